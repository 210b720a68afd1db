"""Oracle restatement of the L2-projection layer (reference ``src/projection.py``).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__``).
"""

from __future__ import annotations

import math

import numpy as np
import scipy.linalg
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import quad as Q
from .assemble import Coeff
from .trim import TrimConfig

CONDITION_GUARD = 1e12   # src/projection.py:41
DIRECT_LIMIT = 6000      # src/projection.py:44
ELEM_CHUNK = 8192


def default_target(P):
    """sin(2 u1) cos(3 u2) (src/projection.py:51-54)."""
    P = np.atleast_2d(P)
    return np.sin(2.0 * P[:, 0]) * np.cos(3.0 * P[:, 1])


def tensor_tables(space, n_extra):
    """Per-element (p+n_extra)-point Gauss: points, weights, values, first
    (src/projection.py:83-98)."""
    gx, gw = Q.gauss(space.p + n_extra)
    bp = space.bp
    mid, half = 0.5 * (bp[:-1] + bp[1:]), 0.5 * np.diff(bp)
    X = mid[:, None] + half[:, None] * gx[None, :]
    W = half[:, None] * gw[None, :]
    f, V = space.eval_nonzero(X.ravel())
    V = V.reshape(space.nel, gx.size, space.p + 1)
    return X, W, V, f.reshape(space.nel, gx.size)[:, 0]


def _interior_elements(cfg):
    e1, e2 = np.nonzero(cfg.element_class == 0)
    return e1, e2


def assemble_rhs(target, cfg: TrimConfig, coeff: Coeff | None = None, elements=None):
    """b_i = int_valid f B_i c: (p+2)^2 Gauss on interior elements plus the
    cut-cell rule (src/projection.py:101-145)."""
    coeff = coeff or Coeff()
    s1, s2 = cfg.s1, cfg.s2
    X1, W1, V1, F1 = tensor_tables(s1, 2)
    X2, W2, V2, F2 = tensor_tables(s2, 2)
    act = cfg.active()
    col_of = np.full((s1.n, s2.n), -1, np.int64)
    col_of[act[:, 0], act[:, 1]] = np.arange(act.shape[0])
    b = np.zeros(act.shape[0])
    E1, E2 = _interior_elements(cfg) if elements is None else elements
    g1, g2 = X1.shape[1], X2.shape[1]
    q1, q2 = s1.p + 1, s2.p + 1
    for c0 in range(0, E1.size, ELEM_CHUNK):
        e1, e2 = E1[c0: c0 + ELEM_CHUNK], E2[c0: c0 + ELEM_CHUNK]
        P = np.stack([np.broadcast_to(X1[e1][:, :, None], (e1.size, g1, g2)),
                      np.broadcast_to(X2[e2][:, None, :], (e1.size, g1, g2))], axis=-1).reshape(-1, 2)
        cw = (target(P) * coeff.at(P)).reshape(e1.size, g1, g2) * W1[e1][:, :, None] * W2[e2][:, None, :]
        loc = np.einsum("eab,eak,ebl->ekl", cw, V1[e1], V2[e2])
        comp = col_of[F1[e1][:, None, None] + np.arange(q1)[None, :, None],
                      F2[e2][:, None, None] + np.arange(q2)[None, None, :]]
        ok = comp >= 0
        np.add.at(b, comp[ok], loc[ok])
    rule = cfg.cut_cell_rule(max(s1.p, s2.p))
    for (e1, e2), (P, W) in rule.rules.items():
        if P.shape[0] == 0:
            continue
        f1, Va = s1.eval_nonzero(P[:, 0])
        f2, Vb = s2.eval_nonzero(P[:, 1])
        cw = target(P) * coeff.at(P) * W
        keys = f1 * (s2.n + 1) + f2
        for key in np.unique(keys):
            sel = keys == key
            loc = np.einsum("k,ka,kb->ab", cw[sel], Va[sel], Vb[sel])
            a1, a2 = int(f1[sel][0]), int(f2[sel][0])
            comp = col_of[a1: a1 + q1, a2: a2 + q2].ravel()
            ok = comp >= 0
            np.add.at(b, comp[ok], loc.ravel()[ok])
    return b


def l2_error_parts(coeffs, target, cfg: TrimConfig, active=None):
    """(num, den) of the relative L2 error with (p+3)^2 Gauss on interior
    elements and the cut-cell rule (src/projection.py:221-260)."""
    s1, s2 = cfg.s1, cfg.s2
    act = cfg.active() if active is None else active
    C = np.zeros((s1.n, s2.n))
    C[act[:, 0], act[:, 1]] = coeffs
    X1, W1, V1, F1 = tensor_tables(s1, 3)
    X2, W2, V2, F2 = tensor_tables(s2, 3)
    q1, q2 = s1.p + 1, s2.p + 1
    E1, E2 = _interior_elements(cfg)
    g1, g2 = X1.shape[1], X2.shape[1]
    num = den = 0.0
    for c0 in range(0, E1.size, ELEM_CHUNK):
        e1, e2 = E1[c0: c0 + ELEM_CHUNK], E2[c0: c0 + ELEM_CHUNK]
        Ce = C[F1[e1][:, None, None] + np.arange(q1)[None, :, None],
               F2[e2][:, None, None] + np.arange(q2)[None, None, :]]
        uh = np.einsum("eak,ekl,ebl->eab", V1[e1], Ce, V2[e2])
        P = np.stack([np.broadcast_to(X1[e1][:, :, None], (e1.size, g1, g2)),
                      np.broadcast_to(X2[e2][:, None, :], (e1.size, g1, g2))], axis=-1).reshape(-1, 2)
        f = target(P).reshape(e1.size, g1, g2)
        w = W1[e1][:, :, None] * W2[e2][:, None, :]
        num += float(np.sum(w * (uh - f) ** 2))
        den += float(np.sum(w * f ** 2))
    rule = cfg.cut_cell_rule(max(s1.p, s2.p))
    for (e1, e2), (P, W) in rule.rules.items():
        if P.shape[0] == 0:
            continue
        f1, Va = s1.eval_nonzero(P[:, 0])
        f2, Vb = s2.eval_nonzero(P[:, 1])
        i1 = f1[:, None] + np.arange(q1)[None, :]
        i2 = f2[:, None] + np.arange(q2)[None, :]
        uh = np.einsum("ka,kb,kab->k", Va, Vb, C[i1[:, :, None], i2[:, None, :]])
        f = target(P)
        num += float(np.sum(W * (uh - f) ** 2))
        den += float(np.sum(W * f ** 2))
    return num, den


def l2_error(coeffs, target, cfg, active=None):
    num, den = l2_error_parts(coeffs, target, cfg, active)
    if den <= 0.0:
        raise ValueError("target function has zero norm on the valid region")
    return math.sqrt(num / den)


def solve_spd(A, b):
    """Jacobi-scaled Cholesky (n<=6000) or CG to 1e-13 (src/projection.py:148-211)."""
    A = sp.csr_matrix(A)
    b = np.asarray(b, float)
    n = A.shape[0]
    d = A.diagonal()
    if np.any(d <= 0.0):
        raise ValueError("matrix is not positive definite (non-positive diagonal)")
    s = 1.0 / np.sqrt(d)
    As = sp.diags(s) @ A @ sp.diags(s)
    bs = s * b
    if n <= DIRECT_LIMIT:
        D = As.toarray()
        cho = scipy.linalg.cho_factor(0.5 * (D + D.T), lower=True, check_finite=False)
        solve = lambda r: scipy.linalg.cho_solve(cho, r, check_finite=False)
    else:
        def solve(r):
            x, info = spla.cg(As, r, rtol=1e-14, atol=0.0, maxiter=10 * n)
            if info > 0:
                x = x + spla.cg(As, r - As @ x, rtol=1e-10, atol=0.0, maxiter=n)[0]
            return x
    y = solve(bs)
    bn = np.linalg.norm(bs) or 1.0
    for _ in range(4):
        r = bs - As @ y
        if np.linalg.norm(r) <= 1e-14 * bn:
            break
        y = y + solve(r)
    return s * y
