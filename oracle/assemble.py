"""Oracle restatement of mass-matrix formation (reference ``src/assembly.py``).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__``).

Contributions are collected as COO triplets and summed into a raw matrix,
then symmetrized exactly like ``_Run.finish`` (src/assembly.py:400-404):
``0.5*(M + M.T)`` with scipy CSR addition (which drops exact zeros) and
``sort_indices`` -- the final pattern is therefore the reference's.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import quad as Q
from .trim import CUT, EXTERIOR, INTERIOR, TrimConfig

STRATEGIES = ("reference", "wq", "hybrid", "dwq")   # src/assembly.py:51
ROW_CHUNK = 20000


class Coeff:
    """CoefficientField (src/assembly.py:54-85): None means c == 1."""

    def __init__(self, fn=None):
        self.fn = fn

    @property
    def identity(self):
        return self.fn is None

    def at(self, P):
        P = np.atleast_2d(P)
        if self.fn is None:
            return np.ones(P.shape[0])
        return np.asarray(self.fn(P), float).reshape(P.shape[0])

    def grid(self, x1, x2):
        if self.fn is None:
            return np.ones((x1.size, x2.size))
        P = np.column_stack([np.repeat(x1, x2.size), np.tile(x2, x1.size)])
        return self.at(P).reshape(x1.size, x2.size)


@dataclass
class Report:
    """FormationReport (src/assembly.py:123-138)."""
    strategy: str
    t_weights: float = 0.0
    t_interior: float = 0.0
    t_cut_regular: float = 0.0
    t_cut_elements: float = 0.0
    t_total: float = 0.0
    n_wq_points: int = 0
    n_gauss_elements: int = 0
    n_cutcell_points: int = 0


@dataclass
class Mass:
    data: sp.csr_matrix
    active: np.ndarray


def pattern(cfg: TrimConfig):
    """Support-overlap CSR of the active functions (src/assembly.py:145-171).
    Returns (active, col_of, indptr int64, indices int64)."""
    s1, s2 = cfg.s1, cfg.s2
    act = cfg.active()
    col_of = np.full((s1.n, s2.n), -1, dtype=np.int64)
    col_of[act[:, 0], act[:, 1]] = np.arange(act.shape[0])
    cols = []
    for i1, i2 in act:
        c = col_of[s1.ov_lo[i1]: s1.ov_hi[i1] + 1, s2.ov_lo[i2]: s2.ov_hi[i2] + 1].ravel()
        cols.append(c[c >= 0])   # row-major window order is already ascending
    lens = np.array([c.size for c in cols], dtype=np.int64)
    indptr = np.concatenate([[0], np.cumsum(lens)])
    indices = np.concatenate(cols) if cols else np.empty(0, np.int64)
    return act, col_of, indptr, indices


class _Gauss1D:
    """(p+1)-point element Gauss tables per direction (src/assembly.py:198-211)."""

    def __init__(self, space, npts):
        gx, gw = Q.gauss(npts)
        bp = space.bp
        mid, half = 0.5 * (bp[:-1] + bp[1:]), 0.5 * np.diff(bp)
        self.x = mid[:, None] + half[:, None] * gx[None, :]
        self.w = half[:, None] * gw[None, :]
        f, v = space.eval_nonzero(self.x.ravel())
        self.v = v.reshape(space.nel, npts, space.p + 1)
        self.first = f.reshape(space.nel, npts)[:, 0]


class _Run:
    def __init__(self, cfg: TrimConfig, coeff: Coeff):
        self.cfg = cfg
        self.coeff = coeff
        self.s1, self.s2 = cfg.s1, cfg.s2
        self.act, self.col_of, _, _ = pattern(cfg)
        self.K = self.act.shape[0]
        self.g1 = _Gauss1D(self.s1, self.s1.p + 1)
        self.g2 = _Gauss1D(self.s2, self.s2.p + 1)
        self.R, self.C, self.V = [], [], []
        self._blk = {}
        self.report = Report("")

    def add(self, r, c, v):
        self.R.append(np.asarray(r, np.int64).ravel())
        self.C.append(np.asarray(c, np.int64).ravel())
        self.V.append(np.asarray(v, float).ravel())

    def element_block(self, e1, e2):
        """Gauss block B2d^T diag(cw) B2d of a full element (src/assembly.py:310-332)."""
        key = (e1, e2)
        if key in self._blk:
            return self._blk[key]
        g1, g2 = self.g1, self.g2
        V1, V2 = g1.v[e1], g2.v[e2]
        cw = np.outer(g1.w[e1], g2.w[e2])
        if not self.coeff.identity:
            P = np.column_stack([np.repeat(g1.x[e1], g2.x[e2].size), np.tile(g2.x[e2], g1.x[e1].size)])
            cw = self.coeff.at(P).reshape(V1.shape[0], V2.shape[0]) * cw
        B = (V1[:, None, :, None] * V2[None, :, None, :]).reshape(V1.shape[0] * V2.shape[0], -1)
        blk = B.T @ (cw.reshape(-1)[:, None] * B)
        self._blk[key] = blk
        self.report.n_gauss_elements += 1
        return blk

    def elem_fns(self, e1, e2):
        a1 = self.s1.espan[e1] - self.s1.p
        a2 = self.s2.espan[e2] - self.s2.p
        f1 = np.arange(a1, a1 + self.s1.p + 1)
        f2 = np.arange(a2, a2 + self.s2.p + 1)
        return self.col_of[f1[:, None], f2[None, :]].ravel()

    def scatter_element(self, e1, e2, blk, rows_keep):
        """src/assembly.py:334-356: rows filtered, columns = active functions."""
        comp = self.elem_fns(e1, e2)
        ok = comp >= 0
        ri = np.nonzero(rows_keep)[0]
        ci = np.nonzero(ok)[0]
        if ri.size == 0:
            return
        self.add(np.repeat(comp[ri], ci.size), np.tile(comp[ci], ri.size), blk[np.ix_(ri, ci)])

    def scatter_row_block(self, i1, i2, j1lo, j2lo, blk):
        """src/assembly.py:358-365."""
        row = self.col_of[i1, i2]
        comp = self.col_of[j1lo: j1lo + blk.shape[0], j2lo: j2lo + blk.shape[1]].ravel()
        ok = comp >= 0
        self.add(np.full(int(ok.sum()), row), comp[ok], blk.ravel()[ok])

    def flush(self):
        """Sum the accumulated contributions into the CSR -- the analogue of
        the reference's ``flush`` scatter (src/assembly.py:299-306), which
        ``assemble_mass`` runs INSIDE its clock (:525-546)."""
        if self.R:
            r, c, v = np.concatenate(self.R), np.concatenate(self.C), np.concatenate(self.V)
        else:
            r = c = np.empty(0, np.int64)
            v = np.empty(0)
        self.R, self.C, self.V = [], [], []
        M = sp.csr_matrix((v, (r, c)), shape=(self.K, self.K))
        self._M = M if getattr(self, "_M", None) is None else self._M + M

    def finish(self):
        """0.5*(M+M^T), zero-drop, sorted (src/assembly.py:400-404)."""
        self.flush()
        M = self._M
        self._M = None
        M = 0.5 * (M + M.T)
        M.sort_indices()
        return Mass(M.tocsr(), self.act)


def sum_factor_row(i1, i2, r1: Q.RuleSet, r2: Q.RuleSet, grid, mask=None, point_box=None):
    """One row by two nested 1-D contractions (src/assembly.py:218-252).
    Collocation slices are evaluated directly on the rule layouts."""
    s1, s2 = r1.space, r2.space
    k1, w1 = r1.row(i1)
    k2, w2 = r2.row(i2)
    a1, b1_ = k1, k1 + w1.size
    a2, b2_ = k2, k2 + w2.size
    if point_box is not None:
        a1, b1_ = max(a1, point_box[0]), min(b1_, point_box[1])
        a2, b2_ = max(a2, point_box[2]), min(b2_, point_box[3])
    j1lo, j1hi = int(s1.ov_lo[i1]), int(s1.ov_hi[i1])
    j2lo, j2hi = int(s2.ov_lo[i2]), int(s2.ov_hi[i2])
    if a1 >= b1_ or a2 >= b2_:
        return j1lo, j2lo, np.zeros((j1hi - j1lo + 1, j2hi - j2lo + 1))
    B1 = s1.colloc_block(r1.layout.points[a1:b1_], j1lo, j1hi) * w1[a1 - k1: b1_ - k1, None]
    B2 = s2.colloc_block(r2.layout.points[a2:b2_], j2lo, j2hi) * w2[a2 - k2: b2_ - k2, None]
    G = grid[a1:b1_, a2:b2_]
    if mask is not None:
        G = G * mask
    inner = B2.T @ G.T
    return j1lo, j2lo, B1.T @ inner.T


def sum_factor_op_count(i1, i2, r1, r2):
    """src/assembly.py:255-265."""
    n1, n2 = r1.row(i1)[1].size, r2.row(i2)[1].size
    t1 = r1.space.ov_hi[i1] - r1.space.ov_lo[i1] + 1
    t2 = r2.space.ov_hi[i2] - r2.space.ov_lo[i2] + 1
    return int(t2 * n1 * n2 + t1 * t2 * n1)


def interior_rows(run: _Run, rows, r1: Q.RuleSet, r2: Q.RuleSet, C1, C2, grid):
    """Batched sum factorization grouped by shape (src/assembly.py:409-449)."""
    s1, s2 = run.s1, run.s2
    if len(rows) == 0:
        return
    k1s, w1l = zip(*[r1.row(int(i)) for i in rows[:, 0]])
    k2s, w2l = zip(*[r2.row(int(i)) for i in rows[:, 1]])
    n1 = np.array([w.size for w in w1l])
    n2 = np.array([w.size for w in w2l])
    t1 = s1.ov_hi[rows[:, 0]] - s1.ov_lo[rows[:, 0]] + 1
    t2 = s2.ov_hi[rows[:, 1]] - s2.ov_lo[rows[:, 1]] + 1
    keys = np.stack([n1, n2, t1, t2], axis=1)
    uk, inv = np.unique(keys, axis=0, return_inverse=True)
    inv = inv.ravel()
    for g, (gn1, gn2, gt1, gt2) in enumerate(uk):
        members = np.nonzero(inv == g)[0]
        for c0 in range(0, members.size, ROW_CHUNK):
            sel = members[c0: c0 + ROW_CHUNK]
            R = sel.size
            i1, i2 = rows[sel, 0], rows[sel, 1]
            K1 = np.array([k1s[s] for s in sel])[:, None] + np.arange(gn1)[None, :]
            K2 = np.array([k2s[s] for s in sel])[:, None] + np.arange(gn2)[None, :]
            J1 = s1.ov_lo[i1][:, None] + np.arange(gt1)[None, :]
            J2 = s2.ov_lo[i2][:, None] + np.arange(gt2)[None, :]
            W1 = np.stack([w1l[s] for s in sel])
            W2 = np.stack([w2l[s] for s in sel])
            B1 = C1[K1[:, :, None], J1[:, None, :]] * W1[:, :, None]
            B2 = C2[K2[:, :, None], J2[:, None, :]] * W2[:, :, None]
            G = grid[K1[:, :, None], K2[:, None, :]]
            inner = np.matmul(B2.transpose(0, 2, 1), G.transpose(0, 2, 1))
            blocks = np.matmul(B1.transpose(0, 2, 1), inner.transpose(0, 2, 1))
            rr = run.col_of[i1, i2]
            comp = run.col_of[J1[:, :, None], J2[:, None, :]].reshape(R, -1)
            ok = comp >= 0
            run.add(np.repeat(rr, gt1 * gt2)[ok.ravel()], comp[ok], blocks.reshape(R, -1)[ok])


def build_rules(run: _Run, need_dwq: bool):
    """Standard rules per direction + DWQ sets per (dir, u_disc) (src/assembly.py:454-489)."""
    r1 = Q.compute_wq_rules(run.s1, Q.place_wq_points(run.s1))
    r2 = Q.compute_wq_rules(run.s2, Q.place_wq_points(run.s2))
    dwq = {}
    if need_dwq:
        needed = {}
        fc = run.cfg.func_class
        for i1, i2 in run.act:
            if fc[i1, i2] != CUT:
                continue
            info = run.cfg.dwq_info(i1, i2)
            if info.eligible and info.box is not None:
                for d, u in enumerate(info.u_disc):
                    if u is not None:
                        needed.setdefault((d, float(u)), set()).add(int((i1, i2)[d]))
        for key in sorted(needed):
            d, u = key
            sp_ = (run.s1, run.s2)[d]
            base = (r1, r2)[d].layout
            dwq[key] = Q.build_dwq(sp_, base, u, only_rows=sorted(needed[key]))
    return r1, r2, dwq


def gauss_rows_by_element(run: _Run, rows):
    """Element Gauss over interior elements, restricted to given rows (src/assembly.py:623-643)."""
    if len(rows) == 0:
        return
    marks = np.zeros(run.K, bool)
    marks[run.col_of[rows[:, 0], rows[:, 1]]] = True
    for (e1, e2) in run.cfg.interior_elements:
        comp = run.elem_fns(e1, e2)
        keep = (comp >= 0) & marks[np.clip(comp, 0, None)]
        if not np.any(keep):
            continue
        run.scatter_element(e1, e2, run.element_block(e1, e2), keep)


def cut_regular_rows(run: _Run, rows, strategy, r1, r2, grid, dwq):
    """src/assembly.py:553-610."""
    if len(rows) == 0:
        return
    cfg = run.cfg
    if strategy == "wq":
        inter = cfg.element_class == INTERIOR
        el1, el2 = r1.layout.elem_of_point, r2.layout.elem_of_point
        for i1, i2 in rows:
            k1, w1 = r1.row(int(i1))
            k2, w2 = r2.row(int(i2))
            mask = inter[el1[k1: k1 + w1.size][:, None], el2[k2: k2 + w2.size][None, :]]
            j1lo, j2lo, blk = sum_factor_row(int(i1), int(i2), r1, r2, grid, mask=mask)
            run.scatter_row_block(int(i1), int(i2), j1lo, j2lo, blk)
        return
    if strategy == "hybrid":
        gauss_rows_by_element(run, rows)
        return
    fallback = []
    grids = {}
    for i1, i2 in rows:
        info = cfg.dwq_info(int(i1), int(i2))
        if not info.eligible or info.box is None:
            fallback.append((int(i1), int(i2)))
            continue
        d1 = dwq.get((0, float(info.u_disc[0]))) if info.u_disc[0] is not None else None
        d2 = dwq.get((1, float(info.u_disc[1]))) if info.u_disc[1] is not None else None
        q1 = d1 if d1 is not None else r1
        q2 = d2 if d2 is not None else r2
        gk = (id(q1.layout), id(q2.layout))
        if gk not in grids:
            grids[gk] = grid if (q1 is r1 and q2 is r2) else run.coeff.grid(q1.layout.points, q2.layout.points)
        (a1, b1), (a2, b2) = info.box
        box = (int(q1.layout.offsets[a1]), int(q1.layout.offsets[b1 + 1]),
               int(q2.layout.offsets[a2]), int(q2.layout.offsets[b2 + 1]))
        j1lo, j2lo, blk = sum_factor_row(int(i1), int(i2), q1, q2, grids[gk], point_box=box)
        run.scatter_row_block(int(i1), int(i2), j1lo, j2lo, blk)
        row = run.col_of[i1, i2]
        for (e1, e2) in info.residual:
            comp = run.elem_fns(e1, e2)
            run.scatter_element(e1, e2, run.element_block(e1, e2), comp == row)
    if fallback:
        gauss_rows_by_element(run, np.asarray(fallback))


def add_cut_blocks(run: _Run, rule):
    """Cut-element blocks grouped by span key (src/assembly.py:369-398)."""
    s1, s2 = run.s1, run.s2
    for (e1, e2), (P, W) in rule.rules.items():
        if P.shape[0] == 0:
            continue
        f1, V1 = s1.eval_nonzero(P[:, 0])
        f2, V2 = s2.eval_nonzero(P[:, 1])
        cw = run.coeff.at(P) * W
        run.report.n_cutcell_points += P.shape[0]
        keys = f1 * (s2.n + 1) + f2
        for key in np.unique(keys):
            sel = keys == key
            a1, a2 = int(f1[sel][0]), int(f2[sel][0])
            B = (V1[sel][:, :, None] * V2[sel][:, None, :]).reshape(int(sel.sum()), -1)
            blk = B.T @ (cw[sel][:, None] * B)
            comp = run.col_of[np.arange(a1, a1 + s1.p + 1)[:, None], np.arange(a2, a2 + s2.p + 1)[None, :]].ravel()
            ok = np.nonzero(comp >= 0)[0]
            run.add(np.repeat(comp[ok], ok.size), np.tile(comp[ok], ok.size), blk[np.ix_(ok, ok)])


def assemble_mass(cfg: TrimConfig, coeff: Coeff | None = None, strategy="reference",
                  report: Report | None = None, rules=None) -> Mass:
    """Strategy dispatch with the four timed phases (src/assembly.py:492-550).

    ``rules``: optional precomputed (r1, r2, dwq) -- the weight-import path
    used to compare GPU rows against the oracle at c != 1.
    """
    if strategy not in STRATEGIES:
        raise ValueError(f"unknown strategy {strategy!r}; choose from {STRATEGIES}")
    coeff = coeff or Coeff()
    run = _Run(cfg, coeff)
    if report is not None:
        run.report = report
    run.report.strategy = strategy
    q = max(cfg.s1.p, cfg.s2.p)
    cut_rule = cfg.cut_cell_rule(q)
    t0 = time.perf_counter()
    if strategy == "reference":
        r1 = r2 = None
        dwq = {}
    else:
        r1, r2, dwq = rules if rules is not None else build_rules(run, strategy == "dwq")
        run.report.n_wq_points = r1.layout.npts + r2.layout.npts
    t1 = time.perf_counter()
    run.report.t_weights = t1 - t0
    fc = cfg.func_class
    is_cut = fc[run.act[:, 0], run.act[:, 1]] == CUT
    if strategy == "reference":
        comp_all = None
        for (e1, e2) in cfg.interior_elements:
            comp_all = run.elem_fns(e1, e2)
            run.scatter_element(e1, e2, run.element_block(e1, e2), comp_all >= 0)
        t2 = t3 = time.perf_counter()
        run.report.t_interior = t2 - t1
    else:
        C1 = run.s1.collocation(r1.layout.points)
        C2 = run.s2.collocation(r2.layout.points)
        grid = coeff.grid(r1.layout.points, r2.layout.points)
        interior_rows(run, run.act[~is_cut], r1, r2, C1, C2, grid)
        t2 = time.perf_counter()
        run.report.t_interior = t2 - t1
        cut_regular_rows(run, run.act[is_cut], strategy, r1, r2, grid, dwq)
        t3 = time.perf_counter()
        run.report.t_cut_regular = t3 - t2
    add_cut_blocks(run, cut_rule)
    run.flush()               # the scatter is timed, as in the reference
    t4 = time.perf_counter()
    run.report.t_cut_elements = t4 - t3
    run.report.t_total = t4 - t0
    return run.finish()


def form_with_timings(strategy, cfg: TrimConfig, coeff=None):
    """src/assembly.py:651-665: cut rule warmed outside the clock."""
    cfg.cut_cell_rule(max(cfg.s1.p, cfg.s2.p))
    rep = Report(strategy)
    M = assemble_mass(cfg, coeff, strategy, report=rep)
    return M, rep
