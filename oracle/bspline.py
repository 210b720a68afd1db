"""Oracle restatement of the univariate B-spline layer (reference ``src/splines.py``).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__``).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

KNOT_TOL = 1e-12  # src/splines.py:29


def merge_breakpoints(knots: np.ndarray, tol: float = KNOT_TOL):
    """Unique knot values with multiplicities; a value joins the running
    unique value when within ``tol`` of it (src/splines.py:156-166)."""
    uniq = [float(knots[0])]
    mult = [1]
    for v in knots[1:]:
        if v - uniq[-1] <= tol:
            mult[-1] += 1
        else:
            uniq.append(float(v))
            mult.append(1)
    return np.asarray(uniq), np.asarray(mult, dtype=np.int64)


class Space1D:
    """Open knot vector + degree + support bookkeeping.

    Restates ``KnotVector`` (src/splines.py:32-153) and the index bookkeeping
    of ``Basis1D`` (src/splines.py:169-232) in one object.
    """

    def __init__(self, knots, p: int):
        knots = np.ascontiguousarray(knots, dtype=float)
        p = int(p)
        if p < 0:
            raise ValueError("negative degree")
        if knots.ndim != 1 or knots.size < 2 * (p + 1):
            raise ValueError("knot vector too short for the requested degree")
        if np.any(np.diff(knots) < 0):
            raise ValueError("knots must be non-decreasing")
        bp, mult = merge_breakpoints(knots)
        if mult[0] != p + 1 or mult[-1] != p + 1:
            raise ValueError("open knot vector required")
        if mult.size > 2 and np.any(mult[1:-1] > p + 1):
            raise ValueError("interior knot multiplicity too high")
        self.knots = knots
        self.p = p
        self.bp = bp
        self.mult = mult
        self.n = knots.size - p - 1
        self.nel = bp.size - 1
        # knot-span index of each element (src/splines.py:69)
        self.espan = np.cumsum(mult)[:-1] - 1
        # support element range of each function: elements whose span lies in
        # [i, i+p] (src/splines.py:178-190); spans are strictly increasing.
        i = np.arange(self.n)
        self.el_first = np.searchsorted(self.espan, i, side="left")
        self.el_last = np.searchsorted(self.espan, i + p, side="right") - 1
        # trial window: first function on the first support element to the
        # last function on the last one (src/splines.py:222-232)
        self.ov_lo = self.espan[self.el_first] - p
        self.ov_hi = self.espan[self.el_last]

    # -- queries -------------------------------------------------------------
    @property
    def domain(self):
        return float(self.knots[0]), float(self.knots[-1])

    def spans(self, u) -> np.ndarray:
        """src/splines.py:114-122: searchsorted(side=right)-1, clipped."""
        u = np.asarray(u, dtype=float)
        lo, hi = self.domain
        if np.any(u < lo) or np.any(u > hi):
            raise ValueError("coordinate outside the knot domain")
        s = np.searchsorted(self.knots, u, side="right") - 1
        return np.clip(s, self.p, self.n - 1)

    def element_of(self, u) -> np.ndarray:
        """src/splines.py:124-127."""
        e = np.searchsorted(self.bp, np.asarray(u, dtype=float), side="right") - 1
        return np.clip(e, 0, self.nel - 1)

    def fns_on_element(self, e: int):
        s = int(self.espan[e])
        return s - self.p, s

    def support_interval(self, i: int):
        return float(self.knots[i]), float(self.knots[i + self.p + 1])

    def multiplicity_of(self, u: float) -> int:
        return int(np.sum(np.abs(self.knots - u) <= KNOT_TOL))

    def n_trials(self) -> np.ndarray:
        return self.ov_hi - self.ov_lo + 1

    # -- evaluation ----------------------------------------------------------
    def eval_nonzero(self, u):
        """Cox-de Boor triangle (NURBS book A2.2) at many points.

        Restates src/splines.py:245-269; returns (first index, (N, p+1) values).
        """
        u = np.asarray(u, dtype=float).reshape(-1)
        sp_ = self.spans(u)
        p, kn = self.p, self.knots
        N = np.ones((u.size, p + 1))
        lft = np.empty((u.size, max(p, 1)))
        rgt = np.empty((u.size, max(p, 1)))
        for j in range(1, p + 1):
            lft[:, j - 1] = u - kn[sp_ + 1 - j]
            rgt[:, j - 1] = kn[sp_ + j] - u
            carry = np.zeros(u.size)
            for r in range(j):
                q = N[:, r] / (rgt[:, r] + lft[:, j - r - 1])
                N[:, r] = carry + rgt[:, r] * q
                carry = lft[:, j - r - 1] * q
            N[:, j] = carry
        return sp_ - p, N

    def eval_nonzero_ders(self, u):
        """Values and first derivatives of the p+1 non-zero functions.

        Not in the reference; derivative from the degree p-1
        values on the same span: B'_{i,p} = p/(t_{i+p}-t_i) B_{i,p-1}
        - p/(t_{i+p+1}-t_{i+1}) B_{i+1,p-1}.
        """
        u = np.asarray(u, dtype=float).reshape(-1)
        first, N = self.eval_nonzero(u)
        p, kn = self.p, self.knots
        D = np.zeros_like(N)
        if p == 0:
            return first, N, D
        sp_ = first + p
        # degree p-1 values of functions sp-p+1 .. sp on the span
        Nl = np.ones((u.size, p))
        lft = np.empty((u.size, p))
        rgt = np.empty((u.size, p))
        for j in range(1, p):
            lft[:, j - 1] = u - kn[sp_ + 1 - j]
            rgt[:, j - 1] = kn[sp_ + j] - u
            carry = np.zeros(u.size)
            for r in range(j):
                q = Nl[:, r] / (rgt[:, r] + lft[:, j - r - 1])
                Nl[:, r] = carry + rgt[:, r] * q
                carry = lft[:, j - r - 1] * q
            Nl[:, j] = carry
        # Nl[:, k] = B_{sp-p+1+k, p-1}
        for k in range(p + 1):
            i = sp_ - p + k
            acc = np.zeros(u.size)
            if k >= 1:  # term with B_{i,p-1} = Nl[:, k-1]
                den = kn[i + p] - kn[i]
                acc += np.where(den > 0, p / np.where(den > 0, den, 1.0), 0.0) * Nl[:, k - 1]
            if k <= p - 1:  # term with B_{i+1,p-1} = Nl[:, k]
                den = kn[i + p + 1] - kn[i + 1]
                acc -= np.where(den > 0, p / np.where(den > 0, den, 1.0), 0.0) * Nl[:, k]
            D[:, k] = acc
        return first, N, D

    def colloc_block(self, pts, j0: int, j1: int) -> np.ndarray:
        """Dense slice C[k, j-j0] = B_j(pts[k]) for j in [j0, j1]
        (the needed window of src/splines.py:282-290)."""
        first, vals = self.eval_nonzero(pts)
        C = np.zeros((np.size(pts), j1 - j0 + 1))
        for r in range(self.p + 1):
            col = first + r - j0
            ok = (col >= 0) & (col <= j1 - j0)
            C[np.nonzero(ok)[0], col[ok]] = vals[ok, r]
        return C

    def collocation(self, pts) -> np.ndarray:
        return self.colloc_block(pts, 0, self.n - 1)

    # -- refinement ----------------------------------------------------------
    def insert(self, ubar: float):
        """Single knot insertion -> (refined space, S (n+1)x n sparse).

        Restates src/splines.py:369-403 (alpha coefficients, PAPER Eq. 9).
        """
        p, n, kn = self.p, self.n, self.knots
        lo, hi = self.domain
        if not (lo <= ubar <= hi):
            raise ValueError("insertion point outside the domain")
        if self.multiplicity_of(ubar) >= p + 1:
            raise ValueError("multiplicity would exceed p+1")
        span = int(self.spans(np.asarray([ubar]))[0])
        alpha = np.zeros(n + 1)
        alpha[: span - p + 1] = 1.0
        for k in range(max(span - p + 1, 0), span + 1):
            alpha[k] = (ubar - kn[k]) / (kn[k + p] - kn[k])
        rows = np.concatenate([np.arange(n), np.arange(1, n + 1)])
        cols = np.concatenate([np.arange(n), np.arange(n)])
        vals = np.concatenate([alpha[:n], 1.0 - alpha[1:]])
        S = sp.coo_matrix((vals, (rows, cols)), shape=(n + 1, n)).tocsr()
        S.eliminate_zeros()
        at = int(np.searchsorted(kn, ubar, side="right"))
        return Space1D(np.insert(kn, at, ubar), p), S


def uniform_knots(nel: int, p: int, a: float = 0.0, b: float = 1.0) -> np.ndarray:
    """src/splines.py:445-451."""
    if nel < 1:
        raise ValueError("need at least one element")
    inner = np.linspace(a, b, nel + 1)[1:-1]
    return np.concatenate([np.full(p + 1, a), inner, np.full(p + 1, b)])


def uniform_space(nel: int, p: int) -> Space1D:
    return Space1D(uniform_knots(nel, p), p)
