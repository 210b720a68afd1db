"""Oracle restatement of the quadrature layer (reference ``src/quadrature.py``).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__``).
"""

from __future__ import annotations

import math
from functools import lru_cache

import numpy as np
import scipy.linalg

from .bspline import Space1D

FIT_TOL = 1e-12     # src/quadrature.py:40
MAX_RETRIES = 5     # src/quadrature.py:43


class RuleConstructionError(RuntimeError):
    """src/quadrature.py:46-47."""


@lru_cache(maxsize=None)
def gauss(n: int):
    """n-point Gauss-Legendre on [-1, 1] (src/quadrature.py:63-71)."""
    if n < 1:
        raise ValueError("point count must be positive")
    x, w = np.polynomial.legendre.leggauss(n)
    return x, w


def gauss_mapped(n: int, a, b):
    """mid + half*x, half*w (src/quadrature.py:57-60)."""
    x, w = gauss(n)
    mid, half = 0.5 * (a + b), 0.5 * (b - a)
    return mid + half * x, half * w


class Layout:
    """Sorted points grouped by element, strictly interior (src/quadrature.py:74-121)."""

    def __init__(self, bp, groups):
        self.bp = np.asarray(bp, dtype=float)
        counts = np.array([len(g) for g in groups], dtype=np.int64)
        self.offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        self.points = np.concatenate(groups) if self.offsets[-1] else np.empty(0)
        self.elem_of_point = np.repeat(np.arange(counts.size), counts)
        for e, g in enumerate(groups):
            if len(g) and not (np.all(g > self.bp[e]) and np.all(g < self.bp[e + 1])):
                raise ValueError(f"points of element {e} not strictly interior")

    @property
    def npts(self) -> int:
        return int(self.offsets[-1])

    def counts(self) -> np.ndarray:
        return np.diff(self.offsets)

    def element_points(self, e):
        return self.points[self.offsets[e]: self.offsets[e + 1]]

    def range_for(self, e0, e1):
        return int(self.offsets[e0]), int(self.offsets[e1 + 1])


def interior_points(a, b, count):
    """a + (b-a)*k/(count+1), k=1..count (src/quadrature.py:124-127)."""
    k = np.arange(1, count + 1)
    return a + (b - a) * k / (count + 1)


def required_counts(sp_: Space1D) -> np.ndarray:
    """Per-element max over tests of ceil(#trials/#support elements)
    (src/quadrature.py:130-143)."""
    req = np.zeros(sp_.nel, dtype=np.int64)
    trials = sp_.ov_hi - sp_.ov_lo + 1
    els = sp_.el_last - sp_.el_first + 1
    need = -(-trials // els)  # ceil for positive ints
    for i in range(sp_.n):
        a, b = sp_.el_first[i], sp_.el_last[i]
        np.maximum(req[a: b + 1], need[i], out=req[a: b + 1])
    return req


def layout_from_counts(sp_: Space1D, counts) -> Layout:
    """src/quadrature.py:146-152."""
    bp = sp_.bp
    return Layout(bp, [interior_points(bp[e], bp[e + 1], int(counts[e])) for e in range(sp_.nel)])


def place_wq_points(sp_: Space1D) -> Layout:
    """src/quadrature.py:155-157."""
    return layout_from_counts(sp_, required_counts(sp_))


def mass_1d(sp_: Space1D) -> np.ndarray:
    """Exact dense 1-D mass matrix by (p+1)-point Gauss per element
    (src/quadrature.py:160-188)."""
    x0, w0 = gauss(sp_.p + 1)
    bp = sp_.bp
    nel, g = sp_.nel, x0.size
    mid = 0.5 * (bp[:-1] + bp[1:])
    half = 0.5 * np.diff(bp)
    x = (mid[:, None] + half[:, None] * x0[None, :]).ravel()
    w = (half[:, None] * w0[None, :]).ravel()
    f, v = sp_.eval_nonzero(x)
    v = v.reshape(nel, g, -1)
    blocks = np.einsum("egk,egl,eg->ekl", v, v, w.reshape(nel, g))
    M = np.zeros((sp_.n, sp_.n))
    i0 = f.reshape(nel, g)[:, 0]
    q = sp_.p + 1
    r = np.broadcast_to(i0[:, None, None] + np.arange(q)[None, :, None], (nel, q, q))
    c = np.broadcast_to(i0[:, None, None] + np.arange(q)[None, None, :], (nel, q, q))
    np.add.at(M, (r.ravel(), c.ravel()), blocks.ravel())
    return M


def qr_basic(A: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Basic LS solution by column-pivoted QR (LAPACK dgeqp3) with the
    rank rule |R_kk| > max(t,m)*eps*|R_00| (src/quadrature.py:263-278)."""
    Q, R, piv = scipy.linalg.qr(A, mode="economic", pivoting=True)
    d = np.abs(np.diag(R))
    thr = max(A.shape) * np.finfo(float).eps * (d[0] if d.size else 0.0)
    r = int(np.sum(d > thr))
    w = np.zeros(A.shape[1])
    if r:
        w[piv[:r]] = scipy.linalg.solve_triangular(R[:r, :r], (Q.T @ b)[:r])
    return w


class RuleSet:
    """Per-test weight rows over one layout: rows[i] = (k0, w) or None
    (src/quadrature.py:201-260)."""

    def __init__(self, sp_, layout, rows, u_disc=None, S=None, refined=None, base_layout=None):
        self.space = sp_
        self.layout = layout
        self.rows = rows
        self.u_disc = u_disc
        self.S = S
        self.refined = refined
        self.base_layout = base_layout

    def row(self, i):
        return self.rows[i]

    def row_full(self, i):
        k0, w = self.rows[i]
        out = np.zeros(self.layout.npts)
        out[k0: k0 + w.size] = w
        return out

    def packed(self):
        """(k0[int64], wptr[int64], w[float64]) with -1 for missing rows."""
        k0 = np.full(len(self.rows), -1, dtype=np.int64)
        lens = np.zeros(len(self.rows), dtype=np.int64)
        chunks = []
        for i, r in enumerate(self.rows):
            if r is None:
                continue
            k0[i] = r[0]
            lens[i] = r[1].size
            chunks.append(r[1])
        wptr = np.concatenate([[0], np.cumsum(lens)])
        w = np.concatenate(chunks) if chunks else np.empty(0)
        return k0, wptr, w


def solve_rows(sp_: Space1D, layout: Layout, which=None):
    """Moment fit of each test row on a fixed layout (src/quadrature.py:281-303)."""
    M = mass_1d(sp_)
    f, V = sp_.eval_nonzero(layout.points)
    rows = [None] * sp_.n
    failing = []
    for i in (range(sp_.n) if which is None else which):
        k0, k1 = layout.range_for(sp_.el_first[i], sp_.el_last[i])
        j0, j1 = int(sp_.ov_lo[i]), int(sp_.ov_hi[i])
        A = np.zeros((j1 - j0 + 1, k1 - k0))
        for r in range(sp_.p + 1):
            jj = f[k0:k1] + r - j0
            ok = (jj >= 0) & (jj <= j1 - j0)
            A[jj[ok], np.nonzero(ok)[0]] = V[k0:k1][ok, r]
        b = M[i, j0: j1 + 1]
        w = qr_basic(A, b)
        if np.max(np.abs(A @ w - b)) > FIT_TOL * max(np.max(np.abs(b)), 1e-300):
            failing.append(i)
        rows[i] = (k0, w)
    return rows, failing


def least_covered(sp_: Space1D, layout: Layout, i: int) -> int:
    """src/quadrature.py:306-309 (first minimum)."""
    a, b = sp_.el_first[i], sp_.el_last[i]
    return int(a + np.argmin(layout.counts()[a: b + 1]))


def compute_wq_rules(sp_: Space1D, layout: Layout | None = None) -> RuleSet:
    """Standard WQ rules with enrichment retries (src/quadrature.py:312-337)."""
    layout = layout if layout is not None else place_wq_points(sp_)
    counts = layout.counts().copy()
    for attempt in range(MAX_RETRIES + 1):
        rows, failing = solve_rows(sp_, layout)
        if not failing:
            return RuleSet(sp_, layout, rows)
        if attempt == MAX_RETRIES:
            break
        for i in failing:
            counts[least_covered(sp_, layout, i)] += 1
        layout = layout_from_counts(sp_, counts)
    raise RuleConstructionError(f"moment fit failed for rows {failing}")


def split_largest_gap(pts, a, b):
    """Midpoint of the first largest gap of [a, *pts, b] (src/quadrature.py:340-345)."""
    fence = [a, *pts, b]
    g = int(np.argmax(np.diff(fence)))
    return 0.5 * (fence[g] + fence[g + 1])


def augment_nested(layout: Layout, extra) -> Layout:
    """src/quadrature.py:348-363."""
    groups = []
    for e in range(layout.bp.size - 1):
        pts = sorted(layout.element_points(e).tolist())
        for _ in range(int(extra[e])):
            pts.append(split_largest_gap(pts, layout.bp[e], layout.bp[e + 1]))
            pts.sort()
        groups.append(np.asarray(pts))
    return Layout(layout.bp, groups)


def refine_to_c_minus_1(sp_: Space1D, u: float):
    """Insert u until multiplicity p+1 -> (refined space, composite S csr)."""
    missing = sp_.p + 1 - sp_.multiplicity_of(u)
    cur = sp_
    S = scipy.sparse.identity(sp_.n, format="csr")
    for _ in range(missing):
        cur, step = cur.insert(u)
        S = step @ S
    return cur, S.tocsr()


def dwq_layout(sp_: Space1D, layout: Layout, u: float):
    """Integer/point part of src/quadrature.py:382-407: refined space, S and
    the nested augmented layout (before any fit retries)."""
    refined, S = refine_to_c_minus_1(sp_, u)
    need = required_counts(refined)
    extra = np.maximum(need - layout.counts(), 0)
    aug = augment_nested(layout, extra) if np.any(extra) else layout
    for i in range(refined.n):
        e0, e1 = refined.el_first[i], refined.el_last[i]
        t = refined.ov_hi[i] - refined.ov_lo[i] + 1
        while aug.offsets[e1 + 1] - aug.offsets[e0] < t:
            bump = np.zeros(aug.bp.size - 1, dtype=np.int64)
            bump[least_covered(refined, aug, i)] = 1
            aug = augment_nested(aug, bump)
    return refined, S, aug


def build_dwq(sp_: Space1D, layout: Layout, u_disc: float, only_rows=None) -> RuleSet:
    """Discontinuous WQ in four steps (src/quadrature.py:366-449)."""
    bp = sp_.bp
    if not np.any(np.abs(bp - u_disc) <= 1e-12):
        raise ValueError(f"{u_disc} is not a breakpoint")
    u = float(bp[np.argmin(np.abs(bp - u_disc))])
    refined, S, aug = dwq_layout(sp_, layout, u)
    Sc = S.tocsc()
    wanted = list(range(sp_.n)) if only_rows is None else sorted(set(only_rows))
    fine_needed = None
    if only_rows is not None:
        seen = set()
        for j in wanted:
            seen.update(int(i) for i in Sc.indices[Sc.indptr[j]: Sc.indptr[j + 1]])
        fine_needed = sorted(seen)
    for attempt in range(MAX_RETRIES + 1):
        fine_rows, failing = solve_rows(refined, aug, which=fine_needed)
        if not failing:
            break
        if attempt == MAX_RETRIES:
            raise RuleConstructionError(f"dwq fit failed for {failing} at {u}")
        bump = np.zeros(aug.bp.size - 1, dtype=np.int64)
        for i in failing:
            bump[least_covered(refined, aug, i)] += 1
        aug = augment_nested(aug, bump)
    rows = [None] * sp_.n
    for j in wanted:
        k0, k1 = aug.range_for(sp_.el_first[j], sp_.el_last[j])
        w = np.zeros(k1 - k0)
        for i, s in zip(Sc.indices[Sc.indptr[j]: Sc.indptr[j + 1]], Sc.data[Sc.indptr[j]: Sc.indptr[j + 1]]):
            fk0, fw = fine_rows[i]
            w[fk0 - k0: fk0 - k0 + fw.size] += s * fw
        rows[j] = (k0, w)
    return RuleSet(sp_, aug, rows, u_disc=u, S=S, refined=refined, base_layout=layout)
