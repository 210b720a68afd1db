"""Quadrature rules: Gauss, WQ point layouts, GPU moment fits, DWQ.

Drop-in for ``trimquad.quadrature`` (src/quadrature.py:25-449).  Host side:
point-layout integer logic (counts, nested augmentation, knot insertion),
which is O(n) bookkeeping.  Device side: basis tables, exact 1-D moments,
the batched pivoted-QR moment fits and the DWQ combination
(``tq_moments_1d_g``, ``tq_wq_solve``, ``tq_dwq_combine``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import lru_cache

import ctypes as C

import bisect

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib as L
from ._lib import RuleConstructionError
from .splines import Basis1D, refine_to_c_minus_1

FIT_TOL = 1e-12       # src/quadrature.py:40
MAX_RETRIES = 5       # src/quadrature.py:43


@dataclass(frozen=True)
class GaussRule:
    """src/quadrature.py:50-60."""
    points: np.ndarray
    weights: np.ndarray

    def mapped(self, a, b):
        mid, half = 0.5 * (a + b), 0.5 * (b - a)
        return mid + half * self.points, half * self.weights


@lru_cache(maxsize=None)
def gauss_legendre(n: int) -> GaussRule:
    """n-point Gauss-Legendre rule on [-1,1] (src/quadrature.py:63-71)."""
    if n < 1:
        raise ValueError(f"point count must be positive, got {n}")
    x, w = np.polynomial.legendre.leggauss(n)
    x.setflags(write=False)
    w.setflags(write=False)
    return GaussRule(x, w)


_gauss_dev = {}


def gauss_device(n):
    if n not in _gauss_dev:
        g = gauss_legendre(n)
        _gauss_dev[n] = (L.dev(g.points, torch.float64), L.dev(g.weights, torch.float64))
    return _gauss_dev[n]


class PointLayout:
    """Points grouped by element, strictly interior (src/quadrature.py:74-121)."""

    def __init__(self, breakpoints, per_element=None, *, points=None, offsets=None, check=True):
        self.breakpoints = np.asarray(breakpoints, dtype=float)
        if per_element is not None:
            counts = np.array([len(g) for g in per_element], dtype=np.int64)
            self.offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
            self.points = np.concatenate(per_element) if self.offsets[-1] else np.empty(0)
        else:
            self.points = np.asarray(points, dtype=float)
            self.offsets = np.asarray(offsets, dtype=np.int64)
        counts = np.diff(self.offsets)
        self.element_of_point = np.repeat(np.arange(counts.size), counts)
        if check and self.points.size:
            e = self.element_of_point
            if np.any(self.points <= self.breakpoints[e]) or np.any(self.points >= self.breakpoints[e + 1]):
                bad = int(e[np.nonzero((self.points <= self.breakpoints[e]) |
                                       (self.points >= self.breakpoints[e + 1]))[0][0]])
                raise ValueError(f"points of element {bad} not strictly interior")
        self._dev = None

    num_points = property(lambda self: int(self.offsets[-1]))
    num_elements = property(lambda self: self.breakpoints.size - 1)

    def counts(self):
        return np.diff(self.offsets)

    def element_points(self, e):
        return self.points[self.offsets[e]: self.offsets[e + 1]]

    def range_for_elements(self, e0, e1):
        return int(self.offsets[e0]), int(self.offsets[e1 + 1])

    def contains(self, other, tol=1e-12):
        idx = np.clip(np.searchsorted(self.points, other.points), 0, self.num_points - 1)
        near = np.abs(self.points[idx] - other.points) <= tol
        idx2 = np.clip(idx - 1, 0, self.num_points - 1)
        near |= np.abs(self.points[idx2] - other.points) <= tol
        return bool(np.all(near))

    def device(self):
        if self._dev is None:
            pts, off = L.dev_many([(self.points, torch.float64), (self.offsets, torch.int32)])
            self._dev = (L.Layout(L.ptr(pts), L.ptr(off), self.num_points, self.num_elements), pts, off)
        return self._dev[0]

    def device_points(self):
        self.device()
        return self._dev[1]


def _required_counts(basis: Basis1D) -> np.ndarray:
    """max over tests of ceil(#trials / #support elements) (src/quadrature.py:130-143)."""
    t = basis._ov_hi - basis._ov_lo + 1
    ne = basis._el_last - basis._el_first + 1
    need = -(-t // ne)
    req = np.zeros(basis.num_elements, dtype=np.int64)
    # each function raises its support elements to its need
    for off in range(int(ne.max()) if ne.size else 0):
        e = basis._el_first + off
        ok = e <= basis._el_last
        np.maximum.at(req, e[ok], need[ok])
    return req


def _layout_from_counts(basis: Basis1D, counts) -> PointLayout:
    """a + (b-a)*k/(count+1), k = 1..count per element (src/quadrature.py:124-152)."""
    bp = basis.breakpoints
    counts = np.asarray(counts, dtype=np.int64)
    offsets = np.concatenate([[0], np.cumsum(counts)])
    e = np.repeat(np.arange(counts.size), counts)
    k = np.arange(offsets[-1]) - offsets[e] + 1
    a, b = bp[e], bp[e + 1]
    pts = a + (b - a) * k / (counts[e] + 1)
    return PointLayout(bp, points=pts, offsets=offsets)


def place_wq_points(basis: Basis1D) -> PointLayout:
    """src/quadrature.py:155-157."""
    from . import _adapt
    basis = _adapt.basis1d(basis)
    return _layout_from_counts(basis, _required_counts(basis))


_TAG = [""]     # timeline probe: prefix of the fit-chain stamps


def _st(name):
    from . import assembly as A
    if A.STAMPS is not None:
        A.STAMPS(_TAG[0] + name)


def moments_device(basis: Basis1D):
    """Banded exact 1-D mass matrix on the GPU, n x (2p+1); recomputed on
    every call like mass_matrix_1d inside the reference's _solve_rows."""
    gx, gw = gauss_device(basis.p + 1)
    mom = torch.empty((basis.n, 2 * basis.p + 1), dtype=torch.float64, device=L.device())
    L.call("tq_moments_1d_g", basis.device(), L.ptr(gx), L.ptr(gw), basis.p + 1, L.ptr(mom), L.stream())
    return mom


def mass_matrix_1d(basis: Basis1D, trial_basis=None) -> np.ndarray:
    """Exact 1-D mass matrix (src/quadrature.py:160-188), formed on the GPU:
    the banded moments (tq_moments_1d_g) for one space, the dense mixed
    matrix (tq_mass_1d_mixed) against another trial space on the same
    breakpoints."""
    from . import _adapt
    basis, trial_basis = _adapt.basis1d(basis), _adapt.basis1d(trial_basis)
    if trial_basis is not None and trial_basis is not basis:
        nb = max(basis.p, trial_basis.p) + 1
        gx, gw = gauss_device(nb)
        M = torch.empty((basis.n, trial_basis.n), dtype=torch.float64, device=L.device())
        L.call("tq_mass_1d_mixed", basis.device(), trial_basis.device(), L.ptr(gx), L.ptr(gw), nb, L.ptr(M),
               L.stream())
        return M.cpu().numpy()
    band = moments_device(basis).cpu().numpy()
    n, p = basis.n, basis.p
    M = np.zeros((n, n))
    i = np.repeat(np.arange(n), 2 * p + 1)
    j = i - p + np.tile(np.arange(2 * p + 1), n)
    ok = (j >= 0) & (j < n)
    M[i[ok], j[ok]] = band.ravel()[ok]
    return M


def exact_moments(basis, i):
    j0, j1 = basis.overlapping(i)
    return j0, mass_matrix_1d(basis)[i, j0: j1 + 1].copy()


class WeightedRuleSet:
    """Per-test weight rows on one layout, stored on the device
    (src/quadrature.py:201-232).  ``rows`` materializes host copies lazily."""

    def __init__(self, basis, layout, wptr, k0, w, direction=None):
        self.basis = basis
        self.layout = layout
        self.wptr, self.k0, self.w = wptr, k0, w     # device tensors
        self.direction = direction
        self._rows = None
        self._basis_tab = None

    def device(self):
        return L.Rules(L.ptr(self.wptr), L.ptr(self.k0), L.ptr(self.w))

    @property
    def rows(self):
        if self._rows is None:
            wptr = self.wptr.cpu().numpy()
            k0 = self.k0.cpu().numpy()
            w = self.w.cpu().numpy()
            self._rows = [None if k0[i] < 0 else (int(k0[i]), w[wptr[i]: wptr[i + 1]].copy())
                          for i in range(k0.size)]
        return self._rows

    def row(self, i):
        return self.rows[i]

    def row_full(self, i):
        k0, w = self.rows[i]
        full = np.zeros(self.layout.num_points)
        full[k0: k0 + w.size] = w
        return full

    def total_points(self):
        return self.layout.num_points

    def apply(self, i, values_at_points):
        k0, w = self.rows[i]
        return float(np.dot(w, values_at_points[k0: k0 + w.size]))

    def basis_table(self):
        """(first, vals) of the basis at this layout's points (device)."""
        if self._basis_tab is None:
            self._basis_tab = self.basis.eval_device(self.layout.device_points(), check=False)
        return self._basis_tab


class DiscontinuousRuleSet(WeightedRuleSet):
    """src/quadrature.py:235-260."""

    def __init__(self, basis, layout, wptr, k0, w, u_disc, subdivision, refined_basis, base_layout,
                 direction=None, regular_side=None):
        super().__init__(basis, layout, wptr, k0, w, direction)
        self.u_disc = float(u_disc)
        self.subdivision = subdivision
        self.refined_basis = refined_basis
        self.base_layout = base_layout
        self.regular_side = regular_side

    def side_points(self, side):
        if side == "left":
            return np.nonzero(self.layout.points < self.u_disc)[0]
        if side == "right":
            return np.nonzero(self.layout.points > self.u_disc)[0]
        raise ValueError(f"side must be 'left' or 'right', got {side!r}")


def _row_lengths(basis, layout):
    e0, e1 = basis._el_first, basis._el_last
    return layout.offsets[e1 + 1] - layout.offsets[e0]


class _FitPlan:
    """Host-side description of one batch of moment fits (sizes, row list,
    weight offsets) with its device copies; depends on geometry only."""

    def __init__(self, basis, layout, which=None):
        self.basis, self.layout = basis, layout
        lens = _row_lengths(basis, layout)
        self.wptr_h = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        self.rows_h = np.arange(basis.n, dtype=np.int32) if which is None else np.asarray(which, dtype=np.int32)
        t = basis._ov_hi - basis._ov_lo + 1
        self.tmax = int(t[self.rows_h].max()) if self.rows_h.size else 1
        self.mmax = int(lens[self.rows_h].max()) if self.rows_h.size else 1
        self.wptr, self.rows = L.dev_many([(self.wptr_h, torch.int64), (self.rows_h, torch.int32)])


def _solve_rows_async_t(plan: _FitPlan, init=None, products=None):
    """Launch the GPU moment fits of a plan (src/quadrature.py:281-303).
    Returns ((wptr, k0, w, fail), (first, vals) basis table at the layout
    points or None) as device tensors; no host sync.  The solve writes k0,
    the weights and the fail flag of every plan row; rows outside the plan
    are initialised (k0 = -1, w = 0) only when ``init`` (default: the plan
    leaves rows out), so a full plan launches no fill kernels."""
    basis, layout = plan.basis, plan.layout
    dev = L.device()
    init = plan.rows_h.size < basis.n if init is None else init
    if init:
        k0 = torch.full((basis.n,), -1, dtype=torch.int32, device=dev)
        w = torch.zeros(max(int(plan.wptr_h[-1]), 1), dtype=torch.float64, device=dev)
    else:
        k0 = torch.empty((basis.n,), dtype=torch.int32, device=dev)
        w = torch.empty(max(int(plan.wptr_h[-1]), 1), dtype=torch.float64, device=dev)
    fail = (torch.empty if plan.rows_h.size else torch.zeros)(max(plan.rows_h.size, 1), dtype=torch.int32, device=dev)
    tab = None
    if plan.rows_h.size:
        tab = basis.eval_device(layout.device_points(), check=False)
        _st("eval")
        first, vals = tab
        mom = moments_device(basis)
        _st("mom")
        L.call("tq_wq_solve", basis.device(), layout.device(), L.ptr(first), L.ptr(vals), L.ptr(mom),
               L.ptr(plan.rows), plan.rows_h.size, plan.tmax, plan.mmax, L.ptr(plan.wptr), L.ptr(k0), L.ptr(w),
               L.ptr(fail), L.ptr(products), L.stream())
        _st("solve")
    return (plan.wptr, k0, w, fail), tab


def fit_sets_async(plans, products=None, inits=None):
    """Every plan's moment fits in one fused launch per TQ_FIT_MAX_SETS plans
    (tq_wq_fit_sets: warp per system, its own moments and collocation block,
    LAPACK pivoting).  Returns [(wptr, k0, w, fail)] per plan as device
    tensors; no host sync.  Rows outside a plan are initialised (k0 = -1,
    w = 0) when ``inits[k]`` (default: the plan leaves rows out)."""
    dev = L.device()
    products = products or [None] * len(plans)
    inits = inits or [None] * len(plans)
    outs = []
    p = None
    for pl in plans:
        if p is not None and pl.basis.p != p:
            raise ValueError("one fused fit takes rule sets of one degree")
        p = pl.basis.p
    for c0 in range(0, len(plans), L.FIT_MAX_SETS):
        batch = L.FitBatch()
        tmax = mmax = 1
        chunk = list(zip(plans, products, inits))[c0: c0 + L.FIT_MAX_SETS]
        for k, (pl, prod, init) in enumerate(chunk):
            basis, layout = pl.basis, pl.layout
            init = pl.rows_h.size < basis.n if init is None else init
            if init:
                k0 = torch.full((basis.n,), -1, dtype=torch.int32, device=dev)
                w = torch.zeros(max(int(pl.wptr_h[-1]), 1), dtype=torch.float64, device=dev)
            else:
                k0 = torch.empty((basis.n,), dtype=torch.int32, device=dev)
                w = torch.empty(max(int(pl.wptr_h[-1]), 1), dtype=torch.float64, device=dev)
            fail = (torch.empty if pl.rows_h.size else torch.zeros)(max(pl.rows_h.size, 1), dtype=torch.int32,
                                                                    device=dev)
            outs.append((pl.wptr, k0, w, fail))
            batch.set[k] = L.FitSet(basis.device(), layout.device(), L.ptr(pl.rows), int(pl.rows_h.size),
                                    L.ptr(pl.wptr), L.ptr(k0), L.ptr(w), L.ptr(fail), L.ptr(prod))
            tmax, mmax = max(tmax, pl.tmax), max(mmax, pl.mmax)
        batch.nsets = len(chunk)
        gx, gw = gauss_device(p + 1)
        batch.gx, batch.gw = L.ptr(gx), L.ptr(gw)
        L.call("tq_wq_fit_sets", C.byref(batch), tmax, mmax, L.stream())
    return outs


def combine_sets_async(dplans, fine_outs):
    """w = S^T w~ of every DWQ plan, one launch per TQ_FIT_MAX_SETS plans
    (tq_dwq_combine_sets); returns the weight tensors."""
    dev = L.device()
    ws = []
    pairs = list(zip(dplans, fine_outs))
    for c0 in range(0, len(pairs), L.FIT_MAX_SETS):
        batch = L.CombineBatch()
        chunk = pairs[c0: c0 + L.FIT_MAX_SETS]
        for k, (pl, (fwptr, fk0, fw, _)) in enumerate(chunk):
            w = torch.empty(max(int(pl.wptr_h[-1]), 1), dtype=torch.float64, device=dev)
            ws.append(w)
            batch.set[k] = L.CombineSet(L.ptr(pl.rows), int(pl.wanted.size), L.ptr(pl.cp), L.ptr(pl.ri),
                                        L.ptr(pl.sv), L.Rules(L.ptr(fwptr), L.ptr(fk0), L.ptr(fw)),
                                        L.Rules(L.ptr(pl.wptr), L.ptr(pl.k0), L.ptr(w)))
        batch.nsets = len(chunk)
        L.call("tq_dwq_combine_sets", C.byref(batch), L.stream())
    return ws


def _solve_rows_async(plan: _FitPlan, init=None):
    """(wptr, k0, w, fail) of ``_solve_rows_async_t``."""
    return _solve_rows_async_t(plan, init)[0]


def _failing(plan, fail):
    return plan.rows_h[fail[: plan.rows_h.size].cpu().numpy() != 0].tolist() if plan.rows_h.size else []


def _solve_rows(basis: Basis1D, layout: PointLayout, which=None):
    """Synchronous variant: (wptr, k0, w device tensors, failing rows)."""
    plan = _FitPlan(basis, layout, which)
    wptr, k0, w, fail = _solve_rows_async(plan)
    return wptr, k0, w, _failing(plan, fail)


def _least_covered_element(basis, layout, i):
    """src/quadrature.py:306-309."""
    e0, e1 = basis.support_elements(i)
    return int(e0 + np.argmin(layout.counts()[e0: e1 + 1]))


def compute_wq_rules(basis: Basis1D, layout: PointLayout | None = None, direction=None) -> WeightedRuleSet:
    """WQ rules for every test function, GPU fits + enrichment retries
    (src/quadrature.py:312-337)."""
    from . import _adapt
    basis, layout = _adapt.basis1d(basis), _adapt.layout(layout)
    if layout is None:
        layout = place_wq_points(basis)
    counts = layout.counts().copy()
    failing = []
    for attempt in range(MAX_RETRIES + 1):
        wptr, k0, w, failing = _solve_rows(basis, layout)
        if not failing:
            return WeightedRuleSet(basis, layout, wptr, k0, w, direction)
        if attempt == MAX_RETRIES:
            break
        for i in failing:
            counts[_least_covered_element(basis, layout, i)] += 1
        layout = _layout_from_counts(basis, counts)
    raise RuleConstructionError(f"moment fit residual above {FIT_TOL:g} for test functions {failing} "
                                f"after {MAX_RETRIES} enrichment retries")


def _split_largest_gap(pts, a, b):
    """Midpoint of the first largest gap of [a, *pts, b] (src/quadrature.py:340-345)."""
    fence = np.concatenate([[a], pts, [b]])
    g = int(np.argmax(np.diff(fence)))
    return 0.5 * (fence[g] + fence[g + 1])


def _augment_nested(layout: PointLayout, extra) -> PointLayout:
    """Nested largest-gap augmentation (src/quadrature.py:348-363); only the
    elements with extra > 0 are rebuilt, the rest are spliced through."""
    extra = np.asarray(extra)
    touched = np.nonzero(extra > 0)[0]
    if touched.size == 0:
        return layout
    bp, off, pts = layout.breakpoints, layout.offsets, layout.points
    pieces, counts = [], np.diff(off).copy()
    prev = 0
    for e in touched:
        pieces.append(pts[off[prev]: off[e]])
        # a handful of points per element: plain floats (the same IEEE
        # arithmetic as _split_largest_gap, first largest gap, sorted insert)
        g = sorted(pts[off[e]: off[e + 1]].tolist())
        a, b = float(bp[e]), float(bp[e + 1])
        for _ in range(int(extra[e])):
            fence = [a, *g, b]
            gaps = [fence[k + 1] - fence[k] for k in range(len(fence) - 1)]
            k = gaps.index(max(gaps))
            bisect.insort(g, 0.5 * (fence[k] + fence[k + 1]))
        pieces.append(np.asarray(g, dtype=float))
        counts[e] = len(g)
        prev = e + 1
    pieces.append(pts[off[prev]:])
    new_off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    return PointLayout(bp, points=np.concatenate(pieces), offsets=new_off)


def dwq_layout(basis: Basis1D, layout: PointLayout, u: float):
    """Integer/point part of DWQ (src/quadrature.py:382-407):
    refined basis, subdivision matrix, nested augmented layout."""
    refined, S = refine_to_c_minus_1(basis, u)
    need = _required_counts(refined)
    aug = _augment_nested(layout, np.maximum(need - layout.counts(), 0))
    t = refined._ov_hi - refined._ov_lo + 1
    e0, e1 = refined._el_first, refined._el_last
    short = np.nonzero(aug.offsets[e1 + 1] - aug.offsets[e0] < t)[0]
    for i in short:        # top-up loop, in function order (usually empty)
        i = int(i)
        while aug.offsets[e1[i] + 1] - aug.offsets[e0[i]] < t[i]:
            bump = np.zeros(aug.num_elements, dtype=np.int64)
            bump[_least_covered_element(refined, aug, i)] = 1
            aug = _augment_nested(aug, bump)
    return refined, S, aug


class DwqPlan:
    """Geometry of one DWQ set (src/quadrature.py:382-418): refined basis,
    subdivision matrix S, nested augmented layout, the refined rows to fit
    and the output row layout.  Depends only on (basis, base layout, u_disc,
    rows), never on weights."""

    def __init__(self, basis, layout, u_disc, only_rows=None):
        bp = basis.breakpoints
        if not np.any(np.abs(bp - u_disc) <= 1e-12):
            raise ValueError(f"{u_disc} is not a breakpoint of the basis")
        self.basis, self.base_layout = basis, layout
        self.u = float(bp[np.argmin(np.abs(bp - u_disc))])
        self.refined, self.S, self.aug = dwq_layout(basis, layout, self.u)
        Sc = self.S.matrix.tocsc()
        Sc.sort_indices()
        self.Sc = Sc
        self.wanted = (np.arange(basis.n) if only_rows is None
                       else np.array(sorted(set(int(r) for r in only_rows)), dtype=np.int64))
        self.fine_needed = None
        if only_rows is not None:
            seen = set()
            for j in self.wanted:
                seen.update(Sc.indices[Sc.indptr[j]: Sc.indptr[j + 1]].tolist())
            self.fine_needed = sorted(seen)
        self._finalize()

    def _finalize(self):
        basis, aug = self.basis, self.aug
        self.fit = _FitPlan(self.refined, aug, self.fine_needed)
        lens = _row_lengths(basis, aug)
        sel = np.zeros(basis.n, dtype=bool)
        sel[self.wanted] = True
        lens = np.where(sel, lens, 0)
        self.wptr_h = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        k0_h = np.where(sel, aug.offsets[basis._el_first], -1).astype(np.int32)
        self.wptr, self.k0, self.cp, self.ri, self.sv, self.rows = L.dev_many([
            (self.wptr_h, torch.int64), (k0_h, torch.int32), (self.Sc.indptr, torch.int32),
            (self.Sc.indices, torch.int32), (self.Sc.data, torch.float64), (self.wanted, torch.int32)])

    def bump(self, failing):
        """Enrichment retry of the refined fit (src/quadrature.py:420-432)."""
        bump = np.zeros(self.aug.num_elements, dtype=np.int64)
        for i in failing:
            bump[_least_covered_element(self.refined, self.aug, i)] += 1
        self.aug = _augment_nested(self.aug, bump)
        self._finalize()


def dwq_solve_async(plan: DwqPlan, direction=None, regular_side=None):
    """Numeric part of DWQ on the GPU: refined fits, then w = S^T w~
    (src/quadrature.py:420-444).  Returns (rule set, fail tensor)."""
    # refined fits: read only by the combine, and only on their own rows
    fwptr, fk0, fw, fail = _solve_rows_async(plan.fit, init=False)
    # the combine writes every wanted row; other rows have empty ranges
    w = torch.empty(max(int(plan.wptr_h[-1]), 1), dtype=torch.float64, device=L.device())
    L.call("tq_dwq_combine", L.ptr(plan.rows), plan.wanted.size, L.ptr(plan.cp), L.ptr(plan.ri), L.ptr(plan.sv),
           L.Rules(L.ptr(fwptr), L.ptr(fk0), L.ptr(fw)), L.Rules(L.ptr(plan.wptr), L.ptr(plan.k0), L.ptr(w)),
           L.stream())
    _st("combine")
    rs = DiscontinuousRuleSet(plan.basis, plan.aug, plan.wptr, plan.k0, w, plan.u, plan.S, plan.refined,
                              plan.base_layout, direction, regular_side)
    return rs, fail


def build_dwq(basis: Basis1D, layout: PointLayout, u_disc: float, direction=None,
              regular_side=None, only_rows=None, plan=None) -> DiscontinuousRuleSet:
    """Discontinuous WQ (src/quadrature.py:366-449): host layout plan, GPU
    fits of the refined rows with enrichment retries, GPU w = S^T w~."""
    from . import _adapt
    basis, layout = _adapt.basis1d(basis), _adapt.layout(layout)
    plan = plan or DwqPlan(basis, layout, u_disc, only_rows)
    for attempt in range(MAX_RETRIES + 1):
        rs, fail = dwq_solve_async(plan, direction, regular_side)
        failing = _failing(plan.fit, fail)
        if not failing:
            return rs
        if attempt == MAX_RETRIES:
            raise RuleConstructionError(f"discontinuous rule fit failed for refined test functions "
                                        f"{failing} at u_disc={plan.u}")
        plan.bump(failing)


def rules_from_arrays(basis, points, offsets, k0, wptr, w, direction=None, u_disc=None):
    """Import a weight table computed elsewhere (WQ weights are not
    unique, so c != 1 parity compares against the same weights)."""
    lay = PointLayout(basis.breakpoints, points=np.asarray(points, float), offsets=np.asarray(offsets, np.int64))
    args = (basis, lay, L.dev(np.asarray(wptr, np.int64), torch.int64), L.dev(np.asarray(k0, np.int32), torch.int32),
            L.dev(np.asarray(w, float) if len(w) else np.zeros(1), torch.float64))
    if u_disc is None:
        return WeightedRuleSet(*args, direction=direction)
    return DiscontinuousRuleSet(*args, u_disc, None, None, None, direction=direction)
