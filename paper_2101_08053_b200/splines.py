"""Univariate and tensor-product B-spline spaces (host metadata + device mirror).

Drop-in for the reference ``trimquad.splines`` types (src/splines.py:17-455):
same class names, constructor arguments, properties and errors.  The index
bookkeeping is O(n) host work; evaluation runs on the GPU
(``Basis1D.eval_nonzero_batch`` -> ``tq_basis_eval``).
"""

from __future__ import annotations

import json

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib as L

KNOT_TOL = 1e-12  # src/splines.py:29


def _breakpoints(knots, tol=KNOT_TOL):
    """Unique values merging entries within tol of the running value
    (src/splines.py:156-166).  Vectorized when no gap lies in (0, tol]
    (then the running-value rule and plain gap splitting coincide)."""
    d = np.diff(knots)
    if not np.any((d > 0) & (d <= tol)):
        start = np.concatenate([[0], np.nonzero(d > tol)[0] + 1])
        mult = np.diff(np.concatenate([start, [knots.size]])).astype(np.int64)
        return knots[start], mult
    keep = [0]
    mult = [1]
    for k in range(1, knots.size):
        if knots[k] - knots[keep[-1]] <= tol:
            mult[-1] += 1
        else:
            keep.append(k)
            mult.append(1)
    return knots[np.asarray(keep)], np.asarray(mult, dtype=np.int64)


class KnotVector:
    """Open knot vector + degree (src/splines.py:32-153)."""

    def __init__(self, knots, degree: int):
        knots = np.ascontiguousarray(knots, dtype=float)
        degree = int(degree)
        if degree < 0:
            raise ValueError(f"degree must be non-negative, got {degree}")
        if knots.ndim != 1 or knots.size < 2 * (degree + 1):
            raise ValueError("knot vector too short for the requested degree")
        if np.any(np.diff(knots) < 0):
            raise ValueError("knots must be non-decreasing")
        bp, mult = _breakpoints(knots)
        if mult[0] != degree + 1 or mult[-1] != degree + 1:
            raise ValueError("open knot vector required: boundary knots must have "
                             f"multiplicity exactly {degree + 1}")
        if mult.size > 2 and np.any(mult[1:-1] > degree + 1):
            raise ValueError(f"interior knot multiplicity exceeds {degree + 1}")
        self.knots = knots
        self.knots.setflags(write=False)
        self.degree = degree
        self.breakpoints = bp
        self.multiplicities = mult
        self.element_spans = np.cumsum(mult)[:-1] - 1

    @property
    def num_elements(self):
        return self.breakpoints.size - 1

    @property
    def num_functions(self):
        return self.knots.size - self.degree - 1

    @property
    def domain(self):
        return float(self.knots[0]), float(self.knots[-1])

    def multiplicity_of(self, u):
        return int(np.sum(np.abs(self.knots - u) <= KNOT_TOL))

    def find_spans(self, u):
        u = np.asarray(u, dtype=float)
        lo, hi = self.domain
        if np.any(u < lo) or np.any(u > hi):
            bad = u[(u < lo) | (u > hi)][0]
            raise ValueError(f"coordinate {bad} outside domain [{lo}, {hi}]")
        s = np.searchsorted(self.knots, u, side="right") - 1
        return np.clip(s, self.degree, self.num_functions - 1)

    def find_span(self, u):
        return int(self.find_spans(np.asarray([u]))[0])

    def element_of(self, u):
        e = np.searchsorted(self.breakpoints, np.asarray(u, dtype=float), side="right") - 1
        return np.clip(e, 0, self.num_elements - 1)

    def insert(self, ubar):
        at = int(np.searchsorted(self.knots, ubar, side="right"))
        return KnotVector(np.insert(self.knots, at, ubar), self.degree)

    def to_json(self):
        return json.dumps({"degree": self.degree, "knots": self.knots.tolist()})

    @classmethod
    def from_json(cls, text):
        d = json.loads(text)
        return cls(d["knots"], d["degree"])

    def __eq__(self, other):
        return (isinstance(other, KnotVector) and self.degree == other.degree
                and self.knots.size == other.knots.size
                and bool(np.all(np.abs(self.knots - other.knots) <= KNOT_TOL)))

    def __repr__(self):
        return f"KnotVector(degree={self.degree}, n={self.num_functions})"


class Basis1D:
    """B-spline basis over a KnotVector (src/splines.py:169-300)."""

    def __init__(self, kv: KnotVector):
        self.kv = kv
        spans = kv.element_spans
        i = np.arange(kv.num_functions)
        # support elements: spans in [i, i+p] (src/splines.py:178-190)
        self._el_first = np.searchsorted(spans, i, side="left")
        self._el_last = np.searchsorted(spans, i + kv.degree, side="right") - 1
        self._ov_lo = spans[self._el_first] - kv.degree
        self._ov_hi = spans[self._el_last]
        self._dev = None

    p = property(lambda self: self.kv.degree)
    n = property(lambda self: self.kv.num_functions)
    breakpoints = property(lambda self: self.kv.breakpoints)
    num_elements = property(lambda self: self.kv.num_elements)
    domain = property(lambda self: self.kv.domain)

    def support_elements(self, i):
        return int(self._el_first[i]), int(self._el_last[i])

    def support_interval(self, i):
        kn = self.kv.knots
        return float(kn[i]), float(kn[i + self.p + 1])

    def functions_on_element(self, e):
        s = int(self.kv.element_spans[e])
        return s - self.p, s

    def overlapping(self, i):
        return int(self._ov_lo[i]), int(self._ov_hi[i])

    # -- device mirror ---------------------------------------------------------
    def device(self):
        """tq_space1d view with device arrays (cached)."""
        if self._dev is None:
            names = ("knots", "bp", "espan", "el_first", "el_last", "ov_lo", "ov_hi")
            f64, i32 = torch.float64, torch.int32
            keep = dict(zip(names, L.dev_many([      # one upload for the seven tables
                (self.kv.knots, f64), (self.breakpoints, f64), (self.kv.element_spans, i32),
                (self._el_first, i32), (self._el_last, i32), (self._ov_lo, i32), (self._ov_hi, i32)])))
            st = L.Space1D(*(L.ptr(keep[k]) for k in ("knots", "bp", "espan", "el_first", "el_last",
                                                     "ov_lo", "ov_hi")),
                           self.kv.knots.size, self.p, self.n, self.num_elements)
            self._dev = (st, keep)
        return self._dev[0]

    def device_arrays(self):
        self.device()
        return self._dev[1]

    def eval_device(self, u_dev, ders=False, check=True):
        """GPU Cox-de Boor at device points -> (first int32, vals[, ders]).
        ``check`` reads the domain status back (a stream sync); internal
        callers whose points are in the domain by construction skip it."""
        n = u_dev.numel()
        first = torch.empty(n, dtype=torch.int32, device=u_dev.device)
        vals = torch.empty((n, self.p + 1), dtype=torch.float64, device=u_dev.device)
        dv = torch.empty_like(vals) if ders else None
        status = torch.zeros(1, dtype=torch.int32, device=u_dev.device) if check else None
        L.call("tq_basis_eval", self.device(), L.ptr(u_dev), n, L.ptr(first), L.ptr(vals), L.ptr(dv),
               L.ptr(status), L.stream())
        if check and int(status.item()) & 1:
            raise ValueError("coordinate outside the knot domain")
        return (first, vals, dv) if ders else (first, vals)

    def eval_nonzero_batch(self, u):
        """(first, values) like src/splines.py:245-269, computed on the GPU."""
        u = np.asarray(u, dtype=float).reshape(-1)
        self.kv.find_spans(u)  # domain check with the reference's message
        first, vals = self.eval_device(L.dev(u, torch.float64))
        return first.cpu().numpy().astype(np.int64), vals.cpu().numpy()

    def eval_nonzero(self, u):
        f, v = self.eval_nonzero_batch(np.asarray([u]))
        return int(f[0]), v[0]

    def eval_single(self, i, u):
        a, b = self.support_interval(i)
        if u < a or u > b:
            return 0.0
        f, v = self.eval_nonzero(u)
        k = i - f
        return float(v[k]) if 0 <= k <= self.p else 0.0

    def collocation(self, points):
        points = np.asarray(points, dtype=float)
        f, v = self.eval_nonzero_batch(points)
        C = np.zeros((points.size, self.n))
        rows = np.repeat(np.arange(points.size), self.p + 1)
        cols = (f[:, None] + np.arange(self.p + 1)[None, :]).ravel()
        C[rows, cols] = v.ravel()
        return C

    def spline_value(self, coeffs, u):
        f, v = self.eval_nonzero_batch(u)
        idx = f[:, None] + np.arange(self.p + 1)[None, :]
        return np.einsum("kj,kj->k", np.asarray(coeffs)[idx], v)

    def __repr__(self):
        return f"Basis1D(p={self.p}, n={self.n}, elements={self.num_elements})"


class TensorBasis2D:
    """src/splines.py:303-330."""

    def __init__(self, basis1: Basis1D, basis2: Basis1D):
        self.dir = (basis1, basis2)

    shape = property(lambda self: (self.dir[0].n, self.dir[1].n))
    degrees = property(lambda self: (self.dir[0].p, self.dir[1].p))
    num_elements = property(lambda self: (self.dir[0].num_elements, self.dir[1].num_elements))

    def value(self, index, u1, u2):
        return self.dir[0].eval_single(index[0], u1) * self.dir[1].eval_single(index[1], u2)

    def __repr__(self):
        return f"TensorBasis2D(p={self.degrees}, n={self.shape})"


class SubdivisionMatrix:
    """Sparse coarse->fine coefficient map (src/splines.py:333-366)."""

    def __init__(self, matrix, source, target):
        self.matrix = sp.csr_matrix(matrix)
        self.source = source
        self.target = target

    shape = property(lambda self: self.matrix.shape)

    def apply(self, coeffs):
        return self.matrix @ np.asarray(coeffs)

    def bandwidth(self):
        """max |row - col| over the stored entries (src/splines.py:356-360)."""
        m = self.matrix.tocoo()
        return int(np.max(np.abs(m.row - m.col))) if m.nnz else 0

    def __matmul__(self, other):
        return SubdivisionMatrix(self.matrix @ other.matrix, other.source, self.target)

    def __repr__(self):
        return f"SubdivisionMatrix({self.shape[0]}x{self.shape[1]})"


def insert_knot(basis: Basis1D, ubar: float):
    """One knot insertion with its subdivision map (src/splines.py:369-403;
    PAPER Eq. 9 alpha coefficients)."""
    kv = basis.kv
    p, n, kn = kv.degree, kv.num_functions, kv.knots
    lo, hi = kv.domain
    if not (lo <= ubar <= hi):
        raise ValueError(f"insertion point {ubar} outside domain [{lo}, {hi}]")
    if kv.multiplicity_of(ubar) >= p + 1:
        raise ValueError(f"multiplicity of {ubar} would exceed {p + 1}")
    l = kv.find_span(ubar)
    k = np.arange(n + 1)
    alpha = np.where(k <= l - p, 1.0, 0.0)
    mid = np.arange(max(l - p + 1, 0), l + 1)
    alpha[mid] = (ubar - kn[mid]) / (kn[mid + p] - kn[mid])
    r = np.concatenate([np.arange(n), np.arange(1, n + 1)])
    c = np.concatenate([np.arange(n), np.arange(n)])
    S = sp.coo_matrix((np.concatenate([alpha[:n], 1.0 - alpha[1:]]), (r, c)), shape=(n + 1, n)).tocsr()
    S.eliminate_zeros()
    fine = Basis1D(kv.insert(ubar))
    return fine, SubdivisionMatrix(S, basis, fine)


def _insertion_matrix(kn, p, ubar):
    """Single-insertion map on a raw knot array (PAPER Eq. 9; the alpha rule
    of src/splines.py:369-403)."""
    n = kn.size - p - 1
    l = int(np.clip(np.searchsorted(kn, ubar, side="right") - 1, p, n - 1))
    k = np.arange(n + 1)
    alpha = np.where(k <= l - p, 1.0, 0.0)
    mid = np.arange(max(l - p + 1, 0), l + 1)
    alpha[mid] = (ubar - kn[mid]) / (kn[mid + p] - kn[mid])
    r = np.concatenate([np.arange(n), np.arange(1, n + 1)])
    c = np.concatenate([np.arange(n), np.arange(n)])
    S = sp.coo_matrix((np.concatenate([alpha[:n], 1.0 - alpha[1:]]), (r, c)), shape=(n + 1, n)).tocsr()
    S.eliminate_zeros()
    at = int(np.searchsorted(kn, ubar, side="right"))
    return np.insert(kn, at, ubar), S


def _multiset_difference(a, b, tol=KNOT_TOL):
    """Values of the sorted knot sequence ``a`` not matched by ``b`` (multiset
    semantics within the knot tolerance): a two-pointer walk over the two
    sorted sequences."""
    a, b = np.asarray(a, float), np.asarray(b, float)
    out, j = [], 0
    for v in a:
        while j < b.size and b[j] < v - tol:
            j += 1
        if j < b.size and abs(b[j] - v) <= tol:
            j += 1
        else:
            out.append(v)
    return np.asarray(out, float)


def subdivision_matrix_to(basis: Basis1D, target_knots) -> SubdivisionMatrix:
    """Composite subdivision map onto a nested, finer knot vector of the same
    degree (src/splines.py:406-428): the product of single knot insertions,
    in ascending order of the missing knots.  ``target_knots``: a KnotVector
    or a knot sequence; it must contain the source knots as a multiset."""
    target = target_knots if isinstance(target_knots, KnotVector) else KnotVector(target_knots, basis.p)
    if target.degree != basis.p:
        raise ValueError("target knot vector must have the same degree")
    if _multiset_difference(basis.kv.knots, target.knots).size:
        raise ValueError("target knot vector is not a refinement of the source")
    current, S = basis, sp.identity(basis.n, format="csr")
    for ubar in _multiset_difference(target.knots, basis.kv.knots):
        current, step = insert_knot(current, float(ubar))
        S = step.matrix @ S
    return SubdivisionMatrix(S, basis, current)


def refine_to_c_minus_1(basis: Basis1D, u: float):
    """Insert u up to multiplicity p+1 -> (refined basis, SubdivisionMatrix);
    the composite of single insertions (src/splines.py:406-428)."""
    kv = basis.kv
    if not (kv.domain[0] <= u <= kv.domain[1]):
        raise ValueError(f"insertion point {u} outside domain {kv.domain}")
    kn, S = _repeated_insertion(kv.knots, basis.p, u, basis.p + 1 - kv.multiplicity_of(u))
    fine = Basis1D(KnotVector(kn, basis.p))
    return fine, SubdivisionMatrix(S, basis, fine)


def _repeated_insertion(kn, p, u, r):
    """Composite of r insertions of the same knot u (the product of the
    single-insertion maps of _insertion_matrix, bit-identical).  Outside a
    window around u the map is the identity above and an identity shifted by
    r below, so only that window is composed, densely: a step's new row k is
    alpha_k row_k + (1 - alpha_k) row_{k-1}, the two-term sum of the sparse
    product."""
    kn = np.asarray(kn, float)
    n = kn.size - p - 1
    if r <= 0:
        return kn.copy(), sp.identity(n, format="csr")
    at = int(np.searchsorted(kn, u, side="right"))       # every copy of u goes in here
    l0 = min(max(at - 1, p), n - 1)
    lo = max(l0 - p, 0)
    w = l0 - lo + 1
    B = np.eye(w)                        # rows = coefficients lo .., cols = source lo .. l0
    zrow = np.zeros((1, w))
    for s in range(r):
        nc = kn.size - p - 1
        l = min(max(at + s - 1, p), nc - 1)
        nb = B.shape[0]
        g = lo + np.arange(nb + 1)       # global coefficient index after the insertion
        mid = (g > l - p) & (g < l + 1)
        gm = g[mid]
        a = np.where(g <= l - p, 1.0, 0.0)
        a[mid] = (u - kn[gm]) / (kn[gm + p] - kn[gm])
        # rows above the span copy B[k] (a = 1), rows below copy B[k - 1]
        # (a = 0): 1 * x + 0 * y is exact, so this is the scalar recurrence
        new = a[:, None] * np.concatenate([B, zrow]) + (1.0 - a)[:, None] * np.concatenate([zrow, B])
        B = new
        kn = np.concatenate([kn[: at + s], [u], kn[at + s:]])
    nb = B.shape[0]
    bi, bj = np.nonzero(B)               # row-major: sorted by row, then column
    tail = np.arange(lo + nb, n + r)
    counts = np.concatenate([np.ones(lo, np.int64), np.bincount(bi, minlength=nb), np.ones(tail.size, np.int64)])
    indptr = np.concatenate([[0], np.cumsum(counts)])
    indices = np.concatenate([np.arange(lo), lo + bj, tail - r])
    vals = np.concatenate([np.ones(lo), B[bi, bj], np.ones(tail.size)])
    S = sp.csr_matrix((vals, indices.astype(np.int32), indptr.astype(np.int32)), shape=(n + r, n))
    S.has_sorted_indices = True
    return kn, S


def make_uniform_knots(num_elements, degree, a=0.0, b=1.0):
    """src/splines.py:445-451."""
    if num_elements < 1:
        raise ValueError("need at least one element")
    inner = np.linspace(a, b, num_elements + 1)[1:-1]
    return KnotVector(np.concatenate([np.full(degree + 1, a), inner, np.full(degree + 1, b)]), degree)


def make_uniform_basis(num_elements, degree, a=0.0, b=1.0):
    return Basis1D(make_uniform_knots(num_elements, degree, a, b))
