"""Trimming curves, GPU element/function classification, cut-cell quadrature.

Drop-in for ``trimquad.trimming`` (src/trimming.py:22-1130).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from ._lib import CUT, EXTERIOR, INTERIOR, TrimmingConfigurationError
from .splines import TensorBasis2D

ON_CURVE_TOL = 1e-12   # src/trimming.py:40
SNAP_REL_TOL = 1e-10   # src/trimming.py:43
MAX_SPLIT_DEPTH = 4    # src/trimming.py:46


class ElementClass:
    """src/trimming.py:53-56."""
    INTERIOR = INTERIOR
    CUT = CUT
    EXTERIOR = EXTERIOR


@dataclass
class DwqInfo:
    """src/trimming.py:410-425."""
    eligible: bool
    u_disc: tuple
    box: tuple | None
    regular_side: tuple
    residual: list
    cut: list


@dataclass(frozen=True)
class Intersection:
    """A curve/edge intersection (src/trimming.py:59-66)."""
    t: float
    coord: float
    point: tuple
    tangential: bool = False


@dataclass
class SubCell:
    """One mapped integration cell with its quadrature (src/trimming.py:740-746).
    The device decomposition does not report the cell shape: ``kind`` is
    'cell'."""
    kind: str
    points: np.ndarray
    weights: np.ndarray


def _integral_image(a):
    out = np.zeros((a.shape[0] + 1, a.shape[1] + 1), dtype=np.int64)
    out[1:, 1:] = np.cumsum(np.cumsum(a, axis=0), axis=1)
    return out


def _host_copy(t):
    """Device tensor -> numpy array backed by pinned memory (one DMA)."""
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return h.numpy()


class TrimConfiguration:
    """Element and function classification of a trimmed tensor space
    (src/trimming.py:428-594).  Classes are produced on the GPU; host copies
    are kept for the Python-level queries."""

    def __init__(self, basis2d: TensorBasis2D, curves, element_class_dev, func_class_dev,
                 face1, face2):
        self.basis2d = basis2d
        self.curves = list(curves)
        self.element_class_dev = element_class_dev
        self.func_class_dev = func_class_dev
        self._element_class = None       # host copies: made on first use
        self._func_class = None
        b1, b2 = basis2d.dir
        self.u_disc = (np.asarray(b1.breakpoints[1:-1][face1], dtype=float),
                       np.asarray(b2.breakpoints[1:-1][face2], dtype=float))
        self._cut_rules = {}
        self._cut_pending = {}
        self._dwq_cache = {}
        self._active = None
        self._active_fns = None
        self._cum_int = None

    @property
    def element_class(self):
        """Host copy of the element classes (int8 nel1 x nel2; D2H on first use)."""
        if self._element_class is None:
            self._element_class = _host_copy(self.element_class_dev)
        return self._element_class

    @property
    def func_class(self):
        """Host copy of the function classes (int8 n1 x n2; D2H on first use)."""
        if self._func_class is None:
            self._func_class = _host_copy(self.func_class_dev)
        return self._func_class

    @property
    def num_elements(self):
        return tuple(self.element_class_dev.shape)

    def element_bounds(self, e1, e2):
        bp1 = self.basis2d.dir[0].breakpoints
        bp2 = self.basis2d.dir[1].breakpoints
        return float(bp1[e1]), float(bp1[e1 + 1]), float(bp2[e2]), float(bp2[e2 + 1])

    @property
    def cut_elements(self):
        e1, e2 = np.nonzero(self.element_class == CUT)
        return list(zip(e1.tolist(), e2.tolist()))

    def has_cuts(self):
        if not hasattr(self, "_has_cuts"):
            if self._element_class is not None:
                self._has_cuts = bool(np.any(self._element_class == CUT))
            else:        # on the device: one flag read back
                self._has_cuts = bool((self.element_class_dev == CUT).any().item())
        return self._has_cuts

    @property
    def interior_elements(self):
        e1, e2 = np.nonzero(self.element_class == INTERIOR)
        return list(zip(e1.tolist(), e2.tolist()))

    def active_functions(self):
        """src/trimming.py:514-517 (row-major): (K, 2) int64 (i1, i2) pairs,
        built on the device from the active index and copied once through
        pinned memory (cached: geometry)."""
        if self._active_fns is None:
            idx, _ = self.active_index()
            act = idx["active"][: idx["K"]].long()
            n2 = self.basis2d.shape[1]
            pairs = torch.stack((act // n2, act % n2), dim=1)
            h = torch.empty(pairs.shape, dtype=torch.int64, pin_memory=True)
            h.copy_(pairs, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            self._active_fns = (h, h.numpy())
        return self._active_fns[1]

    def active_index(self):
        """Device col_of (n1*n2), active list (K) -- tq_active_index."""
        if self._active is None:
            n1, n2 = self.basis2d.shape
            dev = L.device()
            col_of = torch.empty(n1 * n2, dtype=torch.int32, device=dev)
            active = torch.empty(n1 * n2, dtype=torch.int32, device=dev)
            K = L.i32(0)
            L.call("tq_active_index", L.ptr(self.func_class_dev), n1 * n2, L.ptr(col_of), L.ptr(active),
                   L.C.byref(K), L.stream())
            self._active = ({"col_of": col_of, "active": active, "K": int(K.value)}, None)
        return self._active

    def support_block(self, i1, i2):
        a1, b1 = self.basis2d.dir[0].support_elements(i1)
        a2, b2 = self.basis2d.dir[1].support_elements(i2)
        return a1, b1, a2, b2

    def cut_cell_rule(self, q, cache=True):
        """Cut-element quadrature, host-native C++ (src/trimming.py:588-594,1084-1111)."""
        if cache and q in self._cut_rules:
            return self._cut_rules[q]
        pending = self._cut_pending.pop(q, None) if cache else None
        source = getattr(self, "_cut_rule_source", None)
        if source is not None:            # a caller-built configuration with non-device curves
            from . import _adapt
            rule = _adapt.cut_rule_from(source, q)
        elif pending is not None:         # started by cut_cell_rule_async
            rule = pending.result()
        else:
            from . import _classify
            rule = _classify.cut_cell_rule(self, q)
        if cache:
            self._cut_rules[q] = rule
        return rule

    def cut_cell_rule_async(self, q):
        """Start building the cut-element quadrature on a worker thread (the
        C++ decomposition runs without the GIL); ``cut_cell_rule(q)`` joins."""
        if q in self._cut_rules or q in self._cut_pending or not self.has_cuts():
            return
        if getattr(self, "_cut_rule_source", None) is not None:
            return
        if self.element_class_dev is not None and self.element_class_dev.is_cuda:
            # decomposed on the device: queued now (outside stream capture),
            # joined on first use, so the kernel and the read-back of its
            # summary overlap the caller's host work
            if not torch.cuda.is_current_stream_capturing():
                from . import _classify
                self._cut_pending[q] = _classify.start_cut_cell_rule_device(self, q)
            return
        from . import _classify
        self._cut_pending[q] = _classify.submit(_classify.cut_cell_rule, self, q, True)

    def support_split(self, i1, i2):
        a1, b1, a2, b2 = self.support_block(i1, i2)
        blk = self.element_class[a1: b1 + 1, a2: b2 + 1]
        reg = [(a1 + r, a2 + c) for r, c in zip(*np.nonzero(blk == INTERIOR))]
        cut = [(a1 + r, a2 + c) for r, c in zip(*np.nonzero(blk == CUT))]
        return reg, cut

    def is_inside(self, points):
        """Valid-region test of every curve (src/trimming.py:493-498), on the device."""
        pts = np.atleast_2d(np.asarray(points, dtype=float))
        inside = np.ones(pts.shape[0], dtype=bool)
        for curve in self.curves:
            inside &= np.asarray(curve.is_inside(pts), dtype=bool)
        return inside

    def dwq_info(self, i1, i2):
        """DWQ routing of one basis function (src/trimming.py:536-586): the
        device routing kernel (tq_dwq_route, the one the assembly uses) on
        that function, cached like the reference's ``_dwq_cache``."""
        key = (int(i1), int(i2))
        info = self._dwq_cache.get(key)
        if info is None:
            info = self._dwq_cache[key] = _dwq_info(self, *key)
        return info


# ---------------------------------------------------------------------------
# trimming curves: descriptors for the device classifier / host decomposition
# (src/trimming.py:69-351 and the harness closed curves)
# ---------------------------------------------------------------------------

class TrimmingCurve:
    """Oriented curve; the valid domain lies to the left (src/trimming.py:69-95).

    The predicate interface -- ``signed_distance``, ``is_inside`` and
    ``intersect_line`` -- runs on the device (``tq_curve_eval``,
    ``tq_curve_intersect_line``) with the very predicates the classifier and
    the cut-cell decomposition use, for every curve that has a device
    ``descriptor()``.  ``evaluate`` / ``derivative`` are the closed-form
    parametrisations (host).  A subclass without a descriptor keeps its own
    Python predicates; it cannot be classified on the device, but a
    configuration built around it by the reference package can be passed to
    the formation entry points (see ``_adapt``)."""
    straight = False
    closed = False

    def sample(self, n=257):
        return self.evaluate(np.linspace(0.0, 1.0, n))

    def descriptor(self):
        raise NotImplementedError(f"{type(self).__name__} has no device descriptor; use LineTrim, CircleTrim, "
                                  "ClosedCircleTrim, BezierTrim or PeriodicBSplineTrim, or build the "
                                  "configuration with the reference's classify_elements and pass it in")

    def _device_op(self, op, values, width):
        from . import _classify
        x = np.ascontiguousarray(values, dtype=np.float64)
        n = x.shape[0]
        if n == 0:
            return np.empty((0, 2)) if width == 2 else np.empty(0)
        arr, keep = _classify.curve_array([self])
        xin = L.dev(x.reshape(-1), torch.float64)
        out = torch.empty(n * width, dtype=torch.float64, device=L.device())
        L.call("tq_curve_eval", arr, op, L.ptr(xin), n, L.ptr(out), L.stream())
        o = out.cpu().numpy()
        return o.reshape(n, 2) if width == 2 else o

    def signed_distance(self, points):
        """Distance to the curve, positive on the valid side (src/trimming.py:80-82)."""
        return self._device_op(2, np.atleast_2d(np.asarray(points, dtype=float)), 1)

    def is_inside(self, points):
        """True in the valid (left) region, on-curve counts inside (src/trimming.py:76-78)."""
        return self._device_op(3, np.atleast_2d(np.asarray(points, dtype=float)), 1) != 0.0

    def intersect_line(self, axis, level):
        """All (t, cross coordinate) where the curve meets {axis = level},
        'v' = vertical line u1 = level (src/trimming.py:84-93): the hits the
        device classifier sweeps (tangential touches dropped, duplicates
        merged, sorted by cross coordinate)."""
        if axis not in ("v", "h"):
            raise ValueError("axis must be 'v' or 'h'")
        from . import _classify
        arr, keep = _classify.curve_array([self])
        cap = 64
        dev = L.device()
        ht = torch.empty(cap, dtype=torch.float64, device=dev)
        hc = torch.empty(cap, dtype=torch.float64, device=dev)
        cnt = torch.zeros(2, dtype=torch.int32, device=dev)
        L.call("tq_curve_intersect_line", arr, 0 if axis == "v" else 1, float(level), cap, L.ptr(ht), L.ptr(hc),
               L.ptr(cnt), L.stream())
        n, ovf = (int(v) for v in cnt.cpu().tolist())
        if ovf or n > cap:
            raise TrimmingConfigurationError("too many curve crossings on one grid line")
        t, c = ht[:n].cpu().numpy(), hc[:n].cpu().numpy()
        return [(float(a), float(b)) for a, b in zip(t, c)]


class LineTrim(TrimmingCurve):
    """src/trimming.py:98-134."""
    straight = True

    def __init__(self, p0, p1):
        self.p0 = np.asarray(p0, dtype=float)
        self.p1 = np.asarray(p1, dtype=float)
        self.d = self.p1 - self.p0
        if np.hypot(*self.d) == 0.0:
            raise ValueError("degenerate line segment")

    def evaluate(self, t):
        return self.p0 + np.multiply.outer(np.asarray(t, dtype=float), self.d)

    def derivative(self, t):
        t = np.asarray(t, dtype=float)
        return np.broadcast_to(self.d, t.shape + (2,)).copy()

    def descriptor(self):
        return 1, 0, np.array([*self.p0, *self.p1])


class CircleTrim(TrimmingCurve):
    """Circular arc theta0 -> theta1 (src/trimming.py:137-201)."""

    def __init__(self, center, radius, theta0=0.0, theta1=0.5 * np.pi):
        self.center = np.asarray(center, dtype=float)
        self.radius = float(radius)
        self.theta0, self.theta1 = float(theta0), float(theta1)
        if self.radius <= 0 or self.theta0 == self.theta1:
            raise ValueError("degenerate circular arc")

    def _th(self, t):
        return self.theta0 + np.asarray(t, dtype=float) * (self.theta1 - self.theta0)

    def evaluate(self, t):
        th = self._th(t)
        return self.center + self.radius * np.stack([np.cos(th), np.sin(th)], axis=-1)

    def derivative(self, t):
        th = self._th(t)
        return self.radius * (self.theta1 - self.theta0) * np.stack([-np.sin(th), np.cos(th)], axis=-1)

    def descriptor(self):
        return 2, 0, np.array([*self.center, self.radius, self.theta0, self.theta1])


class ClosedCircleTrim(CircleTrim):
    """Full circle with a movable seam; ccw keeps the disc (harness)."""
    closed = True

    def __init__(self, center, radius, ccw=False, seam=np.pi):
        self.ccw = bool(ccw)
        self.seam = float(seam)
        s = 1.0 if ccw else -1.0
        super().__init__(center, radius, seam, seam + s * 2.0 * np.pi)

    def descriptor(self):
        return 3, 0, np.array([*self.center, self.radius, 1.0 if self.ccw else 0.0, self.seam,
                               self.theta1 - self.theta0])


class PeriodicBSplineTrim(TrimmingCurve):
    """Closed uniform periodic cubic B-spline (harness); valid
    side to the left of the control-polygon orientation."""
    closed = True

    def __init__(self, ctrl, shift=0.0):
        self.ctrl = np.asarray(ctrl, dtype=float)
        self.m = self.ctrl.shape[0]
        self.shift = float(shift) % 1.0
        P = self.ctrl
        self.ccw = float(np.sum(P[:, 0] * np.roll(P[:, 1], -1) - np.roll(P[:, 0], -1) * P[:, 1])) > 0

    def _pw(self):
        m = self.m
        G = self.ctrl[(np.arange(m)[:, None] + np.arange(4)[None, :]) % m]
        P0, P1, P2, P3 = G[:, 0], G[:, 1], G[:, 2], G[:, 3]
        return np.stack([(-P0 + 3.0 * P1 - 3.0 * P2 + P3) / 6.0, (3.0 * P0 - 6.0 * P1 + 3.0 * P2) / 6.0,
                         (-3.0 * P0 + 3.0 * P2) / 6.0, (P0 + 4.0 * P1 + P2) / 6.0], axis=1)

    def _seg(self, t):
        s = ((np.asarray(t, dtype=float) + self.shift) % 1.0) * self.m
        k = np.minimum(np.floor(s).astype(np.int64), self.m - 1)
        return k, s - k

    def evaluate(self, t):
        k, u = self._seg(t)
        c = self._pw()[k]
        u = np.asarray(u)[..., None]
        return ((c[..., 0, :] * u + c[..., 1, :]) * u + c[..., 2, :]) * u + c[..., 3, :]

    def derivative(self, t):
        k, u = self._seg(t)
        c = self._pw()[k]
        u = np.asarray(u)[..., None]
        return self.m * ((3.0 * c[..., 0, :] * u + 2.0 * c[..., 1, :]) * u + c[..., 2, :])

    def descriptor(self):
        return 5, self.m, np.concatenate([[self.shift, 1.0 if self.ccw else 0.0], self.ctrl.ravel()])


class BezierTrim(TrimmingCurve):
    """Cubic Bezier trimming curve with its endpoints on the domain boundary
    (src/trimming.py:204-351).  The device predicates (csrc/curves.cuh
    bz_*) classify points by crossing parity of the segment to a valid
    anchor (cubic roots), with the reference's grazing retries and
    nearest-point tangent fallback."""

    def __init__(self, control_points, anchors=((0.05, 0.05), (0.08, 0.03), (0.03, 0.09))):
        self.ctrl = np.asarray(control_points, dtype=float)
        if self.ctrl.shape != (4, 2):
            raise ValueError("cubic Bezier needs 4 control points")
        c0, c1, c2, c3 = self.ctrl
        # power-basis coefficients, highest degree first (same as the reference)
        self._pow = np.stack([-c0 + 3 * c1 - 3 * c2 + c3, 3 * c0 - 6 * c1 + 3 * c2, -3 * c0 + 3 * c1, c0])
        self.anchors = [np.asarray(a, dtype=float) for a in anchors]
        if len(self.anchors) != 3:
            raise ValueError("the device predicates take three anchors")

    def evaluate(self, t):
        a, b, c, d = self._pow
        tt = np.asarray(t, dtype=float)[..., None]
        return a * tt ** 3 + b * tt ** 2 + c * tt + d

    def derivative(self, t):
        a, b, c, _ = self._pow
        tt = np.asarray(t, dtype=float)[..., None]
        return 3 * a * tt ** 2 + 2 * b * tt + c

    def descriptor(self):
        return 4, 0, np.concatenate([self.ctrl.ravel(), np.concatenate(self.anchors)])


def classify_point(curves, point):
    """True where ``point`` lies in the valid region of every curve
    (src/trimming.py:371-377): a bool for one point, else a bool array."""
    pts = np.atleast_2d(np.asarray(point, dtype=float))
    inside = np.ones(pts.shape[0], dtype=bool)
    for curve in curves:
        inside &= np.asarray(curve.is_inside(pts), dtype=bool)
    return bool(inside.all()) if pts.shape[0] == 1 else inside


def _is_tangential(curve, t, axis):
    """src/trimming.py:399-403."""
    d = np.asarray(curve.derivative(t)).reshape(-1)
    k = 0 if axis == "v" else 1
    return abs(d[k]) < 1e-9 * max(np.hypot(d[0], d[1]), 1e-30)


def intersect_edge(curve, axis, level, lo, hi):
    """Intersections of a curve with the axis-aligned segment {axis = level}
    x [lo, hi], tangential touches flagged, sorted along the edge
    (src/trimming.py:380-396)."""
    hits = []
    for item in curve.intersect_line(axis, level):
        t, coord = item[0], item[1]
        tangential = _is_tangential(curve, t, axis)
        if lo - 1e-12 <= coord <= hi + 1e-12:
            pt = (level, coord) if axis == "v" else (coord, level)
            hits.append(Intersection(t, float(coord), pt, tangential))
    hits.sort(key=lambda h: h.coord)
    return hits


# sub-cell capacity of a single-element decomposition (the split depth is at
# most 4: far fewer cells than this are ever produced)
_DECOMP_CELLS = 256


def decompose_cut_element(bounds, curve, q):
    """Sub-cells of one cut element with (q+1)^2 Gauss points each
    (src/trimming.py:938-1056), decomposed on the device by the kernel the
    configurations use (tq_cutcell_device_slots on a one-element mesh)."""
    from . import _classify
    if q < 1:
        raise ValueError("Lagrange degree q must be >= 1")
    x0, x1, y0, y1 = (float(v) for v in bounds)
    dev = L.device()
    arr, keep = _classify.curve_array([curve])
    tabs = _classify.cell_tables(q)
    bp1 = L.dev(np.array([x0, x1]), torch.float64)
    bp2 = L.dev(np.array([y0, y1]), torch.float64)
    el = torch.zeros(2, dtype=torch.int32, device=dev)
    m = (q + 1) ** 2
    cap = _DECOMP_CELLS * m
    sP = torch.empty(2 * cap, dtype=torch.float64, device=dev)
    sW = torch.empty(cap, dtype=torch.float64, device=dev)
    ptr = torch.zeros(2, dtype=torch.int64, device=dev)
    nc = torch.zeros(1, dtype=torch.int32, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    L.call("tq_cutcell_device_slots", arr, 1, L.ptr(bp1), L.ptr(bp2), L.ptr(el), 1, q, tabs.ctypes.data_as(L.vp),
           cap, L.ptr(sP), L.ptr(sW), L.ptr(ptr), L.ptr(nc), L.ptr(st), L.stream())
    status, npts, ncells = int(st.item()), int(ptr[1].item()), int(nc.item())
    if status:
        raise TrimmingConfigurationError(_classify._CUT_ERRORS.get(status, "decomposition failed"))
    if npts > cap or npts != ncells * m:
        raise RuntimeError(f"cut-cell decomposition returned {npts} points for {ncells} cells")
    P = sP[:2 * npts].reshape(npts, 2).cpu().numpy()
    W = sW[:npts].cpu().numpy()
    return [SubCell("cell", P[k * m:(k + 1) * m], W[k * m:(k + 1) * m]) for k in range(ncells)]


def cut_cell_quadrature(config, q):
    """Quadrature of every cut element of a configuration (src/trimming.py:1084-1111):
    1 <= q <= 6 as in the reference (the formation path itself calls
    ``config.cut_cell_rule`` without that cap), decomposed on the
    device."""
    if q < 1 or q > 6:
        raise ValueError("Lagrange degree q must be within 1..6")
    return config.cut_cell_rule(q, cache=False)


def _dwq_info(config, i1, i2):
    """src/trimming.py:545-586 through tq_dwq_route (fclass.cu k_dwq_route)."""
    b1, b2 = config.basis2d.dir
    n2 = b2.n
    u1, u2 = config.u_disc
    dev = L.device()
    du1 = L.dev(u1 if u1.size else np.zeros(1), torch.float64)
    du2 = L.dev(u2 if u2.size else np.zeros(1), torch.float64)
    rows = torch.tensor([i1 * n2 + i2], dtype=torch.int32, device=dev)
    out = torch.empty(8, dtype=torch.int32, device=dev)
    L.call("tq_dwq_route", b1.device(), b2.device(), L.ptr(config.element_class_dev), L.ptr(du1), u1.size,
           L.ptr(du2), u2.size, L.ptr(rows), 1, L.ptr(out), L.stream())
    r = [int(v) for v in out.cpu().tolist()]
    reg, cut = config.support_split(i1, i2)
    if r[0] == 0:
        return DwqInfo(False, (None, None), None, (None, None), reg, cut)
    if r[3] < 0:
        return DwqInfo(True, (None, None), None, (None, None), reg, cut)
    box = ((r[3], r[4]), (r[5], r[6]))
    used, sides = [], []
    for iu, ud, basis, (lo, _hi) in ((r[1], u1, b1, box[0]), (r[2], u2, b2, box[1])):
        if iu < 0:
            used.append(None)
            sides.append(None)
            continue
        u = float(ud[iu])
        k = int(np.argmin(np.abs(basis.breakpoints - u)))
        used.append(u)
        sides.append("right" if lo == k else "left")
    residual = [(f1, f2) for (f1, f2) in reg
                if not (box[0][0] <= f1 <= box[0][1] and box[1][0] <= f2 <= box[1][1])]
    return DwqInfo(True, tuple(used), box, tuple(sides), residual, cut)


def classify_elements(basis2d: TensorBasis2D, curves) -> TrimConfiguration:
    """Classify elements and functions on the GPU (src/trimming.py:607-733).
    Reference-built bases and catalog curves are accepted (``_adapt``); a
    curve the device cannot evaluate raises TypeError."""
    from . import _adapt
    basis2d = _adapt.basis2d(basis2d)
    src = list(curves)
    curves, known = _adapt.curves(src)
    if not known:
        bad = [type(c).__name__ for c in src if _adapt.curve(c) is None]
        raise TypeError(f"curves {bad} cannot be evaluated on the device; classify with the reference's "
                        "classify_elements and pass that configuration to the formation entry points")
    b1, b2 = basis2d.dir
    if curves:
        from . import _classify
        ec = _classify.classify_device(basis2d, curves)
    else:
        ec = torch.full((b1.num_elements, b2.num_elements), INTERIOR, dtype=torch.int8, device=L.device())
    return configuration_from_classes(basis2d, curves, ec)


def configuration_from_classes(basis2d: TensorBasis2D, curves, element_class) -> TrimConfiguration:
    """Function classes, discontinuity faces and the configuration from
    element classes (device int8 nel1 x nel2, or a host array that is
    uploaded): src/trimming.py:431-484 on the GPU (tq_function_classes)."""
    b1, b2 = basis2d.dir
    dev = L.device()
    nel1, nel2 = b1.num_elements, b2.num_elements
    n1, n2 = basis2d.shape
    if not isinstance(element_class, torch.Tensor):
        ec_h = np.asarray(element_class)
        if ec_h.shape != (nel1, nel2):
            raise ValueError(f"element classes of shape {ec_h.shape} for a {nel1} x {nel2} mesh")
        element_class = L.dev(ec_h.astype(np.int8), torch.int8)
    ec = element_class.reshape(nel1, nel2)
    fc = torch.empty((n1, n2), dtype=torch.int8, device=dev)
    face1 = torch.zeros(max(nel1 - 1, 1), dtype=torch.int32, device=dev)
    face2 = torch.zeros(max(nel2 - 1, 1), dtype=torch.int32, device=dev)
    L.call("tq_function_classes", b1.device(), b2.device(), L.ptr(ec), L.ptr(fc), L.ptr(face1),
           L.ptr(face2), L.stream())
    f1 = face1.cpu().numpy()[: max(nel1 - 1, 0)] != 0
    f2 = face2.cpu().numpy()[: max(nel2 - 1, 0)] != 0
    return TrimConfiguration(basis2d, curves, ec, fc, f1, f2)


def __getattr__(name):
    # the reference's name for the cut-cell rule container (src/trimming.py:749-766)
    if name == "CutCellQuadrature":
        from ._classify import CutCellRule
        return CutCellRule
    raise AttributeError(name)
