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
        if pending is not None:           # started by cut_cell_rule_async
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
        if self.element_class_dev is not None and self.element_class_dev.is_cuda:
            return          # decomposed on the device on first use (tq_cutcell_device)
        from . import _classify
        self._cut_pending[q] = _classify.submit(_classify.cut_cell_rule, self, q, True)

    def support_split(self, i1, i2):
        a1, b1, a2, b2 = self.support_block(i1, i2)
        blk = self.element_class[a1: b1 + 1, a2: b2 + 1]
        reg = [(a1 + r, a2 + c) for r, c in zip(*np.nonzero(blk == INTERIOR))]
        cut = [(a1 + r, a2 + c) for r, c in zip(*np.nonzero(blk == CUT))]
        return reg, cut


# ---------------------------------------------------------------------------
# trimming curves: descriptors for the device classifier / host decomposition
# (src/trimming.py:69-351 and the harness closed curves)
# ---------------------------------------------------------------------------

class TrimmingCurve:
    """Oriented curve; the valid domain lies to the left (src/trimming.py:69-95)."""
    straight = False
    closed = False

    def sample(self, n=257):
        return self.evaluate(np.linspace(0.0, 1.0, n))

    def descriptor(self):
        raise NotImplementedError


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


def classify_elements(basis2d: TensorBasis2D, curves) -> TrimConfiguration:
    """Classify elements and functions on the GPU (src/trimming.py:607-733)."""
    curves = list(curves)
    b1, b2 = basis2d.dir
    dev = L.device()
    nel1, nel2 = b1.num_elements, b2.num_elements
    n1, n2 = basis2d.shape
    if curves:
        from . import _classify
        ec = _classify.classify_device(basis2d, curves)
    else:
        ec = torch.full((nel1, nel2), INTERIOR, dtype=torch.int8, device=dev)
    fc = torch.empty((n1, n2), dtype=torch.int8, device=dev)
    face1 = torch.zeros(max(nel1 - 1, 1), dtype=torch.int32, device=dev)
    face2 = torch.zeros(max(nel2 - 1, 1), dtype=torch.int32, device=dev)
    fn = L.optional("tq_function_classes", [L.Space1D, L.Space1D, L.vp, L.vp, L.vp, L.vp, L.vp])
    if fn is None:
        raise RuntimeError("native library lacks tq_function_classes")
    L.call("tq_function_classes", b1.device(), b2.device(), L.ptr(ec), L.ptr(fc), L.ptr(face1),
           L.ptr(face2), L.stream())
    f1 = face1.cpu().numpy()[: max(nel1 - 1, 0)] != 0
    f2 = face2.cpu().numpy()[: max(nel2 - 1, 0)] != 0
    return TrimConfiguration(basis2d, curves, ec, fc, f1, f2)
