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
        self.element_class = element_class_dev.cpu().numpy()
        self.func_class = func_class_dev.cpu().numpy()
        b1, b2 = basis2d.dir
        self.u_disc = (np.asarray(b1.breakpoints[1:-1][face1], dtype=float),
                       np.asarray(b2.breakpoints[1:-1][face2], dtype=float))
        self._cut_rules = {}
        self._dwq_cache = {}
        self._active = None
        self._cum_int = None

    @property
    def num_elements(self):
        return self.element_class.shape

    def element_bounds(self, e1, e2):
        bp1 = self.basis2d.dir[0].breakpoints
        bp2 = self.basis2d.dir[1].breakpoints
        return float(bp1[e1]), float(bp1[e1 + 1]), float(bp2[e2]), float(bp2[e2 + 1])

    @property
    def cut_elements(self):
        e1, e2 = np.nonzero(self.element_class == CUT)
        return list(zip(e1.tolist(), e2.tolist()))

    @property
    def interior_elements(self):
        e1, e2 = np.nonzero(self.element_class == INTERIOR)
        return list(zip(e1.tolist(), e2.tolist()))

    def active_functions(self):
        """src/trimming.py:514-517 (row-major), from the device index."""
        idx, _ = self.active_index()
        act = idx["active"][: idx["K"]].cpu().numpy().astype(np.int64)
        n2 = self.basis2d.shape[1]
        return np.column_stack([act // n2, act % n2])

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

    def support_split(self, i1, i2):
        a1, b1, a2, b2 = self.support_block(i1, i2)
        blk = self.element_class[a1: b1 + 1, a2: b2 + 1]
        reg = [(a1 + r, a2 + c) for r, c in zip(*np.nonzero(blk == INTERIOR))]
        cut = [(a1 + r, a2 + c) for r, c in zip(*np.nonzero(blk == CUT))]
        return reg, cut


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
