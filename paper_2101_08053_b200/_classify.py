"""Curve descriptors -> tq_curve, GPU classification and host cut-cell rules."""

from __future__ import annotations

import ctypes as C
from functools import lru_cache

import numpy as np
import torch

from . import _lib as L
from ._lib import TrimmingConfigurationError

TQ_CURVE_LINE, TQ_CURVE_ARC, TQ_CURVE_CLOSED_CIRCLE, TQ_CURVE_BEZIER, TQ_CURVE_BSPLINE = 1, 2, 3, 4, 5


def curve_array(curves):
    """ctypes array of tq_curve with host data (kept alive by the return)."""
    keep = []
    arr = (L.Curve * max(len(curves), 1))()
    for k, cv in enumerate(curves):
        kind, m, data = cv.descriptor()
        data = np.ascontiguousarray(data, dtype=np.float64)
        keep.append(data)
        arr[k] = L.Curve(kind, m, data.ctypes.data_as(L.vp))
    return arr, keep


def classify_device(basis2d, curves):
    b1, b2 = basis2d.dir
    arr, keep = curve_array(curves)
    ec = torch.empty((b1.num_elements, b2.num_elements), dtype=torch.int8, device=L.device())
    status = torch.zeros(1, dtype=torch.int32, device=L.device())
    fn = L.optional("tq_classify_elements", [C.POINTER(L.Curve), L.i32, L.Space1D, L.Space1D, L.vp, L.vp, L.vp])
    L.call("tq_classify_elements", arr, len(curves), b1.device(), b2.device(), L.ptr(ec), L.ptr(status),
           L.stream())
    return ec


@lru_cache(maxsize=None)
def cell_tables(q):
    """Lobatto nodes, Gauss rule on [0,1] and Lagrange tables, computed the
    way the reference does (src/trimming.py:769-798)."""
    if q == 1:
        x = np.array([-1.0, 1.0])
    else:
        c = np.zeros(q + 1)
        c[q] = 1.0
        x = np.concatenate([[-1.0], np.polynomial.legendre.legroots(np.polynomial.legendre.legder(c)), [1.0]])
    nodes = 0.5 * (x + 1.0)
    gx, gw = np.polynomial.legendre.leggauss(q + 1)
    xi, wx = 0.5 * (gx + 1.0), 0.5 * gw
    V = np.vander(nodes, q + 1, increasing=True)
    co = np.linalg.solve(V, np.eye(q + 1))
    Lt = np.vander(xi, q + 1, increasing=True) @ co
    dco = co[1:, :] * np.arange(1, q + 1)[:, None]
    dLt = np.vander(xi, q, increasing=True) @ dco
    return np.concatenate([nodes, xi, wx, Lt.ravel(), dLt.ravel()])


class CutCellRule:
    """Cut-element quadrature (src/trimming.py:749-766) with packed arrays.
    A rule decomposed on the device keeps its arrays there (``dev``); the
    host copies are made on first use."""

    def __init__(self, q, elements, ptr, pts, wts, ncells, dev=None):
        self.q = q
        self.elements = elements          # (ncut, 2) row-major element order
        self._host = None if dev is not None else (ptr, pts, wts, ncells)
        self.dev = dev
        self._npts = int(ptr[-1]) if dev is None else dev["npts"]
        self._rules = None
        self._counts = None

    def _h(self):
        if self._host is None:
            d = self.dev
            self._host = (d["ptr"].cpu().numpy(), d["P"].cpu().numpy(), d["W"].cpu().numpy(),
                          d["ncells"].cpu().numpy())
        return self._host

    @property
    def ptr(self):                        # (ncut+1) int64
        return self._h()[0]

    @property
    def points(self):                     # (P, 2)
        return self._h()[1]

    @property
    def weights(self):                    # (P,)
        return self._h()[2]

    @property
    def _ncells(self):
        return self._h()[3]

    @property
    def rules(self):
        """{(e1, e2): (points, weights)} views (built on first use)."""
        if self._rules is None:
            pts, wts, ptr = self.points, self.weights, self.ptr
            self._rules = {(int(e1), int(e2)): (pts[ptr[k]:ptr[k + 1]], wts[ptr[k]:ptr[k + 1]])
                           for k, (e1, e2) in enumerate(self.elements)}
        return self._rules

    @property
    def subcell_counts(self):
        if self._counts is None:
            self._counts = {(int(e1), int(e2)): int(n) for (e1, e2), n in zip(self.elements, self._ncells)}
        return self._counts

    def element_rule(self, e1, e2):
        return self.rules[(e1, e2)]

    def total_points(self):
        return self._npts

    def all_points(self):
        return self.points


_POOL = None


def _worker_init():
    """The worker's OpenMP team leaves two cores to the launching thread
    (nthreads is a per-thread setting of the OpenMP runtime)."""
    import os
    try:
        gomp = C.CDLL("libgomp.so.1")
        gomp.omp_set_num_threads(max(1, len(os.sched_getaffinity(0)) - 2))
    except OSError:
        pass


def submit(fn, *args):
    """Run ``fn(*args)`` on the module's worker thread (host geometry)."""
    global _POOL
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(max_workers=1, thread_name_prefix="tq-cutcells", initializer=_worker_init)
    return _POOL.submit(fn, *args)


_CUT_ERRORS = {1: "cannot decompose cell at maximum split depth 4", 2: "folded sub-cell",
               3: "cell is not crossed by exactly one curve", 4: "cut-cell capacity exceeded"}


# slot capacity of the single-decomposition schedule, in sub-cells of
# (q+1)^2 points (config 5 averages 1.7 sub-cells per cut element)
SLOT_CELLS = 4


class _DeviceRulePending:
    """A device cut-cell decomposition in flight (start_cut_cell_rule_device):
    the slots kernel is queued and its summary is on its way to pinned host
    memory; ``result()`` waits for that copy and packs the rule."""

    def __init__(self, config, q, slot_cells=None):
        if q < 1:
            raise ValueError("Lagrange degree q must be >= 1")
        b1, b2 = config.basis2d.dir
        ec = config.element_class_dev.reshape(b1.num_elements, b2.num_elements)
        el = torch.nonzero(ec == 1).to(torch.int32).contiguous()
        ncut = el.shape[0]
        dev = el.device
        arr, keep = curve_array(config.curves)
        tabs = cell_tables(q)
        bp1, bp2 = b1.device_arrays()["bp"], b2.device_arrays()["bp"]
        cap = (SLOT_CELLS if slot_cells is None else slot_cells) * (q + 1) ** 2
        ptr = torch.zeros(ncut + 1, dtype=torch.int64, device=dev)
        ncells = torch.zeros(max(ncut, 1), dtype=torch.int32, device=dev)
        status = torch.zeros(max(ncut, 1), dtype=torch.int32, device=dev)
        sP = torch.empty(max(ncut, 1) * cap * 2, dtype=torch.float64, device=dev)
        sW = torch.empty(max(ncut, 1) * cap, dtype=torch.float64, device=dev)
        common = (arr, len(config.curves), L.ptr(bp1), L.ptr(bp2), L.ptr(el), ncut, q, tabs.ctypes.data_as(L.vp), cap)
        L.call("tq_cutcell_device_slots", *common, L.ptr(sP), L.ptr(sW), L.ptr(ptr), L.ptr(ncells), L.ptr(status),
               L.stream())
        self.summary = self.event = None
        if ncut:
            cnt = ptr[1:]
            summary = torch.stack([status[:ncut].max().to(torch.int64), cnt.max(), cnt.sum()])
            self.summary = torch.empty(3, dtype=torch.int64, pin_memory=True)
            self.summary.copy_(summary, non_blocking=True)
            self.event = torch.cuda.Event()
            self.event.record()
        self.el_host = torch.empty(el.shape, dtype=torch.int32, pin_memory=True)
        self.el_host.copy_(el, non_blocking=True)
        self.el_event = torch.cuda.Event()
        self.el_event.record()
        self.s = dict(q=q, el=el, ncut=ncut, common=common, keep=(keep, tabs, bp1, bp2), cap=cap, ptr=ptr,
                      ncells=ncells, status=status, sP=sP, sW=sW)

    def result(self):
        s = self.s
        q, el, ncut, cap, ptr, status = s["q"], s["el"], s["ncut"], s["cap"], s["ptr"], s["status"]
        over = 0
        if ncut:
            self.event.synchronize()
            summary = self.summary.tolist()
            if summary[0]:
                bad = torch.nonzero(status[:ncut]).flatten()
                z = int(bad[0])
                e1, e2 = (int(v) for v in el[z].tolist())
                raise TrimmingConfigurationError(f"element ({e1}, {e2}): {_CUT_ERRORS.get(int(status[z]), 'error')}")
            over = int(summary[1] > cap)
            ptr[1:] = torch.cumsum(ptr[1:], 0)
            npts = int(summary[2])
        else:
            npts = 0
        dev = el.device
        P = torch.empty((max(npts, 1), 2), dtype=torch.float64, device=dev)
        W = torch.empty(max(npts, 1), dtype=torch.float64, device=dev)
        L.call("tq_cutcell_device_pack", *s["common"], L.ptr(s["sP"]), L.ptr(s["sW"]), L.ptr(ptr), L.ptr(P), L.ptr(W),
               over, L.stream())
        self.el_event.synchronize()
        elements = self.el_host.numpy().astype(np.int64).reshape(-1, 2)
        return CutCellRule(q, elements, None, None, None, None,
                           dev=dict(P=P[:npts], W=W[:npts], ptr=ptr, el=el, ncells=s["ncells"][:ncut], npts=npts))


def start_cut_cell_rule_device(config, q, slot_cells=None):
    """Queue the device decomposition and return at once; ``.result()``
    joins (called by TrimConfiguration.cut_cell_rule).  The kernel and its
    read-back then overlap the host's plan building of the formation."""
    return _DeviceRulePending(config, q, slot_cells)


def cut_cell_rule_device(config, q, slot_cells=None):
    """Cut-element quadrature decomposed on the GPU (one thread per cut
    element; same decomposition as the host C++): one decomposition into
    fixed-capacity slots (tq_cutcell_device_slots), one read-back of the
    status and point count, then the slots are packed to their offsets
    (tq_cutcell_device_pack; overflowing elements are decomposed again).
    The rule's device arrays are kept on it (``rule.dev``)."""
    return _DeviceRulePending(config, q, slot_cells).result()


def cut_cell_rule(config, q, host_only=False):
    """Cut-element quadrature of the configuration.  On the device when the
    classes live there (tq_cutcell_device); ``host_only`` (worker threads,
    host-only configurations) runs the host C++ decomposition."""
    if q < 1:
        raise ValueError("Lagrange degree q must be >= 1")
    if not host_only and getattr(config, "element_class_dev", None) is not None:
        return cut_cell_rule_device(config, q)
    b1, b2 = config.basis2d.dir
    # cut elements (class 1) in row-major order (found on the device when the
    # classes live there; host-only configurations use the host array)
    dev = None if host_only else getattr(config, "element_class_dev", None)
    if dev is not None:
        nz = torch.nonzero(dev.reshape(config.num_elements) == 1)
        el = np.ascontiguousarray(nz.to(torch.int32).cpu().numpy()).reshape(-1, 2)
    else:
        e1, e2 = np.nonzero(config.element_class == 1)
        el = np.ascontiguousarray(np.column_stack([e1, e2]).astype(np.int32))
    arr, keep = curve_array(config.curves)
    tabs = cell_tables(q)
    bp1 = np.ascontiguousarray(b1.breakpoints, dtype=np.float64)
    bp2 = np.ascontiguousarray(b2.breakpoints, dtype=np.float64)
    lib = L.lib()
    build = lib.tq_cutcell_build
    build.argtypes = [C.POINTER(L.Curve), L.i32, L.vp, L.i32, L.vp, L.i32, L.vp, L.i32, L.i32, L.vp,
                      C.POINTER(L.i32)]
    build.restype = L.vp
    st = L.i32(0)
    h = build(arr, len(config.curves), bp1.ctypes.data_as(L.vp), b1.num_elements, bp2.ctypes.data_as(L.vp),
              b2.num_elements, el.ctypes.data_as(L.vp), el.shape[0], q, tabs.ctypes.data_as(L.vp), C.byref(st))
    if not h:
        msg = lib.tq_last_error().decode(errors="replace")
        raise L._EXC.get(st.value, RuntimeError)(msg)
    lib.tq_cutcell_npoints.argtypes = [L.vp]
    lib.tq_cutcell_npoints.restype = L.i64
    npts = lib.tq_cutcell_npoints(h)
    ptr = np.empty(el.shape[0] + 1, np.int64)
    P = np.empty((npts, 2))
    W = np.empty(npts)
    nc = np.empty(el.shape[0], np.int32)
    lib.tq_cutcell_copy.argtypes = [L.vp, L.vp, L.vp, L.vp, L.vp]
    lib.tq_cutcell_copy(h, ptr.ctypes.data_as(L.vp), P.ctypes.data_as(L.vp), W.ctypes.data_as(L.vp),
                        nc.ctypes.data_as(L.vp))
    lib.tq_cutcell_free.argtypes = [L.vp]
    lib.tq_cutcell_free(h)
    return CutCellRule(q, el.astype(np.int64), ptr, P, W, nc)
