"""ctypes binding of the C ABI in ``include/trimquad_b200.h``.

The library is built in-tree (``paper_2101_08053_b200/libtq_b200.so``).  There
is no CPU fallback: importing a formation entry point without the library or
without a CUDA device raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TQ_LIB") or os.path.join(HERE, "libtq_b200.so")   # TQ_LIB: A/B builds

TQ_OK, TQ_EINVAL, TQ_ERULE, TQ_ETRIM, TQ_EPATTERN, TQ_ECUDA, TQ_EOVERFLOW = range(7)
INTERIOR, CUT, EXTERIOR = 0, 1, 2


class RuleConstructionError(RuntimeError):
    """A weight row cannot satisfy its moment system (src/quadrature.py:46-47)."""


class TrimmingConfigurationError(RuntimeError):
    """Trimming layout outside the supported catalog (src/trimming.py:49-50)."""


class NativeError(RuntimeError):
    """CUDA / native failure."""


_EXC = {TQ_EINVAL: ValueError, TQ_ERULE: RuleConstructionError, TQ_ETRIM: TrimmingConfigurationError,
        TQ_EPATTERN: RuntimeError, TQ_ECUDA: NativeError, TQ_EOVERFLOW: OverflowError}

vp = C.c_void_p
i32, i64, f64 = C.c_int32, C.c_int64, C.c_double


class Space1D(C.Structure):
    _fields_ = [("knots", vp), ("bp", vp), ("espan", vp), ("el_first", vp), ("el_last", vp),
                ("ov_lo", vp), ("ov_hi", vp), ("nknots", i32), ("p", i32), ("n", i32), ("nel", i32)]


class Layout(C.Structure):
    _fields_ = [("pts", vp), ("offsets", vp), ("npts", i32), ("nel", i32)]


class Rules(C.Structure):
    _fields_ = [("wptr", vp), ("k0", vp), ("w", vp)]


class Curve(C.Structure):
    _fields_ = [("kind", i32), ("m", i32), ("data", vp)]


FIT_MAX_SETS = 16      # TQ_FIT_MAX_SETS


class FitSet(C.Structure):
    _fields_ = [("s", Space1D), ("lay", Layout), ("rows", vp), ("nrows", i32), ("wptr", vp), ("k0", vp),
                ("w", vp), ("fail", vp), ("products", vp)]


class FitBatch(C.Structure):
    _fields_ = [("set", FitSet * FIT_MAX_SETS), ("nsets", i32), ("start", i32 * (FIT_MAX_SETS + 1)),
                ("gx", vp), ("gw", vp)]


class CombineSet(C.Structure):
    _fields_ = [("rows", vp), ("nrows", i32), ("colptr", vp), ("rowidx", vp), ("sval", vp), ("fine", Rules),
                ("out", Rules)]


class CombineBatch(C.Structure):
    _fields_ = [("set", CombineSet * FIT_MAX_SETS), ("nsets", i32), ("start", i32 * (FIT_MAX_SETS + 1))]


EVAL_MAX_TASKS = 16    # TQ_EVAL_MAX_TASKS


class EvalTask(C.Structure):
    _fields_ = [("s", Space1D), ("u", vp), ("n", i64), ("first", vp), ("vals", vp)]


class EvalBatch(C.Structure):
    _fields_ = [("task", EvalTask * EVAL_MAX_TASKS), ("ntasks", i32), ("block_start", i32 * (EVAL_MAX_TASKS + 1)),
                ("stage_bytes", i32)]


def eval_many(jobs):
    """[(basis, device points)] -> [(first, vals)]: one launch per degree
    (and per EVAL_MAX_TASKS jobs) of tq_basis_eval_multi."""
    outs = [None] * len(jobs)
    by_p = {}
    for k, (basis, u) in enumerate(jobs):
        by_p.setdefault(basis.p, []).append(k)
    for ks in by_p.values():
        for c0 in range(0, len(ks), EVAL_MAX_TASKS):
            chunk = ks[c0: c0 + EVAL_MAX_TASKS]
            batch = EvalBatch()
            for slot, k in enumerate(chunk):
                basis, u = jobs[k]
                n = u.numel()
                first = torch.empty(n, dtype=torch.int32, device=u.device)
                vals = torch.empty((n, basis.p + 1), dtype=torch.float64, device=u.device)
                outs[k] = (first, vals)
                batch.task[slot] = EvalTask(basis.device(), ptr(u), n, ptr(first), ptr(vals))
            batch.ntasks = len(chunk)
            call("tq_basis_eval_multi", C.byref(batch), stream())
    return outs


class Coeff(C.Structure):
    _fields_ = [("kind", i32), ("p", i32), ("n", i32), ("knots", vp), ("X", vp), ("Y", vp)]


class RowCtx(C.Structure):
    _fields_ = [("n1", i32), ("n2", i32), ("p1", i32), ("p2", i32),
                ("ov_lo1", vp), ("ov_hi1", vp), ("ov_lo2", vp), ("ov_hi2", vp),
                ("col_of", vp), ("active", vp), ("slot", vp), ("a1", vp), ("a2", vp), ("raw", vp),
                ("deep", vp), ("rowfast", vp), ("row_begin", i32), ("row_end", i32), ("counts", vp), ("tiles", vp),
                ("raw_ld", i64), ("fclass", vp), ("pos", vp)]


_lib = None


def lib():
    """Load the native library (once).  Fails loudly: no fallback exists."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"native library missing: {LIB_PATH} (run __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    sig = {
        "tq_version": ([], i32),
        "tq_pool_keep": ([i32], i32),
        "tq_graph_instantiate": ([vp, i32, C.POINTER(vp)], i32),
        "tq_graph_launch": ([vp, vp], i32),
        "tq_graph_exec_destroy": ([vp], i32),
        "tq_graph_node_priorities": ([vp, C.POINTER(i32), C.POINTER(i32)], i32),
        "tq_graph_node_types": ([vp, C.POINTER(i32)], i32),
        "tq_last_error": ([], C.c_char_p),
        "tq_device_sync": ([vp], i32),
        "tq_debug_stamp": ([vp, i32, vp], i32),
        "tq_basis_eval": ([Space1D, vp, i64, vp, vp, vp, vp, vp], i32),
        "tq_moments_1d_g": ([Space1D, vp, vp, i32, vp, vp], i32),
        "tq_wq_solve": ([Space1D, Layout, vp, vp, vp, vp, i32, i32, i32, vp, vp, vp, vp, vp, vp], i32),
        "tq_dwq_combine": ([vp, i32, vp, vp, vp, Rules, Rules, vp], i32),
        "tq_wq_products": ([Space1D, Layout, vp, vp, Rules, vp, vp], i32),
        "tq_row_counts": ([RowCtx, vp, vp], i32),
        "tq_row_counts_deep": ([RowCtx, vp, vp, vp], i32),
        "tq_row_counts_geo": ([RowCtx, vp, vp, vp, vp, vp], i32),
        "tq_row_counts_rest": ([RowCtx, vp, vp, vp], i32),
        "tq_list_record_bytes": ([], i64),
        "tq_list_geometry": ([RowCtx, vp, vp, vp], i32),
        "tq_row_counts_rest_rec": ([RowCtx, vp, vp, vp, vp], i32),
        "tq_row_counts_spec": ([RowCtx, vp, vp, vp, vp], i32),
        "tq_row_counts_cached": ([RowCtx, vp, vp, vp, vp, vp, vp, vp, vp], i32),
        "tq_row_counts_verify": ([RowCtx, vp, vp, vp, vp, vp, vp], i32),
        "tq_scan_indptr": ([vp, i32, vp, C.POINTER(i64), vp], i32),
        "tq_scan_workspace_bytes": ([i32], i64),
        "tq_scan_indptr_ws": ([vp, i32, vp, vp, C.POINTER(i64), vp], i32),
        "tq_fill_rows": ([RowCtx, vp, vp, vp, vp], i32),
        "tq_scan_tiles": ([RowCtx, vp, C.POINTER(i64), vp], i32),
        "tq_tiles_expect": ([RowCtx, i64, vp], i32),
        "tq_scan_tiles_early": ([RowCtx, i64, i32, vp], i32),
        "tq_fill_fast_part": ([RowCtx, vp, vp, vp, i32, i32, vp], i32),
        "tq_fill_fast": ([RowCtx, vp, vp, vp, vp], i32),
        "tq_fill_listed": ([RowCtx, vp, vp, vp, vp, vp], i32),
        "tq_active_index": ([vp, i64, vp, vp, C.POINTER(i32), vp], i32),
        "tq_deep_flags": ([RowCtx, vp, vp, i32, vp, vp], i32),
        "tq_deep_geometry": ([RowCtx, vp, vp, i32, vp, vp], i32),
        "tq_deep_apply": ([RowCtx, vp, vp, vp], i32),
        "tq_csr_diag": ([vp, vp, vp, i32, vp, vp], i32),
        "tq_spmv": ([vp, vp, vp, i32, vp, vp, vp, vp, vp], i32),
        "tq_cg_workspace_bytes": ([i32], i64),
        "tq_cg_scaled": ([vp, vp, vp, i32, vp, vp, vp, C.c_double, i32, vp, vp, vp, vp], i32),
        "tq_cutcell_device": ([C.POINTER(Curve), i32, vp, vp, vp, i32, i32, vp, vp, vp, vp, vp, vp, vp], i32),
        "tq_cutcell_device_slots": ([C.POINTER(Curve), i32, vp, vp, vp, i32, i32, vp, i64, vp, vp, vp, vp, vp,
                                     vp], i32),
        "tq_cutcell_device_pack": ([C.POINTER(Curve), i32, vp, vp, vp, i32, i32, vp, i64, vp, vp, vp, vp, vp, i32,
                                    vp], i32),
        "tq_dwq_route": ([Space1D, Space1D, vp, vp, i32, vp, i32, vp, i32, vp, vp], i32),
        "tq_function_classes": ([Space1D, Space1D, vp, vp, vp, vp, vp], i32),
        "tq_wq_fit_sets": ([C.POINTER(FitBatch), i32, i32, vp], i32),
        "tq_dwq_combine_sets": ([C.POINTER(CombineBatch), vp], i32),
        "tq_basis_eval_multi": ([C.POINTER(EvalBatch), vp], i32),
        "tq_mass_1d_mixed": ([Space1D, Space1D, vp, vp, i32, vp, vp], i32),
        "tq_curve_eval": ([C.POINTER(Curve), i32, vp, i64, vp, vp], i32),
        "tq_curve_intersect_line": ([C.POINTER(Curve), i32, f64, i32, vp, vp, vp, vp], i32),
        "tq_sum_factor_rows": ([i32, vp, vp, vp, vp, vp, vp, vp], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def optional(name, args, res=i32):
    """Bind an entry point added after the first release (absent -> None)."""
    L = lib()
    fn = getattr(L, name, None)
    if fn is not None:
        fn.argtypes = args
        fn.restype = res
    return fn


def call(name, *args):
    fn = getattr(lib(), name)
    rc = fn(*args)
    if rc != TQ_OK:
        msg = lib().tq_last_error().decode(errors="replace")
        raise _EXC.get(rc, RuntimeError)(f"{name}: {msg}")


class Stamps:
    """Timeline probe (TQ_STAMPS=1): device global-timer stamps recorded in
    stream order at named points; ``report()`` gives µs from the first."""

    def __init__(self, n=1024):
        self.buf = torch.zeros(n, dtype=torch.int64, device=device())
        self.names = []

    def __call__(self, name):
        self.names.append(name)
        call("tq_debug_stamp", ptr(self.buf), len(self.names) - 1, stream())

    def report(self):
        t = self.buf[:len(self.names)].cpu().numpy()
        return {n: (int(v) - int(t[0])) / 1e3 for n, v in zip(self.names, t)}


_POOLS_KEPT = set()
_HAVE_CUDA = []


def device():
    if not _HAVE_CUDA:        # (torch.cuda.is_available queries NVML: once per process)
        if not torch.cuda.is_available():
            raise RuntimeError("trimquad_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists")
        _HAVE_CUDA.append(True)
    d = torch.cuda.current_device()
    if d not in _POOLS_KEPT:      # once per device: freed scratch stays in the stream-ordered pool
        _POOLS_KEPT.add(d)
        lib().tq_pool_keep(d)
    return torch.device("cuda", d)


def stream():
    return vp(torch.cuda.current_stream().cuda_stream)


def tile_pad(nrows):
    """TQ_TILE_PAD of the header: tile sums (padded), then the bases."""
    return ((nrows + 31) // 32 + 3) // 4 * 4


def tile_ctl(nrows):
    """TQ_TILE_CTL: first control word of a tile-mode buffer."""
    return tile_pad(nrows) + 2 * ((nrows + 31) // 32) + 2


def tile_ints(nrows):
    """TQ_TILE_INTS: ints of a tile-mode buffer (tq_rowctx.tiles): sums |
    bases, total, overflow | early bases | nine control words."""
    return tile_pad(nrows) + 2 * ((nrows + 31) // 32) + 11


def ptr(t):
    return vp(t.data_ptr()) if t is not None else vp(0)


_pinned_keep = []
_NP_DTYPE = {torch.float64: np.float64, torch.float32: np.float32, torch.int64: np.int64,
             torch.int32: np.int32, torch.int8: np.int8, torch.uint8: np.uint8, torch.int16: np.int16}
_PAGEABLE_UPLOADS = os.environ.get("TQ_PAGEABLE_UPLOADS", "0") == "1"     # A/B knob


class _StagingRing:
    """Pinned host ring for small uploads: the array is written into the
    next free slot and copied from there (no per-upload pinned allocation).
    A slot is reused only after the copy that read it has run: an event per
    use, and a new lap of the ring waits for every copy of the previous one."""

    SIZE = 8 << 20

    def __init__(self):
        import collections
        self.buf = torch.empty(self.SIZE, dtype=torch.uint8, pin_memory=True)
        self.host = self.buf.numpy()
        self.head = 0
        self.pending = collections.deque()       # events of this lap's copies

    def stage(self, a):
        n = (a.nbytes + 255) & ~255
        if n > self.SIZE // 4:
            return None
        if self.head + n > self.SIZE:
            # a new lap: every copy of the previous one must have run (rare:
            # 8 MB of small uploads per lap); within a lap slots never overlap
            while self.pending:
                self.pending.popleft().synchronize()
            self.head = 0
        while self.pending and self.pending[0].query():
            self.pending.popleft()
        lo = self.head
        self.host[lo: lo + a.nbytes] = a.reshape(-1).view(np.uint8)
        self.head = lo + n
        return self.buf[lo: lo + a.nbytes]

    def reserve(self, n):
        """Offset of n free bytes (256-aligned) in the ring, or None."""
        n = (n + 255) & ~255
        if n > self.SIZE // 4:
            return None
        if self.head + n > self.SIZE:
            while self.pending:
                self.pending.popleft().synchronize()
            self.head = 0
        while self.pending and self.pending[0].query():
            self.pending.popleft()
        lo = self.head
        self.head = lo + n
        return lo

    def done(self, view):
        ev = torch.cuda.Event()
        ev.record()
        self.pending.append(ev)


_RINGS = {}


def dev(x, dtype):
    """Upload a host array (numpy) as a contiguous device tensor, copied
    asynchronously on the current stream (no host sync).  Small arrays go
    through a pinned staging ring (_StagingRing); larger ones are staged in
    pinned memory from torch's caching host allocator, which keeps the block
    until the copy has run.  Under CUDA stream capture the pinned source is
    kept alive for good (every replay reads it again)."""
    a = np.ascontiguousarray(x, dtype=_NP_DTYPE.get(dtype))
    if a.size == 0:
        return torch.empty(a.shape, dtype=dtype, device=device())
    capturing = torch.cuda.is_current_stream_capturing()
    if _PAGEABLE_UPLOADS and not capturing:
        return torch.from_numpy(a.copy()).to(device=device(), dtype=dtype, non_blocking=False).contiguous()
    if not capturing and dtype in _NP_DTYPE:
        d = device()
        ring = _RINGS.get(d.index)
        if ring is None:
            ring = _RINGS[d.index] = _StagingRing()
        view = ring.stage(a)
        if view is not None:
            out = torch.empty(a.shape, dtype=dtype, device=d)
            out.view(-1).view(torch.uint8).copy_(view, non_blocking=True)
            ring.done(view)
            return out
    src = torch.from_numpy(a.copy() if not a.flags.writeable else a)
    src = src.pin_memory()
    if capturing:
        _pinned_keep.append(src)
    out = src.to(device=device(), non_blocking=True)
    return out if out.dtype == dtype else out.to(dtype)


_DEV_MANY = os.environ.get("TQ_DEV_MANY", "1") == "1"      # A/B knob


def dev_many(items):
    """Upload several small host arrays with ONE copy: ``items`` is a list of
    (array, torch dtype); returns the device tensors (views of one device
    block, each 256-byte aligned) in order.  Same stream semantics as
    ``dev``; falls back to one upload per array under stream capture or when
    the batch does not fit a ring slot."""
    arrs = [np.ascontiguousarray(x, dtype=_NP_DTYPE.get(dt)) for x, dt in items]
    offs, total = [], 0
    for a in arrs:
        offs.append(total)
        total += (a.nbytes + 255) & ~255
    ok = (_DEV_MANY and total > 0 and not _PAGEABLE_UPLOADS and all(dt in _NP_DTYPE for _, dt in items)
          and not torch.cuda.is_current_stream_capturing())
    lo = None
    if ok:
        d = device()
        ring = _RINGS.get(d.index)
        if ring is None:
            ring = _RINGS[d.index] = _StagingRing()
        lo = ring.reserve(total)
    if lo is None:
        return [dev(a, dt) for a, (_, dt) in zip(arrs, items)]
    host = ring.host
    for a, o in zip(arrs, offs):
        if a.nbytes:
            host[lo + o: lo + o + a.nbytes] = a.reshape(-1).view(np.uint8)
    block = torch.empty(total, dtype=torch.uint8, device=d)
    block.copy_(ring.buf[lo: lo + total], non_blocking=True)
    ring.done(None)
    out = []
    for a, o, (_, dt) in zip(arrs, offs, items):
        if a.size == 0:
            out.append(torch.empty(a.shape, dtype=dt, device=d))
        else:
            out.append(block[o: o + a.nbytes].view(dt).view(a.shape))
    return out


def dev_bytes(buf):
    """Upload raw bytes (e.g. a ctypes struct array) as a uint8 device tensor."""
    import numpy as np
    return dev(np.frombuffer(bytes(buf), dtype=np.uint8), torch.uint8)


def sync():
    call("tq_device_sync", stream())
