"""Mass-matrix formation on the GPU with the reference's four strategies.

Drop-in for ``trimquad.assembly`` (src/assembly.py:40-665): same entry points
(``assemble_mass``, ``form_with_timings``, ``sum_factor_row``,
``sum_factor_op_count``), types (``CoefficientField``, ``SparseMatrix``,
``FormationReport``) and errors.  Every formation step runs in sm_100a
kernels; the host only orchestrates and (optionally) copies the final CSR
back into a scipy matrix.

Row sources:
  * separable rows -- interior test functions with c == 1 under wq/hybrid/
    dwq: M_ij = a1[i1,j1] a2[i2,j2], never materialised before the CSR write;
  * raw rows -- everything else (cut rows, c != 1, the ``reference``
    strategy): a dense local block per row written by ``tq_raw_rows``.
The symmetrised, zero-dropped CSR is then counted, scanned and filled.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field

import contextlib

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib as L
from ._lib import CUT, EXTERIOR, INTERIOR
from ._lib import RuleConstructionError as RuleConstructionError_
from .quadrature import compute_wq_rules, place_wq_points
from .splines import TensorBasis2D
from .trimming import TrimConfiguration

STRATEGIES = ("reference", "wq", "hybrid", "dwq")   # src/assembly.py:51


class CoefficientField:
    """Scalar coefficient c(u1,u2) (src/assembly.py:54-85).

    ``fn`` is a host callable (N,2)->(N,) evaluated on the host at the
    requested point sets and uploaded; ``device`` is an optional on-device
    description (``GeometryMap``) evaluated by the GPU instead.
    """

    def __init__(self, fn=None, device=None):
        self._fn = fn
        self._device = device
        self._grids = {}

    @property
    def identity(self):
        return self._fn is None and self._device is None

    def at(self, points):
        points = np.atleast_2d(points)
        if self.identity:
            return np.ones(points.shape[0])
        if self._fn is None:
            return self._device.at_host(points)
        return np.asarray(self._fn(points), dtype=float).reshape(points.shape[0])

    def grid(self, pts1, pts2):
        key = (id(pts1), id(pts2))
        if key not in self._grids:
            if self.identity:
                self._grids[key] = np.ones((pts1.size, pts2.size))
            else:
                P = np.column_stack([np.repeat(pts1, pts2.size), np.tile(pts2, pts1.size)])
                self._grids[key] = self.at(P).reshape(pts1.size, pts2.size)
        return self._grids[key]

    # -- device evaluation ----------------------------------------------------
    def at_device(self, P_dev):
        """c at device points (N,2) -> device (N,)."""
        if self.identity:
            return torch.ones(P_dev.shape[0], dtype=torch.float64, device=P_dev.device)
        if self._device is not None:
            return self._device.at_device(P_dev)
        return L.dev(self.at(P_dev.cpu().numpy()), torch.float64)

    def grid_device(self, x1_dev, x2_dev, out=None):
        """c on the tensor grid x1 x x2 -> device (N1, N2) (into ``out``, a
        ``_padded_grid``, when given)."""
        if self._device is not None:
            return self._device.grid_device(x1_dev, x2_dev, out)
        g = self.grid(x1_dev.cpu().numpy(), x2_dev.cpu().numpy())
        out = _padded_grid(g.shape[0], g.shape[1], x1_dev.device) if out is None else out
        out.copy_(torch.as_tensor(g, dtype=torch.float64))
        return out


def _padded_grid(n1, n2, device):
    """(n1, n2) coefficient grid with two doubles of slack after its end: the
    strips kernel reads rows with 16-byte bulk copies rounded up to an even
    length (tq_sf_strips)."""
    buf = torch.empty(n1 * n2 + 2, dtype=torch.float64, device=device)
    return buf[: n1 * n2].view(n1, n2)


class GeometryMap:
    """c = det J of a B-spline geometry map x(u,v) = sum N_i(u) N_j(v) P_ij,
    evaluated on the GPU (``tq_coeff_grid`` / ``tq_coeff_points``).  Same
    knot vector and degree in both directions; X, Y are (n, n) control nets."""

    def __init__(self, knots, p, X, Y):
        self.knots = np.ascontiguousarray(knots, dtype=float)
        self.p = int(p)
        self.X = np.ascontiguousarray(X, dtype=float)
        self.Y = np.ascontiguousarray(Y, dtype=float)
        self.n = self.X.shape[0]
        self._dev = None

    def device(self):
        if self._dev is None:
            from . import _rawrows
            _rawrows._bind()
            k, X, Y = (L.dev(a, torch.float64) for a in (self.knots, self.X.ravel(), self.Y.ravel()))
            self._dev = (L.Coeff(1, self.p, self.n, L.ptr(k), L.ptr(X), L.ptr(Y)), (k, X, Y))
        return self._dev[0]

    def grid_device(self, x1, x2, out=None):
        out = _padded_grid(x1.numel(), x2.numel(), x1.device) if out is None else out
        L.call("tq_coeff_grid", self.device(), L.ptr(x1), x1.numel(), L.ptr(x2), x2.numel(), L.ptr(out), L.stream())
        return out

    def at_device(self, P):
        P = P.contiguous()
        out = torch.empty(P.shape[0], dtype=torch.float64, device=P.device)
        L.call("tq_coeff_points", self.device(), L.ptr(P), P.shape[0], L.vp(0), L.ptr(out), L.stream())
        return out

    def at_host(self, points):
        return self.at_device(L.dev(np.atleast_2d(points), torch.float64)).cpu().numpy()


class SparseMatrix:
    """Row-compressed symmetric mass matrix over the active functions
    (src/assembly.py:88-120).  ``device`` keeps the GPU CSR (indptr, indices,
    data) when it was formed on the device."""

    def __init__(self, data, active, basis2d, device=None):
        self.data = data
        self._active = active          # (K, 2) array, or a callable producing it on first use
        self.basis2d = basis2d
        self.symmetric = True
        self.device = device

    @property
    def active(self):
        """(K, 2) active (i1, i2) pairs in row order (src/assembly.py:88-120),
        fetched from the device on first access."""
        if callable(self._active):
            self._active = self._active()
        return self._active

    @active.setter
    def active(self, value):
        self._active = value

    @property
    def shape(self):
        return self.data.shape

    def index_of(self):
        n1, n2 = self.basis2d.shape
        out = np.full((n1, n2), -1, dtype=np.int64)
        out[self.active[:, 0], self.active[:, 1]] = np.arange(self.active.shape[0])
        return out

    def frobenius(self):
        return float(sp.linalg.norm(self.data))

    def asymmetry(self):
        return float(sp.linalg.norm(self.data - self.data.T))

    def toarray(self):
        return self.data.toarray()


@dataclass
class FormationReport:
    """Phase breakdown of one formation (src/assembly.py:123-138), seconds.
    ``t_finish`` (symmetrise + compact + CSR write) is reported separately
    because the fused row writer runs there; ``t_total`` includes it."""
    strategy: str
    t_weights: float = 0.0
    t_interior: float = 0.0
    t_cut_regular: float = 0.0
    t_cut_elements: float = 0.0
    t_finish: float = 0.0
    t_total: float = 0.0
    n_wq_points: int = 0
    n_gauss_elements: int = 0
    n_cutcell_points: int = 0
    nnz: int = 0
    kernels: dict = field(default_factory=dict)

    def components(self):
        return (self.t_weights, self.t_interior, self.t_cut_regular, self.t_cut_elements)


class _Clock:
    """Phase timer: device-synchronised wall clock (the reference's
    perf_counter boundaries).  Inactive (no syncs) under stream capture."""

    def __init__(self, active=True):
        self.active = active
        if active:
            torch.cuda.synchronize()
        self.t = time.perf_counter()

    def lap(self):
        if not self.active:
            return 0.0
        torch.cuda.synchronize()
        now = time.perf_counter()
        dt, self.t = now - self.t, now
        return dt


@dataclass
class DeviceCSR:
    indptr: torch.Tensor    # int32 (rows+1)
    indices: torch.Tensor   # int32 (nnz)
    data: torch.Tensor      # float64 (nnz)
    row_begin: int
    row_end: int
    nnz: int

    def to_host(self):
        """(indptr, indices, data) as numpy arrays backed by pinned host
        memory (torch's caching host allocator reuses freed blocks), copied
        with asynchronous DMA."""
        out = []
        for t in (self.indptr, self.indices, self.data):
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t, non_blocking=True)
            out.append(h)
        torch.cuda.current_stream().synchronize()
        return tuple(h.numpy() for h in out)

    def to_scipy(self, shape):
        ptr, ind, dat = self.to_host()
        return sp.csr_matrix((dat, ind, ptr), shape=shape)


class _KernelTimer:
    """CUDA events around named native calls on the launching stream."""

    def __init__(self):
        self.events = {}

    def __call__(self, name):
        timer = self

        class _Ctx:
            def __enter__(self_):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                timer.events.setdefault(name, []).append((s, e))
                s.record()

            def __exit__(self_, *a):
                timer.events[name][-1][1].record()
        return _Ctx()

    def ms(self):
        torch.cuda.synchronize()
        return {k: sum(s.elapsed_time(e) for s, e in v) for k, v in self.events.items()}


class _NoTimer:
    class _C:
        def __enter__(self):
            pass

        def __exit__(self, *a):
            pass

    _c = _C()

    def __call__(self, name):
        return self._c


class Formation:
    """Device state of one assembly run (the analogue of ``_Run``,
    src/assembly.py:272-404)."""

    def __init__(self, basis2d: TensorBasis2D, config: TrimConfiguration, coeff, strategy, timer=None,
                 capture=None):
        if strategy not in STRATEGIES:
            raise ValueError(f"unknown strategy {strategy!r}; choose from {STRATEGIES}")
        self.basis2d = basis2d
        self.config = config
        self.coeff = coeff or CoefficientField()
        self.strategy = strategy
        self.b1, self.b2 = basis2d.dir
        idx, _ = config.active_index()
        self.col_of, self.active, self.K = idx["col_of"], idx["active"], idx["K"]
        self.dev = L.device()
        n1, n2 = basis2d.shape
        # raw-row slot per function (-1: separable); geometry, cached per
        # configuration -- the raw phase swaps in the map of its row plan
        from ._rawrows import _geo
        g = _geo(config)
        if "slot_none" not in g:
            g["slot_none"] = torch.full((n1 * n2,), -1, dtype=torch.int32, device=self.dev)
        self.slot = g["slot_none"]
        self.a1 = self.a2 = None
        self.raw = None
        self.raw_list = torch.empty(0, dtype=torch.int32, device=self.dev)   # raw-row function ids
        self.deep = None
        self.rowfast = None
        self.rules = None
        self.report = FormationReport(strategy)
        self.timer = timer or _NoTimer()
        # capture: None (eager) or dict(nnz=...) -- a CUDA-graph capture pass
        # with no host syncs; sizes come from the preceding eager pass
        self.capture = capture

    # -- phases -------------------------------------------------------------------
    def build_weights(self, rules=None):
        if self.strategy == "reference":
            return
        if rules is None:
            from . import _rawrows
            rules = _rawrows.build_all_rules(self)
        self.rules = rules
        self.report.n_wq_points = rules[0].layout.num_points + rules[1].layout.num_points

    def separable(self):
        return self.strategy != "reference" and self.coeff.identity

    def interior_products(self):
        """Direction-wise WQ contractions a_d (c == 1)."""
        if not self.separable():
            return
        pre = [getattr(r, "_products", None) for r in self.rules[:2]]
        if all(a is not None for a in pre):      # written by the fits (tq_wq_solve)
            self.a1, self.a2 = pre
            return
        from ._rawrows import _forked, _keep_on, _named_stream
        main = torch.cuda.current_stream()
        side = _named_stream("products", priority=-2)
        out = []
        for d, (b, r) in enumerate(zip((self.b1, self.b2), self.rules[:2])):
            first, vals = r.basis_table()
            a = torch.empty((b.n, 2 * b.p + 1), dtype=torch.float64, device=self.dev)
            with _forked(main, side) if d == 1 else contextlib.nullcontext():   # the two directions overlap
                L.call("tq_wq_products", b.device(), r.layout.device(), L.ptr(first), L.ptr(vals), r.device(),
                       L.ptr(a), L.stream())
            out.append(a)
        main.wait_stream(side)
        _keep_on(main, out[1:])
        self.a1, self.a2 = out

    def raw_rows(self, phase):
        """Raw blocks of the non-separable rows (phase 'interior'/'cut'/'cutcells')."""
        from . import _rawrows
        _rawrows.run_phase(self, phase)

    def rowctx(self, row_begin=0, row_end=None):
        b1, b2 = self.b1, self.b2
        d1, d2 = b1.device_arrays(), b2.device_arrays()
        dummy = self.slot
        return L.RowCtx(b1.n, b2.n, b1.p, b2.p,
                        L.ptr(d1["ov_lo"]), L.ptr(d1["ov_hi"]), L.ptr(d2["ov_lo"]), L.ptr(d2["ov_hi"]),
                        L.ptr(self.col_of), L.ptr(self.active), L.ptr(self.slot),
                        L.ptr(self.a1 if self.a1 is not None else dummy),
                        L.ptr(self.a2 if self.a2 is not None else dummy),
                        L.ptr(self.raw if self.raw is not None else dummy),
                        L.ptr(self.deep), L.ptr(self.rowfast), row_begin, self.K if row_end is None else row_end)

    def fill(self, ctx, indptr, indices, data, part=0):
        """Fast rows by warp tiles on the current stream; the rows listed by
        the count pass concurrently on a side stream."""
        from ._rawrows import _named_stream
        main = torch.cuda.current_stream()
        ev_side = None
        if FILL_EVENTS is not None:
            # fill-start timing event (external: an event node when captured)
            # on its own branch, so no node is added to the fill's critical path
            ev_side = _named_stream("fill_event", priority=0)
            ev_side.wait_stream(main)
            FILL_EVENTS[0].record(ev_side)
        # lowest priority: the tile fill's warps dispatch first, the listed
        # rows take the slots it leaves (measured best)
        side = _named_stream("fill_listed", priority=0)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            L.call("tq_fill_listed", ctx, L.ptr(indptr), L.ptr(indices), L.ptr(data), L.ptr(self.work), L.stream())
            _stamp("fill_listed")
        L.call("tq_fill_fast_part", ctx, L.ptr(indptr), L.ptr(indices), L.ptr(data), part, 0, L.stream())
        _stamp("fill_tiles")
        main.wait_stream(side)
        if ev_side is not None:
            main.wait_stream(ev_side)
        if not torch.cuda.is_current_stream_capturing():
            for t in (indptr, indices, data, self.work) + self._count_bufs:
                t.record_stream(side)

    def finish(self, row_begin=0, row_end=None, join=None) -> DeviceCSR:
        """Count -> scan -> fill: symmetrised, zero-dropped, sorted CSR rows
        [row_begin, row_end) (src/assembly.py:400-404).  ``join``: a side
        stream still computing the raw rows; the deep-row pass overlaps it."""
        row_end = self.K if row_end is None else row_end
        nrows = row_end - row_begin
        from ._rawrows import join_cut_blocks, planes
        if self.raw is not None and planes(self):
            return self._finish_planes(row_begin, row_end, join)
        if self.deep is None and self.a1 is not None:
            n1, n2 = self.basis2d.shape
            # geometric flags: cached per row plan (keyed by its raw-row list)
            from ._rawrows import _geo
            g = _geo(self.config)
            gkey = ("deep_geo", id(self.raw_list) if self.raw_list.numel() else None)
            if gkey not in g:
                geo = torch.empty(n1 * n2, dtype=torch.int8, device=self.dev)
                L.call("tq_deep_geometry", self.rowctx(), L.ptr(self.config.func_class_dev), L.ptr(self.raw_list),
                       self.raw_list.numel(), L.ptr(geo), L.stream())
                g[gkey] = (geo, self.raw_list)     # the list is kept alive with its key
            # the count pass applies the factor positivity inline and hands the
            # deep / not-deep split to the fill through its row lists: the
            # context carries the geometric flags, no deep array is formed
            self.deep = g[gkey][0]
            _stamp("deep_flags")
        spec = getattr(self, "_spec", None)
        if spec is not None and (spec["rows"] != (row_begin, row_end) or self.a1 is None):
            raise RuntimeError("speculative count pass launched for another row range")
        # count pass 1 depends on the row plan's geometry and, through the
        # factor positivity, on values only in a corner case: its arrays are
        # cached per configuration like the reference's sparsity pattern
        # (_pattern_for, src/assembly.py:186-195) and a captured pass checks
        # the positivity against them on the device (tq_row_counts_cached)
        from ._rawrows import _geo
        ckey = ("counts1", row_begin, row_end, id(self.deep)) if self.a1 is not None else None
        cached = _geo(self.config).get(ckey) if (ckey is not None and spec is None) else None
        if spec is not None:       # count pass 1 ran at pass start (prelaunch_counts)
            self.rowfast, counts, work, tiles = spec["rowfast"], spec["counts"], spec["work"], spec["tiles"]
        elif cached is not None and self.capture is not None:
            self.rowfast, counts, work = cached["rowfast"], cached["counts"], cached["work"]
            tiles = torch.empty(L.tile_ints(nrows), dtype=torch.int32, device=self.dev)
        else:
            self.rowfast = torch.empty(max(nrows, 1), dtype=torch.int8, device=self.dev)   # written for every row
            counts = torch.empty(max(nrows, 1), dtype=torch.int32, device=self.dev)
            work = torch.empty(2 * nrows + 2, dtype=torch.int32, device=self.dev)
            # tile mode: the count passes leave per-32-row sums, one small scan
            # turns them into bases and the fill derives (and writes) indptr
            tiles = torch.empty(L.tile_ints(nrows), dtype=torch.int32, device=self.dev)
        ctx = self.rowctx(row_begin, row_end)
        ctx.counts, ctx.tiles = L.ptr(counts), L.ptr(tiles)
        self._count_bufs = (counts, tiles)
        self._nrows = nrows
        with self.timer("counts"):
            if spec is not None:
                # the factors exist now: positivity check, redo only if a line is not positive
                torch.cuda.current_stream().wait_stream(spec["stream"])
                pos = torch.empty(self.b1.n + self.b2.n, dtype=torch.int8, device=self.dev)
                L.call("tq_row_counts_verify", ctx, L.ptr(self.deep), L.ptr(pos), L.ptr(spec["bad"]),
                       L.ptr(counts), L.ptr(work), L.stream())
            elif cached is not None and self.capture is not None:
                pos = torch.empty(self.b1.n + self.b2.n, dtype=torch.int8, device=self.dev)
                L.call("tq_row_counts_cached", ctx, L.ptr(self.deep), L.ptr(pos), L.ptr(cached["pos"]),
                       L.ptr(cached["flags"]), L.ptr(counts), L.ptr(work), L.ptr(cached["tiles0"]), L.stream())
            elif self.a1 is not None:
                pos = torch.empty(self.b1.n + self.b2.n, dtype=torch.int8, device=self.dev)
                L.call("tq_row_counts_geo", ctx, L.ptr(self.deep), L.ptr(pos), L.ptr(counts), L.ptr(work),
                       L.stream())
                if ckey is not None and cached is None and self.capture is None:
                    # snapshot right after pass 1 (pass 2 adds to the tile sums)
                    _geo(self.config)[ckey] = dict(
                        rowfast=self.rowfast.clone(), counts=counts.clone(), work=work.clone(),
                        tiles0=tiles.clone(), pos=pos.clone(),
                        flags=torch.zeros(3, dtype=torch.int32, device=self.dev))
            else:
                L.call("tq_row_counts_deep", ctx, L.ptr(counts), L.ptr(work), L.stream())
            rec = None
            if self.a1 is not None and GEOMETRIC_NEAR:
                # interior separable rows on positive lines are counted
                # geometrically by pass 2 and verified by the fill (rowctx.fclass)
                ctx.fclass, ctx.pos = L.ptr(self.config.func_class_dev), L.ptr(pos)
                self._near_pos = pos
                # the listed rows' geometry records, before the join (pass 2
                # starts from them: one load per row)
                rec = torch.empty(max(nrows, 1) * int(L.lib().tq_list_record_bytes()), dtype=torch.uint8,
                                  device=self.dev)
                L.call("tq_list_geometry", ctx, L.ptr(work), L.ptr(rec), L.stream())
                self._list_rec = rec
            _stamp("counts_deep")
            head = None
            if self.capture is not None and HEAD_FILL:
                # the output exists before the scan (nnz known): the tiles
                # before the first / after the last list-A row have final
                # offsets now (the tail ones from nnz; the full scan checks
                # it) -- fill them on a low-priority stream with a capped grid
                # while the raw rows and count pass 2 finish
                out = self._alloc_out(nrows, self.capture["nnz"])
                L.call("tq_scan_tiles_early", ctx, self.capture["nnz"], EARLY_TAIL, L.stream())
                main = torch.cuda.current_stream()
                from ._rawrows import _named_stream
                head = _named_stream("fill_head", priority=0)
                head.wait_stream(main)
                with torch.cuda.stream(head):
                    L.call("tq_fill_fast_part", ctx, *map(L.ptr, out), 1, HEAD_BLOCKS_PER_SM, L.stream())
                    _stamp("head_fill")
            # count pass 2 reads raw values: the pass-start stream (Gauss
            # parts, cut-element blocks) and the cut-row side stream rejoin
            # here, after pass 1 (which needs neither)
            join_cut_blocks(self)
            if join is not None:
                torch.cuda.current_stream().wait_stream(join)
            _stamp("join")
            if rec is not None:
                L.call("tq_row_counts_rest_rec", ctx, L.ptr(counts), L.ptr(work), L.ptr(rec), L.stream())
            else:
                L.call("tq_row_counts_rest", ctx, L.ptr(counts), L.ptr(work), L.stream())
            _stamp("counts_rest")
        nnz = L.i64(0)
        if head is None:
            indptr = torch.empty(nrows + 1, dtype=torch.int32, device=self.dev)
        else:
            indptr, indices, data = out
        with self.timer("scan"):
            if self.capture is not None and head is None:
                # a replay must reproduce the captured nnz (its buffers' size):
                # checked by the scan, the fill writes nothing otherwise
                L.call("tq_tiles_expect", ctx, self.capture["nnz"], L.stream())
            L.call("tq_scan_tiles", ctx, L.ptr(indptr), None if self.capture else L.C.byref(nnz), L.stream())
        _stamp("scan")
        nnz = self.capture["nnz"] if self.capture else int(nnz.value)
        if head is None:
            indices = torch.empty(max(nnz, 1), dtype=torch.int32, device=self.dev)
            data = torch.empty(max(nnz, 1), dtype=torch.float64, device=self.dev)
        self.work = work
        with self.timer("fill"):
            self.fill(ctx, indptr, indices, data, part=0 if head is None else 2)
        if head is not None:
            torch.cuda.current_stream().wait_stream(head)
        for st in getattr(self, "_status_streams", []):       # status reductions rejoin
            torch.cuda.current_stream().wait_stream(st)
        _stamp("fill")
        if self.capture is None and nrows > 0 and ctx.fclass and int(tiles[L.tile_ctl(nrows) + 8].item()):
            raise RuntimeError("a geometrically counted row dropped an entry (rowctx.fclass): pattern inconsistent")
        return DeviceCSR(indptr, indices[:nnz], data[:nnz], row_begin, row_end, nnz)

    def _finish_planes(self, row_begin, row_end, join):
        """All-raw formation: symmetrise / zero-drop / CSR in one pass over
        the planes (tq_planes_csr).  The output is sized by the window total
        (an upper bound of nnz) so no count pass precedes it."""
        from ._rawrows import join_cut_blocks, planes_geo
        nrows = row_end - row_begin
        pg = planes_geo(self)
        join_cut_blocks(self)
        if join is not None:
            torch.cuda.current_stream().wait_stream(join)
        _stamp("join")
        W = (2 * self.b1.p + 1) * (2 * self.b2.p + 1)
        cap = max(nrows * W, 1)
        indptr = torch.empty(nrows + 1, dtype=torch.int32, device=self.dev)
        indices = torch.empty(cap, dtype=torch.int32, device=self.dev)
        data = torch.empty(cap, dtype=torch.float64, device=self.dev)
        state = torch.empty((L.lib().tq_planes_state_bytes(nrows) + 7) // 8, dtype=torch.int64, device=self.dev)
        ctl = torch.zeros(3, dtype=torch.int32, device=self.dev)
        ctx = self.rowctx(row_begin, row_end)
        ctx.raw_ld = pg["ld"]
        expect = self.capture["nnz"] if self.capture else -1
        nnz = L.i64(0)
        with self.timer("fill"):
            L.call("tq_planes_csr", ctx, pg["base"], L.ptr(indptr), L.ptr(indices), L.ptr(data), cap, L.ptr(state),
                   L.ptr(ctl), expect, None if self.capture else L.C.byref(nnz), L.stream())
        self._planes_ctl = ctl
        self._count_bufs = (indptr, state)
        self._nrows = nrows
        for st in getattr(self, "_status_streams", []):       # status reductions rejoin
            torch.cuda.current_stream().wait_stream(st)
        st = getattr(self, "_planes_status", None)
        if st is not None and self.capture is None and int(st.item()):
            raise RuntimeError(f"planes path status {int(st.item())}: a strip workspace bound (1, 2) or an element "
                               "block (4) missed")
        _stamp("fill")
        nnz = self.capture["nnz"] if self.capture else int(nnz.value)
        return DeviceCSR(indptr, indices[:nnz], data[:nnz], row_begin, row_end, nnz)

    def _alloc_out(self, nrows, nnz):
        return (torch.empty(nrows + 1, dtype=torch.int32, device=self.dev),
                torch.empty(max(nnz, 1), dtype=torch.int32, device=self.dev),
                torch.empty(max(nnz, 1), dtype=torch.float64, device=self.dev))


STAMPS = None     # timeline probe (an _lib.Stamps) -- development aid
# captured passes can fill the tiles before the first list-A row early, on a
# low-priority stream with this many fill blocks per SM (tuning knobs; off by
# default since the single-stage fill: the early fill's memory traffic slows
# the latency-bound count pass 2 by more than it saves, measured at config 5)
HEAD_FILL = int(os.environ.get("TQ_HEAD_FILL", "0"))
# TQ_GRAPH_PRIO=1: replayed graphs honour the capture streams' priorities
# (instantiated by the library with per-node priorities; the kernel nodes do
# carry them, GraphFormation.node_priorities).  Default off: measured equal
# at config 4 and 3-5 us slower at config 5 than torch's instantiation, which
# runs every node at the launch stream's priority
GRAPH_NODE_PRIORITY = os.environ.get("TQ_GRAPH_PRIO", "0") == "1"
# count pass 2 counts interior separable rows on positive factor lines
# geometrically (their partner sums are positive; the fill verifies them)
GEOMETRIC_NEAR = os.environ.get("TQ_GEOMETRIC_NEAR", "1") == "1"
HEAD_BLOCKS_PER_SM = int(os.environ.get("TQ_HEAD_BPS", "3"))
# ... and the tiles after the last list-A row too (their offsets from the
# captured nnz): measured slower at config 5 (the early fill then delays the
# latency-bound count pass 2), off by default
EARLY_TAIL = int(os.environ.get("TQ_EARLY_TAIL", "0"))


def _stamp(name):
    if STAMPS is not None:
        STAMPS(name)


def form(basis2d, config, coeff=None, strategy="reference", rules=None, row_range=None, timer=None,
         capture=None, timed=True):
    """Run every formation phase on the device; returns (Formation, DeviceCSR).

    Eager passes run the phases in order with synchronised phase timers (the
    reference's FormationReport boundaries).  A capture pass (``capture`` =
    dict(nnz=...), used by GraphFormation) schedules the cut-row chain on a
    side stream, overlapping the deep-row flags and counts.  ``timed=False``
    drops the phase clock's synchronisations (nobody reads the report)."""
    f = Formation(basis2d, config, coeff, strategy, timer, capture)
    f.row_range = row_range        # a row block forms only the raw rows its rows read
    rep = f.report
    if config.has_cuts():     # shared geometry (src/assembly.py:505-508)
        if capture is None:
            # the cut-row list and the DWQ routing read two small results
            # back: before the cut-cell kernel is queued, not behind it
            from ._rawrows import cut_rows_host, dwq_keys
            cut_rows_host(f)
            if strategy == "dwq":
                dwq_keys(f)
        # queued now (device) or built on a worker thread (host), joined on
        # first use: it runs while the host builds the plans and the fits run
        config.cut_cell_rule_async(max(basis2d.degrees))
    clk = _Clock(active=capture is None and timed)
    _stamp("start")
    if capture is not None:
        from ._rawrows import prelaunch_counts, prelaunch_geometry, prelaunch_grids
        prelaunch_counts(f)
        prelaunch_grids(f)
        prelaunch_geometry(f)
    f.build_weights(rules)
    _stamp("weights")
    rep.t_weights = clk.lap()
    f.interior_products()
    _stamp("products")
    f.raw_rows("interior")
    _stamp("raw_interior")
    rep.t_interior = clk.lap()
    rb, re_ = (0, f.K) if row_range is None else row_range
    if capture is not None:
        from ._rawrows import _forked, _side_streams
        main = torch.cuda.current_stream()
        side = _side_streams(1)[0]
        with _forked(main, side):
            f.raw_rows("cut")
            _stamp("side:raw_cut")
            f.raw_rows("cutcells")
            _stamp("side:cutcells")
        csr = f.finish(rb, re_, join=side)
    else:
        f.raw_rows("cut")
        rep.t_cut_regular = clk.lap()
        f.raw_rows("cutcells")
        rep.t_cut_elements = clk.lap()
        csr = f.finish(rb, re_)
        rep.t_finish = clk.lap()
    rep.t_total = rep.t_weights + rep.t_interior + rep.t_cut_regular + rep.t_cut_elements + rep.t_finish
    rep.nnz = csr.nnz
    return f, csr


# (start,) timing event recorded where the fill starts while a pass is
# captured (GraphFormation(fill_events=...)); None otherwise
FILL_EVENTS = None


def _graph_handle(graph):
    """cudaGraph_t of a torch CUDAGraph(keep_graph=True) as an int."""
    h = graph.raw_cuda_graph()
    if isinstance(h, int):
        return h
    for conv in (int, lambda x: int(x.getPtr()), lambda x: x.value):
        try:
            return int(conv(h))
        except Exception:
            continue
    raise RuntimeError(f"cannot read the cudaGraph_t handle from {type(h)}")


class GraphFormation:
    """One formation pass captured as a CUDA graph and replayed.

    The first call runs eagerly (it builds the cached geometry plans and
    learns nnz and the fit status); the pass is then captured with no host
    syncs and every ``run()`` replays all of its kernels -- weights, DWQ
    sets, interior products, raw and cut rows, symmetrise/compact/CSR fill --
    into the same static device buffers.  The moment-fit residual flags are
    re-checked after each replay (``check()``)."""

    def __init__(self, basis2d, config, coeff=None, strategy="dwq", row_range=None, fill_events=None):
        """``fill_events``: an optional 1-tuple holding a timing event
        created with ``external=True``; it is captured where the fill
        (tiles and listed rows) starts, on a side branch of the graph, so an
        event recorded after the replay times the fill inside the step."""
        global FILL_EVENTS
        self.args = (basis2d, config, coeff, strategy)
        self.row_range = row_range
        f, csr = form(basis2d, config, coeff, strategy, row_range=row_range)
        self.nnz = csr.nnz
        self.report = f.report
        del f, csr
        torch.cuda.synchronize()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):   # warm the capture path once (allocator, attributes)
            form(*self.args, row_range=row_range, capture={"nnz": self.nnz})
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph(keep_graph=True)
        lib = L.lib()
        lib.tq_launch_count.restype = L.C.c_longlong
        n0 = lib.tq_launch_count()
        from ._rawrows import _named_stream
        cap = _named_stream("capture", priority=-2)      # the main chain outranks the bulk side streams
        FILL_EVENTS = fill_events
        try:
            with torch.cuda.graph(self.graph, stream=cap):
                self.f, self.csr = form(*self.args, row_range=row_range, capture={"nnz": self.nnz})
        finally:
            FILL_EVENTS = None
        self.launches_per_pass = int(lib.tq_launch_count() - n0)
        # instantiated by the library with per-node priorities: the capture
        # streams' priorities (fit chain, pass-start chains, bulk work) hold
        # in every replay (a default instantiation runs all nodes at the
        # launch stream's priority)
        self._exec = None
        if GRAPH_NODE_PRIORITY:
            ex = L.vp()
            L.call("tq_graph_instantiate", L.vp(_graph_handle(self.graph)), 1, L.C.byref(ex))
            self._exec = ex
        else:
            self.graph.instantiate()
        torch.cuda.synchronize()

    def node_priorities(self):
        """Kernel nodes of the captured graph by priority (hist[k]: -k)."""
        hist, nk = (L.i32 * 8)(), L.i32(0)
        L.call("tq_graph_node_priorities", L.vp(_graph_handle(self.graph)), hist, L.C.byref(nk))
        return list(hist), int(nk.value)

    def node_types(self):
        """Graph nodes by type: kernel, memcpy, memset, host, graph, empty,
        event wait, event record, ... (cudaGraphNodeType order)."""
        counts = (L.i32 * 12)()
        L.call("tq_graph_node_types", L.vp(_graph_handle(self.graph)), counts)
        names = ["kernel", "memcpy", "memset", "host", "graph", "empty", "wait_event", "event_record",
                 "ext_sem_signal", "ext_sem_wait", "mem_alloc", "mem_free"]
        return {n: int(c) for n, c in zip(names, counts) if c}

    def run(self):
        if self._exec is not None:
            L.call("tq_graph_launch", self._exec, L.stream())
        else:
            self.graph.replay()
        return self.csr

    def __del__(self):
        ex = getattr(self, "_exec", None)
        if ex is not None and L is not None:
            try:
                L.lib().tq_graph_exec_destroy(ex)
            except Exception:
                pass

    def check(self):
        """Status of the last replay (host reads after the pass; the
        reductions ran inside the graph)."""
        fail = getattr(self.f, "_fail_any", None)
        if fail is not None and bool(fail.item()):
            raise RuleConstructionError_("moment-fit residual above tolerance in a replayed pass")
        ctl = getattr(self.f, "_planes_ctl", None)
        if ctl is not None:
            if int(ctl[2].item()):
                raise RuntimeError("replayed pass formed a different nnz than the captured one")
            st = getattr(self.f, "_planes_status", None)
            if st is not None and int(st.item()):
                raise RuntimeError("planes path status word set in a replayed pass (tq_sf_strips / tq_cut_rows_gather)")
        elif self.f._nrows > 0:
            ctl = self.f._count_bufs[1][L.tile_ctl(self.f._nrows):].cpu()
            if int(ctl[4]):
                raise RuntimeError("replayed pass formed a different nnz than the captured one")
            if int(ctl[8]):
                raise RuntimeError("a geometrically counted row dropped an entry in a replayed pass")


def assemble_mass(basis2d: TensorBasis2D, config: TrimConfiguration, coeff=None, strategy="reference",
                  parallel=False, report=None, *, rules=None) -> SparseMatrix:
    """Assemble the mass matrix with the chosen strategy (src/assembly.py:492-550).
    ``parallel`` is accepted for signature parity (the GPU path is always
    parallel); ``rules`` imports precomputed weight tables."""
    if strategy not in STRATEGIES:
        raise ValueError(f"unknown strategy {strategy!r}; choose from {STRATEGIES}")
    from . import _adapt         # reference-built objects are accepted (duck-typed)
    basis2d, config = _adapt.space(basis2d, config)
    coeff = _adapt.coefficient(coeff)
    f, csr = form(basis2d, config, coeff, strategy, rules, timed=report is not None)
    if report is not None:
        # report-only geometry count (cached per row plan), off the formation path
        from ._rawrows import gauss_element_count, needs_raw
        f.report.n_gauss_elements = gauss_element_count(f) if needs_raw(f) else 0
        for k, v in f.report.__dict__.items():
            if k != "strategy":
                setattr(report, k, v)
        report.strategy = strategy
    M = csr.to_scipy((f.K, f.K))
    return SparseMatrix(M, config.active_functions, basis2d, device=csr)


def form_with_timings(strategy, basis2d, config, coeff=None, parallel=False):
    """src/assembly.py:651-665: shared geometry warmed outside the clock."""
    from . import _adapt
    basis2d, config = _adapt.space(basis2d, config)
    coeff = _adapt.coefficient(coeff)
    q = max(basis2d.degrees)
    if config.has_cuts():
        config.cut_cell_rule(q)
    config.active_index()
    report = FormationReport(strategy=strategy)
    M = assemble_mass(basis2d, config, coeff, strategy, parallel, report=report)
    return M, report


def sum_factor_row(i1, i2, rules1, rules2, colloc1, colloc2, grid, mask=None, point_box=None):
    """One mass-matrix row by two nested univariate contractions
    (src/assembly.py:218-252), on the device: ``(j1lo, j2lo, block)`` with
    block[o1][o2] = sum_k1 B1[k1][o1] sum_k2 B2[k2][o2] G[k1][k2].  See
    :func:`sum_factor_rows` for the batched form."""
    m = None if mask is None else [mask]
    pb = None if point_box is None else [point_box]
    return sum_factor_rows([(i1, i2)], rules1, rules2, colloc1, colloc2, grid, m, pb)[0]


def sum_factor_rows(rows, rules1, rules2, colloc1, colloc2, grid, masks=None, point_boxes=None):
    """Batched :func:`sum_factor_row`: the operand windows of every row --
    collocation slices colloc_d[s_d:e_d, jlo_d:jhi_d+1], weight rows, the
    coefficient window grid[s1:e1, s2:e2] (and its mask) -- are packed on
    the host and contracted on the device in one launch
    (tq_sum_factor_rows).  ``rules*`` may be this package's or the
    reference's rule sets (only ``row`` and ``basis.overlapping`` are used).
    Returns a list of (j1lo, j2lo, block)."""
    b1, b2 = rules1.basis, rules2.basis
    colloc1 = np.asarray(colloc1, dtype=np.float64)
    colloc2 = np.asarray(colloc2, dtype=np.float64)
    grid = np.asarray(grid, dtype=np.float64)
    chunks, dims, offs, outs, res = [], [], [], [], []
    pos = scratch = out_pos = 0

    def put(a):
        nonlocal pos
        a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
        chunks.append(a)
        pos += a.size
        return pos - a.size

    for r, (i1, i2) in enumerate(rows):
        i1, i2 = int(i1), int(i2)
        k1, w1 = rules1.row(i1)
        k2, w2 = rules2.row(i2)
        w1, w2 = np.asarray(w1, dtype=np.float64), np.asarray(w2, dtype=np.float64)
        s1, e1, s2, e2 = k1, k1 + w1.size, k2, k2 + w2.size
        pb = None if point_boxes is None else point_boxes[r]
        if pb is not None:
            s1, e1 = max(s1, pb[0]), min(e1, pb[1])
            s2, e2 = max(s2, pb[2]), min(e2, pb[3])
        j1lo, j1hi = b1.overlapping(i1)
        j2lo, j2hi = b2.overlapping(i2)
        t1, t2 = j1hi - j1lo + 1, j2hi - j2lo + 1
        if s1 >= e1 or s2 >= e2:
            res.append((j1lo, j2lo, np.zeros((t1, t2))))
            continue
        n1, n2 = e1 - s1, e2 - s2
        G = grid[s1:e1, s2:e2]
        mk = None if masks is None else masks[r]
        if mk is not None and np.shape(mk) != G.shape:
            raise ValueError(f"mask of shape {np.shape(mk)} for a {G.shape} coefficient window")
        o = [put(colloc1[s1:e1, j1lo:j1hi + 1]), put(w1[s1 - k1:e1 - k1]),
             put(colloc2[s2:e2, j2lo:j2hi + 1]), put(w2[s2 - k2:e2 - k2]), put(G),
             put(mk) if mk is not None else -1, scratch]
        scratch += t2 * n1
        dims.append((n1, n2, t1, t2))
        offs.append(o)
        outs.append(out_pos)
        res.append((j1lo, j2lo, (len(outs) - 1, t1, t2)))
        out_pos += t1 * t2
    if outs:
        dev = L.device()
        data = L.dev(np.concatenate(chunks), torch.float64)
        d_dims = L.dev(np.asarray(dims, np.int32), torch.int32)
        d_offs = L.dev(np.asarray(offs, np.int64), torch.int64)
        d_out_off = L.dev(np.asarray(outs, np.int64), torch.int64)
        work = torch.empty(max(scratch, 1), dtype=torch.float64, device=dev)
        out = torch.empty(max(out_pos, 1), dtype=torch.float64, device=dev)
        L.call("tq_sum_factor_rows", len(outs), L.ptr(d_dims), L.ptr(d_offs), L.ptr(d_out_off), L.ptr(data),
               L.ptr(work), L.ptr(out), L.stream())
        host = out.cpu().numpy()
        for k, (j1lo, j2lo, blk) in enumerate(res):
            if isinstance(blk, tuple):
                idx, t1, t2 = blk
                res[k] = (j1lo, j2lo, host[outs[idx]:outs[idx] + t1 * t2].reshape(t1, t2).copy())
    return res


def sum_factor_op_count(i1, i2, rules1, rules2):
    """Multiply-add count of one sum-factorized row (src/assembly.py:255-265)."""
    b1, b2 = rules1.basis, rules2.basis
    n1 = int(rules1.wptr[i1 + 1] - rules1.wptr[i1])
    n2 = int(rules2.wptr[i2 + 1] - rules2.wptr[i2])
    j1lo, j1hi = b1.overlapping(i1)
    j2lo, j2hi = b2.overlapping(i2)
    t1, t2 = j1hi - j1lo + 1, j2hi - j2lo + 1
    return t2 * n1 * n2 + t1 * t2 * n1
