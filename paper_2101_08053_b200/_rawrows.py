"""Raw (non-separable) rows: orchestration of ``tq_raw_regular`` /
``tq_raw_cutcells`` and of the DWQ routing.

Which rows are raw (src/assembly.py:492-610):
  * strategy ``reference``: every active row, element Gauss (GAUSS);
  * c != 1 under wq/hybrid/dwq: interior rows by full-support sum
    factorization over the standard rules (BOX with the full support box);
  * cut rows: hybrid -> GAUSS; wq -> MASK (naive, masked sum factorization);
    dwq -> BOX on the DWQ rule sets for eligible rows with a box, else GAUSS.
Every raw row also collects the cut-element points (``tq_raw_cutcells``).
"""

from __future__ import annotations

import contextlib
import os
import ctypes as C

import weakref

import numpy as np
import torch

from . import _lib as L
from ._lib import CUT, INTERIOR
from .quadrature import (_TAG as _QT, fit_sets_async, combine_sets_async, DiscontinuousRuleSet, _st, DwqPlan, WeightedRuleSet, _FitPlan, _failing, _solve_rows_async_t, build_dwq,
                         compute_wq_rules, dwq_solve_async, gauss_legendre, place_wq_points)

MODE_GAUSS, MODE_BOX, MODE_MASK = 0, 1, 2


class RuleSetDev(C.Structure):
    _fields_ = [("rules", L.Rules), ("lay", L.Layout), ("first", L.vp), ("vals", L.vp)]


class RawCtx(C.Structure):
    _fields_ = ([(k, L.i32) for k in ("n1", "n2", "p1", "p2", "nel1", "nel2")]
                + [(k, L.vp) for k in ("el_first1", "el_last1", "el_first2", "el_last2", "ov_lo1", "ov_hi1",
                                       "ov_lo2", "ov_hi2", "espan1", "espan2", "elem_class")]
                + [("ng1", L.i32), ("ng2", L.i32)]
                + [(k, L.vp) for k in ("ew1", "ev1", "ew2", "ev2", "em1", "em2", "cg", "sets1", "sets2")]
                + [("nsets1", L.i32), ("nsets2", L.i32)]
                + [(k, L.vp) for k in ("grids", "cutidx", "cut_ptr", "cut_cw", "cfirst1", "cvals1", "cfirst2",
                                       "cvals2", "grp_ptr", "grp_key", "grp_pts", "grp_perm", "grp_blocks")]
                + [("ngroups", L.i32), ("desc", L.vp)]
                + [("nraw", L.i32), ("nmax1", L.i32), ("nmax2", L.i32), ("raw", L.vp), ("store", L.vp),
                   ("raw_ld", L.i64)])


def _bind():
    L.optional("tq_raw_regular", [RawCtx, L.i32, L.i32, L.vp])
    L.optional("tq_raw_cutcells", [RawCtx, L.i32, L.i32, L.vp])
    L.optional("tq_row_groups", [RawCtx, L.i32, L.i32, L.vp, L.vp, L.vp])
    L.optional("tq_raw_cutcells_list", [RawCtx, L.i32, L.i32, L.vp, L.vp, L.vp])
    L.optional("tq_cut_blocks", [RawCtx, L.vp])
    L.optional("tq_raw_gauss", [RawCtx, L.i32, L.i32, L.vp])
    L.optional("tq_raw_sumfactor", [RawCtx, L.i32, L.i32, L.vp])
    L.optional("tq_elem_mass", [L.vp, L.vp, L.i32, L.i32, L.i32, L.vp, L.vp])
    L.optional("tq_dwq_route", [L.Space1D, L.Space1D, L.vp, L.vp, L.i32, L.vp, L.i32, L.vp, L.i32, L.vp, L.vp])
    L.optional("tq_coeff_grid", [L.Coeff, L.vp, L.i32, L.vp, L.i32, L.vp, L.vp])
    L.optional("tq_coeff_points", [L.Coeff, L.vp, L.i64, L.vp, L.vp, L.vp])
    L.optional("tq_sf_strips", [RawCtx, L.i32, L.vp, L.i32, L.i32, L.i32, L.i32, L.i32, L.vp, L.vp, L.vp])
    L.optional("tq_bw_tables", [RawCtx, L.vp, L.vp, L.vp])
    L.optional("tq_sf_strips_occupancy", [L.i32] * 6)
    L.optional("tq_gauss_pairs", [RawCtx, L.Coeff, L.vp, L.vp, L.vp, L.i32, L.vp, L.vp, L.vp, L.vp, L.vp, L.vp,
                                  L.vp])
    L.optional("tq_geo_lines", [L.Coeff, L.vp, L.i32, L.vp, L.vp, L.vp])
    L.optional("tq_cut_pairs", [RawCtx, L.vp, L.i32, L.vp, L.vp, L.vp, L.vp])
    L.optional("tq_cut_pair_piece", [], L.i32)
    L.optional("tq_cut_rows_gather", [RawCtx, L.i32, L.i32, L.vp, L.vp, L.vp, L.vp, L.vp, L.vp, L.vp])
    L.optional("tq_pair_block_doubles", [L.i32], L.i64)
    L.optional("tq_bw_table_doubles", [RawCtx], L.i64)
    L.optional("tq_planes_csr", [L.RowCtx, L.i32, L.vp, L.vp, L.vp, L.i64, L.vp, L.vp, L.i64, L.vp, L.vp])
    L.optional("tq_planes_state_bytes", [L.i32], L.i64)


def _geo(config):
    """Config-level cache of geometry-derived data, the analogue of the
    reference's per-configuration caches (cut_cell_rule, _assembly_cache,
    _dwq_cache: src/trimming.py:437-438, 588-594, src/assembly.py:186-195)."""
    g = config.__dict__.get("_geo")
    if g is None:
        g = config.__dict__["_geo"] = {}
    return g


def active_host(f):
    g = _geo(f.config)
    if "active" not in g:
        g["active"] = f.active[: f.K].cpu().numpy().astype(np.int64)
    return g["active"]


def cut_rows_host(f):
    """Active cut functions in active (row-major) order -> function ids
    (filtered on the device; only the cut rows come back)."""
    g = _geo(f.config)
    if "cut_fids" not in g:
        act = f.active[: f.K]
        fc = f.config.func_class_dev.reshape(-1)
        g["cut_fids"] = act[fc[act.long()] == CUT].cpu().numpy().astype(np.int32)
    return g["cut_fids"]


def route_cut_rows(f):
    """DWQ routing on the GPU (src/trimming.py:545-586) -> (cut fids, routes);
    cached per configuration like the reference's dwq_info cache."""
    _bind()
    g = _geo(f.config)
    if "routes" in g:
        return g["routes"]
    cut = cut_rows_host(f)
    routes = np.full((cut.size, 8), -1, np.int32)
    if cut.size:
        u1, u2 = f.config.u_disc
        du1 = L.dev(u1 if u1.size else np.zeros(1), torch.float64)
        du2 = L.dev(u2 if u2.size else np.zeros(1), torch.float64)
        rows = L.dev(cut, torch.int32)
        out = torch.empty((cut.size, 8), dtype=torch.int32, device=f.dev)
        L.call("tq_dwq_route", f.b1.device(), f.b2.device(), L.ptr(f.config.element_class_dev), L.ptr(du1),
               u1.size, L.ptr(du2), u2.size, L.ptr(rows), cut.size, L.ptr(out), L.stream())
        routes = out.cpu().numpy()
    g["routes"] = (cut, routes)
    return g["routes"]


def cut_point_tables(f):
    """Device copy of the host cut-cell rule (cached per configuration)."""
    g = _geo(f.config)
    rule = f.config.cut_cell_rule(max(f.b1.p, f.b2.p))
    if g.get("cutpts_src") is not rule:      # rebuilt when the rule object changes
        b1, b2 = f.b1, f.b2
        ddev = getattr(rule, "dev", None)       # decomposed on the device: no upload
        if ddev is not None:
            P, Wd, ptr_d = ddev["P"], ddev["W"], ddev["ptr"]
        else:
            P = L.dev(rule.points.reshape(-1, 2), torch.float64)
            Wd, ptr_d = L.dev(rule.weights, torch.float64), L.dev(rule.ptr, torch.int64)
        dev = f.dev
        ncut = rule.elements.shape[0]
        el = ddev["el"] if ddev is not None else L.dev(rule.elements.astype(np.int32).reshape(-1, 2), torch.int32)
        cutidx = torch.full((b1.num_elements * b2.num_elements,), -1, dtype=torch.int32, device=dev)
        if ncut:
            cutidx[el[:, 0].long() * b2.num_elements + el[:, 1].long()] = torch.arange(
                ncut, dtype=torch.int32, device=dev)
        t = dict(P=P, x=P[:, 0].contiguous(), y=P[:, 1].contiguous(),
                 W=Wd, idx=cutidx, ptr=ptr_d, npts=rule.total_points())
        # span-key groups per cut element (src/assembly.py:380-388): points of
        # one element grouped by (first1, first2), keys in np.unique order --
        # a stable sort by (element, key) on the device (= np.lexsort with the
        # point index as the last key)
        f1, _ = b1.eval_device(t["x"], check=False)
        f2, _ = b2.eval_device(t["y"], check=False)
        npts = int(t["npts"])
        elem = torch.repeat_interleave(torch.arange(ncut, device=dev), (ptr_d[1:] - ptr_d[:-1]).long())
        key = f1.long() * (b2.n + 1) + f2.long()
        comp = elem * (b1.n * (b2.n + 1) + b2.n + 1) + key
        comp_s, perm = torch.sort(comp, stable=True)
        if npts:
            first = torch.ones(npts, dtype=torch.bool, device=dev)
            first[1:] = comp_s[1:] != comp_s[:-1]
            start = torch.nonzero(first).flatten()
        else:
            start = torch.zeros(0, dtype=torch.int64, device=dev)
        gpts = torch.cat([start, torch.tensor([npts], dtype=torch.int64, device=dev)])
        gelem = elem[perm][start]
        gptr = torch.searchsorted(gelem, torch.arange(ncut + 1, device=dev), right=False).to(torch.int32)
        gkey = torch.stack([f1[perm][start], f2[perm][start]], dim=1).to(torch.int32).contiguous()
        t["grp_ptr"] = gptr
        t["grp_key"] = gkey
        t["grp_pts"] = gpts.contiguous()
        t["grp_perm"] = perm.contiguous() if npts else torch.zeros(1, dtype=torch.int64, device=dev)
        t["ngroups"] = int(start.numel())
        g["cutpts"] = t
        g["cutpts_src"] = rule
    return g["cutpts"]


def element_points(f):
    g = _geo(f.config)
    if "eg" not in g:
        out = []
        for b in (f.b1, f.b2):
            gl = gauss_legendre(b.p + 1)
            bp = b.breakpoints
            mid, half = 0.5 * (bp[:-1] + bp[1:]), 0.5 * np.diff(bp)
            X = mid[:, None] + half[:, None] * gl.points[None, :]
            Wt = half[:, None] * gl.weights[None, :]
            out.append((L.dev(X.ravel(), torch.float64), L.dev(Wt.ravel(), torch.float64)))
        g["eg"] = out
    return g["eg"]


def dwq_keys(f):
    """(direction, u_disc) -> sorted rows, for eligible boxed cut rows
    (src/assembly.py:460-471)."""
    g = _geo(f.config)
    if "dwq_keys" not in g:
        cut, routes = route_cut_rows(f)
        n2 = f.b2.n
        box = (routes[:, 0] == 1) & (routes[:, 3] >= 0)
        ij = (cut.astype(np.int64) // n2, cut.astype(np.int64) % n2)
        needed = {}
        for d in (0, 1):
            iu = routes[:, 1 + d]
            sel = box & (iu >= 0)
            if not np.any(sel):
                continue
            pairs = np.unique(np.stack([iu[sel], ij[d][sel]], axis=1), axis=0)   # (u index, row), sorted
            for k in np.unique(pairs[:, 0]):
                needed[(d, float(f.config.u_disc[d][k]))] = pairs[pairs[:, 0] == k, 1].tolist()
        g["dwq_keys"] = {k: v for k, v in sorted(needed.items())}
    return g["dwq_keys"]


_SIDE = {}


def _side_streams(n):
    dev = torch.cuda.current_device()
    lst = _SIDE.setdefault(dev, [])
    while len(lst) < n:
        # high priority: the fit chains are short latency-bound kernels that
        # must not queue behind the bulk raw-row work of the pass-start stream
        lst.append(torch.cuda.Stream(priority=int(os.environ.get("TQ_PRIO_FITS", -3))))
    return lst[:n]


class _forked:
    """Run a block on a side stream that starts after the main stream."""

    def __init__(self, main, side):
        self.main, self.side = main, side

    def __enter__(self):
        self.side.wait_stream(self.main)
        self.ctx = torch.cuda.stream(self.side)
        self.ctx.__enter__()

    def __exit__(self, *a):
        self.ctx.__exit__(*a)


def _keep_on(stream, tensors):
    """Tensors made on a side stream and consumed on `stream`."""
    for t in tensors:
        if t is not None and not torch.cuda.is_current_stream_capturing():
            t.record_stream(stream)


def build_all_rules(f):
    """Standard WQ rules per direction and the DWQ sets (src/assembly.py:454-489).
    Point layouts and DWQ refinement plans are geometry (cached per
    configuration); every fit -- basis tables, exact moments, pivoted-QR
    solves, S^T combination -- is recomputed on the GPU each call, with a
    single host sync to read back all residual flags."""
    g = _geo(f.config)
    if "std_plans" not in g:
        g["std_plans"] = [_FitPlan(b, place_wq_points(b)) for b in (f.b1, f.b2)]
        # identical directions (same knot vector, hence the same layout and
        # the same moment systems): one set of fits serves both
        g["std_same"] = (f.b1.p == f.b2.p and np.array_equal(f.b1.kv.knots, f.b2.kv.knots))
    same = g["std_same"]
    plans = g["std_plans"]
    fit_plans = plans[:1] if same else plans
    dplans = {}
    if f.strategy == "dwq":
        for (d, u), rows in dwq_keys(f).items():
            pk = ("dwq_plan", d, u)
            if pk not in g:
                g[pk] = DwqPlan((f.b1, f.b2)[d], plans[d].layout, u, only_rows=rows)
            dplans[(d, u)] = g[pk]
    # every fit of the pass in ONE fused launch (tq_wq_fit_sets: warp per
    # moment system, own moments and collocation block), then every DWQ
    # combination in one launch; the basis tables the raw rows read at the
    # layout points (geometry: no dependence on the weights) go to a side
    # stream and overlap the fits
    main = torch.cuda.current_stream()
    sep = f.strategy != "reference" and f.coeff.identity       # the direction products are needed
    prods = [torch.empty((pl.basis.n, 2 * pl.basis.p + 1), dtype=torch.float64, device=f.dev)
             if sep and pl.rows_h.size == pl.basis.n else None for pl in fit_plans]
    dkeys = list(dplans)
    side = _side_streams(1)[0]
    with _forked(main, side):
        tabs = L.eval_many([(pl.basis, pl.layout.device_points()) for pl in fit_plans]
                           + [(dplans[k].basis, dplans[k].aug.device_points()) for k in dkeys])
        tables, dtables = tabs[: len(fit_plans)], tabs[len(fit_plans):]
        _st("tables")
        _keep_on(main, [t for tb in tables + dtables for t in tb])
    # the fits gate the whole pass: the highest stream priority, so their
    # blocks (and the combine's) dispatch ahead of the pass-start bulk work
    fs = _named_stream("fits", priority=-5)
    with _forked(main, fs):
        _QT[0] = "fit:"
        outs = fit_sets_async(fit_plans + [dplans[k].fit for k in dkeys], prods + [None] * len(dkeys),
                              [None] * len(fit_plans) + [False] * len(dkeys))
        _st("fits")
        fine = outs[len(fit_plans):]
        ws = combine_sets_async([dplans[k] for k in dkeys], fine)
        _st("combine")
        _QT[0] = ""
        _keep_on(main, [t for o in outs for t in o[1:]] + list(ws) + [p_ for p_ in prods if p_ is not None])
    main.wait_stream(fs)
    std = outs[: len(fit_plans)]
    if same:      # direction 2 reads direction 1's fits
        std, tables, prods = std * 2, tables * 2, prods * 2
    dwq_pending = {}
    for k, key, w, fo, tab in zip(range(len(dkeys)), dkeys, ws, fine, dtables):
        pl = dplans[key]
        rs = DiscontinuousRuleSet(pl.basis, pl.aug, pl.wptr, pl.k0, w, pl.u, pl.S, pl.refined, pl.base_layout,
                                  key[0], None)
        rs._basis_tab = tab
        dwq_pending[key] = (pl, rs, fo[3])
    main.wait_stream(side)
    _st("fits_joined")
    flags = [fl[: max(pl.rows_h.size, 1)] for pl, (_, _, _, fl) in zip(plans, std)]
    flags += [fl[: max(pl.fit.rows_h.size, 1)] for pl, _, fl in dwq_pending.values()]
    if f.capture is not None:
        # graph capture: the replay reduces the flags on a side stream (off
        # the critical path, joined at the end of the pass); the host reads
        # the one status word after the replay (GraphFormation.check)
        f._fail_any = None
        if flags:
            s = _named_stream("fit_status", priority=0)
            s.wait_stream(main)
            with torch.cuda.stream(s):
                f._fail_any = torch.cat(flags).any()
            f._status_streams = getattr(f, "_status_streams", []) + [s]
        any_fail = False
    else:
        any_fail = bool(torch.cat(flags).any().item()) if flags else False
    rules = []
    for d, (pl, (wptr, k0, w, fail)) in enumerate(zip(plans, std)):
        if any_fail and _failing(pl, fail):
            rules.append(compute_wq_rules(pl.basis, pl.layout, direction=d))   # enrichment retries
        else:
            rs = WeightedRuleSet(pl.basis, pl.layout, wptr, k0, w, d)
            if tables[d] is not None:
                rs._basis_tab = tables[d]      # the fit's own table at the same points
            rs._products = prods[d]            # direction products written by the solve
            rules.append(rs)
    dwq = {}
    for key, (pl, rs, fail) in dwq_pending.items():
        if any_fail and _failing(pl.fit, fail):
            rs = build_dwq(pl.basis, pl.base_layout, key[1], direction=key[0], plan=pl)
        dwq[key] = rs
    return rules[0], rules[1], dwq


def needs_raw(f):
    if f.strategy == "reference" or not f.coeff.identity:
        return True
    return cut_rows_host(f).size > 0


# the all-raw path (every active row raw: c != 1 or the `reference`
# strategy) keeps its raw blocks in the planes layout and forms the CSR in
# one pass (csrc/planes.cu); TQ_PLANES=0 selects the row-major blocks and the
# two count passes (A/B and the parity tests)
PLANES = os.environ.get("TQ_PLANES", "1") != "0"
STRIP_ROWS = 16
# 8-row strips of their own for the long-rule functions at the ends of
# direction 2 (smaller shared stage for the other strips); measured: more
# total kernel time at config 4 p = 8 (fixed per-strip cost), off
EDGE_STRIPS = os.environ.get("TQ_EDGE_STRIPS", "0") == "1"
# one strips launch (packed B2 rows) instead of one per shared-memory class:
# by occupancy (default), TQ_MERGED_STRIPS=1 always, =0 never
MERGED_STRIPS = os.environ.get("TQ_MERGED_STRIPS")


def planes(f):
    """Does this formation use the planes layout?"""
    return (PLANES and (f.strategy == "reference" or not f.coeff.identity) and f.b1.p == f.b2.p
            and 1 <= f.b1.p <= 10)


def planes_geo(f):
    """Storage map of the planes layout for this formation's row plan
    (geometry, cached): storage index of a row = its active index minus the
    plan's first one (the plan holds every active row of its lines), the
    per-function slot map with those indices, and the strips of the interior
    (whole-support box) rows for tq_sf_strips."""
    desc, nint = _plan(f)
    g = _geo(f.config)
    key = ("planes", id(desc))
    if key not in g:
        col_of = _col_of_host(f)
        fid = desc[:, 0].astype(np.int64)
        col = col_of[fid].astype(np.int64)
        base = int(col.min()) if col.size else 0
        store = col - base
        if col.size and not (store.max() == col.size - 1 and np.unique(store).size == col.size):
            raise RuntimeError("planes layout needs every active row of the plan's lines in the plan")
        slot = torch.full((f.b1.n * f.b2.n,), -1, dtype=torch.int32, device=f.dev)
        if fid.size:
            slot[torch.as_tensor(fid, device=f.dev)] = torch.as_tensor(store.astype(np.int32), device=f.dev)
        # interior rows [0, nint) for the strips (grouped per layout in strip_classes)
        n2 = f.b2.n
        i1, i2 = fid[:nint] // n2, fid[:nint] % n2
        full = ((desc[:nint, 1] == MODE_BOX) & (desc[:nint, 2] == 0) & (desc[:nint, 3] == 0)
                & (desc[:nint, 4] == f.b1._el_first[i1]) & (desc[:nint, 5] == f.b1._el_last[i1])
                & (desc[:nint, 6] == f.b2._el_first[i2]) & (desc[:nint, 7] == f.b2._el_last[i2]))
        interior = (i1, i2, store[:nint])
        g[key] = dict(base=base, store=L.dev(store.astype(np.int32), torch.int32), slot=slot,
                      interior=interior, strip_ok=bool(nint == 0 or full.all()), ld=int(col.size))
    return g[key]


def strip_classes(f, pg, layout1, layout2):
    """The interior rows grouped into strips and the strips split into
    launches by shared-memory need (cached per plan and layouts).  A WQ rule
    row lies in its support's points, so the support point counts bound the
    rows (the kernel flags any row that breaks them).  The functions at the
    ends of direction 2 whose rules are longer than the median (the boundary
    functions of an open knot vector) form 8-row strips of their own; the
    rest form 16-row strips aligned after them.  Launches: 16-row strips on
    regular lines, 16-row strips on long-rule lines, 8-row edge strips --
    each [(rows per strip, strips_dev, nstrips, n1m, n2m, nu_max, b2cap)]
    (b2cap: doubles of the packed B2 stage, tq_sf_strips)."""
    g = _geo(f.config)
    key = ("strip_classes", id(pg), id(layout1), id(layout2))
    if key not in g:
        i1, i2, sto = pg["interior"]
        out = []
        if i1.size:
            b1, b2 = f.b1, f.b2
            o1, o2 = layout1.offsets, layout2.offsets
            cnt1 = o1[b1._el_last + 1] - o1[b1._el_first]
            cnt2 = o2[b2._el_last + 1] - o2[b2._el_first]
            med1, med2 = int(np.median(cnt1)), int(np.median(cnt2))
            long2 = (cnt2 > med2) & EDGE_STRIPS
            half = b2.n // 2
            lo_l, hi_l = np.nonzero(long2[:half])[0], np.nonzero(long2[half:])[0]
            e_lo = int(lo_l.max()) + 1 if lo_l.size else 0                 # edge: [0, e_lo)
            mid_end = half + int(hi_l.min()) if hi_l.size else b2.n         # edge: [mid_end, n2)
            edge = (i2 < e_lo) | (i2 >= mid_end)
            # column chunk start of every interior row
            start = np.where(i2 < e_lo, (i2 // 8) * 8,
                             np.where(i2 >= mid_end, mid_end + ((i2 - mid_end) // 8) * 8,
                                      e_lo + ((i2 - e_lo) // STRIP_ROWS) * STRIP_ROWS))
            for ts, sel_rows in ((STRIP_ROWS, ~edge), (8, edge)):
                if not sel_rows.any():
                    continue
                r1_, s_, t_, st_ = i1[sel_rows], start[sel_rows], i2[sel_rows] - start[sel_rows], sto[sel_rows]
                skey = r1_.astype(np.int64) * (b2.n + 1) + s_
                uk, inv = np.unique(skey, return_inverse=True)
                strips = np.full((uk.size, 2 + ts), -1, np.int32)
                strips[inv, 0] = r1_
                strips[inv, 1] = s_
                strips[inv, 2 + t_] = st_
                rows = strips[:, 2:] >= 0
                t = np.arange(ts)
                ii2 = np.minimum(strips[:, 1:2] + t[None, :], b2.n - 1)
                lo = np.where(rows, t[None, :], ts).min(axis=1)
                hi = np.where(rows, t[None, :], -1).max(axis=1)
                c1 = cnt1[strips[:, 0]]
                c2 = np.where(rows, cnt2[ii2], 0).max(axis=1)
                nu = o2[b2._el_last[strips[:, 1] + hi] + 1] - o2[b2._el_first[strips[:, 1] + lo]]
                reg = (c1 <= med1) & (c2 <= med2)
                groups = (reg, ~reg) if ts == STRIP_ROWS else (c1 <= med1, c1 > med1)
                # packed B2 stage: each row sized by its own rule-length bound
                wp = 3 * ((2 * b1.p + 3) // 3)
                lens = np.where(rows, cnt2[ii2], 0)
                alloc = np.where(lens > 0, 2 * (((lens * wp + 1) // 2) | 1), 0).sum(axis=1)
                if ts == STRIP_ROWS and reg.any() and (~reg).any():
                    # one launch (packed rows) when it keeps the regular
                    # class's resident blocks per SM: no tail of a second
                    # launch (config 4 p = 8: 0.496 -> 0.478 ms)
                    occ = L.lib().tq_sf_strips_occupancy
                    merged = occ(b1.p, ts, int(c1.max()), int(c2.max()), max(int(nu.max()), 1), int(alloc.max()))
                    regular = occ(b1.p, ts, int(c1[reg].max()), int(c2[reg].max()), max(int(nu[reg].max()), 1), 0)
                    if MERGED_STRIPS == "1" or (MERGED_STRIPS is None and merged >= regular > 0):
                        groups = (np.ones_like(reg), )
                for k, sel in enumerate(groups):
                    if sel.any():
                        # the regular class keeps a fixed row stride (every row
                        # an equal odd number of 16-byte units: conflict-free
                        # stage-B reads); the long-rule class packs its rows
                        # (two blocks per SM instead of one)
                        packed = (k > 0 or len(groups) == 1) and ts == STRIP_ROWS
                        out.append((ts, L.dev(np.ascontiguousarray(strips[sel]), torch.int32), int(sel.sum()),
                                    int(c1[sel].max()), int(c2[sel].max()), max(int(nu[sel].max()), 1),
                                    int(alloc[sel].max()) if packed else 0))
        g[key] = out
        g[key + ("keep",)] = (layout1, layout2)       # the ids stay valid
    return g[key]


def _col_of_host(f):
    g = _geo(f.config)
    if "col_of_h" not in g:
        g["col_of_h"] = f.col_of.cpu().numpy()
    return g["col_of_h"]


def raw_buffer(f, ndesc):
    """Raw blocks of the plan: row-major (ndesc x W) or planes (W x ld)."""
    W = (2 * f.b1.p + 1) * (2 * f.b2.p + 1)
    if planes(f):
        return torch.empty((W, max(ndesc, 1)), dtype=torch.float64, device=f.dev)
    return torch.empty((max(ndesc, 1), W), dtype=torch.float64, device=f.dev)


def pairs_mode(f):
    """c != 1 planes path whose cut rows are formed element-centric from
    pair-form element blocks (csrc/cutrows.cu)."""
    return planes(f) and not f.coeff.identity and f.strategy != "reference" and f.b1.p <= 8


def gauss_elements(f):
    """Interior elements whose element-Gauss block a row of the plan reads
    (GAUSS rows: every interior support element; BOX rows: those outside the
    box) -- geometry of the plan, cached: element list (device, nslot x 2),
    element -> slot map, and the point gather indices of their Gauss grids."""
    desc, _ = _plan(f)
    g = _geo(f.config)
    key = ("gauss_el", id(desc))
    if key not in g:
        b1, b2 = f.b1, f.b2
        nel1, nel2 = b1.num_elements, b2.num_elements
        ec = f.config.element_class
        mark = np.zeros((nel1, nel2), bool)
        sel = desc[(desc[:, 1] == MODE_GAUSS) | (desc[:, 1] == MODE_BOX)]
        if sel.shape[0]:
            i1, i2 = sel[:, 0] // b2.n, sel[:, 0] % b2.n
            o1, o2 = np.arange(b1.p + 1), np.arange(b2.p + 1)
            e1 = b1._el_first[i1][:, None, None] + o1[None, :, None]
            e2 = b2._el_first[i2][:, None, None] + o2[None, None, :]
            e1, e2 = np.broadcast_arrays(e1, e2)
            ok = (e1 <= b1._el_last[i1][:, None, None]) & (e2 <= b2._el_last[i2][:, None, None])
            e1c, e2c = np.minimum(e1, nel1 - 1), np.minimum(e2, nel2 - 1)
            ok &= ec[e1c, e2c] == INTERIOR
            box = (sel[:, 1] == MODE_BOX) & (sel[:, 4] >= 0)
            inbox = (box[:, None, None] & (e1 >= sel[:, 4, None, None]) & (e1 <= sel[:, 5, None, None])
                     & (e2 >= sel[:, 6, None, None]) & (e2 <= sel[:, 7, None, None]))
            ok &= ~inbox
            mark[e1c[ok], e2c[ok]] = True
        el = np.argwhere(mark).astype(np.int32)        # row-major element order
        slot = np.full(nel1 * nel2, -1, np.int32)
        slot[el[:, 0].astype(np.int64) * nel2 + el[:, 1]] = np.arange(el.shape[0], dtype=np.int32)
        q1, q2 = b1.p + 1, b2.p + 1
        gi = (el[:, 0].astype(np.int64)[:, None, None] * q1 + np.arange(q1)[None, :, None])
        gj = (el[:, 1].astype(np.int64)[:, None, None] * q2 + np.arange(q2)[None, None, :])
        gi, gj = np.broadcast_arrays(gi, gj)
        g[key] = dict(n=int(el.shape[0]), gel=L.dev(el if el.size else np.zeros((1, 2), np.int32), torch.int32),
                      gslot=L.dev(slot, torch.int32),
                      idx1=L.dev(gi.reshape(-1) if el.size else np.zeros(1, np.int64), torch.int64),
                      idx2=L.dev(gj.reshape(-1) if el.size else np.zeros(1, np.int64), torch.int64))
    return g[key]


def _gauss_pairs(f, eg, em):
    """Element-Gauss blocks (pair form) of the plan's Gauss elements on the
    current stream; c = det J computed in the kernel for a geometry map,
    else evaluated at just their Gauss points."""
    from .assembly import GeometryMap
    ge = gauss_elements(f)
    npair = int(L.lib().tq_pair_block_doubles(f.b1.p))
    E = torch.empty(max(ge["n"], 1) * npair, dtype=torch.float64, device=f.dev)
    if ge["n"]:
        ctx = _gauss_ctx(f, eg, em, None, _desc_dev(f)[0], torch.empty(1, dtype=torch.float64, device=f.dev), 0)
        dev = getattr(f.coeff, "_device", None) or f.coeff
        lines = [None] * 4
        if isinstance(dev, GeometryMap):
            geo, cgp = dev.device(), None
            lines = []
            for d in range(2):      # line tables of the element Gauss points (tiny; per pass)
                X = eg[d][3]
                sp = torch.empty(X.numel(), dtype=torch.int32, device=f.dev)
                nd = torch.empty(X.numel() * 2 * (dev.p + 1), dtype=torch.float64, device=f.dev)
                L.call("tq_geo_lines", geo, L.ptr(X), X.numel(), L.ptr(sp), L.ptr(nd), L.stream())
                lines += [sp, nd]
            f._keep_pairs = getattr(f, "_keep_pairs", []) + lines
        else:
            P = torch.stack([eg[0][3][ge["idx1"]], eg[1][3][ge["idx2"]]], dim=1)
            geo, cgp = L.Coeff(), f.coeff.at_device(P)
            f._keep_pairs = getattr(f, "_keep_pairs", []) + [P, cgp]
        L.call("tq_gauss_pairs", ctx, geo, L.ptr(eg[0][3]), L.ptr(eg[1][3]), L.ptr(ge["gel"]), ge["n"], L.ptr(cgp),
               L.ptr(E), *[L.ptr(t) for t in lines], L.stream())
    return E, ge["gslot"]


def _cut_pieces(f, cut):
    """Pieces of the span-key groups for tq_cut_pairs (geometry, cached with
    the cut-point tables): (pieces npieces x 2 int64, gpiece int32, npieces)."""
    t = cut_point_tables(f)
    if "pieces" not in t:
        kp = int(L.lib().tq_cut_pair_piece())
        gp = t["grp_pts"]
        ng = t["ngroups"]
        lens = gp[1:] - gp[:-1]
        npc = (lens + kp - 1) // kp
        gpiece = torch.zeros(ng + 1, dtype=torch.int64, device=f.dev)
        gpiece[1:] = torch.cumsum(npc, 0)
        npieces = int(gpiece[-1].item()) if ng else 0
        grp = torch.repeat_interleave(torch.arange(ng, device=f.dev), npc)
        within = torch.arange(npieces, device=f.dev) - gpiece[:-1][grp]
        pieces = torch.stack([grp, gp[:-1][grp] + kp * within], dim=1).contiguous()
        t["pieces"] = (pieces if npieces else torch.zeros((1, 2), dtype=torch.int64, device=f.dev),
                       gpiece.to(torch.int32), npieces)
    return t["pieces"]


# the cut-cell rows gathered over per-row group lists (geometry, built once
# per plan on the device) instead of scanning each row's element window
CUTCELL_LISTS = os.environ.get("TQ_CUTCELL_LISTS", "1") == "1"


def raw_row_groups(f):
    """Span-key groups of every raw row of the plan, in tq_raw_cutcells's
    order (tq_row_groups: counts, prefix, triplets) -- geometry, cached per
    plan and cut-point tables: (rg_ptr int32 ndesc + 1, rg int32 3 x total)."""
    desc, _ = _plan(f)
    t = cut_point_tables(f)
    g = _geo(f.config)
    key = ("raw_row_groups", id(desc), id(t))
    if key not in g:
        n = int(f._ndesc)
        counts = torch.empty(max(n, 1), dtype=torch.int32, device=f.dev)
        L.call("tq_row_groups", f._ctx, 0, n, None, L.ptr(counts), L.stream())
        rg_ptr = torch.zeros(n + 1, dtype=torch.int32, device=f.dev)
        if n:
            rg_ptr[1:] = torch.cumsum(counts[:n], 0)
        # a (row, group) pair appears once and a group reaches the (p1+1)(p2+1)
        # functions of its key: that bounds the total without a host read
        cap = int(t["ngroups"]) * (f.b1.p + 1) * (f.b2.p + 1)
        rg = torch.empty(max(3 * cap, 3), dtype=torch.int32, device=f.dev)
        L.call("tq_row_groups", f._ctx, 0, n, L.ptr(rg_ptr), L.ptr(rg), L.stream())
        g[key] = (rg_ptr, rg)
        g[key + ("keep",)] = (desc, t)
    return g[key]


def cut_row_groups(f, r0, r1):
    """Span-key groups each cut row [r0, r1) of the plan reads (cut elements
    within one element of its support, groups in element / key order, key
    within the row's reach) -- geometry, cached: (rg_ptr, rg) device int32."""
    desc, _ = _plan(f)
    t = cut_point_tables(f)
    g = _geo(f.config)
    key = ("row_groups", id(desc), id(t), r0, r1)
    if key not in g:
        b1, b2 = f.b1, f.b2
        nel1, nel2 = b1.num_elements, b2.num_elements
        if "host" not in t:
            t["host"] = (t["idx"].cpu().numpy(), t["grp_ptr"].cpu().numpy().astype(np.int64),
                         t["grp_key"].cpu().numpy())
        cutidx, gptr, gkey = t["host"]
        fid = desc[r0:r1, 0].astype(np.int64)
        i1, i2 = fid // b2.n, fid % b2.n
        ea1 = np.maximum(b1._el_first[i1] - 1, 0)
        eb1 = np.minimum(b1._el_last[i1] + 1, nel1 - 1)
        ea2 = np.maximum(b2._el_first[i2] - 1, 0)
        eb2 = np.minimum(b2._el_last[i2] + 1, nel2 - 1)
        w1 = int(np.max(eb1 - ea1 + 1)) if fid.size else 0
        w2 = int(np.max(eb2 - ea2 + 1)) if fid.size else 0
        e1 = ea1[:, None, None] + np.arange(w1)[None, :, None]
        e2 = ea2[:, None, None] + np.arange(w2)[None, None, :]
        e1, e2 = np.broadcast_arrays(e1, e2)
        ok = (e1 <= eb1[:, None, None]) & (e2 <= eb2[:, None, None])
        row = np.broadcast_to(np.arange(fid.size)[:, None, None], e1.shape)[ok]
        cid = cutidx[np.minimum(e1, nel1 - 1)[ok].astype(np.int64) * nel2 + np.minimum(e2, nel2 - 1)[ok]]
        row, cid = row[cid >= 0], cid[cid >= 0]
        cnt = gptr[cid + 1] - gptr[cid]
        rrow = np.repeat(row, cnt)
        start = np.repeat(gptr[cid], cnt)
        off = np.arange(rrow.size) - np.repeat(np.cumsum(cnt) - cnt, cnt)
        grp = (start + off).astype(np.int64)
        k1, k2 = gkey[grp, 0], gkey[grp, 1]
        a1, a2 = i1[rrow] - k1, i2[rrow] - k2
        keep = (a1 >= 0) & (a1 <= b1.p) & (a2 >= 0) & (a2 <= b2.p)
        rrow, grp, k1, k2 = rrow[keep], grp[keep], k1[keep], k2[keep]
        rg_ptr = np.zeros(fid.size + 1, np.int32)
        rg_ptr[1:] = np.cumsum(np.bincount(rrow, minlength=fid.size))
        rg = np.stack([grp, k1, k2], axis=1).astype(np.int32)
        g[key] = (L.dev(rg_ptr, torch.int32), L.dev(rg if rg.size else np.zeros((1, 3), np.int32), torch.int32))
        g[key + ("keep",)] = t
    return g[key]


def _cut_pairs(f, cut):
    """Span-key group blocks (pair form) of the cut elements (current stream)."""
    npair = int(L.lib().tq_pair_block_doubles(f.b1.p))
    E = torch.empty(max(cut["ngroups"], 1) * npair, dtype=torch.float64, device=f.dev)
    pieces, gpiece, npieces = _cut_pieces(f, cut)
    if cut["ngroups"]:
        part = torch.empty(max(npieces, 1) * npair, dtype=torch.float64, device=f.dev)
        # every group (the pieces index groups absolutely; a row block's
        # rows read only some, the rest is small replicated work)
        L.call("tq_cut_pairs", _cut_blocks_ctx(f, cut), L.ptr(pieces), npieces,
               L.ptr(gpiece), L.ptr(part), L.ptr(E), L.stream())
        f._keep_pairs = getattr(f, "_keep_pairs", []) + [part]
    return E


class _Setup:
    """Device tables shared by the raw-row kernels of one formation."""

    def __init__(self, f):
        _bind()
        self.keep = []
        b1, b2 = f.b1, f.b2
        cfg = f.config
        dev = f.dev
        # (a proxy: the formation owns this object, and a strong reference
        # back would leave the pass's device tables to the cyclic collector)
        self.f = weakref.proxy(f)
        # element Gauss tables, (p+1) points (src/assembly.py:198-211);
        # basis values evaluated per formation as in the reference's _Run
        pre = getattr(f, "_elem_pre", None)
        self.eg, self.em, self.cg = pre if pre is not None else _elem_tables(f, with_grid=not pairs_mode(f))
        # rule sets
        self.sets = ([], [])
        self.grids = None
        self.grids_all = None          # event: every rule-set pair's grid evaluated
        self.key_index = _key_index(f)
        if f.rules is not None:
            r1, r2, dwq = f.rules
            self.sets[0].append(r1)
            self.sets[1].append(r2)
            ki = ({}, {})
            for (d, u), rs in sorted(dwq.items()):
                ki[d][u] = len(self.sets[d])
                self.sets[d].append(rs)
            self.key_index = ki       # imported rules may carry extra keys
            self.sets_dev = []
            for d, b in enumerate((b1, b2)):
                arr = (RuleSetDev * len(self.sets[d]))()
                for k, rs in enumerate(self.sets[d]):
                    first, vals = rs.basis_table()
                    arr[k] = RuleSetDev(rs.device(), rs.layout.device(), L.ptr(first), L.ptr(vals))
                t = L.dev_bytes(bytearray(arr))
                self.sets_dev.append(t)
            self.nmax = []
            self.nmax_std = []      # the standard rules alone (interior rows read set 0 only)
            for d, b in enumerate((b1, b2)):
                ms = []
                for rs in self.sets[d]:
                    off = rs.layout.offsets
                    ms.append(int(np.max(off[b._el_last + 1] - off[b._el_first])))
                self.nmax.append(max(ms))
                self.nmax_std.append(ms[0])
            if not f.coeff.identity:
                pre = getattr(f, "_grids_pre", None)
                lays = ([s.layout for s in self.sets[0]], [s.layout for s in self.sets[1]])
                if pre is not None and all(len(a) == len(b) and all(x is y for x, y in zip(a, b))
                                           for a, b in zip(pre[0], lays)):
                    # computed at pass start on its own stream (prelaunch_grids):
                    # the interior rows read the standard grid only; the
                    # launches that read the DWQ sets' grids wait for all
                    # (wait_all_grids)
                    torch.cuda.current_stream().wait_event(pre[4])
                    self.grids = pre[1]
                    self.grids_all = pre[2]
                else:
                    ptrs = np.zeros(len(self.sets[0]) * len(self.sets[1]), dtype=np.uint64)
                    for a, s1 in enumerate(self.sets[0]):
                        for c, s2 in enumerate(self.sets[1]):
                            g = f.coeff.grid_device(s1.layout.device_points(), s2.layout.device_points())
                            self.keep.append(g)
                            ptrs[a * len(self.sets[1]) + c] = g.data_ptr()
                    self.grids = L.dev(ptrs.view(np.int64), torch.int64)
                _st("grids")
        else:
            self.sets_dev = [None, None]
            self.nmax = [1, 1]
            self.nmax_std = [1, 1]
        # cut-element points (host C++ geometry, device basis tables); taken
        # from the pass-start launch when the pass made one
        pre = getattr(f, "_cut_pre", None)
        self.cut = pre if pre is not None else (_cut_tables(f) if f.config.has_cuts() else None)

    def wait_all_grids(self):
        """Current stream waits until every rule-set pair's coefficient grid
        exists (the pass-start grids signal the standard one first)."""
        if self.grids_all is not None:
            torch.cuda.current_stream().wait_event(self.grids_all)

    def ctx(self, desc, raw, nraw):
        f = self.f
        d1, d2 = f.b1.device_arrays(), f.b2.device_arrays()
        cut = self.cut or {}
        P = L.ptr
        ctx = RawCtx(f.b1.n, f.b2.n, f.b1.p, f.b2.p, f.b1.num_elements, f.b2.num_elements,
                      P(d1["el_first"]), P(d1["el_last"]), P(d2["el_first"]), P(d2["el_last"]),
                      P(d1["ov_lo"]), P(d1["ov_hi"]), P(d2["ov_lo"]), P(d2["ov_hi"]),
                      P(d1["espan"]), P(d2["espan"]), P(f.config.element_class_dev),
                      f.b1.p + 1, f.b2.p + 1,
                      P(self.eg[0][1]), P(self.eg[0][2]), P(self.eg[1][1]), P(self.eg[1][2]), P(self.em[0]),
                      P(self.em[1]),
                      P(self.cg), P(self.sets_dev[0]), P(self.sets_dev[1]),
                      len(self.sets[0]), len(self.sets[1]), P(self.grids),
                      P(cut.get("idx")), P(cut.get("ptr")), P(cut.get("cw")), P(cut.get("f1")), P(cut.get("v1")),
                      P(cut.get("f2")), P(cut.get("v2")), P(cut.get("grp_ptr")), P(cut.get("grp_key")),
                      P(cut.get("grp_pts")), P(cut.get("grp_perm")), P(cut.get("blocks")), cut.get("ngroups", 0),
                      P(desc), nraw, self.nmax[0], self.nmax[1], P(raw))
        if planes(f):
            pg = planes_geo(f)
            ctx.store, ctx.raw_ld = P(pg["store"]), pg["ld"]
        return ctx


def _elem_tables(f, with_grid=True):
    """Element Gauss tables ((p+1) points, src/assembly.py:198-211), the
    per-element 1-D mass blocks and (c != 1) the coefficient on the Gauss
    grid; basis values evaluated per formation as in the reference's _Run."""
    eg, em = [], []
    pts = element_points(f)
    same = f.b1.p == f.b2.p and np.array_equal(f.b1.kv.knots, f.b2.kv.knots)   # one table serves both
    dirs = ((f.b1, pts[0]),) if same else tuple(zip((f.b1, f.b2), pts))
    tabs = L.eval_many([(b, Xd) for b, (Xd, _) in dirs])
    for b, (Xd, Wd), (_, vals) in zip([d[0] for d in dirs], [d[1] for d in dirs], tabs):
        eg.append((None, Wd, vals, Xd))
        m = torch.empty(b.num_elements * (b.p + 1) ** 2, dtype=torch.float64, device=f.dev)
        L.call("tq_elem_mass", L.ptr(vals), L.ptr(Wd), b.num_elements, b.p + 1, b.p, L.ptr(m), L.stream())
        em.append(m)
    if same:
        eg, em = eg * 2, em * 2
    cg = None if (f.coeff.identity or not with_grid) else f.coeff.grid_device(eg[0][3], eg[1][3])
    return eg, em, cg


def _key_index(f):
    """Rule-set index per DWQ key and direction: 0 = standard rules, then
    the DWQ sets in sorted key order (geometry: known before the fits)."""
    ki = ({}, {})
    if f.strategy == "dwq":
        cnt = [1, 1]
        for d, u in sorted(dwq_keys(f)):
            ki[d][u] = cnt[d]
            cnt[d] += 1
    return ki


def _gauss_ctx(f, eg, em, cg, desc, raw, nraw):
    """Context of the element-Gauss part of the raw rows (no rule sets)."""
    d1, d2 = f.b1.device_arrays(), f.b2.device_arrays()
    P = L.ptr
    ctx = RawCtx(n1=f.b1.n, n2=f.b2.n, p1=f.b1.p, p2=f.b2.p, nel1=f.b1.num_elements, nel2=f.b2.num_elements,
                  el_first1=P(d1["el_first"]), el_last1=P(d1["el_last"]), el_first2=P(d2["el_first"]),
                  el_last2=P(d2["el_last"]), ov_lo1=P(d1["ov_lo"]), ov_hi1=P(d1["ov_hi"]), ov_lo2=P(d2["ov_lo"]),
                  ov_hi2=P(d2["ov_hi"]), espan1=P(d1["espan"]), espan2=P(d2["espan"]),
                  elem_class=P(f.config.element_class_dev), ng1=f.b1.p + 1, ng2=f.b2.p + 1,
                  ew1=P(eg[0][1]), ev1=P(eg[0][2]), ew2=P(eg[1][1]), ev2=P(eg[1][2]), em1=P(em[0]), em2=P(em[1]),
                  cg=P(cg), desc=P(desc), nraw=nraw, nmax1=1, nmax2=1, raw=P(raw))
    if planes(f):
        pg = planes_geo(f)
        ctx.store, ctx.raw_ld = P(pg["store"]), pg["ld"]
    return ctx


def _cut_tables(f):
    """Cut-element point tables, their basis values and weights (no
    dependence on the WQ fits)."""
    b1, b2 = f.b1, f.b2
    t = cut_point_tables(f)
    (f1, v1), (f2, v2) = L.eval_many([(b1, t["x"]), (b2, t["y"])])
    cw = f.coeff.at_device(t["P"]) * t["W"] if not f.coeff.identity else t["W"]
    Q = (b1.p + 1) * (b2.p + 1)
    f.report.n_cutcell_points = t["npts"]
    return dict(idx=t["idx"], ptr=t["ptr"], cw=cw.contiguous(), f1=f1, v1=v1, f2=f2, v2=v2,
                npts=t["npts"], grp_ptr=t["grp_ptr"], grp_key=t["grp_key"], grp_pts=t["grp_pts"],
                grp_perm=t["grp_perm"], ngroups=t["ngroups"],
                blocks=torch.empty(1 if pairs_mode(f) else max(t["ngroups"], 1) * Q * Q, dtype=torch.float64,
                                   device=f.dev))


def _group_range(f, cut):
    """Span-key groups of the cut elements a row block reads: elements in
    the supports of the block's raw-row window (cut elements and their
    groups are stored in row-major element order: one contiguous range)."""
    win = line_window(f)
    if win is None:
        return 0, cut["ngroups"]
    g = _geo(f.config)
    key = ("groups", win, id(cut["grp_ptr"]))
    if key not in g:
        rule = f.config.cut_cell_rule(max(f.b1.p, f.b2.p))
        e1 = rule.elements[:, 0]
        # the gather reads one element beyond each raw row's support
        lo_e = max(int(f.b1._el_first[win[0]]) - 1, 0) if win[1] >= win[0] else 0
        hi_e = min(int(f.b1._el_last[win[1]]) + 1, f.b1.num_elements - 1) if win[1] >= win[0] else -1
        c0 = int(np.searchsorted(e1, lo_e, side="left"))
        c1 = int(np.searchsorted(e1, hi_e, side="right"))
        gp = cut["grp_ptr"].cpu().numpy()
        g[key] = (int(gp[c0]), int(gp[c1]))
    return g[key]


def _cut_blocks_ctx(f, cut, groups=None):
    """tq_cut_blocks context; ``groups`` = (g0, g1) restricts the launch to
    that group range (pointer offsets, no kernel change)."""
    P = L.ptr
    g0, g1 = groups if groups is not None else (0, cut["ngroups"])
    Q = (f.b1.p + 1) * (f.b2.p + 1)
    return RawCtx(n1=f.b1.n, n2=f.b2.n, p1=f.b1.p, p2=f.b2.p, nel1=f.b1.num_elements, nel2=f.b2.num_elements,
                  cutidx=P(cut["idx"]), cut_ptr=P(cut["ptr"]), cut_cw=P(cut["cw"]), cfirst1=P(cut["f1"]),
                  cvals1=P(cut["v1"]), cfirst2=P(cut["f2"]), cvals2=P(cut["v2"]), grp_ptr=P(cut["grp_ptr"]),
                  grp_key=P(cut["grp_key"]), grp_pts=L.vp(cut["grp_pts"].data_ptr() + 8 * g0),
                  grp_perm=P(cut["grp_perm"]), grp_blocks=L.vp(cut["blocks"].data_ptr() + 8 * Q * Q * g0),
                  ngroups=max(g1 - g0, 0))


_NAMED = {}


def _named_stream(name, priority=0):
    """Cached side stream.  Priorities (lower = more urgent): fit chains -3;
    the captured main chain and the pass-start streams (Gauss part of the raw
    rows, cut-element blocks: both gate the cut-row chain) -2."""
    dev = torch.cuda.current_device()
    key = (dev, name)
    if key not in _NAMED:
        priority = int(os.environ.get("TQ_PRIO_" + name.upper(), priority))   # tuning knob
        _NAMED[key] = torch.cuda.Stream(priority=priority)
    return _NAMED[key]


def prelaunch_grids(f):
    """Coefficient grids of every rule-set pair at pass start, on their own
    stream (they depend on the point layouts -- geometry, cached by the eager
    pass -- and the coefficient field, not on the weights)."""
    if f.coeff.identity or f.strategy == "reference":
        return
    g = _geo(f.config)
    if "std_plans" not in g:
        return
    lays = [[g["std_plans"][d].layout] for d in (0, 1)]
    if f.strategy == "dwq":
        for (d, u) in dwq_keys(f):
            pk = ("dwq_plan", d, u)
            if pk not in g:
                return
            lays[d].append(g[pk].aug)
    s = _named_stream("grids", priority=-3)
    main = torch.cuda.current_stream()
    from .assembly import _padded_grid
    with _forked(main, s):
        # every grid buffer first, so the pointer table is uploaded ahead of
        # the evaluations; the standard x standard grid (the only one the
        # interior strips read) is evaluated first and signalled on its own
        pts = ([l.device_points() for l in lays[0]], [l.device_points() for l in lays[1]])
        keep = [[_padded_grid(x1.numel(), x2.numel(), f.dev) for x2 in pts[1]] for x1 in pts[0]]
        ptrs = np.array([g.data_ptr() for row in keep for g in row], dtype=np.uint64)
        table = L.dev(ptrs.view(np.int64), torch.int64)
        ev_std = None
        for a, x1 in enumerate(pts[0]):
            for c, x2 in enumerate(pts[1]):
                f.coeff.grid_device(x1, x2, out=keep[a][c])
                if ev_std is None:
                    ev_std = torch.cuda.Event()
                    ev_std.record()
        keep = [g for row in keep for g in row]
        ev = torch.cuda.Event()
        ev.record()
    for st in (main, _side_streams(1)[0]):
        _keep_on(st, keep + [table])
    f._grids_pre = (lays, table, ev, keep, ev_std)


def _gather_ctx(f, eg, em, cut, desc_dev, raw, ndesc):
    """Context of tq_cut_rows_gather before the rule sets exist."""
    ctx = _gauss_ctx(f, eg, em, None, desc_dev, raw, ndesc)
    if cut is not None:
        cc = _cut_blocks_ctx(f, cut)
        for k in ("cutidx", "cut_ptr", "cut_cw", "cfirst1", "cvals1", "cfirst2", "cvals2", "grp_ptr", "grp_key",
                  "grp_pts", "grp_perm", "ngroups"):
            setattr(ctx, k, getattr(cc, k))
    return ctx


# launch order at pass start: the cut-element chain (tables -> blocks) before
# the element-Gauss chain in pairs mode (config 4: p = 8 0.524 -> 0.522 ms,
# p = 6 0.300 -> 0.294 ms), after it otherwise (config 5: 0.703 vs 0.711 ms);
# TQ_CUT_FIRST=0/1 forces either
CUT_FIRST = os.environ.get("TQ_CUT_FIRST")


def prelaunch_geometry(f):
    """Start the WQ-independent raw-row work of a captured pass on its own
    stream, overlapping the fits: element tables, the element-Gauss part of
    every raw row (tq_raw_gauss), the cut-element tables and blocks.  The
    interior phase waits for the Gauss part (event), the cut-cell gather
    joins the stream (``join_cut_blocks``)."""
    if not needs_raw(f):
        return
    _bind()
    # priority of the main chain: the Gauss part gates the cut-row chain (measured best)
    s = _named_stream("cut_blocks", priority=-2)
    s2 = _named_stream("cut_blocks2", priority=-2)
    main = torch.cuda.current_stream()
    pm = pairs_mode(f)
    st = {}

    def gauss_part():
        with _forked(main, s):
            f._elem_pre = st["eg"] = _elem_tables(f, with_grid=not pm)
            eg, em, cg = st["eg"]
            _st("preA:elem")
            st["desc"] = desc_dev, ndesc = _desc_dev(f)
            f._desc_pre = desc_dev
            f._raw_pre = raw_buffer(f, ndesc)
            if pm:
                f._gpairs = _gauss_pairs(f, eg, em)
            elif ndesc:
                L.call("tq_raw_gauss", _gauss_ctx(f, eg, em, cg, desc_dev, f._raw_pre, ndesc), 0, ndesc, L.stream())
            _st("preA:gauss")
            f._elem_event = torch.cuda.Event()
            f._elem_event.record()

    def cut_part():
        # cut-element tables and blocks: an independent chain on a second stream
        cut = None
        with _forked(main, s2):
            if f.config.has_cuts():
                cut = _cut_tables(f)
                _st("preB:tables")
                if pm:
                    f._cpairs = _cut_pairs(f, cut)
                else:
                    L.call("tq_cut_blocks", _cut_blocks_ctx(f, cut, _group_range(f, cut)), L.stream())
            from .assembly import _stamp
            _stamp("cutpre:blocks")
        st["cut"] = cut

    cut_first = pm if CUT_FIRST is None else CUT_FIRST == "1"
    for part in ((cut_part, gauss_part) if cut_first else (gauss_part, cut_part)):
        part()
    eg, em, cg = st["eg"]
    desc_dev, ndesc = st["desc"]
    cut = st["cut"]
    s.wait_stream(s2)         # one stream to join later
    if pm:
        # the cut rows' element parts need no weights: gathered on the
        # pass-start stream as soon as both block sets exist
        desc, nint = _plan(f)
        if ndesc > nint:
            f._planes_status = torch.zeros(1, dtype=torch.int32, device=f.dev)     # (main: before every user)
            with _forked(main, s):
                Eg, gslot = f._gpairs
                Ec = getattr(f, "_cpairs", None)
                rg_ptr, rg = cut_row_groups(f, nint, ndesc) if Ec is not None else (None, None)
                L.call("tq_cut_rows_gather", _gather_ctx(f, eg, em, cut, desc_dev, f._raw_pre, ndesc), nint, ndesc,
                       L.ptr(gslot), L.ptr(Eg), L.ptr(Ec), L.ptr(rg_ptr), L.ptr(rg), L.ptr(f._planes_status),
                       L.stream())
                _st("preA:gather")
            f._gathered = True
    # tensors made here are consumed on the main and raw side streams
    tensors = [t for t in (cut or {}).values() if isinstance(t, torch.Tensor)]
    tensors += [t for e in eg for t in e if isinstance(t, torch.Tensor)] + list(em) + [f._raw_pre]
    tensors += [cg] if cg is not None else []
    tensors += list(getattr(f, "_gpairs", ())) + ([f._cpairs] if getattr(f, "_cpairs", None) is not None else [])
    tensors += getattr(f, "_keep_pairs", [])
    for st in (main, _side_streams(1)[0]):
        _keep_on(st, tensors)
    f._cut_pre = cut
    f._cut_stream = s


# count pass 1 launched speculatively at pass start (captured passes).  Off:
# measured 0.737 -> 0.743 ms per step at config 5 -- the pre-fill phase is
# throughput-bound across its concurrent streams, so starting the pass
# earlier only delays the pass-start streams (the cut-row chain gates the
# join).  Kept (and tested) for passes where the count pass is the gate.
SPEC_COUNTS = os.environ.get("TQ_SPEC_COUNTS", "0") == "1"


def prelaunch_counts(f):
    """Count pass 1 of a captured pass at pass start, on its own stream,
    overlapping the fits: it reads only the cached geometric deep flags and
    assumes every line's factors positive (tq_row_counts_spec); ``finish``
    checks the positivity once the factors exist and redoes the pass on the
    device only if some line is not positive (tq_row_counts_verify).  Needs
    the geometry cached by an earlier eager pass of the same plan."""
    if not SPEC_COUNTS or not f.separable():
        return
    g = _geo(f.config)
    raw_list = f.raw_list
    if needs_raw(f):
        desc, _ = _plan(f)
        skey = ("slot", id(desc))
        if skey not in g:
            return
        raw_list = g[skey][1]
    gkey = ("deep_geo", id(raw_list) if raw_list.numel() else None)
    if gkey not in g:
        return
    rb, re_ = (0, f.K) if f.row_range is None else f.row_range
    nrows = re_ - rb
    f.deep = g[gkey][0]
    spec = dict(rows=(rb, re_),
                rowfast=torch.empty(max(nrows, 1), dtype=torch.int8, device=f.dev),
                counts=torch.empty(max(nrows, 1), dtype=torch.int32, device=f.dev),
                work=torch.empty(2 * nrows + 2, dtype=torch.int32, device=f.dev),
                tiles=torch.empty(L.tile_ints(nrows), dtype=torch.int32, device=f.dev),
                bad=torch.empty(1, dtype=torch.int32, device=f.dev))
    f.rowfast = spec["rowfast"]
    ctx = f.rowctx(rb, re_)
    ctx.counts, ctx.tiles = L.ptr(spec["counts"]), L.ptr(spec["tiles"])
    s = _named_stream("counts_spec", priority=-2)
    main = torch.cuda.current_stream()
    with _forked(main, s):
        L.call("tq_row_counts_spec", ctx, L.ptr(f.deep), L.ptr(spec["counts"]), L.ptr(spec["work"]), L.stream())
        from .assembly import _stamp
        _stamp("spec:counts")
    spec["stream"] = s
    f._spec = spec


def join_cut_blocks(f):
    s = getattr(f, "_cut_stream", None)
    if s is not None:
        torch.cuda.current_stream().wait_stream(s)
        f._cut_stream = None


def _plan_full(f):
    """Raw rows and their descriptors for the whole matrix (host bookkeeping,
    cached per configuration / strategy / coefficient kind / DWQ key set)."""
    setup = getattr(f, "_setup", None)
    ki = setup.key_index if setup is not None else _key_index(f)
    key = ("plan", f.strategy, f.coeff.identity, tuple(sorted(ki[0].items())), tuple(sorted(ki[1].items())))
    g = _geo(f.config)
    if key not in g:
        g[key] = _plan_uncached(f, ki)
    return g[key]


def line_window(f):
    """Direction-1 lines [lo, hi] whose raw rows a row block needs: its own
    lines and the partner lines within p1 (|j1 - i1| <= p1 for every entry
    of a block row).  None: the whole matrix."""
    rr = getattr(f, "row_range", None)
    if rr is None or (rr[0] <= 0 and rr[1] >= f.K):
        return None
    g = _geo(f.config)
    key = ("lines", tuple(rr))
    if key not in g:
        n2 = f.b2.n
        if rr[1] <= rr[0]:
            g[key] = (0, -1)
        else:
            a = int(f.active[rr[0]].item()) // n2
            b = int(f.active[rr[1] - 1].item()) // n2
            g[key] = (max(a - f.b1.p, 0), min(b + f.b1.p, f.b1.n - 1))
    return g[key]


def _plan(f):
    """The raw-row plan of this formation: the whole matrix, or -- for a row
    block (multi-GPU sharding) -- only the raw rows on the block's line
    window, so each rank forms the raw rows its block reads."""
    desc, nint = _plan_full(f)
    win = line_window(f)
    if win is None:
        return desc, nint
    g = _geo(f.config)
    key = ("plan_window", id(desc), win)
    if key not in g:
        i1 = desc[:, 0] // f.b2.n
        keep = (i1 >= win[0]) & (i1 <= win[1])
        g[key] = (desc[keep], int(np.count_nonzero(keep[:nint])), desc)   # (the full plan kept alive)
    d, n, _ = g[key]
    return d, n


def gauss_element_count(f):
    """Distinct interior elements whose element-Gauss block the strategy
    computes (FormationReport.n_gauss_elements; src/assembly.py:310-332):
    the supports of GAUSS rows and the residual (outside-box) supports of
    BOX rows, interior elements only.  Geometry of the row plan, cached."""
    desc, _ = _plan_full(f)
    g = _geo(f.config)
    key = ("ngauss", id(desc))
    if key not in g:
        sel = desc[(desc[:, 1] == MODE_GAUSS) | (desc[:, 1] == MODE_BOX)]
        b1, b2 = f.b1, f.b2
        ec = f.config.element_class
        mark = np.zeros(ec.shape, bool)
        if sel.shape[0]:
            i1, i2 = sel[:, 0] // b2.n, sel[:, 0] % b2.n
            o1 = np.arange(b1.p + 1)
            o2 = np.arange(b2.p + 1)
            e1 = b1._el_first[i1][:, None, None] + o1[None, :, None]
            e2 = b2._el_first[i2][:, None, None] + o2[None, None, :]
            e1, e2 = np.broadcast_arrays(e1, e2)
            ok = (e1 <= b1._el_last[i1][:, None, None]) & (e2 <= b2._el_last[i2][:, None, None])
            e1c = np.minimum(e1, ec.shape[0] - 1)
            e2c = np.minimum(e2, ec.shape[1] - 1)
            ok &= ec[e1c, e2c] == INTERIOR
            box = (sel[:, 1] == MODE_BOX) & (sel[:, 4] >= 0)
            inbox = (box[:, None, None] & (e1 >= sel[:, 4, None, None]) & (e1 <= sel[:, 5, None, None])
                     & (e2 >= sel[:, 6, None, None]) & (e2 <= sel[:, 7, None, None]))
            ok &= ~inbox
            mark[e1c[ok], e2c[ok]] = True
        g[key] = int(mark.sum())
    return g[key]


def _desc_dev(f):
    """Device copy of the row plan's descriptors (cached) and its size."""
    desc, _ = _plan(f)
    g = _geo(f.config)
    dkey = ("desc", id(desc))
    if dkey not in g:
        g[dkey] = L.dev(desc, torch.int32)
    return g[dkey], desc.shape[0]


def _plan_uncached(f, key_index):
    n2 = f.b2.n
    interior_raw = f.strategy == "reference" or not f.coeff.identity
    rows_cut = cut_rows_host(f).astype(np.int64)
    if interior_raw:
        fc = f.config.func_class.ravel()
        act = active_host(f)
        rows_int = act[fc[act] != CUT]
    else:
        rows_int = np.empty(0, np.int64)
    descs = []
    # interior rows
    if rows_int.size:
        d = np.full((rows_int.size, 8), -1, np.int32)
        d[:, 0] = rows_int
        if f.strategy == "reference":
            d[:, 1] = MODE_GAUSS
        else:
            i1, i2 = rows_int // n2, rows_int % n2
            d[:, 1] = MODE_BOX
            d[:, 2] = 0
            d[:, 3] = 0
            d[:, 4] = f.b1._el_first[i1]
            d[:, 5] = f.b1._el_last[i1]
            d[:, 6] = f.b2._el_first[i2]
            d[:, 7] = f.b2._el_last[i2]
        descs.append(d)
    # cut rows
    if rows_cut.size:
        d = np.full((rows_cut.size, 8), -1, np.int32)
        d[:, 0] = rows_cut
        if f.strategy in ("reference", "hybrid"):
            d[:, 1] = MODE_GAUSS
        elif f.strategy == "wq":
            d[:, 1] = MODE_MASK
            d[:, 2] = 0
            d[:, 3] = 0
        else:  # dwq
            cut, routes = route_cut_rows(f)
            assert np.array_equal(cut, rows_cut)
            box = (routes[:, 0] == 1) & (routes[:, 3] >= 0)
            d[~box, 1] = MODE_GAUSS
            d[box, 1] = MODE_BOX
            for dd in (0, 1):
                # rule-set index per u_disc position (0: no discontinuity inside)
                ud = f.config.u_disc[dd]
                lut = np.array([key_index[dd].get(float(u), -1) for u in ud] + [0], np.int32)
                iu = routes[:, 1 + dd]
                sidx = np.where(iu >= 0, lut[np.where(iu >= 0, iu, ud.size)], 0)
                if np.any(box & (sidx < 0)):
                    raise KeyError("missing DWQ rule set for a boxed cut row")
                d[box, 2 + dd] = sidx[box]
            d[box, 4:8] = routes[box, 3:7]
        descs.append(d)
    desc = np.concatenate(descs) if descs else np.empty((0, 8), np.int32)
    return desc, int(rows_int.size)


def run_phase(f, phase):
    if not needs_raw(f):
        return
    if phase == "interior":
        f._setup = _Setup(f)
        desc, nint = _plan(f)
        f._nint = nint
        f._ndesc = desc.shape[0]
        g = _geo(f.config)
        f._desc, _ = _desc_dev(f)
        if getattr(f, "_raw_pre", None) is not None and f._desc is not f._desc_pre:
            raise RuntimeError("row plan changed between the pass-start launch and the raw phase")
        pre = getattr(f, "_raw_pre", None)
        f.raw = pre if pre is not None else raw_buffer(f, desc.shape[0])
        skey = ("slot", id(desc))
        if skey not in g:
            if planes(f):
                slot = planes_geo(f)["slot"]
            else:
                slot = torch.full_like(f.slot, -1)
                slot[f._desc[:, 0].long()] = torch.arange(desc.shape[0], dtype=torch.int32, device=f.dev)
            g[skey] = (slot, f._desc[:, 0].contiguous())
        f.slot, f.raw_list = g[skey]
        f._ctx = f._setup.ctx(f._desc, f.raw, desc.shape[0])
        pg = planes_geo(f) if planes(f) else None
        if nint and pg is not None and pg["strip_ok"] and f._setup.grids is not None:
            # interior rows by strips (no element-Gauss part: disjoint from
            # the pass-start launch, no wait)
            ctx_int = RawCtx.from_buffer_copy(f._ctx)
            ctx_int.nmax1, ctx_int.nmax2 = f._setup.nmax_std
            f._ctx_int = ctx_int
            if getattr(f, "_planes_status", None) is None:
                f._planes_status = torch.zeros(1, dtype=torch.int32, device=f.dev)
            f._bw = torch.empty(max(int(L.lib().tq_bw_table_doubles(ctx_int)), 1), dtype=torch.float64,
                                device=f.dev)
            L.call("tq_bw_tables", ctx_int, L.ptr(f._bw), L.ptr(f._planes_status), L.stream())
            # the launches write disjoint rows: the smaller ones run beside
            # the main one on side streams (their tails overlap)
            classes = strip_classes(f, pg, f._setup.sets[0][0].layout, f._setup.sets[1][0].layout)
            main = torch.cuda.current_stream()
            sides = []
            for k, (ts, strips, ns, n1m, n2m, nu, b2cap) in enumerate(classes):
                st = main if k == 0 else _named_stream(f"strips{k}", priority=-2)
                with (contextlib.nullcontext() if k == 0 else _forked(main, st)):
                    L.call("tq_sf_strips", ctx_int, ts, L.ptr(strips), ns, n1m, n2m, nu, b2cap, L.ptr(f._bw),
                           L.ptr(f._planes_status), L.stream())
                if k:
                    sides.append(st)
            for st in sides:
                main.wait_stream(st)
            _st("strips")
        elif nint:
            f._setup.wait_all_grids()
            if pre is not None:      # the sum-factor part adds onto the pass-start Gauss part
                torch.cuda.current_stream().wait_event(f._elem_event)
            # interior rows read the standard rules only: their launch sizes its
            # per-row workspace by those (more rows resident per SM)
            ctx_int = RawCtx.from_buffer_copy(f._ctx)
            ctx_int.nmax1, ctx_int.nmax2 = f._setup.nmax_std
            f._ctx_int = ctx_int
            L.call("tq_raw_sumfactor" if pre is not None else "tq_raw_regular", ctx_int, 0, nint, L.stream())
    elif phase == "cut" and pairs_mode(f):
        if f._ndesc > f._nint:
            pre = getattr(f, "_raw_pre", None) is not None
            if pre:
                torch.cuda.current_stream().wait_event(f._elem_event)
                join_cut_blocks(f)
                Eg, gslot = f._gpairs
                Ec = getattr(f, "_cpairs", None)
                if getattr(f, "_gathered", False):       # gathered at pass start
                    f._setup.wait_all_grids()
                    L.call("tq_raw_sumfactor", f._ctx, f._nint, f._ndesc, L.stream())
                    return
            else:
                Eg, gslot = _gauss_pairs(f, f._setup.eg, f._setup.em)
                Ec = _cut_pairs(f, f._setup.cut) if f._setup.cut is not None else None
                f._eager_pairs = (Eg, Ec)
            if getattr(f, "_planes_status", None) is None:
                f._planes_status = torch.zeros(1, dtype=torch.int32, device=f.dev)
            rg_ptr, rg = (cut_row_groups(f, f._nint, f._ndesc) if Ec is not None
                          else (None, None))
            L.call("tq_cut_rows_gather", f._ctx, f._nint, f._ndesc, L.ptr(gslot), L.ptr(Eg), L.ptr(Ec),
                   L.ptr(rg_ptr), L.ptr(rg), L.ptr(f._planes_status), L.stream())
            f._setup.wait_all_grids()
            L.call("tq_raw_sumfactor", f._ctx, f._nint, f._ndesc, L.stream())
    elif phase == "cutcells" and pairs_mode(f):
        pass          # in the cut phase (tq_cut_rows_gather)
    elif phase == "cut":
        if f._ndesc > f._nint:
            pre = getattr(f, "_raw_pre", None) is not None
            if pre:
                torch.cuda.current_stream().wait_event(f._elem_event)
            f._setup.wait_all_grids()
            L.call("tq_raw_sumfactor" if pre else "tq_raw_regular", f._ctx, f._nint, f._ndesc, L.stream())
    elif phase == "cutcells":
        if f._setup.cut is not None:
            if getattr(f, "_cut_pre", None) is None:
                L.call("tq_cut_blocks", _cut_blocks_ctx(f, f._setup.cut, _group_range(f, f._setup.cut)),
                       L.stream())
            join_cut_blocks(f)
            if CUTCELL_LISTS:
                rg_ptr, rg = raw_row_groups(f)
                L.call("tq_raw_cutcells_list", f._ctx, 0, f._ndesc, L.ptr(rg_ptr), L.ptr(rg), L.stream())
            else:
                L.call("tq_raw_cutcells", f._ctx, 0, f._ndesc, L.stream())
