#!/usr/bin/env python
"""Headline benchmark: FP64 mass-matrix nonzeros formed per second.

Workload (BASELINE.json config 5, the row-sharded configuration): unit square
trimmed by the seeded periodic cubic B-spline (24 control points, seed 0),
p = 4, 2048 x 2048 elements, c == 1, DWQ strategy, FP64; synthetic inputs.

One step = one full formation pass on the GPU (the analogue of the
reference's ``form_with_timings`` t_total: WQ/DWQ weights, DWQ routing,
sum-factorized interior rows, cut rows, cut-cell rows, and the fused
symmetrise / zero-drop / CSR write), with the classification and the
cut-cell geometry resident beforehand (the reference also keeps them outside
its clock, src/assembly.py:651-665).  Rows are sharded in contiguous blocks
across ranks; no collective runs inside the formation.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "FP64 mass-matrix nonzeros formed/sec"
UNIT = "nnz/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--nel", type=int, default=2048)
    ap.add_argument("--p", type=int, default=4)
    ap.add_argument("--strategy", default="dwq")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-nel", type=int, default=512, help="oracle sample size (mesh) for the CPU legs")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--no-config4", action="store_true",
                    help="skip the secondary config-4 (c = det J, p = 6/8) formation measurement")
    ap.add_argument("--no-fill-events", action="store_true",
                    help="do not capture timing events around the fill (the roofline falls back to the standalone fill)")
    ap.add_argument("--profile-eager", action="store_true",
                    help="ncu mode: run the captured schedule eagerly each step (ncu cannot profile launches "
                         "made under stream capture); numbers printed in this mode are not bench values")
    return ap.parse_args()


def config_dict(args, world):
    return {"workload": f"config5: B-spline-trimmed unit square, p={args.p}, {args.nel}x{args.nel} elements, "
                        f"c=1, {args.strategy}, seed {args.seed}",
            "nel": args.nel, "p": args.p, "strategy": args.strategy, "seed": args.seed,
            "parallelism": f"row-block x{world}", "l2": "flushed between steps (256 MiB write)",
            "row_sharding": "contiguous active-row blocks balanced by window size (nnz proxy), no collective "
                            "during formation"}


def sample_config(args, world, nnz):
    """The reference arm's config: what it actually ran (a bounded sample of
    the config-5 workload)."""
    c = config_dict(args, world)
    c.update({"workload": f"bounded sample of config5: B-spline-trimmed unit square, p={args.p}, "
                          f"{args.cpu_nel}x{args.cpu_nel} elements (full workload {args.nel}x{args.nel}), "
                          f"c=1, {args.strategy}, seed {args.seed}",
              "nel": args.cpu_nel, "full_workload_nel": args.nel, "sample_nnz": int(nnz),
              "impl": "oracle port (CPU)", "parallelism": "host CPU", "l2": "n/a (CPU)"})
    c.pop("row_sharding", None)
    return c


# ---------------------------------------------------------------------------
# CPU legs (oracle port = the reference algorithm restated in numpy)
# ---------------------------------------------------------------------------

def cpu_threads():
    return len(os.sched_getaffinity(0))


def oracle_sample(nel, p, strategy, seed, repeats=3, threads=None):
    """Reference CPU path (oracle port) on a bounded sample of the workload:
    the same trim, degree and strategy on an nel x nel mesh, after one
    warm-up, with ``threads`` BLAS threads (default: all host cores).
    Returns (median nnz/s over the repeats, description)."""
    from threadpoolctl import threadpool_limits
    from oracle import assemble as OA
    from oracle import configs as OC
    threads = threads or cpu_threads()
    with threadpool_limits(limits=threads):
        c = OC.config(5, seed=seed, nel=nel, p=p)
        cfg = OC.build_space(c["curves"], nel, p)
        cfg.cut_cell_rule(p)
        OA.form_with_timings(strategy, cfg)          # warm-up (median after warm-up)
        rates = []
        for _ in range(repeats):
            M, rep = OA.form_with_timings(strategy, cfg)
            rates.append(M.data.nnz / rep.t_total)
    sample = (f"oracle/ (numpy restatement of trimquad) form_with_timings t_total, same trim/p/strategy on "
              f"{nel}x{nel} elements ({M.data.nnz} nnz), {threads} thread(s), median of {repeats} after a warm-up")
    return statistics.median(rates), sample


def run_reference(args, rank, world):
    if rank != 0:
        return
    from threadpoolctl import threadpool_limits
    from oracle import assemble as OA
    from oracle import configs as OC
    cores = cpu_threads()
    with threadpool_limits(limits=cores):
        c = OC.config(5, seed=args.seed, nel=args.cpu_nel, p=args.p)
        cfg = OC.build_space(c["curves"], args.cpu_nel, args.p)
        cfg.cut_cell_rule(args.p)
        for _ in range(args.warmup):
            OA.form_with_timings(args.strategy, cfg)
        ts, nnz = [], 0
        for _ in range(args.steps):
            M, rep = OA.form_with_timings(args.strategy, cfg)
            ts.append(rep.t_total)
            nnz = M.data.nnz
    ms = 1e3 * sum(ts) / len(ts)
    value = nnz / (ms / 1e3)
    sample = (f"oracle port (numpy restatement of the reference trimquad; the Python reference cannot travel "
              f"to this box) form_with_timings t_total per step -- weights, interior, cut rows, cut-cell rows "
              f"and the scatter into the CSR, as the reference clocks them -- on a bounded sample of the "
              f"config-5 workload: the same trim/p/strategy on {args.cpu_nel}x{args.cpu_nel} elements "
              f"({nnz} nnz), {cores} BLAS threads")
    out = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
           "config": sample_config(args, world, nnz),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def loop():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.1)
        self._t = threading.Thread(target=loop, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if len(r) > 2 + k and r[2 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peak_hbm():
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def profile_traffic():
    """Per-launch DRAM bytes of the fill kernel from the committed ncu summary."""
    try:
        with open(os.path.join(HERE, "profiles", "fill_ncu_summary.json")) as fh:
            return json.load(fh).get("dram_bytes_per_launch")
    except Exception:
        return None


def config4_secondary(p, nel=256, steps=20, seed=0):
    """BASELINE config 4 (B-spline trim, c = det J of the perturbed geometry
    map, DWQ): one formation pass as a CUDA graph, replayed with L2 flushed
    between steps, against the algorithmic roofline of SURVEY §8(d):
    B_alg = 12 nnz + 4 (rows + 1) + 8 N1 N2 (coefficient grid) over the
    measured HBM peak, F_alg = 2 sum over interior rows of
    sum_factor_op_count over the measured DFMA peak."""
    import torch
    from paper_2101_08053_b200 import cases as C
    from paper_2101_08053_b200.assembly import GraphFormation
    c4 = C.baseline_config(4, seed=seed, p=p, nel=nel)
    b2d, cfg = C.build_space(None, nel, p, curves=c4["curves"])
    gf = GraphFormation(b2d, cfg, c4["coeff"], "dwq")
    K = cfg.active_index()[0]["K"]
    flush = torch.empty(256 * 2**20 // 8, dtype=torch.float64, device="cuda")
    for _ in range(3):
        gf.run()
    ts = []
    for _ in range(steps):
        flush.fill_(1.0)
        s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_.record()
        gf.run()
        e_.record()
        torch.cuda.synchronize()
        gf.check()
        ts.append(s_.elapsed_time(e_))
    ms = float(np.mean(ts))
    r1, r2 = gf.f.rules[0], gf.f.rules[1]
    b1, b2 = b2d.dir
    act = cfg.active_functions()
    fc = cfg.func_class
    inter = act[fc[act[:, 0], act[:, 1]] == 0]
    i1, i2 = inter[:, 0], inter[:, 1]
    n1 = np.diff(r1.wptr.cpu().numpy())[i1].astype(np.float64)     # rule-row lengths (standard rules)
    n2 = np.diff(r2.wptr.cpu().numpy())[i2].astype(np.float64)
    t1 = (b1._ov_hi - b1._ov_lo + 1)[i1].astype(np.float64)
    t2 = (b2._ov_hi - b2._ov_lo + 1)[i2].astype(np.float64)
    F = 2.0 * float(np.sum(t2 * n1 * n2 + t1 * t2 * n1))
    B = 12.0 * gf.nnz + 4.0 * (K + 1) + 8.0 * r1.layout.num_points * r2.layout.num_points
    bw = measured_peak_hbm()[0] * 1e9
    try:
        pf = float(json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                                               "fp64_peaks.json")))["dfma_tflops"]) * 1e12
    except Exception:
        pf = 33.6e12
    t_star = max(B / bw, F / pf)
    # the c != 1 interior-row sum factorization alone (tq_bw_tables +
    # tq_sf_strips, the pass's launch re-issued on resident inputs): its
    # algorithmic rate is F_alg (the reference's sum_factor_row multiply-adds
    # of the interior rows) over the kernel time
    sf = None
    try:
        from paper_2101_08053_b200 import _lib as L, _rawrows as R
        f = gf.f
        pg = R.planes_geo(f)
        classes = R.strip_classes(f, pg, f._setup.sets[0][0].layout, f._setup.sets[1][0].layout)
        st = torch.zeros(1, dtype=torch.int32, device="cuda")

        main = torch.cuda.current_stream()
        sides = [torch.cuda.Stream(priority=-2) for _ in classes[1:]]

        def strips():
            # as the pass issues them (_rawrows.run_phase): the tables, then
            # the launches of the shared-memory classes on concurrent streams
            # (they write disjoint rows), joined
            L.call("tq_bw_tables", f._ctx_int, L.ptr(f._bw), L.ptr(st), L.stream())
            for k, (ts, sd, ns, n1m, n2m, nu, b2cap) in enumerate(classes):
                stream = main if k == 0 else sides[k - 1]
                if k:
                    stream.wait_stream(main)
                with torch.cuda.stream(stream):
                    L.call("tq_sf_strips", f._ctx_int, ts, L.ptr(sd), ns, n1m, n2m, nu, b2cap, L.ptr(f._bw),
                           L.ptr(st), L.stream())
            for sd_ in sides:
                main.wait_stream(sd_)
        for _ in range(3):
            strips()
        kts = []
        for _ in range(steps):
            flush.fill_(1.0)
            s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s_.record()
            strips()
            e_.record()
            torch.cuda.synchronize()
            kts.append(s_.elapsed_time(e_))
        kms = float(np.median(kts))
        sf = {"kernel": "tq_bw_tables + tq_sf_strips (interior rows, c = det J)", "ms": kms,
              "achieved_tflops_alg": F / (kms / 1e3) / 1e12, "peak_tflops": pf / 1e12,
              "frac_alg": (F / (kms / 1e3)) / pf, "strips": int(sum(c[2] for c in classes)),
              "timing": "standalone re-issue on resident inputs as the pass issues it (shared-memory classes "
                        "on concurrent streams), L2 flushed, median"}
    except Exception as exc:      # (reported, never fatal for the headline)
        sf = {"error": repr(exc)}
    return {"workload": f"config4: B-spline trim, c = det J, p={p}, {nel}x{nel} elements, dwq, seed {seed}",
            "rows": int(K), "nnz": int(gf.nnz), "ms_per_step": ms, "value": gf.nnz / (ms / 1e3), "unit": "nnz/s",
            "B_alg": B, "F_alg": F, "T_star_us": 1e6 * t_star, "bound": "fp64" if F / pf > B / bw else "hbm",
            "step_frac_of_roofline": t_star / (ms / 1e3), "sum_factorization": sf,
            "step": "CUDA-graph replay of one full formation pass, L2 flushed between steps, mean of "
                    f"{steps}"}


def golden_check(args, world, csr, rb=0, re_=None):
    """The timed CSR against the reference's own config-5 golden
    (tests/golden/config5.npz, written by make_golden.py --huge): nnz, the
    pattern sha256 and the sampled rows (max bar 1e-12); for a row block
    (N > 1) the block's per-row nnz and the sampled rows that fall in it
    (columns and values).  Runs after the timed steps on the graph's output
    buffers; raises on any mismatch so a bench number never stands for a
    wrong matrix.  -> summary dict or None when no golden matches the
    workload."""
    import hashlib
    gpath = os.path.join(HERE, "tests", "golden", "config5.npz")
    if (args.nel, args.p, args.seed) != (2048, 4, 0) or args.strategy not in ("dwq", "hybrid") \
            or not os.path.exists(gpath):
        return None
    g = np.load(gpath)
    s = args.strategy
    if f"{s}_hash" not in g:
        return None
    ptr = csr.indptr.cpu().numpy()
    ind = csr.indices[:csr.nnz].cpu().numpy()
    rows = g[f"{s}_rows"]
    gptr = g[f"{s}_rowsptr"]
    if world == 1:
        if csr.nnz != int(g[f"{s}_nnz"]):
            raise SystemExit(f"bench: nnz {csr.nnz} != reference golden {int(g[f'{s}_nnz'])}")
        h = hashlib.sha256()
        for a in (ptr, ind):
            h.update(str(a.dtype).encode())
            h.update(np.ascontiguousarray(a).tobytes())
        if h.hexdigest() != str(g[f"{s}_hash"]):
            raise SystemExit("bench: CSR pattern sha256 differs from the reference golden")
        mine = np.arange(rows.size)
    else:
        re_ = int(ptr.size - 1 + rb) if re_ is None else re_
        if not np.array_equal(np.diff(ptr), g[f"{s}_row_nnz"][rb:re_]):
            raise SystemExit(f"bench: row block [{rb}, {re_}) per-row nnz differs from the reference golden")
        mine = np.nonzero((rows >= rb) & (rows < re_))[0]
    sel = np.concatenate([np.arange(ptr[r - rb], ptr[r - rb + 1]) for r in rows[mine]]) if mine.size else \
        np.zeros(0, np.int64)
    gsel = np.concatenate([np.arange(gptr[k], gptr[k + 1]) for k in mine]) if mine.size else np.zeros(0, np.int64)
    if not np.array_equal(ind[sel], g[f"{s}_rowsidx"][gsel]):
        raise SystemExit("bench: sampled rows' columns differ from the reference golden")
    got = csr.data[torch_index(sel, csr.data.device)].cpu().numpy()
    ref = g[f"{s}_rowsdata"][gsel]
    err = float(np.max(np.abs(got - ref)) / np.max(np.abs(ref))) if sel.size else 0.0
    if not err <= 1e-12:
        raise SystemExit(f"bench: sampled rows differ from the reference golden (max rel {err:.3g})")
    out = {"golden": "tests/golden/config5.npz (reference run at 2048^2)", "rows_checked": int(mine.size),
           "entries_checked": int(sel.size), "max_abs_err_over_max_abs": err}
    if world == 1:
        out.update({"nnz": "equal", "pattern_sha256": "equal"})
    else:
        out.update({"row_block": [int(rb), int(re_)], "row_nnz": "equal (this rank's block)"})
    return out


def torch_index(sel, device):
    import torch
    return torch.from_numpy(sel.astype(np.int64)).to(device)


def rhs_secondary(b2d, cfg, steps=20, cpu_nel=256, seed=0):
    """The L2-projection legs of config 5 (src/projection.py:101-145, 221-260):
    assemble_rhs of f = sin(2 pi x) cos(3 pi y) and l2_error of a seeded
    coefficient vector, kernels only on resident inputs (ResidentProjection,
    one CUDA graph of both, replayed with L2 flushed between steps), plus the
    oracle port on a bounded sample (cpu_nel^2) for the CPU figure."""
    import torch
    from paper_2101_08053_b200 import cases as C, projection as PR
    prob = PR.ProjectionProblem(C.f_config5, b2d, cfg, strategy="dwq")
    rp = PR.ResidentProjection(prob)
    x = torch.from_numpy(np.random.default_rng(5).standard_normal(rp.K)).to("cuda")
    flush = torch.empty(256 * 2**20 // 8, dtype=torch.float64, device="cuda")
    s_rhs = torch.cuda.Stream()
    s_rhs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s_rhs):       # warm the launch paths, then capture both legs
        for _ in range(2):
            rp.rhs(); rp.l2_parts(x)
    torch.cuda.current_stream().wait_stream(s_rhs)
    torch.cuda.synchronize()
    graphs = {}
    for name, fn in (("rhs", rp.rhs), ("l2", lambda: rp.l2_parts(x))):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        graphs[name] = g
    torch.cuda.synchronize()
    res = {}
    for name, g in graphs.items():
        ts = []
        for _ in range(steps):
            flush.fill_(1.0)
            a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); g.replay(); b_.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b_))
        res[name] = float(np.median(ts))
    nd = rp.nd.cpu().numpy()
    e = float(np.sqrt(nd[0] / nd[1]))
    # algorithmic figures: RHS points = (p+2)^2 Gauss points per interior
    # element + cut-cell points; L2: (p+3)^2 points, F_alg = 2 * per-element
    # FMA of the sum-factorised u_h ((p+3)(p+1)^2 + (p+3)^2 (p+1)) + 3 per point
    p = b2d.dir[0].p
    n_int = int((cfg.element_class_dev == 0).sum().item())
    ncut = rp.cut.n if rp.cut is not None else 0
    rhs_pts = n_int * (p + 2) ** 2 + ncut
    l2_pts = n_int * (p + 3) ** 2 + ncut
    G, Q = p + 3, p + 1
    F_l2 = 2.0 * n_int * (G * Q * Q + G * G * Q + 3 * G * G)
    try:
        pf = float(json.load(open(os.path.join(HERE, "profiles", "fp64_peaks.json")))["dfma_tflops"])
    except Exception:
        pf = 33.6
    l2_tf = F_l2 / (res["l2"] / 1e3) / 1e12
    out = {"workload": "config5 L2 projection legs: assemble_rhs(f = sin(2 pi x) cos(3 pi y)) and "
                       "l2_error(seeded coefficients), 2048^2, p=4",
           "rhs_ms": res["rhs"], "l2_error_ms": res["l2"], "l2_error_value": e,
           "rhs_points_per_s": rhs_pts / (res["rhs"] / 1e3), "l2_points_per_s": l2_pts / (res["l2"] / 1e3),
           "rhs_rows_per_s": rp.K / (res["rhs"] / 1e3),
           "rhs_bound": "latency (five small kernels: separable target tabulated per Gauss coordinate, 1-D element "
                        "integrals, interior rows as products of 1-D sums, cut rows masked + cut-cell points)",
           "l2_roofline": {"bound": "fp64", "achieved": l2_tf, "peak": pf, "unit": "TFLOP/s", "frac": l2_tf / pf,
                           "F_alg": F_l2, "peak_source": "profiles/fp64_peaks.json (DFMA loop)"},
           "step": "CUDA graph of the kernels on resident inputs, L2 flushed between steps, median of "
                   f"{steps}"}
    try:                   # the reference algorithm (oracle port) on a bounded sample
        from threadpoolctl import threadpool_limits
        from oracle import configs as OC, project as OP
        with threadpool_limits(limits=cpu_threads()):
            oc = OC.config(5, seed=seed, nel=cpu_nel, p=p)
            ocfg = OC.build_space(oc["curves"], cpu_nel, p)
            ocfg.cut_cell_rule(p)
            t0 = time.perf_counter()
            rb = OP.assemble_rhs(oc["target"], ocfg)
            t1 = time.perf_counter()
            xs = np.random.default_rng(5).standard_normal(rb.size)
            OP.l2_error(xs, oc["target"], ocfg)
            t2 = time.perf_counter()
        out["cpu_baseline"] = {"rhs_rows_per_s": rb.size / (t1 - t0), "l2_elements_per_s": cpu_nel ** 2 / (t2 - t1),
                               "cores": cpu_threads(), "kind": "port",
                               "sample": f"oracle/project.py assemble_rhs + l2_error on {cpu_nel}x{cpu_nel} elements "
                                         f"of the config-5 recipe ({rb.size} rows), one run each"}
    except Exception as exc:
        out["cpu_baseline"] = {"failed": str(exc)}
    return out


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2101_08053_b200 as P
    from paper_2101_08053_b200 import _lib as L
    from paper_2101_08053_b200 import cases as C
    from paper_2101_08053_b200.assembly import GraphFormation, form

    torch.cuda.set_device(local_rank)
    lib = L.lib()
    lib.tq_launch_count.restype = L.C.c_longlong
    dev = torch.device("cuda", local_rank)

    def barrier():
        if world > 1:
            dist.barrier()

    # setup (untimed, resident): basis, GPU classification, host cut-cell rule
    c5 = C.baseline_config(5, seed=args.seed, p=args.p, nel=args.nel)
    b2d, cfg = C.build_space(None, args.nel, args.p, curves=c5["curves"])
    cfg.cut_cell_rule(args.p)
    idx, _ = cfg.active_index()
    K = idx["K"]
    from paper_2101_08053_b200.distributed import row_block, window_counts
    rb, re_ = row_block(K, world, rank, window_counts(cfg) if world > 1 else None)   # nnz-balanced blocks
    flush = torch.empty(256 * 2**20 // 8, dtype=torch.float64, device=dev)

    # the timed step: one full formation pass captured as a CUDA graph
    # (GraphFormation: every kernel of the pass replays each step) plus the
    # host read-back of the moment-fit residual flags
    fill_ev = None
    if args.profile_eager:
        class _Eager:     # same kernels and schedule as the captured pass, launched eagerly
            def __init__(self):
                f, csr = form(b2d, cfg, None, args.strategy, row_range=(rb, re_))
                self.nnz, self.report = csr.nnz, f.report
                self.cap = {"nnz": csr.nnz}
                lib.tq_launch_count.restype = L.C.c_longlong
                n0 = lib.tq_launch_count()
                self.run()
                self.launches_per_pass = int(lib.tq_launch_count() - n0)

            def run(self):
                self.f, self.csr = form(b2d, cfg, None, args.strategy, row_range=(rb, re_), capture=self.cap)
                return self.csr

            def check(self):
                pass
        gf = _Eager()
    else:
        # timing events captured around the fill inside the step (event nodes of the graph)
        fill_ev = None if args.no_fill_events else (torch.cuda.Event(enable_timing=True, external=True),)
        gf = GraphFormation(b2d, cfg, None, args.strategy, row_range=(rb, re_), fill_events=fill_ev)
    rep = gf.report

    def step():
        return gf.run()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(local_rank)
    sampler.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = lib.tq_launch_count()
    fill_in_step = []
    for k in range(args.steps):
        flush.fill_(float(k))            # L2 flush between timed steps (untimed)
        barrier()
        torch.cuda.synchronize()
        ev[k][0].record()
        csr = step()
        ev[k][1].record()
        torch.cuda.synchronize()
        if fill_ev is not None:
            # fill start (event node in the graph) -> the step's end event: the
            # fill is the pass's last phase, so this bounds it from above
            fill_in_step.append(fill_ev[0].elapsed_time(ev[k][1]))
        gf.check()                       # the pass's status (reduced in the graph), read after it
        barrier()
    nnz_local = gf.nnz
    clocks = sampler.stop()
    parity = golden_check(args, world, gf.csr, rb, re_)
    # kernels per step: the captured pass replays exactly the launches of one eager pass
    launches = gf.launches_per_pass * args.steps
    step_ms = [s.elapsed_time(e) for s, e in ev]
    total_ms = sum(step_ms)

    gather_ms = None
    if world > 1:       # NCCL gather of the CSR blocks to rank 0, timed separately
        from paper_2101_08053_b200.distributed import gather_csr
        barrier()
        torch.cuda.synchronize()
        g0 = time.perf_counter()
        gather_csr(gf.csr.indptr, gf.csr.indices, gf.csr.data, rank, world)
        torch.cuda.synchronize()
        barrier()
        gather_ms = 1e3 * (time.perf_counter() - g0)

    # fill kernels alone (the roofline kernels) on the captured pass's buffers
    kms = {}
    ctx = gf.f.rowctx(rb, re_)
    # (its two launches -- tiles, and the listed rows forked onto a second
    # stream and joined -- timed between events on the launching stream)
    class _FillEager:
        def replay(self):
            gf.f.fill(ctx, gf.csr.indptr, gf.csr.indices, gf.csr.data)
    fill_graph = _FillEager()
    fill_graph.replay()
    fe = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(21)]
    for s_, e_ in fe:
        flush.fill_(1.0)
        s_.record()
        fill_graph.replay()
        e_.record()
    torch.cuda.synchronize()
    kms["fill"] = float(np.median([s_.elapsed_time(e_) for s_, e_ in fe[1:]])) * args.steps
    # the tiles kernel alone (diagnostic: the listed rows excluded)
    for s_, e_ in fe:
        flush.fill_(1.0)
        s_.record()
        L.call("tq_fill_fast", ctx, L.ptr(gf.csr.indptr), L.ptr(gf.csr.indices), L.ptr(gf.csr.data), L.stream())
        e_.record()
    torch.cuda.synchronize()
    kms["fill_tiles_only"] = float(np.median([s_.elapsed_time(e_) for s_, e_ in fe[1:]])) * args.steps
    # standalone fill right after the flush (pays the flush's dirty-L2 write-back): diagnostic
    kms["fill_standalone"] = kms.pop("fill")
    if fill_in_step:      # the roofline kernel timed inside the timed steps (events in the graph)
        kms["fill"] = float(np.mean(fill_in_step)) * args.steps
    else:
        kms["fill"] = kms["fill_standalone"]
    t = torch.tensor([total_ms, float(nnz_local), kms.get("fill", 0.0), float(re_ - rb)], dtype=torch.float64,
                     device=dev)
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
    else:
        tmax = tsum = t
    total_ms_max = float(tmax[0])
    nnz_total = int(tsum[1])
    ms_per_step = total_ms_max / args.steps
    value = nnz_total / (ms_per_step / 1e3)

    # roofline of the dominant kernel (fill): algorithmic bytes / event time
    fill_ms = kms.get("fill", float("nan")) / args.steps
    alg_bytes = 12.0 * nnz_local + 4.0 * ((re_ - rb) + 1)
    peak, peak_kind = measured_peak_hbm()
    achieved = alg_bytes / (fill_ms / 1e3) / 1e9
    traffic = profile_traffic()

    # e2e through the public API from host inputs (rank-local row block at N>1)
    e2e = None
    if args.e2e_steps > 0:
        knots = np.ascontiguousarray(P.make_uniform_knots(args.nel, args.p).knots)
        ctrl = np.ascontiguousarray(c5["curves"][0].ctrl)
        # the ~185k objects alive after setup (torch/scipy modules, plans)
        # move to the permanent generation: a full collection landing inside
        # a step then scans only what that step made (~45 ms otherwise,
        # scripts/probes/gc_census.py), the usual serving-process setting
        gc.collect()
        gc.freeze()
        e_ts, e_ph, h2d, d2h = [], [], 0, 0
        # untimed passes first, as many as the device-timed steps get: the
        # caching allocators (device and pinned host) reach their steady
        # footprint within two fresh-configuration calls
        e2e_warm = max(1, args.warmup)
        for k in range(args.e2e_steps + e2e_warm):
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            kv = P.KnotVector(knots.copy(), args.p)
            bb = P.TensorBasis2D(P.Basis1D(kv), P.Basis1D(P.KnotVector(knots.copy(), args.p)))
            cf = P.classify_elements(bb, [P.trimming.PeriodicBSplineTrim(ctrl.copy())])
            t1 = time.perf_counter()
            if world == 1:
                M = P.assemble_mass(bb, cf, None, strategy=args.strategy)
            else:   # row blocks formed per GPU, NCCL gather to rank 0, host copy there
                from paper_2101_08053_b200.distributed import assemble_mass_distributed
                M = assemble_mass_distributed(bb, cf, None, strategy=args.strategy)
            nnz_e = M.data.nnz if M is not None else 0
            rows_e = M.shape[0] if M is not None else 0
            t2 = time.perf_counter()
            del M
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            barrier()
            if k >= e2e_warm:  # the first passes warm the allocators / caches
                e_ts.append(dt)
                e_ph.append((round(t1 - t0, 4), round(t2 - t1, 4), round(time.perf_counter() - t2, 4)))
            if rank == 0:
                h2d = knots.nbytes * 2 + ctrl.nbytes
                d2h = 12 * nnz_e + 4 * (rows_e + 1)
        et = torch.tensor([sum(e_ts) / len(e_ts)], dtype=torch.float64, device=dev)   # mean step; max over ranks
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": nnz_total / float(et[0]), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "seconds_per_step": float(et[0]),
               "warmup_passes": e2e_warm,
               "step_seconds": [round(x, 4) for x in e_ts],
               "median_seconds": float(np.median(e_ts)),
               "phase_seconds": {"classify": [p[0] for p in e_ph], "assemble_mass": [p[1] for p in e_ph],
                                 "release": [p[2] for p in e_ph]},
               "path": "KnotVector/Basis1D -> classify_elements (GPU) -> cut-cell decomposition (GPU) -> "
                       + ("assemble_mass" if world == 1 else "assemble_mass_distributed (NCCL gather to rank 0)")
                       + " -> scipy CSR on host"}

    if rank != 0:
        return
    secondary = None
    if world == 1 and not args.no_config4 and not args.profile_eager:
        secondary = {}
        try:
            secondary["rhs_l2_config5"] = rhs_secondary(b2d, cfg)
        except Exception as exc:
            secondary["rhs_l2_config5"] = {"failed": str(exc)}
        for p4 in (6, 8):
            try:
                secondary[f"config4_p{p4}"] = config4_secondary(p4)
            except Exception as exc:  # the headline stands on its own
                secondary[f"config4_p{p4}"] = {"failed": str(exc)}
    cpu = None
    if world == 1 and not args.no_cpu:
        try:
            v, sample = oracle_sample(args.cpu_nel, args.p, args.strategy, args.seed)
            v1, sample1 = oracle_sample(args.cpu_nel, args.p, args.strategy, args.seed, repeats=1, threads=1)
            cpu = {"value": v, "unit": UNIT, "cores": cpu_threads(), "kind": "port", "sample": sample,
                   "single_thread": {"value": v1, "unit": UNIT, "cores": 1, "sample": sample1}}
        except Exception as exc:  # the GPU number stands on its own
            cpu = {"value": None, "unit": UNIT, "cores": cpu_threads(), "kind": "port", "sample": f"failed: {exc}"}
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE config 5 geometry)",
        "config": config_dict(args, world),
        "nnz": nnz_total, "rows": K,
        "eager_phases_ms": {"weights": 1e3 * rep.t_weights, "interior": 1e3 * rep.t_interior,
                            "cut_regular": 1e3 * rep.t_cut_regular, "cut_elements": 1e3 * rep.t_cut_elements,
                            "finish": 1e3 * rep.t_finish},
        "step": ("eager run of the captured schedule (--profile-eager: ncu mode, not a bench value)"
                 if args.profile_eager else "CUDA-graph replay of one full formation pass (its status -- fit flags, nnz -- reduced in the graph, read after each step)"),
        "kernels_ms_per_step": {k: v / args.steps for k, v in kms.items()},
        "roofline": {"kernel": "fill: k_fill_tiles with k_fill_irregular concurrent (fused symmetrise + zero-drop + CSR write)", "bound": "hbm",
                     "timing": ("mean over the timed steps: event captured at the fill's start inside the step graph -> the step's end event"
                                if fill_in_step else "standalone fill after an L2 flush (median of 20)"),
                     "achieved": achieved, "peak": peak, "peak_source": peak_kind, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "algorithmic_bytes_per_launch": alg_bytes},
        "gpu_launches": int(launches),
        "parity": parity,
        "gather_ms": gather_ms,
        "clocks": clocks,
        "e2e": e2e,
        "secondary": secondary,
        "cpu_baseline": cpu,
    }
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        # TQ_BENCH_BACKEND=gloo (with ranks folded onto the visible GPUs) is
        # the functional test of the N > 1 path on a one-GPU box
        # (tests/test_gpu_bench_multirank.py); its timings are not bench values
        backend = os.environ.get("TQ_BENCH_BACKEND", "nccl")
        if backend != "nccl":
            local_rank %= torch.cuda.device_count()
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
