"""bench.py's N > 1 path end to end (functional): two ranks launched by
torch.distributed.run, each forming its nnz-balanced row block of the
config-5 headline workload, the block checked against the reference golden
(per-row nnz and sampled rows, bench.golden_check), max-over-ranks timing,
the CSR gather and the e2e leg through assemble_mass_distributed.  One GPU
per box here: TQ_BENCH_BACKEND=gloo folds both ranks onto cuda:0 (their
kernels never wait on each other; every exchange goes through the host).
The timings of this run are not bench values."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_ranks_row_blocks_match_reference_golden():
    env = dict(os.environ, TQ_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--no-cpu", "--no-config4", "--e2e-steps", "1"]
    r = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]          # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["nnz"] == 248114979 and d["rows"] == 3078139
    par = d["parity"]
    assert par is not None and par["row_nnz"].startswith("equal") and par["rows_checked"] > 0
    assert par["max_abs_err_over_max_abs"] <= 1e-12
    assert d["gather_ms"] is not None and d["e2e"]["d2h_bytes_per_step"] == 12 * 248114979 + 4 * 3078140
