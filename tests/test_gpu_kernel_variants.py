"""Specialised kernels against their generic counterparts, bit for bit: the
degree-templated c == 1 element-Gauss part of the raw rows
(k_raw_gauss_sep<P>) against the generic k_raw_regular<1>, through the whole
formation (the generic path is forced with TQ_RAW_GAUSS_GENERIC, read when
the library loads -- hence the subprocesses)."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
from paper_2101_08053_b200 import cases as C
from paper_2101_08053_b200.assembly import form
kind, nel, p, strategy = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
if kind == "bspline":
    b2d, cfg = C.build_space(None, nel, p, curves=C.baseline_config(5)["curves"])
else:
    b2d, cfg = C.build_space(kind, nel, p)
_, csr = form(b2d, cfg, None, strategy)
np.savez(sys.argv[5], *[t.cpu().numpy() for t in (csr.indptr, csr.indices, csr.data)])
"""


@pytest.mark.parametrize("kind,nel,p,strategy", [("bspline", 96, 4, "dwq"), ("bspline", 64, 3, "hybrid"),
                                                 ("corner", 24, 2, "hybrid"), ("bspline", 48, 6, "dwq")])
def test_gauss_part_specialisation_bit_identical(tmp_path, kind, nel, p, strategy):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for mode in ("sep", "generic"):
        env = dict(os.environ)
        env.pop("TQ_RAW_GAUSS_GENERIC", None)
        if mode == "generic":
            env["TQ_RAW_GAUSS_GENERIC"] = "1"
        f = tmp_path / f"{mode}.npz"
        subprocess.run([sys.executable, "-c", _SCRIPT.format(root=root), kind, str(nel), str(p), strategy, str(f)],
                       check=True, env=env, timeout=600)
        z = np.load(f)
        out[mode] = [z[k] for k in ("arr_0", "arr_1", "arr_2")]
    for a, b in zip(out["sep"], out["generic"]):
        assert np.array_equal(a, b)
