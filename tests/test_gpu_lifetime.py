"""Device memory of a public-API call is released by reference counting when
the call's objects go out of scope -- no reference cycle may keep a pass's
device tables waiting for the cyclic collector (the caching allocator's
footprint then differs from call to call and it falls back to cudaMalloc,
tens of ms each: the e2e outliers of profiles/r2_e2e_jitter_*.txt)."""

import gc

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _left_after(fn):
    import torch
    for _ in range(2):
        fn()
    gc.collect()
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    gc.disable()
    try:
        fn()
        torch.cuda.synchronize()
        return torch.cuda.memory_allocated() - base
    finally:
        gc.enable()


@pytest.mark.parametrize("strategy", ["reference", "wq", "hybrid", "dwq"])
def test_assemble_mass_releases_device_memory(strategy):
    import paper_2101_08053_b200 as P
    from paper_2101_08053_b200 import cases as C

    def call():
        b2d, cfg = C.build_space(None, 32, 3, curves=[C.closed_circle()])
        P.assemble_mass(b2d, cfg, None, strategy=strategy)

    assert _left_after(call) == 0


def test_detj_and_projection_release_device_memory():
    import paper_2101_08053_b200 as P
    from paper_2101_08053_b200 import cases as C

    def mass():
        c4 = C.baseline_config(4, nel=32, p=3)
        b2d, cfg = C.build_space(None, 32, 3, curves=c4["curves"])
        P.assemble_mass(b2d, cfg, c4["coeff"], strategy="dwq")

    def proj():
        b2d, cfg = C.build_space(None, 32, 3, curves=[C.closed_circle()])
        prob = P.ProjectionProblem(C.f_config23, b2d, cfg)
        P.assemble_rhs(prob)
        P.l2_error(np.ones(cfg.active_functions().shape[0]), prob)

    assert _left_after(mass) == 0
    assert _left_after(proj) == 0
