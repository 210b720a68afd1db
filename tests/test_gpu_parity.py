"""GPU parity: the CUDA formation path against the reference golden vectors
and the CPU oracle (bars as in tests/test_oracle_golden.py)."""

import hashlib

import numpy as np
import pytest
import scipy.sparse as sp

from tests import golden_cases as G

pytestmark = pytest.mark.gpu


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def assert_matrix_close(M, R, tol=1e-12):
    """Pattern bit-exact; rel-Frobenius and per-entry sqrt(M_ii M_jj) bars."""
    assert M.shape == R.shape
    assert M.indptr.dtype == np.int32 and M.indices.dtype == np.int32
    assert np.array_equal(M.indptr, R.indptr)
    assert np.array_equal(M.indices, R.indices)
    d = M.data - R.data
    assert np.linalg.norm(d) <= tol * np.linalg.norm(R.data)
    diag = R.diagonal()
    rows = np.repeat(np.arange(R.shape[0]), np.diff(R.indptr))
    bound = tol * np.sqrt(np.abs(diag[rows] * diag[R.indices])) + 1e-300
    assert np.all(np.abs(d) <= bound)


def golden_matrix(d, s):
    K = d["active"].shape[0]
    return sp.csr_matrix((d[f"{s}_data"], d[f"{s}_indices"], d[f"{s}_indptr"]), shape=(K, K))


def gpu_space(nel, p, curves=()):
    import paper_2101_08053_b200 as P
    b = P.make_uniform_basis(nel, p)
    b2d = P.TensorBasis2D(b, P.make_uniform_basis(nel, p))
    return b2d, P.classify_elements(b2d, list(curves))


@pytest.mark.parametrize("strategy", ["wq", "hybrid", "dwq"])
def test_config1_untrimmed_matches_reference(strategy):
    import paper_2101_08053_b200 as P
    d = G.load("config1")
    b2d, cfg = gpu_space(16, 2)
    assert np.array_equal(cfg.element_class, d["element_class"])
    assert np.array_equal(cfg.func_class, d["func_class"])
    assert np.array_equal(cfg.active_functions(), d["active"])
    M = P.assemble_mass(b2d, cfg, strategy=strategy)
    assert sha(M.data.indptr, M.data.indices) == str(d[f"{strategy}_hash"])
    assert_matrix_close(M.data, golden_matrix(d, strategy))


@pytest.mark.parametrize("nel,p", [(7, 1), (9, 3), (12, 4), (6, 6), (10, 8)])
def test_untrimmed_vs_oracle(nel, p):
    import paper_2101_08053_b200 as P
    from oracle import assemble as OA
    from oracle import configs as OC
    b2d, cfg = gpu_space(nel, p)
    M = P.assemble_mass(b2d, cfg, strategy="wq")
    ref = OA.assemble_mass(OC.build_space([], nel, p), strategy="wq").data
    assert_matrix_close(M.data, ref)


@pytest.mark.parametrize("nel,p", [(9, 1), (9, 2), (7, 4), (10, 6), (12, 8)])
def test_wq_weights_reproduce_moments(nel, p):
    """GPU weights: residual of every moment system <= 1e-12 max|b|
    (src/quadrature.py:299-301), zero off the support."""
    import paper_2101_08053_b200 as P
    b = P.make_uniform_basis(nel, p)
    r = P.compute_wq_rules(b)
    M = P.mass_matrix_1d(b)
    C = b.collocation(r.layout.points)
    for i in range(b.n):
        approx = C.T @ r.row_full(i)
        assert np.max(np.abs(approx - M[i])) <= 1e-12 * np.max(np.abs(M[i]))
        lo, hi = b.support_interval(i)
        full = r.row_full(i)
        outside = (r.layout.points < lo) | (r.layout.points > hi)
        assert np.all(full[outside] == 0.0)


def test_basis_and_moments_vs_oracle():
    import paper_2101_08053_b200 as P
    from oracle import bspline as OB
    from oracle import quad as OQ
    d = dict(np.load(f"{G.HERE}/rules_1d.npz"))
    kn = d["wq_nonuni_knots"]
    b = P.Basis1D(P.KnotVector(kn, 2))
    f, v = b.eval_nonzero_batch(d["eval_nonuni_u"])
    assert np.array_equal(f, d["eval_nonuni_first"])
    assert np.max(np.abs(v - d["eval_nonuni_vals"])) <= 1e-15
    for nel, p in ((9, 3), (10, 6), (12, 8)):
        b = P.make_uniform_basis(nel, p)
        assert np.max(np.abs(P.mass_matrix_1d(b) - d[f"wq_{nel}_{p}_M"])) <= 1e-16
        s = OB.uniform_space(nel, p)
        u = np.linspace(0, 1, 1001)
        f, v = b.eval_nonzero_batch(u)
        fo, vo = s.eval_nonzero(u)
        assert np.array_equal(f, fo) and np.max(np.abs(v - vo)) <= 1e-15
        _, _, Do = s.eval_nonzero_ders(u)
        import torch
        from paper_2101_08053_b200 import _lib as L
        _, _, Dg = b.eval_device(L.dev(u, torch.float64), ders=True)
        assert np.max(np.abs(Dg.cpu().numpy() - Do)) <= 1e-12 * max(1.0, np.max(np.abs(Do)))
