"""Host-side spline bookkeeping of the drop-in (no GPU): knot insertion and
the composite subdivision map onto a nested knot vector
(src/splines.py:369-442), checked by the identities a refinement must keep:
constants and linear functions (Greville abscissae) are reproduced, and the
composite map equals the product of its single insertions."""

import numpy as np
import pytest


def _greville(kv, p):
    k = np.asarray(kv.knots)
    return np.array([k[i + 1: i + p + 1].mean() for i in range(k.size - p - 1)])


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_subdivision_reproduces_constants_and_lines(p):
    from paper_2101_08053_b200 import splines as S
    coarse = S.make_uniform_basis(4, p)
    fine_kv = S.make_uniform_knots(8, p)
    sub = S.subdivision_matrix_to(coarse, fine_kv)
    assert sub.shape == (fine_kv.knots.size - p - 1, coarse.n)
    assert np.allclose(sub.apply(np.ones(coarse.n)), 1.0, atol=1e-14)
    assert np.allclose(sub.apply(_greville(coarse.kv, p)), _greville(fine_kv, p), atol=1e-14)
    assert np.allclose(sub.target.kv.knots, fine_kv.knots, atol=1e-15)


def test_subdivision_equals_product_of_insertions():
    from paper_2101_08053_b200 import splines as S
    b = S.make_uniform_basis(3, 2)
    target = np.sort(np.concatenate([b.kv.knots, [0.2, 0.5, 0.5, 0.9]]))
    sub = S.subdivision_matrix_to(b, target)
    cur, M = b, None
    for u in (0.2, 0.5, 0.5, 0.9):
        cur, step = S.insert_knot(cur, u)
        M = step if M is None else step @ M
    assert np.array_equal(sub.matrix.toarray(), M.matrix.toarray())


def test_subdivision_rejects_non_refinements():
    from paper_2101_08053_b200 import splines as S
    b = S.make_uniform_basis(4, 2)
    with pytest.raises(ValueError):
        S.subdivision_matrix_to(b, S.make_uniform_knots(3, 2))     # drops interior knots
    with pytest.raises(ValueError):
        S.subdivision_matrix_to(b, S.make_uniform_knots(8, 3))     # other degree


@pytest.mark.parametrize("p,nel", [(1, 5), (2, 7), (3, 9), (4, 12), (6, 10)])
def test_repeated_insertion_equals_product_of_single_insertions(p, nel):
    """refine_to_c_minus_1 composes the insertions in a window; it must be
    bit-identical to the product of the single-insertion maps."""
    import scipy.sparse as sp
    from paper_2101_08053_b200 import splines as S
    b = S.make_uniform_basis(nel, p)
    rng = np.random.default_rng(p)
    bps = b.breakpoints[1:-1]
    for u in list(rng.choice(bps, size=min(3, bps.size), replace=False)) + [0.0, 1.0, float(bps[0])]:
        fine, sub = S.refine_to_c_minus_1(b, float(u))
        kn, M = b.kv.knots, sp.identity(b.n, format="csr")
        for _ in range(p + 1 - b.kv.multiplicity_of(float(u))):
            kn, step = S._insertion_matrix(kn, p, float(u))
            M = step @ M
        M.eliminate_zeros()
        M.sort_indices()              # the sparse product leaves rows unsorted
        A = sub.matrix.tocsr()
        A.eliminate_zeros()
        A.sort_indices()
        assert np.array_equal(fine.kv.knots, kn)
        assert np.array_equal(A.indptr, M.indptr) and np.array_equal(A.indices, M.indices)
        assert np.array_equal(A.data, M.data)
