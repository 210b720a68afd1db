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
