"""WQ enrichment retries on the GPU (src/quadrature.py:306-337; VERDICT r1
weak #10): starting layouts with too few points per element, against the
reference's own outcome (tests/golden/rules_retry.npz, make_golden.py
--retry) -- the final per-element point counts bit-exact, every moment
residual of the final rules within 1e-12 max|b|, and
``RuleConstructionError`` where the reference gives up after 5 retries."""

import numpy as np
import pytest

from tests import golden_cases as G

pytestmark = pytest.mark.gpu

D = G.load("rules_retry")
CASES = list(range(int(D["ncases"])))


@pytest.mark.parametrize("k", CASES)
def test_enrichment_retry_matches_reference(k):
    import paper_2101_08053_b200 as P
    from paper_2101_08053_b200.quadrature import _layout_from_counts
    nel, p = (int(v) for v in D[f"c{k}_case"])
    b = P.make_uniform_basis(nel, p)
    lay = _layout_from_counts(b, D[f"c{k}_start"])
    if f"c{k}_error" in D:
        with pytest.raises(P.RuleConstructionError):
            P.compute_wq_rules(b, lay)
        return
    r = P.compute_wq_rules(b, lay)
    assert np.array_equal(r.layout.counts(), D[f"c{k}_final"])
    # exactness of the final rules: sum_k w_i[k] B_j(x_k) = int B_i B_j
    M = P.mass_matrix_1d(b)
    C = b.collocation(r.layout.points)
    for i in range(b.n):
        k0, w = r.row(i)
        got = w @ C[k0:k0 + w.size]
        assert np.max(np.abs(got - M[i])) <= 1e-12 * np.max(np.abs(M[i]))
