"""B200-native formation path of arXiv 2101.08053 (trimquad drop-in).

Weighted-quadrature row assembly with sum factorization for trimmed
bivariate B-spline mass matrices and the L2-projection right-hand side, on
hand-written sm_100a kernels behind a C ABI (``include/trimquad_b200.h``).
The public names mirror the reference package ``trimquad``
(src/__init__.py:8-32).
"""

from .splines import (Basis1D, KnotVector, SubdivisionMatrix, TensorBasis2D, insert_knot, subdivision_matrix_to,
                      make_uniform_basis, make_uniform_knots)
from .quadrature import (DiscontinuousRuleSet, GaussRule, PointLayout, RuleConstructionError,
                         WeightedRuleSet, build_dwq, compute_wq_rules, exact_moments, gauss_legendre,
                         mass_matrix_1d, place_wq_points)
from .trimming import (BezierTrim, CircleTrim, ElementClass, LineTrim, TrimConfiguration, TrimmingConfigurationError,
                       classify_elements, classify_point, cut_cell_quadrature, decompose_cut_element,
                       intersect_edge)
from .assembly import (STRATEGIES, CoefficientField, FormationReport, SparseMatrix, assemble_mass,
                       form_with_timings, sum_factor_op_count, sum_factor_row, sum_factor_rows)

from .projection import (ConditioningError, ProjectionProblem, SeparableTarget, assemble_rhs, default_target,
                         l2_error, project, solve_spd, run_convergence_study, ConvergenceRecord)

__version__ = "0.1.0"
