"""CPU ORACLE — TEST INFRASTRUCTURE ONLY, never the product.

A plain numpy/scipy restatement of the reference algorithm for the hot path of
arXiv 2101.08053 (``trimquad``: weighted-quadrature row assembly of trimmed
B-spline mass matrices and the L2-projection right-hand side).  Every function
cites the reference ``file:line`` it restates (``src/`` = the reference's
``pkg/src/trimquad/``).

Who may import this package: ``tests/``, ``__graft_entry__.smoke()`` (as the
checker) and ``bench.py`` (the ``cpu_baseline`` leg and ``--impl reference``).
The product package ``paper_2101_08053_b200`` never imports it.

Pinning: the restatement is checked against golden vectors produced by running
the reference itself in the build container (``tests/golden/make_golden.py``;
fixtures under ``tests/golden/``), see ``tests/test_oracle_golden.py``.
"""

from . import bspline, quad, trim, assemble, project, configs  # noqa: F401
