"""CPU oracle for the DG-acoustics hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy, the algorithm of the reference
package ``wavekernel`` (``/root/reference/pkg/src/wavekernel``) for the
hot path named in BASELINE.json: the matrix-free sum-factorized DG
operator (``operator.py:149-325``), the low-storage RK and ADER/TCK
steppers (``stepping.py:179-318``) and the 1-D bases they rest on
(``quadrature.py:110-254``).  Every function cites the reference
file:line it follows.

Rules:

* Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  CPU-baseline leg may import this package.  The product package
  ``paper_1805_03981_b200`` never imports it; its GPU path fails loudly
  when the CUDA library is missing instead of falling back here.
* Parity is PINNED: ``tests/test_oracle_golden.py`` checks this
  restatement against golden vectors produced by running the unmodified
  reference (``tests/golden/make_golden.py``, committed with the
  fixtures).
"""

from .quadrature import (gauss_rule, gauss_lobatto_rule, lagrange_matrix,
                         projection_matrix, basis_change)
from .mesh import (OracleMesh, OracleMaterial, OracleGeometry, build_cartesian,
                   precompute_geometry, min_edge_length, map_points)
from .operator import OracleOperator
from .stepping import (LSRK45, LSRK59, lsrk_step, tck_evaluate, ader_step,
                       reduction_schedule, reduction_degrees, compute_dt,
                       state_norm, advance)

__all__ = [
    "gauss_rule", "gauss_lobatto_rule", "lagrange_matrix",
    "projection_matrix", "basis_change", "OracleMesh", "OracleMaterial",
    "OracleGeometry", "build_cartesian", "precompute_geometry",
    "min_edge_length", "map_points", "OracleOperator", "LSRK45", "LSRK59",
    "lsrk_step", "tck_evaluate", "ader_step", "reduction_schedule",
    "reduction_degrees", "compute_dt", "state_norm", "advance",
]
