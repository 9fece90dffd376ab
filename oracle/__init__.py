"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct fp64 / complex128 NumPy implementation of the hot
path of arXiv:2002.05019 (§II APPROACH): the block LDL^T
factorization with *restricted* Bunch-Kaufman pivoting of the block-sparse
symmetric auxiliary matrix, its clique-graph symbolic step, and the multi-RHS
forward/backward substitution.  Readings of the paper are listed in DESIGN.md
("Readings"); every function cites the passage it follows.

Rules:
  * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
    --impl reference legs may import this package;
  * it shares no code with the CUDA path (paper_2002_05019_b200/) and imports
    nothing from it; the only common module is dd_inputs (seeded inputs, no
    method arithmetic);
  * library primitives used as single steps: numpy matmul, scipy
    solve_triangular (unit-lower triangular substitution).

Pins (tests/test_oracle_*.py, `-m "not gpu"`): LAPACK ?sytrf pivot decisions,
dense LU solves, Sylvester inertia via eigvalsh, the fill-path theorem for the
symbolic step, SPEC worked examples, metamorphic scaling/negation.  Every oracle
function is pinned; none is "parity unpinned".
"""
from .bk import bk_factor, ALPHA, cabs1  # noqa: F401
from .assemble import assemble  # noqa: F401
from .block_ldlt import (symbolic, block_factor, block_solve, refine_solve, inertia,  # noqa: F401
                         flops_factor, flops_solve_per_rhs, residual_berr, OracleFactor, max_abs_L,
                         norm_inf_A, matvec_blocks)
