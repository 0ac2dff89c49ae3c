"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the GMRES operator-apply hot
path of the reference `lapbel` package.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this package; the product
(paper_2111_10743_b200) never does and fails loudly without its CUDA library.

Contents (each restating the reference file:line it follows):
  * p2p / p2p_grouped / csr_matvec  -> C library p2p_oracle.c
  * apply_a1/a2/a3, apply_layer      -> operators.py:126-266 (numpy glue)
  * gmres                            -> solver.py:48-103 (numpy)
  * build_tree / build_lists         -> fmm.py:559-715 (pure Python)
Pinning: tests/test_oracle_golden.py checks every function against golden
vectors produced by running the reference itself (scripts/make_golden.py).
"""

from .core import *  # noqa: F401,F403
from .apply import OracleOperator, gmres, solve  # noqa: F401
