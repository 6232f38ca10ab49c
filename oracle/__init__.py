"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, fp64 numpy implementation of what the FRSVT hot path computes,
written from PAPER.md (arXiv 1509.00296). Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference`
leg may import it. The product path (`paper_1509_00296_b200`) never imports,
links or executes anything under `oracle/`, and this package never imports
the product path: the two share no code. Inputs come from `synth/` only.

Modules
  linalg : one-sided Jacobi SVD (exact-SVT backbone), Newton polar
           decomposition, QR with column pivoting (dgeqp3 as in P:177).
  svt    : soft shrinkage, exact SVT (Def. 1), weighted SVT (fn. 1),
           2-norm-ball projection (Def. 3).
  frsvt  : Algorithm 1 (FRSVT) step by step, with range propagation.
  rpca   : textbook inexact-ALM RPCA hosting FRSVT and the
           reweighted WSVT sequence of BASELINE config c4.

Parity status of each function is stated in its docstring ("pinned by ..." or
"parity unpinned") and summarised in DESIGN.md.
"""
from .linalg import jacobi_svd, polar_newton, qr_cp, norm2_power
from .svt import soft_shrink, svt_exact, wsvt_exact, proj_2ball
from .frsvt import frsvt, FrsvtResult
from .rpca import rpca_ialm, reweighted_wsvt

__all__ = ["jacobi_svd", "polar_newton", "qr_cp", "norm2_power", "soft_shrink",
           "svt_exact", "wsvt_exact", "proj_2ball", "frsvt", "FrsvtResult",
           "rpca_ialm", "reweighted_wsvt"]
