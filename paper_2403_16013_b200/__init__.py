"""B200-native (sm_100a) complex multi-component (DD/TD/QD) GEMM and blocked
LU -- the hot path of arXiv:2403.16013 behind the reference package's API
(mpclu).  See DESIGN.md.

The public names mirror mpclu/__init__.py:10-58 for the hot path; the CUDA
library (lib/libmpcb200.so, built by ``python -m
paper_2403_16013_b200.build``) is loaded on first use and there is no CPU
fallback.
"""

from .rmatrix import Expansion, RealMatrix, mat_add, mat_sub, random_matrix, renorm_planes
from .cmatrix import (
    KernelChoice,
    PlanarComplexMatrix,
    cgemm,
    cgemm_3m,
    cgemm_4m,
    real_kernel_calls,
    reset_real_kernel_calls,
    rgemm_blocked,
    rgemm_naive,
    rgemm_strassen,
)
from .lu import (
    ComplexScalar,
    ComplexVector,
    LinearSystem,
    LUFactors,
    SingularMatrixError,
    lu_blocked,
    lu_normal,
    max_rel_err,
    permuted,
    solve,
    trsm_unit_lower,
)
from .ozaki import SplitStack, ozaki_split, rgemm_ozaki, split_exactness_bound
from .expansion import PRECISIONS, PRECISION_BITS, REFERENCE_K, eps_for, digits_for

__version__ = "0.1.0"
