"""B200-native (sm_100a) rank-truncation hot path of arXiv 1803.10270's tensor PDE solvers.

Drop-in mirror of the reference package ``tensorpde`` (``__init__.py:10-39``)
for the hot path named by BASELINE.json: CP tensors, separable operator apply,
ALS truncation, hSVD truncation of hierarchical Tucker tensors, and the
explicit / implicit integrators that call them.  Compute runs in hand-written
CUDA kernels behind the C ABI in ``include/tpde_b200.h``; there is no CPU
fallback.
"""

from ._lib import ConditioningError, StepFailure
from .basis import BasisSpec, FactorKind, factor_matrix, fourier_diff_matrix
from .cp import (ALSApproxConfig, CPTensor, add, cp_approx_als, inner_product, norm, pad_rank,
                 random_cp, rank_reduce_als, scale)
from .ht import DimensionTree, HTTensor, balanced_tree, from_cp, truncate, truncate_batch
from .io import load_tensor, save_tensor
from . import diagnostics
from .operators import (CrankNicolsonPair, SeparableOperator, advection_operator, apply,
                        crank_nicolson_pair, implicit_euler_pair)

__version__ = "0.1.0"

__all__ = [
    "BasisSpec", "FactorKind", "factor_matrix", "fourier_diff_matrix",
    "CPTensor", "ALSApproxConfig", "cp_approx_als", "rank_reduce_als", "inner_product", "norm",
    "add", "scale", "random_cp", "pad_rank", "ConditioningError", "StepFailure",
    "SeparableOperator", "CrankNicolsonPair", "advection_operator", "apply", "crank_nicolson_pair",
    "implicit_euler_pair",
    "HTTensor", "DimensionTree", "balanced_tree", "from_cp", "truncate", "truncate_batch",
    "save_tensor", "load_tensor", "diagnostics",
    "__version__",
]
