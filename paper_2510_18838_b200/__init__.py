"""B200-native field-mapping hot path of PCMS (arXiv 2510.18838).

Drop-in for the pointwise transfer API of the reference package `fieldbridge`
(point search, MLS/RBF fit, prepared-transfer apply), computed by
hand-written sm_100a CUDA kernels behind a C ABI (include/fieldmap.h,
libfieldmap.so).  There is no CPU fallback: without the built library the
compute calls raise.
"""

from . import errors
from .cycle import PointwiseCycle
from .locate import PointGrid, build_point_grid
from .pointwise import (
    AdaptiveRadius,
    ElementPatch,
    FitSpec,
    FixedRadius,
    PreparedTransfer,
    RadialBasisSpec,
    RbfKind,
    eval_rbf,
    fit_local,
    fit_point_cloud,
    n_monomials,
    select_support,
    transfer_extrinsic,
    transfer_pointwise,
)

__version__ = "0.1.0"
kernel_backend = "b200"

__all__ = [
    "errors",
    "PointGrid",
    "PointwiseCycle",
    "build_point_grid",
    "AdaptiveRadius",
    "ElementPatch",
    "FitSpec",
    "FixedRadius",
    "PreparedTransfer",
    "RadialBasisSpec",
    "RbfKind",
    "eval_rbf",
    "fit_local",
    "fit_point_cloud",
    "n_monomials",
    "select_support",
    "transfer_extrinsic",
    "transfer_pointwise",
]
