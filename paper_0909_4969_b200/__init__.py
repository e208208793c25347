"""B200-native MACH (arXiv 0909.4969) hot path: Bernoulli sampler + Tucker
HOSVD/HOOI on the sampled tensor, behind the reference's interface.

The compute lives in libmach_b200.so (hand-written sm_100a CUDA behind the C
ABI in include/mach_b200.h); this package is the ctypes face of it.
"""
from ._lib import build, header_symbols, lib  # noqa: F401
from .api import (  # noqa: F401
    ArgumentError,
    Context,
    ConvergenceError,
    DenseTensor,
    DeviceError,
    HooiConfig,
    HooiSession,
    LeftSingularBasis,
    MachResult,
    ShapeError,
    SparseTensor,
    SparsifyConfig,
    TuckerModel,
    accuracy,
    default_context,
    hooi,
    kernel_stats,
    profile,
    hosvd,
    left_singular_basis,
    mach_hooi,
    mach_hosvd,
    mode_gram,
    mode_product,
    reconstruct,
    sparsify,
    sparsify_slab,
)

__version__ = "0.1.0"
