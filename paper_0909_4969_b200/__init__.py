"""B200-native MACH (arXiv 0909.4969) hot path: Bernoulli sampler + Tucker
HOSVD/HOOI on the sampled tensor, behind the reference's interface.

The compute lives in libmach_b200.so (hand-written sm_100a CUDA behind the C
ABI in include/mach_b200.h); this package is the ctypes face of it.
"""
from ._lib import build, header_symbols, lib  # noqa: F401
from .api import (  # noqa: F401
    ArgumentError,
    IoError,
    ParseError,
    SampleStream,
    achlioptas_bounds,
    load_tensor,
    min_sampling_probability,
    save_tensor,
    tensor_file_info,
    theorem1_bound,
    theorem1_conditions,
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
    TruncatedSvd,
    TuckerModel,
    truncated_svd,
    accuracy,
    comm_unique_id,
    compare,
    default_context,
    hooi,
    kernel_stats,
    profile,
    hosvd,
    leading_left_singular_vectors,
    left_singular_basis,
    low_rank_approx,
    mach_hooi,
    mach_hosvd,
    mode_gram,
    mode_product,
    pc_correlation,
    pearson,
    reconstruct,
    sparsify,
    sparse_row_gram,
    sparsify_slab,
    subspace_sin,
)

__version__ = "0.1.0"
