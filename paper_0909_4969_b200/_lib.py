"""ctypes binding of libmach_b200.so (C ABI: include/mach_b200.h).

The shared library is built in-tree (``make -C paper_0909_4969_b200``); this
module never falls back to anything else — a missing or unloadable library is
an ImportError/OSError at first use.
"""
from __future__ import annotations

import ctypes as C
import os
import re
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.environ.get("MACH_LIB_PATH") or os.path.join(HERE, "libmach_b200.so")  # override: A/B builds
HEADER = os.path.join(ROOT, "include", "mach_b200.h")

_lib = None

MACH_OK, MACH_ERR_ARGUMENT, MACH_ERR_SHAPE, MACH_ERR_CONVERGENCE = 0, 1, 2, 3
MACH_ERR_CUDA, MACH_ERR_OOM, MACH_ERR_NCCL, MACH_ERR_INTERNAL = 4, 5, 6, 7
MACH_ERR_IO, MACH_ERR_PARSE = 8, 9
MACH_F32, MACH_F64 = 0, 1


class BoundMode(C.Structure):
    _fields_ = [("rank", C.c_int), ("x_residual", C.c_double), ("xhat_residual", C.c_double),
                ("x_lowrank_norm", C.c_double), ("t_i", C.c_double)]


class BoundReport(C.Structure):
    _fields_ = [("b", C.c_double), ("p", C.c_double), ("p_min", C.c_double), ("t", C.c_double),
                ("success_probability", C.c_double), ("dims_large_enough", C.c_int), ("dims_balanced", C.c_int),
                ("p_above_min", C.c_int), ("conditions_met", C.c_int)]


def build(force: bool = False) -> str:
    """Compile every CUDA source for sm_100a into libmach_b200.so (in-tree)."""
    if force:
        subprocess.run(["make", "-s", "-C", HERE, "clean"], check=True)
    subprocess.run(["make", "-s", "-j8", "-C", HERE], check=True)
    return LIB_PATH


vp = C.c_void_p
vpp = C.POINTER(C.c_void_p)
ip = C.POINTER(C.c_int)
dp = C.POINTER(C.c_double)
i64 = C.c_int64
i64p = C.POINTER(C.c_int64)

_SIGS = {
    "mach_last_error": (C.c_char_p, []),
    "mach_last_error_index": (C.c_int, []),
    "mach_version": (C.c_char_p, []),
    "mach_ctx_create": (C.c_int, [C.c_int, vpp]),
    "mach_ctx_destroy": (C.c_int, [vp]),
    "mach_ctx_set_stream": (C.c_int, [vp, vp]),
    "mach_ctx_synchronize": (C.c_int, [vp]),
    "mach_ctx_launch_count": (C.c_int, [vp, i64p]),
    "mach_dense_upload": (C.c_int, [vp, C.c_int, C.c_int, ip, vp, vpp]),
    "mach_dense_wrap": (C.c_int, [vp, C.c_int, C.c_int, ip, vp, vpp]),
    "mach_dense_download": (C.c_int, [vp, vp]),
    "mach_dense_free": (C.c_int, [vp]),
    "mach_sparsify": (C.c_int, [vp, vp, C.c_double, C.c_uint64, vpp]),
    "mach_sparsify_host": (C.c_int, [vp, C.c_int, C.c_int, ip, vp, C.c_double, C.c_uint64, i64p,
                                     C.POINTER(i64p), C.POINTER(dp)]),
    "mach_free_host": (None, [vp]),
    "mach_sparse_upload": (C.c_int, [vp, C.c_int, C.c_int, ip, i64, i64p, dp, vpp]),
    "mach_sparse_nnz": (C.c_int, [vp, i64p]),
    "mach_sparse_download": (C.c_int, [vp, i64p, dp]),
    "mach_sparse_norm": (C.c_int, [vp, dp]),
    "mach_sparse_free": (C.c_int, [vp]),
    "mach_hosvd_sparse": (C.c_int, [vp, vp, ip, vpp]),
    "mach_hosvd_dense": (C.c_int, [vp, vp, ip, vpp]),
    "mach_hooi_sparse": (C.c_int, [vp, vp, ip, C.c_int, C.c_double, vpp]),
    "mach_hooi_dense": (C.c_int, [vp, vp, ip, C.c_int, C.c_double, vpp]),
    "mach_mach_hooi": (C.c_int, [vp, vp, ip, C.c_double, C.c_uint64, C.c_int, C.c_double, vpp, vpp]),
    "mach_mach_hosvd": (C.c_int, [vp, vp, ip, C.c_double, C.c_uint64, vpp, vpp]),
    "mach_hooi_begin": (C.c_int, [vp, vp, ip, vpp]),
    "mach_hooi_begin_dense": (C.c_int, [vp, vp, ip, vpp]),
    "mach_hooi_step": (C.c_int, [vp, C.c_int, C.c_double, ip, ip]),
    "mach_hooi_state": (C.c_int, [vp, dp, ip]),
    "mach_hooi_model": (C.c_int, [vp, vpp]),
    "mach_hooi_ttm_bytes": (C.c_int, [vp, C.c_int, C.POINTER(C.c_longlong)]),
    "mach_hooi_begin_from": (C.c_int, [vp, vp, ip, vp, vpp]),
    "mach_hooi_set_norm2": (C.c_int, [vp, C.c_double]),
    "mach_hooi_mode_y": (C.c_int, [vp, C.c_int, vpp, ip, ip]),
    "mach_hooi_mode_update": (C.c_int, [vp, C.c_int]),
    "mach_hooi_sweep_end": (C.c_int, [vp, C.c_double, ip]),
    "mach_sparsify_slab": (C.c_int, [vp, vp, C.c_int, ip, C.c_int64, C.c_double, C.c_uint64, vpp]),
    "mach_sparse_device_view": (C.c_int, [vp, vpp, vpp, ip]),
    "mach_sparse_from_device": (C.c_int, [vp, C.c_int, C.c_int, ip, C.c_int64, vp, vp, vpp]),
    "mach_session_free": (C.c_int, [vp]),
    "mach_ctx_profile": (C.c_int, [vp, C.c_int]),
    "mach_ctx_kernel_stat": (C.c_int, [vp, C.c_int, C.c_char_p, C.c_size_t, i64p, dp]),
    "mach_model_info": (C.c_int, [vp, ip, ip, dp, ip, ip]),
    "mach_model_dims": (C.c_int, [vp, ip, ip]),
    "mach_model_core": (C.c_int, [vp, dp]),
    "mach_model_factor": (C.c_int, [vp, C.c_int, dp]),
    "mach_model_sweep_fits": (C.c_int, [vp, dp]),
    "mach_model_warning": (C.c_int, [vp, C.c_int, C.c_char_p, C.c_size_t]),
    "mach_model_times": (C.c_int, [vp, dp, dp, dp, dp, C.c_int]),
    "mach_model_free": (C.c_int, [vp]),
    "mach_accuracy": (C.c_int, [vp, vp, vp, dp]),
    "mach_reconstruct": (C.c_int, [vp, vp, vpp]),
    "mach_left_singular_basis": (C.c_int, [vp, C.c_int, C.c_int, dp, C.c_int, dp, dp, ip, ip]),
    "mach_mode_product_dense": (C.c_int, [vp, vp, C.c_int, C.c_int, dp, C.c_int, vpp]),
    "mach_mode_product_sparse": (C.c_int, [vp, vp, C.c_int, C.c_int, dp, C.c_int, vpp]),
    "mach_dense_mode_gram": (C.c_int, [vp, vp, C.c_int, dp, ip]),
    "mach_comm_unique_id": (C.c_int, [C.c_char_p]),
    "mach_ctx_comm_init": (C.c_int, [vp, C.c_int, C.c_int, C.c_char_p]),
    "mach_hooi_shard": (C.c_int, [vp]),
    "mach_model_accuracy": (C.c_int, [vp, vp, ip, dp, C.POINTER(dp), dp]),
    "mach_subspace_sin": (C.c_int, [vp, C.c_int, C.c_int, dp, dp, dp]),
    "mach_truncated_svd": (C.c_int, [vp, C.c_int, C.c_int, dp, C.c_int, dp, dp, dp]),
    "mach_low_rank_approx": (C.c_int, [vp, C.c_int, C.c_int, dp, C.c_int, dp]),
    "mach_sparse_row_gram": (C.c_int, [vp, vp, C.c_int, dp]),
    "mach_hosvd_from_grams": (C.c_int, [vp, C.c_int, ip, ip, C.POINTER(dp), vpp]),
    "mach_hooi_refresh_fit": (C.c_int, [vp]),
    "mach_achlioptas_bounds": (C.c_int, [C.c_double, i64, i64, C.c_double, dp, dp]),
    "mach_min_sampling_probability": (C.c_int, [C.c_int, ip, dp]),
    "mach_theorem1_conditions": (C.c_int, [C.c_int, ip, C.c_double, C.POINTER(BoundReport)]),
    "mach_theorem1_bound": (C.c_int, [vp, vp, vp, ip, C.c_double, C.POINTER(BoundReport), C.POINTER(BoundMode)]),
    "mach_stream_begin": (C.c_int, [vp, C.c_int, C.c_int, ip, C.c_double, C.c_uint64, vpp]),
    "mach_stream_append": (C.c_int, [vp, vp]),
    "mach_stream_append_host": (C.c_int, [vp, vp, C.c_int]),
    "mach_stream_append_records": (C.c_int, [vp, i64, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                             dp, C.c_int, C.c_int]),
    "mach_stream_state": (C.c_int, [vp, i64p, i64p]),
    "mach_stream_tensor": (C.c_int, [vp, vpp]),
    "mach_stream_last_slab": (C.c_int, [vp, vpp]),
    "mach_stream_free": (C.c_int, [vp]),
    "mach_dense_save": (C.c_int, [vp, C.c_char_p]),
    "mach_dense_load": (C.c_int, [vp, C.c_char_p, vpp]),
    "mach_sparse_save": (C.c_int, [vp, C.c_char_p]),
    "mach_sparse_load": (C.c_int, [vp, C.c_char_p, vpp]),
    "mach_tensor_file_kind": (C.c_int, [C.c_char_p, ip, ip, ip, ip, i64p]),
}


def header_symbols() -> list[str]:
    """Every function the C ABI header declares."""
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    txt = re.sub(r"//[^\n]*", "", txt)
    return sorted(set(re.findall(r"\b(mach_[a-z0-9_]+)\s*\(", txt)))


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `make -C {HERE}` (or __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
