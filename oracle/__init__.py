"""TEST INFRASTRUCTURE ONLY — ctypes wrapper over the CPU oracle (liboracle.so).

The oracle restates the reference's hot path (/root/reference/proj/src) without
Eigen; see oracle/oracle.hpp.  Only tests/, __graft_entry__.smoke() and
bench.py's CPU arms import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# ORACLE_VARIANT=omp: the all-cores build (-march=native -fopenmp; bit-identical
# results), used by bench.py's reference arm and all-cores CPU baseline line
_OMP = os.environ.get("ORACLE_VARIANT") == "omp"
_LIB_PATH = os.path.join(_HERE, "liboracle_omp.so" if _OMP else "liboracle.so")
_lib = None

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_llp = C.POINTER(C.c_longlong)
_vpp = C.POINTER(C.c_void_p)


class OracleError(Exception):
    def __init__(self, kind: int, msg: str, index: int = 0):
        super().__init__(msg)
        self.kind = kind
        self.singular_index = index


class ArgumentError(OracleError):
    pass


class ShapeError(OracleError):
    pass


class ConvergenceError(OracleError):
    pass


_KINDS = {1: ArgumentError, 2: ShapeError, 3: ConvergenceError}


def build(force: bool = False) -> str:
    """Compile liboracle.so with the committed Makefile (g++, -O3, no -march)."""
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE] + (["omp"] if _OMP else []), check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        L.orc_counter_hash64.restype = C.c_ulonglong
        L.orc_counter_hash64.argtypes = [C.c_ulonglong, C.c_ulonglong]
        L.orc_counter_uniform01.restype = C.c_double
        L.orc_counter_uniform01.argtypes = [C.c_ulonglong, C.c_ulonglong]
        for name in ("orc_tensor_norm_dense", "orc_tensor_norm_sparse", "orc_model_fit", "orc_subspace_gap"):
            getattr(L, name).restype = C.c_double
        L.orc_subspace_gap.argtypes = [C.c_int, C.c_int, _dp, _dp]
        L.orc_sparse_nnz.restype = C.c_longlong
        L.orc_dense_size.restype = C.c_longlong
        for name in ("orc_tensor_norm_dense", "orc_tensor_norm_sparse", "orc_model_fit", "orc_model_iterations",
                     "orc_model_n_sweep_fits", "orc_model_n_warnings", "orc_model_order", "orc_sparse_nnz",
                     "orc_dense_size", "orc_dense_free", "orc_sparse_free", "orc_model_free"):
            getattr(L, name).argtypes = [C.c_void_p]
        L.orc_model_rank.argtypes = [C.c_void_p, C.c_int]
        L.orc_model_dim.argtypes = [C.c_void_p, C.c_int]
        L.orc_sparsify.argtypes = [C.c_void_p, C.c_double, C.c_ulonglong, _vpp]
        L.orc_hooi_dense.argtypes = [C.c_void_p, _ip, C.c_int, C.c_double, _vpp]
        L.orc_hooi_sparse.argtypes = [C.c_void_p, _ip, C.c_int, C.c_double, _vpp]
        L.orc_hosvd_dense.argtypes = [C.c_void_p, _ip, _vpp]
        L.orc_hosvd_sparse.argtypes = [C.c_void_p, _ip, _vpp]
        L.orc_mach_hooi.argtypes = [C.c_void_p, _ip, C.c_double, C.c_ulonglong, C.c_int, C.c_double, _vpp, _vpp]
        L.orc_mach_hosvd.argtypes = [C.c_void_p, _ip, C.c_double, C.c_ulonglong, _vpp, _vpp]
        L.orc_accuracy.argtypes = [C.c_void_p, C.c_void_p, _dp]
        L.orc_random_tensor.argtypes = [C.c_int, _ip, C.c_ulonglong, _dp]
        L.orc_random_matrix.argtypes = [C.c_int, C.c_int, C.c_ulonglong, _dp]
        L.orc_random_orthogonal.argtypes = [C.c_int, C.c_ulonglong, _dp]
        L.orc_model_warning.argtypes = [C.c_void_p, C.c_int, C.c_char_p, C.c_int]
        L.orc_model_factor.argtypes = [C.c_void_p, C.c_int, _dp]
        L.orc_model_core.argtypes = [C.c_void_p, _dp]
        L.orc_model_sweep_fits.argtypes = [C.c_void_p, _dp]
        L.orc_dense_new.argtypes = [C.c_int, _ip, _dp, _vpp]
        L.orc_sparse_new.argtypes = [C.c_int, _ip, C.c_longlong, _llp, _dp, _vpp]
        L.orc_sparse_get.argtypes = [C.c_void_p, _llp, _dp]
        L.orc_densify.argtypes = [C.c_void_p, _dp]
        L.orc_matricize.argtypes = [C.c_void_p, C.c_int, _dp]
        L.orc_mode_product_dense.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, C.c_int, _dp]
        L.orc_mode_product_sparse.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, C.c_int, _dp]
        L.orc_sparse_row_gram.argtypes = [C.c_void_p, C.c_int, _dp]
        L.orc_sym_eig.argtypes = [C.c_int, _dp, _dp, _dp]
        L.orc_jacobi_eig.argtypes = [C.c_int, _dp, _dp, _dp]
        L.orc_left_singular_basis.argtypes = [C.c_int, C.c_int, _dp, C.c_int, _dp, _dp, _ip, _ip]
        L.orc_low_rank_approx.argtypes = [C.c_int, C.c_int, _dp, C.c_int, _dp]
        L.orc_pearson.argtypes = [C.c_int, _dp, _dp, _dp]
        L.orc_pc_correlation.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, _dp, _ip]
        L.orc_compare.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, _dp, _ip, _ip, _dp, _dp, _dp]
        L.orc_truncated_svd.argtypes = [C.c_int, C.c_int, _dp, C.c_int, _dp, _dp, _dp]
        L.orc_reconstruct.argtypes = [C.c_void_p, _dp]
        L.orc_last_error.argtypes = [C.c_char_p, C.c_int]
        L.orc_phase_times.argtypes = [_dp, _dp, _dp, C.c_int, _ip]
        # SURVEY §8(f) rows (oracle_ext.cpp)
        L.orc_ext_last_error.restype = C.c_char_p
        L.orc_theorem1_bound.argtypes = [C.c_void_p, C.c_void_p, _ip, C.c_double, _dp, _ip, _dp]
        L.orc_theorem1_conditions.argtypes = [C.c_int, _ip, C.c_double, _dp, _ip]
        L.orc_min_sampling_probability.argtypes = [C.c_int, _ip, _dp]
        L.orc_ingest_buckets.restype = C.c_longlong
        L.orc_ingest_buckets.argtypes = [C.c_longlong, _llp, C.c_longlong, _llp]
        L.orc_ingest_indexed.argtypes = [C.c_longlong, _ip, _ip, _llp, _dp, C.c_int, C.c_int, C.c_longlong, C.c_int, _dp]
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        buf = C.create_string_buffer(512)
        lib().orc_last_error(buf, 512)
        idx = lib().orc_last_error_index()
        raise _KINDS.get(rc, OracleError)(rc, buf.value.decode(), idx)


def _d(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _dims(dims) -> C.Array:
    return (C.c_int * len(dims))(*[int(d) for d in dims])


# ---------------------------------------------------------------------------
# value types (Fortran order == first mode fastest, column-major matrices)
# ---------------------------------------------------------------------------
class Dense:
    """First-mode-fastest dense tensor (proj/include/mach/tensor.hpp:13-39)."""

    def __init__(self, values: np.ndarray, dims=None):
        values = np.asarray(values, dtype=np.float64)
        if dims is None:
            dims = values.shape
            flat = np.ascontiguousarray(values.reshape(-1, order="F"))
        else:
            flat = np.ascontiguousarray(values.reshape(-1))
        self.dims = tuple(int(d) for d in dims)
        h = C.c_void_p()
        _check(lib().orc_dense_new(len(self.dims), _dims(self.dims), _d(flat), C.byref(h)))
        self.h = h
        self.flat = flat

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_dense_free(self.h)
            self.h = None

    def norm(self) -> float:
        return lib().orc_tensor_norm_dense(self.h)

    def array(self) -> np.ndarray:
        return self.flat.reshape(self.dims, order="F")


class Sparse:
    """Canonical COO (proj/include/mach/tensor.hpp:48-75)."""

    def __init__(self, h, dims):
        self.h = h
        self.dims = tuple(int(d) for d in dims)

    @classmethod
    def from_entries(cls, dims, idx, vals):
        idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int64))
        vals = _f64(vals)
        h = C.c_void_p()
        _check(lib().orc_sparse_new(len(dims), _dims(dims), len(idx), idx.ctypes.data_as(_llp), _d(vals),
                                    C.byref(h)))
        return cls(h, dims)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_sparse_free(self.h)
            self.h = None

    @property
    def nnz(self) -> int:
        return lib().orc_sparse_nnz(self.h)

    def entries(self):
        n = self.nnz
        idx = np.empty(n, dtype=np.int64)
        vals = np.empty(n, dtype=np.float64)
        lib().orc_sparse_get(self.h, idx.ctypes.data_as(_llp), _d(vals))
        return idx, vals

    def densify(self) -> np.ndarray:
        out = np.empty(int(np.prod(self.dims)), dtype=np.float64)
        _check(lib().orc_densify(self.h, _d(out)))
        return out.reshape(self.dims, order="F")

    def norm(self) -> float:
        return lib().orc_tensor_norm_sparse(self.h)


@dataclass
class Model:
    core: np.ndarray
    factors: list
    ranks: tuple
    iterations: int
    fit: float
    sweep_fits: list
    warnings: list = field(default_factory=list)
    _h: object = None

    @classmethod
    def from_handle(cls, h):
        L = lib()
        d = L.orc_model_order(h)
        ranks = tuple(L.orc_model_rank(h, m) for m in range(d))
        dims = tuple(L.orc_model_dim(h, m) for m in range(d))
        core = np.empty(int(np.prod(ranks)), dtype=np.float64)
        L.orc_model_core(h, _d(core))
        factors = []
        for m in range(d):
            f = np.empty(dims[m] * ranks[m], dtype=np.float64)
            L.orc_model_factor(h, m, _d(f))
            factors.append(f.reshape((dims[m], ranks[m]), order="F"))
        n = L.orc_model_n_sweep_fits(h)
        sf = np.empty(n, dtype=np.float64)
        L.orc_model_sweep_fits(h, _d(sf))
        warns = []
        for i in range(L.orc_model_n_warnings(h)):
            buf = C.create_string_buffer(512)
            L.orc_model_warning(h, i, buf, 512)
            warns.append(buf.value.decode())
        m = cls(core.reshape(ranks, order="F"), factors, ranks, L.orc_model_iterations(h), L.orc_model_fit(h),
                list(sf), warns)
        m._h = h
        return m

    def __del__(self):
        if self._h is not None and _lib is not None:
            _lib.orc_model_free(self._h)
            self._h = None


# ---------------------------------------------------------------------------
# functions (names follow proj/include/mach/*.hpp)
# ---------------------------------------------------------------------------
def counter_hash64(seed: int, counter: int) -> int:
    return lib().orc_counter_hash64(seed, counter)


def counter_uniform01(seed: int, counter: int) -> float:
    return lib().orc_counter_uniform01(seed, counter)


def sparsify(t: Dense, p: float, seed: int) -> Sparse:
    h = C.c_void_p()
    _check(lib().orc_sparsify(t.h, float(p), int(seed), C.byref(h)))
    return Sparse(h, t.dims)


def _ranks(ranks):
    return (C.c_int * len(ranks))(*[int(r) for r in ranks])


def hosvd(t, ranks) -> Model:
    h = C.c_void_p()
    fn = lib().orc_hosvd_dense if isinstance(t, Dense) else lib().orc_hosvd_sparse
    if len(ranks) != len(t.dims):
        raise ArgumentError(1, "ranks must name one rank per mode")
    _check(fn(t.h, _ranks(ranks), C.byref(h)))
    return Model.from_handle(h)


def hooi(t, ranks, max_iterations: int = 50, fit_tolerance: float = 1e-4) -> Model:
    h = C.c_void_p()
    fn = lib().orc_hooi_dense if isinstance(t, Dense) else lib().orc_hooi_sparse
    if len(ranks) != len(t.dims):
        raise ArgumentError(1, "ranks must name one rank per mode")
    _check(fn(t.h, _ranks(ranks), int(max_iterations), float(fit_tolerance), C.byref(h)))
    return Model.from_handle(h)


def mach_hooi(t: Dense, ranks, p, seed, max_iterations=50, fit_tolerance=1e-4):
    hm, hs = C.c_void_p(), C.c_void_p()
    _check(lib().orc_mach_hooi(t.h, _ranks(ranks), float(p), int(seed), int(max_iterations), float(fit_tolerance),
                               C.byref(hm), C.byref(hs)))
    return Model.from_handle(hm), Sparse(hs, t.dims)


def mach_hosvd(t: Dense, ranks, p, seed):
    hm, hs = C.c_void_p(), C.c_void_p()
    _check(lib().orc_mach_hosvd(t.h, _ranks(ranks), float(p), int(seed), C.byref(hm), C.byref(hs)))
    return Model.from_handle(hm), Sparse(hs, t.dims)


def accuracy(t: Dense, model: Model) -> float:
    out = C.c_double()
    _check(lib().orc_accuracy(t.h, model._h, C.byref(out)))
    return out.value


def reconstruct(model: Model) -> np.ndarray:
    dims = tuple(f.shape[0] for f in model.factors)
    out = np.empty(int(np.prod(dims)), dtype=np.float64)
    _check(lib().orc_reconstruct(model._h, _d(out)))
    return out.reshape(dims, order="F")


def matricize(t: Dense, mode: int) -> np.ndarray:
    d = t.dims
    if not 0 <= mode < len(d):
        raise ArgumentError(1, "mode out of range")
    rows = d[mode]
    cols = int(np.prod(d)) // rows
    out = np.empty(rows * cols, dtype=np.float64)
    _check(lib().orc_matricize(t.h, mode, _d(out)))
    return out.reshape((rows, cols), order="F")


def mode_product(t, m: np.ndarray, mode: int) -> np.ndarray:
    mf = np.asfortranarray(np.asarray(m, dtype=np.float64))
    od = list(t.dims)
    if not 0 <= mode < len(od):
        raise ArgumentError(1, "mode out of range")
    od[mode] = mf.shape[0]
    out = np.empty(int(np.prod(od)), dtype=np.float64)
    fn = lib().orc_mode_product_dense if isinstance(t, Dense) else lib().orc_mode_product_sparse
    flat = np.ascontiguousarray(mf.reshape(-1, order="F"))
    _check(fn(t.h, mf.shape[0], mf.shape[1], _d(flat), mode, _d(out)))
    return out.reshape(od, order="F")


def sparse_row_gram(t: Sparse, mode: int) -> np.ndarray:
    n = t.dims[mode]
    out = np.empty(n * n, dtype=np.float64)
    _check(lib().orc_sparse_row_gram(t.h, mode, _d(out)))
    return out.reshape((n, n), order="F")


def sym_eig(a: np.ndarray):
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    n = a.shape[0]
    ev = np.empty(n)
    vec = np.empty(n * n)
    flat = np.ascontiguousarray(a.reshape(-1, order="F"))
    _check(lib().orc_sym_eig(n, _d(flat), _d(ev), _d(vec)))
    return ev, vec.reshape((n, n), order="F")


def jacobi_eig(a: np.ndarray):
    a = np.asarray(a, dtype=np.float64)
    n = a.shape[0]
    ev = np.empty(n)
    vec = np.empty(n * n)
    flat = np.ascontiguousarray(a.reshape(-1, order="F"))
    _check(lib().orc_jacobi_eig(n, _d(flat), _d(ev), _d(vec)))
    return ev, vec.reshape((n, n), order="F")


def left_singular_basis(m: np.ndarray, k: int):
    m = np.asarray(m, dtype=np.float64)
    rows, cols = m.shape
    basis = np.empty(rows * max(k, 0) if k > 0 else 1)
    sv = np.empty(max(k, 1))
    nr, comp = C.c_int(), C.c_int()
    flat = np.ascontiguousarray(m.reshape(-1, order="F"))
    _check(lib().orc_left_singular_basis(rows, cols, _d(flat), int(k), _d(basis), _d(sv), C.byref(nr),
                                         C.byref(comp)))
    return basis.reshape((rows, k), order="F"), sv[:k].copy(), nr.value, bool(comp.value)


def pearson(x, y) -> float:
    """metrics.cpp:67-96."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    if x.size != y.size:
        raise ShapeError(2, "correlation inputs have different lengths")
    out = C.c_double()
    _check(lib().orc_pearson(int(x.size), _d(x), _d(y), C.byref(out)))
    return out.value


def pc_correlation(exact: "Model", approx: "Model", mode: int, component: int = 1):
    """metrics.cpp:98-122: (rho, flipped)."""
    out, fl = C.c_double(), C.c_int()
    _check(lib().orc_pc_correlation(exact._h, approx._h, int(mode), int(component), C.byref(out), C.byref(fl)))
    return out.value, bool(fl.value)


def compare(exact: "Model", approx: "Model", reference: "Dense") -> dict:
    """metrics.cpp:124-159 (ComparisonReport)."""
    d = len(exact.factors)
    rho, ts = np.zeros(d), np.zeros(d)
    fl, ti = (C.c_int * d)(), (C.c_int * d)()
    acc, core = np.zeros(2), np.zeros(2)
    _check(lib().orc_compare(exact._h, approx._h, reference.h, _d(rho), fl, ti, _d(ts), _d(acc), _d(core)))
    return {"per_mode_rho": rho, "flipped": [bool(v) for v in fl], "tied": [bool(v) for v in ti],
            "tie_subspace_sin": ts, "accuracy_exact": acc[0], "accuracy_mach": acc[1],
            "core_interaction": (core[0], core[1])}


def truncated_svd(m: np.ndarray, k: int):
    """(left rows x k, singular values k, right cols x k) — linalg.cpp:301-305."""
    m = np.asarray(m, dtype=np.float64)
    rows, cols = m.shape
    left = np.empty(max(rows * k, 1))
    right = np.empty(max(cols * k, 1))
    sv = np.empty(max(k, 1))
    flat = np.ascontiguousarray(m.reshape(-1, order="F"))
    _check(lib().orc_truncated_svd(rows, cols, _d(flat), int(k), _d(left), _d(sv), _d(right)))
    return left[: rows * k].reshape((rows, k), order="F"), sv[:k].copy(), right[: cols * k].reshape((cols, k), order="F")


def low_rank_approx(m: np.ndarray, k: int) -> np.ndarray:
    m = np.asarray(m, dtype=np.float64)
    rows, cols = m.shape
    out = np.empty(rows * cols)
    flat = np.ascontiguousarray(m.reshape(-1, order="F"))
    _check(lib().orc_low_rank_approx(rows, cols, _d(flat), int(k), _d(out)))
    return out.reshape((rows, cols), order="F")


def subspace_gap(a: np.ndarray, b: np.ndarray) -> float:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1, order="F"))
    b2 = np.asarray(b, dtype=np.float64)
    n, k = b2.shape
    b = np.ascontiguousarray(b2.reshape(-1, order="F"))
    return lib().orc_subspace_gap(n, k, _d(a), _d(b))


def _check_ext(rc: int):
    if rc != 0:
        raise _KINDS.get(rc, OracleError)(rc, lib().orc_ext_last_error().decode(), 0)


def _bound_dict(scal, flags, per_mode=None):
    out = {"b": scal[0], "p": scal[1], "p_min": scal[2], "t": scal[3], "success_probability": scal[4],
           "dims_large_enough": bool(flags[0]), "dims_balanced": bool(flags[1]), "p_above_min": bool(flags[2]),
           "conditions_met": bool(flags[3]), "per_mode": []}
    if per_mode is not None:
        for r in per_mode.reshape(-1, 5):
            out["per_mode"].append({"rank": int(r[0]), "x_residual": r[1], "xhat_residual": r[2],
                                    "x_lowrank_norm": r[3], "t_i": r[4]})
    return out


def theorem1_bound(x: "Dense", xhat: "Sparse", ranks, p: float) -> dict:
    """BoundReport as a dict — bounds.cpp:152-184."""
    d = len(x.dims)
    scal = np.zeros(5)
    flags = (C.c_int * 4)()
    pm = np.zeros(5 * d)
    rk = (C.c_int * max(len(ranks), d))(*[int(r) for r in ranks])
    if len(ranks) != d:
        raise ArgumentError(1, "ranks must name one rank per mode")
    _check_ext(lib().orc_theorem1_bound(x.h, xhat.h, rk, float(p), _d(scal), flags, _d(pm)))
    return _bound_dict(scal, flags, pm)


def theorem1_conditions(dims, p: float) -> dict:
    scal = np.zeros(5)
    flags = (C.c_int * 4)()
    _check_ext(lib().orc_theorem1_conditions(len(dims), _dims(dims) if len(dims) else None, float(p), _d(scal), flags))
    return _bound_dict(scal, flags)


def min_sampling_probability(dims) -> float:
    out = np.zeros(1)
    _check_ext(lib().orc_min_sampling_probability(len(dims), _dims(dims) if len(dims) else None, _d(out)))
    return float(out[0])


def ingest_indexed(machine, metric, ts, value, n_machines: int, n_metrics: int, bucket_seconds: int = 300,
                   carry_forward: bool = False):
    """(tensor machines x metrics x buckets, first bucket start) — ingest.cpp:51-135 on pre-indexed records."""
    machine = np.ascontiguousarray(machine, dtype=np.int32)
    metric = np.ascontiguousarray(metric, dtype=np.int32)
    ts = np.ascontiguousarray(ts, dtype=np.int64)
    value = _f64(value)
    n = len(ts)
    llp = C.POINTER(C.c_longlong)
    fb = C.c_longlong(0)
    buckets = lib().orc_ingest_buckets(n, ts.ctypes.data_as(llp), int(bucket_seconds), C.byref(fb))
    out = np.zeros(n_machines * n_metrics * buckets)
    _check_ext(lib().orc_ingest_indexed(n, machine.ctypes.data_as(_ip), metric.ctypes.data_as(_ip),
                                        ts.ctypes.data_as(llp), _d(value), n_machines, n_metrics, int(bucket_seconds),
                                        1 if carry_forward else 0, _d(out)))
    return out.reshape((n_machines, n_metrics, buckets), order="F"), int(fb.value)


def random_tensor(dims, seed: int) -> np.ndarray:
    out = np.empty(int(np.prod(dims)), dtype=np.float64)
    lib().orc_random_tensor(len(dims), _dims(dims), int(seed), _d(out))
    return out.reshape(tuple(dims), order="F")


def random_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    out = np.empty(rows * cols, dtype=np.float64)
    lib().orc_random_matrix(rows, cols, int(seed), _d(out))
    return out.reshape((rows, cols), order="F")


def random_orthogonal(n: int, seed: int) -> np.ndarray:
    out = np.empty(n * n, dtype=np.float64)
    lib().orc_random_orthogonal(n, int(seed), _d(out))
    return out.reshape((n, n), order="F")


def phase_times():
    s, h = C.c_double(), C.c_double()
    n = C.c_int()
    buf = (C.c_double * 1024)()
    lib().orc_phase_times(C.byref(s), C.byref(h), buf, 1024, C.byref(n))
    return s.value, h.value, list(buf[: min(n.value, 1024)])
