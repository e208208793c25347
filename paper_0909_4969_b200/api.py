"""Python face of the B200 MACH sampler + Tucker path.

Names, argument meaning and errors follow the reference interface
(/root/reference/proj/include/mach/{sampling,tucker,linalg,tensor}.hpp):
``sparsify``, ``mach_hosvd``, ``mach_hooi``, ``hosvd``, ``hooi``,
``accuracy``, ``reconstruct``, ``mode_product``, ``left_singular_basis``,
``SparsifyConfig``, ``HooiConfig``, ``TuckerModel`` and the exception types
``ArgumentError``, ``ShapeError``, ``ConvergenceError``.

Every computation runs in libmach_b200.so on the GPU; tensors are
device-resident handles.  Host arrays are numpy arrays whose flat order is
first-mode-fastest (numpy ``order='F'``), exactly the reference layout.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


# ---------------------------------------------------------------------------
# errors (proj/include/mach/errors.hpp:9-47)
# ---------------------------------------------------------------------------
class MachError(Exception):
    code = -1


class ArgumentError(MachError, ValueError):
    code = L.MACH_ERR_ARGUMENT


class ShapeError(MachError, ValueError):
    code = L.MACH_ERR_SHAPE


class ConvergenceError(MachError, RuntimeError):
    code = L.MACH_ERR_CONVERGENCE

    def __init__(self, msg: str, singular_index: int):
        super().__init__(msg)
        self.singular_index = singular_index


class DeviceError(MachError, RuntimeError):
    code = L.MACH_ERR_CUDA


class IoError(MachError, OSError):
    code = L.MACH_ERR_IO


class ParseError(MachError, RuntimeError):
    code = L.MACH_ERR_PARSE


def _check(rc: int):
    if rc == L.MACH_OK:
        return
    lib = L.lib()
    msg = (lib.mach_last_error() or b"").decode()
    if rc == L.MACH_ERR_ARGUMENT:
        raise ArgumentError(msg)
    if rc == L.MACH_ERR_SHAPE:
        raise ShapeError(msg)
    if rc == L.MACH_ERR_CONVERGENCE:
        raise ConvergenceError(msg, lib.mach_last_error_index())
    if rc == L.MACH_ERR_IO:
        raise IoError(msg)
    if rc == L.MACH_ERR_PARSE:
        raise ParseError(msg)
    raise DeviceError(f"[{rc}] {msg}")


# ---------------------------------------------------------------------------
# context
# ---------------------------------------------------------------------------
class Context:
    """Device + stream.  One per host thread (SURVEY §8b threading contract)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(L.lib().mach_ctx_create(int(device), C.byref(h)))
        self.h = h
        self.device = device

    def set_stream(self, cuda_stream_ptr: int | None):
        _check(L.lib().mach_ctx_set_stream(self.h, C.c_void_p(cuda_stream_ptr or 0)))

    def comm_init(self, world: int, rank: int, unique_id: bytes):
        """Bind this context to an NCCL communicator (time-slab shards)."""
        _check(L.lib().mach_ctx_comm_init(self.h, int(world), int(rank), bytes(unique_id)))

    def synchronize(self):
        _check(L.lib().mach_ctx_synchronize(self.h))

    @property
    def launches(self) -> int:
        n = C.c_int64()
        _check(L.lib().mach_ctx_launch_count(self.h, C.byref(n)))
        return n.value

    def close(self):
        if getattr(self, "h", None):
            L.lib().mach_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def comm_unique_id() -> bytes:
    """NCCL unique id for Context.comm_init (rank 0 creates, the caller broadcasts)."""
    buf = C.create_string_buffer(128)
    _check(L.lib().mach_comm_unique_id(buf))
    return buf.raw


def _ctx(ctx):
    return ctx if ctx is not None else default_context()


def _dims_arr(dims):
    return (C.c_int * len(dims))(*[int(d) for d in dims])


_DT = {np.dtype(np.float32): L.MACH_F32, np.dtype(np.float64): L.MACH_F64}


# ---------------------------------------------------------------------------
# tensors
# ---------------------------------------------------------------------------
class DenseTensor:
    """Dense tensor in HBM, first mode fastest (tensor.hpp:13-39)."""

    def __init__(self, h, dims, dtype, ctx, keepalive=None):
        self.h, self.dims, self.dtype, self.ctx = h, tuple(dims), np.dtype(dtype), ctx
        self._keepalive = keepalive

    @classmethod
    def from_numpy(cls, x: np.ndarray, ctx: Context | None = None, dtype=None):
        ctx = _ctx(ctx)
        x = np.asarray(x)
        dt = np.dtype(dtype or (x.dtype if x.dtype in (np.float32, np.float64) else np.float64))
        flat = np.ascontiguousarray(x.astype(dt, copy=False).reshape(-1, order="F"))
        h = C.c_void_p()
        _check(L.lib().mach_dense_upload(ctx.h, _DT[dt], x.ndim, _dims_arr(x.shape), flat.ctypes.data_as(C.c_void_p),
                                         C.byref(h)))
        return cls(h, x.shape, dt, ctx)

    @classmethod
    def from_torch(cls, flat, dims, ctx: Context | None = None):
        """Zero-copy view of a CUDA torch tensor whose memory is first-mode-fastest.

        The library works on its own stream: the producer's pending work on
        torch's current stream is completed first, so the view never reads a
        tensor that is still being written."""
        import torch

        ctx = _ctx(ctx)
        assert flat.is_cuda and flat.is_contiguous()
        torch.cuda.current_stream(flat.device).synchronize()
        dt = {torch.float32: np.float32, torch.float64: np.float64}[flat.dtype]
        h = C.c_void_p()
        _check(L.lib().mach_dense_wrap(ctx.h, _DT[np.dtype(dt)], len(dims), _dims_arr(dims), C.c_void_p(flat.data_ptr()),
                                       C.byref(h)))
        return cls(h, dims, dt, ctx, keepalive=flat)

    def numpy(self) -> np.ndarray:
        out = np.empty(int(np.prod(self.dims)), dtype=self.dtype)
        _check(L.lib().mach_dense_download(self.h, out.ctypes.data_as(C.c_void_p)))
        return out.reshape(self.dims, order="F")

    def free(self):
        if getattr(self, "h", None):
            L.lib().mach_dense_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class SparseTensor:
    """Canonical COO in HBM (tensor.hpp:48-75): ascending flat index."""

    def __init__(self, h, dims, dtype, ctx):
        self.h, self.dims, self.dtype, self.ctx = h, tuple(dims), np.dtype(dtype), ctx

    @classmethod
    def from_entries(cls, dims, idx, vals, dtype=np.float64, ctx: Context | None = None):
        ctx = _ctx(ctx)
        idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int64))
        vals = np.ascontiguousarray(np.asarray(vals, dtype=np.float64))
        h = C.c_void_p()
        _check(L.lib().mach_sparse_upload(ctx.h, _DT[np.dtype(dtype)], len(dims), _dims_arr(dims), len(idx),
                                          idx.ctypes.data_as(L.i64p), vals.ctypes.data_as(L.dp), C.byref(h)))
        return cls(h, dims, dtype, ctx)

    @property
    def nnz(self) -> int:
        n = C.c_int64()
        _check(L.lib().mach_sparse_nnz(self.h, C.byref(n)))
        return n.value

    def size(self) -> int:
        return int(np.prod(self.dims))

    def entries(self):
        n = self.nnz
        idx = np.empty(n, dtype=np.int64)
        vals = np.empty(n, dtype=np.float64)
        _check(L.lib().mach_sparse_download(self.h, idx.ctypes.data_as(L.i64p), vals.ctypes.data_as(L.dp)))
        return idx, vals

    def norm(self) -> float:
        out = C.c_double()
        _check(L.lib().mach_sparse_norm(self.h, C.byref(out)))
        return out.value

    def device_view(self):
        """(idx device pointer, value device pointer, index bytes 4|8)."""
        ip_, vp_, ib = C.c_void_p(), C.c_void_p(), C.c_int()
        _check(L.lib().mach_sparse_device_view(self.h, C.byref(ip_), C.byref(vp_), C.byref(ib)))
        return ip_.value, vp_.value, ib.value

    @classmethod
    def from_device(cls, dims, nnz, idx_ptr, val_ptr, dtype, ctx: Context | None = None):
        """Copy canonical device arrays (ascending unique flat indices)."""
        ctx = _ctx(ctx)
        h = C.c_void_p()
        _check(L.lib().mach_sparse_from_device(ctx.h, _DT[np.dtype(dtype)], len(dims), _dims_arr(dims), int(nnz),
                                               C.c_void_p(idx_ptr), C.c_void_p(val_ptr), C.byref(h)))
        return cls(h, dims, dtype, ctx)

    def densify(self) -> np.ndarray:
        idx, vals = self.entries()
        out = np.zeros(self.size(), dtype=np.float64)
        out[idx] = vals
        return out.reshape(self.dims, order="F")

    def free(self):
        if getattr(self, "h", None):
            L.lib().mach_sparse_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# configs / model (sampling.hpp:14-30, tucker.hpp:14-30)
# ---------------------------------------------------------------------------
@dataclass
class SparsifyConfig:
    p: float = 1.0
    seed: int = 0


@dataclass
class HooiConfig:
    max_iterations: int = 50
    fit_tolerance: float = 1e-4


@dataclass
class TuckerModel:
    core: np.ndarray
    factors: list
    ranks: tuple
    iterations: int
    fit: float
    sweep_fits: list
    warnings: list = field(default_factory=list)
    times: dict = field(default_factory=dict)


def _model_from(h) -> TuckerModel:
    lib = L.lib()
    order, iters, nfits, nwarn = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    fit = C.c_double()
    try:
        _check(lib.mach_model_info(h, C.byref(order), C.byref(iters), C.byref(fit), C.byref(nfits), C.byref(nwarn)))
        d = order.value
        dims = (C.c_int * d)()
        ranks = (C.c_int * d)()
        _check(lib.mach_model_dims(h, dims, ranks))
        dims, ranks = tuple(dims), tuple(ranks)
        core = np.empty(int(np.prod(ranks)))
        _check(lib.mach_model_core(h, core.ctypes.data_as(L.dp)))
        factors = []
        for m in range(d):
            f = np.empty(dims[m] * ranks[m])
            _check(lib.mach_model_factor(h, m, f.ctypes.data_as(L.dp)))
            factors.append(f.reshape((dims[m], ranks[m]), order="F"))
        sf = np.empty(nfits.value)
        _check(lib.mach_model_sweep_fits(h, sf.ctypes.data_as(L.dp)))
        warns = []
        for i in range(nwarn.value):
            buf = C.create_string_buffer(512)
            _check(lib.mach_model_warning(h, i, buf, 512))
            warns.append(buf.value.decode())
        sample, setup, hosvd_ms = C.c_double(), C.c_double(), C.c_double()
        sw = (C.c_double * max(1, iters.value))()
        _check(lib.mach_model_times(h, C.byref(sample), C.byref(setup), C.byref(hosvd_ms), sw, iters.value))
        times = {"sample_ms": sample.value, "setup_ms": setup.value, "hosvd_ms": hosvd_ms.value,
                 "sweep_ms": list(sw)[: iters.value]}
        return TuckerModel(core.reshape(ranks, order="F"), factors, ranks, iters.value, fit.value, list(sf), warns,
                           times)
    finally:
        lib.mach_model_free(h)


# ---------------------------------------------------------------------------
# entry points
# ---------------------------------------------------------------------------
def _dense(t, ctx):
    if isinstance(t, DenseTensor):
        return t
    return DenseTensor.from_numpy(np.asarray(t), ctx)


def sparsify(t, cfg: SparsifyConfig | float = None, seed: int = 0, ctx: Context | None = None) -> SparseTensor:
    """sampling.hpp:22 — keep x_i != 0 with probability p, rescaled by 1/p."""
    if not isinstance(cfg, SparsifyConfig):
        cfg = SparsifyConfig(1.0 if cfg is None else float(cfg), int(seed))
    d = _dense(t, ctx)
    h = C.c_void_p()
    _check(L.lib().mach_sparsify(d.ctx.h, d.h, float(cfg.p), int(cfg.seed) & (2**64 - 1), C.byref(h)))
    return SparseTensor(h, d.dims, d.dtype, d.ctx)



def sparsify_slab(slab, global_dims, offset: int, cfg: "SparsifyConfig", ctx: Context | None = None) -> "SparseTensor":
    """Sample the flat range [offset, offset + slab.size) of a tensor of dims
    global_dims (a time slab): global RNG counter and global indices, so the
    kept set equals the full tensor's restricted to the slab."""
    d = _dense(slab, ctx)
    h = C.c_void_p()
    _check(L.lib().mach_sparsify_slab(d.ctx.h, d.h, len(global_dims), _dims_arr(global_dims), int(offset),
                                      float(cfg.p), int(cfg.seed) & 0xFFFFFFFFFFFFFFFF, C.byref(h)))
    return SparseTensor(h, global_dims, d.dtype, d.ctx)

def _ranks(ranks, d):
    if len(ranks) != d:
        raise ArgumentError("ranks must name one rank per mode")
    return (C.c_int * d)(*[int(r) for r in ranks])


def hosvd(t, ranks, ctx: Context | None = None) -> TuckerModel:
    """tucker.hpp:34,39 — HOSVD of a dense or sparse tensor."""
    h = C.c_void_p()
    if isinstance(t, SparseTensor):
        _check(L.lib().mach_hosvd_sparse(t.ctx.h, t.h, _ranks(ranks, len(t.dims)), C.byref(h)))
    else:
        d = _dense(t, ctx)
        _check(L.lib().mach_hosvd_dense(d.ctx.h, d.h, _ranks(ranks, len(d.dims)), C.byref(h)))
    return _model_from(h)


def hooi(t, ranks, cfg: HooiConfig | None = None, ctx: Context | None = None, max_iterations=None,
         fit_tolerance=None) -> TuckerModel:
    """tucker.hpp:43-44 — HOSVD init then alternating sweeps."""
    cfg = cfg or HooiConfig()
    mi = cfg.max_iterations if max_iterations is None else max_iterations
    tol = cfg.fit_tolerance if fit_tolerance is None else fit_tolerance
    h = C.c_void_p()
    if isinstance(t, SparseTensor):
        _check(L.lib().mach_hooi_sparse(t.ctx.h, t.h, _ranks(ranks, len(t.dims)), int(mi), float(tol), C.byref(h)))
    else:
        d = _dense(t, ctx)
        _check(L.lib().mach_hooi_dense(d.ctx.h, d.h, _ranks(ranks, len(d.dims)), int(mi), float(tol), C.byref(h)))
    return _model_from(h)


@dataclass
class MachResult:
    model: TuckerModel
    sparsified: SparseTensor


def mach_hooi(t, ranks, scfg: SparsifyConfig, hcfg: HooiConfig | None = None, ctx: Context | None = None) -> MachResult:
    """sampling.hpp:35-36 — sparsify then hooi; returns both."""
    hcfg = hcfg or HooiConfig()
    d = _dense(t, ctx)
    hm, hs = C.c_void_p(), C.c_void_p()
    _check(L.lib().mach_mach_hooi(d.ctx.h, d.h, _ranks(ranks, len(d.dims)), float(scfg.p), int(scfg.seed),
                                  int(hcfg.max_iterations), float(hcfg.fit_tolerance), C.byref(hm), C.byref(hs)))
    return MachResult(_model_from(hm), SparseTensor(hs, d.dims, d.dtype, d.ctx))


def mach_hosvd(t, ranks, scfg: SparsifyConfig, ctx: Context | None = None) -> MachResult:
    """sampling.hpp:32-33."""
    d = _dense(t, ctx)
    hm, hs = C.c_void_p(), C.c_void_p()
    _check(L.lib().mach_mach_hosvd(d.ctx.h, d.h, _ranks(ranks, len(d.dims)), float(scfg.p), int(scfg.seed),
                                   C.byref(hm), C.byref(hs)))
    return MachResult(_model_from(hm), SparseTensor(hs, d.dims, d.dtype, d.ctx))


def reconstruct(model: TuckerModel, ctx: Context | None = None) -> np.ndarray:
    """tucker.hpp:50 — core x_1 U_1 ... x_d U_d (device mode products)."""
    y = DenseTensor.from_numpy(np.asarray(model.core, dtype=np.float64), ctx)
    for m, f in enumerate(model.factors):
        y = mode_product(y, f, m, ctx=ctx, keep_on_device=True)
    return y.numpy()


def accuracy(t, model: TuckerModel, ctx: Context | None = None) -> float:
    """tucker.hpp:55 — 1 - |t - reconstruct(model)| / |t|, one fused device
    pass over t (the reconstruction is never materialised)."""
    d = _dense(t, ctx)
    if len(model.factors) != len(d.dims) or any(f.shape[0] != n for f, n in zip(model.factors, d.dims)):
        raise ShapeError("model reconstructs to a different shape")
    core = np.ascontiguousarray(np.asarray(model.core, dtype=np.float64).reshape(-1, order="F"))
    fs = [np.ascontiguousarray(np.asarray(f, dtype=np.float64).reshape(-1, order="F")) for f in model.factors]
    fp = (L.dp * len(fs))(*[f.ctypes.data_as(L.dp) for f in fs])
    out = C.c_double()
    _check(L.lib().mach_model_accuracy(d.ctx.h, d.h, _ranks(model.ranks, len(d.dims)), core.ctypes.data_as(L.dp), fp,
                                       C.byref(out)))
    return out.value


def subspace_sin(a: np.ndarray, b: np.ndarray, r: int | None = None, ctx: Context | None = None) -> float:
    """metrics.cpp:59-66 — largest principal-angle sine between the spans of
    the leading r columns of a and b (on the device)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    r = min(a.shape[1], b.shape[1]) if r is None else int(r)
    if a.shape[0] != b.shape[0]:
        raise ShapeError("subspace_sin needs matrices with the same rows")
    fa = np.ascontiguousarray(a[:, :r].reshape(-1, order="F"))
    fb = np.ascontiguousarray(b[:, :r].reshape(-1, order="F"))
    out = C.c_double()
    _check(L.lib().mach_subspace_sin(_ctx(ctx).h, a.shape[0], r, fa.ctypes.data_as(L.dp), fb.ctypes.data_as(L.dp),
                                     C.byref(out)))
    return out.value


def _pairwise(v: np.ndarray) -> float:
    """internal.hpp:36-46 cascade (base 64) — the reference's summation order."""
    n = v.size
    if n <= 64:
        s = 0.0
        for x in v.tolist():
            s += x
        return s
    mid = n // 2
    return _pairwise(v[:mid]) + _pairwise(v[mid:])


def pearson(x, y) -> float:
    """metrics.cpp:67-96 (same summation order and errors)."""
    x = np.asarray(x, dtype=np.float64).ravel()
    y = np.asarray(y, dtype=np.float64).ravel()
    if x.size != y.size:
        raise ShapeError(f"correlation inputs have lengths {x.size} and {y.size}")
    n = x.size
    if n < 2:
        raise ArgumentError("correlation needs at least 2 samples")
    if np.all(x == x[0]) or np.all(y == y[0]):
        raise ArgumentError("correlation is undefined for a zero-variance input")
    mx = _pairwise(x) / n
    my = _pairwise(y) / n
    dx, dy = x - mx, y - my
    sxx, syy, sxy = _pairwise(dx * dx), _pairwise(dy * dy), _pairwise(dx * dy)
    if sxx == 0.0 or syy == 0.0:
        raise ArgumentError("correlation is undefined for a zero-variance input")
    return sxy / float(np.sqrt(sxx * syy))


def pc_correlation(exact: TuckerModel, approx: TuckerModel, mode: int, component: int = 1):
    """metrics.cpp:98-122 — (rho, flipped)."""
    if len(exact.factors) != len(approx.factors):
        raise ShapeError("models have different orders")
    if not 0 <= mode < len(exact.factors):
        raise ArgumentError(f"mode {mode + 1} out of range for order {len(exact.factors)}")
    limit = min(exact.ranks[mode], approx.ranks[mode])
    if not 1 <= component <= limit:
        raise ArgumentError(f"component {component} out of range; mode {mode + 1} has at most {limit} shared components")
    a = np.asarray(exact.factors[mode][:, component - 1], dtype=np.float64)
    b = np.asarray(approx.factors[mode][:, component - 1], dtype=np.float64)
    if a.size != b.size:
        raise ShapeError("factor columns of different lengths")
    flip = _pairwise(a * b) < 0.0
    return pearson(a, -b if flip else b), bool(flip)


def compare(exact: TuckerModel, approx: TuckerModel, reference, ctx: Context | None = None) -> dict:
    """metrics.cpp:124-159 (ComparisonReport): component-1 correlations per
    mode, tie detection from the core slice norms with the subspace sine,
    both accuracies (fused device passes), the leading core entries."""
    ref = _dense(reference, ctx)
    d = len(ref.dims)
    if len(exact.factors) != d or len(approx.factors) != d:
        raise ShapeError("reference and models have different orders")
    rep = {"per_mode_rho": [], "flipped": [], "tied": [], "tie_subspace_sin": []}

    def slice_norms(core, m):
        return np.sqrt((np.moveaxis(np.asarray(core), m, 0).reshape(core.shape[m], -1) ** 2).sum(axis=1))

    def tied(n):
        n = np.sort(n)[::-1]
        return n.size >= 2 and n[0] - n[1] <= 1e-6 * n[0]

    for m in range(d):
        rho, fl = pc_correlation(exact, approx, m, 1)
        rep["per_mode_rho"].append(rho)
        rep["flipped"].append(fl)
        t = tied(slice_norms(exact.core, m)) or tied(slice_norms(approx.core, m))
        rep["tied"].append(bool(t))
        r = min(exact.ranks[m], approx.ranks[m])
        rep["tie_subspace_sin"].append(subspace_sin(exact.factors[m], approx.factors[m], r, ctx) if t else 0.0)
    rep["accuracy_exact"] = accuracy(ref, exact)
    rep["accuracy_mach"] = accuracy(ref, approx)
    rep["core_interaction"] = (float(np.asarray(exact.core).reshape(-1, order="F")[0]),
                               float(np.asarray(approx.core).reshape(-1, order="F")[0]))
    return rep


def mode_product(t, m: np.ndarray, mode: int, ctx: Context | None = None, keep_on_device=False):
    """tensor.hpp:129,132 — t x_mode m (m is J x I_mode)."""
    mf = np.asfortranarray(np.asarray(m, dtype=np.float64))
    flat = np.ascontiguousarray(mf.reshape(-1, order="F"))
    h = C.c_void_p()
    if isinstance(t, SparseTensor):
        dims, c = t.dims, t.ctx
        _check(L.lib().mach_mode_product_sparse(c.h, t.h, mf.shape[0], mf.shape[1], flat.ctypes.data_as(L.dp), int(mode),
                                                C.byref(h)))
    else:
        d = _dense(t, ctx)
        dims, c = d.dims, d.ctx
        _check(L.lib().mach_mode_product_dense(c.h, d.h, mf.shape[0], mf.shape[1], flat.ctypes.data_as(L.dp), int(mode),
                                               C.byref(h)))
    od = list(dims)
    od[mode] = mf.shape[0]
    out = DenseTensor(h, od, np.float64, c)
    return out if keep_on_device else out.numpy()


def sparse_row_gram(t: "SparseTensor", mode: int) -> np.ndarray:
    """Row Gram X_(mode) X_(mode)^T of a sampled tensor (I x I, fp64)."""
    n = int(t.dims[mode])
    out = np.empty(n * n, dtype=np.float64)
    _check(L.lib().mach_sparse_row_gram(t.ctx.h, t.h, int(mode), out.ctypes.data_as(L.dp)))
    return out.reshape((n, n), order="F")


def mode_gram(t, mode: int, ctx: Context | None = None):
    """X_(mode) X_(mode)^T of a dense tensor (the dense HOSVD's row-side Gram,
    linalg.cpp:340).  Returns (G, tensor_cores): fp32 tensors of supported
    shape go through the tcgen05 TF32 kernel (tensor_cores True)."""
    d = _dense(t, ctx)
    R = d.dims[mode]
    g = np.empty(R * R, dtype=np.float64)
    tc = C.c_int(0)
    _check(L.lib().mach_dense_mode_gram(d.ctx.h, d.h, int(mode), g.ctypes.data_as(L.dp), C.byref(tc)))
    return g.reshape((R, R), order="F"), bool(tc.value)


@dataclass
class TruncatedSvd:
    left: np.ndarray
    singular_values: np.ndarray
    right: np.ndarray


def truncated_svd(m: np.ndarray, k: int, ctx: Context | None = None) -> TruncatedSvd:
    """linalg.hpp:23 — top-k singular triplets (reference sign rule), on the device."""
    m = np.asarray(m, dtype=np.float64)
    rows, cols = m.shape
    c = _ctx(ctx)
    kk = max(int(k), 1)
    left, sv, right = np.empty(rows * kk), np.empty(kk), np.empty(cols * kk)
    flat = np.ascontiguousarray(m.reshape(-1, order="F"))
    _check(L.lib().mach_truncated_svd(c.h, rows, cols, flat.ctypes.data_as(L.dp), int(k), left.ctypes.data_as(L.dp),
                                      sv.ctypes.data_as(L.dp), right.ctypes.data_as(L.dp)))
    return TruncatedSvd(left.reshape((rows, kk), order="F"), sv, right.reshape((cols, kk), order="F"))


def leading_left_singular_vectors(m: np.ndarray, k: int, ctx: Context | None = None) -> np.ndarray:
    """linalg.hpp:26 — the left factor of truncated_svd."""
    return truncated_svd(m, k, ctx).left


def low_rank_approx(m: np.ndarray, k: int, ctx: Context | None = None) -> np.ndarray:
    """linalg.hpp:29 — left diag(sv) right^T of truncated_svd, on the device."""
    m = np.asarray(m, dtype=np.float64)
    rows, cols = m.shape
    c = _ctx(ctx)
    out = np.empty(rows * cols)
    flat = np.ascontiguousarray(m.reshape(-1, order="F"))
    _check(L.lib().mach_low_rank_approx(c.h, rows, cols, flat.ctypes.data_as(L.dp), int(k), out.ctypes.data_as(L.dp)))
    return out.reshape((rows, cols), order="F")


@dataclass
class LeftSingularBasis:
    basis: np.ndarray
    singular_values: np.ndarray
    numerical_rank: int
    completed: bool


def left_singular_basis(m: np.ndarray, k: int, ctx: Context | None = None) -> LeftSingularBasis:
    """linalg.hpp:42 — on-device eigen step for a host matrix."""
    ctx = _ctx(ctx)
    m = np.asarray(m, dtype=np.float64)
    if m.ndim != 2 or m.shape[0] < 1 or m.shape[1] < 1:
        raise ArgumentError("matrix must be nonempty")
    rows, cols = m.shape
    if k < 1 or k > rows:
        raise ArgumentError("k must satisfy 1 <= k <= rows")
    flat = np.ascontiguousarray(m.reshape(-1, order="F"))
    basis = np.empty(rows * k)
    sv = np.empty(k)
    nr, comp = C.c_int(), C.c_int()
    _check(L.lib().mach_left_singular_basis(ctx.h, rows, cols, flat.ctypes.data_as(L.dp), int(k),
                                            basis.ctypes.data_as(L.dp), sv.ctypes.data_as(L.dp), C.byref(nr),
                                            C.byref(comp)))
    return LeftSingularBasis(basis.reshape((rows, k), order="F"), sv, nr.value, bool(comp.value))


# ---------------------------------------------------------------------------
# incremental HOOI (hooi_loop split into begin / step), for streaming use and
# for timing sweeps one by one
# ---------------------------------------------------------------------------
class HooiSession:
    """Setup + HOSVD on construction; ``step(n)`` runs sweeps with the
    reference stop rule (tucker.cpp:102)."""

    def __init__(self, t, ranks, ctx: Context | None = None):
        h = C.c_void_p()
        if isinstance(t, SparseTensor):
            self.ctx = t.ctx
            _check(L.lib().mach_hooi_begin(t.ctx.h, t.h, _ranks(ranks, len(t.dims)), C.byref(h)))
        else:
            d = _dense(t, ctx)
            self.ctx = d.ctx
            _check(L.lib().mach_hooi_begin_dense(d.ctx.h, d.h, _ranks(ranks, len(d.dims)), C.byref(h)))
        self.h = h
        self._src = t

    def step(self, n: int = 1, fit_tolerance: float = 0.0):
        done, stopped = C.c_int(), C.c_int()
        _check(L.lib().mach_hooi_step(self.h, int(n), float(fit_tolerance), C.byref(done), C.byref(stopped)))
        return done.value, bool(stopped.value)

    @property
    def fit(self) -> float:
        f, it = C.c_double(), C.c_int()
        _check(L.lib().mach_hooi_state(self.h, C.byref(f), C.byref(it)))
        return f.value

    def model(self) -> TuckerModel:
        hm = C.c_void_p()
        _check(L.lib().mach_hooi_model(self.h, C.byref(hm)))
        return _model_from(hm)

    @classmethod
    def from_session(cls, t: "SparseTensor", ranks, init: "HooiSession"):
        """Session on `t` starting from `init`'s current factors (no HOSVD)."""
        hm = C.c_void_p()
        _check(L.lib().mach_hooi_model(init.h, C.byref(hm)))
        try:
            h = C.c_void_p()
            _check(L.lib().mach_hooi_begin_from(t.ctx.h, t.h, _ranks(ranks, len(t.dims)), hm, C.byref(h)))
        finally:
            L.lib().mach_model_free(hm)
        self = cls.__new__(cls)
        self.h, self.ctx, self._src = h, t.ctx, t
        return self

    @classmethod
    def from_grams(cls, t: "SparseTensor", ranks, grams):
        """Shard session on `t` whose HOSVD factors come from the full row Grams
        `grams` (one I_n x I_n array per mode; partial Grams summed
        over the shards).  Call refresh_fit() once mode_y(last) is reduced."""
        d = len(t.dims)
        gs = [np.ascontiguousarray(np.asarray(g, dtype=np.float64).reshape(-1, order="F")) for g in grams]
        ptrs = (L.dp * d)(*[g.ctypes.data_as(L.dp) for g in gs])
        hm = C.c_void_p()
        _check(L.lib().mach_hosvd_from_grams(t.ctx.h, d, _dims_arr(t.dims), _ranks(ranks, d), ptrs, C.byref(hm)))
        try:
            h = C.c_void_p()
            _check(L.lib().mach_hooi_begin_from(t.ctx.h, t.h, _ranks(ranks, d), hm, C.byref(h)))
        finally:
            L.lib().mach_model_free(hm)
        self = cls.__new__(cls)
        self.h, self.ctx, self._src = h, t.ctx, t
        return self

    def refresh_fit(self):
        """Starting fit (sweep_fits[0]) from the last mode's (reduced) Y."""
        _check(L.lib().mach_hooi_refresh_fit(self.h))

    def shard(self):
        """Make this session one time-slab shard over its context's NCCL
        communicator: |X|^2 summed over the shards, and every step()
        all-reduces each mode's partial Y_(n) inside the library."""
        _check(L.lib().mach_hooi_shard(self.h))

    def set_norm2(self, norm2: float):
        _check(L.lib().mach_hooi_set_norm2(self.h, float(norm2)))

    def mode_y(self, mode: int):
        """TTM of the local nonzeros: (device pointer, rows, cols) of Y_(mode)."""
        y, r, c = C.c_void_p(), C.c_int(), C.c_int()
        _check(L.lib().mach_hooi_mode_y(self.h, int(mode), C.byref(y), C.byref(r), C.byref(c)))
        return y.value, r.value, c.value

    def mode_update(self, mode: int):
        _check(L.lib().mach_hooi_mode_update(self.h, int(mode)))

    def sweep_end(self, fit_tolerance: float = 0.0) -> bool:
        st = C.c_int()
        _check(L.lib().mach_hooi_sweep_end(self.h, float(fit_tolerance), C.byref(st)))
        return bool(st.value)

    def ttm_bytes(self, mode: int) -> int:
        """Algorithmic bytes of one mode-`mode` TTM launch (-1 on the dense route)."""
        b = C.c_longlong()
        _check(L.lib().mach_hooi_ttm_bytes(self.h, int(mode), C.byref(b)))
        return int(b.value)

    def free(self):
        if getattr(self, "h", None):
            L.lib().mach_session_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def profile(ctx: Context, enable: bool = True):
    _check(L.lib().mach_ctx_profile(ctx.h, 1 if enable else 0))


def kernel_stats(ctx: Context) -> dict:
    """{kernel name: (launches, total device ms)} since profile(ctx, True)."""
    out = {}
    i = 0
    while True:
        buf = C.create_string_buffer(256)
        n, ms = C.c_int64(), C.c_double()
        rc = L.lib().mach_ctx_kernel_stat(ctx.h, i, buf, 256, C.byref(n), C.byref(ms))
        if rc != L.MACH_OK:
            break
        out[buf.value.decode()] = (n.value, ms.value)
        i += 1
    return out


# ---------------------------------------------------------------------------
# Theorem-1 bound (bounds.hpp:10-66), SURVEY 8f.3
# ---------------------------------------------------------------------------
def _bound_dict(rep, modes=None) -> dict:
    out = {k: getattr(rep, k) for k in ("b", "p", "p_min", "t", "success_probability")}
    for k in ("dims_large_enough", "dims_balanced", "p_above_min", "conditions_met"):
        out[k] = bool(getattr(rep, k))
    out["per_mode"] = [] if modes is None else [
        {k: getattr(m, k) for k in ("rank", "x_residual", "xhat_residual", "x_lowrank_norm", "t_i")} for m in modes]
    return out


def achlioptas_bounds(b: float, n: int, k: int, p: float):
    """(two_norm, frobenius) — bounds.hpp:17."""
    a, f = C.c_double(), C.c_double()
    _check(L.lib().mach_achlioptas_bounds(float(b), int(n), int(k), float(p), C.byref(a), C.byref(f)))
    return a.value, f.value


def min_sampling_probability(dims) -> float:
    out = C.c_double()
    _check(L.lib().mach_min_sampling_probability(len(dims), _dims_arr(dims) if len(dims) else None, C.byref(out)))
    return out.value


def theorem1_conditions(dims, p: float) -> dict:
    rep = L.BoundReport()
    _check(L.lib().mach_theorem1_conditions(len(dims), _dims_arr(dims) if len(dims) else None, float(p), C.byref(rep)))
    return _bound_dict(rep)


def theorem1_bound(x: "DenseTensor", xhat: "SparseTensor", ranks, p: float, ctx: Context | None = None) -> dict:
    """BoundReport as a dict; the mode spectra are computed on the device (bounds.hpp:62)."""
    ctx = _ctx(ctx or x.ctx)
    d = len(x.dims)
    if len(ranks) != d:
        raise ArgumentError("ranks must name one rank per mode")
    rep = L.BoundReport()
    modes = (L.BoundMode * d)()
    _check(L.lib().mach_theorem1_bound(ctx.h, x.h, xhat.h, (C.c_int * d)(*[int(r) for r in ranks]), float(p),
                                       C.byref(rep), modes))
    return _bound_dict(rep, modes)


# ---------------------------------------------------------------------------
# streaming sample-on-arrival ingest
# ---------------------------------------------------------------------------
class SampleStream:
    """A tensor growing along its last (time) mode, sampled slab by slab on the device.

    dims: the leading dims and, last, the capacity in time ticks.  At any time
    `tensor()` equals sparsify() of everything appended so far, bit for bit."""

    def __init__(self, dims, cfg: "SparsifyConfig", dtype=np.float32, ctx: Context | None = None):
        self.ctx = _ctx(ctx)
        self.dims, self.dtype = tuple(int(d) for d in dims), np.dtype(dtype)
        self.h = C.c_void_p()
        _check(L.lib().mach_stream_begin(self.ctx.h, _DT[self.dtype], len(self.dims), _dims_arr(self.dims), float(cfg.p),
                                         int(cfg.seed), C.byref(self.h)))

    def append(self, slab):
        """slab: a DenseTensor in HBM, or a numpy array (leading dims x ticks) copied from the host."""
        if isinstance(slab, DenseTensor):
            _check(L.lib().mach_stream_append(self.h, slab.h))
            return
        a = np.asarray(slab)
        if a.shape[:-1] != self.dims[:-1]:
            raise ShapeError("slab leading dims differ from the stream's")
        flat = np.ascontiguousarray(a.astype(self.dtype, copy=False).reshape(-1, order="F"))
        _check(L.lib().mach_stream_append_host(self.h, flat.ctypes.data_as(C.c_void_p), int(a.shape[-1])))
        self._last_ticks = int(a.shape[-1])

    def append_host_ptr(self, ptr: int, ticks: int):
        """Host slab by address (e.g. a pinned torch tensor's data_ptr())."""
        _check(L.lib().mach_stream_append_host(self.h, C.c_void_p(ptr), int(ticks)))
        self._last_ticks = int(ticks)

    def append_records(self, machine, metric, tick, value, ticks: int, carry_forward: bool = False):
        """One time slab of pre-indexed measurement records (ingest.cpp:90-134 on the device)."""
        m = np.ascontiguousarray(machine, dtype=np.int32)
        j = np.ascontiguousarray(metric, dtype=np.int32)
        t = np.ascontiguousarray(tick, dtype=np.int32)
        v = np.ascontiguousarray(value, dtype=np.float64)
        i32p = C.POINTER(C.c_int32)
        _check(L.lib().mach_stream_append_records(self.h, len(v), m.ctypes.data_as(i32p), j.ctypes.data_as(i32p),
                                                  t.ctypes.data_as(i32p), v.ctypes.data_as(L.dp), int(ticks),
                                                  1 if carry_forward else 0))
        self._last_ticks = int(ticks)

    def state(self):
        t, z = C.c_int64(), C.c_int64()
        _check(L.lib().mach_stream_state(self.h, C.byref(t), C.byref(z)))
        return t.value, z.value

    def tensor(self) -> "SparseTensor":
        h = C.c_void_p()
        _check(L.lib().mach_stream_tensor(self.h, C.byref(h)))
        ticks, _ = self.state()
        return SparseTensor(h, self.dims[:-1] + (ticks,), self.dtype, self.ctx)

    def last_slab(self) -> "DenseTensor":
        h = C.c_void_p()
        _check(L.lib().mach_stream_last_slab(self.h, C.byref(h)))
        return DenseTensor(h, self.dims[:-1] + (self._last_ticks,), self.dtype, self.ctx)

    def free(self):
        if getattr(self, "h", None):
            L.lib().mach_stream_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# binary tensor files
# ---------------------------------------------------------------------------
def tensor_file_info(path: str) -> dict:
    kind, dt, order, nnz = C.c_int(), C.c_int(), C.c_int(), C.c_int64()
    dims = (C.c_int * 8)()
    _check(L.lib().mach_tensor_file_kind(str(path).encode(), C.byref(kind), C.byref(dt), C.byref(order), dims, C.byref(nnz)))
    return {"kind": "sparse" if kind.value else "dense", "dtype": np.dtype(np.float64 if dt.value else np.float32),
            "dims": tuple(dims[i] for i in range(order.value)), "count": nnz.value}


def save_tensor(t, path: str):
    fn = L.lib().mach_sparse_save if isinstance(t, SparseTensor) else L.lib().mach_dense_save
    _check(fn(t.h, str(path).encode()))


def load_tensor(path: str, ctx: Context | None = None):
    """DenseTensor or SparseTensor in HBM from a MACHB2 binary file."""
    ctx = _ctx(ctx)
    info = tensor_file_info(path)
    h = C.c_void_p()
    if info["kind"] == "sparse":
        _check(L.lib().mach_sparse_load(ctx.h, str(path).encode(), C.byref(h)))
        return SparseTensor(h, info["dims"], info["dtype"], ctx)
    _check(L.lib().mach_dense_load(ctx.h, str(path).encode(), C.byref(h)))
    return DenseTensor(h, info["dims"], info["dtype"], ctx)
