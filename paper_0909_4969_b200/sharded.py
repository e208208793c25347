"""Time-slab sharded MACH-HOOI across the GPUs of one box.

Partition: rank g owns the time slab t in [t_g, t_{g+1}) of the LAST mode.
Under first-mode-fastest layout a slab is the contiguous flat range
[t_g S, t_{g+1} S), S = prod(dims[:-1]); the sampler's RNG counter is the
global flat index (sampling.cpp:27), so per-rank sampling
(`sparsify_slab`) reproduces the single-GPU kept set bit for bit.

Every rank keeps its nonzeros in a tensor of the GLOBAL dims.  Mode-n TTM of
the local nonzeros gives a partial Y_(n) whose rank-sum is the full Y_(n) for
every mode (for the time mode the row blocks are disjoint), so one sweep is,
per mode, TTM -> all-reduce(sum) of Y_(n) (<= 0.5 MB at the configs) ->
replicated factor update (identical inputs on every rank give identical
factors, so no broadcast), and the core/fit come from the last mode's summed
Y.  |X|^2 is all-reduced once.  HOSVD runs once on the all-gathered sampled
tensor (replicated: the time mode's row Gram has cross-slab blocks, SURVEY
§8e).  With an NCCL group the per-mode all-reduce runs inside the library
(mach_ctx_comm_init + mach_hooi_shard: on the library stream, inside the
sweep's CUDA graph, overlapped stage 1 kept); `sharded_sweeps` is the same
exchange driven from the host, used with `gloo` (CPU tests, and a 2-process
test of the real CUDA engine).
"""
from __future__ import annotations

import math
import os

import numpy as np


def slab_bounds(extent: int, world: int, rank: int):
    """Balanced [t0, t1) of the last mode for `rank` of `world`."""
    q, r = divmod(extent, world)
    t0 = rank * q + min(rank, r)
    return t0, t0 + q + (1 if rank < r else 0)


def sharded_sweeps(engine, allreduce_sum_, d: int, sweeps: int, fit_tolerance: float):
    """One HOOI sweep per iteration (tucker.cpp:80-106): for every mode the
    engine's partial Y_(m) is summed over the ranks in place, then the factor
    is updated from it; the sweep ends with core, fit and the stop rule."""
    done = 0
    for _ in range(sweeps):
        for m in range(d):
            y = engine.mode_y(m)
            allreduce_sum_(y)
            engine.mode_update(m)
        done += 1
        if engine.sweep_end(fit_tolerance):
            break
    return done


class _CAI:
    """Zero-copy __cuda_array_interface__ over a device pointer."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


def device_view(ptr: int, n: int, dtype, device):
    import torch
    ts = {np.dtype(np.float32): "<f4", np.dtype(np.float64): "<f8", np.dtype(np.int32): "<i4",
          np.dtype(np.int64): "<i8"}[np.dtype(dtype)]
    return torch.as_tensor(_CAI(ptr, n, ts), device=device)


class CudaEngine:
    """Split sweep on libmach_b200 (mach_hooi_mode_y / _mode_update / _sweep_end)."""

    def __init__(self, session, dtype, device):
        self.s, self.dtype, self.device = session, np.dtype(dtype), device

    def mode_y(self, m):
        ptr, rows, cols = self.s.mode_y(m)
        return device_view(ptr, rows * cols, self.dtype, self.device)

    def mode_update(self, m):
        self.s.mode_update(m)

    def sweep_end(self, tol):
        return self.s.sweep_end(tol)


def _host_staged(group) -> bool:
    """gloo exchanges go through host tensors (its CUDA paths are not used)."""
    import torch.distributed as dist
    return dist.get_backend(group) == "gloo"


def _allgather_varlen(t, group):
    """All-gather 1-D tensors of per-rank lengths, concatenated in rank order."""
    import torch
    import torch.distributed as dist
    if _host_staged(group) and t.is_cuda:
        return _allgather_varlen(t.cpu(), group).to(t.device)
    world = dist.get_world_size(group)
    n = torch.tensor([t.numel()], device=t.device, dtype=torch.int64)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    ns = [int(v.item()) for v in ns]
    mx = max(ns) if ns else 0
    pad = torch.zeros(mx, device=t.device, dtype=t.dtype)
    pad[: t.numel()] = t
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return torch.cat([o[:k] for o, k in zip(outs, ns)])


def sharded_mach_hooi(slab_flat, global_dims, ranks, p: float, seed: int, sweeps: int, fit_tolerance: float = 0.0,
                      group=None, ctx=None, in_library=None):
    """MACH-HOOI of a tensor whose time slabs live on the ranks of `group`.

    slab_flat: this rank's slab (torch CUDA tensor, first-mode-fastest, the
    flat range slab_bounds(global_dims[-1]) * prod(global_dims[:-1])).
    Returns (TuckerModel, local SparseTensor).  Identical model on every rank.
    """
    import torch
    import torch.distributed as dist

    from . import api as A

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if in_library is None:  # the library's NCCL exchange when the group is NCCL, else the host loop
        in_library = dist.get_backend(group) == "nccl"
    dims = list(global_dims)
    S = math.prod(dims[:-1])
    t0, t1 = slab_bounds(dims[-1], world, rank)
    if slab_flat.numel() != S * (t1 - t0):
        raise A.ShapeError("slab does not match slab_bounds for this rank")
    dev = slab_flat.device
    ctx = ctx or A.Context(dev.index)
    # one explicit stream for the library, torch's collectives and copies (a
    # null handle would give the library a stream of its own)
    stream = torch.cuda.Stream(device=dev)
    stream.wait_stream(torch.cuda.current_stream(dev))
    ctx.set_stream(stream.cuda_stream)
    ctx._stream_keepalive = stream  # the context (and the returned tensors) keep using it
    with torch.cuda.stream(stream):
        out = _sharded_body(slab_flat, dims_=list(global_dims), ranks=ranks, p=p, seed=seed, sweeps=sweeps,
                            fit_tolerance=fit_tolerance, group=group, ctx=ctx, in_library=in_library, dev=dev)
    stream.synchronize()
    return out


def _sharded_body(slab_flat, dims_, ranks, p, seed, sweeps, fit_tolerance, group, ctx, in_library, dev):
    import torch
    import torch.distributed as dist

    from . import api as A

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    dims = dims_
    d = len(dims)
    S = math.prod(dims[:-1])
    t0, t1 = slab_bounds(dims[-1], world, rank)
    dtype = np.float32 if slab_flat.dtype == torch.float32 else np.float64
    slab = A.DenseTensor.from_torch(slab_flat, dims[:-1] + [t1 - t0], ctx)
    sp = A.sparsify_slab(slab, dims, t0 * S, A.SparsifyConfig(p, seed), ctx)

    # HOSVD.  Every mode but the last: the row Gram of X_(n) is a
    # sum over its columns, which the time slabs partition, so each rank forms
    # the Gram of its own nonzeros and the Grams are all-reduced.  The last
    # mode's Gram has cross-slab blocks: it is formed once from the gathered
    # nonzeros.  The eigen step runs replicated on identical Grams.  (Modes
    # whose unfolding is taller than wide take the replicated route below.)
    numel = math.prod(dims)
    partial = all(dims[m] <= numel // dims[m] for m in range(d)) and os.environ.get("MACH_SHARD_REPLICATED_HOSVD") is None
    ip, vp, ib = sp.device_view()
    nnz = sp.nnz
    idx = device_view(ip, nnz, np.int32 if ib == 4 else np.int64, dev) if nnz else torch.zeros(0, dtype=torch.int32, device=dev)
    val = device_view(vp, nnz, dtype, dev) if nnz else torch.zeros(0, dtype=slab_flat.dtype, device=dev)
    gidx = _allgather_varlen(idx, group)
    gval = _allgather_varlen(val, group)
    full = A.SparseTensor.from_device(dims, gidx.numel(), gidx.data_ptr(), gval.data_ptr(), dtype, ctx)
    if partial:
        grams = []
        for m in range(d - 1):
            g = torch.from_numpy(np.ascontiguousarray(A.sparse_row_gram(sp, m)))
            if _host_staged(group):
                dist.all_reduce(g, group=group)
            else:
                gd = g.to(dev)
                dist.all_reduce(gd, group=group)
                g = gd.cpu()
            grams.append(g.numpy())
        grams.append(A.sparse_row_gram(full, d - 1))
        full.free()
        sess = A.HooiSession.from_grams(sp, ranks, grams)
    else:  # replicated on the gathered tensor
        hs = A.HooiSession(full, ranks)
        sess = A.HooiSession.from_session(sp, ranks, hs)
        hs.free()
        full.free()

    def start_fit(allreduce):
        """sweep_fits[0] of the shard session: the last mode's partial Y summed over the ranks."""
        if not partial:
            return
        ptr, rows, cols = sess.mode_y(d - 1)
        allreduce(device_view(ptr, rows * cols, dtype, dev))
        sess.refresh_fit()

    if in_library:
        # NCCL inside the library: the exchange rides the library stream and
        # the sweep graph (overlapped stage 1 kept)
        bind_comm(ctx, group)
        sess.shard()
        start_fit(lambda y: dist.all_reduce(y, group=group))
        sess.step(sweeps, fit_tolerance)
    else:
        host = _host_staged(group)
        n2 = (val.double() ** 2).sum().reshape(1)
        n2 = n2.cpu() if host else n2
        dist.all_reduce(n2, group=group)
        sess.set_norm2(float(n2.item()))

        def allreduce_sum_(y):
            if host:
                torch.cuda.current_stream(dev).synchronize()  # the library's Y_(m) is written
                yh = y.cpu()
                dist.all_reduce(yh, group=group)
                y.copy_(yh)
            else:
                dist.all_reduce(y, group=group)

        start_fit(allreduce_sum_)
        sharded_sweeps(CudaEngine(sess, dtype, dev), allreduce_sum_, d, sweeps, fit_tolerance)
    model = sess.model()
    sess.free()
    return model, sp


def bind_comm(ctx, group=None):
    """Give `ctx` an NCCL communicator over the ranks of `group` (the unique
    id travels by torch.distributed, whatever its backend)."""
    import torch.distributed as dist

    from . import api as A

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    obj = [A.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    ctx.comm_init(world, rank, obj[0])
