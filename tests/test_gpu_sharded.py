"""Time-slab sharded path on the B200 (world size 1 over NCCL: the GPU box
has one GPU; the 2-rank exchange logic is covered on CPU in test_sharded.py).

Checks the device pieces the sharded sweep is built from: slab sampling
reproduces the full kept set bit for bit, the gathered tensor and the split
sweep (mode_y -> all-reduce -> mode_update -> sweep_end) reproduce the
single-GPU session.
"""
import os
import socket

import numpy as np
import pytest

import oracle as O
from tests.helpers import align_core, rel, subspace_sin

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_slab_sampling_bitexact():
    import paper_0909_4969_b200 as mb
    dims = (20, 16, 30)
    x = O.random_tensor(list(dims), 5)
    full = mb.sparsify(x, mb.SparsifyConfig(0.2, 11))
    fi, fv = full.entries()
    S = 20 * 16
    got_i, got_v = [], []
    for t0, t1 in ((0, 7), (7, 19), (19, 30)):
        slab = np.ascontiguousarray(x[..., t0:t1])
        sp = mb.sparsify_slab(slab, dims, t0 * S, mb.SparsifyConfig(0.2, 11))
        i, v = sp.entries()
        got_i.append(i)
        got_v.append(v)
    assert np.array_equal(np.concatenate(got_i), fi)
    assert np.array_equal(np.concatenate(got_v).view(np.uint64), fv.view(np.uint64))


@pytest.mark.parametrize("dtype,in_library,dims,ranks", [
    ("float64", False, (40, 30, 36), (4, 3, 5)), ("float32", False, (40, 30, 36), (4, 3, 5)),
    ("float64", True, (40, 30, 36), (4, 3, 5)), ("float32", True, (40, 30, 36), (4, 3, 5)),
    ("float32", True, (12, 10, 8, 14), (3, 3, 2, 4))])
def test_sharded_world1_matches_session(dtype, in_library, dims, ranks):
    """in_library: the exchange inside the library (mach_ctx_comm_init +
    mach_hooi_shard, NCCL on the library stream, sweep graph and overlapped
    stage 1 kept); otherwise the host loop over torch.distributed."""
    import torch
    import torch.distributed as dist

    import paper_0909_4969_b200 as mb
    from paper_0909_4969_b200.sharded import sharded_mach_hooi

    p, seed, sweeps = 0.2, 7, 3
    x = O.random_tensor(list(dims), 13).astype(dtype)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        flat = torch.from_numpy(x.reshape(-1, order="F").copy()).cuda()
        model, sp = sharded_mach_hooi(flat, dims, ranks, p, seed, sweeps, 0.0, in_library=in_library)
    finally:
        dist.destroy_process_group()
    ref = mb.mach_hooi(mb.DenseTensor.from_numpy(x), ranks, mb.SparsifyConfig(p, seed),
                       mb.HooiConfig(sweeps, 0.0)).model
    tol = 1e-9 if dtype == "float64" else 1e-4
    assert model.iterations == ref.iterations
    assert np.abs(np.array(model.sweep_fits) - np.array(ref.sweep_fits)).max() <= tol
    for a, b in zip(model.factors, ref.factors):
        assert subspace_sin(a, b) <= (1e-9 if dtype == "float64" else 1e-3)
    assert rel(align_core(model.core, model.factors, ref.factors), ref.core) <= tol


def _two_rank_worker(rank, port, dims, ranks, p, seed, sweeps, q):
    """One of two processes sharing cuda:0: its slab, the real CUDA engine,
    the per-mode exchange over gloo (host staging; no kernel waits on the
    other process)."""
    import torch
    import torch.distributed as dist

    from paper_0909_4969_b200.sharded import sharded_mach_hooi, slab_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        x = O.random_tensor(list(dims), 13).astype("float32")
        S = int(np.prod(dims[:-1]))
        t0, t1 = slab_bounds(dims[-1], 2, rank)
        flat = torch.from_numpy(x.reshape(-1, order="F")[t0 * S: t1 * S].copy()).cuda()
        model, sp = sharded_mach_hooi(flat, dims, ranks, p, seed, sweeps, 0.0, in_library=False)
        q.put((rank, model.iterations, list(model.sweep_fits), [f.copy() for f in model.factors], model.core.copy(),
               sp.nnz))
    finally:
        dist.destroy_process_group()


def test_sharded_two_processes_cuda_engine_gloo():
    """World size 2 of the product engine (CudaEngine over libmach_b200) on
    one GPU: every rank ends with the single-GPU model (fp32 bars)."""
    import torch.multiprocessing as tmp

    import paper_0909_4969_b200 as mb

    dims, ranks, p, seed, sweeps = (40, 30, 36), (4, 3, 5), 0.2, 7, 3
    ctxm = tmp.get_context("spawn")
    q = ctxm.Queue()
    port = _port()
    procs = [ctxm.Process(target=_two_rank_worker, args=(r, port, dims, ranks, p, seed, sweeps, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    outs = [q.get(timeout=600) for _ in range(2)]
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    x = O.random_tensor(list(dims), 13).astype("float32")
    res = mb.mach_hooi(mb.DenseTensor.from_numpy(x), ranks, mb.SparsifyConfig(p, seed), mb.HooiConfig(sweeps, 0.0))
    ref = res.model
    assert sum(o[5] for o in outs) == res.sparsified.nnz  # the slabs partition the kept set
    for rank, its, fits, factors, core, _ in outs:
        assert its == ref.iterations
        assert np.abs(np.array(fits) - np.array(ref.sweep_fits)).max() <= 1e-4
        for a, b in zip(factors, ref.factors):
            assert subspace_sin(a, b) <= 1e-3
        assert rel(align_core(core, factors, ref.factors), ref.core) <= 1e-4


def test_partial_grams_sum_to_the_full_gram_and_give_the_hosvd():
    """for every mode but the last the time slabs partition the
    columns of X_(n), so the shards' row Grams add up to the full one; the
    HOSVD from the summed Grams (+ the last mode's Gram of the gathered
    nonzeros) equals the one-shot sparse HOSVD."""
    import paper_0909_4969_b200 as mb
    from tests.helpers import subspace_sin
    dims, ranks, p, seed = (30, 24, 40), (3, 4, 5), 0.3, 11
    x = O.random_tensor(list(dims), 8)
    full = mb.sparsify(x, mb.SparsifyConfig(p, seed))
    S = dims[0] * dims[1]
    parts = [mb.sparsify_slab(np.ascontiguousarray(x[..., t0:t1]), dims, t0 * S, mb.SparsifyConfig(p, seed))
             for t0, t1 in ((0, 13), (13, 14), (14, 40))]
    d = full.densify()
    for m in range(2):
        a = np.moveaxis(d, m, 0).reshape(dims[m], -1, order="F")
        g = sum(mb.sparse_row_gram(sp, m) for sp in parts)
        assert np.abs(g - a @ a.T).max() <= 1e-12 * np.abs(a @ a.T).max()
        assert np.abs(g - mb.sparse_row_gram(full, m)).max() <= 1e-12 * np.abs(g).max()
    grams = [sum(mb.sparse_row_gram(sp, m) for sp in parts) for m in range(2)] + [mb.sparse_row_gram(full, 2)]
    ref = mb.hosvd(full, ranks)
    sess = mb.HooiSession.from_grams(full, ranks, grams)  # (one shard holding everything)
    sess.mode_y(2)
    sess.refresh_fit()
    got = sess.model()
    assert abs(got.fit - ref.fit) <= 1e-12 and got.sweep_fits[0] == got.fit
    for fd, fr in zip(got.factors, ref.factors):
        assert subspace_sin(fd, fr) <= 1e-10
    with pytest.raises(mb.ArgumentError):
        mb.sparse_row_gram(mb.sparsify(O.random_tensor([50, 3, 4], 1), mb.SparsifyConfig(0.5, 1)), 0)  # rows > columns
