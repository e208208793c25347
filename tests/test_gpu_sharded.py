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


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_sharded_world1_matches_session(dtype):
    import torch
    import torch.distributed as dist

    import paper_0909_4969_b200 as mb
    from paper_0909_4969_b200.sharded import sharded_mach_hooi

    dims, ranks, p, seed, sweeps = (40, 30, 36), (4, 3, 5), 0.2, 7, 3
    x = O.random_tensor(list(dims), 13).astype(dtype)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        flat = torch.from_numpy(x.reshape(-1, order="F").copy()).cuda()
        model, sp = sharded_mach_hooi(flat, dims, ranks, p, seed, sweeps, 0.0)
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
