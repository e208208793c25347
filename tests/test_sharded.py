"""Time-slab sharding host logic (paper_0909_4969_b200/sharded.py) on CPU.

`sharded_sweeps` — the per-sweep exchange the CUDA path runs over NCCL — is
driven here over `gloo` with world size 2 (127.0.0.1) by a numpy engine whose
local steps restate the reference (tensor.cpp:241-259 TTM, linalg.cpp
left_singular_basis via the oracle, tucker.cpp:80-106 loop).  Checks: the
slab sampler partition reproduces the full kept set, the 2-rank result equals
the 1-rank result and the oracle's mach_hooi.  The engine is test
infrastructure; the product engine is CudaEngine (tests/test_gpu_sharded.py).
"""
import os
import socket

import numpy as np
import pytest

import oracle as O
from paper_0909_4969_b200.sharded import sharded_sweeps, slab_bounds
from tests.helpers import align_core, rel, subspace_sin

DIMS, RANKS, P, SEED, SWEEPS = (14, 10, 12), (3, 2, 4), 0.3, 7, 4


def tensor():
    return O.random_tensor(list(DIMS), 41)


class NumpyEngine:
    """Local steps of one rank: dense numpy stand-in of the device session."""

    def __init__(self, idx, vals, factors, norm2, fit0):
        import torch
        self.torch = torch
        x = np.zeros(int(np.prod(DIMS)))
        x[idx] = vals
        self.x = x.reshape(DIMS, order="F")
        self.U = [f.copy() for f in factors]
        self.norm2, self.fit, self.prev, self.fits = norm2, fit0, fit0, [fit0]

    def mode_y(self, m):
        y = self.x
        for j in range(len(DIMS)):
            if j != m:
                y = np.moveaxis(np.tensordot(self.U[j].T, y, axes=([1], [j])), 0, j)
        self.ym_shape = (DIMS[m], y.size // DIMS[m])
        self.y = self.torch.from_numpy(np.moveaxis(y, m, 0).reshape(self.ym_shape, order="F").reshape(-1, order="F").copy())
        return self.y

    def mode_update(self, m):
        ym = self.y.numpy().reshape(self.ym_shape, order="F")
        self.U[m] = O.left_singular_basis(ym, RANKS[m])[0]
        self.last = (m, ym)

    def sweep_end(self, tol):
        m, ym = self.last
        g = self.U[m].T @ ym
        others = [RANKS[j] for j in range(len(DIMS)) if j != m]
        self.core = np.moveaxis(g.reshape([RANKS[m]] + others, order="F"), 0, m)
        e2 = max(self.norm2 - float((self.core ** 2).sum()), 0.0)
        self.fit = 1.0 - np.sqrt(e2) / np.sqrt(self.norm2)
        self.fits.append(self.fit)
        stop = tol >= 0 and self.fit - self.prev < tol
        self.prev = self.fit
        return stop


def local_engine(rank, world):
    x = tensor()
    full = O.sparsify(O.Dense(x), P, SEED)
    idx, vals = full.entries()
    S = int(np.prod(DIMS[:-1]))
    t0, t1 = slab_bounds(DIMS[-1], world, rank)
    keep = (idx >= t0 * S) & (idx < t1 * S)
    h = O.hosvd(full, list(RANKS))
    # global |X|^2 (the CUDA path all-reduces the per-rank partial sums)
    return NumpyEngine(idx[keep], vals[keep], h.factors, float((vals ** 2).sum()), h.fit), (idx, vals, keep)


def worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    eng, _ = local_engine(rank, world)
    sharded_sweeps(eng, lambda y: dist.all_reduce(y), len(DIMS), SWEEPS, 0.0)
    if rank == 0:
        np.savez(out, *eng.U, core=eng.core, fits=np.array(eng.fits))
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_world(world, tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / f"w{world}.npz")
    mp.spawn(worker, args=(world, free_port(), out), nprocs=world, join=True)
    z = np.load(out)
    return [z[f"arr_{i}"] for i in range(len(DIMS))], z["core"], z["fits"]


def test_slab_bounds_partition():
    for extent in (1, 7, 12, 65536):
        for world in (1, 2, 3, 8):
            b = [slab_bounds(extent, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == extent
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            assert max(t1 - t0 for t0, t1 in b) - min(t1 - t0 for t0, t1 in b) <= 1


def test_slab_sampling_partition_is_the_full_kept_set():
    # the kept set depends only on (seed, global flat index): slabs partition it
    x = tensor()
    idx, vals = O.sparsify(O.Dense(x), P, SEED).entries()
    S = int(np.prod(DIMS[:-1]))
    parts = []
    for r in range(3):
        t0, t1 = slab_bounds(DIMS[-1], 3, r)
        slab = np.zeros_like(x)
        slab[..., t0:t1] = x[..., t0:t1]
        pi, pv = O.sparsify(O.Dense(slab), P, SEED).entries()
        assert np.all((pi >= t0 * S) & (pi < t1 * S))
        parts.append((pi, pv))
    assert np.array_equal(np.concatenate([p[0] for p in parts]), idx)
    assert np.array_equal(np.concatenate([p[1] for p in parts]), vals)


def test_sharded_sweeps_gloo_world2_matches_world1_and_oracle(tmp_path):
    f1, c1, fits1 = run_world(1, tmp_path)
    f2, c2, fits2 = run_world(2, tmp_path)
    ref, _ = O.mach_hooi(O.Dense(tensor()), list(RANKS), P, SEED, SWEEPS, 0.0)
    for a, b, r in zip(f2, f1, ref.factors):
        assert subspace_sin(a, b) <= 1e-12
        assert subspace_sin(a, r) <= 1e-9
    assert rel(c2, c1) <= 1e-12
    assert rel(align_core(c2, f2, ref.factors), ref.core) <= 1e-9
    n = min(len(fits2), len(ref.sweep_fits))
    assert np.abs(fits2[:n] - np.array(ref.sweep_fits[:n])).max() <= 1e-9
