"""Sampler parity on the B200: kept-index set bit-exact against the oracle.

The device path is mach_sparsify (sampler.cu) through the C ABI; the checker
is the CPU oracle's restatement of proj/src/sampling.cpp:21-31, itself pinned
to SplitMix64's published outputs (tests/test_oracle_pins.py).
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mb():
    import paper_0909_4969_b200 as mb
    return mb


CASES = [
    ((4, 3, 2), 0.5, 7),
    ((1000,), 0.1, 0),
    ((1000,), 0.05, 1),
    ((37, 41, 13), 0.3, 12345),
    ((100, 12, 1024), 0.1, 7),          # C1 shape
    ((64, 64, 64), 0.05, 2**63 + 11),   # large seed
    ((5, 6, 7), 1.0, 99),               # keep everything
    ((257, 3), 0.001, 5),
    ((4097,), 0.9, 3),                  # tile tail
    ((1,), 0.5, 0),
]


@pytest.mark.parametrize("dims,p,seed", CASES)
def test_kept_set_bitexact_fp64(mb, dims, p, seed):
    x = O.random_tensor(list(dims), 17)
    x.reshape(-1, order="F")[::7] = 0.0  # zeros are never emitted
    s = mb.sparsify(x, mb.SparsifyConfig(p, seed))
    idx, vals = s.entries()
    oi, ov = O.sparsify(O.Dense(x), p, seed).entries()
    assert np.array_equal(idx, oi)
    assert np.array_equal(vals.view(np.uint64), ov.view(np.uint64))  # x / p bit for bit


@pytest.mark.parametrize("dims,p,seed", CASES[:6])
def test_kept_set_bitexact_fp32(mb, dims, p, seed):
    x = O.random_tensor(list(dims), 23).astype(np.float32)
    s = mb.sparsify(mb.DenseTensor.from_numpy(x), mb.SparsifyConfig(p, seed))
    idx, vals = s.entries()
    oi, ov = O.sparsify(O.Dense(x.astype(np.float64)), p, seed).entries()
    assert np.array_equal(idx, oi)
    # fp32 values are the reference's fp64 x/p rounded once to fp32
    assert np.array_equal(vals.astype(np.float32), ov.astype(np.float32))


def test_p_one_is_identity_and_zeros_dropped(mb):
    x = np.zeros((3, 3))
    x[1, 1] = 4.0
    x[2, 0] = -2.5
    s = mb.sparsify(x, mb.SparsifyConfig(1.0, 0))
    assert s.nnz == 2
    assert np.array_equal(s.densify(), x)
    y = O.random_tensor([5, 6, 7], 40)
    assert np.array_equal(mb.sparsify(y, mb.SparsifyConfig(1.0, 3)).densify(), y)


def test_validation(mb):
    x = O.random_tensor([3, 3], 45)
    for p in (0.0, -0.2, 1.5, float("nan")):
        with pytest.raises(mb.ArgumentError):
            mb.sparsify(x, mb.SparsifyConfig(p, 0))
    bad = x.copy()
    bad[0, 0] = np.inf
    with pytest.raises(mb.ArgumentError):
        mb.sparsify(bad, mb.SparsifyConfig(0.5, 0))


def test_large_size_properties(mb):
    """Full-size property checks where the oracle would be slow: count within
    a binomial band, ascending unique indices, exact 1/p scaling."""
    import torch
    from paper_0909_4969_b200.synth import lowrank_torch

    dims = (256, 256, 512)
    x = lowrank_torch(dims, (10, 10, 10), 0.01, seed=2, dtype="float32")
    t = mb.DenseTensor.from_torch(x, dims)
    p = 0.05
    s = mb.sparsify(t, mb.SparsifyConfig(p, 7))
    idx, vals = s.entries()
    n = x.numel()
    assert abs(len(idx) - n * p) < 6 * np.sqrt(n * p)
    assert np.all(np.diff(idx) > 0)
    xh = x.cpu().numpy()
    assert np.array_equal((xh[idx].astype(np.float64) / p).astype(np.float32), vals.astype(np.float32))
    # spot-check the keep rule on a slice with the numpy restatement of the hash
    from tests.test_oracle_pins import np_hash
    lo = 123456
    cs = np.arange(lo, lo + 20000, dtype=np.uint64)
    keep = (np_hash(7, cs) >> np.uint64(11)) < np.uint64(int(np.ceil(p * 2.0**53)))
    keep &= xh[lo:lo + 20000] != 0
    want = np.nonzero(keep)[0] + lo
    got = idx[(idx >= lo) & (idx < lo + 20000)]
    assert np.array_equal(got, want)
    del torch


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", [1, 4095, 4096, 4097, 70001])
def test_keep_all_path_p1(mb, dtype, n):
    """p = 1 (sampling.cpp:25-27: every nonzero entry, values unchanged) runs the
    two-pass keep-all kernels: kept set and values equal the oracle's, zeros
    (and -0.0) skipped, ragged sizes, slab offsets, non-finite input rejected."""
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n).astype(dtype)
    x[rng.random(n) < 0.3] = 0.0
    if n > 10:
        x[7] = -0.0
    dims = (n, 1, 1) if n < 100 else (n,)
    x = x.reshape(dims)
    ref_idx, ref_val = O.sparsify(O.Dense(x.astype(np.float64)), 1.0, 3).entries()
    sp = mb.sparsify(mb.DenseTensor.from_numpy(x), mb.SparsifyConfig(1.0, 3))
    idx, val = sp.entries()
    assert np.array_equal(idx, ref_idx) and np.array_equal(val, ref_val)
    if n > 4096:
        off = 1000
        part = mb.sparsify_slab(mb.DenseTensor.from_numpy(x.reshape(-1)[off:].reshape(-1)), (n,), off, mb.SparsifyConfig(1.0, 3))
        pi, pv = part.entries()
        assert np.array_equal(pi, ref_idx[ref_idx >= off]) and np.array_equal(pv, ref_val[ref_idx >= off])
        bad = x.copy().reshape(-1)
        bad[n // 2] = np.inf
        with pytest.raises(mb.ArgumentError):
            mb.sparsify(mb.DenseTensor.from_numpy(bad), mb.SparsifyConfig(1.0, 3))
    z = mb.sparsify(mb.DenseTensor.from_numpy(np.zeros((5, 4), dtype=dtype)), mb.SparsifyConfig(1.0, 3))
    assert z.nnz == 0
