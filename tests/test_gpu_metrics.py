"""SURVEY §8(f)1 on the GPU: accuracy as one fused device pass (no dense
reconstruction), subspace_sin on the device, and pearson / pc_correlation /
compare (proj/src/metrics.cpp:59-159) against the oracle's restatement.

Bars: fp64 accuracy within 1e-12 of the oracle; pearson bit-identical (same
pairwise summation order); compare's correlations, flips and tie flags equal,
its accuracies within 1e-12, tie sines within 1e-10.
"""
import numpy as np
import pytest

import oracle as O
from paper_0909_4969_b200.synth import lowrank_numpy

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mb():
    import paper_0909_4969_b200 as mb
    return mb


@pytest.mark.parametrize("dims,ranks", [((30, 24, 20), (3, 4, 2)), ((12, 10, 8, 6), (2, 3, 2, 2)), ((200, 9, 70), (6, 3, 5))])
def test_fused_accuracy_matches_oracle(mb, dims, ranks):
    x = lowrank_numpy(dims, ranks, 0.05, seed=sum(dims))
    model = O.hooi(O.Dense(x), ranks, 3, 0.0)
    ref = O.accuracy(O.Dense(x), model)
    dev = mb.accuracy(mb.DenseTensor.from_numpy(x), model)
    assert abs(dev - ref) <= 1e-12, (dev, ref)


def test_fused_accuracy_fp32_reference_tensor(mb):
    dims, ranks = (256, 96, 64), (8, 6, 5)
    x = lowrank_numpy(dims, ranks, 0.02, seed=4).astype(np.float32)
    model = mb.hooi(mb.DenseTensor.from_numpy(x), ranks, mb.HooiConfig(2, 0.0))
    rec = np.asarray(model.core)
    for m, f in enumerate(model.factors):
        rec = np.moveaxis(np.tensordot(f, rec, axes=([1], [m])), 0, m)
    x64 = x.astype(np.float64)
    ref = 1.0 - np.linalg.norm(x64 - rec) / np.linalg.norm(x64)
    assert abs(mb.accuracy(mb.DenseTensor.from_numpy(x), model) - ref) <= 1e-10


def test_subspace_sin_on_device(mb):
    rng = np.random.default_rng(3)
    a, _ = np.linalg.qr(rng.standard_normal((80, 6)))
    b, _ = np.linalg.qr(a + 1e-3 * rng.standard_normal((80, 6)))
    ref = O.subspace_gap(a, b)
    assert abs(mb.subspace_sin(a, b) - ref) <= 1e-12
    assert mb.subspace_sin(a, a) <= 1e-7


@pytest.mark.parametrize("n", [2, 5, 64, 65, 1000, 4097])
def test_pearson_bit_identical(mb, n):
    rng = np.random.default_rng(n)
    x, y = rng.standard_normal(n), rng.standard_normal(n) + 0.3 * np.arange(n)
    assert mb.pearson(x, y) == O.pearson(x, y)
    assert mb.pearson(x, x) == 1.0 and mb.pearson(x, -x) == -1.0
    with pytest.raises(mb.ArgumentError):
        mb.pearson(np.ones(n), y)
    with pytest.raises(mb.ShapeError):
        mb.pearson(x, y[:-1])


def models_pair(dims, ranks, p, seed, tie=False):
    if tie:  # exactly low rank with equal core slice norms: component 1 is not identifiable
        rng = np.random.default_rng(seed)
        core = np.zeros(ranks)
        for i in range(min(ranks)):
            core[(i,) * len(ranks)] = 5.0
        x = core
        for m, (n, r) in enumerate(zip(dims, ranks)):
            q, _ = np.linalg.qr(rng.standard_normal((n, r)))
            x = np.moveaxis(np.tensordot(q, x, axes=([1], [m])), 0, m)
    else:
        x = lowrank_numpy(dims, ranks, 0.02, seed=seed)
    exact = O.hooi(O.Dense(x), ranks, 4, 0.0)
    approx, _ = O.mach_hooi(O.Dense(x), ranks, p, 7, 4, 0.0)
    return x, exact, approx


@pytest.mark.parametrize("tie", [False, True])
def test_compare_matches_oracle(mb, tie):
    x, exact, approx = models_pair((40, 30, 24), (3, 3, 3), 0.3, 11, tie)
    dev = mb.compare(exact, approx, x)
    ref = O.compare(exact, approx, O.Dense(x))
    assert dev["flipped"] == ref["flipped"]
    assert dev["tied"] == ref["tied"]
    assert np.array_equal(np.array(dev["per_mode_rho"]), ref["per_mode_rho"])
    assert np.abs(np.array(dev["tie_subspace_sin"]) - ref["tie_subspace_sin"]).max() <= 1e-10
    assert abs(dev["accuracy_exact"] - ref["accuracy_exact"]) <= 1e-12
    assert abs(dev["accuracy_mach"] - ref["accuracy_mach"]) <= 1e-12
    assert dev["core_interaction"] == ref["core_interaction"]
    if tie:
        assert any(dev["tied"])
    for m in range(3):
        rho, fl = mb.pc_correlation(exact, approx, m, 2)
        r2, f2 = O.pc_correlation(exact, approx, m, 2)
        assert rho == r2 and fl == f2
    with pytest.raises(mb.ArgumentError):
        mb.pc_correlation(exact, approx, 0, 4)
