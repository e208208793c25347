"""Dense route on the tensor cores (gram_tc.cu): the mode-n Gram X_(n) X_(n)^T
through tcgen05 kind::tf32 against an fp64 Gram, and the fp32 dense HOSVD /
HOOI that uses it against the CPU oracle.

Reference: hosvd(DenseTensor) (proj/src/tucker.cpp:135-150) -> row-side Gram
a * a^T (proj/src/linalg.cpp:340).  Tolerances: the Gram carries TF32
operands (10-bit mantissa): entrywise error <= 2e-3 of the largest diagonal
entry; the leading eigen-subspace of a low-rank + noise Gram within sine
1e-4 of the fp64 one; the HOSVD / HOOI model within the north_star fp32 bars
(sine <= 1e-3, fit and core 1e-4 relative).
"""
import numpy as np
import pytest

import oracle as O
from paper_0909_4969_b200.synth import lowrank_numpy
from tests.helpers import align_core, rel, subspace_sin

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mb():
    import paper_0909_4969_b200 as mb
    return mb


def unfold(x, mode):
    return np.moveaxis(x, mode, 0).reshape(x.shape[mode], -1, order="F")


@pytest.mark.parametrize("dims", [(256, 96, 80), (130, 68, 300), (64, 512, 36), (200, 16, 24, 40)])
def test_mode_gram_tf32_matches_fp64(mb, dims):
    rng = np.random.default_rng(sum(dims))
    x = rng.standard_normal(dims).astype(np.float32)
    t = mb.DenseTensor.from_numpy(x)
    for m in range(len(dims)):
        g, tc = mb.mode_gram(t, m)
        a = unfold(x.astype(np.float64), m)
        ref = a @ a.T
        if dims[m] >= 64 and a.shape[1] >= 4096 and (m == 0 and dims[0] % 4 == 0 or m > 0 and np.prod(dims[:m]) % 4 == 0):
            assert tc, f"mode {m} of {dims} should take the tensor-core Gram"
        assert np.array_equal(g, g.T), "Gram must be exactly symmetric"
        scale = np.abs(np.diag(ref)).max()
        assert np.abs(g - ref).max() <= 2e-3 * scale, (m, np.abs(g - ref).max() / scale)


def test_mode_gram_tf32_subspace(mb):
    dims, ranks = (256, 192, 160), (6, 5, 7)
    x = lowrank_numpy(dims, ranks, 0.01, seed=11).astype(np.float32)
    t = mb.DenseTensor.from_numpy(x)
    for m in range(3):
        g, tc = mb.mode_gram(t, m)
        assert tc
        a = unfold(x.astype(np.float64), m)
        ref = a @ a.T
        k = ranks[m]
        _, vd = np.linalg.eigh(g)
        _, vr = np.linalg.eigh(ref)
        assert subspace_sin(vd[:, -k:], vr[:, -k:]) <= 1e-4


def test_dense_hosvd_fp32_tensor_cores_match_oracle(mb):
    dims, ranks = (256, 128, 192), (8, 6, 7)
    x = lowrank_numpy(dims, ranks, 0.01, seed=5)
    xf = x.astype(np.float32)
    dev = mb.hosvd(mb.DenseTensor.from_numpy(xf), ranks)
    ref = O.hosvd(O.Dense(xf.astype(np.float64)), ranks)
    for fd, fr in zip(dev.factors, ref.factors):
        assert subspace_sin(fd, fr) <= 1e-3
    assert abs(dev.fit - ref.fit) <= 1e-4 * abs(ref.fit)
    core = align_core(dev.core, dev.factors, ref.factors)
    assert rel(core, ref.core) <= 1e-4


def test_dense_hooi_fp32_tensor_cores_match_oracle(mb):
    dims, ranks = (192, 160, 128), (5, 5, 5)
    x = lowrank_numpy(dims, ranks, 0.02, seed=9).astype(np.float32)
    dev = mb.hooi(mb.DenseTensor.from_numpy(x), ranks, mb.HooiConfig(3, 0.0))
    ref = O.hooi(O.Dense(x.astype(np.float64)), ranks, 3, 0.0)
    for fd, fr in zip(dev.factors, ref.factors):
        assert subspace_sin(fd, fr) <= 1e-3
    n = min(len(dev.sweep_fits), len(ref.sweep_fits))
    assert np.abs(np.array(dev.sweep_fits[:n]) - np.array(ref.sweep_fits[:n])).max() <= 1e-4
    core = align_core(dev.core, dev.factors, ref.factors)
    assert rel(core, ref.core) <= 1e-4


@pytest.mark.parametrize("dims,mode,r", [((256, 64, 80), 0, 16), ((256, 64, 80), 1, 10), ((256, 64, 80), 2, 16),
                                          ((130, 50, 300), 1, 32), ((200, 33, 257), 0, 5), ((512, 40, 70), 2, 24)])
def test_mode_product_tf32x3_matches_fp64(mb, dims, mode, r):
    """x_m U^T on tcgen05 with 3xTF32 (ttm_tc.cu) against numpy fp64: the
    split keeps ~2^-22 relative accuracy per product (no truncation bias)."""
    rng = np.random.default_rng(sum(dims) + mode + r)
    x = rng.standard_normal(dims).astype(np.float32)
    m = rng.standard_normal((r, dims[mode]))
    got = mb.mode_product(mb.DenseTensor.from_numpy(x), m, mode)
    ref = np.moveaxis(np.tensordot(m, x.astype(np.float64), axes=([1], [mode])), 0, mode)
    scale = np.sqrt(dims[mode])  # typical magnitude of an output entry
    assert np.abs(got - ref).max() <= 2e-6 * scale, np.abs(got - ref).max() / scale


def test_sampled_hosvd_gram_on_tensor_cores_when_dense_enough(monkeypatch):
    """a sampled fp32 tensor whose mode fibres are long
    (p^2 I_n / 2 >= 1.5 pair products per element) takes its HOSVD row Grams
    from the densified tcgen05 Gram instead of the per-pair nonzero route.
    Bars (north_star, fp32): factor sine <= 1e-3 against the oracle, fit and
    core within 1e-4 relative; the two device routes agree the same way."""
    import paper_0909_4969_b200 as mb

    dims, ranks, p, seed = (256, 192, 320), (8, 6, 7), 0.2, 5  # below the 0.25 densify switch
    x = lowrank_numpy(dims, ranks, 0.01, seed=9).astype(np.float32)
    ctx = mb.Context(0)
    xd = mb.DenseTensor.from_numpy(x, ctx)
    mb.profile(ctx, True)
    tc = mb.mach_hosvd(xd, ranks, mb.SparsifyConfig(p, seed), ctx=ctx)
    ctx.synchronize()
    stats = mb.kernel_stats(ctx)
    mb.profile(ctx, False)
    assert any("gram_tc" in k for k in stats), sorted(stats)
    assert not any("row_gram_kernel" in k for k in stats), sorted(stats)
    monkeypatch.setenv("MACH_SPARSE_GRAM_TC_MIN", "0")
    mb.profile(ctx, True)
    nz = mb.mach_hosvd(xd, ranks, mb.SparsifyConfig(p, seed), ctx=ctx)
    ctx.synchronize()
    stats = mb.kernel_stats(ctx)
    mb.profile(ctx, False)
    assert any("row_gram_kernel" in k for k in stats) and not any("gram_tc" in k for k in stats)
    monkeypatch.delenv("MACH_SPARSE_GRAM_TC_MIN")
    ref, ref_sp = O.mach_hosvd(O.Dense(x.astype(np.float64)), ranks, p, seed)
    assert np.array_equal(tc.sparsified.entries()[0], ref_sp.entries()[0])
    for got in (tc.model, nz.model):
        for fd, fr in zip(got.factors, ref.factors):
            assert subspace_sin(fd, fr) <= 1e-3
        assert abs(got.fit - ref.fit) <= 1e-4 * max(abs(ref.fit), 1e-30) + 1e-6
        assert rel(align_core(got.core, got.factors, ref.factors), ref.core) <= 1e-4
    # and through HOOI (the Grams only seed it)
    h = mb.mach_hooi(xd, ranks, mb.SparsifyConfig(p, seed), mb.HooiConfig(3, 0.0), ctx=ctx)
    href, _ = O.mach_hooi(O.Dense(x.astype(np.float64)), ranks, p, seed, 3, 0.0)
    assert h.model.iterations == href.iterations
    assert abs(h.model.fit - href.fit) <= 1e-4 * abs(href.fit) + 1e-6
    for fd, fr in zip(h.model.factors, href.factors):
        assert subspace_sin(fd, fr) <= 1e-3
