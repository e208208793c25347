"""HOSVD / HOOI parity on the B200 against the CPU oracle.

North-star bars (BASELINE.json): factors equal up to column sign with the
largest principal-angle sine <= 1e-9 (fp64) / <= 1e-3 (fp32); core and fit
within 1e-4 relative (fp32); iterations and sweep_fits compared.  fp64 cases
are held to fp64-level tolerances (1e-9).
"""
import numpy as np
import pytest

import oracle as O
from paper_0909_4969_b200.synth import lowrank_numpy
from tests.helpers import align_core, canonical_cols, rel, subspace_sin

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mb():
    import paper_0909_4969_b200 as mb
    return mb


def assert_same_iterations(dev, ref, fit_tol):
    """The stop rule (fit - prev < tol, tucker.cpp:102) is compared, not
    assumed.  With tol = 0 a converged model stops on a rounding-level fit
    decrease, which either side may hit first; that is the only accepted
    difference, and the shared prefix of sweep_fits must agree."""
    n = min(len(dev.sweep_fits), len(ref.sweep_fits))
    assert np.abs(np.array(dev.sweep_fits[:n]) - np.array(ref.sweep_fits[:n])).max() <= fit_tol
    if dev.iterations != ref.iterations:
        short = dev if dev.iterations < ref.iterations else ref
        k = short.iterations
        assert abs(short.sweep_fits[k] - short.sweep_fits[k - 1]) <= 1e-12, (dev.sweep_fits, ref.sweep_fits)
        return False
    return True


def assert_model_close(dev, ref, sin_tol, rel_tol, fit_tol):
    if assert_same_iterations(dev, ref, fit_tol):
        assert len(dev.sweep_fits) == len(ref.sweep_fits)
        assert np.abs(np.array(dev.sweep_fits) - np.array(ref.sweep_fits)).max() <= fit_tol
    assert abs(dev.fit - ref.fit) <= fit_tol
    for fd, fr in zip(dev.factors, ref.factors):
        assert fd.shape == fr.shape
        assert subspace_sin(fd, fr) <= sin_tol
        assert np.abs(fd.T @ fd - np.eye(fd.shape[1])).max() < 1e-10
    core = align_core(dev.core, dev.factors, ref.factors)
    assert rel(core, ref.core) <= rel_tol
    assert dev.warnings == ref.warnings


# ---------------------------------------------------------------------------
# sparse route, fp64 (C1-style and small shapes)
# ---------------------------------------------------------------------------
SPARSE64 = [
    ((20, 15, 30), (3, 2, 4), 0.2, 5, 10),
    ((30, 25, 20), (4, 4, 4), 0.1, 9, 5),
    ((64, 8, 40), (5, 3, 6), 0.15, 3, 8),
    ((40, 50), (4, 3), 0.1, 2, 6),       # order 2
]


@pytest.mark.parametrize("dims,ranks,p,seed,sweeps", SPARSE64)
def test_mach_hooi_fp64_matches_oracle(mb, dims, ranks, p, seed, sweeps):
    x = lowrank_numpy(dims, ranks, 0.01, seed=seed)
    res = mb.mach_hooi(x, ranks, mb.SparsifyConfig(p, 7), mb.HooiConfig(sweeps, 0.0))
    ref_model, ref_sparse = O.mach_hooi(O.Dense(x), ranks, p, 7, sweeps, 0.0)
    idx, vals = res.sparsified.entries()
    oi, ov = ref_sparse.entries()
    assert np.array_equal(idx, oi) and np.array_equal(vals, ov)
    assert_model_close(res.model, ref_model, 1e-9, 1e-9, 1e-9)


def test_c1_config_fp64(mb):
    """BASELINE configs[0]: 100x12x1024 fp64, ranks (5,5,5), p=0.1, HOSVD + 3 sweeps."""
    dims, ranks = (100, 12, 1024), (5, 5, 5)
    x = lowrank_numpy(dims, ranks, 0.01, seed=1)
    res = mb.mach_hooi(x, ranks, mb.SparsifyConfig(0.1, 7), mb.HooiConfig(3, 0.0))
    ref_model, _ = O.mach_hooi(O.Dense(x), ranks, 0.1, 7, 3, 0.0)
    assert_model_close(res.model, ref_model, 1e-9, 1e-8, 1e-9)


def test_sparse_hosvd_tall_mode_column_side(mb):
    # mode 0 taller than the product of the others -> column-side Gram + products
    rng = np.random.default_rng(77)
    dims = (30, 4, 5)
    idx = rng.choice(600, size=60, replace=False)
    vals = rng.standard_normal(60)
    st = mb.SparseTensor.from_entries(dims, idx, vals)
    ref = O.hosvd(O.Sparse.from_entries(dims, idx, vals), [3, 2, 2])
    dev = mb.hosvd(st, [3, 2, 2])
    assert_model_close(dev, ref, 1e-9, 1e-9, 1e-12)
    for fd, fr in zip(dev.factors, ref.factors):
        assert np.abs(canonical_cols(fd) - canonical_cols(fr)).max() < 1e-9


def test_sparse_hooi_random_sparse(mb):
    rng = np.random.default_rng(123)
    dims = (8, 9, 10)
    idx = rng.choice(720, size=70, replace=False)
    vals = rng.standard_normal(70)
    dev = mb.hooi(mb.SparseTensor.from_entries(dims, idx, vals), [2, 2, 2])
    ref = O.hooi(O.Sparse.from_entries(dims, idx, vals), [2, 2, 2])
    assert_model_close(dev, ref, 1e-9, 1e-9, 1e-12)


# ---------------------------------------------------------------------------
# fp32 sparse route (C2/C3/C5-like shapes at test scale)
# ---------------------------------------------------------------------------
SPARSE32 = [
    ((64, 64, 64), (10, 10, 10), 0.05, 1, 5),
    ((96, 80, 128), (16, 16, 16), 0.1, 2, 3),
    ((100, 16, 512), (10, 6, 12), 0.05, 3, 3),
]


@pytest.mark.parametrize("dims,ranks,p,seed,sweeps", SPARSE32)
def test_mach_hooi_fp32_matches_oracle(mb, dims, ranks, p, seed, sweeps):
    x = lowrank_numpy(dims, ranks, 0.01, seed=seed, dtype=np.float32)
    res = mb.mach_hooi(mb.DenseTensor.from_numpy(x), ranks, mb.SparsifyConfig(p, 7), mb.HooiConfig(sweeps, 0.0))
    ref_model, ref_sparse = O.mach_hooi(O.Dense(x.astype(np.float64)), ranks, p, 7, sweeps, 0.0)
    assert np.array_equal(res.sparsified.entries()[0], ref_sparse.entries()[0])
    m = res.model
    assert m.iterations == ref_model.iterations
    for fd, fr in zip(m.factors, ref_model.factors):
        assert subspace_sin(fd, fr) <= 1e-3
    assert rel(align_core(m.core, m.factors, ref_model.factors), ref_model.core) <= 1e-4
    assert abs(m.fit - ref_model.fit) <= 1e-4 * abs(ref_model.fit)
    assert np.allclose(m.sweep_fits, ref_model.sweep_fits, rtol=1e-4, atol=0)


# ---------------------------------------------------------------------------
# dense route (density >= 0.25 switch, dense inputs, general orders)
# ---------------------------------------------------------------------------
def test_dense_hooi_matches_oracle(mb):
    x = O.random_tensor([6, 7, 8], 42)
    dev = mb.hooi(x, [2, 2, 2], mb.HooiConfig(50, 0.0))
    ref = O.hooi(O.Dense(x), [2, 2, 2], 50, 0.0)
    assert_model_close(dev, ref, 1e-9, 1e-8, 1e-12)


def test_keep_everything_rides_dense_route(mb):
    x = O.random_tensor([6, 7, 8], 46)
    res = mb.mach_hooi(x, [2, 3, 2], mb.SparsifyConfig(1.0, 31))
    ref = O.hooi(O.Dense(x), [2, 3, 2])
    assert res.sparsified.nnz == x.size
    assert_model_close(res.model, ref, 1e-9, 1e-8, 1e-12)


def test_four_way_matches_oracle(mb):
    x = lowrank_numpy((12, 10, 8, 14), (3, 3, 2, 4), 0.02, seed=4)
    res = mb.mach_hooi(x, (3, 3, 2, 4), mb.SparsifyConfig(0.2, 5), mb.HooiConfig(4, 0.0))
    ref, _ = O.mach_hooi(O.Dense(x), (3, 3, 2, 4), 0.2, 5, 4, 0.0)
    assert_model_close(res.model, ref, 1e-9, 1e-8, 1e-9)


# order-4 sparse route (stage 1 fibre sums + dimension-tree stage 2), C3-like
FOURWAY = [
    ((20, 18, 9, 30), (3, 4, 2, 5), 0.05, np.float64, 3),
    ((32, 32, 16, 64), (8, 8, 8, 8), 0.02, np.float32, 3),
    ((24, 40, 7, 50), (5, 6, 3, 4), 0.1, np.float32, 4),
]


@pytest.mark.parametrize("dims,ranks,p,dt,sweeps", FOURWAY)
def test_four_way_sparse_route_matches_oracle(mb, dims, ranks, p, dt, sweeps):
    x = lowrank_numpy(dims, ranks, 0.02, seed=8, dtype=dt)
    res = mb.mach_hooi(mb.DenseTensor.from_numpy(x), ranks, mb.SparsifyConfig(p, 7), mb.HooiConfig(sweeps, 0.0))
    ref, ref_sp = O.mach_hooi(O.Dense(x.astype(np.float64)), ranks, p, 7, sweeps, 0.0)
    assert np.array_equal(res.sparsified.entries()[0], ref_sp.entries()[0])
    assert res.sparsified.nnz < 0.25 * x.size  # sparse route (below the densify switch)
    if dt == np.float64:
        assert_model_close(res.model, ref, 1e-9, 1e-8, 1e-9)
        return
    m = res.model
    assert m.iterations == ref.iterations
    for fd, fr in zip(m.factors, ref.factors):
        assert subspace_sin(fd, fr) <= 1e-3
    assert rel(align_core(m.core, m.factors, ref.factors), ref.core) <= 1e-4
    assert np.allclose(m.sweep_fits, ref.sweep_fits, rtol=1e-4, atol=0)


def test_order_one(mb):
    x = O.random_tensor([9], 77)
    assert mb.hosvd(x, [1]).fit >= 1 - 1e-10
    assert len(mb.hosvd(x, [3]).warnings) == 1
    h = mb.hooi(x, [2])
    assert h.iterations == 1 and h.fit >= 1 - 1e-10


# ---------------------------------------------------------------------------
# reference known answers (proj/tests/test_tucker.cpp) on the device path
# ---------------------------------------------------------------------------
def test_separable_rank_one(mb):
    from tests.test_oracle_pins import separable3
    t = separable3(4, 5, 6, 7.0, 21)
    m = mb.hosvd(t, [1, 1, 1])
    assert abs(abs(m.core.reshape(-1)[0]) - 7.0) < 1e-12
    assert m.fit >= 1 - 1e-10 and m.warnings == []
    assert mb.accuracy(t, m) >= 1 - 1e-10


def test_exact_low_rank_one_sweep(mb):
    from tests.test_oracle_pins import exact_rank_tensor
    t = exact_rank_tensor([6, 7, 8], [2, 2, 2], 3)
    m = mb.hooi(t, [2, 2, 2])
    assert m.iterations == 1 and abs(m.fit - 1) < 1e-10 and len(m.sweep_fits) == 2


def test_completion_warnings(mb):
    from tests.test_oracle_pins import separable3
    m = mb.hosvd(separable3(4, 5, 6, 3.0, 9), [2, 2, 2])
    assert len(m.warnings) == 3 and "mode 1" in m.warnings[0] and "mode 3" in m.warnings[2]
    assert m.fit >= 1 - 1e-10


def test_monotone_and_stop_rule(mb):
    x = O.random_tensor([6, 7, 8], 42)
    m = mb.hooi(x, [2, 2, 2], mb.HooiConfig(50, 0.0))
    assert all(b >= a - 1e-12 for a, b in zip(m.sweep_fits, m.sweep_fits[1:]))
    assert mb.hooi(x, [2, 2, 2], mb.HooiConfig(50, 0.5)).iterations == 1
    c = mb.hooi(x, [2, 2, 2], mb.HooiConfig(2, 0.0))
    assert c.iterations <= 2 and len(c.sweep_fits) == c.iterations + 1


def test_validation_errors(mb):
    x = O.random_tensor([4, 5, 6], 2)
    for r in ([0, 2, 2], [2, 2, 7], [2, 2]):
        with pytest.raises(mb.ArgumentError):
            mb.hosvd(x, r)
    for cfg in (mb.HooiConfig(0, 1e-4), mb.HooiConfig(10, -1.0), mb.HooiConfig(10, float("nan"))):
        with pytest.raises(mb.ArgumentError):
            mb.hooi(x, [2, 2, 2], cfg)


def test_bitwise_deterministic(mb):
    x = lowrank_numpy((40, 30, 50), (4, 3, 5), 0.01, seed=8, dtype=np.float32)
    a = mb.mach_hooi(mb.DenseTensor.from_numpy(x), (4, 3, 5), mb.SparsifyConfig(0.1, 3), mb.HooiConfig(4, 0.0)).model
    b = mb.mach_hooi(mb.DenseTensor.from_numpy(x), (4, 3, 5), mb.SparsifyConfig(0.1, 3), mb.HooiConfig(4, 0.0)).model
    assert np.array_equal(a.core, b.core) and a.sweep_fits == b.sweep_fits
    for fa, fb in zip(a.factors, b.factors):
        assert np.array_equal(fa, fb)


# ---------------------------------------------------------------------------
# eigen step in isolation (linalg.cpp:319-353)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("shape,k", [((6, 9), 3), ((40, 12), 5), ((12, 40), 12), ((150, 150), 10),
                                     ((300, 500), 8), ((7, 3), 5)])
def test_left_singular_basis_matches_oracle(mb, shape, k):
    a = O.random_matrix(shape[0], shape[1], 515 + shape[0])
    dev = mb.left_singular_basis(a, k)
    b, sv, nr, comp = O.left_singular_basis(a, k)
    assert dev.numerical_rank == nr and dev.completed == comp
    assert np.abs(dev.singular_values - sv).max() <= 1e-10 * max(1.0, sv.max())
    assert np.abs(dev.basis - b).max() < 1e-8  # same canonical signs, same completions


def test_left_singular_basis_zero(mb):
    dev = mb.left_singular_basis(np.zeros((4, 3)), 4)
    assert dev.numerical_rank == 0 and dev.completed
    assert np.abs(dev.basis - np.eye(4)).max() == 0


# ---------------------------------------------------------------------------
# large row Grams: the multi-kernel eigensolver (n beyond one CTA's shared
# memory) against the oracle and against the single-CTA global-memory solver
# ---------------------------------------------------------------------------
def _hosvd_env(mb, monkeypatch, st, ranks, **env):
    monkeypatch.delenv("MACH_EIG_LARGE_OFF", raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    return mb.hosvd(st, ranks)


@pytest.mark.parametrize("dims,ranks,p", [((300, 30, 40), (5, 4, 4), 0.2), ((600, 20, 24), (8, 3, 3), 0.3),
                                          ((520, 16, 70), (10, 4, 6), 0.1),
                                          ((300, 40, 40), (20, 6, 6), 0.2),    # block size 24
                                          ((260, 36, 36), (28, 4, 4), 0.3)])   # block size 32
def test_large_gram_eigensolver(mb, monkeypatch, dims, ranks, p):
    x = lowrank_numpy(dims, ranks, 0.01, seed=4)
    rng = np.random.default_rng(5)
    keep = rng.random(x.size) < p
    idx = np.flatnonzero(keep)
    vals = x.reshape(-1, order="F")[idx]
    st = mb.SparseTensor.from_entries(dims, idx, vals)
    ref = O.hosvd(O.Sparse.from_entries(dims, idx, vals), list(ranks))
    large = _hosvd_env(mb, monkeypatch, st, ranks)
    assert_model_close(large, ref, 1e-9, 1e-9, 1e-12)
    single = _hosvd_env(mb, monkeypatch, st, ranks, MACH_EIG_LARGE_OFF="1")
    assert_model_close(single, ref, 1e-9, 1e-9, 1e-12)


def test_mode_basis_fallback_inside_sweep_graph(mb, monkeypatch):
    """The fused mode-basis kernel hands off to flag-gated fallback kernels
    that sit in every sweep (and in the captured sweep graph); forcing the
    fallback on every mode must give the same model as the fast path (and
    the oracle)."""
    dims, ranks, p, sweeps = (64, 64, 64), (10, 10, 10), 0.05, 5
    x = lowrank_numpy(dims, ranks, 0.01, seed=1, dtype=np.float32)

    def run(force):
        if force:
            monkeypatch.setenv("MACH_FORCE_MB_FALLBACK", "1")
        else:
            monkeypatch.delenv("MACH_FORCE_MB_FALLBACK", raising=False)
        return mb.mach_hooi(mb.DenseTensor.from_numpy(x), ranks, mb.SparsifyConfig(p, 7),
                            mb.HooiConfig(sweeps, 0.0)).model

    fast, forced = run(False), run(True)
    ref, _ = O.mach_hooi(O.Dense(x.astype(np.float64)), ranks, p, 7, sweeps, 0.0)
    assert forced.iterations == fast.iterations >= 3  # >= 2 sweeps replayed from the graph
    for a, b, r in zip(fast.factors, forced.factors, ref.factors):
        assert subspace_sin(a, b) <= 1e-6
        assert subspace_sin(b, r) <= 1e-3
    assert np.allclose(forced.sweep_fits, fast.sweep_fits, rtol=1e-6, atol=0)
    n = min(len(forced.sweep_fits), len(ref.sweep_fits))
    assert np.allclose(forced.sweep_fits[:n], ref.sweep_fits[:n], rtol=1e-4, atol=0)


@pytest.mark.parametrize("dims,ranks", [((30, 25, 20), (4, 4, 4)), ((64, 40, 50), (5, 3, 6)), ((40, 70, 33), (6, 20, 5))])
def test_sweep_variants_match_full_ttm(mb, monkeypatch, dims, ranks):
    """The overlapped sweep (split TTM, default), the fibre-sum reuse sweep
    (MACH_NO_OVERLAP) and plain full TTMs for every mode (both off) give the
    same model to fp64 rounding."""
    x = lowrank_numpy(dims, ranks, 0.01, seed=6)

    def run(**env):
        for k in ("MACH_NO_OVERLAP", "MACH_NO_FIBRE_REUSE"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        return mb.mach_hooi(x, ranks, mb.SparsifyConfig(0.2, 3), mb.HooiConfig(6, 0.0)).model

    full = run(MACH_NO_OVERLAP="1", MACH_NO_FIBRE_REUSE="1")
    for m in (run(), run(MACH_NO_OVERLAP="1")):
        assert m.iterations == full.iterations
        for fa, fb in zip(m.factors, full.factors):
            assert subspace_sin(fa, fb) <= 1e-10
        assert np.abs(np.array(m.sweep_fits) - np.array(full.sweep_fits)).max() <= 1e-12


def test_side_stream_grams_bitwise_equal(mb, monkeypatch):
    """HOSVD's row Grams computed on a side stream during setup (default) give
    the same fixed-point Grams, hence bitwise the same model, as computing
    them in line (MACH_NO_ASYNC_GRAMS)."""
    x = lowrank_numpy((70, 60, 50), (5, 4, 6), 0.01, seed=12, dtype=np.float32)

    def run(off):
        if off:
            monkeypatch.setenv("MACH_NO_ASYNC_GRAMS", "1")
        else:
            monkeypatch.delenv("MACH_NO_ASYNC_GRAMS", raising=False)
        return mb.mach_hooi(mb.DenseTensor.from_numpy(x), (5, 4, 6), mb.SparsifyConfig(0.1, 5),
                            mb.HooiConfig(3, 0.0)).model

    a, b = run(False), run(True)
    assert np.array_equal(a.core, b.core) and a.sweep_fits == b.sweep_fits
    for fa, fb in zip(a.factors, b.factors):
        assert np.array_equal(fa, fb)
