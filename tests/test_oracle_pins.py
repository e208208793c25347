"""Pin the CPU oracle before trusting it (CPU only).

The reference (/root/reference/proj) cannot be built here (Eigen3 missing,
proj/CMakeLists.txt:10), so the oracle is a restatement.  These tests pin it to
  * the published SplitMix64 known answers (the reference RNG is exactly
    SplitMix64's output function on a counter, src/internal.hpp:68-77),
  * the reference's own test suites, restated case by case
    (proj/tests/test_sampling.cpp, test_tucker.cpp, test_tensor.cpp,
    test_linalg.cpp, acceptance.cpp) with the same fixtures
    (proj/tests/oracles.hpp random_tensor: mt19937_64 + libstdc++ normal),
  * numpy.linalg.eigh for the eigensolver.
"""
import math

import numpy as np
import pytest

import oracle as O


# ---------------------------------------------------------------------------
# RNG: published SplitMix64 outputs (state 0 → first three outputs) and an
# independent numpy restatement of src/internal.hpp:68-77.
# ---------------------------------------------------------------------------
SPLITMIX64_SEED0 = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def np_hash(seed, counters):
    c = np.asarray(counters, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (c + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def test_splitmix64_known_answers():
    for i, want in enumerate(SPLITMIX64_SEED0):
        assert O.counter_hash64(0, i) == want


def test_hash_matches_numpy_restatement():
    for seed in (0, 1, 7, 0xDEADBEEF, 2**63 + 5):
        cs = [0, 1, 2, 3, 1000, 2**32 - 1, 2**32, 2**40 + 17]
        got = [O.counter_hash64(seed, c) for c in cs]
        assert got == [int(x) for x in np_hash(seed, cs)]


def test_uniform_is_top53_bits():
    for c in range(50):
        h = O.counter_hash64(3, c)
        assert O.counter_uniform01(3, c) == (h >> 11) * 2.0**-53


def test_integer_threshold_equivalent_to_uniform_compare():
    """keep iff u < p  <=>  (h >> 11) < ceil(p * 2^53): the GPU sampler's test."""
    cs = np.arange(4000, dtype=np.uint64)
    top = np_hash(11, cs) >> np.uint64(11)
    u = top.astype(np.float64) * 2.0**-53
    ps = [1.0, 0.5, 0.25, 0.1, 0.05, 0.02, 0.01, 0.001, 1e-7, 0.3, 1 / 3, 0.999999, 2.0**-53, 0.7 + 1e-16]
    ps += list(np.random.default_rng(0).uniform(0, 1, 200))
    for p in ps:
        thr = np.uint64(math.ceil(p * 2.0**53))
        assert np.array_equal(u < p, top < thr), p
    # boundary cases: p exactly on a representable u value
    for c in range(64):
        uv = int(top[c]) * 2.0**-53
        if uv > 0:
            thr = np.uint64(math.ceil(uv * 2.0**53))
            assert np.array_equal(u < uv, top < thr)


# spot values derived by restating internal.hpp:68-77 + sampling.cpp:21-31
# (SURVEY.md §8c); regression pins for the restatement
def test_sampler_spot_values():
    s = O.sparsify(O.Dense(np.ones((4, 3, 2))), 0.5, 7)
    assert list(s.entries()[0]) == [0, 1, 4, 5, 6, 7, 8, 9, 10, 17, 21, 22, 23]
    assert O.sparsify(O.Dense(np.ones(1000)), 0.1, 0).nnz == 92
    assert list(O.sparsify(O.Dense(np.ones(1000)), 0.05, 1).entries()[0][:8]) == [25, 28, 66, 67, 98, 107, 135, 137]


# ---------------------------------------------------------------------------
# proj/tests/test_sampling.cpp restated
# ---------------------------------------------------------------------------
def test_keep_everything_densifies_back_exactly():          # :55-60
    t = O.random_tensor([5, 6, 7], 40)
    sp = O.sparsify(O.Dense(t), 1.0, 99)
    assert sp.nnz == t.size
    assert np.array_equal(sp.densify(), t)


def test_kept_entries_scaled_by_inverse_p():                # :62-70
    t = O.random_tensor([6, 6, 6], 41)
    sp = O.sparsify(O.Dense(t), 0.5, 7)
    idx, vals = sp.entries()
    assert 0 < len(idx) < t.size
    assert np.array_equal(vals * 0.5, t.reshape(-1, order="F")[idx])


def test_zero_entries_never_emitted():                      # :72-79
    t = np.zeros((3, 3))
    t[1, 1] = 4.0
    t[2, 0] = -2.5
    sp = O.sparsify(O.Dense(t), 1.0, 0)
    assert sp.nnz == 2
    assert np.array_equal(sp.densify(), t)


def test_pure_function_of_tensor_p_seed():                  # :81-87
    t = O.Dense(O.random_tensor([7, 5, 4], 42))
    a, b = O.sparsify(t, 0.3, 1234).entries(), O.sparsify(t, 0.3, 1234).entries()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    c = O.sparsify(t, 0.3, 1235).entries()
    assert not (len(a[0]) == len(c[0]) and np.array_equal(a[0], c[0]))


def test_unbiased():                                        # :89-106
    t = O.random_tensor([3, 3, 3], 43)
    d = O.Dense(t)
    p, trials = 0.1, 2000
    sums = np.zeros(t.size)
    for s in range(trials):
        idx, vals = O.sparsify(d, p, s).entries()
        sums[idx] += vals
    x = t.reshape(-1, order="F")
    se = np.abs(x) * math.sqrt((1 - p) / (p * trials))
    assert np.all(np.abs(sums / trials - x) <= 3 * se)


def test_binomial_counts():                                 # :108-123
    t = O.Dense(O.random_tensor([20, 20, 20], 44))
    n, p, z = 8000.0, 0.1, 3.8906
    sd = math.sqrt(n * p * (1 - p))
    for s in range(100):
        nnz = O.sparsify(t, p, 5000 + s).nnz
        assert n * p - z * sd <= nnz <= n * p + z * sd


def test_p_validation():                                    # :125-131
    t = O.Dense(O.random_tensor([3, 3], 45))
    for p in (0.0, -0.2, 1.5, float("nan")):
        with pytest.raises(O.ArgumentError):
            O.sparsify(t, p, 0)


def _same_model(a, b):
    return (np.array_equal(a.core, b.core) and all(np.array_equal(x, y) for x, y in zip(a.factors, b.factors))
            and a.fit == b.fit and a.sweep_fits == b.sweep_fits and a.iterations == b.iterations)


def test_keep_everything_pipelines_bitwise():              # :133-142
    t = O.Dense(O.random_tensor([6, 7, 8], 46))
    m, sp = O.mach_hosvd(t, [2, 3, 2], 1.0, 31)
    assert _same_model(m, O.hosvd(t, [2, 3, 2])) and sp.nnz == 336
    m2, _ = O.mach_hooi(t, [2, 3, 2], 1.0, 31)
    assert _same_model(m2, O.hooi(t, [2, 3, 2]))


def test_pipelines_decompose_returned_tensor():             # :144-154
    t = O.Dense(O.random_tensor([8, 9, 10], 47))
    m, sp = O.mach_hosvd(t, [2, 2, 2], 0.15, 77)
    assert _same_model(m, O.hosvd(sp, [2, 2, 2]))
    m2, sp2 = O.mach_hooi(t, [2, 2, 2], 0.15, 77)
    assert _same_model(m2, O.hooi(sp2, [2, 2, 2]))


def cauchy(n):
    i = np.arange(1, n + 1)
    return 1.0 / (i[:, None, None] + i[None, :, None] + i[None, None, :])


def test_accuracy_increases_with_p():                       # :156-172
    t = cauchy(30)
    d = O.Dense(t)
    means = []
    for p in (0.05, 0.1, 0.3, 1.0):
        acc = [O.accuracy(d, O.mach_hooi(d, [3, 3, 3], p, s)[0]) for s in range(10)]
        means.append(sum(acc) / 10)
    assert all(means[i] <= means[i + 1] + 1e-9 for i in range(3))
    assert means[-1] > 0.99


# ---------------------------------------------------------------------------
# proj/tests/test_tucker.cpp restated
# ---------------------------------------------------------------------------
def separable3(a, b, c, scale, seed):
    # unit vectors from mt19937_64 normal streams seeded seed, seed+1, seed+2
    u = O.random_matrix(a, 1, seed)[:, 0]
    v = O.random_matrix(b, 1, seed + 1)[:, 0]
    w = O.random_matrix(c, 1, seed + 2)[:, 0]
    u, v, w = u / np.sqrt((u * u).sum()), v / np.sqrt((v * v).sum()), w / np.sqrt((w * w).sum())
    return scale * np.einsum("i,j,k->ijk", u, v, w)


def exact_rank_tensor(dims, ranks, seed):
    t = O.random_tensor(ranks, seed)
    for m, (n, r) in enumerate(zip(dims, ranks)):
        u = O.random_orthogonal(n, seed + 11 * (m + 1))[:, :r]
        t = O.mode_product(O.Dense(t), u, m)
    return t


def random_sparse(dims, nnz, seed):
    total = int(np.prod(dims))
    rng = np.random.default_rng(seed)
    idx = rng.choice(total, size=nnz, replace=False)
    return O.Sparse.from_entries(dims, idx, rng.standard_normal(nnz))


def test_separable_rank_one():                              # :162-171
    t = separable3(4, 5, 6, 7.0, 21)
    d = O.Dense(t)
    m = O.hosvd(d, [1, 1, 1])
    assert abs(abs(m.core.reshape(-1)[0]) - 7.0) < 1e-12
    assert O.accuracy(d, m) >= 1 - 1e-10 and m.fit >= 1 - 1e-10
    assert np.abs(O.reconstruct(m) - t).max() < 1e-12
    assert m.warnings == []


def test_full_rank_reproduces():                            # :173-179
    t = O.random_tensor([4, 3, 5], 33)
    d = O.Dense(t)
    m = O.hosvd(d, [4, 3, 5])
    assert O.accuracy(d, m) >= 1 - 1e-10
    for f in m.factors:
        assert np.abs(f.T @ f - np.eye(f.shape[1])).max() < 1e-10


def test_hosvd_matches_jacobi_gram_oracle():                # :181-191
    t = O.random_tensor([6, 7, 8], 5)
    d = O.Dense(t)
    ranks = [2, 3, 4]
    m = O.hosvd(d, ranks)
    for mode in range(3):
        x = O.matricize(d, mode)
        ev, vec = O.jacobi_eig(x @ x.T)
        assert O.subspace_gap(m.factors[mode], vec[:, : ranks[mode]]) < 1e-8


def test_hosvd_warns_and_completes():                       # :193-204
    t = separable3(4, 5, 6, 3.0, 9)
    m = O.hosvd(O.Dense(t), [2, 2, 2])
    assert len(m.warnings) == 3
    assert "mode 1" in m.warnings[0] and "mode 3" in m.warnings[2]
    assert m.fit >= 1 - 1e-10


def test_sparse_hosvd_matches_dense():                      # :206-217
    st = random_sparse([8, 9, 10], 70, 123)
    dt = O.Dense(st.densify())
    a, b = O.hosvd(st, [3, 3, 3]), O.hosvd(dt, [3, 3, 3])
    for x, y in zip(a.factors, b.factors):
        assert np.abs(x - y).max() < 1e-10
    assert np.abs(a.core - b.core).max() < 1e-10 and abs(a.fit - b.fit) < 1e-12


def test_sparse_hosvd_tall_mode():                          # :219-231
    st = random_sparse([30, 4, 5], 60, 77)
    dt = O.Dense(st.densify())
    a, b = O.hosvd(st, [3, 2, 2]), O.hosvd(dt, [3, 2, 2])
    for x, y in zip(a.factors, b.factors):
        assert np.abs(x - y).max() < 1e-9
    assert abs(a.fit - b.fit) < 1e-12


def test_densify_switch_bitwise():                          # :233-239
    st = random_sparse([4, 5, 6], 40, 15)
    dt = O.Dense(st.densify())
    assert _same_model(O.hosvd(st, [2, 2, 2]), O.hosvd(dt, [2, 2, 2]))
    assert _same_model(O.hooi(st, [2, 2, 2]), O.hooi(dt, [2, 2, 2]))


def test_hooi_exact_low_rank_one_sweep():                   # :241-248
    t = exact_rank_tensor([6, 7, 8], [2, 2, 2], 3)
    m = O.hooi(O.Dense(t), [2, 2, 2])
    assert m.iterations == 1 and abs(m.fit - 1) < 1e-10 and len(m.sweep_fits) == 2


def test_hooi_monotone():                                   # :250-263
    d = O.Dense(O.random_tensor([6, 7, 8], 42))
    base = O.hosvd(d, [2, 2, 2])
    m = O.hooi(d, [2, 2, 2], 50, 0.0)
    assert m.fit >= base.fit - 1e-12 and m.sweep_fits[0] == base.fit
    assert m.iterations == len(m.sweep_fits) - 1
    assert all(b >= a - 1e-12 for a, b in zip(m.sweep_fits, m.sweep_fits[1:]))
    assert abs(m.fit - O.accuracy(d, m)) < 1e-12


def test_hooi_stop_rule():                                  # :265-272
    d = O.Dense(O.random_tensor([6, 7, 8], 42))
    assert O.hooi(d, [2, 2, 2], 50, 0.5).iterations == 1
    c = O.hooi(d, [2, 2, 2], 2, 0.0)
    assert c.iterations <= 2 and len(c.sweep_fits) == c.iterations + 1


def test_sparse_hooi_matches_dense():                       # :274-286
    st = random_sparse([8, 9, 10], 70, 123)
    dt = O.Dense(st.densify())
    a, b = O.hooi(st, [2, 2, 2]), O.hooi(dt, [2, 2, 2])
    assert a.iterations == b.iterations
    for x, y in zip(a.factors, b.factors):
        assert np.abs(x - y).max() < 1e-9
    assert abs(a.fit - b.fit) < 1e-12 and abs(a.fit - O.accuracy(dt, a)) < 1e-12


def test_order_one():                                       # :288-300
    d = O.Dense(O.random_tensor([9], 77))
    assert O.hosvd(d, [1]).fit >= 1 - 1e-10
    assert len(O.hosvd(d, [3]).warnings) == 1
    h = O.hooi(d, [2])
    assert h.iterations == 1 and h.fit >= 1 - 1e-10


def test_validation():                                      # :385-393
    d = O.Dense(O.random_tensor([4, 5, 6], 2))
    for r in ([0, 2, 2], [2, 2, 7]):
        with pytest.raises(O.ArgumentError):
            O.hosvd(d, r)
    with pytest.raises(O.ArgumentError):
        O.hooi(d, [2, 2, 2], 0, 1e-4)
    with pytest.raises(O.ArgumentError):
        O.hooi(d, [2, 2, 2], 10, -1.0)
    with pytest.raises(O.ArgumentError):
        O.hooi(d, [2, 2, 2], 10, float("nan"))


def test_random_shapes():                                   # :395-418 (numpy-drawn shapes)
    rng = np.random.default_rng(2024)
    for trial in range(10):
        order = int(rng.integers(1, 5))
        dims = [int(rng.integers(2, 8)) for _ in range(order)]
        ranks = [1 + int(rng.integers(0, d)) for d in dims]
        d = O.Dense(O.random_tensor(dims, 900 + trial))
        m = O.hosvd(d, ranks)
        for f in m.factors:
            assert np.abs(f.T @ f - np.eye(f.shape[1])).max() < 1e-10
        assert abs(m.fit - O.accuracy(d, m)) < 1e-12


# ---------------------------------------------------------------------------
# eigensolver / linalg pins (test_linalg.cpp, acceptance.cpp:366-388)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n", [1, 2, 5, 17, 64, 130])
def test_sym_eig_vs_numpy(n):
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n))
    a = a + a.T
    ev, vec = O.sym_eig(a)
    ev2 = np.linalg.eigh(a)[0]
    assert np.abs(ev - ev2).max() < 1e-12 * max(1, np.abs(ev2).max()) * n
    assert np.abs(vec.T @ vec - np.eye(n)).max() < 1e-12 * n
    assert np.abs(a @ vec - vec * ev).max() < 1e-12 * n * np.abs(ev).max()


def test_rank_k_error_matches_jacobi():                     # acceptance.cpp:366-388
    rng = np.random.default_rng(41)
    for i in range(20):
        rows, cols = 2 + int(rng.integers(0, 29)), 2 + int(rng.integers(0, 39))
        a = O.random_matrix(rows, cols, 1000 + i)
        k = 1 + int(rng.integers(0, max(1, min(rows, cols) - 1)))
        err = np.sqrt(((a - O.low_rank_approx(a, k)) ** 2).sum())
        g = a @ a.T if rows <= cols else a.T @ a
        sv = np.sqrt(np.maximum(0, O.jacobi_eig(g)[0]))
        want = np.sqrt((sv[k:] ** 2).sum())
        assert abs(err - want) <= 1e-8 * max(want, 1e-12)


def test_left_basis_zero_and_completion():                  # test_linalg.cpp:221-244
    b, sv, nr, comp = O.left_singular_basis(np.zeros((4, 3)), 4)
    assert nr == 0 and comp and np.abs(b.T @ b - np.eye(4)).max() < 1e-12
    b, sv, nr, comp = O.left_singular_basis(O.random_matrix(6, 9, 515), 3)
    assert nr == 3 and not comp


def test_sparse_row_gram_is_xxt():
    st = random_sparse([7, 6, 5], 60, 3)
    x = O.matricize(O.Dense(st.densify()), 1)
    assert np.abs(O.sparse_row_gram(st, 1) - x @ x.T).max() < 1e-12


def test_mode_product_vs_einsum():                          # test_tensor.cpp:160-169, :218-235
    t = O.random_tensor([3, 4, 5], 7)
    m = O.random_matrix(6, 4, 8)
    y = O.mode_product(O.Dense(t), m, 1)
    assert np.abs(y - np.einsum("ijk,qj->iqk", t, m)).max() < 1e-12
    st = random_sparse([3, 4, 5], 12, 9)
    ys = O.mode_product(st, m, 1)
    assert np.abs(ys - np.einsum("ijk,qj->iqk", st.densify(), m)).max() < 1e-12
