"""The drop-in boundary on the GPU: the C++ mirror of the reference headers
driven by a reference-style caller (tests/cpp/api_smoke.cpp), and the
truncated-SVD family (linalg.hpp:11-30) against the CPU oracle's restatement
of linalg.cpp:196-317.  fp64 inputs: subspaces to 1e-10, values to 1e-10
relative, factors column by column (the sign rule fixes them)."""
import os
import subprocess

import numpy as np
import pytest

import oracle as O
from paper_0909_4969_b200 import _lib

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def mb():
    import paper_0909_4969_b200 as mb
    return mb


def test_cxx_mirror_reference_style_caller_runs():
    src = os.path.join(ROOT, "tests", "cpp", "api_smoke.cpp")
    exe = os.path.join(ROOT, "tests", "cpp", "api_smoke")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), src, "-o", exe, _lib.LIB_PATH,
                    f"-Wl,-rpath,{os.path.dirname(_lib.LIB_PATH)}"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "api_smoke: 0 failures" in r.stdout


def lowrank_matrix(rows, cols, rank, seed, noise=1e-3):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((rows, rank)) @ rng.standard_normal((rank, cols)) + noise * rng.standard_normal((rows, cols))


@pytest.mark.parametrize("rows,cols,k", [(40, 300, 5), (300, 40, 6), (64, 64, 10), (17, 23, 17), (600, 90, 8)])
def test_truncated_svd_matches_oracle(mb, rows, cols, k):
    a = lowrank_matrix(rows, cols, max(k, 3), rows * cols + k)
    dev = mb.truncated_svd(a, k)
    ref_l, ref_s, ref_r = O.truncated_svd(a, k)
    assert np.abs(dev.singular_values - ref_s).max() <= 1e-10 * ref_s[0]
    # well-separated values: columns equal up to rounding (signs fixed by the rule)
    gaps = np.abs(np.diff(ref_s)) / ref_s[0]
    if gaps.min() > 1e-6:
        assert np.abs(dev.left - ref_l).max() <= 1e-8
        assert np.abs(dev.right - ref_r).max() <= 1e-8
    assert np.abs(dev.left.T @ dev.left - np.eye(k)).max() <= 1e-12
    assert np.abs(dev.right.T @ dev.right - np.eye(k)).max() <= 1e-12
    assert np.array_equal(mb.leading_left_singular_vectors(a, k), dev.left)
    lr = mb.low_rank_approx(a, k)
    assert np.abs(lr - O.low_rank_approx(a, k)).max() <= 1e-9 * np.abs(a).max()


def test_truncated_svd_rank_deficient_and_zero(mb):
    a = lowrank_matrix(30, 50, 2, 3, noise=0.0)  # rank 2, ask for 4
    dev = mb.truncated_svd(a, 4)
    ref_l, ref_s, ref_r = O.truncated_svd(a, 4)
    assert np.abs(dev.singular_values[:2] - ref_s[:2]).max() <= 1e-10 * ref_s[0]
    assert np.abs(dev.singular_values[2:]).max() <= 1e-6 * ref_s[0]
    assert np.abs(dev.left.T @ dev.left - np.eye(4)).max() <= 1e-12
    assert np.abs(dev.right.T @ dev.right - np.eye(4)).max() <= 1e-12
    z = mb.truncated_svd(np.zeros((5, 7)), 3)  # zero_matrix_svd, linalg.cpp:196-207
    assert np.array_equal(z.left, np.eye(5)[:, :3]) and np.array_equal(z.right, np.eye(7)[:, :3])
    assert np.array_equal(z.singular_values, np.zeros(3))


def test_truncated_svd_argument_errors(mb):
    with pytest.raises(mb.ArgumentError):
        mb.truncated_svd(np.ones((4, 6)), 5)
    with pytest.raises(mb.ArgumentError):
        mb.low_rank_approx(np.ones((4, 6)), 0)


@pytest.mark.parametrize("dims,p", [((9, 7, 11), 0.3), ((5, 6, 4, 7), 0.2), ((40, 1, 33), 0.1)])
def test_sparse_mode_product_bit_exact(mb, dims, p):
    """mode_product(SparseTensor) straight from the nonzeros, in the reference's
    summation order (tensor.cpp:241-259): bit-identical to the oracle."""
    rng = np.random.default_rng(len(dims) * 100 + dims[0])
    x = rng.standard_normal(dims)
    sp_ref = O.sparsify(O.Dense(x), p, 5)
    idx, vals = sp_ref.entries()
    sp = mb.SparseTensor.from_entries(dims, idx, vals)
    for mode in range(len(dims)):
        m = rng.standard_normal((3, dims[mode]))
        got = mb.mode_product(sp, m, mode)
        ref = O.mode_product(sp_ref, m, mode)
        assert got.shape == ref.shape
        assert np.array_equal(got, ref), np.abs(got - ref).max()


@pytest.mark.parametrize("rows,cols,k", [(256, 900, 16), (130, 400, 8), (300, 2000, 10)])
def test_left_singular_basis_large_gram_matches_oracle(mb, rows, cols, k):
    """Row Grams of 130-300 rows exceed one CTA's shared memory: the
    cluster-distributed eigensolver (eig_cluster.cuh) takes them."""
    a = lowrank_matrix(rows, cols, k + 4, rows + cols, noise=1e-2)
    dev = mb.left_singular_basis(a, k)
    ref_b, ref_s, ref_nr, ref_c = O.left_singular_basis(a, k)
    assert np.abs(dev.singular_values - ref_s).max() <= 1e-10 * ref_s[0]
    r = dev.basis - ref_b @ (ref_b.T @ dev.basis)
    assert np.linalg.norm(r, 2) <= 1e-9


def test_next_row_mirrors_reference_style_caller_runs(tmp_path):
    """bounds / ingest (+ sample-on-arrival) / tensor files / CLI through the C++ mirror (tests/cpp/ext_smoke.cpp)."""
    src = os.path.join(ROOT, "tests", "cpp", "ext_smoke.cpp")
    exe = os.path.join(ROOT, "tests", "cpp", "ext_smoke")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), src, "-o", exe, _lib.LIB_PATH,
                    f"-Wl,-rpath,{os.path.dirname(_lib.LIB_PATH)}"], check=True)
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "ext_smoke: 0 failures" in r.stdout
