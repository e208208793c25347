"""Tall-mode basis: a mode taller than the product
of the others takes the column side in the reference (sparse_kernels.cpp:82-89,
linalg.cpp:335-352).  Past `MACH_TALL_MIN_COLS` columns (4096 by default: C4's
time mode has 64000) the device replaces the column Gram by an implicit
subspace iteration on X_(n) X_(n)^T (tall_basis.cu, linalg.cpp:128-193
semantics).  These tests lower the threshold so the path runs at shapes the
oracle (which always forms the column Gram) finishes in seconds.
"""
import numpy as np
import pytest

import oracle as O
from paper_0909_4969_b200.synth import lowrank_numpy
from tests.helpers import align_core, rel, subspace_sin

pytestmark = pytest.mark.gpu


@pytest.fixture()
def mb(monkeypatch):
    import paper_0909_4969_b200 as mb
    monkeypatch.setenv("MACH_TALL_MIN_COLS", "48")
    return mb


def test_tall_hosvd_fp64_matches_oracle(mb):
    dims, ranks = (10, 6, 400), (3, 2, 5)  # X_(2): 400 x 60 -> tall path
    x = lowrank_numpy(dims, ranks, 0.02, seed=11, kind="stream")
    res = mb.mach_hosvd(x, ranks, mb.SparsifyConfig(0.3, 7))
    ref, ref_sp = O.mach_hosvd(O.Dense(x), ranks, 0.3, 7)
    assert np.array_equal(res.sparsified.entries()[0], ref_sp.entries()[0])
    m = res.model
    for fd, fr in zip(m.factors, ref.factors):
        assert subspace_sin(fd, fr) <= 1e-9
        assert np.abs(fd.T @ fd - np.eye(fd.shape[1])).max() < 1e-10
    assert rel(align_core(m.core, m.factors, ref.factors), ref.core) <= 1e-9
    assert abs(m.fit - ref.fit) <= 1e-9
    assert m.warnings == ref.warnings


def test_tall_hooi_fp64_matches_oracle(mb):
    dims, ranks = (12, 5, 360), (3, 2, 6)
    x = lowrank_numpy(dims, ranks, 0.05, seed=5, kind="stream")
    res = mb.mach_hooi(x, ranks, mb.SparsifyConfig(0.2, 3), mb.HooiConfig(3, 0.0))
    ref, _ = O.mach_hooi(O.Dense(x), ranks, 0.2, 3, 3, 0.0)
    m = res.model
    n = min(len(m.sweep_fits), len(ref.sweep_fits))
    assert np.abs(np.array(m.sweep_fits[:n]) - np.array(ref.sweep_fits[:n])).max() <= 1e-9
    for fd, fr in zip(m.factors, ref.factors):
        assert subspace_sin(fd, fr) <= 1e-9


def test_tall_fp32_c4_shape_matches_oracle(mb):
    """C4's generator (lognormal host loads, daily harmonics) at 40 x 8 x 2048,
    ranks (10, 6, 20), p = 0.05: the time mode (2048 > 320) takes the tall path."""
    dims, ranks = (40, 8, 2048), (10, 6, 20)
    x = lowrank_numpy(dims, ranks, 0.05, seed=4, dtype=np.float32, kind="stream")
    res = mb.mach_hooi(mb.DenseTensor.from_numpy(x), ranks, mb.SparsifyConfig(0.05, 7), mb.HooiConfig(3, 0.0))
    ref, ref_sp = O.mach_hooi(O.Dense(x.astype(np.float64)), ranks, 0.05, 7, 3, 0.0)
    assert np.array_equal(res.sparsified.entries()[0], ref_sp.entries()[0])
    m = res.model
    assert m.iterations == ref.iterations
    for fd, fr in zip(m.factors, ref.factors):
        assert subspace_sin(fd, fr) <= 1e-3
    assert rel(align_core(m.core, m.factors, ref.factors), ref.core) <= 1e-4
    assert np.allclose(m.sweep_fits, ref.sweep_fits, rtol=1e-4, atol=0)


def test_tall_dense_route_matches_oracle(mb):
    """Dense HOSVD with a tall mode (column side past the threshold)."""
    dims, ranks = (7, 8, 300), (2, 3, 4)
    x = lowrank_numpy(dims, ranks, 0.01, seed=9)
    dev = mb.hosvd(x, ranks)
    ref = O.hosvd(O.Dense(x), ranks)
    for fd, fr in zip(dev.factors, ref.factors):
        assert subspace_sin(fd, fr) <= 1e-9
    assert abs(dev.fit - ref.fit) <= 1e-9
