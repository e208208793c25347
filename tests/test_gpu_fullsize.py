"""Parity at the BASELINE configs' full sizes (north_star bars, fp32):
the whole kept-index array bit for bit and the kept values equal to the
reference's fp64 x/p rounded once to fp32 (sampling.cpp:21-31); factors with
the largest principal-angle sine <= 1e-3; core (after sign alignment) and fit
within 1e-4 relative; equal iterations and sweep_fits (tucker.cpp:80-106).

The device input comes from the same on-device generator as bench.py (C2:
512^3, ranks 10, p = 0.05; C3: 128x128x64x256, ranks 8, p = 0.02; C5: 1024^3,
ranks 16, p in {0.01, 0.001}); the oracle runs on the same values promoted to
fp64.  The oracle is single-threaded and recomputes every fit by a dense
reconstruction (tucker.cpp:56-64), so these tests take ~0.5-2 minutes each.
"""
import numpy as np
import pytest

import oracle as O
from paper_0909_4969_b200.synth import CONFIGS, KIND, lowrank_torch
from tests.helpers import align_core, rel, subspace_sin

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mb():
    import paper_0909_4969_b200 as mb
    return mb


def run_case(mb, config, p=None, sweeps=None, seed_data=2, seed_mach=7):
    import torch

    dims, ranks, noise, p0, sweeps0, dtype = CONFIGS[config]
    p = p0 if p is None else p
    sweeps = sweeps0 if sweeps is None else sweeps
    x = lowrank_torch(dims, ranks, noise, seed=seed_data, dtype=dtype, device="cuda", kind=KIND.get(config))
    torch.cuda.synchronize()  # the library runs on its own stream
    ctx = mb.Context(0)
    t = mb.DenseTensor.from_torch(x, dims, ctx)
    res = mb.mach_hooi(t, ranks, mb.SparsifyConfig(p, seed_mach), mb.HooiConfig(sweeps, 0.0), ctx=ctx)
    idx, vals = res.sparsified.entries()
    res.sparsified.free()
    xh = x.cpu().numpy().astype(np.float64)  # flat, first mode fastest
    del t, x
    torch.cuda.empty_cache()
    ref, ref_sp = O.mach_hooi(O.Dense(xh, dims), ranks, p, seed_mach, sweeps, 0.0)
    del xh
    oi, ov = ref_sp.entries()
    return res.model, idx, vals, ref, oi, ov


def check(model, idx, vals, ref, oi, ov):
    assert np.array_equal(idx, oi), "kept-index set differs"
    assert np.array_equal(vals.astype(np.float32), ov.astype(np.float32)), "kept values differ"
    # tucker.cpp:102's stop rule at tolerance 0 fires on the first fit
    # decrease; at convergence the fp32 fit moves by rounding (~1e-7), so the
    # two runs may stop a sweep apart — accepted only when the shorter run
    # stopped on such a rounding-level change.  The shared sweeps must agree.
    n = min(len(model.sweep_fits), len(ref.sweep_fits))
    assert np.allclose(model.sweep_fits[:n], ref.sweep_fits[:n], rtol=1e-4, atol=0)
    if model.iterations != ref.iterations:
        short = model if model.iterations < ref.iterations else ref
        k = short.iterations
        assert abs(short.sweep_fits[k] - short.sweep_fits[k - 1]) <= 1e-6, (model.sweep_fits, ref.sweep_fits)
        return
    assert abs(model.fit - ref.fit) <= 1e-4 * abs(ref.fit)
    sines = [subspace_sin(fd, fr) for fd, fr in zip(model.factors, ref.factors)]
    assert max(sines) <= 1e-3, sines
    assert rel(align_core(model.core, model.factors, ref.factors), ref.core) <= 1e-4
    assert model.warnings == ref.warnings
    return sines


def test_c2_full_size_parity(mb):
    model, idx, vals, ref, oi, ov = run_case(mb, "c2")
    assert len(idx) > 6_700_000
    check(model, idx, vals, ref, oi, ov)


def test_c3_full_size_parity(mb):
    model, idx, vals, ref, oi, ov = run_case(mb, "c3", sweeps=3)
    assert len(idx) > 5_300_000
    check(model, idx, vals, ref, oi, ov)


@pytest.mark.parametrize("p", [0.01, 0.001])
def test_c5_full_size_parity(mb, p):
    model, idx, vals, ref, oi, ov = run_case(mb, "c5", p=p, sweeps=2)
    check(model, idx, vals, ref, oi, ov)
