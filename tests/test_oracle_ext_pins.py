"""Pins of the oracle's §8(f) restatements (oracle/oracle_ext.cpp) against the
reference's own known answers: proj/tests/test_bounds.cpp (closed forms,
full-rank residuals exactly zero, amplitude from the original tensor, the
assembly re-evaluated independently with numpy, the p-halving identity, the
measured error under the bound) and proj/tests/test_io.cpp:187-345 (ingest)."""
import math

import numpy as np
import pytest

import oracle as O


def _split(a, r):
    s = np.linalg.svd(a, compute_uv=False)
    return math.sqrt((s[:r] ** 2).sum()), math.sqrt((s[r:] ** 2).sum())


def _unfold(x, m):
    return np.moveaxis(x, m, 0).reshape(x.shape[m], -1, order="F")


def test_min_sampling_probability_closed_form():  # test_bounds.cpp:82-109
    dims = (10, 20, 30)
    terms = []
    for j in range(3):
        others = [d for k, d in enumerate(dims) if k != j]
        terms.append((8.0 * sum(math.log(d) for d in others)) ** 4 / math.prod(others))
    assert O.min_sampling_probability(dims) == pytest.approx(max(terms), rel=1e-12)
    assert O.min_sampling_probability(dims) > 1.0
    for bad in [(5,), (5, 1), ()]:
        with pytest.raises(O.ArgumentError):
            O.min_sampling_probability(bad)


def test_full_rank_bound_isolates_amplitude_terms():  # test_bounds.cpp:112-126
    x = O.random_tensor((10, 12, 9), 60)
    X = O.Dense(x)
    rep = O.theorem1_bound(X, O.sparsify(X, 1.0, 1), (10, 12, 9), 1.0)
    for m in rep["per_mode"]:
        assert m["x_residual"] == 0.0 and m["xhat_residual"] == 0.0 and m["t_i"] > 0.0
    assert rep["t"] == min(m["t_i"] for m in rep["per_mode"])
    assert not rep["dims_large_enough"] and not rep["p_above_min"] and not rep["conditions_met"]


def test_amplitude_from_original():  # test_bounds.cpp:128-136
    x = np.clip(O.random_tensor((6, 6, 6), 61), -3.0, 3.0)
    x[2, 4, 1] = -3.7
    X = O.Dense(x)
    assert O.theorem1_bound(X, O.sparsify(X, 0.5, 2), (2, 2, 2), 0.5)["b"] == 3.7


def test_bound_assembly_independent():  # test_bounds.cpp:138-183
    x = O.random_tensor((7, 6, 5), 62)
    p, ranks = 0.35, (2, 3, 2)
    X = O.Dense(x)
    sp = O.sparsify(X, p, 9)
    xh = sp.densify()
    rep = O.theorem1_bound(X, sp, ranks, p)
    b = np.abs(x).max()
    assert rep["b"] == b and rep["p"] == p
    hres = [_split(_unfold(xh, j), ranks[j])[1] for j in range(3)]
    ts = []
    for i in range(3):
        low, res = _split(_unfold(x, i), ranks[i])
        m = rep["per_mode"][i]
        assert m["rank"] == ranks[i]
        assert m["x_residual"] == pytest.approx(res, rel=1e-9)
        assert m["x_lowrank_norm"] == pytest.approx(low, rel=1e-9)
        assert m["xhat_residual"] == pytest.approx(hres[i], rel=1e-9)
        ratio = ranks[i] / p * math.prod(d for k, d in enumerate(x.shape) if k != i)
        ts.append(res + 4 * b * math.sqrt(ratio) + 4 * math.sqrt(low * b) * ratio ** 0.25 + sum(hres) - hres[i])
        assert m["t_i"] == pytest.approx(ts[-1], rel=1e-9)
    assert rep["t"] == pytest.approx(min(ts), rel=1e-9)


def test_halving_p():  # test_bounds.cpp:185-203
    x = O.random_tensor((8, 7, 6), 63)
    X = O.Dense(x)
    sp = O.sparsify(X, 0.4, 3)
    full = O.theorem1_bound(X, sp, (2, 2, 2), 0.4)
    half = O.theorem1_bound(X, sp, (2, 2, 2), 0.2)
    for i in range(3):
        m = full["per_mode"][i]
        ratio = m["rank"] / 0.4 * math.prod(d for k, d in enumerate(x.shape) if k != i)
        t2 = 4 * full["b"] * math.sqrt(ratio)
        t3 = 4 * math.sqrt(m["x_lowrank_norm"] * full["b"]) * ratio ** 0.25
        pred = (math.sqrt(2) - 1) * t2 + (2 ** 0.25 - 1) * t3
        assert half["per_mode"][i]["t_i"] - m["t_i"] == pytest.approx(pred, rel=1e-10)
        assert half["per_mode"][i]["x_residual"] == m["x_residual"]


def test_measured_error_under_bound():  # test_bounds.cpp:205-215
    x = O.random_tensor((12, 12, 12), 64)
    X = O.Dense(x)
    for s in range(4):
        model, sp = O.mach_hosvd(X, (3, 3, 3), 0.3, s)
        rep = O.theorem1_bound(X, sp, (3, 3, 3), 0.3)
        assert (1.0 - O.accuracy(X, model)) * np.linalg.norm(x) <= rep["t"]


def test_conditions_and_validation():  # test_bounds.cpp:217-264
    big = (200, 200, 200)
    pmin = O.min_sampling_probability(big)
    x = O.random_tensor((4, 4, 4), 1)
    X = O.Dense(x)
    ok = O.sparsify(X, 0.5, 1)
    wrong = O.sparsify(O.Dense(O.random_tensor((4, 4, 5), 1)), 0.5, 1)
    with pytest.raises(O.ShapeError):
        O.theorem1_bound(X, wrong, (2, 2, 2), 0.5)
    for ranks, p in [((2, 2), 0.5), ((2, 2, 9), 0.5), ((0, 2, 2), 0.5), ((2, 2, 2), 0.0), ((2, 2, 2), 1.2)]:
        with pytest.raises(O.ArgumentError):
            O.theorem1_bound(X, ok, ranks, p)
    shape = O.theorem1_conditions((4, 4, 4), 0.5)
    full = O.theorem1_bound(X, ok, (2, 2, 2), 0.5)
    for k in ("p", "p_min", "success_probability", "dims_large_enough", "dims_balanced", "p_above_min", "conditions_met"):
        assert shape[k] == full[k]
    assert shape["per_mode"] == [] and shape["b"] == 0.0 and shape["t"] == 0.0
    assert pmin > 0


# ---- ingest (test_io.cpp:187-345) ----
def test_ingest_single_series_and_duplicates():
    t, first = O.ingest_indexed([0, 0, 0], [0, 0, 0], [1000, 1060, 1120], [1.0, 2.0, 3.0], 1, 1, 60)
    assert t.shape == (1, 1, 3) and list(t[0, 0]) == [1.0, 2.0, 3.0] and first == 960
    t, _ = O.ingest_indexed([0, 0], [0, 0], [10, 20], [4.0, 6.0], 1, 1, 100)
    assert t.shape == (1, 1, 1) and t[0, 0, 0] == 5.0
    t, first = O.ingest_indexed([0, 0], [0, 0], [-10, 10], [1.0, 2.0], 1, 1, 60)
    assert t.shape == (1, 1, 2) and first == -60 and list(t[0, 0]) == [1.0, 2.0]


def test_ingest_order_invariant():
    rec = [(0, 0, 5, 1e16), (0, 0, 15, 1.0), (0, 0, 25, -1e16), (0, 0, 35, 2.0), (0, 0, 45, 0.125), (1, 0, 12, -7.5),
           (0, 1, 22, 3.25), (1, 1, 91, 2.5), (1, 1, 33, 2.5)]
    base, _ = O.ingest_indexed(*zip(*rec), 2, 2, 100)
    rng = np.random.default_rng(77)
    for _ in range(20):
        perm = rng.permutation(len(rec))
        sh, _ = O.ingest_indexed(*zip(*[rec[i] for i in perm]), 2, 2, 100)
        assert sh.tobytes() == base.tobytes()


def test_ingest_missing_policy():
    rec = [(0, 0, 0, 2.0), (0, 0, 200, 8.0), (0, 1, 100, 5.0)]
    z, _ = O.ingest_indexed(*zip(*rec), 1, 2, 100)
    assert z[0, 0, 1] == 0.0 and z[0, 1, 0] == 0.0 and z[0, 1, 2] == 0.0
    c, _ = O.ingest_indexed(*zip(*rec), 1, 2, 100, carry_forward=True)
    assert c[0, 0, 1] == 2.0 and c[0, 0, 2] == 8.0 and c[0, 1, 0] == 0.0 and c[0, 1, 2] == 5.0
    with pytest.raises(O.ArgumentError):
        O.ingest_indexed([0], [0], [0], [float("nan")], 1, 1, 60)
    with pytest.raises(O.ArgumentError):
        O.ingest_indexed([0], [0], [0], [1.0], 1, 1, 0)
