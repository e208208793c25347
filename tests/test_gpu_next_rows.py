"""SURVEY §8(f) rows 2-4 on the GPU, through the C ABI, against the oracle.

(f)3 Theorem-1 bound (bounds.cpp:152-184): every field of the report within
     1e-9 relative of the oracle in fp64 (full device spectra), exact flags,
     exact amplitude; the reference's own known answers (test_bounds.cpp).
(f)2 streaming sample-on-arrival ingest: the streamed kept set equals
     sparsify() of the whole tensor bit for bit for ragged slab sizes, device
     and host slabs; HOOI on the streamed tensor equals the one-shot result;
     device record binning equals the oracle's ingest bit for bit.
(f)4 binary tensor files: value-exact round trips, malformed files rejected.
"""
import os

import numpy as np
import pytest

import oracle as O
from paper_0909_4969_b200.synth import lowrank_numpy

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mb():
    import paper_0909_4969_b200 as mb
    return mb


# ---------------------------------------------------------------- (f)3 bound
@pytest.mark.parametrize("dims,ranks,p,seed", [((7, 6, 5), (2, 3, 2), 0.35, 9), ((40, 30, 50), (4, 3, 5), 0.2, 3),
                                               ((12, 10, 8, 6), (2, 3, 2, 2), 0.5, 1), ((90, 4, 3), (3, 2, 2), 0.4, 5)])
def test_bound_matches_oracle_fp64(mb, dims, ranks, p, seed):
    x = lowrank_numpy(dims, ranks, 0.05, seed=seed) if len(dims) == 3 and dims[0] > 10 else O.random_tensor(dims, 62)
    X = O.Dense(x)
    ref = O.theorem1_bound(X, O.sparsify(X, p, seed), ranks, p)
    xd = mb.DenseTensor.from_numpy(x)
    sp = mb.sparsify(xd, mb.SparsifyConfig(p, seed))
    dev = mb.theorem1_bound(xd, sp, ranks, p)
    assert dev["b"] == ref["b"] and dev["p"] == ref["p"]
    for k in ("p_min", "success_probability", "t"):
        assert dev[k] == pytest.approx(ref[k], rel=1e-9), k
    for k in ("dims_large_enough", "dims_balanced", "p_above_min", "conditions_met"):
        assert dev[k] == ref[k]
    scale = np.linalg.norm(x)
    for md, mr in zip(dev["per_mode"], ref["per_mode"]):
        assert md["rank"] == mr["rank"]
        for k in ("x_residual", "xhat_residual", "x_lowrank_norm", "t_i"):
            assert abs(md[k] - mr[k]) <= 1e-9 * max(scale, abs(mr[k])), (k, md[k], mr[k])


def test_bound_reference_known_answers(mb):
    # full rank, unsampled: both residuals exactly zero (test_bounds.cpp:112-126)
    x = O.random_tensor((10, 12, 9), 60)
    xd = mb.DenseTensor.from_numpy(x)
    rep = mb.theorem1_bound(xd, mb.sparsify(xd, mb.SparsifyConfig(1.0, 1)), (10, 12, 9), 1.0)
    for m in rep["per_mode"]:
        assert m["x_residual"] == 0.0 and m["xhat_residual"] == 0.0 and m["t_i"] > 0.0
    assert rep["t"] == min(m["t_i"] for m in rep["per_mode"])
    assert not rep["dims_large_enough"] and not rep["conditions_met"]
    # amplitude from the original tensor (test_bounds.cpp:128-136)
    y = np.clip(O.random_tensor((6, 6, 6), 61), -3.0, 3.0)
    y[2, 4, 1] = -3.7
    yd = mb.DenseTensor.from_numpy(y)
    assert mb.theorem1_bound(yd, mb.sparsify(yd, mb.SparsifyConfig(0.5, 2)), (2, 2, 2), 0.5)["b"] == 3.7
    # validation (test_bounds.cpp:254-264)
    wrong = mb.sparsify(mb.DenseTensor.from_numpy(O.random_tensor((6, 6, 7), 1)), mb.SparsifyConfig(0.5, 1))
    ok = mb.sparsify(yd, mb.SparsifyConfig(0.5, 1))
    with pytest.raises(mb.ShapeError):
        mb.theorem1_bound(yd, wrong, (2, 2, 2), 0.5)
    for ranks, p in [((2, 2, 9), 0.5), ((0, 2, 2), 0.5), ((2, 2, 2), 0.0), ((2, 2, 2), 1.2)]:
        with pytest.raises(mb.ArgumentError):
            mb.theorem1_bound(yd, ok, ranks, p)


def test_bound_fp32_monitoring_shape(mb):
    """C1-like fp32 tensor: measured MACH-HOSVD error sits under the bound; fp32 parity 1e-5 relative."""
    dims, ranks, p = (100, 12, 256), (5, 5, 5), 0.1
    x = lowrank_numpy(dims, ranks, 0.01, seed=11).astype(np.float32)
    xd = mb.DenseTensor.from_numpy(x)
    res = mb.mach_hosvd(xd, ranks, mb.SparsifyConfig(p, 7))
    rep = mb.theorem1_bound(xd, res.sparsified, ranks, p)
    X = O.Dense(x.astype(np.float64))
    idx, vals = res.sparsified.entries()
    ref = O.theorem1_bound(X, O.Sparse.from_entries(dims, idx, vals), ranks, p)
    assert rep["t"] == pytest.approx(ref["t"], rel=1e-5)
    for md, mr in zip(rep["per_mode"], ref["per_mode"]):
        assert md["x_residual"] == pytest.approx(mr["x_residual"], rel=1e-5)
        assert md["xhat_residual"] == pytest.approx(mr["xhat_residual"], rel=1e-5)
    measured = (1.0 - mb.accuracy(xd, res.model)) * float(np.linalg.norm(x.astype(np.float64)))
    assert measured <= rep["t"]


# --------------------------------------------------------------- (f)2 stream
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("slabs", [[1, 7, 0, 24, 3, 29], [64], [5] * 12 + [4]])
def test_stream_equals_offline_sampler(mb, dtype, slabs):
    dims, p, seed = (37, 11, sum(slabs)), 0.13, 21
    x = lowrank_numpy(dims, (3, 3, 3), 0.05, seed=8).astype(dtype)
    ref_idx, ref_val = O.sparsify(O.Dense(x.astype(np.float64)), p, seed).entries()
    for host in (True, False):
        st = mb.SampleStream(dims[:2] + (dims[2] + 5,), mb.SparsifyConfig(p, seed), dtype=dtype)
        t0 = 0
        for n in slabs:
            slab = np.asfortranarray(x[:, :, t0:t0 + n])
            if host:
                st.append(slab)
            elif n > 0:
                st.append(mb.DenseTensor.from_numpy(slab))
            t0 += n
            if n and t0 < dims[2]:  # the prefix property holds at every point of the stream
                i_now, _ = st.tensor().entries()
                assert np.array_equal(i_now, ref_idx[ref_idx < 37 * 11 * t0])
        sp = st.tensor()
        idx, val = sp.entries()
        assert sp.dims == dims and st.state() == (dims[2], len(ref_idx))
        assert np.array_equal(idx, ref_idx)
        if dtype == np.float64:
            assert np.array_equal(val, ref_val)
        else:
            assert np.array_equal(val, (x.reshape(-1, order="F")[ref_idx] * np.float32(1.0 / p)).astype(np.float64)) or \
                np.allclose(val, ref_val, rtol=3e-7)
        st.free()


def test_stream_hooi_matches_one_shot(mb):
    dims, ranks, p, seed = (60, 12, 200), (4, 3, 5), 0.2, 5
    x = lowrank_numpy(dims, ranks, 0.02, seed=2)
    st = mb.SampleStream(dims, mb.SparsifyConfig(p, seed), dtype=np.float64)
    for t0 in range(0, 200, 40):
        st.append(np.asfortranarray(x[:, :, t0:t0 + 40]))
    got = mb.hooi(st.tensor(), ranks, mb.HooiConfig(3, 0.0))
    ref, _ = O.mach_hooi(O.Dense(x), ranks, p, seed, 3, 0.0)
    assert got.iterations == ref.iterations
    assert abs(got.fit - ref.fit) <= 1e-9
    for fd, fr in zip(got.factors, ref.factors):
        assert np.linalg.norm(fd - fr @ (fr.T @ fd), 2) <= 1e-9
    with pytest.raises(mb.ShapeError):
        st.append(np.zeros((60, 12, 1)))  # capacity exceeded


def test_stream_validation(mb):
    with pytest.raises(mb.ArgumentError):
        mb.SampleStream((5,), mb.SparsifyConfig(0.5, 1))
    with pytest.raises(mb.ArgumentError):
        mb.SampleStream((5, 5), mb.SparsifyConfig(0.0, 1))
    st = mb.SampleStream((4, 3, 10), mb.SparsifyConfig(0.5, 1))
    with pytest.raises(mb.ShapeError):
        st.tensor()  # no ticks yet
    with pytest.raises(mb.ShapeError):
        st.append(mb.DenseTensor.from_numpy(np.zeros((4, 2, 1), dtype=np.float32)))
    with pytest.raises(mb.ArgumentError):
        st.append(np.full((4, 3, 1), np.nan, dtype=np.float32))
        st.state()  # host slabs are sampled when the next call needs them


@pytest.mark.parametrize("carry", [False, True])
def test_record_ingest_matches_oracle(mb, carry):
    rng = np.random.default_rng(4)
    M, J, T, bucket = 9, 4, 48, 300
    n = 3000
    machine = rng.integers(0, M, n)
    metric = rng.integers(0, J, n)
    ts = rng.integers(0, T * bucket, n)
    ts[:2] = [0, T * bucket - 1]  # span every bucket
    gaps = rng.random(n) < 0.35
    gaps[:2] = False
    machine, metric, ts = machine[~gaps], metric[~gaps], ts[~gaps]
    value = rng.standard_normal(len(ts)) * 10.0 ** rng.integers(-3, 12, len(ts))  # cancellation-prone
    ref, first = O.ingest_indexed(machine, metric, ts, value, M, J, bucket, carry_forward=carry)
    assert ref.shape == (M, J, T) and first == 0
    st = mb.SampleStream((M, J, T), mb.SparsifyConfig(1.0, 3), dtype=np.float64)
    tick = ts // bucket
    got = []
    for t0, t1 in [(0, 5), (5, 6), (6, 30), (30, 48)]:  # ragged time slabs; state carries across them
        sel = (tick >= t0) & (tick < t1)
        perm = rng.permutation(int(sel.sum()))  # arrival order must not matter
        st.append_records(machine[sel][perm], metric[sel][perm], (tick[sel] - t0)[perm], value[sel][perm], t1 - t0, carry)
        got.append(st.last_slab().numpy())
    dev = np.concatenate(got, axis=2)
    assert np.array_equal(dev, ref)
    idx, val = st.tensor().entries()  # p = 1: every nonzero cell kept (sampling.cpp:21-31)
    assert np.array_equal(val, ref.reshape(-1, order="F")[idx])
    with pytest.raises(mb.ArgumentError):
        st2 = mb.SampleStream((M, J, 4), mb.SparsifyConfig(1.0, 3), dtype=np.float64)
        st2.append_records([0], [0], [7], [1.0], 2)


def test_record_ingest_reference_known_answers(mb):
    # test_io.cpp:202-209 (duplicates average), :262-283 (missing policy), :211-226 (order invariance)
    st = mb.SampleStream((1, 1, 1), mb.SparsifyConfig(1.0, 1), dtype=np.float64)
    st.append_records([0, 0], [0, 0], [0, 0], [4.0, 6.0], 1)
    assert st.last_slab().numpy()[0, 0, 0] == 5.0
    st = mb.SampleStream((1, 2, 3), mb.SparsifyConfig(1.0, 1), dtype=np.float64)
    st.append_records([0, 0, 0], [0, 0, 1], [0, 2, 1], [2.0, 8.0, 5.0], 3, carry_forward=True)
    c = st.last_slab().numpy()
    assert c[0, 0, 1] == 2.0 and c[0, 0, 2] == 8.0 and c[0, 1, 0] == 0.0 and c[0, 1, 2] == 5.0
    rec = [(0, 0, 0, 1e16), (0, 0, 0, 1.0), (0, 0, 0, -1e16), (0, 0, 0, 2.0), (0, 0, 0, 0.125), (1, 0, 0, -7.5),
           (0, 1, 0, 3.25), (1, 1, 0, 2.5), (1, 1, 0, 2.5)]
    base = None
    rng = np.random.default_rng(77)
    for trial in range(6):
        perm = rng.permutation(len(rec))
        m, j, t, v = zip(*[rec[i] for i in perm])
        st = mb.SampleStream((2, 2, 1), mb.SparsifyConfig(1.0, 1), dtype=np.float64)
        st.append_records(m, j, t, v, 1)
        cur = st.last_slab().numpy().tobytes()
        base = base or cur
        assert cur == base
    ref, _ = O.ingest_indexed(*zip(*[(m, j, 5, v) for m, j, _, v in rec]), 2, 2, 100)
    assert base == np.asfortranarray(ref).tobytes()


# ------------------------------------------------------------ (f)4 binary I/O
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_binary_round_trip(mb, tmp_path, dtype):
    dims = (33, 17, 29)
    x = lowrank_numpy(dims, (3, 3, 3), 0.1, seed=6).astype(dtype)
    xd = mb.DenseTensor.from_numpy(x)
    sp = mb.sparsify(xd, mb.SparsifyConfig(0.2, 4))
    pd, ps = str(tmp_path / "x.machb"), str(tmp_path / "s.machb")
    mb.save_tensor(xd, pd)
    mb.save_tensor(sp, ps)
    assert os.path.getsize(pd) == 72 + x.size * x.itemsize
    info = mb.tensor_file_info(ps)
    assert info["kind"] == "sparse" and info["dims"] == dims and info["count"] == sp.nnz and info["dtype"] == np.dtype(dtype)
    xr, sr = mb.load_tensor(pd), mb.load_tensor(ps)
    assert isinstance(xr, mb.DenseTensor) and xr.numpy().tobytes() == np.asfortranarray(x).tobytes()
    i0, v0 = sp.entries()
    i1, v1 = sr.entries()
    assert np.array_equal(i0, i1) and np.array_equal(v0, v1)
    # the loaded tensors drive the decomposition exactly like the originals
    a = mb.hooi(sp, (3, 3, 3), mb.HooiConfig(2, 0.0))
    b = mb.hooi(sr, (3, 3, 3), mb.HooiConfig(2, 0.0))
    assert a.fit == b.fit


def test_binary_rejects_malformed(mb, tmp_path):
    with pytest.raises(mb.IoError):
        mb.load_tensor(str(tmp_path / "missing.machb"))
    bad = tmp_path / "bad.machb"
    bad.write_bytes(b"not a tensor file at all, just text padded past the header size ......................")
    with pytest.raises(mb.ParseError):
        mb.load_tensor(str(bad))
    x = mb.DenseTensor.from_numpy(np.arange(24, dtype=np.float64).reshape(2, 3, 4))
    good = tmp_path / "good.machb"
    mb.save_tensor(x, str(good))
    (tmp_path / "trunc.machb").write_bytes(good.read_bytes()[:-8])
    with pytest.raises(mb.ParseError):
        mb.load_tensor(str(tmp_path / "trunc.machb"))
    sp = mb.SparseTensor.from_entries((2, 3, 4), [1, 5, 9], [1.0, 2.0, 3.0])
    mb.save_tensor(sp, str(tmp_path / "s.machb"))
    raw = bytearray((tmp_path / "s.machb").read_bytes())
    raw[72:76], raw[76:80] = raw[76:80], raw[72:76]  # swap two indices: no longer ascending
    (tmp_path / "unsorted.machb").write_bytes(bytes(raw))
    with pytest.raises(mb.ParseError):
        mb.load_tensor(str(tmp_path / "unsorted.machb"))
    with pytest.raises(mb.IoError):
        mb.save_tensor(x, str(tmp_path / "no_such_dir" / "x.machb"))


def test_stream_wide_capacity_narrows_indices(mb):
    """A stream whose capacity exceeds 2^32 elements stores 64-bit indices; a
    snapshot that still fits 32 bits is narrowed to the canonical u32 layout
    and equals the offline sampler's kept set."""
    lead, ticks, p, seed = (2048, 128), 6, 0.05, 9
    rng = np.random.default_rng(1)
    x = rng.standard_normal(lead + (ticks,)).astype(np.float32)
    st = mb.SampleStream(lead + (20000,), mb.SparsifyConfig(p, seed), dtype=np.float32)  # 5.2e9 > 2^32
    st.append(np.asfortranarray(x[:, :, :4]))
    st.append(mb.DenseTensor.from_numpy(np.asfortranarray(x[:, :, 4:])))
    sp = st.tensor()
    idx, val = sp.entries()
    ref_idx, _ = O.sparsify(O.Dense(x.astype(np.float64)), p, seed).entries()
    assert sp.dims == lead + (ticks,) and np.array_equal(idx, ref_idx)
    m = mb.hosvd(sp, (3, 3, 2))
    assert m.fit == m.fit  # the narrowed tensor drives the decomposition


def test_cli_decomposes_fp32_binary_in_place(mb, tmp_path):
    """(f)4: an fp32 MACHB2 file goes file -> HBM -> mach-hooi in its stored
    precision (no fp64 host round trip); the CLI's model equals the API's."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cli = os.path.join(root, "paper_0909_4969_b200", "mach_b200")
    dims, ranks, p, seed = (64, 48, 80), (4, 3, 5), 0.3, 6
    x = lowrank_numpy(dims, ranks, 0.02, seed=12).astype(np.float32)
    xd = mb.DenseTensor.from_numpy(x)
    src = str(tmp_path / "x.machb")
    mb.save_tensor(xd, src)
    out, sp_path = str(tmp_path / "model"), str(tmp_path / "s.machb")
    r = subprocess.run([cli, "mach-hooi", "--input", src, "--ranks", ",".join(map(str, ranks)), "--p", str(p), "--seed", str(seed),
                        "--max-iters", "3", "--fit-tol", "0", "--output", out, "--sparsified", sp_path],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    ref = mb.mach_hooi(xd, ranks, mb.SparsifyConfig(p, seed), mb.HooiConfig(3, 0.0))
    meta = dict(ln.split(":", 1) for ln in open(os.path.join(out, "metadata")).read().splitlines() if ":" in ln)
    assert float(meta["fit"]) == ref.model.fit and int(meta["iterations"]) == ref.model.iterations
    info = mb.tensor_file_info(sp_path)
    assert info["kind"] == "sparse" and info["dtype"] == np.dtype(np.float32) and info["count"] == ref.sparsified.nnz
    i0, v0 = mb.load_tensor(sp_path).entries()
    i1, v1 = ref.sparsified.entries()
    assert np.array_equal(i0, i1) and np.array_equal(v0, v1)
    # exit codes (cli.hpp:9-14): data error for a missing file, usage error for a bad p
    assert subprocess.run([cli, "hosvd", "--input", str(tmp_path / "none"), "--ranks", "2,2,2", "--output", out]).returncode == 3
    assert subprocess.run([cli, "sparsify", "--input", src, "--p", "0", "--output", sp_path], capture_output=True).returncode == 2
