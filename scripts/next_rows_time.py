"""Timing of the SURVEY 8(f) rows on one B200: streaming sample-on-arrival ingest
(host slabs from pinned memory vs the PCIe copy alone; device-resident slabs vs
the one-shot sampler), device record binning, the Theorem-1 bound, binary files.
Prints one JSON line per measurement."""
import json
import math
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0909_4969_b200 as mb  # noqa: E402
from paper_0909_4969_b200.synth import lowrank_torch  # noqa: E402

ctx = mb.Context(0)


def out(**kw):
    print(json.dumps(kw), flush=True)


def wall(fn, reps=3):
    best = 1e30
    for _ in range(reps):
        ctx.synchronize()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ctx.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


# ---- stream: monitoring-shaped tensor 1000 x 64 x T fp32 (C4's leading dims), p = 0.01 ----
M, J, T, slab_t, p = 1000, 64, 8192, 512, 0.01
x = lowrank_torch((M, J, T), (10, 6, 20), 0.05, seed=2, dtype="float32")  # flat, first mode fastest
host = x.cpu().pin_memory()
dense = mb.DenseTensor.from_torch(x, (M, J, T), ctx)
cfg = mb.SparsifyConfig(p, 7)
one_shot = wall(lambda: mb.sparsify(dense, cfg).free())
ref = mb.sparsify(dense, cfg)
ref_idx, _ = ref.entries()
slab_elems = M * J * slab_t


def stream_host():
    st = mb.SampleStream((M, J, T), cfg, dtype=np.float32, ctx=ctx)
    for t0 in range(0, T, slab_t):
        st.append_host_ptr(host.data_ptr() + 4 * M * J * t0, slab_t)
    st.state()
    return st


def stream_dev():
    st = mb.SampleStream((M, J, T), cfg, dtype=np.float32, ctx=ctx)
    for t0 in range(0, T, slab_t):
        v = x[M * J * t0:M * J * (t0 + slab_t)]
        st.append(mb.DenseTensor.from_torch(v, (M, J, slab_t), ctx))
    st.state()
    return st


st = stream_host()
idx, _ = st.tensor().entries()
assert np.array_equal(idx, ref_idx), "streamed kept set differs from the one-shot sampler"
st.free()
dev_buf = torch.empty_like(x)
def copy_all():
    dev_buf.copy_(host, non_blocking=True)
    torch.cuda.synchronize()


copy_only = wall(copy_all)
t_host = wall(lambda: stream_host().free())
t_dev = wall(lambda: stream_dev().free())
gb = x.numel() * 4 / 1e9
out(what="stream_ingest", dims=[M, J, T], slab_ticks=slab_t, p=p, nnz=int(len(ref_idx)), GB=round(gb, 3),
    one_shot_sampler_ms=round(one_shot * 1e3, 3), host_slabs_ms=round(t_host * 1e3, 3),
    host_slabs_GBps=round(gb / t_host, 1), h2d_copy_only_ms=round(copy_only * 1e3, 3),
    h2d_copy_only_GBps=round(gb / copy_only, 1), frac_of_pcie_copy=round(copy_only / t_host, 3),
    device_slabs_ms=round(t_dev * 1e3, 3), device_slabs_GBps=round(gb / t_dev, 1),
    kept_set="equal to the one-shot sampler's")
del dev_buf, host

# ---- record binning: 1000 x 64 x 288 buckets, 3 records per cell ----
rng = np.random.default_rng(1)
Tb = 288
n = M * J * Tb * 3
machine = rng.integers(0, M, n).astype(np.int32)
metric = rng.integers(0, J, n).astype(np.int32)
tick = rng.integers(0, Tb, n).astype(np.int32)
value = rng.standard_normal(n)


def bin_records():
    s2 = mb.SampleStream((M, J, Tb), mb.SparsifyConfig(0.1, 3), dtype=np.float32, ctx=ctx)
    s2.append_records(machine, metric, tick, value, Tb, carry_forward=True)
    s2.state()
    s2.free()


t_bin = wall(bin_records)
out(what="record_ingest", records=n, cells=M * J * Tb, ms=round(t_bin * 1e3, 2), Mrecords_per_s=round(n / t_bin / 1e6, 1),
    note="wall clock incl. the 20 B/record host->device copy from pageable memory")

# ---- Theorem-1 bound ----
for name, dims, ranks, pp, dtype in [("c1", (100, 12, 1024), (5, 5, 5), 0.1, "float64"),
                                     ("c2", (512, 512, 512), (10, 10, 10), 0.05, "float32")]:
    xx = lowrank_torch(dims, ranks, 0.01, seed=2, dtype=dtype)
    d = mb.DenseTensor.from_torch(xx, dims, ctx)
    sp = mb.sparsify(d, mb.SparsifyConfig(pp, 7))
    rep = None

    def run():
        global rep
        rep = mb.theorem1_bound(d, sp, ranks, pp, ctx=ctx)

    t_b = wall(run, reps=2)
    out(what="theorem1_bound", config=name, dims=list(dims), ms=round(t_b * 1e3, 2), t=rep["t"], b=rep["b"],
        x_residual=[m["x_residual"] for m in rep["per_mode"]], conditions_met=rep["conditions_met"])
    del xx

# ---- binary files ----
with tempfile.TemporaryDirectory() as tmp:
    pth = os.path.join(tmp, "x.machb")
    t_save = wall(lambda: mb.save_tensor(dense, pth), reps=1)
    t_load = wall(lambda: mb.load_tensor(pth, ctx).free(), reps=2)
    out(what="binary_file", GB=round(gb, 3), save_ms=round(t_save * 1e3, 1), load_ms=round(t_load * 1e3, 1),
        load_GBps=round(gb / t_load, 2), note="tmpfs/page-cache file; 64 MiB pinned chunks")
