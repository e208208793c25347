"""Sampler kernel time at the configs (CUDA events around the kernel via the
library's profiling mode) and the HBM fraction: (numel*s + nnz*(4+s)) / t."""
import json, math, sys
import torch
import paper_0909_4969_b200 as mb
from paper_0909_4969_b200.synth import CONFIGS, KIND, lowrank_torch
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if __import__("os").path.exists("MEASURED_PEAKS.json") else 6456.8
for cfg, p in [("c2", None), ("c5", 0.1), ("c5", 0.01), ("c4", None)]:
    dims, ranks, noise, p0, _, dtype = CONFIGS[cfg]
    p = p0 if p is None else p
    x = lowrank_torch(dims, ranks, noise, seed=2, dtype=dtype, kind=KIND.get(cfg))
    ctx = mb.Context(0)
    t = mb.DenseTensor.from_torch(x, dims, ctx)
    mb.sparsify(t, mb.SparsifyConfig(p, 8), ctx=ctx).free()
    ms = []
    for rep in range(5):
        mb.profile(ctx, True)
        s = mb.sparsify(t, mb.SparsifyConfig(p, 7), ctx=ctx)
        st = mb.kernel_stats(ctx)
        mb.profile(ctx, False)
        nnz = s.nnz
        s.free()
        ms.append(sum(v[1] for k, v in st.items() if "sample_kernel" in k))
    kms = min(ms)
    vs = 4 if dtype == "float32" else 8
    by = math.prod(dims) * vs + nnz * (4 + vs)
    print(json.dumps({"config": cfg, "p": p, "nnz": nnz, "kernel_ms": round(kms, 4), "GB_s": round(by / kms / 1e6, 1),
                      "frac": round(by / kms / 1e6 / peak, 3)}), flush=True)
    del t, x
    torch.cuda.empty_cache()
