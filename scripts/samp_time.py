"""Sampler timing: sample_kernel device time (library profiler) per config, median of 7."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0909_4969_b200 as mb  # noqa: E402
from paper_0909_4969_b200.synth import CONFIGS, lowrank_torch  # noqa: E402

peak = 6536.7
try:
    peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    pass
cfgs = sys.argv[1:] or ["c2", "c5", "c5p01", "c5p001"]
ctx = mb.Context(0)
for name in cfgs:
    dims, ranks, noise, p, _, dtype = CONFIGS[name]
    x = lowrank_torch(dims, ranks, noise, seed=2, dtype=dtype)
    t = mb.DenseTensor.from_torch(x, dims, ctx)
    vs = 4 if dtype == "float32" or str(dtype).endswith("32") else 8
    ms = []
    nnz = 0
    for it in range(8):
        mb.profile(ctx, True)
        sp = mb.sparsify(t, mb.SparsifyConfig(p, 7))
        ctx.synchronize()
        st = mb.kernel_stats(ctx)
        mb.profile(ctx, False)
        nnz = sp.nnz
        sp.free()
        k = [v for kname, v in st.items() if "sample" in kname]
        if it:
            ms.append(k[0][1] / k[0][0])
    ms.sort()
    med = ms[len(ms) // 2]
    numel = math.prod(dims)
    byt = numel * vs + nnz * (4 + vs)
    print(json.dumps({"config": name, "p": p, "nnz": nnz, "ms": round(med, 4), "min_ms": round(ms[0], 4),
                      "GB_s": round(byt / med / 1e6, 1), "frac": round(byt / med / 1e6 / peak, 3)}), flush=True)
    t.free()
    del x
    torch.cuda.empty_cache()
