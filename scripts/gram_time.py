"""Time the tcgen05 dense mode Gram (gram_tc.cu) at C5 (1024^3 fp32) with CUDA
events (library profiling: per-kernel device ms on the library's stream)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0909_4969_b200 as mb  # noqa: E402

dims = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1024,1024,1024").split(","))
reps = 3
x = torch.randn(int(np.prod(dims)), device="cuda", dtype=torch.float32)
ctx = mb.Context(0)
t = mb.DenseTensor.from_torch(x, dims, ctx)
out = {"dims": dims}
peak_tf32 = json.load(open("MEASURED_PEAKS.json"))["bf16_tflops"] / 2 if os.path.exists("MEASURED_PEAKS.json") else 821.0
for m in range(len(dims)):
    mb.mode_gram(t, m)  # warm-up
    mb.profile(ctx, True)
    for _ in range(reps):
        g, tc = mb.mode_gram(t, m)
    st = mb.kernel_stats(ctx)
    mb.profile(ctx, False)
    kern = {k: v[1] / v[0] for k, v in st.items()}
    main = [v for k, v in kern.items() if "gram_tc_kernel" in k or "gram_kernel" in k or "gram_mma" in k]
    ms = main[0] if main else float("nan")
    flops = 2.0 * dims[m] * np.prod(dims)  # full Gram (algorithmic, as SURVEY 8d)
    out[f"mode{m}"] = {"tensor_cores": tc, "kernel_ms": ms, "all_ms": kern,
                       "tflops_full": flops / ms / 1e9, "frac_of_tf32_peak": flops / ms / 1e9 / peak_tf32}
print(json.dumps(out))
