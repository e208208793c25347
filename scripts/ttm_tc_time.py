"""Time the tcgen05 dense mode product (ttm_tc.cu) alone at C5 size."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_0909_4969_b200 as mb
dims = (1024, 1024, 1024)
x = torch.randn(int(np.prod(dims)), device="cuda", dtype=torch.float32)
ctx = mb.Context(0)
t = mb.DenseTensor.from_torch(x, dims, ctx)
m = np.random.default_rng(0).standard_normal((16, 1024))
for mode in (0, 1):
    mb.mode_product(t, m, mode, ctx=ctx, keep_on_device=True).free()
    mb.profile(ctx, True)
    for _ in range(3):
        mb.mode_product(t, m, mode, ctx=ctx, keep_on_device=True).free()
    st = mb.kernel_stats(ctx)
    mb.profile(ctx, False)
    k = [v for n, v in st.items() if "ttm_tc" in n][0]
    ms = k[1] / k[0]
    print(f"mode {mode}: {ms:.3f} ms  {4.295e9 / ms / 1e6:.0f} GB/s")
