"""Per-kernel device times of a few HOOI sweeps of one config (profiling on)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0909_4969_b200 as mb  # noqa: E402
from paper_0909_4969_b200.synth import CONFIGS, lowrank_torch  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
dims, ranks, noise, p, _, dtype = CONFIGS[cfg]
x = lowrank_torch(dims, ranks, noise, seed=2, dtype=dtype)
ctx = mb.Context(0)
t = mb.DenseTensor.from_torch(x, dims, ctx)
sp = mb.sparsify(t, mb.SparsifyConfig(p, 7))
s = mb.HooiSession(sp, ranks)
s.step(2, -1.0)
ctx.synchronize()
mb.profile(ctx, True)
s.step(4, -1.0)
ctx.synchronize()
st = mb.kernel_stats(ctx)
mb.profile(ctx, False)
tag = os.environ.get("MACH_TTM_W", "-")
for k, v in sorted(st.items(), key=lambda kv: -kv[1][1])[:int(os.environ.get("TOPK", "3"))]:
    print(f"W={tag:>3} {k[:50]:50s} n={v[0]:4d} ms/launch={v[1] / max(1, v[0]):.4f}")
