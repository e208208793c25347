"""Per-kernel device times of one HOSVD initialisation (session setup) of a config."""
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
mb.HooiSession(sp, ranks).free()  # warm-up
ctx.synchronize()
mb.profile(ctx, True)
s = mb.HooiSession(sp, ranks)
ctx.synchronize()
st = mb.kernel_stats(ctx)
mb.profile(ctx, False)
tot = sum(v[1] for v in st.values())
print(f"total device ms (serialised events) {tot:.3f}")
for k, v in sorted(st.items(), key=lambda kv: -kv[1][1])[:int(os.environ.get("TOPK", "20"))]:
    print(f"{k[:60]:60s} n={v[0]:4d} ms={v[1]:.4f} ms/launch={v[1] / max(1, v[0]):.4f}")
