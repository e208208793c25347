"""C5 p = 1 dense route timing (HOSVD + sweeps) with per-kernel device ms."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0909_4969_b200 as mb  # noqa: E402
from paper_0909_4969_b200.synth import lowrank_torch  # noqa: E402

dims = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1024,1024,1024").split(","))
ranks = tuple(int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "16,16,16").split(","))
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
x = lowrank_torch(dims, ranks, 0.01, seed=2)
ctx = mb.Context(0)
t = mb.DenseTensor.from_torch(x, dims, ctx)
mb.profile(ctx, True)
s = mb.HooiSession(t, ranks, ctx)
st0 = mb.kernel_stats(ctx)
s.step(sweeps, -1.0)
ctx.synchronize()
st1 = mb.kernel_stats(ctx)
m = s.model()
sweep_k = {k: round((v[1] - st0.get(k, (0, 0.0))[1]) / sweeps, 4) for k, v in st1.items() if v[1] - st0.get(k, (0, 0.0))[1] > 0}
print(json.dumps({"dims": dims, "ranks": ranks, "hosvd_ms": m.times["hosvd_ms"], "sweep_ms": m.times["sweep_ms"],
                  "fits": m.sweep_fits, "hosvd_kernels_ms": {k: round(v[1], 3) for k, v in st0.items()},
                  "sweep_kernels_ms": sweep_k}))
