"""Profiling driver: the C2 sampler twice (for ncu -k sample_kernel -s 1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0909_4969_b200 as mb  # noqa: E402
from paper_0909_4969_b200.synth import CONFIGS, lowrank_torch  # noqa: E402

dims, ranks, noise, p, _, dtype = CONFIGS["c2"]
x = lowrank_torch(dims, ranks, noise, seed=2, dtype=dtype)
ctx = mb.Context(0)
t = mb.DenseTensor.from_torch(x, dims, ctx)
for _ in range(2):
    mb.sparsify(t, mb.SparsifyConfig(p, 7)).free()
ctx.synchronize()
print("ok")
