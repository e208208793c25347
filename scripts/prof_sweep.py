"""Profiling driver: one config, setup + HOSVD + a few HOOI sweeps (for ncu)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_0909_4969_b200 as mb  # noqa: E402
from paper_0909_4969_b200.synth import CONFIGS, lowrank_torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--sweeps", type=int, default=3)
a = ap.parse_args()
dims, ranks, noise, p, _, dtype = CONFIGS[a.config]
x = lowrank_torch(dims, ranks, noise, seed=2, dtype=dtype)
ctx = mb.Context(0)
t = mb.DenseTensor.from_torch(x, dims, ctx)
sp = mb.sparsify(t, mb.SparsifyConfig(p, 7))
s = mb.HooiSession(sp, ranks)
s.step(a.sweeps, -1.0)
ctx.synchronize()
print("nnz", sp.nnz, "fit", s.fit)
