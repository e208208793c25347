import numpy as np, torch
import oracle as O, paper_0909_4969_b200 as mb
from paper_0909_4969_b200.synth import CONFIGS, KIND, lowrank_torch
dims, ranks, noise, p, sweeps, dtype = CONFIGS["c3"]
x = lowrank_torch(dims, ranks, noise, seed=2, dtype=dtype, device="cuda")
ctx = mb.Context(0)
t = mb.DenseTensor.from_torch(x, dims, ctx)
s = mb.sparsify(t, mb.SparsifyConfig(p, 7), ctx=ctx)
idx, vals = s.entries()
xh = x.cpu().numpy().astype(np.float64)
oi, ov = O.sparsify(O.Dense(xh, dims), p, 7).entries()
d = np.setxor1d(idx, oi)
print("diff", d, len(idx), len(oi))
for i in d:
    h = O.counter_hash64(7, int(i))
    T = int(np.ceil(p * 2**53))
    print(i, "x=", xh[i], repr(np.float32(xh[i])), "h>>11=", h >> 11, "T=", T, "u=", O.counter_uniform01(7, int(i)), "in gpu", i in set(idx.tolist()), "tie_hi", (h >> 32) == ((T << 11) >> 32))
