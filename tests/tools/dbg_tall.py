import os, numpy as np
os.environ["MACH_TALL_MIN_COLS"]="48"; os.environ["MACH_DEBUG_TALL"]="1"
import oracle as O, paper_0909_4969_b200 as mb
from paper_0909_4969_b200.synth import lowrank_numpy
from tests.helpers import subspace_sin
dims, ranks = (10, 6, 400), (3, 2, 5)
x = lowrank_numpy(dims, ranks, 0.02, seed=11, kind="stream")
for deg in ["1", "8"]:
    res = mb.mach_hosvd(x, ranks, mb.SparsifyConfig(0.3, 7))
    ref, ref_sp = O.mach_hosvd(O.Dense(x), ranks, 0.3, 7)
    print([subspace_sin(a, b) for a, b in zip(res.model.factors, ref.factors)])
    # direct: leading left singular vectors of X_(2)
    idx, vals = res.sparsified.entries()
    d = np.zeros(int(np.prod(dims))); d[idx] = vals
    X2 = d.reshape(dims, order="F").transpose(2, 0, 1).reshape(400, -1, order="F")
    u, s, vt = np.linalg.svd(X2, full_matrices=False)
    print("svals", s[:8])
    print("dev vs svd", subspace_sin(res.model.factors[2], u[:, :5]), "ref vs svd", subspace_sin(ref.factors[2], u[:, :5]))
    break
