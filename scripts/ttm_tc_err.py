"""Accuracy of the tcgen05 3xTF32 mode product vs fp64 as the contracted length grows."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_0909_4969_b200 as mb
rng = np.random.default_rng(0)
for mode in (0, 1):
    for L in (64, 256, 1024, 4096):
        dims = (L, 256, 64) if mode == 0 else (256, L, 64)
        x = rng.standard_normal(dims).astype(np.float32) + 0.5  # nonzero mean: partial sums grow
        m = rng.standard_normal((16, L)) / np.sqrt(L) + 1.0 / L
        got = mb.mode_product(mb.DenseTensor.from_numpy(x), m, mode)
        ref = np.moveaxis(np.tensordot(m, x.astype(np.float64), axes=([1], [mode])), 0, mode)
        err = got - ref
        print(f"mode {mode} L {L}: max rel err {np.abs(err).max() / np.abs(ref).max():.2e}  mean signed err / mean|ref| {err.mean() / np.abs(ref).mean():+.2e}")
