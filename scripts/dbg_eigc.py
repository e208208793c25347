import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0909_4969_b200 as mb
rng = np.random.default_rng(0)
for rows, k in ((256, 16), (130, 8), (64, 8)):
    a = rng.standard_normal((rows, k + 4)) @ rng.standard_normal((k + 4, 3 * rows)) + 1e-2 * rng.standard_normal((rows, 3 * rows))
    b = mb.left_singular_basis(a, k)
    print(rows, k, b.singular_values[:3], flush=True)
