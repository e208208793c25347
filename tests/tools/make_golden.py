"""Generate tests/golden/ fixtures from the pinned CPU oracle.

  python tests/tools/make_golden.py

Inputs are regenerated deterministically from mt19937_64 streams
(oracle.random_tensor), so only the small outputs are stored: sampler kept
sets (flat indices + x/p as hex bit patterns) and a small MACH-HOOI model
(factors up to sign, core, sweep fits).  The oracle itself is pinned in
tests/test_oracle_pins.py; these fixtures let the GPU tests compare against
stored vectors as well as against a live oracle run.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")

SAMPLER = [  # (dims, p, seed, tensor seed)
    ((4, 3, 2), 0.5, 7, 17),
    ((37, 41, 13), 0.3, 12345, 17),
    ((64, 64, 64), 0.05, 2**63 + 11, 17),
    ((4097,), 0.9, 3, 17),
]

HOOI = [  # (dims, ranks, p, seed, sweeps, tensor seed)
    ((30, 20, 25), (4, 3, 5), 0.2, 7, 3, 29),
    ((100, 12, 64), (5, 5, 5), 0.1, 7, 3, 31),
]


def main():
    os.makedirs(OUT, exist_ok=True)
    cases = []
    for dims, p, seed, ts in SAMPLER:
        x = O.random_tensor(list(dims), ts)
        x.reshape(-1, order="F")[::7] = 0.0
        idx, vals = O.sparsify(O.Dense(x), p, seed).entries()
        cases.append({"dims": list(dims), "p": p, "seed": str(seed), "tensor_seed": ts, "zero_every": 7,
                      "idx": idx.tolist(), "vals_hex": [f"{v:016x}" for v in vals.view(np.uint64)]})
    with open(os.path.join(OUT, "sampler.json"), "w") as f:
        json.dump({"generator": "tests/tools/make_golden.py", "cases": cases}, f)
    models = []
    for dims, ranks, p, seed, sweeps, ts in HOOI:
        x = O.random_tensor(list(dims), ts)
        m, sp = O.mach_hooi(O.Dense(x), list(ranks), p, seed, sweeps, 0.0)
        models.append({"dims": list(dims), "ranks": list(ranks), "p": p, "seed": seed, "sweeps": sweeps,
                       "tensor_seed": ts, "nnz": int(sp.nnz), "iterations": int(m.iterations), "fit": m.fit,
                       "sweep_fits": [float(v) for v in m.sweep_fits],
                       "core": m.core.reshape(-1, order="F").tolist(),
                       "factors": [f.reshape(-1, order="F").tolist() for f in m.factors]})
    with open(os.path.join(OUT, "mach_hooi.json"), "w") as f:
        json.dump({"generator": "tests/tools/make_golden.py", "cases": models}, f)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
