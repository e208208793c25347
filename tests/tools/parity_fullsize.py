"""One-off full-size parity run outside the test suite (minutes of CPU oracle time):
  ORACLE_VARIANT=omp python tests/tools/parity_fullsize.py c5 0.1 2
compares the device mach_hooi at a BASELINE config with the oracle on the same
values (kept-index array, sweep_fits, factor sines, core, fit) and prints one
JSON line.  C5 p = 0.1 is the config whose HOSVD Grams run on tcgen05 (TF32)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_0909_4969_b200 as mb  # noqa: E402
from tests.helpers import align_core, rel, subspace_sin  # noqa: E402
from tests.test_gpu_fullsize import run_case  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
p = float(sys.argv[2]) if len(sys.argv) > 2 else None
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else None
t0 = time.time()
model, idx, vals, ref, oi, ov = run_case(mb, cfg, p=p, sweeps=sweeps)
n = min(len(model.sweep_fits), len(ref.sweep_fits))
out = {"config": cfg, "p": p, "sweeps": sweeps, "nnz": int(len(idx)),
       "kept_index_array_equal": bool(np.array_equal(idx, oi)),
       "kept_values_equal_fp32": bool(np.array_equal(vals.astype(np.float32), ov.astype(np.float32))),
       "iterations": [model.iterations, ref.iterations],
       "sweep_fits_device": [float(v) for v in model.sweep_fits], "sweep_fits_oracle": [float(v) for v in ref.sweep_fits],
       "sweep_fits_max_rel": float(np.max(np.abs(np.array(model.sweep_fits[:n]) - np.array(ref.sweep_fits[:n])) /
                                          np.abs(np.array(ref.sweep_fits[:n])))),
       "factor_sines": [float(subspace_sin(fd, fr)) for fd, fr in zip(model.factors, ref.factors)],
       "core_rel": float(rel(align_core(model.core, model.factors, ref.factors), ref.core)),
       "fit_rel": float(abs(model.fit - ref.fit) / abs(ref.fit)), "wall_s": round(time.time() - t0, 1)}
out["pass"] = bool(out["kept_index_array_equal"] and out["kept_values_equal_fp32"] and max(out["factor_sines"]) <= 1e-3 and
                   out["core_rel"] <= 1e-4 and out["fit_rel"] <= 1e-4 and out["sweep_fits_max_rel"] <= 1e-4)
print(json.dumps(out), flush=True)
