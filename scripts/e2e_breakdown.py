"""Wall-clock breakdown of the e2e job (bench.py run_e2e): upload, mach_mach_hooi
(with the model's own sample / setup / HOSVD / sweep device times), download."""
import ctypes as C
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0909_4969_b200 as mb  # noqa: E402
from paper_0909_4969_b200 import _lib as L  # noqa: E402
from paper_0909_4969_b200.synth import CONFIGS, lowrank_torch  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
dims, ranks, noise, p, sweeps, dtype = CONFIGS[cfg]
host = lowrank_torch(dims, ranks, noise, seed=2, dtype=dtype).cpu().pin_memory()
lib = L.lib()
ctx = mb.Context(0)
dt = L.MACH_F32 if dtype == "float32" else L.MACH_F64
dims_c = (C.c_int * len(dims))(*dims)
ranks_c = (C.c_int * len(ranks))(*ranks)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hd = C.c_void_p()
    assert lib.mach_dense_upload(ctx.h, dt, len(dims), dims_c, C.c_void_p(host.data_ptr()), C.byref(hd)) == 0
    lib.mach_ctx_synchronize(ctx.h)
    t1 = time.perf_counter()
    hm, hs = C.c_void_p(), C.c_void_p()
    assert lib.mach_mach_hooi(ctx.h, hd, ranks_c, p, 7, 5, 0.0, C.byref(hm), C.byref(hs)) == 0, lib.mach_last_error()
    t2 = time.perf_counter()
    sample, setup, hosvd = C.c_double(), C.c_double(), C.c_double()
    sw = (C.c_double * 5)()
    lib.mach_model_times(hm, C.byref(sample), C.byref(setup), C.byref(hosvd), sw, 5)
    model = mb.api._model_from(hm)
    t3 = time.perf_counter()
    lib.mach_sparse_free(hs)
    lib.mach_dense_free(hd)
    print(f"rep {rep}: upload {1e3*(t1-t0):.2f} ms ({math.prod(dims)*4/(t1-t0)/1e9:.1f} GB/s), job {1e3*(t2-t1):.2f} ms "
          f"[sample {sample.value:.2f} setup {setup.value:.2f} hosvd {hosvd.value:.2f} sweeps {sum(sw):.2f} = {[round(v, 2) for v in sw]}], "
          f"download {1e3*(t3-t2):.2f} ms, total {1e3*(t3-t0):.2f} ms")
