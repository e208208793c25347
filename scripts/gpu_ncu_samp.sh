cat > /tmp/samp1.py <<'PY'
import torch, paper_0909_4969_b200 as mb
from paper_0909_4969_b200.synth import CONFIGS, lowrank_torch
dims, ranks, noise, p, _, dtype = CONFIGS["c2"]
x = lowrank_torch(dims, ranks, noise, seed=2, dtype=dtype)
t = mb.DenseTensor.from_torch(x, dims)
for i in range(2): mb.sparsify(t, mb.SparsifyConfig(p, 7)).free()
PY
PYTHONPATH=. python /tmp/samp1.py > gpurun_out/plain.log 2>&1 && PYTHONPATH=. ncu --set full --clock-control none --import-source on -k regex:sample_kernel -s 1 -c 1 -o gpurun_out/r02_sampler python /tmp/samp1.py > gpurun_out/ncu.log 2>&1; tail -2 gpurun_out/ncu.log
