python -m pytest tests/test_gpu_tall.py tests/test_gpu_tucker.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --config c4 --no-cpu-baseline --steps 3 --warmup 1 --no-e2e > gpurun_out/r02c_c4.json 2> gpurun_out/r02c_c4.err; tail -3 gpurun_out/r02c_c4.err; python -c "
import json; j=json.load(open('gpurun_out/r02c_c4.json')); print(j['value'], j['ms_per_step'], j['phases_ms']['hosvd'], j['phases_ms']['setup'], j['sampler']); print({k:v['ms_per_sweep'] for k,v in j['kernels'].items()})"
