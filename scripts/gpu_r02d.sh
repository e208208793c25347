timeout 300 python -m pytest tests/test_gpu_tucker.py -x -q -k "four_way or fp32 or variants" 2>&1 | tail -15
timeout 600 python bench.py --config c3 --no-cpu-baseline --steps 10 --warmup 3 --no-e2e > gpurun_out/r02d_c3.json 2> gpurun_out/r02d_c3.err; tail -3 gpurun_out/r02d_c3.err; python -c "
import json; j=json.load(open('gpurun_out/r02d_c3.json')); print(j['value'], j['ms_per_step'], j['phases_ms']['hosvd'], j['phases_ms']['setup'], j['sampler']); print({k:v['ms_per_sweep'] for k,v in j['kernels'].items()})"
timeout 600 python bench.py --no-cpu-baseline --steps 20 --warmup 5 --no-e2e > gpurun_out/r02d_c2.json 2> gpurun_out/r02d_c2.err; tail -3 gpurun_out/r02d_c2.err; python -c "
import json; j=json.load(open('gpurun_out/r02d_c2.json')); print(j['value'], j['ms_per_step'])"
