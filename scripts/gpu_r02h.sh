timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_boundary.py -x -q 2>&1 | tail -8
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r02h_c2.json 2>gpurun_out/r02h_c2.err; tail -2 gpurun_out/r02h_c2.err
timeout 600 python bench.py --sharded --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r02h_c2_sh.json 2>gpurun_out/r02h_c2_sh.err; tail -2 gpurun_out/r02h_c2_sh.err
python -c "
import json
for f in ['r02h_c2','r02h_c2_sh']:
    j=json.load(open('gpurun_out/'+f+'.json')); print(f, j['value'], j['ms_per_step'], j['config']['parallelism'], j['gpu_launches'])"
