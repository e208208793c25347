set -x
timeout 1800 python -m pytest tests/test_gpu_tucker.py tests/test_gpu_fullsize.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -8
for c in c5 c5p01 c5p001 c2; do
timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/r03g_$c.json 2> gpurun_out/r03g_$c.err; tail -2 gpurun_out/r03g_$c.err
python -c "
import json; d=json.loads(open('gpurun_out/r03g_$c.json').read().strip().splitlines()[-1]); print('$c', d['value'], d['ms_per_step'], d['fit'])"
MACH_NO_SIDE_STAGE1=1 timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c no-side', d['value'], d['ms_per_step'], d['fit'])"
done
