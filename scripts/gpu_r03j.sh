timeout 600 python -m pytest tests/test_gpu_tucker.py -x -q 2>&1 | tail -3
for v in 65536 81920; do
for c in c5 c5p01 c5p001 c4; do
MACH_S2_STAGE_MAX=$v timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c stage_max $v', d['value'], d['ms_per_step'], {k[:24]:round(v['ms_per_sweep'],3) for k,v in list(d['kernels'].items()) if 'segments' in k})"
done
done
