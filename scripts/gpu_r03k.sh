timeout 1800 python -m pytest tests/test_gpu_tucker.py tests/test_gpu_fullsize.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -4
for c in c3 c2 c1; do
timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['value'], d['ms_per_step'], d['fit'])"
done
MACH_NO_SIDE_STAGE1=1 timeout 600 python bench.py --config c3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 no-side', d['value'], d['ms_per_step'], d['fit'])"
for r in 24 32 56; do
MACH_OV_RESERVE_SIDE=$r timeout 600 python bench.py --config c3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 reserve $r', d['value'], d['ms_per_step'], d['fit'])"
done
