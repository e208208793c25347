for r in 40 44 48 52 56; do
for c in c5 c5p01 c5p001; do
MACH_OV_RESERVE_SIDE=$r timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c reserve_side $r', d['value'], d['ms_per_step'])"
done
done
