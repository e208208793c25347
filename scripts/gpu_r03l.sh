timeout 900 python -m pytest tests/test_gpu_tucker.py tests/test_gpu_tall.py -x -q 2>&1 | tail -3
for c in c4 c5 c2; do
timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['value'], d['ms_per_step'], d['fit'], {k[:22]:round(v['ms_per_sweep'],3) for k,v in list(d['kernels'].items())[:8]})"
done
