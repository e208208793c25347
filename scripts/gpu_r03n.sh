timeout 1800 python -m pytest tests/test_gpu_tucker.py tests/test_gpu_fullsize.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -3
for c in c5 c5p01 c5p001 c2 c4; do
timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['value'], d['ms_per_step'], d['fit'], {k[:22]:round(v['ms_per_sweep'],3) for k,v in d['kernels'].items() if 'segments' in k})"
done
