timeout 1200 python -m pytest tests/test_gpu_sharded.py -x -q 2>&1 | tail -15
MACH_SHARD_REPLICATED_HOSVD=1 timeout 1200 python -m pytest tests/test_gpu_sharded.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --sharded --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('sharded n1', d['value'], d['ms_per_step'], d['fit'], d['phases_ms'].get('hosvd'))"
