timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/r03q_pytest.txt; cat gpurun_out/r03q_pytest.txt
for c in c2 c3 c4 c5 c5p01 c5p001 c1 c5p1; do
timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/r03q_$c.json 2> gpurun_out/r03q_$c.err; python -c "
import json; d=json.loads(open('gpurun_out/r03q_$c.json').read().strip().splitlines()[-1]); e=d['e2e']; print('$c', d['value'], d['ms_per_step'], 'e2e', e['value'], e['job_seconds'], e['step'][-18:], 'hosvd', d['phases_ms']['hosvd'], 'traffic', d['roofline'].get('traffic'))"
done
timeout 300 python scripts/e2e_breakdown.py c4 2>&1 | tail -1
