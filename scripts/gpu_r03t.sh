for c in c2 c5; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"jds_kernel" --log-file gpurun_out/r03t_$c.csv python scripts/prof_sweep.py --config $c --sweeps 1 > /dev/null 2>&1
done
timeout 600 python -m pytest tests/test_gpu_tucker.py -x -q 2>&1 | tail -2
timeout 600 python bench.py --config c5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5', d['value'], d['ms_per_step'], d['fit'])"
