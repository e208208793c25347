timeout 900 python -m pytest tests/test_gpu_tucker.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -2
for c in c2 c5; do
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum --clock-control none --csv -k regex:"jds_kernel|ttm_mode_kernel" --log-file gpurun_out/r03y_$c.csv python scripts/prof_sweep.py --config $c --sweeps 1 > /dev/null 2>&1
done
for c in c5 c2; do
timeout 600 python bench.py --config $c --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['value'], d['ms_per_step'], d['fit'], 'e2e', d['e2e']['value'], d['e2e']['job_seconds'])"
done
