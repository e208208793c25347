set -x
timeout 900 python scripts/next_rows_time.py > gpurun_out/r03c_next_rows.jsonl 2> gpurun_out/r03c_next_rows.err; tail -3 gpurun_out/r03c_next_rows.err; cat gpurun_out/r03c_next_rows.jsonl
for c in c2 c4 c1 c5; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r03c_launches_$c.csv python scripts/prof_sweep.py --config $c --sweeps 1 > gpurun_out/r03c_ncu_$c.log 2>&1; tail -1 gpurun_out/r03c_ncu_$c.log
done
timeout 300 python scripts/e2e_breakdown.py c2 2>&1 | tail -3
timeout 300 python scripts/e2e_breakdown.py c5 2>&1 | tail -3
