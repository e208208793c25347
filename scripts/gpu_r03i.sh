# round 2 final-state evidence: GPU tests, bench lines (all configs), reference arm, launch lists, ncu captures, 8(f) timings
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 > gpurun_out/r03i_pytest.txt; cat gpurun_out/r03i_pytest.txt
timeout 900 python bench.py > gpurun_out/r03i_c2.json 2> gpurun_out/r03i_c2.err; echo c2 rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r03i_ref.json 2> gpurun_out/r03i_ref.err; echo ref rc=$?
for c in c1 c3 c4 c5 c5p01 c5p001 c5p1; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/r03i_$c.json 2> gpurun_out/r03i_$c.err; echo $c rc=$?
done
timeout 900 python scripts/next_rows_time.py > gpurun_out/r03i_next_rows.jsonl 2> gpurun_out/r03i_next_rows.err; echo next rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r03i_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r03i_ncu_ll.log 2>&1; echo ll rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r03i_launches_c5.csv python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r03i_ncu_ll5.log 2>&1; echo ll5 rc=$?
CMD="python scripts/prof_sweep.py --config c2 --sweeps 3"
$CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:ttm_mode_kernel -s 3 -c 1 -o gpurun_out/r03i_ttm_stage1 $CMD > gpurun_out/ncu1.log 2>&1; echo ncu1 rc=$?
$CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:mode_basis_kernel -s 6 -c 1 -o gpurun_out/r03i_mode_basis $CMD > gpurun_out/ncu2.log 2>&1; echo ncu2 rc=$?
python scripts/samp_prof.py > gpurun_out/plain_s.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:sample_kernel -s 1 -c 1 -o gpurun_out/r03i_sampler python scripts/samp_prof.py > gpurun_out/ncu3.log 2>&1; echo ncu3 rc=$?
CMD5="python scripts/prof_sweep.py --config c5 --sweeps 2"
$CMD5 > gpurun_out/plain5.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_tc_kernel -s 1 -c 1 -o gpurun_out/r03i_gram_tc_sampled $CMD5 > gpurun_out/ncu5.log 2>&1; echo ncu5 rc=$?
$CMD5 > gpurun_out/plain5.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:ttm_mode_kernel -s 4 -c 1 -o gpurun_out/r03i_ttm_stage1_c5 $CMD5 > gpurun_out/ncu6.log 2>&1; echo ncu6 rc=$?
CMD1="python scripts/prof_sweep.py --config c5p1 --sweeps 1"
$CMD1 > gpurun_out/plain1.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:keep_all_write_kernel -c 1 -o gpurun_out/r03i_keep_all $CMD1 > gpurun_out/ncu7.log 2>&1; echo ncu7 rc=$?
ls -la gpurun_out/r03i_*.ncu-rep
