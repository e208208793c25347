# round 2 final-state evidence: GPU tests, bench lines (all configs), reference arm, launch lists, ncu captures
# (summarised on the box: the .ncu-rep files are too large to bring back), 8(f) timings
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 > gpurun_out/r03z_pytest.txt; cat gpurun_out/r03z_pytest.txt
timeout 900 python bench.py > gpurun_out/r03z_c2.json 2> gpurun_out/r03z_c2.err; echo c2 rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r03z_ref.json 2> gpurun_out/r03z_ref.err; echo ref rc=$?
for c in c1 c3 c4 c5 c5p01 c5p001 c5p1; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/r03z_$c.json 2> gpurun_out/r03z_$c.err; echo $c rc=$?
done
timeout 900 python scripts/next_rows_time.py > gpurun_out/r03z_next_rows.jsonl 2> gpurun_out/r03z_next_rows.err; echo next rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r03z_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r03z_ncu_ll.log 2>&1; echo ll rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r03z_launches_c5.csv python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r03z_ncu_ll5.log 2>&1; echo ll5 rc=$?
cap() {  # cap <tag> <config> <kernel regex> <skip> <command...>
  local tag=$1 cfg=$2 k=$3 skip=$4; shift 4
  "$@" > gpurun_out/plain.log 2>&1 || { echo "$tag plain run failed"; return; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -o /tmp/$tag "$@" > gpurun_out/ncu_$tag.log 2>&1
  echo "$tag ncu rc=$?"
  python scripts/ncu_summary.py /tmp/$tag.ncu-rep --config $cfg --tag $tag > /dev/null 2>&1 && cp profiles/$tag.json profiles/$tag.md gpurun_out/
  ncu -i /tmp/$tag.ncu-rep --page source --csv > /tmp/$tag.src.csv 2>/dev/null && python scripts/ncu_hot.py /tmp/$tag.src.csv 25 > gpurun_out/${tag}_hotlines.txt 2>/dev/null
  rm -f /tmp/$tag.ncu-rep
}
cap r03z_ttm_stage1_ncu c2 ttm_mode_kernel 3 python scripts/prof_sweep.py --config c2 --sweeps 3
cap r03z_mode_basis_ncu c2 mode_basis_kernel 6 python scripts/prof_sweep.py --config c2 --sweeps 3
cap r03z_sampler_ncu c2 sample_kernel 1 python scripts/samp_prof.py
cap r03z_ttm_stage1_c5_ncu c5 ttm_mode_kernel 4 python scripts/prof_sweep.py --config c5 --sweeps 2
cap r03z_gram_tc_sampled_ncu c5 gram_tc_kernel 1 python scripts/prof_sweep.py --config c5 --sweeps 1
cap r03z_stage2_c5_ncu c5 y_from_segments_kernel 4 python scripts/prof_sweep.py --config c5 --sweeps 2
cap r03z_keep_all_ncu c5p1 keep_all_write_kernel 0 python scripts/prof_sweep.py --config c5p1 --sweeps 1
du -sh gpurun_out
