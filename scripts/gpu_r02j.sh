# round 2 final-state evidence: bench lines (all configs), reference arm, C2 launch list, ncu captures
timeout 900 python bench.py > gpurun_out/r02j_c2.json 2> gpurun_out/r02j_c2.err; echo c2 rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02j_ref.json 2> gpurun_out/r02j_ref.err; echo ref rc=$?
for c in c1 c3 c4 c5 c5p01 c5p001 c5p1; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02j_$c.json 2> gpurun_out/r02j_$c.err; echo $c rc=$?
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02j_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02j_ncu_ll.log 2>&1; echo ll rc=$?
CMD="python scripts/prof_sweep.py --config c2 --sweeps 3"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:ttm_mode_kernel -s 3 -c 1 -o gpurun_out/r02j_ttm_stage1 $CMD > gpurun_out/ncu1.log 2>&1; echo ncu1 rc=$?
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:mode_basis_kernel -s 6 -c 1 -o gpurun_out/r02j_mode_basis $CMD > gpurun_out/ncu2.log 2>&1; echo ncu2 rc=$?
python scripts/samp_prof.py > gpurun_out/plain_s.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sample_kernel -s 1 -c 1 -o gpurun_out/r02j_sampler python scripts/samp_prof.py > gpurun_out/ncu3.log 2>&1; echo ncu3 rc=$?
CMD2="python scripts/prof_sweep.py --config c5p01 --sweeps 2"
$CMD2 > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:eig_cluster_kernel -s 4 -c 1 -o gpurun_out/r02j_eig_cluster $CMD2 > gpurun_out/ncu4.log 2>&1; echo ncu4 rc=$?
ls -la gpurun_out/r02j_*.ncu-rep
