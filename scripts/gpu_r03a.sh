# restored build after the sampler rewrite: GPU tests, all benches, launch list
set -x
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r03a_pytest.txt; cat gpurun_out/r03a_pytest.txt
timeout 600 python bench.py > gpurun_out/r03a_c2.json 2> gpurun_out/r03a_c2.err; tail -3 gpurun_out/r03a_c2.err; cat gpurun_out/r03a_c2.json
for c in c3 c4 c5p1 c5p01 c5p001 c5 c1; do
timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/r03a_$c.json 2> gpurun_out/r03a_$c.err; tail -2 gpurun_out/r03a_$c.err; cat gpurun_out/r03a_$c.json
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r03a_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r03a_ncu.log 2>&1; tail -2 gpurun_out/r03a_ncu.log
