CMD="python bench.py --config c3 --no-cpu-baseline --steps 2 --warmup 1 --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:stage2_4way -s 4 -c 4 -o gpurun_out/r02_s2_4way $CMD > gpurun_out/ncu.log 2>&1; tail -3 gpurun_out/ncu.log
