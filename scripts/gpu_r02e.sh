# round 2 baseline on the restored build: GPU tests, C2 bench (both arms), launch list
set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r02e_pytest.txt; cat gpurun_out/r02e_pytest.txt
timeout 600 python bench.py > gpurun_out/r02e_c2.json 2> gpurun_out/r02e_c2.err; tail -3 gpurun_out/r02e_c2.err; cat gpurun_out/r02e_c2.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02e_ref.json 2> gpurun_out/r02e_ref.err; tail -2 gpurun_out/r02e_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02e_ncu.log 2>&1; tail -2 gpurun_out/r02e_ncu.log
