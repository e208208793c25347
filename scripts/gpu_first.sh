set -x
nproc; free -g; lscpu | grep "Model name"; nvidia-smi --query-gpu=name,memory.total --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r02a_c2.json 2> gpurun_out/r02a_c2.err
tail -c 600 gpurun_out/r02a_c2.json
timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 5 > gpurun_out/r02a_c3.json 2> gpurun_out/r02a_c3.err; tail -3 gpurun_out/r02a_c3.err; tail -c 300 gpurun_out/r02a_c3.json
timeout 300 python bench.py --config c4 --no-cpu-baseline --steps 3 --no-e2e > gpurun_out/r02a_c4.json 2> gpurun_out/r02a_c4.err; tail -3 gpurun_out/r02a_c4.err
