python -m pytest tests/test_gpu_tall.py -x -q 2>&1 | tail -15
MACH_DEBUG_TALL=1 timeout 600 python bench.py --config c4 --no-cpu-baseline --steps 3 --warmup 1 --no-e2e > gpurun_out/r02b_c4.json 2> gpurun_out/r02b_c4.err; grep -v "\[tall\]" gpurun_out/r02b_c4.err | tail -5; grep -c "\[tall\]" gpurun_out/r02b_c4.err; tail -c 1500 gpurun_out/r02b_c4.json
