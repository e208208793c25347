timeout 900 python -m pytest tests/test_gpu_dense_tc.py -x -q 2>&1 | tail -15
timeout 600 python scripts/dense_time.py > gpurun_out/dense1.json 2>gpurun_out/dense1.err; tail -3 gpurun_out/dense1.err; cat gpurun_out/dense1.json
