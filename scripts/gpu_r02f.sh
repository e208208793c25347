# tcgen05 dense Gram: parity tests, then C5-size timing
timeout 600 python -m pytest tests/test_gpu_dense_tc.py -x -q 2>&1 | tail -15
timeout 300 python scripts/gram_time.py > gpurun_out/r02f_gram.json 2> gpurun_out/r02f_gram.err; tail -3 gpurun_out/r02f_gram.err; cat gpurun_out/r02f_gram.json
