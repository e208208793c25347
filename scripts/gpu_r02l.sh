# sampler rewrite: parity + timing
timeout 900 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r02l_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r02l_pytest.log
timeout 600 python scripts/samp_time.py c2 c5 c5p01 c5p001 c3 c4 c1 c5p1 > gpurun_out/r02l_samp.txt 2>&1; echo st rc=$?; cat gpurun_out/r02l_samp.txt
