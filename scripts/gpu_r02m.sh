# pipelined persistent sampler: parity + timing (TB 128 / 64)
timeout 900 python -m pytest tests/test_gpu_sampler.py -x -q > gpurun_out/r02m_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r02m_pytest.log
timeout 600 python scripts/samp_time.py c2 c5 c5p01 c3 c4 c1 c5p1 > gpurun_out/r02m_samp128.txt 2>&1; echo st rc=$?; cat gpurun_out/r02m_samp128.txt
MACH_SAMPLER_TB=64 timeout 600 python scripts/samp_time.py c2 c5 c5p01 c3 c4 c1 c5p1 > gpurun_out/r02m_samp64.txt 2>&1; echo st rc=$?; cat gpurun_out/r02m_samp64.txt
