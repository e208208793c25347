timeout 300 python -m pytest tests/test_gpu_sampler.py -x -q 2>&1 | tail -1
timeout 300 python scripts/samp_time.py c2 c5 c5p01 c4 c3 2>&1
python scripts/samp_prof.py > gpurun_out/plain_s.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:sample_kernel -s 1 -c 1 -o gpurun_out/r02p_sampler python scripts/samp_prof.py > gpurun_out/ncu_s.log 2>&1; echo ncu rc=$?
