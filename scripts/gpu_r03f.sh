set -x
timeout 900 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_tucker.py tests/test_gpu_dense_tc.py tests/test_gpu_next_rows.py -x -q 2>&1 | tail -8
timeout 300 python scripts/e2e_breakdown.py c5p1 2>&1 | tail -2
timeout 300 python scripts/samp_time.py c5p1 c2 2>&1 | tail -2
