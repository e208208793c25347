set -x
timeout 900 python -m pytest tests/test_gpu_dense_tc.py -x -q 2>&1 | tail -25
