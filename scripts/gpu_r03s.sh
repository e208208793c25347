timeout 300 python scripts/e2e_breakdown.py c2 2>&1 | tail -2
MACH_SPARSE_GRAM_TC_MIN=0.5 timeout 300 python scripts/e2e_breakdown.py c2 2>&1 | tail -2
MACH_SPARSE_GRAM_TC_MIN=0.5 timeout 1200 python -m pytest tests/test_gpu_tucker.py tests/test_gpu_fullsize.py -x -q -k "not c5 and not c3" 2>&1 | tail -3
