set -x
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/r03e_pytest.txt; cat gpurun_out/r03e_pytest.txt
timeout 300 python scripts/e2e_breakdown.py c2 2>&1 | tail -2
timeout 300 python scripts/e2e_breakdown.py c4 2>&1 | tail -2
timeout 300 python scripts/e2e_breakdown.py c3 2>&1 | tail -2
timeout 300 python scripts/e2e_breakdown.py c1 2>&1 | tail -2
timeout 300 python scripts/e2e_breakdown.py c5p1 2>&1 | tail -2
