# new SURVEY 8(f) rows: bound, stream, binary files, C++ mirror + CLI
timeout 900 python -m pytest tests/test_gpu_next_rows.py tests/test_gpu_boundary.py -x -q 2>&1 | tail -40
