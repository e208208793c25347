# round 2 (session 3): state check after the restored container
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02k_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r02k_pytest.log
timeout 600 python bench.py > gpurun_out/r02k_c2.json 2> gpurun_out/r02k_c2.err; echo c2 rc=$?; cat gpurun_out/r02k_c2.json | head -c 600; echo
./scripts/micro/hash_probe > gpurun_out/r02k_hash_probe.txt 2>&1; cat gpurun_out/r02k_hash_probe.txt
