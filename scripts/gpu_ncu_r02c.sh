# ncu captures (round 2): mode basis at C2, tcgen05 Gram and TTM at C5 p=1
python scripts/prof_sweep.py --config c2 --sweeps 3 > gpurun_out/plain_mb.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mode_basis_kernel -s 6 -c 1 -o gpurun_out/r02c_mode_basis python scripts/prof_sweep.py --config c2 --sweeps 3 > gpurun_out/ncu_mb.log 2>&1
tail -2 gpurun_out/ncu_mb.log
python scripts/dense_time.py 1024,1024,1024 16,16,16 1 > gpurun_out/plain_dense.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gram_tc_kernel -s 1 -c 1 -o gpurun_out/r02c_gram_tc python scripts/dense_time.py 1024,1024,1024 16,16,16 1 > gpurun_out/ncu_gram.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ttm_tc_kernel -s 1 -c 1 -o gpurun_out/r02c_ttm_tc python scripts/dense_time.py 1024,1024,1024 16,16,16 1 > gpurun_out/ncu_ttm.log 2>&1
tail -2 gpurun_out/ncu_gram.log gpurun_out/ncu_ttm.log
ls -la gpurun_out/*.ncu-rep
