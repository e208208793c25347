tag=r03x_jds_ncu
python scripts/prof_sweep.py --config c2 --sweeps 1 > gpurun_out/plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jds_kernel -s 1 -c 1 -o /tmp/$tag python scripts/prof_sweep.py --config c2 --sweeps 1 > gpurun_out/ncu_$tag.log 2>&1
python scripts/ncu_summary.py /tmp/$tag.ncu-rep --config c2 --tag $tag > /dev/null 2>&1 && cp profiles/$tag.json profiles/$tag.md gpurun_out/
ncu -i /tmp/$tag.ncu-rep --page source --csv > /tmp/$tag.src.csv 2>/dev/null && python scripts/ncu_hot.py /tmp/$tag.src.csv 30 > gpurun_out/${tag}_hotlines.txt 2>/dev/null
ncu -i /tmp/$tag.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; v=rows[2]
for k in ('launch__occupancy_limit_registers','launch__occupancy_limit_shared_mem','sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','launch__grid_size','launch__block_size','smsp__cycles_active.avg','l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum','l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum','sm__cycles_elapsed.max','smsp__inst_executed.sum','launch__waves_per_multiprocessor'):
    if k in h: print(k, v[h.index(k)])
" > gpurun_out/${tag}_extra.txt
