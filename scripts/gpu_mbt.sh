# mode-basis phase stamps (MACH_DEBUG_EIG_T) at C2 and C1
MACH_DEBUG_EIG_T=1 timeout 300 python scripts/prof_sweep.py --config c2 --sweeps 4 > gpurun_out/mbt_c2.log 2>&1
grep -c mb-t gpurun_out/mbt_c2.log; tail -12 gpurun_out/mbt_c2.log
