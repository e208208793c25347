# sampler variants A/B (MACH_LIB_PATH)
for v in base v1 v3 v4; do
  if [ $v = base ]; then L=""; else L=paper_0909_4969_b200/build/var/lib_$v.so; fi
  TBV=128; [ $v = v4 ] && TBV=64
  echo "== $v"
  MACH_SAMPLER_TB=$TBV MACH_LIB_PATH=$L timeout 300 python -m pytest tests/test_gpu_sampler.py -x -q 2>&1 | tail -1
  MACH_SAMPLER_TB=$TBV MACH_LIB_PATH=$L timeout 300 python scripts/samp_time.py c2 c5 c5p01 2>&1
done
