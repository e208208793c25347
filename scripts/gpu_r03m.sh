timeout 1800 python -m pytest tests/test_gpu_tucker.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3
for c in c5 c2 c3 c4; do
timeout 600 python bench.py --config $c --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['value'], d['ms_per_step'], d['fit'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['phases_ms']['setup'], d['e2e']['value'], d['e2e']['job_seconds'])"
done
cap() {
  local tag=$1 cfg=$2 k=$3 skip=$4; shift 4
  "$@" > gpurun_out/plain.log 2>&1 || { echo "$tag plain run failed"; return; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -o /tmp/$tag "$@" > gpurun_out/ncu_$tag.log 2>&1
  echo "$tag ncu rc=$?"
  python scripts/ncu_summary.py /tmp/$tag.ncu-rep --config $cfg --tag $tag > /dev/null 2>&1 && cp profiles/$tag.json profiles/$tag.md gpurun_out/
  rm -f /tmp/$tag.ncu-rep
}
cap r03m_ttm_stage1_ncu c2 ttm_mode_kernel 3 python scripts/prof_sweep.py --config c2 --sweeps 3
cap r03m_ttm_stage1_c5_ncu c5 ttm_mode_kernel 4 python scripts/prof_sweep.py --config c5 --sweeps 2
