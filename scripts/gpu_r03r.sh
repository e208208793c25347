for i in 1 2 3; do
for v in cur old; do
if [ $v = old ]; then L=$PWD/paper_0909_4969_b200/build/var/lib_r03i.so; else L=""; fi
MACH_LIB_PATH=$L timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2 $v', d['value'], d['ms_per_step'], d['in_job_sweeps']['ms'], d['e2e']['value'])"
done
done
