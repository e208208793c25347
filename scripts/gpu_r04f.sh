# final validation of the last build: full GPU suite, smoke, default bench and the reference arm
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/r04f_pytest.txt; cat gpurun_out/r04f_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py > gpurun_out/r04f_c2.json 2> gpurun_out/r04f_c2.err; echo c2 rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r04f_ref.json 2> gpurun_out/r04f_ref.err; echo ref rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/r04f_c2.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['traffic'], d['gpu_launches'])
r=json.loads(open('gpurun_out/r04f_ref.json').read().strip().splitlines()[-1]); print(r['value'], r['e2e'])"
