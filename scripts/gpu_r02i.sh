# round 2 bench lines: C2 (full contract), reference arm, and every other config
timeout 900 python bench.py > gpurun_out/r02i_c2.json 2> gpurun_out/r02i_c2.err; echo c2 rc=$?; tail -2 gpurun_out/r02i_c2.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02i_ref.json 2> gpurun_out/r02i_ref.err; echo ref rc=$?; tail -2 gpurun_out/r02i_ref.err
for c in c1 c3 c5 c5p01 c5p001 c5p1 c4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02i_$c.json 2> gpurun_out/r02i_$c.err; echo $c rc=$?; tail -2 gpurun_out/r02i_$c.err
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/r02i_*.json")):
    try:
        j = json.load(open(f))
    except Exception as e:
        print(f, "bad", e); continue
    r = j.get("roofline") or {}
    print(f, j.get("value"), j.get("ms_per_step"), j.get("phases_ms", {}).get("hosvd"), r.get("frac"), j.get("in_job_sweeps", {}).get("value_sweeps_2_to_n"), (j.get("cpu_baseline_allcores") or {}).get("value"))
PY
