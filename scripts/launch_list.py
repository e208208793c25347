"""Per-sweep kernel table from an ncu launch list.

  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file L.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e
  python scripts/launch_list.py L.csv --sweeps 2 --tag r01_launches_c2

A sweep ends with core_sumsq_kernel (or, in older builds, core_from_last ->
sumsq_partial -> sum_final); the last --sweeps sweeps are tabulated (library kernels
only; the bench's L2-flush fill is listed separately).  Writes
profiles/<tag>.csv (the raw list) and profiles/<tag>.md.
"""
import argparse
import csv
import os
import shutil

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--sweeps", type=int, default=2)
ap.add_argument("--tag", required=True)
ap.add_argument("--command", default="ncu --metrics gpu__time_duration.sum --clock-control none --csv "
                "python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e")
a = ap.parse_args()

rows = []
with open(a.csv) as fh:
    lines = [ln for ln in fh if ln.startswith('"')]
rd = csv.reader(lines)
hdr = None
for r in rd:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "ns")
    us = v / 1e3 if unit in ("ns", "nsecond") else (v if unit in ("us", "usecond") else v * 1e3)
    rows.append((d["Kernel Name"], us))

ends = [i for i, (k, _) in enumerate(rows) if "core_sumsq_kernel" in k or (
    "sum_final_kernel" in k and i >= 2 and "sumsq_partial_kernel" in rows[i - 1][0]
    and "core_from_last_kernel" in rows[i - 2][0])]
assert len(ends) > a.sweeps, f"found {len(ends)} sweeps"
sel = rows[ends[-a.sweeps - 1] + 1: ends[-1] + 1]
lib = [(k, us) for k, us in sel if "machb" in k or "ttm::" in k]
other = [(k, us) for k, us in sel if not ("machb" in k or "ttm::" in k)]
agg = {}
for k, us in lib:
    n, t = agg.get(k, (0, 0.0))
    agg[k] = (n + 1, t + us)
tot = sum(t for _, t in agg.values())
out = [f"# {a.tag}: C2 sweep kernels (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised)", "",
       f"command: `{a.command}`", "",
       f"last {a.sweeps} sweeps: {len(lib)} library launches, {tot:.1f} us total, {tot / a.sweeps:.1f} us per sweep "
       "(sum of kernel durations under ncu's serialisation; the un-profiled graph replay overlaps launches with PDL)", "",
       "| kernel | launches/sweep | us/sweep | share |", "|---|---|---|---|"]
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    out.append(f"| `{k[:110]}` | {n / a.sweeps:.1f} | {t / a.sweeps:.1f} | {100 * t / tot:.1f}% |")
if other:
    out += ["", "Not library kernels (bench L2 flush between timed sweeps): " +
            ", ".join(f"`{k[:60]}` {us:.1f} us" for k, us in other)]
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
with open(os.path.join(ROOT, "profiles", a.tag + ".md"), "w") as fh:
    fh.write("\n".join(out) + "\n")
shutil.copy(a.csv, os.path.join(ROOT, "profiles", a.tag + ".csv"))
print("\n".join(out))
