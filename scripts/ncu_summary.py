"""Summarise one kernel of an `ncu --set full` report into profiles/.

  python scripts/ncu_summary.py REPORT.ncu-rep --config c2 --tag r01_ttm_ncu [--index 0]

Writes profiles/<tag>.json (per-launch DRAM bytes, duration, throughputs,
occupancy, stall mix) and profiles/<tag>.md.  Run here on a report copied back
from gpurun_out/ (ncu -i works without a GPU).
"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smem_ld_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "smem_ld_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smem_pipe_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "inst_executed": "smsp__inst_executed.sum",
    "registers": "launch__registers_per_thread",
    "block": "launch__block_size",
    "grid": "launch__grid_size",
    "dyn_smem": "launch__shared_mem_per_block_dynamic",
}


def ttm_src_sha():
    """Hash of the sources that define the sparse TTM kernels: bench.py only
    takes a capture's DRAM traffic when it matches the build it measures."""
    import hashlib
    h = hashlib.sha256()
    for name in ("ttm_kernel.cuh", "sparse_ttm.cu", "sparse_ttm.cuh", "common.cuh"):
        with open(os.path.join(ROOT, "paper_0909_4969_b200", "csrc", name), "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--config", default="c2")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--index", type=int, default=0)
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    d = dict(zip(head, data[a.index]))
    u = dict(zip(head, units))
    out = {"config": a.config, "report": os.path.basename(a.report), "kernel": d.get("Kernel Name", ""),
           "ttm_src_sha": ttm_src_sha()}
    for k, m in KEYS.items():
        out[k] = num(d.get(m))
    # ncu reports bytes in the unit row (byte / Kbyte / Mbyte ...); normalise
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for k in ("dram_read", "dram_write"):
        m = KEYS[k]
        if out[k] is not None:
            out[k] *= scale.get(u.get(m, "byte"), 1)
    dur_scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    out["duration_us"] = out["duration_us"] * dur_scale.get(u.get(KEYS["duration_us"], "ns"), 1e-3)
    out["dram_bytes_per_launch"] = (out["dram_read"] or 0) + (out["dram_write"] or 0)
    stalls = {}
    for h in head:
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            v = num(d.get(h))
            if v:
                stalls[h[len("smsp__pcsamp_warps_issue_stalled_"):]] = v
    tot = sum(stalls.values()) or 1.0
    out["stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", a.tag + ".json"), "w") as f:
        json.dump(out, f, indent=1)
    lines = [f"# {a.tag}: {out['kernel'][:100]}", "", f"report: `{out['report']}` (ncu --set full --clock-control none)", ""]
    for k in KEYS:
        lines.append(f"- {k}: {out[k]}")
    lines.append(f"- dram_bytes_per_launch: {out['dram_bytes_per_launch']:.0f}")
    lines.append(f"- stalls (% of samples): {out['stalls_pct']}")
    with open(os.path.join(ROOT, "profiles", a.tag + ".md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
