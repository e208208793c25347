"""Top SASS lines by warp-stall samples from `ncu --page source --csv` output."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
h = rows[1]
ix = {c: i for i, c in enumerate(h)}
body = [r for r in rows[2:] if len(r) == len(h) and r[0] != h[0]]
tot = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
body.sort(key=lambda r: -float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
for r in body[:n]:
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    top = sorted(((float(r[ix[c]] or 0), c[6:]) for c in stalls), reverse=True)[:2]
    conf = r[ix["L1 Conflicts Shared N-Way"]]
    print(f"{100*s/tot:5.1f}% {r[ix['Address']][-5:]} {r[ix['Source']].strip()[:60]:60s} "
          f"{','.join(f'{b}:{int(a)}' for a, b in top if a)} nway={conf}")
