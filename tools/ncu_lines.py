"""Aggregate an `ncu --page source --csv --print-source cuda,sass` dump per CUDA source line:
warp-level instructions executed and stall samples. Tooling.
  python tools/ncu_lines.py dump.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = defaultdict(lambda: [0, 0, ""])
f, line, hdr = "?", None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0]:
        line = (f, int(r[0]))
        agg[line][2] = r[1][:70]
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        agg[line][0] += int(d.get("Instructions Executed", "0") or 0)
        agg[line][1] += int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        pass
tot_i = sum(v[0] for v in agg.values())
tot_s = sum(v[1] for v in agg.values())
print(f"total warp instructions {tot_i:.3e}, stall samples {tot_s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100 * v[0] / tot_i:5.1f}% inst {100 * v[1] / max(tot_s, 1):5.1f}% samples  {k[0]}:{k[1]:<5} {v[2]}")
