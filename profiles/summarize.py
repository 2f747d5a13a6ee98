#!/usr/bin/env python3
"""Summarise ncu outputs into profiles/ (committed evidence).

  python profiles/summarize.py launches <launches.csv>      -> per-kernel share of one timed step
  python profiles/summarize.py full <report.ncu-rep>        -> key metrics of a --set full capture
"""
import collections
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        name = name.replace("ngsb::<unnamed>::", "").replace("void ", "")[:60]
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
        agg[name][0] += 1
        agg[name][1] += v * scale
    tot = sum(v[1] for v in agg.values())
    print(f"# one timed Newton step, serialised cold-cache launches (ncu gpu__time_duration.sum)")
    print(f"# total {tot / 1e3:.3f} ms over {sum(v[0] for v in agg.values())} launches")
    print(f"{'us':>10} {'share':>6} {'n':>4}  kernel")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t:10.1f} {100 * t / tot:5.1f}% {n:4d}  {k}")


WANT = ["Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Executed Ipc Active", "Issue Slots Busy", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Warp Cycles Per Issued Instruction", "Block Limit Registers", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    I = {k: i for i, k in enumerate(h)}
    print(f"# ncu --set full: {path}")
    seen = set()
    for r in rows[1:]:
        key = (r[I["ID"]], r[I["Metric Name"]])
        if r[I["Metric Name"]] in WANT and key not in seen:
            seen.add(key)
            print(f"{r[I['ID']]:>3} {r[I['Kernel Name']][:48]:48s} {r[I['Metric Name']]:36s} {r[I['Metric Value']]:>12} {r[I['Metric Unit']]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if rr:
        hh = rr[0]
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
                  "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum",
                  "sm__inst_executed.sum", "gpu__time_duration.sum"):
            if m in hh:
                j = hh.index(m)
                for r in rr[2:]:
                    print(f"raw {m:55s} {r[j]} {rr[1][j]}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
