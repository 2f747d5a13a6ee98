"""Cross-check of the 290 flop/record constant of the position backward (bench.py roofline):
run under
  ncu --profile-from-start off --metrics <FP32 instruction counters> -k regex:backward_k --csv \
      --log-file flops.csv python tools/flop_crosscheck.py run
then `python tools/flop_crosscheck.py summarize flops.csv records.json` writes
profiles/r2_flops_backward.json: executed FP32 flops of the primary view's position launch
(2 FFMA + 4 FFMA2 + FMUL + 2 FMUL2 + FADD + 2 FADD2 per thread instruction) per contributing
record of that launch. Tooling."""
import collections
import csv
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def run(out_json):
    import torch
    from paper_2501_13975_b200 import capi
    from paper_2501_13975_b200.workload import CONFIGS, cameras_for, make_scenes
    cfg = CONFIGS["c2"]
    lib = capi.product()
    ctx = lib.context(0)
    truth, init = make_scenes(cfg)
    cams = cameras_for(cfg)
    ctx.set_scene(truth)
    targets = [ctx.render(c) for c in cams]
    ctx.set_scene(init)
    ctx.trainer_configure(lib.default_train(), cams, targets, list(range(cfg.views)))
    order = [int(v) for v in np.random.default_rng(7).permutation(cfg.views)]
    for i in range(3):
        ctx.trainer_step(order[i])
    ctx.profile_reset()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    ctx.trainer_step(order[3])
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    p = ctx.profile_read()
    json.dump({"primary_contrib_pairs": p["primary_contrib_pairs"], "contrib_pairs": p["contrib_pairs"]},
              open(out_json, "w"))


def summarize(csv_path, rec_json):
    rows = list(csv.reader(open(csv_path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) > vi:
            per.setdefault((r[ii], r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
    first = next((k, m) for k, m in per.items() if "backward_k<4, 16>" in k[1] or "backward_k<(int)4, (int)16>" in k[1])
    m = first[1]
    pre = "smsp__sass_thread_inst_executed_op_"
    flops = (2 * m[pre + "ffma_pred_on.sum"] + 4 * m[pre + "ffma2_pred_on.sum"] + m[pre + "fmul_pred_on.sum"] +
             2 * m[pre + "fmul2_pred_on.sum"] + m[pre + "fadd_pred_on.sum"] + 2 * m[pre + "fadd2_pred_on.sum"])
    rec = json.load(open(rec_json))["primary_contrib_pairs"][0]
    t_ms = m["gpu__time_duration.sum"] / 1e6
    out = {"kernel": "backward_k<PositionUV,16>, primary view, c2 (ncu, one launch)",
           "executed_fp32_flops": flops, "contributing_records": rec, "executed_flops_per_record": flops / rec,
           "algorithmic_flops_per_record": 290, "ncu_duration_ms": t_ms,
           "executed_tflops_under_ncu": flops / (t_ms * 1e-3) / 1e12,
           "source": "profiles/r2_flops_backward.csv (ncu --metrics sass_thread_inst_executed_op_*)"}
    json.dump(out, open(os.path.join(REPO, "profiles", "r2_flops_backward.json"), "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/flop_records.json")
    else:
        summarize(sys.argv[2], sys.argv[3])
