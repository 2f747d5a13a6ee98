"""One Newton step of a BASELINE config bracketed by cudaProfilerStart/Stop (for
`ncu --profile-from-start off`), plus the library's per-stage device times of a few
serialised steps. Tooling, not product code.

  python tools/step_profile.py [c1|c2|c3] [steps]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_13975_b200 import capi  # noqa: E402
from paper_2501_13975_b200.workload import CONFIGS, cameras_for, make_scenes  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
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
    ctx.trainer_step(order[(i) % len(order)])
torch.cuda.synchronize()
torch.cuda.profiler.start()
rep = ctx.trainer_step(order[(3) % len(order)])
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"{cfg.name}: profiled step {rep.dt_ms:.3f} ms")
ctx.profile_reset()
ctx.profile_enable(True)
dts = [ctx.trainer_step(order[(4 + i) % len(order)]).dt_ms for i in range(steps)]
p = ctx.profile_read()
print(f"{cfg.name}: serialised steps {np.mean(dts):.3f} ms; stage ms/step",
      {k: round(v / steps, 3) for k, v in p["ms"].items()}, "pairs", [x / steps for x in p["contrib_pairs"]],
      "raster pairs", p["raster_pairs"] / steps)
if p.get("color_channels") and os.environ.get("NGS_COLOR_FUSED", "0") != "0":  # fused colour solve only
    print(f"{cfg.name}: colour channel solves on the fast path {p['color_fast_channels'] / p['color_channels']:.4f}")
ctx.profile_enable(False)
dts = [ctx.trainer_step(order[(10 + i) % len(order)]).dt_ms for i in range(steps)]
print(f"{cfg.name}: concurrent steps {np.mean(dts):.3f} ms")

# Timeline of one concurrent step (per-launch events, views NOT serialised).
ctx.profile_timeline(True)
rep = ctx.trainer_step(order[(20) % len(order)])
rows = ctx.read_timeline()
ctx.profile_timeline(False)
streams = {}
for st, sid, t0, t1 in sorted(rows, key=lambda r: r[2]):
    streams.setdefault(sid, len(streams))
print(f"{cfg.name}: timeline of one concurrent step ({rep.dt_ms:.3f} ms), rows: stage stream start end (ms)")
for st, sid, t0, t1 in sorted(rows, key=lambda r: r[2]):
    print(f"  {st:18s} s{streams[sid]} {t0:8.3f} {t1:8.3f} {t1 - t0:7.3f}")
