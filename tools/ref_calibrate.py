"""Calibrates bench.py's reference slice: ONE full c2 Trainer::step of the reference (all host
threads) against the 1/64 slice bench.py --impl reference times. Targets are rendered (reference
render, threaded) only for the step's primary and its K neighbours; the other views' targets
are never read by one step. Tooling."""
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
import bench  # noqa: E402
from paper_2501_13975_b200.workload import CONFIGS, cameras_for, make_scenes  # noqa: E402
from refimpl import ref  # noqa: E402

cfg = CONFIGS["c2"]
lib = ref()
threads = os.cpu_count() or 1
truth, init = make_scenes(cfg)
cams = cameras_for(cfg)
view = int(np.random.default_rng(7).permutation(cfg.views)[0])
zeros = [np.zeros((c.height, c.width, 3)) for c in cams]
tc = lib.default_train()
tc.threads = threads
probe = lib.context()
probe.set_scene(init)
probe.trainer_configure(tc, cams, zeros, list(range(cfg.views)))
nbrs = probe.trainer_neighbors(view)
probe.close()
rctx = lib.context()
rctx.set_scene(truth)
ro = lib.default_raster()
ro.threads = threads
targets = list(zeros)
for v in [view] + nbrs:
    targets[v] = rctx.render(cams[v], ro)
ctx = lib.context()
ctx.set_scene(init)
ctx.trainer_configure(tc, cams, targets, list(range(cfg.views)))
t0 = time.time()
rep = ctx.trainer_step(view)
full_s = time.time() - t0
sl = bench.run_reference_sample(cfg, 2, 1, 8)
print(f"full c2 reference step: {rep.dt_ms / 1e3:.1f} s ({threads} threads) = {1e3 / rep.dt_ms:.5f} views/s; "
      f"1/64 slice: {sl['ms_per_sample_step'] / 1e3:.2f} s/step = {sl['value']:.5f} views/s "
      f"(slice x64 = {64 * sl['ms_per_sample_step'] / 1e3:.1f} s; ratio full / (64 x slice) = "
      f"{rep.dt_ms / (64 * sl['ms_per_sample_step']):.3f})")
