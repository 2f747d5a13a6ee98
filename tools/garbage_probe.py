"""Uninitialised-memory probe: fill most of the device memory with a garbage pattern and
release it to the driver before creating the contexts (cudaMalloc hands the pages back
unzeroed within a process), then run deterministic Newton steps and first-order Adam
steps; the printed norms must match a run without garbage. Tooling (GPU).
  python tools/garbage_probe.py [nan|big|rand|none]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
mode = sys.argv[1] if len(sys.argv) > 1 else "none"
if mode != "none":
    free, _ = torch.cuda.mem_get_info()
    n = int(free * 0.85) // 4
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    if mode == "nan":
        x.fill_(float("nan"))
    elif mode == "big":
        x.fill_(3e38)
    else:
        x.random_()
    torch.cuda.synchronize()
    del x
    torch.cuda.empty_cache()
from paper_2501_13975_b200 import capi  # noqa: E402
from paper_2501_13975_b200.workload import Config, cameras_for, make_scenes  # noqa: E402
from refimpl import synth  # noqa: E402

gpu = capi.product()
out = {}
# Newton, deterministic: small synthetic scene (8x8-tile, chunked primary) and a mid-size one
for name, cfg in (("small", None), ("mid", Config("g", 40_000, 6, 256, 192, 3, 0.45))):
    if cfg is None:
        d = synth(seed=23, kernels=60, views=4, probe_views=0, width=48, height=48, perturbation=0.5,
                  secondary_downsample=2)
        init, cams, targets, train = d["init"], d["cameras"], d["targets"], d["train"]
    else:
        truth, init = make_scenes(cfg, seed=2)
        cams = cameras_for(cfg)
        c = gpu.context()
        c.set_scene(truth)
        targets = [c.render(x) for x in cams]
        c.close()
        train = list(range(cfg.views))
    ctx = gpu.context()
    ctx.set_deterministic(True)
    ctx.set_scene(init)
    tc = gpu.default_train()
    tc.knn = 2
    ctx.trainer_configure(tc, cams, targets, train)
    norms = [list(ctx.trainer_step(v).delta_norms) for v in train[:3]]
    s = ctx.get_scene()
    out[name] = (norms, float(np.sum(s.position)), float(np.sum(s.sh)))
    ctx.close()
# first-order Adam (the flaky test's path)
d = synth(seed=32, kernels=200, views=4, probe_views=0, width=48, height=48, perturbation=0.5, secondary_downsample=2)
cfg = gpu.default_train()
cfg.optimizer = capi.OPT_ADAM
ctx = gpu.context()
ctx.set_deterministic(True)
ctx.set_scene(d["init"])
ctx.trainer_configure(cfg, d["cameras"], d["targets"], d["train"])
out["adam"] = [list(ctx.trainer_step(v).delta_norms) for v in d["train"][:3]]
ctx.close()
print(mode, repr(out))
