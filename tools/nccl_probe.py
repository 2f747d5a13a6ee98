"""Local vs 1-rank NCCL trainer steps on a small scene: run-to-run and exchange differences. Tooling (GPU)."""
import os, sys
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from paper_2501_13975_b200 import capi
from refimpl import synth
gpu = capi.product()
d = synth(seed=23, kernels=20, views=4, probe_views=0, width=48, height=48, perturbation=0.5, secondary_downsample=2)
def run(use_nccl, det=False):
    ctx = gpu.context()
    ctx.set_scene(d["init"])
    if use_nccl:
        ctx.dist_init(capi.dist_unique_id(gpu), 0, 1)
    cfg = gpu.default_train(); cfg.knn = 2; cfg.secondary_downsample = 2
    ctx.trainer_configure(cfg, d["cameras"], d["targets"], d["train"], [], d["secondary"], d["secondary_downsample"])
    for v in (0, 2): ctx.trainer_step(v)
    s = ctx.get_scene(); ctx.close(); return s
def diff(a, b):
    return {f: float(np.max(np.abs(getattr(a, f) - getattr(b, f)))) for f in ("position", "scale", "quaternion", "sigma", "sh")}
a = run(False); b = run(False); c = run(True)
print(os.environ.get("NGS_BWD_CHUNKS"), "local-vs-local", diff(a, b))
print(os.environ.get("NGS_BWD_CHUNKS"), "local-vs-nccl", diff(a, c))
