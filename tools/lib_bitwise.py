"""Bitwise comparison of two libngs_b200.so builds: deterministic-mode trainer steps on a
mid-size synthetic scene must give identical parameters. Tooling (GPU).
  python tools/lib_bitwise.py libA.so libB.so"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2501_13975_b200 import capi  # noqa: E402
from paper_2501_13975_b200.workload import Config, cameras_for, make_scenes  # noqa: E402

cfg = Config("bitwise", 60_000, 8, 320, 256, 3, 0.45)
truth, init = make_scenes(cfg, seed=11)
cams = cameras_for(cfg)
outs = []
for path in sys.argv[1:3]:
    lib = capi.NgsLibrary(path)
    c = lib.context(0)
    c.set_scene(truth)
    targets = [c.render(x) for x in cams]
    c.close()
    ctx = lib.context(0)
    ctx.set_deterministic(True)
    ctx.set_scene(init)
    ctx.trainer_configure(lib.default_train(), cams, targets, list(range(cfg.views)))
    for v in (0, 3, 5):
        ctx.trainer_step(v)
    outs.append(ctx.get_scene())
    ctx.close()
same = all(np.array_equal(getattr(outs[0], f), getattr(outs[1], f)) for f in ("position", "scale", "quaternion", "sigma", "sh"))
print("bitwise identical" if same else "DIFFERENT", {f: float(np.max(np.abs(getattr(outs[0], f) - getattr(outs[1], f))))
                                                   for f in ("position", "scale", "quaternion", "sigma", "sh")})
sys.exit(0 if same else 1)
