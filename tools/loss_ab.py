"""Bitwise A/B of the view loss (value, gradient and diagonal Hessian fields) between two
builds of libngs_b200.so, on BASELINE-size and odd-size views. Tooling (GPU).
  python tools/loss_ab.py paper_2501_13975_b200/lib/base.so paper_2501_13975_b200/lib/libngs_b200.so"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2501_13975_b200 import capi  # noqa: E402
from paper_2501_13975_b200.workload import CONFIGS, cameras_for, make_scenes  # noqa: E402

libs = [capi.NgsLibrary(p) for p in sys.argv[1:3]]
ok = True
for name, (w, h) in (("c2", (800, 800)), ("c2", (801, 603)), ("c2", (962, 540)), ("c1", (256, 256)),
                     ("c2", (200, 200))):
    cfg = CONFIGS[name]
    truth, init = make_scenes(cfg)
    cam = cameras_for(cfg)[0]
    cam.width, cam.height = w, h
    outs = []
    for lib in libs:
        ctx = lib.context(0)
        ctx.set_scene(truth)
        target = ctx.render(cam)
        ctx.set_scene(init)
        val = ctx.build_view(0, cam, target)
        g, hh = ctx.view_loss_derivs(0)
        outs.append((val, g, hh))
        ctx.close()
    (v0, g0, h0), (v1, g1, h1) = outs
    same = v0 == v1 and np.array_equal(g0, g1) and np.array_equal(h0, h1)
    ok &= same
    print(f"{name} {w}x{h}: loss {v0!r} vs {v1!r}; grad max|d| {np.max(np.abs(g0 - g1)):.3e}, "
          f"hess max|d| {np.max(np.abs(h0 - h1)):.3e}: {'bit-identical' if same else 'DIFFERENT'}")
sys.exit(0 if ok else 1)
