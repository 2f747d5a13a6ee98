"""BASELINE config 5 (rasterizer fwd+bwd microbenchmark): 6M Gaussians at 3840x2160, SH3,
large heavily overlapping splats. Times one view's render + loss (ngs_build_view) and its
position backward (ngs_accumulate) through the C-ABI on cuda:0. Inputs exceed the L2.

  python tools/c5_bench.py [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_13975_b200 import capi  # noqa: E402
from paper_2501_13975_b200.workload import Config, cameras_for, footprint_factor, make_scenes  # noqa: E402

C5 = Config("c5", 6_000_000, 1, 3840, 2160, 3, 4.0 * footprint_factor(6_000_000))
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
lib = capi.product()
truth, init = make_scenes(C5, seed=77)
cam = cameras_for(C5, total=8)[3]
ctx = lib.context(0)
ctx.set_scene(truth)
target = ctx.render(cam)
ctx.set_scene(init)


for _ in range(2):  # warm-up (allocations, capacities)
    ctx.build_view(0, cam, target)
    ctx.accumulate(0, 0)
# Device time per stage from the library's per-launch CUDA events (ngs_profile_*): the
# host-side target upload and the accumulator read-back of the API calls are excluded.
ctx.profile_reset()
ctx.profile_enable(True)
for _ in range(reps):
    ctx.build_view(0, cam, target)
    ctx.accumulate(0, 0)
prof = ctx.profile_read()
ms = {k: v / reps for k, v in prof["ms"].items() if v > 0}
info = ctx.view_info(0)
fw = sum(ms.get(k, 0.0) for k in ("project", "sort", "raster", "loss"))
bw = sum(ms.get(k, 0.0) for k in ("consts", "bwd_position"))
print(f"c5: {info.entries} projected, {info.pairs} (tile, splat) pairs")
print("  device ms per view:", {k: round(v, 3) for k, v in ms.items()})
print(f"  forward (project + sort + raster + loss) {fw:.2f} ms = {info.pairs / fw / 1e6:.2f} G pairs/s; "
      f"position backward (world-axis terms, constants + traversal) {bw:.2f} ms; mean of {reps}")
