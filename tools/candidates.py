"""Phase-1 candidate statistics of the backward (debug build): how many warp-level splat
iterations phase 1 runs, how many of them yield >= 1 contributing record, and the records.
  tools/build_variant.sh cand -DNGS_COUNT_CANDIDATES=1
  python tools/candidates.py paper_2501_13975_b200/lib/cand.so     (GPU box; stats on stderr)
Tooling."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_13975_b200 import capi  # noqa: E402
from paper_2501_13975_b200.workload import CONFIGS, cameras_for, make_scenes  # noqa: E402

lib = capi.NgsLibrary(sys.argv[1])
cfg = CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "c2"]
ctx = lib.context(0)
truth, init = make_scenes(cfg)
cams = cameras_for(cfg)
ctx.set_scene(truth)
targets = [ctx.render(c) for c in cams]
ctx.set_scene(init)
ctx.trainer_configure(lib.default_train(), cams, targets, list(range(cfg.views)))
for i in range(3):
    ctx.trainer_step(i)
ctx.profile_read()  # prints and clears the warm-up counts
ctx.profile_reset()
ctx.trainer_step(5)
p = ctx.profile_read()  # one step
print(cfg.name, "records per pass", p["contrib_pairs"], "primary", p["primary_contrib_pairs"])
