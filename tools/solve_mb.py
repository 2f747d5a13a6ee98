"""Colour/Newton solve microbenchmark (BASELINE config 4) for one library build: python tools/solve_mb.py [lib.so]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_13975_b200 import capi  # noqa: E402

lib = capi.NgsLibrary(sys.argv[1]) if len(sys.argv) > 1 else capi.product()
ctx = lib.context(0)
for _ in range(2):
    ms = ctx.microbench_solve(10_000_000, sh_degree=3, views=4, reps=5)
print(os.path.basename(sys.argv[1]) if len(sys.argv) > 1 else "product", "ms per group", [round(x, 3) for x in ms],
      "total", round(sum(ms), 3), "colour fast-path fraction", round(ctx.last_color_fast_frac, 4))
