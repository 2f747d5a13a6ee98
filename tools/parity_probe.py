"""Dump per-pass solved deltas of the GPU library, the reference, and the reference on
1-FP32-ulp-perturbed inputs (the intrinsic sensitivity of the computation) at C1 / the
C2-shaped slice, for offline analysis. Test tooling, not product code."""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
from paper_2501_13975_b200 import capi  # noqa: E402
from refimpl import ref  # noqa: E402
import test_gpu_scale_parity as T  # noqa: E402


def main(name, out):
    d = T.make_fixture(10_000, 0, 1.0, 1000) if name == "c1" else T.make_fixture(30_000, 3, T.C2_SLICE_SCALE, 1001)
    gpu = capi.product()
    tr = ref().context()
    tr.set_scene(d["init"])
    tr.trainer_configure(ref().default_train(), d["cameras"], d["targets"], d["train"], d["probe"])
    view = d["train"][0]
    nbrs = tr.trainer_neighbors(view)
    tr.close()
    views = [(d["cameras"][view], d["targets"][view])]
    for nb in nbrs:
        views.append((d["cameras"][nb].downsampled(4), T.box_downsample(d["targets"][nb], 4)))
    ro = ref().default_raster()
    ro.threads = os.cpu_count() or 1
    res = {}
    scene = d["init"]
    for attr in T.ATTRS:
        a = capi.ATTRIBUTES[attr]
        for tag, lib, sc in (("gpu", gpu, scene), ("ref", ref(), scene), ("refp", ref(), T.perturb_ulp(scene, attr))):
            c = lib.context()
            c.set_scene(sc)
            for slot, (cam, tgt) in enumerate(views):
                c.build_view(slot, cam, tgt, raster=ro if lib is ref() else None)
            g_, h_, v_ = c.accumulate(attr, 0, list(range(1, len(views))))
            if attr != capi.COLOR:  # dense SH3 colour blocks are 6 KB per Gaussian: too big to ship back
                res[f"{a}.{tag}.grad"], res[f"{a}.{tag}.hess"] = g_.astype(np.float32), h_.astype(np.float32)
            res[f"{a}.{tag}.visible"] = v_
            r = c.newton_step(attr, 0, list(range(1, len(views))))
            res[f"{a}.{tag}.delta"] = r["delta"]
            res[f"{a}.{tag}.accepted"] = r["accepted"]
            res[f"{a}.{tag}.degenerate"] = r["degenerate"]
            if tag == "ref":
                nxt = T.f32(c.get_scene())
            c.close()
        e = T.rel_dist(res[f"{a}.gpu.delta"], res[f"{a}.ref.delta"])
        ep = T.rel_dist(res[f"{a}.refp.delta"], res[f"{a}.ref.delta"])
        print(f"{name} {a}: gpu-vs-ref {e}  refp-vs-ref {ep}", flush=True)
        for k, v in (("position", scene.position), ("scale", scene.scale), ("quaternion", scene.quaternion),
                     ("sigma", scene.sigma)):
            res[f"{a}.scene.{k}"] = v
        scene = nxt
    np.savez_compressed(out, **res)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
