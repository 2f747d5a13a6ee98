#!/usr/bin/env python3
"""Generate tests/golden/*.npz from the REFERENCE itself.

Runs the unmodified reference (oracle/_ref/libngs_ref.so: /root/reference
headers compiled against oracle/eigen_shim) on the reference's own fixture
generators and stores inputs + outputs. These vectors pin both the numpy
restatement (oracle/ngs_oracle.py) and, on the GPU box, the CUDA library.

  python tests/golden/make_golden.py      (needs oracle/_ref built: make -C oracle)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from paper_2501_13975_b200 import capi  # noqa: E402
from refimpl import check_fixture, random_scene, ref, synth, test_camera  # noqa: E402


def scene_arrays(s, prefix):
    return {f"{prefix}position": s.position, f"{prefix}scale": s.scale, f"{prefix}quaternion": s.quaternion,
            f"{prefix}sigma": s.sigma, f"{prefix}sh": s.sh, f"{prefix}background": s.background,
            f"{prefix}sh_degree": np.array(s.sh_degree)}


def cam_arrays(c, prefix):
    return {f"{prefix}view": np.asarray(c.view), f"{prefix}proj": np.asarray(c.proj),
            f"{prefix}size": np.array([c.width, c.height])}


def f32(s):
    s = s.copy()
    for f in ("position", "scale", "quaternion", "sigma", "sh"):
        setattr(s, f, getattr(s, f).astype(np.float32).astype(np.float64))
    return s


def render_golden():
    L = ref()
    scene = f32(random_scene(103, 30))
    cam = test_camera((0.3, -0.2, -3.4), 48, 32)
    ctx = L.context()
    ctx.set_scene(scene)
    out = dict(scene_arrays(scene, "s_"), **cam_arrays(cam, "c_"))
    out["image_default"] = ctx.render(cam)
    out["image_reference"] = ctx.render(cam, L.reference_raster())
    ctx.build_view(0, cam, np.zeros((32, 48, 3)))
    sp = ctx.view_splats(0)
    for k in ("kernel", "pixel", "depth", "cov2d", "view_color", "clamped", "bbox", "tile_offsets", "tile_indices"):
        out["splat_" + k] = sp[k]
    np.savez_compressed(os.path.join(HERE, "render.npz"), **out)


def newton_golden():
    L = ref()
    scene, cam, target = check_fixture(7)
    scene = f32(scene)
    r = L.context()
    r.set_scene(scene)
    secs = []
    for eye in [(1.0, 0.5, -3.0), (-1.2, 0.3, -2.9)]:
        c = test_camera(eye, 24, 24)
        secs.append((c, r.render(c)))
    out = dict(scene_arrays(scene, "s_"), **cam_arrays(cam, "c_"), target=target)
    for i, (c, t) in enumerate(secs):
        out.update(cam_arrays(c, f"sec{i}_"))
        out[f"sec{i}_target"] = t

    def views(ctx):
        ctx.set_scene(scene)
        lv = ctx.build_view(0, cam, target)
        for i, (c, t) in enumerate(secs):
            ctx.build_view(1 + i, c, t)
        return lv

    ctx = L.context()
    out["loss_value"] = np.array(views(ctx))
    out["image"] = ctx.view_image(0)
    out["loss_grad"], out["loss_hess"] = ctx.view_loss_derivs(0)
    for attr, name in enumerate(capi.ATTRIBUTES):
        g, h, vis = ctx.accumulate(attr, 0, [1, 2])
        out[f"terms_{name}_grad"], out[f"terms_{name}_hess"], out[f"terms_{name}_visible"] = g, h, vis
    for attr, name in enumerate(capi.ATTRIBUTES):
        c2 = L.context()
        views(c2)
        res = c2.newton_step(attr, 0, [1, 2])
        out[f"solve_{name}_delta"] = res["delta"]
        out[f"solve_{name}_accepted"] = res["accepted"]
        out[f"solve_{name}_degenerate"] = res["degenerate"]
        out[f"solve_{name}_norm_sq"] = np.array(res["delta_norm_sq"])
    np.savez_compressed(os.path.join(HERE, "newton.npz"), **out)


def trainer_golden():
    L = ref()
    d = synth(seed=23, kernels=20, views=4, probe_views=0, width=48, height=48, perturbation=0.5,
              secondary_downsample=2)
    ctx = L.context()
    ctx.set_scene(d["init"])
    cfg = L.default_train()
    cfg.knn = 2
    cfg.secondary_downsample = 2
    ctx.trainer_configure(cfg, d["cameras"], d["targets"], d["train"], d["probe"], d["secondary"],
                          d["secondary_downsample"])
    out = dict(scene_arrays(d["init"], "init_"))
    for i, c in enumerate(d["cameras"]):
        out.update(cam_arrays(c, f"cam{i}_"))
        out[f"target{i}"] = d["targets"][i]
        out[f"sec_target{i}"] = d["secondary"][i]
    out["neighbors0"] = np.array(ctx.trainer_neighbors(0))
    rep = ctx.trainer_step(0)
    out["delta_norms"] = np.array(list(rep.delta_norms))
    out.update(scene_arrays(ctx.get_scene(), "post_"))
    np.savez_compressed(os.path.join(HERE, "trainer.npz"), **out)


EVAL_RUN = dict(epochs=1, seed=7, probe_cadence=2)


def eval_golden():
    """total_loss_value / psnr / ssim_metric, probe_metrics and run (metrics.hpp,
    loss.hpp:359-375, trainer.hpp:215-277) on a synth dataset with probe views."""
    L = ref()
    d = synth(seed=29, kernels=20, views=4, probe_views=2, width=48, height=48, perturbation=0.5,
              secondary_downsample=2)
    ctx = L.context()
    ctx.set_scene(d["init"])
    out = dict(scene_arrays(d["init"], "init_"))
    n = len(d["cameras"])
    for i, c in enumerate(d["cameras"]):
        out.update(cam_arrays(c, f"cam{i}_"))
        out[f"target{i}"] = d["targets"][i]
        out[f"sec_target{i}"] = d["secondary"][i]
    out["train"], out["probe"] = np.array(d["train"]), np.array(d["probe"])
    m = ctx.view_metrics(d["cameras"][0], d["targets"][0])
    out["view_metrics"] = np.array([m.loss, m.psnr, m.ssim])
    lc = L.default_loss()
    lc.lambda_ = 0.0
    m = ctx.view_metrics(d["cameras"][1], d["targets"][1], loss=lc)
    out["view_metrics_l2"] = np.array([m.loss, m.psnr, m.ssim])
    cfg = L.default_train()
    cfg.knn = 2
    cfg.secondary_downsample = 2
    cfg.epochs, cfg.seed, cfg.probe_cadence = EVAL_RUN["epochs"], EVAL_RUN["seed"], EVAL_RUN["probe_cadence"]
    ctx.trainer_configure(cfg, d["cameras"], d["targets"], d["train"], d["probe"], d["secondary"],
                          d["secondary_downsample"])
    m = ctx.trainer_probe()
    out["probe0"] = np.array([m.loss, m.psnr, m.ssim])
    rows = ctx.trainer_run(cfg.epochs, len(d["train"]))
    out["run_ids"] = np.array([[r.step, r.image_id] for r in rows])
    out["run_probe"] = np.array([[r.probe_loss, r.probe_psnr, r.probe_ssim] for r in rows])
    out["run_norms"] = np.array([list(r.delta_norms) for r in rows])
    out["barrier_after"] = np.array(ctx.barrier_weight())
    out["run_cfg"] = np.array([EVAL_RUN["epochs"], EVAL_RUN["seed"], EVAL_RUN["probe_cadence"]])
    out.update(scene_arrays(ctx.get_scene(), "post_"))
    np.savez_compressed(os.path.join(HERE, "eval.npz"), **out)


FO_STEPS = (1, 3)  # view ids of the two first-order steps


def first_order_golden():
    """first_order_step (trainer.hpp:419-509): two GD and two Adam steps."""
    L = ref()
    d = synth(seed=31, kernels=20, views=4, probe_views=0, width=48, height=48, perturbation=0.5,
              secondary_downsample=2)
    out = dict(scene_arrays(d["init"], "init_"))
    for i, c in enumerate(d["cameras"]):
        out.update(cam_arrays(c, f"cam{i}_"))
        out[f"target{i}"] = d["targets"][i]
    for name, opt in (("gd", 1), ("adam", 2)):
        ctx = L.context()
        ctx.set_scene(d["init"])
        cfg = L.default_train()
        cfg.optimizer = opt
        ctx.trainer_configure(cfg, d["cameras"], d["targets"], d["train"], [], d["secondary"],
                              d["secondary_downsample"])
        norms = [list(ctx.trainer_step(v).delta_norms) for v in FO_STEPS]
        out[f"{name}_norms"] = np.array(norms)
        out.update(scene_arrays(ctx.get_scene(), f"{name}_post_"))
    lr = L.default_train()
    out["gd_lr"] = np.array([lr.gd_lr.position, lr.gd_lr.rotation, lr.gd_lr.scaling, lr.gd_lr.opacity, lr.gd_lr.color])
    out["adam_lr"] = np.array([lr.adam_lr.position, lr.adam_lr.rotation, lr.adam_lr.scaling, lr.adam_lr.opacity,
                               lr.adam_lr.color])
    out["steps"] = np.array(FO_STEPS)
    np.savez_compressed(os.path.join(HERE, "first_order.npz"), **out)


if __name__ == "__main__":
    render_golden()
    newton_golden()
    trainer_golden()
    eval_golden()
    first_order_golden()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
