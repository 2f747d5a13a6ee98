"""GPU parity against the committed golden vectors (tests/golden, produced by the
reference itself): runs without the oracle libraries, through the C-ABI only."""
import os

import numpy as np
import pytest

from paper_2501_13975_b200 import capi
from test_oracle import cam_from, load, scene_from

pytestmark = pytest.mark.gpu
FLOOR = 1e-3


def qerr(a, b, floor_frac=FLOOR):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    floor = max(floor_frac * float(np.max(np.abs(b))), 1e-300)
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)))


@pytest.fixture(scope="module")
def gpu():
    return capi.product()


def test_golden_render_and_binning(gpu):
    g = load("render.npz")
    ctx = gpu.context()
    ctx.set_scene(scene_from(g, "s_"))
    cam = cam_from(g, "c_")
    assert np.max(np.abs(ctx.render(cam) - g["image_default"])) < 1e-6
    assert np.max(np.abs(ctx.render(cam, gpu.reference_raster()) - g["image_reference"])) < 1e-6
    ctx.build_view(0, cam, np.zeros((32, 48, 3)))
    sp = ctx.view_splats(0)
    assert np.array_equal(sp["kernel"], g["splat_kernel"])
    assert np.array_equal(sp["tile_offsets"], g["splat_tile_offsets"])
    assert np.array_equal(sp["tile_indices"], g["splat_tile_indices"])


@pytest.mark.parametrize("attr", range(5))
def test_golden_terms_and_solves(gpu, attr):
    g = load("newton.npz")
    name = capi.ATTRIBUTES[attr]

    def views(ctx):
        ctx.set_scene(scene_from(g, "s_"))
        lv = ctx.build_view(0, cam_from(g, "c_"), g["target"])
        for i in range(2):
            ctx.build_view(1 + i, cam_from(g, f"sec{i}_"), g[f"sec{i}_target"])
        return lv

    ctx = gpu.context()
    lv = views(ctx)
    assert abs(lv - float(g["loss_value"])) <= 1e-5 * abs(float(g["loss_value"]))
    gg, hh, vis = ctx.accumulate(attr, 0, [1, 2])
    assert np.array_equal(vis, g[f"terms_{name}_visible"])
    # colour gradients are sums of gl * w whose terms cancel most (TOL_DELTA-level)
    assert qerr(gg, g[f"terms_{name}_grad"]) < (2e-3 if attr == capi.COLOR else 1e-3)
    assert qerr(hh, g[f"terms_{name}_hess"]) < 1e-3
    ctx2 = gpu.context()
    views(ctx2)
    res = ctx2.newton_step(attr, 0, [1, 2])
    # The safeguarded solve amplifies gradient error by at most 1 / eig_floor_rel = 20 along the
    # weakest kept eigen-direction; colour systems (rank <= views) sit at that bound most often.
    assert qerr(res["delta"], g[f"solve_{name}_delta"]) < (1e-2 if attr == capi.COLOR else 2e-3)
    assert np.array_equal(res["accepted"], g[f"solve_{name}_accepted"])


def test_golden_trainer_step(gpu):
    g = load("trainer.npz")
    ctx = gpu.context()
    ctx.set_scene(scene_from(g, "init_"))
    n = len([k for k in g if k.startswith("cam") and k.endswith("_view")])
    cfg = gpu.default_train()
    cfg.knn = 2
    cfg.secondary_downsample = 2
    ctx.trainer_configure(cfg, [cam_from(g, f"cam{i}_") for i in range(n)], [g[f"target{i}"] for i in range(n)],
                          list(range(n)), [], [g[f"sec_target{i}"] for i in range(n)], 2)
    assert ctx.trainer_neighbors(0) == list(g["neighbors0"])
    rep = ctx.trainer_step(0)
    assert qerr(list(rep.delta_norms), g["delta_norms"]) < 1e-3
    post = ctx.get_scene()
    for f in ("position", "scale", "sigma", "sh"):
        assert qerr(getattr(post, f), g["post_" + f]) < 1e-4, f
    # orientation: rotation angle between GPU and reference quaternions; the solved spin
    # theta (|2 theta| <= pi) carries the ~1e-4 relative error of the rotation terms
    dots = np.abs(np.sum(post.quaternion * g["post_quaternion"], axis=1))
    assert np.max(2 * np.arccos(np.clip(dots, -1, 1))) < 1e-3


# ---------------------------------------------------------------------------
# Evaluation path: metrics, probe_metrics, run
# ---------------------------------------------------------------------------

def _eval_ctx(gpu, g):
    ctx = gpu.context()
    ctx.set_scene(scene_from(g, "init_"))
    n = len([k for k in g if k.startswith("cam") and k.endswith("_view")])
    cams = [cam_from(g, f"cam{i}_") for i in range(n)]
    return ctx, cams, [g[f"target{i}"] for i in range(n)]


def test_golden_view_metrics(gpu):
    """total_loss_value / psnr / ssim_metric of the GPU render (loss.hpp:359-375, metrics.hpp)."""
    g = load("eval.npz")
    ctx, cams, targets = _eval_ctx(gpu, g)
    m = ctx.view_metrics(cams[0], targets[0])
    assert qerr([m.loss, m.psnr, m.ssim], g["view_metrics"]) < 1e-5
    lc = gpu.default_loss()
    lc.lambda_ = 0.0
    m = ctx.view_metrics(cams[1], targets[1], loss=lc)
    assert qerr([m.loss, m.psnr, m.ssim], g["view_metrics_l2"]) < 1e-5
    own = ctx.render(cams[1])
    m = ctx.view_metrics(cams[1], own)
    assert m.psnr == float("inf") and abs(m.ssim - 1.0) < 1e-9 and m.loss < 1e-12


def test_golden_probe_and_run(gpu):
    """Trainer::probe_metrics + Trainer::run: same shuffled view order (exact), probe
    rows and delta norms within the trainer-step tolerances."""
    g = load("eval.npz")
    ctx, cams, targets = _eval_ctx(gpu, g)
    epochs, seed, cadence = (int(x) for x in g["run_cfg"])
    cfg = gpu.default_train()
    cfg.knn = 2
    cfg.secondary_downsample = 2
    cfg.epochs, cfg.seed, cfg.probe_cadence = epochs, seed, cadence
    ctx.trainer_configure(cfg, cams, targets, list(g["train"]), list(g["probe"]),
                          [g[f"sec_target{i}"] for i in range(len(cams))], 2)
    p0 = ctx.trainer_probe()
    assert qerr([p0.loss, p0.psnr, p0.ssim], g["probe0"]) < 1e-5
    rows = ctx.trainer_run(epochs, len(g["train"]))
    assert [[r.step, r.image_id] for r in rows] == g["run_ids"].tolist()
    assert qerr([[r.probe_loss, r.probe_psnr, r.probe_ssim] for r in rows], g["run_probe"]) < 1e-4
    assert qerr([list(r.delta_norms) for r in rows], g["run_norms"]) < 2e-3
    assert ctx.barrier_weight() == pytest.approx(float(g["barrier_after"]), rel=1e-12)


def test_golden_first_order(gpu):
    """GD / Adam baselines on the GPU (one image-space gradient traversal + chain kernel)."""
    g = load("first_order.npz")
    n = len([k for k in g if k.startswith("cam") and k.endswith("_view")])
    cams = [cam_from(g, f"cam{i}_") for i in range(n)]
    for name, opt in (("gd", 1), ("adam", 2)):
        ctx = gpu.context()
        ctx.set_scene(scene_from(g, "init_"))
        cfg = gpu.default_train()
        cfg.optimizer = opt
        ctx.trainer_configure(cfg, cams, [g[f"target{i}"] for i in range(n)], list(range(n)))
        norms = [list(ctx.trainer_step(int(v)).delta_norms) for v in g["steps"]]
        print(name, np.array(norms), g[f"{name}_norms"])
        assert qerr(norms, g[f"{name}_norms"]) < 2e-3, name
        post = ctx.get_scene()
        for f in ("position", "scale", "sigma", "sh"):
            assert qerr(getattr(post, f), g[f"{name}_post_" + f]) < 1e-4, (name, f)
        dots = np.abs(np.sum(post.quaternion * g[f"{name}_post_quaternion"], axis=1))
        assert np.max(2 * np.arccos(np.clip(dots, -1, 1))) < 1e-3, name
