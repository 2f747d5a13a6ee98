"""CPU suite: the numpy restatement (oracle/ngs_oracle.py) pinned against golden
vectors produced by the reference itself (tests/golden/make_golden.py), plus the
reference's closed-form known answers.
"""
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REPO, "oracle"))

import ngs_oracle as O  # noqa: E402
from paper_2501_13975_b200 import capi  # noqa: E402

GOLD = os.path.join(REPO, "tests", "golden")
TOL = 1e-7  # float64 restatement vs float64 reference: summation order (numpy vs loops), eigen routines


def load(name):
    return dict(np.load(os.path.join(GOLD, name)))


def scene_from(g, p):
    return capi.Scene(g[p + "position"], g[p + "scale"], g[p + "quaternion"], g[p + "sigma"], g[p + "sh"],
                      g[p + "background"], int(g[p + "sh_degree"]))


def cam_from(g, p):
    w, h = g[p + "size"]
    return capi.Camera(g[p + "view"], g[p + "proj"], int(w), int(h))


def rel(a, b, floor_frac=1e-6):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    floor = max(floor_frac * float(np.max(np.abs(b))) if b.size else 0, 1e-300)
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor))) if b.size else 0.0


@pytest.fixture(scope="module")
def render_gold():
    return load("render.npz")


@pytest.fixture(scope="module")
def newton_gold():
    return load("newton.npz")


@pytest.fixture(scope="module")
def newton_ctx(newton_gold):
    g = newton_gold
    ctx = O.OracleContext()
    ctx.set_scene(scene_from(g, "s_"))
    lv = ctx.build_view(0, cam_from(g, "c_"), g["target"])
    for i in range(2):
        ctx.build_view(1 + i, cam_from(g, f"sec{i}_"), g[f"sec{i}_target"])
    return ctx, lv


def test_oracle_render_default(render_gold):
    g = render_gold
    ctx = O.OracleContext()
    ctx.set_scene(scene_from(g, "s_"))
    img = ctx.render(cam_from(g, "c_"))
    assert np.max(np.abs(img - g["image_default"])) < 1e-12


def test_oracle_render_reference_mode(render_gold):
    g = render_gold
    ctx = O.OracleContext()
    ctx.set_scene(scene_from(g, "s_"))
    img = ctx.render(cam_from(g, "c_"), O.REFERENCE_RASTER)
    assert np.max(np.abs(img - g["image_reference"])) < 1e-12


def test_oracle_binning_exact(render_gold):
    g = render_gold
    ctx = O.OracleContext()
    ctx.set_scene(scene_from(g, "s_"))
    ctx.build_view(0, cam_from(g, "c_"), np.zeros((32, 48, 3)))
    sp = ctx.view_splats(0)
    assert np.array_equal(sp["kernel"], g["splat_kernel"])
    assert np.array_equal(sp["tile_offsets"], g["splat_tile_offsets"])
    assert np.array_equal(sp["tile_indices"], g["splat_tile_indices"])


def test_bin_entries_reproduces_reference_csr(render_gold):
    """The sort+bin contract (rasterizer.hpp:228-263) on supplied depth/bbox —
    the function the GPU binning test applies to the GPU's own entries."""
    g = render_gold
    order = np.argsort(np.random.default_rng(0).random(len(g["splat_kernel"])))  # scrambled input order
    kern, offs, idx = O.bin_entries(list(g["splat_kernel"][order]), list(g["splat_depth"][order]),
                                    list(g["splat_bbox"][order]), 48, 32)
    assert np.array_equal(np.array(kern), g["splat_kernel"])
    assert np.array_equal(offs, g["splat_tile_offsets"])
    assert np.array_equal(idx, g["splat_tile_indices"])


def test_oracle_loss_fields(newton_gold, newton_ctx):
    ctx, lv = newton_ctx
    g = newton_gold
    assert abs(lv - float(g["loss_value"])) <= 1e-12 * abs(float(g["loss_value"]))
    gr, hs = ctx.view_loss_derivs(0)
    assert np.max(np.abs(ctx.view_image(0) - g["image"])) < 1e-12
    assert rel(gr, g["loss_grad"]) < TOL
    assert rel(hs, g["loss_hess"]) < TOL


@pytest.mark.parametrize("attr", range(5))
def test_oracle_terms(newton_gold, newton_ctx, attr):
    ctx, _ = newton_ctx
    name = capi.ATTRIBUTES[attr]
    gg, hh, vis = ctx.accumulate(attr, 0, [1, 2])
    assert np.array_equal(vis, newton_gold[f"terms_{name}_visible"])
    assert rel(gg, newton_gold[f"terms_{name}_grad"]) < TOL
    assert rel(hh, newton_gold[f"terms_{name}_hess"]) < TOL


@pytest.mark.parametrize("attr", range(5))
def test_oracle_solves(newton_gold, attr):
    g = newton_gold
    name = capi.ATTRIBUTES[attr]
    ctx = O.OracleContext()
    ctx.set_scene(scene_from(g, "s_"))
    ctx.build_view(0, cam_from(g, "c_"), g["target"])
    for i in range(2):
        ctx.build_view(1 + i, cam_from(g, f"sec{i}_"), g[f"sec{i}_target"])
    res = ctx.newton_step(attr, 0, [1, 2])
    assert rel(res["delta"], g[f"solve_{name}_delta"]) < 1e-7
    assert np.array_equal(res["accepted"], g[f"solve_{name}_accepted"])
    assert np.array_equal(res["degenerate"], g[f"solve_{name}_degenerate"])
    assert abs(res["delta_norm_sq"] - float(g[f"solve_{name}_norm_sq"])) <= 1e-7 * abs(float(g[f"solve_{name}_norm_sq"]))


# ---- closed-form known answers from the reference's own suites -------------

def test_psd_safeguard_known_answers():
    """test_newton.cpp:58-72."""
    s = O.psd_safeguard(np.diag([2.0, -1.0]))
    assert np.allclose(s, np.diag([2.0, 1.0]), atol=1e-12)
    assert O.psd_safeguard(np.array([[-1e-12]]))[0, 0] == pytest.approx(O.K_RIDGE_MIN)
    h = np.array([[3.0, 0.5], [0.5, 1.0]])
    assert np.array_equal(O.psd_safeguard(h), h)


def test_gaussian_weight_stationary_point():
    """test_rasterizer.cpp:36-44."""
    S = np.array([[2.0, 0.3], [0.3, 1.5]])
    d = O.gaussian_weight(S, np.array([10.0, 20.0]), np.array([10.0, 20.0]))
    assert d["g"] == 1.0 and np.linalg.norm(d["d_pi"]) == 0.0
    assert np.max(np.abs(d["d2_pi"] + np.linalg.inv(S))) < 1e-14


def test_l2_gradient_known_answer():
    """test_loss.cpp:72-80: L2 gradient (c - c^t) / (3N)."""
    img = np.full((16, 16, 3), 0.5)
    tgt = img.copy()
    tgt[3, 4, 1] = 0.5 - 0.768
    cfg = dict(O.DEFAULT_LOSS)
    cfg["lambda"] = 0.0
    _, g, h = O.total_loss_derivs(img, tgt, cfg)
    assert g[3, 4, 1] == pytest.approx(0.768 / (3 * 256))
    assert h[0, 0, 0] == pytest.approx(1.0 / (3 * 256))


def test_single_centered_kernel():
    """test_rasterizer.cpp:218-229 (pixel (32, 32) == 0.8)."""
    from paper_2501_13975_b200.workload import make_lookat_view, make_perspective_proj
    cam = capi.Camera(make_lookat_view([0, 0, -4], [0, 0, 0], [0, 1, 0]),
                      make_perspective_proj(np.pi / 3, 1.0, 0.05, 100.0), 65, 65)
    s = capi.Scene.empty(1, 3)
    s.scale[:] = 0.05
    s.sigma[:] = 0.8
    s.sh[0, :, 0] = (np.array([1.0, 0.0, 0.0]) - 0.5) / O.SH0
    ctx = O.OracleContext()
    ctx.set_scene(s)
    img = ctx.render(cam)
    assert img[32, 32, 0] == pytest.approx(0.8, rel=1e-12)
    assert img[32, 32, 1] == 0.0


def test_oracle_trainer_step_matches_reference():
    """Trainer::step (trainer.hpp:185-207, 299-417) on the reference's synth fixture."""
    g = load("trainer.npz")
    ctx = O.OracleContext()
    ctx.set_scene(scene_from(g, "init_"))
    n_cams = len([k for k in g if k.startswith("cam") and k.endswith("_view")])
    cams = [cam_from(g, f"cam{i}_") for i in range(n_cams)]
    tr = O.OracleTrainer(ctx, cams, [g[f"target{i}"] for i in range(n_cams)], list(range(n_cams)),
                         [g[f"sec_target{i}"] for i in range(n_cams)], 2, knn=2, downsample=2)
    assert tr.neighbors[0] == list(g["neighbors0"])
    norms = tr.step(0)
    assert rel(norms, g["delta_norms"]) < 1e-7
    post = ctx.get_scene_arrays()
    for f in ("position", "scale", "quaternion", "sigma", "sh"):
        assert rel(post[f], g["post_" + f]) < 1e-7, f


# ---------------------------------------------------------------------------
# Evaluation path: metrics, probe_metrics, run
# ---------------------------------------------------------------------------

def test_rng_is_mt19937_64():
    """ngs::Rng wraps std::mt19937_64 (core.hpp:52-83): the C++ standard's
    known answer ([rand.predef]: 10000th output of the default engine)."""
    r = O.Rng(5489)
    assert r.next() == 14514284786278117030
    r = O.Rng(5489)
    for _ in range(9999):
        r.next()
    assert r.next() == 9981545732273789042
    v = O.Rng(3).shuffle(list(range(10)))
    assert sorted(v) == list(range(10)) and v != list(range(10))


def _eval_fixture():
    g = load("eval.npz")
    n = len([k for k in g if k.startswith("cam") and k.endswith("_view")])
    cams = [cam_from(g, f"cam{i}_") for i in range(n)]
    targets = [g[f"target{i}"] for i in range(n)]
    return g, cams, targets


def test_oracle_metrics_match_reference():
    """total_loss_value / psnr / ssim_metric (loss.hpp:359-375, metrics.hpp:14-30)."""
    g, cams, targets = _eval_fixture()
    ctx = O.OracleContext()
    ctx.set_scene(scene_from(g, "init_"))
    img = ctx.render(cams[0])
    got = [O.total_loss_value(img, targets[0], O.DEFAULT_LOSS), O.psnr(img, targets[0]),
           O.ssim_mean_value(img, targets[0], O.DEFAULT_LOSS)]
    assert rel(got, g["view_metrics"]) < TOL
    img = ctx.render(cams[1])
    l2 = dict(O.DEFAULT_LOSS, **{"lambda": 0.0})
    got = [O.total_loss_value(img, targets[1], l2), O.psnr(img, targets[1]), O.ssim_mean_value(img, targets[1], l2)]
    assert rel(got, g["view_metrics_l2"]) < TOL
    assert O.psnr(img, img) == float("inf")


def test_oracle_run_matches_reference():
    """Trainer::run (trainer.hpp:238-277): shuffled order, probe cadence, barrier decay."""
    g, cams, targets = _eval_fixture()
    epochs, seed, cadence = (int(x) for x in g["run_cfg"])
    ctx = O.OracleContext()
    ctx.set_scene(scene_from(g, "init_"))
    n = len(cams)
    tr = O.OracleTrainer(ctx, cams, targets, list(g["train"]), [g[f"sec_target{i}"] for i in range(n)], 2, knn=2,
                         downsample=2)
    p0 = tr.probe_metrics(list(g["probe"]))
    assert rel(p0, g["probe0"]) < TOL
    rows = tr.run(epochs=epochs, seed=seed, probe_cadence=cadence, probe_ids=list(g["probe"]))
    assert [[r[0], r[1]] for r in rows] == g["run_ids"].tolist()
    assert rel([r[2] for r in rows], g["run_probe"]) < TOL
    assert rel([r[3] for r in rows], g["run_norms"]) < TOL
    assert tr.barrier == pytest.approx(float(g["barrier_after"]), rel=1e-15)
    post = ctx.get_scene_arrays()
    for f in ("position", "scale", "quaternion", "sigma", "sh"):
        assert rel(post[f], g["post_" + f]) < TOL, f


def test_oracle_first_order_matches_reference():
    """first_order_step (trainer.hpp:419-509): GD and Adam baselines, two steps each."""
    g = load("first_order.npz")
    n = len([k for k in g if k.startswith("cam") and k.endswith("_view")])
    cams = [cam_from(g, f"cam{i}_") for i in range(n)]
    targets = [g[f"target{i}"] for i in range(n)]
    for name, adam in (("gd", False), ("adam", True)):
        ctx = O.OracleContext()
        ctx.set_scene(scene_from(g, "init_"))
        tr = O.OracleTrainer(ctx, cams, targets, list(range(n)), knn=0)
        state = dict(t=0, m=np.zeros((ctx.scene["n"], 56)), v=np.zeros((ctx.scene["n"], 56)))
        norms = [tr.first_order_step(int(v), adam, g[f"{name}_lr"], state) for v in g["steps"]]
        assert rel(norms, g[f"{name}_norms"]) < TOL, name
        post = ctx.get_scene_arrays()
        for f in ("position", "scale", "quaternion", "sigma", "sh"):
            assert rel(post[f], g[f"{name}_post_" + f]) < TOL, (name, f)
