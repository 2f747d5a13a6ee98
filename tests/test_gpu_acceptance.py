"""The reference's acceptance criteria and trainer tests that pin this path, re-run
against the CUDA library (SURVEY.md §4 "must be re-run against
the GPU build"):

  * criterion 2, rasterizer oracle over 100 scenes (proj/tests/acceptance.cpp:67-113);
  * criterion 7, kernel invariants and determinism over a 504-step run (:180-238);
  * criterion 8, fixed point of training against its own renders (:243-274);
  * test_trainer.cpp:69-85 (self-rendered fixed point) and :101-118 (same seed ->
    same curve).

Where the reference's bound is a float64 statement the GPU's FP32 hot loop cannot
meet literally (criterion 2's 1e-12 for the cutoff-free tiled render), the bound
used here is stated next to it.
"""
import numpy as np
import pytest

from paper_2501_13975_b200 import capi
from refimpl import accept_raster_scene, ref, render_reference, synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    return capi.product()


def test_criterion2_rasterizer_oracle(gpu):
    """100 random scenes (20..200 kernels, SH3, 64x64): the GPU's cutoff-free render against
    the reference's exact per-pixel render (render_reference, rasterizer.hpp:452-458) and the
    GPU's default render against it. Reference bounds: 1e-12 (float64) and 2e-3. GPU bounds:
    1e-5 for the cutoff-free render (FP32 alpha/T hot loop, FP64 colour sums) and the
    reference's own 2e-3 for the default render."""
    worst_exact = worst_default = 0.0
    g = gpu.context()
    r = ref().context()
    for trial in range(100):
        scene, cam = accept_raster_scene(trial)
        g.set_scene(scene)
        r.set_scene(scene)
        exact = render_reference(r, cam)
        tiled = g.render(cam, gpu.reference_raster())
        fast = g.render(cam)
        worst_exact = max(worst_exact, float(np.max(np.abs(tiled - exact))))
        worst_default = max(worst_default, float(np.max(np.abs(fast - exact))))
    print(f"criterion 2 on the GPU: cutoffs-off max dev {worst_exact:.3e}, default max dev {worst_default:.3e}")
    assert worst_exact <= 1e-5
    assert worst_default <= 2e-3


def _self_consistent(gpu_lib, synth_kw):
    """Scene = truth with sigma = 0.5 (barrier-stationary), targets rendered by the GPU's own
    trainer render path (test_trainer.cpp:29-39; acceptance.cpp:244-261)."""
    d = synth(**synth_kw)
    scene = d["truth"].copy()
    scene.sigma[:] = 0.5
    c = gpu_lib.context()
    c.set_scene(scene)
    targets = [c.render(cam) for cam in d["cameras"]]
    c.close()
    return scene, d, targets


@pytest.mark.parametrize("which", ["criterion8", "test_trainer_fixed_point"])
def test_fixed_point_against_own_renders(gpu, which):
    if which == "criterion8":  # standard_fixture(777) with perturbation 0, 2 epochs (16 steps)
        kw = dict(seed=777, kernels=100, views=8, probe_views=4, width=64, height=64, perturbation=0.0,
                  secondary_downsample=1)
        epochs = 2
    else:  # self_consistent_fixture(21): small_params(21, 0.0), 1 epoch
        kw = dict(seed=21, kernels=20, views=4, probe_views=0, width=48, height=48, perturbation=0.0,
                  secondary_downsample=2)
        epochs = 1
    scene, d, targets = _self_consistent(gpu, kw)
    c = gpu.context()
    c.set_scene(scene)
    cfg = gpu.default_train()
    cfg.epochs = epochs
    cfg.knn = 0  # box-filtered secondaries are never matched exactly: single-view objective
    c.trainer_configure(cfg, d["cameras"], targets, d["train"], d["probe"])
    rows = c.trainer_run(epochs, len(d["train"]))
    assert len(rows) > 1
    worst_delta = max(max(rows[i].delta_norms) for i in range(1, min(len(rows), 11)))
    worst_drift = max(abs(rows[i].probe_loss - rows[0].probe_loss) for i in range(1, min(len(rows), 11)))
    print(f"{which}: {len(rows) - 1} steps, max delta norm {worst_delta:.3e}, probe drift {worst_drift:.3e}")
    assert worst_delta < 1e-8
    assert worst_drift < 1e-10


def test_same_seed_reproduces_the_curve(gpu):
    """test_trainer.cpp:101-118 (small_params(29, 0.7), seed 77, 1 epoch): identical image
    ids, probe losses and delta norms. The reference is deterministic for a fixed thread
    count; the GPU's equivalent is ngs_set_deterministic (exact fixed-point accumulation)."""
    d = synth(seed=29, kernels=20, views=4, probe_views=0, width=48, height=48, perturbation=0.7,
              secondary_downsample=2)
    runs = []
    for _ in range(2):
        c = gpu.context()
        c.set_deterministic(True)
        c.set_scene(d["init"])
        cfg = gpu.default_train()
        cfg.epochs = 1
        cfg.seed = 77
        c.trainer_configure(cfg, d["cameras"], d["targets"], d["train"], d["probe"], d["secondary"],
                            d["secondary_downsample"])
        runs.append([(r.image_id, r.probe_loss, tuple(r.delta_norms)) for r in c.trainer_run(1, len(d["train"]))])
        c.close()
    assert runs[0] == runs[1]


def test_criterion7_invariants_and_determinism(gpu):
    """Criterion 7 (acceptance.cpp:180-238): standard_fixture(4242), bench_train_config
    (newton, seed 4242, probe every step, full-resolution secondaries), 63 epochs = 504
    steps on 8 views: unit quaternions, sigma inside (1e-4, 1 - 1e-4), positive scales; two
    runs give identical curves (deterministic mode)."""
    d = synth(seed=4242, kernels=100, views=8, probe_views=4, width=64, height=64, perturbation=0.5,
              secondary_downsample=1)
    runs = []
    for _ in range(2):
        c = gpu.context()
        c.set_deterministic(True)
        c.set_scene(d["init"])
        cfg = gpu.default_train()
        cfg.epochs = 63
        cfg.seed = 4242
        cfg.secondary_downsample = 1
        cfg.probe_cadence = 1
        c.trainer_configure(cfg, d["cameras"], d["targets"], d["train"], d["probe"])
        rows = c.trainer_run(63, len(d["train"]))
        runs.append(([(r.image_id, r.probe_loss, r.probe_psnr, r.probe_ssim, tuple(r.delta_norms)) for r in rows],
                     c.get_scene()))
        c.close()
    (rows_a, scene_a), (rows_b, _) = runs
    assert len(rows_a) == 505
    assert rows_a == rows_b
    assert np.all(np.abs(np.linalg.norm(scene_a.quaternion, axis=1) - 1.0) < 1e-6)  # FP32 storage (ref: 1e-9)
    assert np.all(scene_a.sigma > 1e-4) and np.all(scene_a.sigma < 1 - 1e-4)
    assert np.all(scene_a.scale > 0)
    print(f"criterion 7: {len(rows_a) - 1} steps, probe loss {rows_a[0][1]:.5f} -> {rows_a[-1][1]:.5f}")
