"""Error behaviour of the drop-in boundary: invalid inputs raise the same
exception kind from the CUDA library as from the reference (InvalidInput /
DegenerateGeometry / NumericalError, core.hpp:30-48), through the C-ABI."""
import numpy as np
import pytest

from paper_2501_13975_b200 import capi
from refimpl import check_fixture, ref, synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    return capi.product()


def _scene_cases():
    base, _, _ = check_fixture(1)

    def mod(f):
        s = base.copy()
        for k in ("position", "scale", "quaternion", "sigma", "sh"):
            setattr(s, k, getattr(s, k).copy())
        f(s)
        return s

    return {
        "non-unit quaternion": mod(lambda s: s.quaternion.__setitem__((0, 0), 2.0)),
        "zero scale": mod(lambda s: s.scale.__setitem__((1, 2), 0.0)),
        "opacity at 1": mod(lambda s: s.sigma.__setitem__(2, 1.0)),
        "opacity at 0": mod(lambda s: s.sigma.__setitem__(3, 0.0)),
        "background > 1": mod(lambda s: setattr(s, "background", np.array([0.1, 1.5, 0.1]))),
    }


@pytest.mark.parametrize("case", list(_scene_cases()))
def test_invalid_scene_rejected_like_the_reference(gpu, case):
    scene = _scene_cases()[case]
    kinds = []
    for lib in (gpu, ref()):
        ctx = lib.context()
        with pytest.raises(capi.NgsError) as e:
            ctx.set_scene(scene)
        kinds.append(type(e.value))
    assert kinds[0] is kinds[1] is capi.InvalidInput


@pytest.mark.parametrize("case", ["duplicate order", "negative knn", "negative epochs", "even window"])
def test_invalid_train_config_rejected_like_the_reference(gpu, case):
    d = synth(seed=23, kernels=20, views=4, probe_views=0, width=48, height=48, perturbation=0.5,
              secondary_downsample=2)
    kinds = []
    for lib in (gpu, ref()):
        ctx = lib.context()
        ctx.set_scene(d["init"])
        cfg = lib.default_train()
        if case == "duplicate order":
            cfg.order[1] = cfg.order[0]
        elif case == "negative knn":
            cfg.knn = -1
        elif case == "negative epochs":
            cfg.epochs = -1
        else:
            cfg.loss.window = 10
        with pytest.raises(capi.NgsError) as e:
            ctx.trainer_configure(cfg, d["cameras"], d["targets"], d["train"], [], d["secondary"], 2)
            ctx.trainer_step(d["train"][0])
        kinds.append(type(e.value))
    assert kinds[0] is kinds[1] is capi.InvalidInput, kinds


def test_small_image_and_bad_camera_rejected(gpu):
    scene, cam, target = check_fixture(1)
    for lib in (gpu, ref()):
        ctx = lib.context()
        ctx.set_scene(scene)
        small = capi.Camera(cam.view, cam.proj, 8, 8)  # camera.hpp: width and height must be >= 16
        with pytest.raises(capi.InvalidInput):
            ctx.render(small)
        lc = lib.default_loss()  # ssim window larger than the image (loss.hpp:166-168)
        lc.window = 21
        tiny = capi.Camera(cam.view, cam.proj, 16, 16)
        with pytest.raises(capi.InvalidInput):
            ctx.build_view(0, tiny, np.zeros((16, 16, 3)), loss=lc)


def test_pair_count_beyond_the_sort_limit_is_rejected(gpu):
    """more than 2^30 - 1 (tile, splat) pairs in one view (the onesweep's 30-bit
    running counts) must raise InvalidInput, not corrupt the tile lists. 40K Gaussians with
    the cutoff-free reference raster options put every splat in every tile of a 3840x2160
    view (32400 tiles): 1.3e9 pairs."""
    from paper_2501_13975_b200.workload import Config, cameras_for, make_scenes
    cfg = Config("pairs", 40_000, 1, 3840, 2160, 0, 1.0)
    truth, _ = make_scenes(cfg, seed=3)
    ctx = gpu.context()
    ctx.set_scene(truth)
    with pytest.raises(capi.InvalidInput, match="2\\^30"):
        ctx.render(cameras_for(cfg)[0], gpu.reference_raster())
    # the context stays usable for a view within the limit
    img = ctx.render(capi.Camera(cameras_for(cfg)[0].view, cameras_for(cfg)[0].proj, 64, 36))
    assert np.all(np.isfinite(img))


def test_adam_moments_follow_the_scene(gpu):
    """Adam moments are sized for one scene; set_scene with more Gaussians after an
    Adam step must restart them (AdamState(n)), not index past the old allocation."""
    d = synth(seed=31, kernels=20, views=4, probe_views=0, width=48, height=48, perturbation=0.5,
              secondary_downsample=2)
    ctx = gpu.context()
    ctx.set_scene(d["init"])
    cfg = gpu.default_train()
    cfg.optimizer = capi.OPT_ADAM
    ctx.trainer_configure(cfg, d["cameras"], d["targets"], d["train"])
    ctx.trainer_step(d["train"][0])
    big = synth(seed=32, kernels=200, views=4, probe_views=0, width=48, height=48, perturbation=0.5,
                secondary_downsample=2)
    ctx.set_scene(big["init"])
    ctx.trainer_configure(cfg, big["cameras"], big["targets"], big["train"])
    r1 = ctx.trainer_step(big["train"][0])
    # a fresh context on the same scene takes the identical first Adam step
    fresh = gpu.context()
    fresh.set_deterministic(False)
    fresh.set_scene(big["init"])
    fresh.trainer_configure(cfg, big["cameras"], big["targets"], big["train"])
    r2 = fresh.trainer_step(big["train"][0])
    for a, b in zip(r1.delta_norms, r2.delta_norms):
        assert abs(a - b) <= 1e-6 * max(abs(b), 1e-12)


def test_first_order_reported_norms_match_the_update(gpu):
    """The first-order kernel reduces five per-attribute norms with back-to-back block
    reductions; the reported |delta| of position and colour must equal the parameter change
    actually committed (a shared-memory reuse race there once corrupted the first step's
    report). Held to the FP32 parameter storage rounding (2e-3 relative)."""
    d = synth(seed=32, kernels=200, views=4, probe_views=0, width=48, height=48, perturbation=0.5,
              secondary_downsample=2)
    for opt in (capi.OPT_ADAM, capi.OPT_GD):
        ctx = gpu.context()
        ctx.set_scene(d["init"])
        cfg = gpu.default_train()
        cfg.optimizer = opt
        ctx.trainer_configure(cfg, d["cameras"], d["targets"], d["train"])
        for v in d["train"][:3]:
            before = ctx.get_scene()
            rep = ctx.trainer_step(v)
            after = ctx.get_scene()
            for a, f in ((capi.POSITION, "position"), (capi.COLOR, "sh")):
                moved = float(np.linalg.norm(getattr(after, f) - getattr(before, f)))
                got = rep.delta_norms[a]
                assert abs(got - moved) <= 2e-3 * max(moved, 1e-9), (opt, v, f, got, moved)
        ctx.close()
