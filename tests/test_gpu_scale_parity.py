"""GPU parity at BASELINE scale: C1 (10K Gaussians, 16 views 256x256, SH0, K=3,
downsample 4) and a C2-shaped slice (30K Gaussians, 256x256, SH3, c2's footprint
law), the CUDA library (libngs_b200.so) against the compiled reference
(oracle/_ref/libngs_ref.so) through the same C-ABI.

A third fixture, c3slice, is C3-shaped (16:9 at 320x180 with ragged edge tiles, SH3,
c3's footprint law). Fixture: the reference's own ``synth_scene`` (synth.hpp:71-154) generates the
scenes and cameras. Its images are rendered at 16x16 only to keep the
generator's single-threaded ``render_reference`` cheap: the RNG stream, the
kernels, the jittered init and the view/proj matrices do not depend on the
image size (aspect 1 either way), so the cameras are then re-sized to 256x256
and the targets are rendered by the reference's threaded default render from
the truth scene. Both libraries receive bit-identical inputs (init rounded to
FP32, the device's storage type).

Checks (VERDICT r1 "next round" item 1; SURVEY.md §8a parity contract):
  * binning bit-exact at 10K / 30K Gaussians (entry order, tile offsets, per-tile
    lists), with FP32-vs-FP64 depth near-ties and bbox near-tile-edge counts reported;
  * per-pass solved deltas of all five attributes from identical inputs (each pass
    starts both libraries from the reference's FP32-rounded post-commit scene), as
    an error distribution per quantity;
  * one full Trainer::step: delta norms and the post-step update.
Bound: the GPU's per-Gaussian error distribution must not be wider than the
reference's own response to a one-ulp FP32 perturbation of its input (a second
reference run), i.e. the GPU is as close to the reference as FP32 storage of
the parameters allows (within_sensitivity).
Measured errors are printed and, with NGS_PARITY_REPORT=<path>, written as JSON
(DESIGN.md §3 quotes them).
"""
import json
import os

import numpy as np
import pytest

from paper_2501_13975_b200 import capi
from refimpl import ref, synth

pytestmark = pytest.mark.gpu

FLOOR = 1e-3
ATTRS = [capi.POSITION, capi.ROTATION, capi.SCALING, capi.OPACITY, capi.COLOR]
REPORT = {}


def _report(key, value):
    REPORT[key] = value
    path = os.environ.get("NGS_PARITY_REPORT")
    if path:
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "w") as f:
            json.dump(REPORT, f, indent=1, sort_keys=True)


def rel_dist(gpu, refv, floor_frac=FLOOR):
    """rel_error (fd.hpp:31-34) with an absolute floor of floor_frac*max|ref|:
    (max, p99, p50) over all entries."""
    g = np.asarray(gpu, np.float64).ravel()
    r = np.asarray(refv, np.float64).ravel()
    if r.size == 0:
        return dict(max=0.0, p99=0.0, p50=0.0)
    floor = max(floor_frac * float(np.max(np.abs(r))), 1e-300)
    e = np.abs(g - r) / np.maximum(np.maximum(np.abs(g), np.abs(r)), floor)
    return dict(max=float(e.max()), p99=float(np.quantile(e, 0.99)), p50=float(np.quantile(e, 0.5)))


def f32(scene):
    s = scene.copy()
    for f in ("position", "scale", "quaternion", "sigma", "sh"):
        setattr(s, f, getattr(s, f).astype(np.float32).astype(np.float64))
    # committed opacities may sit at the reference's clamp nextafter(1e-4, 1) (newton.hpp:772-774),
    # whose FP32 rounding falls outside validate_kernel's open interval
    lo = float(np.nextafter(np.float32(1e-4), np.float32(1)))
    hi = float(np.nextafter(np.float32(1 - 1e-4), np.float32(0)))
    s.sigma = np.clip(s.sigma, lo, hi)
    return s


def box_downsample(img, f):
    """downsample_box (image.hpp:39-62) for sizes divisible by f."""
    h, w, _ = img.shape
    return img[: h // f * f, : w // f * f].reshape(h // f, f, w // f, f, 3).mean(axis=(1, 3))


def make_fixture(kernels, sh_degree, scale_mul, seed, width=256, height=256):
    # synth_scene's images are rendered small (16x16, or 1/10 of a 16:9 size): the aspect fixes the projection
    # matrix (synth.hpp:108-110); the RNG stream and the scene do not depend on the size.
    aspect = width / height
    sw, sh = (16, 16) if width == height else (width // 10, height // 10)  # 320x180 -> 32x18: same aspect
    p = dict(seed=seed, kernels=kernels, views=16, probe_views=4, width=sw, height=sh,
             sh_degree=sh_degree, secondary_downsample=1)
    if scale_mul != 1.0:
        p.update(kernel_scale_min=0.05 * scale_mul, kernel_scale_max=0.12 * scale_mul)
    d = synth(**p)
    assert abs(d["cameras"][0].width / d["cameras"][0].height - aspect) < 1e-12
    cams = [capi.Camera(c.view, c.proj, width, height) for c in d["cameras"]]
    r = ref().context()
    r.set_scene(d["truth"])
    ro = ref().default_raster()
    ro.threads = os.cpu_count() or 1
    targets = [r.render(c, ro) for c in cams]
    r.close()
    return dict(init=f32(d["init"]), cameras=cams, targets=targets, train=d["train"], probe=d["probe"])


# C2's footprint law at 256x256: c2 scales kernels by (100/300K)^(1/3) at 800x800; the same
# pixel footprint at 256x256 is that factor x 800/256, and 30K/256^2 keeps c2's splats per pixel.
C2_SLICE_SCALE = (100.0 / 300_000) ** (1.0 / 3.0) * 800.0 / 256.0


# C3's 16:9 aspect with ragged edge tiles (320x180: 20 x 11.25 tiles; secondaries 80x45
# with 8x8 tiles), SH3, the c3 footprint law at this width (3M at 1920 -> 20K at 320 keeps
# the splats per pixel).
C3_SLICE_SCALE = (100.0 / 3_000_000) ** (1.0 / 3.0) * 1920.0 / 320.0


@pytest.fixture(scope="module", params=["c1", "c2slice", "c3slice"])
def fixture(request):
    if request.param == "c1":
        return request.param, make_fixture(10_000, 0, 1.0, 1000)
    if request.param == "c2slice":
        return request.param, make_fixture(30_000, 3, C2_SLICE_SCALE, 1001)
    return request.param, make_fixture(20_000, 3, C3_SLICE_SCALE, 1002, 320, 180)


@pytest.fixture(scope="module")
def gpu():
    return capi.product()


def _near_ties(splats_ref, width, height, tile=16):
    """Counts of FP32-vs-FP64 depth near-ties (adjacent entries within 4 FP32 ulp)
    and bbox edges within 1e-4 px of a tile boundary (SURVEY.md §8a parity contract)."""
    d = np.sort(splats_ref["depth"])
    ulp = np.spacing(np.abs(d[:-1]).astype(np.float32)).astype(np.float64)
    ties = int(np.sum(np.abs(np.diff(d)) <= 4 * ulp))
    bb = splats_ref["bbox"]
    edge = np.abs(bb / tile - np.round(bb / tile)) * tile
    return ties, int(np.sum(edge < 1e-4))


def test_binning_bit_exact_at_scale(gpu, fixture):
    name, d = fixture
    for view in (d["train"][0], d["train"][7]):
        cam = d["cameras"][view]
        g, r = gpu.context(), ref().context()
        for c in (g, r):
            c.set_scene(d["init"])
            c.build_view(0, cam, d["targets"][view])
        sg, sr = g.view_splats(0), r.view_splats(0)
        ties, edges = _near_ties(sr, cam.width, cam.height)
        info = sg["info"]
        print(f"{name} view {view}: entries {info.entries}, pairs {info.pairs}, depth near-ties {ties}, "
              f"bbox near-edges {edges}")
        _report(f"{name}.binning.view{view}", dict(entries=int(info.entries), pairs=int(info.pairs),
                                                  depth_near_ties=ties, bbox_near_tile_edges=edges))
        assert np.array_equal(sg["kernel"], sr["kernel"])
        assert np.array_equal(sg["tile_offsets"], sr["tile_offsets"])
        assert np.array_equal(sg["tile_indices"], sr["tile_indices"])
        img_err = float(np.max(np.abs(g.view_image(0) - r.view_image(0))))
        _report(f"{name}.image_abs.view{view}", img_err)
        assert img_err < 1e-4
        g.close()
        r.close()


def perturb_ulp(scene, seed):
    """Half of the parameters moved by one FP32 ulp (random direction): the reference run on
    this input measures how far the reference itself moves when its FP32-representable input
    moves by the storage precision — the intrinsic sensitivity the GPU is held to."""
    rng = np.random.default_rng(seed)
    s = scene.copy()
    for f in ("position", "scale", "sigma", "sh"):
        a = getattr(s, f).astype(np.float32)
        m = rng.random(a.shape) < 0.5
        up = rng.random(a.shape) < 0.5
        b = np.where(m, np.where(up, np.nextafter(a, np.float32(np.inf)), np.nextafter(a, np.float32(-np.inf))), a)
        setattr(s, f, b.astype(np.float64))
    return f32(s)


def per_kernel_err(gpu, refv, floor_frac=FLOOR):
    """Per-Gaussian max of rel_error (fd.hpp:31-34) over its components, with an absolute floor
    of floor_frac * max|ref| of the whole quantity."""
    g = np.asarray(gpu, np.float64).reshape(len(gpu), -1)
    r = np.asarray(refv, np.float64).reshape(len(refv), -1)
    if r.size == 0:
        return np.zeros(len(r))
    floor = max(floor_frac * float(np.max(np.abs(r))), 1e-300)
    return (np.abs(g - r) / np.maximum(np.maximum(np.abs(g), np.abs(r)), floor)).max(axis=1)


def summary(e):
    return dict(p50=float(np.quantile(e, 0.5)), p99=float(np.quantile(e, 0.99)), p999=float(np.quantile(e, 0.999)),
                max=float(e.max()), n_gt_1e4=int(np.sum(e > 1e-4)), n_gt_1e3=int(np.sum(e > 1e-3)),
                n_gt_1e2=int(np.sum(e > 1e-2)))


def within_sensitivity(eg, ep, what, max_cap=5e-2):
    """The GPU's per-Gaussian error distribution against the reference must not be wider than
    the reference's own response to a one-ulp FP32 perturbation of its input (x2 + 1e-5 slack
    on the p99 quantile, x3 + 1e-5 on p99.9, x3 + 5 on the count of Gaussians above 1e-3). For one
    solve, no single Gaussian may be off by more than `max_cap` (discrete-branch outliers:
    eigengap, caps, clamps). A full step re-renders between passes, so single Gaussians
    inherit their neighbours' branch flips: the reference itself moves individual SH
    coefficients by O(1) on a one-ulp input change there, and only the distribution is held
    (max_cap=None, the maximum is reported)."""
    sg, sp = summary(eg), summary(ep)
    assert sg["p99"] <= 2 * sp["p99"] + 1e-5, (what, sg, sp)
    assert sg["p999"] <= 3 * sp["p999"] + 1e-5, (what, sg, sp)   # p99.9 of 1e4 Gaussians: the 10th largest
    assert sg["n_gt_1e3"] <= 3 * sp["n_gt_1e3"] + 5, (what, sg, sp)
    if max_cap is not None:
        assert sg["max"] < max_cap, (what, sg, sp)


def step_views(d):
    tr = ref().context()
    tr.set_scene(d["init"])
    tr.trainer_configure(ref().default_train(), d["cameras"], d["targets"], d["train"], d["probe"])
    view = d["train"][0]
    nbrs = tr.trainer_neighbors(view)
    tr.close()
    views = [(d["cameras"][view], d["targets"][view])]
    for nb in nbrs:
        views.append((d["cameras"][nb].downsampled(4), box_downsample(d["targets"][nb], 4)))
    return views


def test_per_pass_deltas_at_scale(gpu, fixture):
    """Each of the five passes of newton_step (trainer.hpp:331-405) solved from identical
    inputs on both libraries: primary at 256x256, K=3 neighbours at 64x64 with
    box-downsampled targets (trainer.hpp:151-168). Each pass starts from the reference's
    FP32-rounded post-commit scene of the previous pass."""
    name, d = fixture
    views = step_views(d)
    ro = ref().default_raster()
    ro.threads = os.cpu_count() or 1
    scene = d["init"]
    failures = []
    for attr in ATTRS:
        a = capi.ATTRIBUTES[attr]
        out = {}
        for tag, lib, sc in (("gpu", gpu, scene), ("ref", ref(), scene), ("refp", ref(), perturb_ulp(scene, attr))):
            c = lib.context()
            c.set_scene(sc)
            for slot, (cam, tgt) in enumerate(views):
                c.build_view(slot, cam, tgt, raster=ro if lib is ref() else None)
            out[tag] = c.newton_step(attr, 0, list(range(1, len(views))))
            if tag == "ref":
                nxt = f32(c.get_scene())
            c.close()
        eg = per_kernel_err(out["gpu"]["delta"], out["ref"]["delta"])
        ep = per_kernel_err(out["refp"]["delta"], out["ref"]["delta"])
        flips = int(np.sum(out["gpu"]["accepted"] != out["ref"]["accepted"]))
        flips_p = int(np.sum(out["refp"]["accepted"] != out["ref"]["accepted"]))
        deg = int(np.sum(out["gpu"]["degenerate"] != out["ref"]["degenerate"]))
        deg_p = int(np.sum(out["refp"]["degenerate"] != out["ref"]["degenerate"]))
        nsq = (out["gpu"]["delta_norm_sq"], out["ref"]["delta_norm_sq"])
        print(f"{name} {a}: gpu {summary(eg)}\n    ref(1-ulp input) {summary(ep)}\n    accepted flips "
              f"{flips} (ref-ulp {flips_p}), degenerate flips {deg} (ref-ulp {deg_p}); |delta|^2 {nsq[0]:.9g} vs "
              f"{nsq[1]:.9g}")
        _report(f"{name}.delta.{a}", dict(gpu=summary(eg), ref_ulp=summary(ep), accepted_flips=flips,
                                          accepted_flips_ref_ulp=flips_p, degenerate_flips=deg,
                                          degenerate_flips_ref_ulp=deg_p, norm_sq_gpu=nsq[0], norm_sq_ref=nsq[1]))
        try:
            within_sensitivity(eg, ep, a)
            assert flips <= 2 * flips_p + 1e-3 * len(eg) and deg <= 2 * deg_p + 1e-3 * len(eg)
            assert abs(nsq[0] - nsq[1]) <= 1e-4 * abs(nsq[1]) + 1e-30
        except AssertionError as e:  # report every pass before failing
            failures.append(str(e))
        scene = nxt
    assert not failures, failures


def test_trainer_step_at_scale(gpu, fixture):
    """One full Trainer::step (trainer.hpp:185-207, 299-417) on both libraries; the post-step
    update (post - init, so |p| ~ 1 does not hide it) is held to the same sensitivity bound,
    measured with a second reference step from the one-ulp-perturbed init."""
    name, d = fixture
    runs = {}
    for tag, lib, init in (("gpu", gpu, d["init"]), ("ref", ref(), d["init"]), ("refp", ref(), perturb_ulp(d["init"], 9))):
        c = lib.context()
        c.set_scene(init)
        cfg = lib.default_train()
        cfg.threads = os.cpu_count() or 1
        c.trainer_configure(cfg, d["cameras"], d["targets"], d["train"], d["probe"])
        rep = c.trainer_step(d["train"][0])
        runs[tag] = (rep, c.get_scene(), init)
        if tag == "gpu":
            nb = c.trainer_neighbors(d["train"][0])
        else:
            assert c.trainer_neighbors(d["train"][0]) == nb
        c.close()
    norms = [(runs["gpu"][0].delta_norms[i], runs["ref"][0].delta_norms[i]) for i in range(5)]
    res = {"delta_norms": norms, "gpu_ms": runs["gpu"][0].dt_ms, "ref_ms": runs["ref"][0].dt_ms}
    failures = []
    for f in ("position", "scale", "quaternion", "sigma", "sh"):
        upd = {t: getattr(runs[t][1], f) - getattr(runs[t][2], f) for t in runs}
        eg = per_kernel_err(upd["gpu"], upd["ref"])
        ep = per_kernel_err(upd["refp"], upd["ref"])
        res[f] = dict(gpu=summary(eg), ref_ulp=summary(ep),
                      param_max=float(np.max(np.abs(getattr(runs["gpu"][1], f) - getattr(runs["ref"][1], f)))))
        print(f"{name} step {f} update: gpu {summary(eg)}\n    ref(1-ulp input) {summary(ep)}")
        try:
            within_sensitivity(eg, ep, f, max_cap=None)
        except AssertionError as e:
            failures.append(str(e))
    print(f"{name} step delta norms gpu/ref: {norms}; gpu {res['gpu_ms']:.2f} ms, ref {res['ref_ms']:.0f} ms")
    _report(f"{name}.trainer_step", res)
    for a, b in norms:
        assert abs(a - b) <= 1e-4 * max(abs(b), 1e-9)
    assert not failures, failures
