"""Test helper: the reference oracle (oracle/_ref/libngs_ref.so) and its fixture generators.

TEST INFRASTRUCTURE ONLY. ``libngs_ref.so`` is the unmodified reference
(/root/reference/proj/include/ngs) compiled against oracle/eigen_shim; it
implements the same C-ABI as the CUDA product plus oracle-only generators
(oracle/ref_fixtures.inc) that run the reference's own fixture code.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2501_13975_b200.capi import (Camera, NgsLibrary, Scene, _dptr, _iptr, ngs_camera, ngs_scene)

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_LIB = os.path.join(REPO, "oracle", "_ref", "libngs_ref.so")



class ngsref_synth_params(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("kernels", C.c_int32), ("views", C.c_int32), ("probe_views", C.c_int32),
                ("width", C.c_int32), ("height", C.c_int32), ("layout", C.c_int32), ("camera_radius", C.c_double),
                ("fov_deg", C.c_double), ("perturbation", C.c_double), ("sh_degree", C.c_int32),
                ("secondary_downsample", C.c_int32), ("kernel_scale_min", C.c_double),
                ("kernel_scale_max", C.c_double), ("position_radius", C.c_double), ("sigma_min", C.c_double),
                ("sigma_max", C.c_double)]


_ref = None


def ref() -> NgsLibrary:
    global _ref
    if _ref is None:
        _ref = NgsLibrary(REF_LIB)
        assert _ref.backend == "reference-cpu"
    return _ref


def _scene_struct(n: int, sh_degree: int = 3):
    s = Scene.empty(n, sh_degree)
    cs = ngs_scene()
    cs.count = n
    cs.position, cs.scale, cs.quaternion = _dptr(s.position), _dptr(s.scale), _dptr(s.quaternion)
    cs.sigma, cs.sh = _dptr(s.sigma), _dptr(s.sh)
    return s, cs


def _finish(s: Scene, cs: ngs_scene) -> Scene:
    s.background = np.array(cs.background[:])
    s.sh_degree = cs.sh_degree
    return s


def camera_from_c(c: ngs_camera) -> Camera:
    return Camera(np.array(c.view[:]).reshape(4, 4), np.array(c.proj[:]).reshape(4, 4), c.width, c.height)


def random_scene(seed: int, kernels: int, sh_degree: int = 3) -> Scene:
    """testutil::random_scene(Rng(seed), kernels, sh_degree) (tests/test_util.hpp:38-44)."""
    L = ref()
    s, cs = _scene_struct(kernels, sh_degree)
    L.check(L.lib.ngsref_random_scene(C.c_uint64(seed), C.c_int32(kernels), C.c_int32(sh_degree), C.byref(cs)))
    return _finish(s, cs)


def test_camera(eye, width=64, height=64, fov_deg=60.0, target=(0.0, 0.0, 0.0)) -> Camera:
    """testutil::make_test_camera (tests/test_util.hpp:9-15)."""
    L = ref()
    c = ngs_camera()
    e = np.asarray(eye, np.float64)
    t = np.asarray(target, np.float64)
    L.check(L.lib.ngsref_test_camera(_dptr(e), C.c_int32(width), C.c_int32(height), C.c_double(fov_deg), _dptr(t),
                                     C.byref(c)))
    return camera_from_c(c)


test_camera.__test__ = False  # not a pytest test


def check_fixture(seed: int):
    """make_check_fixture(seed) (check.hpp:99-131): scene, 48x48 camera, target."""
    L = ref()
    cnt = C.c_int32()
    L.check(L.lib.ngsref_check_fixture(C.c_uint64(seed), None, None, None, C.byref(cnt)))
    s, cs = _scene_struct(cnt.value)
    cam = ngs_camera()
    target = np.zeros((48, 48, 3))
    L.check(L.lib.ngsref_check_fixture(C.c_uint64(seed), C.byref(cs), C.byref(cam), _dptr(target), C.byref(cnt)))
    return _finish(s, cs), camera_from_c(cam), target


def synth(**kw):
    """synth_scene(SynthParams) (synth.hpp:71-154) -> dict(init, truth, cameras, targets, secondary, train, probe)."""
    L = ref()
    p = ngsref_synth_params()
    L.lib.ngsref_synth_params_default(C.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    total = p.views + p.probe_views
    init, ci = _scene_struct(p.kernels, p.sh_degree)
    truth, ct = _scene_struct(p.kernels, p.sh_degree)
    cams = (ngs_camera * total)()
    targets = np.zeros(total * p.height * p.width * 3)
    f = max(1, p.secondary_downsample)
    while f > 1 and (p.width // f < 16 or p.height // f < 16):
        f -= 1
    dw, dh = p.width // f, p.height // f
    sec = np.zeros(total * dw * dh * 3) if p.secondary_downsample > 1 else None
    train = np.zeros(p.views, np.int32)
    probe = np.zeros(max(p.probe_views, 1), np.int32)
    L.check(L.lib.ngsref_synth(C.byref(p), C.byref(ci), C.byref(ct), cams, _dptr(targets), _dptr(sec), _iptr(train),
                               _iptr(probe)))
    cameras = [camera_from_c(cams[i]) for i in range(total)]
    tg = targets.reshape(total, p.height, p.width, 3)
    sc = sec.reshape(total, dh, dw, 3) if sec is not None else None
    return dict(init=_finish(init, ci), truth=_finish(truth, ct), cameras=cameras, targets=list(tg),
                secondary=list(sc) if sc is not None else None, secondary_downsample=p.secondary_downsample,
                train=train.tolist(), probe=probe[: p.probe_views].tolist())


def render_reference(ctx, camera: Camera) -> np.ndarray:
    """render_reference on a reference context's scene (rasterizer.hpp:452-458)."""
    out = np.zeros((camera.height, camera.width, 3))
    ctx.L.check(ctx.L.lib.ngsref_render_reference(ctx.ptr, C.byref(camera.to_c()), _dptr(out)))
    return out


def rel_error(a, b, floor=1e-9):
    """fd::rel_error (fd.hpp:31-34), elementwise."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    scale = np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)
    return np.abs(a - b) / scale


def accept_raster_scene(trial: int):
    """Scene + 64x64 camera of acceptance criterion 2's trial `trial` (acceptance.cpp:67-99)."""
    L = ref()
    cnt = C.c_int32()
    L.check(L.lib.ngsref_accept_raster_scene(C.c_int32(trial), None, None, C.byref(cnt)))
    s, cs = _scene_struct(cnt.value)
    cam = ngs_camera()
    L.check(L.lib.ngsref_accept_raster_scene(C.c_int32(trial), C.byref(cs), C.byref(cam), C.byref(cnt)))
    return _finish(s, cs), camera_from_c(cam)
