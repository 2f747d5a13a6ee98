"""ctypes binding of include/ngs_b200.h.

One binding drives every implementation of the C-ABI:
  * the product, ``paper_2501_13975_b200/lib/libngs_b200.so`` (CUDA sm_100a), and
  * the test oracle ``oracle/_ref/libngs_ref.so`` (the unmodified reference
    headers, /root/reference/proj/include/ngs, compiled against an Eigen shim),
so parity tests read like the reference's own: same call, same arguments,
same error behaviour (status codes map onto the reference exception types,
/root/reference/proj/include/ngs/core.hpp:30-48).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
PRODUCT_LIB = os.path.join(_HERE, "lib", "libngs_b200.so")

# ---- status codes / exceptions (core.hpp:30-48) ---------------------------
NGS_OK = 0


class NgsError(RuntimeError):
    code = 7


class InvalidInput(NgsError):
    code = 1


class DegenerateGeometry(NgsError):
    code = 2


class NumericalError(NgsError):
    code = 3


class IoError(NgsError):
    code = 4


class CudaError(NgsError):
    code = 5


_ERRORS = {1: InvalidInput, 2: DegenerateGeometry, 3: NumericalError, 4: IoError, 5: CudaError}

POSITION, ROTATION, SCALING, OPACITY, COLOR = range(5)
ATTRIBUTES = ("position", "rotation", "scaling", "opacity", "color")


# ---- structs ---------------------------------------------------------------
class ngs_scene(C.Structure):
    _fields_ = [("count", C.c_int32), ("sh_degree", C.c_int32), ("background", C.c_double * 3),
                ("position", C.POINTER(C.c_double)), ("scale", C.POINTER(C.c_double)),
                ("quaternion", C.POINTER(C.c_double)), ("sigma", C.POINTER(C.c_double)),
                ("sh", C.POINTER(C.c_double))]


class ngs_camera(C.Structure):
    _fields_ = [("view", C.c_double * 16), ("proj", C.c_double * 16), ("width", C.c_int32), ("height", C.c_int32)]


class ngs_raster_options(C.Structure):
    _fields_ = [("lambda_lp", C.c_double), ("alpha_cutoff", C.c_double), ("t_min", C.c_double),
                ("tiled", C.c_int32), ("threads", C.c_int32)]


class ngs_loss_config(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("c1", C.c_double), ("c2", C.c_double), ("window", C.c_int32),
                ("window_sigma", C.c_double)]


class ngs_newton_options(C.Structure):
    _fields_ = [("mu_min", C.c_double), ("eig_floor_rel", C.c_double), ("step_cap_factor", C.c_double),
                ("scale_cap_factor", C.c_double), ("color_cap", C.c_double), ("theta_cap", C.c_double),
                ("barrier_weight", C.c_double), ("max_backtrack", C.c_int32), ("eigengap_rel", C.c_double)]


OPT_NEWTON, OPT_GD, OPT_ADAM = 0, 1, 2  # ngs_optimizer


class ngs_learning_rates(C.Structure):
    _fields_ = [("position", C.c_double), ("rotation", C.c_double), ("scaling", C.c_double),
                ("opacity", C.c_double), ("color", C.c_double)]


class ngs_train_config(C.Structure):
    _fields_ = [("order", C.c_int32 * 5), ("epochs", C.c_int32), ("seed", C.c_uint64), ("knn", C.c_int32),
                ("secondary_downsample", C.c_int32), ("threads", C.c_int32), ("barrier_decay", C.c_double),
                ("barrier_floor", C.c_double), ("newton", ngs_newton_options), ("raster", ngs_raster_options),
                ("loss", ngs_loss_config), ("host_targets", C.c_int32), ("probe_cadence", C.c_int32),
                ("optimizer", C.c_int32), ("gd_lr", ngs_learning_rates), ("adam_lr", ngs_learning_rates)]


class ngs_metrics(C.Structure):
    _fields_ = [("loss", C.c_double), ("psnr", C.c_double), ("ssim", C.c_double)]


class ngs_iteration_report(C.Structure):
    _fields_ = [("step", C.c_int32), ("image_id", C.c_int32), ("probe_loss", C.c_double),
                ("probe_psnr", C.c_double), ("probe_ssim", C.c_double), ("delta_norms", C.c_double * 5),
                ("dt_ms", C.c_double)]


class ngs_view_info(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("tiles_x", C.c_int32), ("tiles_y", C.c_int32),
                ("entries", C.c_int32), ("pairs", C.c_int32)]


class ngs_splat_list(C.Structure):
    _fields_ = [("kernel", C.POINTER(C.c_int32)), ("pixel", C.POINTER(C.c_double)),
                ("depth", C.POINTER(C.c_double)), ("cov2d", C.POINTER(C.c_double)),
                ("view_color", C.POINTER(C.c_double)), ("clamped", C.POINTER(C.c_uint8)),
                ("bbox", C.POINTER(C.c_double)), ("tile_offsets", C.POINTER(C.c_int32)),
                ("tile_indices", C.POINTER(C.c_int32))]


STAGES = ("project", "sort", "raster", "loss", "consts", "bwd_position", "bwd_rotation", "bwd_scaling",
          "bwd_opacity_color", "solve", "other")


class ngs_profile_stats(C.Structure):
    _fields_ = [("ms", C.c_double * 11), ("launches", C.c_int64 * 11), ("total_launches", C.c_int64),
                ("contrib_pairs", C.c_int64 * 4), ("raster_pairs", C.c_int64), ("renders", C.c_int64),
                ("group_ms", C.c_double * 6), ("allreduce_calls", C.c_int64), ("allreduce_bytes", C.c_int64),
                ("primary_bwd_ms", C.c_double * 4), ("primary_contrib_pairs", C.c_int64 * 4),
                ("color_channels", C.c_int64), ("color_fast_channels", C.c_int64)]


class ngs_terms(C.Structure):
    _fields_ = [("grad", C.POINTER(C.c_double)), ("hess", C.POINTER(C.c_double)),
                ("visible", C.POINTER(C.c_uint8))]


class ngs_solve_result(C.Structure):
    _fields_ = [("delta", C.POINTER(C.c_double)), ("accepted", C.POINTER(C.c_uint8)),
                ("degenerate", C.POINTER(C.c_uint8)), ("delta_norm_sq", C.c_double)]


# Every symbol the header declares (checked by the CPU test suite).
EXPORTED_SYMBOLS = (
    "ngs_abi_version", "ngs_backend", "ngs_last_error", "ngs_raster_options_default",
    "ngs_raster_options_reference", "ngs_loss_config_default", "ngs_newton_options_default",
    "ngs_train_config_default", "ngs_context_create", "ngs_context_destroy", "ngs_set_scene",
    "ngs_get_scene_info", "ngs_get_scene", "ngs_render", "ngs_build_view", "ngs_get_view_info",
    "ngs_view_splats", "ngs_view_image", "ngs_view_loss_derivs", "ngs_accumulate", "ngs_newton_step",
    "ngs_trainer_configure", "ngs_trainer_neighbors", "ngs_trainer_step", "ngs_trainer_barrier_weight",
    "ngs_trainer_probe", "ngs_trainer_run", "ngs_view_metrics", "ngs_set_deterministic",
)


def _dptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _iptr(a):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _bptr(a):
    if a is None:
        return None
    assert a.dtype == np.uint8 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


# ---- host data model (scene.hpp:16-28, camera.hpp:17-45) --------------------
@dataclass
class Scene:
    """Scene as per-field float64 arrays (GaussianKernel fields over kernels)."""
    position: np.ndarray            # (n, 3)
    scale: np.ndarray               # (n, 3)
    quaternion: np.ndarray          # (n, 4) (w, x, y, z)
    sigma: np.ndarray               # (n,)
    sh: np.ndarray                  # (n, 3, 16) channel-major
    background: np.ndarray = field(default_factory=lambda: np.zeros(3))
    sh_degree: int = 3

    @property
    def count(self) -> int:
        return int(self.position.shape[0])

    def copy(self) -> "Scene":
        return Scene(self.position.copy(), self.scale.copy(), self.quaternion.copy(), self.sigma.copy(),
                     self.sh.copy(), self.background.copy(), self.sh_degree)

    @staticmethod
    def empty(n: int, sh_degree: int = 3) -> "Scene":
        return Scene(np.zeros((n, 3)), np.ones((n, 3)), np.tile([1.0, 0, 0, 0], (n, 1)), np.full(n, 0.5),
                     np.zeros((n, 3, 16)), np.zeros(3), sh_degree)

    def contiguous(self) -> "Scene":
        f = lambda a: np.ascontiguousarray(a, dtype=np.float64)
        return Scene(f(self.position), f(self.scale), f(self.quaternion), f(self.sigma), f(self.sh),
                     f(self.background), int(self.sh_degree))


@dataclass
class Camera:
    view: np.ndarray   # (4, 4) world -> camera
    proj: np.ndarray   # (4, 4) camera -> clip
    width: int
    height: int

    def to_c(self) -> ngs_camera:
        c = ngs_camera()
        c.view[:] = [float(v) for v in np.asarray(self.view, dtype=np.float64).reshape(-1)]
        c.proj[:] = [float(v) for v in np.asarray(self.proj, dtype=np.float64).reshape(-1)]
        c.width, c.height = int(self.width), int(self.height)
        return c

    @property
    def center(self) -> np.ndarray:
        r = np.asarray(self.view)[:3, :3]
        return -np.linalg.inv(r) @ np.asarray(self.view)[:3, 3]

    def downsampled(self, factor: int) -> "Camera":
        """make_downsampled_camera (secondary.hpp:85-94)."""
        f = max(1, factor)
        while f > 1 and (self.width // f < 16 or self.height // f < 16):
            f -= 1
        return Camera(self.view, self.proj, self.width // f, self.height // f)


# ---- library ----------------------------------------------------------------
class NgsLibrary:
    """Loads one implementation of the ngs_b200.h C-ABI."""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"ngs C-ABI library not found: {path} (run __graft_entry__.build())")
        self.path = path
        self.lib = C.CDLL(path)
        L = self.lib
        L.ngs_backend.restype = C.c_char_p
        L.ngs_last_error.restype = C.c_char_p
        L.ngs_abi_version.restype = C.c_int32
        for name in EXPORTED_SYMBOLS:
            getattr(L, name)  # raises AttributeError if missing
        self.backend = L.ngs_backend().decode()

    def check(self, status: int):
        if status != NGS_OK:
            msg = self.lib.ngs_last_error().decode()
            raise _ERRORS.get(status, NgsError)(msg)

    def default_raster(self) -> ngs_raster_options:
        o = ngs_raster_options()
        self.lib.ngs_raster_options_default(C.byref(o))
        return o

    def reference_raster(self) -> ngs_raster_options:
        o = ngs_raster_options()
        self.lib.ngs_raster_options_reference(C.byref(o))
        return o

    def default_loss(self) -> ngs_loss_config:
        o = ngs_loss_config()
        self.lib.ngs_loss_config_default(C.byref(o))
        return o

    def default_newton(self) -> ngs_newton_options:
        o = ngs_newton_options()
        self.lib.ngs_newton_options_default(C.byref(o))
        return o

    def default_train(self) -> ngs_train_config:
        o = ngs_train_config()
        self.lib.ngs_train_config_default(C.byref(o))
        return o

    def context(self, device: int = 0) -> "Context":
        return Context(self, device)


class Context:
    """Owns an ngs_context: scene, view slots, trainer."""

    def __init__(self, lib: NgsLibrary, device: int = 0):
        self.L = lib
        self.ptr = C.c_void_p()
        lib.check(lib.lib.ngs_context_create(C.c_int32(device), C.byref(self.ptr)))
        self._keep = []

    def close(self):
        if self.ptr:
            self.L.lib.ngs_context_destroy(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _call(self, name, *args):
        self.L.check(getattr(self.L.lib, name)(self.ptr, *args))

    # scene
    def set_scene(self, scene: Scene):
        s = scene.contiguous()
        cs = ngs_scene()
        cs.count = s.count
        cs.sh_degree = s.sh_degree
        cs.background[:] = [float(v) for v in s.background]
        cs.position, cs.scale, cs.quaternion = _dptr(s.position), _dptr(s.scale), _dptr(s.quaternion)
        cs.sigma, cs.sh = _dptr(s.sigma), _dptr(s.sh)
        self._call("ngs_set_scene", C.byref(cs))

    def get_scene(self) -> Scene:
        n, deg = C.c_int32(), C.c_int32()
        self._call("ngs_get_scene_info", C.byref(n), C.byref(deg))
        s = Scene.empty(n.value, deg.value)
        cs = ngs_scene()
        cs.count = n.value
        cs.position, cs.scale, cs.quaternion = _dptr(s.position), _dptr(s.scale), _dptr(s.quaternion)
        cs.sigma, cs.sh = _dptr(s.sigma), _dptr(s.sh)
        self._call("ngs_get_scene", C.byref(cs))
        s.background = np.array(cs.background[:])
        s.sh_degree = cs.sh_degree
        return s

    # render / views
    def render(self, camera: Camera, options: ngs_raster_options | None = None) -> np.ndarray:
        out = np.zeros((camera.height, camera.width, 3))
        o = options if options is not None else self.L.default_raster()
        self._call("ngs_render", C.byref(camera.to_c()), C.byref(o), _dptr(out))
        return out

    def build_view(self, slot: int, camera: Camera, target: np.ndarray, raster=None, loss=None) -> float:
        t = np.ascontiguousarray(target, dtype=np.float64)
        assert t.shape == (camera.height, camera.width, 3)
        r = raster if raster is not None else self.L.default_raster()
        l = loss if loss is not None else self.L.default_loss()
        v = C.c_double()
        self._call("ngs_build_view", C.c_int32(slot), C.byref(camera.to_c()), _dptr(t), C.byref(r), C.byref(l),
                   C.byref(v))
        return v.value

    def view_info(self, slot: int) -> ngs_view_info:
        info = ngs_view_info()
        self._call("ngs_get_view_info", C.c_int32(slot), C.byref(info))
        return info

    def view_splats(self, slot: int) -> dict:
        info = self.view_info(slot)
        e, tiles, p = info.entries, info.tiles_x * info.tiles_y, info.pairs
        out = dict(kernel=np.zeros(e, np.int32), pixel=np.zeros((e, 2)), depth=np.zeros(e), cov2d=np.zeros((e, 2, 2)),
                   view_color=np.zeros((e, 3)), clamped=np.zeros((e, 3), np.uint8), bbox=np.zeros((e, 4)),
                   tile_offsets=np.zeros(tiles + 1, np.int32), tile_indices=np.zeros(max(p, 1), np.int32))
        sl = ngs_splat_list(_iptr(out["kernel"]), _dptr(out["pixel"]), _dptr(out["depth"]), _dptr(out["cov2d"]),
                            _dptr(out["view_color"]), _bptr(out["clamped"]), _dptr(out["bbox"]),
                            _iptr(out["tile_offsets"]), _iptr(out["tile_indices"]))
        self._call("ngs_view_splats", C.c_int32(slot), C.byref(sl))
        out["tile_indices"] = out["tile_indices"][:p]
        out["info"] = info
        return out

    def view_image(self, slot: int) -> np.ndarray:
        info = self.view_info(slot)
        out = np.zeros((info.height, info.width, 3))
        self._call("ngs_view_image", C.c_int32(slot), _dptr(out))
        return out

    def view_loss_derivs(self, slot: int):
        info = self.view_info(slot)
        g = np.zeros((info.height, info.width, 3))
        h = np.zeros((info.height, info.width, 3))
        self._call("ngs_view_loss_derivs", C.c_int32(slot), _dptr(g), _dptr(h))
        return g, h

    # accumulate / solve
    _GRAD = {POSITION: 3, ROTATION: 1, SCALING: 2, OPACITY: 1, COLOR: 48}
    _HESS = {POSITION: 9, ROTATION: 1, SCALING: 4, OPACITY: 1, COLOR: 768}
    _DELTA = {POSITION: 3, ROTATION: 1, SCALING: 3, OPACITY: 1, COLOR: 48}

    def accumulate(self, attr: int, primary: int, secondaries=(), options=None):
        n = self.scene_count()
        g = np.zeros(n * self._GRAD[attr])
        h = np.zeros(n * self._HESS[attr])
        vis = np.zeros(n, np.uint8)
        t = ngs_terms(_dptr(g), _dptr(h), _bptr(vis))
        secs = np.asarray(list(secondaries), np.int32)
        o = options if options is not None else self.L.default_newton()
        self._call("ngs_accumulate", C.c_int(attr), C.c_int32(primary), _iptr(secs) if len(secs) else None,
                   C.c_int32(len(secs)), C.byref(o), C.byref(t))
        return g.reshape(n, -1), h.reshape(n, -1), vis.astype(bool)

    def newton_step(self, attr: int, primary: int, secondaries=(), options=None, commit: bool = True):
        n = self.scene_count()
        d = np.zeros(n * self._DELTA[attr])
        acc = np.zeros(n, np.uint8)
        deg = np.zeros(n, np.uint8)
        r = ngs_solve_result(_dptr(d), _bptr(acc), _bptr(deg), 0.0)
        secs = np.asarray(list(secondaries), np.int32)
        o = options if options is not None else self.L.default_newton()
        self._call("ngs_newton_step", C.c_int(attr), C.c_int32(primary), _iptr(secs) if len(secs) else None,
                   C.c_int32(len(secs)), C.byref(o), C.c_int32(1 if commit else 0), C.byref(r))
        return dict(delta=d.reshape(n, -1), accepted=acc.astype(bool), degenerate=deg.astype(bool),
                    delta_norm_sq=r.delta_norm_sq)

    def scene_count(self) -> int:
        n, deg = C.c_int32(), C.c_int32()
        self._call("ngs_get_scene_info", C.byref(n), C.byref(deg))
        return n.value

    # trainer
    def trainer_configure(self, config: ngs_train_config, cameras, targets, train_ids, probe_ids=(),
                          secondary_targets=None, secondary_downsample: int = 0):
        cams = (ngs_camera * len(cameras))(*[c.to_c() for c in cameras])
        tg = [np.ascontiguousarray(t, dtype=np.float64) for t in targets]
        self._keep = [tg]
        tptrs = (C.POINTER(C.c_double) * len(tg))(*[_dptr(t) for t in tg])
        sptrs = None
        if secondary_targets is not None:
            st = [np.ascontiguousarray(t, dtype=np.float64) for t in secondary_targets]
            self._keep.append(st)
            sptrs = (C.POINTER(C.c_double) * len(st))(*[_dptr(t) for t in st])
        tr = np.asarray(list(train_ids), np.int32)
        pr = np.asarray(list(probe_ids), np.int32)
        self._call("ngs_trainer_configure", C.byref(config), C.c_int32(len(cameras)), cams, tptrs,
                   C.c_int32(len(tr)), _iptr(tr), C.c_int32(len(pr)), _iptr(pr) if len(pr) else None, sptrs,
                   C.c_int32(secondary_downsample))

    def trainer_neighbors(self, view_id: int):
        buf = np.zeros(64, np.int32)
        n = C.c_int32()
        self._call("ngs_trainer_neighbors", C.c_int32(view_id), _iptr(buf), C.c_int32(64), C.byref(n))
        return buf[: n.value].tolist()

    def trainer_step(self, view_id: int) -> ngs_iteration_report:
        rep = ngs_iteration_report()
        self._call("ngs_trainer_step", C.c_int32(view_id), C.byref(rep))
        return rep

    def set_deterministic(self, on: bool = True):
        """Exact integer fixed-point accumulation: bitwise-reproducible runs."""
        self._call("ngs_set_deterministic", C.c_int32(1 if on else 0))

    def trainer_probe(self) -> ngs_metrics:
        """Trainer::probe_metrics (trainer.hpp:215-233)."""
        m = ngs_metrics()
        self._call("ngs_trainer_probe", C.byref(m))
        return m

    def trainer_run(self, epochs: int, n_train: int) -> list:
        """Trainer::run (trainer.hpp:238-277) without CSV/checkpoints; returns the rows."""
        cap = 1 + max(epochs, 0) * n_train
        rows = (ngs_iteration_report * cap)()
        n = C.c_int32()
        self._call("ngs_trainer_run", rows, C.c_int32(cap), C.byref(n))
        return [rows[i] for i in range(n.value)]

    def view_metrics(self, camera: Camera, target: np.ndarray, raster=None, loss=None) -> ngs_metrics:
        """total_loss_value / psnr / ssim_metric of render(scene, camera) vs target (metrics.hpp)."""
        t = np.ascontiguousarray(target, dtype=np.float64)
        assert t.shape == (camera.height, camera.width, 3)
        r = raster if raster is not None else self.L.default_raster()
        l = loss if loss is not None else self.L.default_loss()
        m = ngs_metrics()
        self._call("ngs_view_metrics", C.byref(camera.to_c()), _dptr(t), C.byref(r), C.byref(l), C.byref(m))
        return m

    # measurement hooks (include/ngs_b200_profile.h; CUDA library only)
    def profile_enable(self, on: bool = True):
        self._call("ngs_profile_enable", C.c_int32(1 if on else 0))

    def profile_reset(self):
        self._call("ngs_profile_reset")

    def profile_read(self) -> dict:
        st = ngs_profile_stats()
        self._call("ngs_profile_read", C.byref(st))
        return dict(ms={k: st.ms[i] for i, k in enumerate(STAGES)},
                    launches={k: st.launches[i] for i, k in enumerate(STAGES)},
                    total_launches=st.total_launches, contrib_pairs=list(st.contrib_pairs),
                    raster_pairs=st.raster_pairs, renders=st.renders,
                    allreduce_calls=st.allreduce_calls, allreduce_bytes=st.allreduce_bytes,
                    primary_bwd_ms=list(st.primary_bwd_ms), primary_contrib_pairs=list(st.primary_contrib_pairs),
                    color_channels=st.color_channels, color_fast_channels=st.color_fast_channels,
                    # Trainer renders are chained per view into the following backward pass, so each
                    # pass group includes the render before it ("render" stays 0 in trainer steps).
                    group_ms=dict(zip(("render", "render+bwd_position", "render+bwd_rotation", "render+bwd_scaling",
                                       "render+bwd_opacity_color", "solve"), list(st.group_ms))))

    def profile_timeline(self, on: bool = True):
        """Per-launch events on the concurrent schedule (views not serialised)."""
        self._call("ngs_profile_timeline", C.c_int32(1 if on else 0))

    def read_timeline(self) -> list:
        """[(stage name, stream id, start_ms, end_ms)] since profile_timeline(True)."""
        class Row(C.Structure):
            _fields_ = [("stage", C.c_int32), ("stream", C.c_int32), ("start_ms", C.c_float), ("end_ms", C.c_float)]
        n = C.c_int32()
        self._call("ngs_profile_read_timeline", None, C.c_int32(0), C.byref(n))
        rows = (Row * max(n.value, 1))()
        self._call("ngs_profile_read_timeline", rows, C.c_int32(n.value), C.byref(n))
        return [(STAGES[r.stage], r.stream, r.start_ms, r.end_ms) for r in rows[: n.value]]

    def set_tile_size(self, tile: int):
        self._call("ngs_set_tile_size", C.c_int32(tile))

    def microbench_fp32(self) -> float:
        v = C.c_double()
        self._call("ngs_microbench_fp32", C.byref(v))
        return v.value

    def microbench_fp64(self) -> float:
        v = C.c_double()
        self._call("ngs_microbench_fp64", C.byref(v))
        return v.value

    def microbench_solve(self, n: int, sh_degree: int = 3, views: int = 4, reps: int = 5) -> list:
        """Mean ms of solve_<attr> over n synthetic Gaussians (ngs_microbench_solve);
        self.last_color_fast_frac = the colour channel solves that took the fast path."""
        out = (C.c_double * 5)()
        frac = C.c_double()
        self._call("ngs_microbench_solve", C.c_int32(n), C.c_int32(sh_degree), C.c_int32(views), C.c_int32(reps),
                   out, C.byref(frac))
        self.last_color_fast_frac = frac.value
        return list(out)

    # multi-GPU sharding (include/ngs_b200_dist.h; CUDA library only)
    def set_shard(self, rank: int, world: int):
        self._call("ngs_set_shard", C.c_int32(rank), C.c_int32(world))

    def dist_init(self, unique_id: bytes, rank: int, world: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        self._call("ngs_dist_init", buf, C.c_int32(rank), C.c_int32(world))

    def barrier_weight(self) -> float:
        v = C.c_double()
        self._call("ngs_trainer_barrier_weight", C.byref(v))
        return v.value


def dist_unique_id(lib: NgsLibrary) -> bytes:
    """ncclGetUniqueId through the library (rank 0); broadcast the bytes to all ranks."""
    buf = (C.c_uint8 * 128)()
    lib.check(lib.lib.ngs_dist_unique_id(buf))
    return bytes(buf)


class ngs_shard_rows(C.Structure):
    _fields_ = [("band_y0", C.c_int32), ("band_y1", C.c_int32), ("own_y0", C.c_int32), ("own_y1", C.c_int32)]


def dist_plan(lib: NgsLibrary, world: int, rank: int, sizes, tiles, loss_window: int = 11):
    """ngs_dist_plan (ngs_b200_dist.h): this rank's (band_y0, band_y1, own_y0, own_y1) tile
    rows of each view of a step, view 0 the primary. Pure host call (no device)."""
    n = len(sizes)
    w = np.asarray([s[0] for s in sizes], np.int32)
    h = np.asarray([s[1] for s in sizes], np.int32)
    t = np.asarray(list(tiles), np.int32)
    out = (ngs_shard_rows * n)()
    lib.check(lib.lib.ngs_dist_plan(C.c_int32(world), C.c_int32(rank), C.c_int32(n), _iptr(w), _iptr(h), _iptr(t),
                                    C.c_int32(loss_window), out))
    return [(r.band_y0, r.band_y1, r.own_y0, r.own_y1) for r in out]


_product = None


def product() -> NgsLibrary:
    """The CUDA implementation. Fails loudly if the extension is not built."""
    global _product
    if _product is None:
        _product = NgsLibrary(PRODUCT_LIB)
        if _product.backend != "cuda-sm_100a":
            raise RuntimeError(f"unexpected backend {_product.backend}")
    return _product
