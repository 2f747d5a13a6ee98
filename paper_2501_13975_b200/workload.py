"""Synthetic workloads for the BASELINE.json configs (host-side data generation).

Follows SynthParams semantics (/root/reference/proj/include/ngs/synth.hpp:19-154):
kernels uniform in the unit ball (radius * cbrt(U)), normalised N(0,1)
quaternions, sigma ~ U[0.35, 0.7], SH DC ~ U[-0.9, 0.9], higher ~ U[-0.12, 0.12],
background (0.05, 0.05, 0.08), Fibonacci-sphere cameras at radius 2 looking at
the origin (fov 60 deg, near 0.05, far 100), and the jittered training init
(synth.hpp:138-152). Bench-scale scenes are drawn with numpy's PCG64 rather
than the reference Rng — they need the right statistics, not bit-identity;
parity fixtures come from the reference's own generator (tests/refimpl.py).

Deviation (stated): kernel scales and the position jitter are
multiplied by (100/N)^(1/3) so footprints stay ~1-3 px and per-pixel splat
depth stays NeRF-synthetic-like as N grows.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .capi import Camera, Scene


def make_lookat_view(eye, target, up_hint) -> np.ndarray:
    """camera.hpp:288-304."""
    eye, target, up = (np.asarray(v, np.float64) for v in (eye, target, up_hint))
    fwd = target - eye
    fwd /= np.linalg.norm(fwd)
    if abs(fwd @ (up / np.linalg.norm(up))) > 0.999:
        up = np.array([0.0, 0.0, 1.0]) if abs(fwd[2]) < 0.9 else np.array([1.0, 0.0, 0.0])
    right = np.cross(up, fwd)
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    view = np.eye(4)
    view[0, :3], view[1, :3], view[2, :3] = right, down, fwd
    view[0, 3], view[1, 3], view[2, 3] = -right @ eye, -down @ eye, -fwd @ eye
    return view


def make_perspective_proj(fov_y_rad, aspect, z_near, z_far) -> np.ndarray:
    """camera.hpp:307-317."""
    fy = 1.0 / math.tan(0.5 * fov_y_rad)
    proj = np.zeros((4, 4))
    proj[0, 0] = fy / aspect
    proj[1, 1] = fy
    proj[2, 2] = (z_far + z_near) / (z_far - z_near)
    proj[2, 3] = -2.0 * z_far * z_near / (z_far - z_near)
    proj[3, 2] = 1.0
    return proj


def fibonacci_dir(i: int, n: int) -> np.ndarray:
    """synth.hpp:51-58."""
    golden = math.pi * (3.0 - math.sqrt(5.0))
    y = 1.0 - 2.0 * (i + 0.5) / n
    r = math.sqrt(max(0.0, 1.0 - y * y))
    phi = golden * i
    return np.array([r * math.cos(phi), y, r * math.sin(phi)])


@dataclass
class Config:
    name: str
    kernels: int
    views: int
    width: int
    height: int
    sh_degree: int
    scale_factor: float = 1.0   # multiplies the kernel-scale range and the position jitter

    @property
    def desc(self) -> str:
        return f"{self.kernels} Gaussians, {self.views} views {self.width}x{self.height}, SH deg {self.sh_degree}"


def footprint_factor(kernels: int) -> float:
    return (100.0 / kernels) ** (1.0 / 3.0)


# BASELINE.json configs (C1 is the reference's own CPU-runnable case).
CONFIGS = {
    "c1": Config("c1", 10_000, 16, 256, 256, 0, 1.0),
    "c2": Config("c2", 300_000, 100, 800, 800, 3, footprint_factor(300_000)),
    "c3": Config("c3", 3_000_000, 200, 1920, 1080, 3, footprint_factor(3_000_000)),
}


def cameras_for(cfg: Config, total: int | None = None, fov_deg: float = 60.0, radius: float = 2.0):
    n = total if total is not None else cfg.views
    proj = make_perspective_proj(math.radians(fov_deg), cfg.width / cfg.height, 0.05, 100.0)
    return [Camera(make_lookat_view(fibonacci_dir(i, n) * radius, np.zeros(3), np.array([0.0, 1.0, 0.0])), proj,
                   cfg.width, cfg.height) for i in range(n)]


def make_scenes(cfg: Config, seed: int = 1000, perturbation: float = 1.0):
    """(truth, init) scenes following synth_scene (synth.hpp:71-101, 138-152)."""
    rng = np.random.default_rng(seed)
    n, f = cfg.kernels, cfg.scale_factor
    d = rng.standard_normal((n, 3))
    d /= np.maximum(np.linalg.norm(d, axis=1, keepdims=True), 1e-12)
    pos = d * np.cbrt(rng.random(n))[:, None]
    scale = rng.uniform(0.05 * f, 0.12 * f, (n, 3))
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    sigma = rng.uniform(0.35, 0.7, n)
    sh = np.zeros((n, 3, 16))
    ncoef = (cfg.sh_degree + 1) ** 2
    sh[:, :, 0] = rng.uniform(-0.9, 0.9, (n, 3))
    if ncoef > 1:
        sh[:, :, 1:ncoef] = rng.uniform(-0.12, 0.12, (n, 3, ncoef - 1))
    truth = Scene(pos, scale, q, sigma, sh, np.array([0.05, 0.05, 0.08]), cfg.sh_degree)
    init = truth.copy()
    p = perturbation
    init.position = pos + p * 0.05 * f * rng.standard_normal((n, 3))
    init.scale = scale * np.exp2(rng.uniform(-1.0, 1.0, (n, 3))) ** p
    init.sigma = np.clip(sigma + p * 0.15 * rng.standard_normal(n), 0.05, 0.95)
    init.sh = sh.copy()
    init.sh[:, :, 0] += p * 0.25 * rng.standard_normal((n, 3))
    init.sh[:, :, 1:] += p * 0.03 * rng.standard_normal((n, 3, 15))
    return truth, init


def float32_exact(scene: Scene) -> Scene:
    s = scene.copy()
    for f in ("position", "scale", "quaternion", "sigma", "sh"):
        setattr(s, f, getattr(s, f).astype(np.float32).astype(np.float64))
    return s
