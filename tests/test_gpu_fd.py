"""GPU derivative audit (the role of check_derivatives,
check.hpp:136-505): the assembled gradient terms of the CUDA library against
central finite differences of the CUDA library's own loss value, on the
reference's derivative-check fixture (make_check_fixture, check.hpp:99-131)."""
import numpy as np
import pytest

from paper_2501_13975_b200 import capi
from refimpl import check_fixture

pytestmark = pytest.mark.gpu
ATTR = dict(position=0, rotation=1, opacity=3, color=4)


@pytest.fixture(scope="module")
def gpu():
    return capi.product()


def _loss(ctx, scene, cam, target):
    ctx.set_scene(scene)
    return ctx.build_view(0, cam, target)


def _rotate(q, axis, th):
    """axis_rotation_quaternion(th, axis) * q (scene.hpp:66-80)."""
    a = np.array([np.cos(th), *(np.sin(th) * axis)])
    w0, x0, y0, z0 = a
    w1, x1, y1, z1 = q
    r = np.array([w0 * w1 - x0 * x1 - y0 * y1 - z0 * z1, w0 * x1 + x0 * w1 + y0 * z1 - z0 * y1,
                  w0 * y1 - x0 * z1 + y0 * w1 + z0 * x1, w0 * z1 + x0 * y1 - y0 * x1 + z0 * w1])
    return r / np.linalg.norm(r)


@pytest.mark.parametrize("seed", [3, 4])
@pytest.mark.parametrize("attr", ["position", "rotation", "opacity", "color"])
def test_terms_match_finite_differences(gpu, seed, attr):
    scene, cam, target = check_fixture(seed)
    for f in ("position", "scale", "quaternion", "sigma", "sh"):
        setattr(scene, f, getattr(scene, f).astype(np.float32).astype(np.float64))
    ctx = gpu.context()
    _loss(ctx, scene, cam, target)
    g, _, vis = ctx.accumulate(ATTR[attr], 0)
    mag = np.abs(g).max(axis=1)
    ks = [int(k) for k in np.argsort(-mag)[:4] if vis[k]]
    center = -np.linalg.inv(np.asarray(cam.view)[:3, :3]) @ np.asarray(cam.view)[:3, 3]
    errs = []
    for k in ks:
        comps = range(3) if attr == "position" else [0]
        for c in comps:
            h = {"position": 1e-3, "rotation": 2e-3, "opacity": 2e-3, "color": 2e-3}[attr]
            vals = []
            for sgn in (1, -1):
                s = scene.copy()
                if attr == "position":
                    s.position = s.position.copy()
                    s.position[k, c] += sgn * h
                elif attr == "rotation":
                    s.quaternion = s.quaternion.copy()
                    r = s.position[k] - center
                    s.quaternion[k] = _rotate(s.quaternion[k], r / np.linalg.norm(r), sgn * h)
                elif attr == "opacity":
                    s.sigma = s.sigma.copy()
                    s.sigma[k] += sgn * h
                else:
                    s.sh = s.sh.copy()
                    s.sh[k, 1, 0] += sgn * h  # green DC coefficient
                vals.append(_loss(ctx, s, cam, target))
            fd = (vals[0] - vals[1]) / (2 * h)
            an = g[k, c] if attr != "color" else g[k, 16 + 0]  # grad[3*16*k + 16*ch + i], ch = 1, i = 0
            errs.append(abs(fd - an) / max(abs(an), 1e-2 * mag.max()))
    print(f"FD {attr} seed {seed}: max rel err {max(errs):.2e} over {len(errs)} probes")
    assert max(errs) < 2e-2
