"""ngs_oracle.py — float64 CPU restatement of the reference 3DGS² Newton path.

TEST INFRASTRUCTURE ONLY (checker, never the product): imported by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg. It restates, in numpy,
the algorithm of /root/reference/proj/include/ngs (citations are
<file>:<line> under proj/include/ngs/), and exposes the same surface as the
C-ABI binding (paper_2501_13975_b200.capi.Context) so parity tests drive it
like the other implementations.

Pinned against golden vectors produced by the reference itself
(oracle/_ref/libngs_ref.so = the unmodified reference compiled against the
test-only Eigen shim), committed under tests/golden/ with their generating
script tests/golden/make_golden.py. Pure-Python loops: small fixtures only.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

K_TILE = 16                    # rasterizer.hpp:18
K_NEAR = 1e-6                  # camera.hpp:11
K_LOWPASS = 0.3                # camera.hpp:12
K_SIGMA_MARGIN = 1e-4          # scene.hpp:10
K_RIDGE_MIN = 1e-8             # newton.hpp:19
K_COLOR_OFFSET = 0.5           # sh.hpp:21
SH0 = 0.28209479177387814      # sh.hpp:13-23
SH1 = 0.4886025119029199
SH2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792, 0.5462742152960396)
SH3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154, -0.4570457994644658,
       1.445305721320277, -0.5900435899266435)


class InvalidInput(ValueError):
    pass


class DegenerateGeometry(ValueError):
    pass


class NumericalError(ArithmeticError):
    pass


# ---------------------------------------------------------------------------
# scene.hpp
# ---------------------------------------------------------------------------

def quaternion_to_rotation(q):
    """scene.hpp:40-53."""
    q = np.asarray(q, np.float64)
    n = np.linalg.norm(q)
    if not (n > 0) or not np.isfinite(n):
        raise InvalidInput("quaternion_to_rotation: zero quaternion")
    if abs(n - 1.0) > 1e-12:
        q = q / n
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def covariance_3d(q, s):
    """build_covariance_3d, scene.hpp:56-63."""
    if not (np.min(s) > 0):
        raise InvalidInput("build_covariance_3d: scale components must be positive")
    rs = quaternion_to_rotation(q) * np.asarray(s)[None, :]
    return rs @ rs.T


def quaternion_multiply(a, b):
    """scene.hpp:66-72 (Hamilton product)."""
    return np.array([a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3],
                     a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2],
                     a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1],
                     a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0]])


# ---------------------------------------------------------------------------
# camera.hpp
# ---------------------------------------------------------------------------

@dataclass
class Cam:
    """Camera, camera.hpp:17-45."""
    view: np.ndarray
    proj: np.ndarray
    width: int
    height: int
    view_proj: np.ndarray = field(init=False)
    rot: np.ndarray = field(init=False)
    trans: np.ndarray = field(init=False)
    center: np.ndarray = field(init=False)

    def __post_init__(self):
        if self.width < 16 or self.height < 16:
            raise InvalidInput("camera: width and height must be >= 16")
        self.view = np.asarray(self.view, np.float64)
        self.proj = np.asarray(self.proj, np.float64)
        self.view_proj = self.proj @ self.view
        self.rot = self.view[:3, :3]
        self.trans = self.view[:3, 3]
        if abs(np.linalg.det(self.rot)) < 1e-12:
            raise InvalidInput("camera: view rotation block is singular")
        self.center = -np.linalg.inv(self.rot) @ self.trans

    @staticmethod
    def of(c) -> "Cam":
        return Cam(np.asarray(c.view).reshape(4, 4), np.asarray(c.proj).reshape(4, 4), int(c.width), int(c.height))


def view_direction_derivs(cam: Cam, p):
    """view_direction / view_direction_derivatives, camera.hpp:63-104."""
    u = p - cam.center
    n = np.linalg.norm(u)
    if not n > 1e-12:
        raise DegenerateGeometry("view_direction: point coincides with camera center")
    r = u / n
    jac = (np.eye(3) - np.outer(r, r)) / n
    hess = np.zeros((3, 3, 3))
    for i in range(3):
        for j in range(3):
            for k in range(3):
                v = 3 * r[i] * r[j] * r[k]
                if i == j:
                    v -= r[k]
                if i == k:
                    v -= r[j]
                if j == k:
                    v -= r[i]
                hess[i, j, k] = v / (n * n)
    return r, jac, hess


def project_center(cam: Cam, p):
    """camera.hpp:106-115."""
    h = cam.view_proj @ np.append(p, 1.0)
    if not h[3] > K_NEAR:
        return None
    px = np.array([0.5 * cam.width * (h[0] / h[3] + 1), 0.5 * cam.height * (h[1] / h[3] + 1)])
    depth = cam.rot[2] @ p + cam.trans[2]
    return px, depth


def projection_derivatives(cam: Cam, p):
    """camera.hpp:124-148: J = dpi/dp (2x3) and H[i] = d2pi_i/dp2."""
    h = cam.view_proj @ np.append(p, 1.0)
    if not h[3] > K_NEAR:
        return None
    a, b, w = cam.view_proj[0, :3], cam.view_proj[1, :3], cam.view_proj[3, :3]
    hw = h[3]
    sx, sy = 0.5 * cam.width, 0.5 * cam.height
    J = np.stack([sx * (a / hw - h[0] / hw ** 2 * w), sy * (b / hw - h[1] / hw ** 2 * w)])
    ww = np.outer(w, w)
    H0 = sx * (-(np.outer(a, w) + np.outer(w, a)) / hw ** 2 + 2 * h[0] * ww / hw ** 3)
    H1 = sy * (-(np.outer(b, w) + np.outer(w, b)) / hw ** 2 + 2 * h[1] * ww / hw ** 3)
    return J, np.stack([H0, H1])


def project_camera_space(cam: Cam, t, second=False):
    """detail::project_camera_space, camera.hpp:163-208 (J, dJ/dt_e, d2J/dt_e dt_f)."""
    h = cam.proj @ np.append(t, 1.0)
    if not h[3] > K_NEAR:
        return None
    a, b, w = cam.proj[0, :3], cam.proj[1, :3], cam.proj[3, :3]
    hw = h[3]
    sx, sy = 0.5 * cam.width, 0.5 * cam.height
    J = np.stack([sx * (a / hw - h[0] / hw ** 2 * w), sy * (b / hw - h[1] / hw ** 2 * w)])
    dJ = np.zeros((3, 2, 3))
    for e in range(3):
        dJ[e, 0] = sx * (-(w[e] * a + a[e] * w) / hw ** 2 + 2 * h[0] * w[e] / hw ** 3 * w)
        dJ[e, 1] = sy * (-(w[e] * b + b[e] * w) / hw ** 2 + 2 * h[1] * w[e] / hw ** 3 * w)
    d2J = np.zeros((3, 3, 2, 3))
    if second:
        for e in range(3):
            for f in range(3):
                d2J[e, f, 0] = sx * (2 * ((w[e] * a + a[e] * w) * w[f] + a[f] * w[e] * w) / hw ** 3 -
                                     6 * h[0] * w[e] * w[f] / hw ** 4 * w)
                d2J[e, f, 1] = sy * (2 * ((w[e] * b + b[e] * w) * w[f] + b[f] * w[e] * w) / hw ** 3 -
                                     6 * h[1] * w[e] * w[f] / hw ** 4 * w)
    return J, dJ, d2J


def project_covariance_2d(cam: Cam, k, lambda_lp=K_LOWPASS):
    """camera.hpp:219-232: Sigma = J W A W^T J^T + lp I (symmetrised) and J."""
    t = cam.rot @ k["p"] + cam.trans
    pr = project_camera_space(cam, t)
    if pr is None:
        return None
    J = pr[0]
    m = cam.rot @ covariance_3d(k["q"], k["s"]) @ cam.rot.T
    S = J @ m @ J.T + lambda_lp * np.eye(2)
    return 0.5 * (S + S.T), J


def cov2d_derivatives(cam: Cam, k):
    """cov2d_derivatives_wrt_position, camera.hpp:241-284: dS/dp_c, d2S/dp_c dp_d."""
    t = cam.rot @ k["p"] + cam.trans
    pr = project_camera_space(cam, t, second=True)
    if pr is None:
        return None
    J, dJ, d2J = pr
    m = cam.rot @ covariance_3d(k["q"], k["s"]) @ cam.rot.T
    W = cam.rot
    djp = np.einsum("eij,ec->cij", dJ, W)
    d2jp = np.einsum("efij,ec,fd->cdij", d2J, W, W)
    mjt = m @ J.T
    dS = np.zeros((3, 2, 2))
    d2S = np.zeros((3, 3, 2, 2))
    for c in range(3):
        term = djp[c] @ mjt
        dS[c] = term + term.T
    for c in range(3):
        for d in range(3):
            t1 = d2jp[c, d] @ mjt
            t2 = djp[c] @ m @ djp[d].T
            d2S[c, d] = t1 + t1.T + t2 + t2.T
    return dS, d2S


def project_kernel(cam: Cam, k, lambda_lp=K_LOWPASS):
    """camera.hpp:319-339."""
    c = project_center(cam, k["p"])
    if c is None:
        return None
    cov = project_covariance_2d(cam, k, lambda_lp)
    if cov is None:
        return None
    S, J = cov
    det = S[0, 0] * S[1, 1] - S[0, 1] * S[1, 0]
    if not det > 0:
        raise NumericalError("project_kernel: projected covariance is not positive definite")
    r, _, _ = view_direction_derivs(cam, k["p"])
    return dict(pixel=c[0], depth=c[1], cov=S, cov_inv=np.linalg.inv(S), J=J, view_dir=r)


# ---------------------------------------------------------------------------
# sh.hpp
# ---------------------------------------------------------------------------

def sh_basis(r, degree):
    """eval_sh_basis, sh.hpp:35-105: values (16), jacobian (16x3), hessian (16x3x3)."""
    x, y, z = r
    v = np.zeros(16)
    jac = np.zeros((16, 3))
    hes = np.zeros((16, 3, 3))
    v[0] = SH0
    if degree < 1:
        return v, jac, hes
    v[1], v[2], v[3] = -SH1 * y, SH1 * z, -SH1 * x
    jac[1, 1], jac[2, 2], jac[3, 0] = -SH1, SH1, -SH1
    if degree < 2:
        return v, jac, hes
    xx, yy, zz = x * x, y * y, z * z
    v[4] = SH2[0] * x * y
    v[5] = SH2[1] * y * z
    v[6] = SH2[2] * (2 * zz - xx - yy)
    v[7] = SH2[3] * x * z
    v[8] = SH2[4] * (xx - yy)
    jac[4] = SH2[0] * np.array([y, x, 0])
    jac[5] = SH2[1] * np.array([0, z, y])
    jac[6] = SH2[2] * np.array([-2 * x, -2 * y, 4 * z])
    jac[7] = SH2[3] * np.array([z, 0, x])
    jac[8] = SH2[4] * np.array([2 * x, -2 * y, 0])
    hes[4] = SH2[0] * np.array([[0, 1, 0], [1, 0, 0], [0, 0, 0]])
    hes[5] = SH2[1] * np.array([[0, 0, 0], [0, 0, 1], [0, 1, 0]])
    hes[6] = SH2[2] * np.diag([-2.0, -2.0, 4.0])
    hes[7] = SH2[3] * np.array([[0, 0, 1], [0, 0, 0], [1, 0, 0]])
    hes[8] = SH2[4] * np.diag([2.0, -2.0, 0.0])
    if degree < 3:
        return v, jac, hes
    v[9] = SH3[0] * y * (3 * xx - yy)
    v[10] = SH3[1] * x * y * z
    v[11] = SH3[2] * y * (4 * zz - xx - yy)
    v[12] = SH3[3] * z * (2 * zz - 3 * xx - 3 * yy)
    v[13] = SH3[4] * x * (4 * zz - xx - yy)
    v[14] = SH3[5] * z * (xx - yy)
    v[15] = SH3[6] * x * (xx - 3 * yy)
    jac[9] = SH3[0] * np.array([6 * x * y, 3 * xx - 3 * yy, 0])
    jac[10] = SH3[1] * np.array([y * z, x * z, x * y])
    jac[11] = SH3[2] * np.array([-2 * x * y, 4 * zz - xx - 3 * yy, 8 * y * z])
    jac[12] = SH3[3] * np.array([-6 * x * z, -6 * y * z, 6 * zz - 3 * xx - 3 * yy])
    jac[13] = SH3[4] * np.array([4 * zz - 3 * xx - yy, -2 * x * y, 8 * x * z])
    jac[14] = SH3[5] * np.array([2 * x * z, -2 * y * z, xx - yy])
    jac[15] = SH3[6] * np.array([3 * xx - 3 * yy, -6 * x * y, 0])
    hes[9] = SH3[0] * np.array([[6 * y, 6 * x, 0], [6 * x, -6 * y, 0], [0, 0, 0]])
    hes[10] = SH3[1] * np.array([[0, z, y], [z, 0, x], [y, x, 0]])
    hes[11] = SH3[2] * np.array([[-2 * y, -2 * x, 0], [-2 * x, -6 * y, 8 * z], [0, 8 * z, 8 * y]])
    hes[12] = SH3[3] * np.array([[-6 * z, 0, -6 * x], [0, -6 * z, -6 * y], [-6 * x, -6 * y, 12 * z]])
    hes[13] = SH3[4] * np.array([[-6 * x, -2 * y, 8 * z], [-2 * y, -2 * x, 0], [8 * z, 0, 8 * x]])
    hes[14] = SH3[5] * np.array([[2 * z, 0, 2 * x], [0, -2 * z, -2 * y], [2 * x, -2 * y, 0]])
    hes[15] = SH3[6] * np.array([[6 * x, -6 * y, 0], [-6 * y, -6 * x, 0], [0, 0, 0]])
    return v, jac, hes


def view_color(basis_v, sh):
    """eval_view_color, sh.hpp:114-123: Phi.c + 0.5 clamped at 0 from below."""
    val = sh @ basis_v + K_COLOR_OFFSET
    clamped = val <= 0
    return np.where(clamped, 0.0, val), clamped


def sh_color_derivs(cam: Cam, k, degree):
    """sh_color_derivs_wrt_position, sh.hpp:134-161: dc~/dp (3x3), d2c~/dp2 (3x3x3)."""
    r, vjac, vhes = view_direction_derivs(cam, k["p"])
    v, bj, bh = sh_basis(r, degree)
    n = (degree + 1) ** 2
    jac = np.zeros((3, 3))
    hes = np.zeros((3, 3, 3))
    for ch in range(3):
        c = k["sh"][ch]
        if c @ v + K_COLOR_OFFSET <= 0:
            continue
        gr = (c[:n, None] * bj[:n]).sum(0)
        hr = (c[:n, None, None] * bh[:n]).sum(0)
        jac[ch] = vjac.T @ gr
        hes[ch] = vjac.T @ hr @ vjac + np.einsum("a,ajk->jk", gr, vhes)
    return jac, hes


# ---------------------------------------------------------------------------
# rasterizer.hpp
# ---------------------------------------------------------------------------

def gaussian_weight(S, pi, x):
    """rasterizer.hpp:116-176: G and derivatives w.r.t. pi and Sigma (symmetrised tensors)."""
    det = S[0, 0] * S[1, 1] - S[0, 1] * S[1, 0]
    if not (det > 0) or not np.isfinite(det):
        raise NumericalError("gaussian_weight: covariance is not positive definite")
    Q = np.linalg.inv(S)
    d = pi - x
    qd = Q @ d
    g = math.exp(-0.5 * d @ qd)
    raw = np.zeros((2, 2, 2, 2))
    for p in range(2):
        for l in range(2):
            for gg in range(2):
                for h in range(2):
                    raw[p, l, gg, h] = g * (0.25 * qd[p] * qd[l] * qd[gg] * qd[h] -
                                            0.5 * (Q[p, gg] * qd[h] * qd[l] + qd[p] * Q[l, gg] * qd[h]))
    sym = np.zeros_like(raw)
    for p in range(2):
        for l in range(2):
            m = 0.5 * (raw[p, l] + raw[l, p])
            sym[p, l] = 0.5 * (m + m.T)
    d2s = np.zeros_like(raw)
    for p in range(2):
        for l in range(2):
            for gg in range(2):
                for h in range(2):
                    d2s[p, l, gg, h] = 0.5 * (sym[p, l, gg, h] + sym[gg, h, p, l])
    mix = np.zeros((2, 2, 2))
    for a in range(2):
        m = np.zeros((2, 2))
        for p in range(2):
            for l in range(2):
                m[p, l] = -0.5 * g * qd[a] * qd[p] * qd[l] + 0.5 * g * (Q[p, a] * qd[l] + qd[p] * Q[l, a])
        mix[a] = 0.5 * (m + m.T)
    return dict(g=g, d_pi=-g * qd, d2_pi=g * (np.outer(qd, qd) - Q), d_sigma=0.5 * g * np.outer(qd, qd),
                d2_sigma=d2s, d2_pi_sigma=mix)


def build_splat_list(scene, cam: Cam, raster):
    """rasterizer.hpp:182-265: entries sorted by (depth, kernel), clamped tile bins."""
    entries = []
    for k in range(scene["n"]):
        kern = kernel_of(scene, k)
        pk = project_kernel(cam, kern, raster["lambda_lp"])
        if pk is None:
            continue
        v, _, _ = sh_basis(pk["view_dir"], scene["deg"])
        col, clamped = view_color(v, kern["sh"])
        if raster["alpha_cutoff"] > 0:
            radius = max(3.0, math.sqrt(2.0 * math.log(1.0 / raster["alpha_cutoff"])))
            rx = radius * math.sqrt(max(pk["cov"][0, 0], 0.0))
            ry = radius * math.sqrt(max(pk["cov"][1, 1], 0.0))
            bmin = pk["pixel"] - np.array([rx, ry])
            bmax = pk["pixel"] + np.array([rx, ry])
        else:
            bmin = np.zeros(2)
            bmax = np.array([cam.width - 1.0, cam.height - 1.0])
        entries.append(dict(kernel=k, proj=pk, color=col, clamped=clamped, sigma=kern["sigma"], bmin=bmin, bmax=bmax))
    entries.sort(key=lambda e: (e["proj"]["depth"], e["kernel"]))
    tiles_x = (cam.width + K_TILE - 1) // K_TILE
    tiles_y = (cam.height + K_TILE - 1) // K_TILE
    bins = [[] for _ in range(tiles_x * tiles_y)]
    for i, e in enumerate(entries):
        if e["bmax"][0] < 0 or e["bmin"][0] >= cam.width or e["bmax"][1] < 0 or e["bmin"][1] >= cam.height:
            continue
        tx0, ty0 = (int(np.clip(math.floor(e["bmin"][a] / K_TILE), 0, lim - 1)) for a, lim in ((0, tiles_x), (1, tiles_y)))
        tx1, ty1 = (int(np.clip(math.floor(e["bmax"][a] / K_TILE), 0, lim - 1)) for a, lim in ((0, tiles_x), (1, tiles_y)))
        for ty in range(ty0, ty1 + 1):
            for tx in range(tx0, tx1 + 1):
                bins[ty * tiles_x + tx].append(i)
    offsets = np.zeros(len(bins) + 1, np.int32)
    for t, b in enumerate(bins):
        offsets[t + 1] = offsets[t] + len(b)
    indices = np.array([i for b in bins for i in b], np.int32)
    return dict(entries=entries, tiles_x=tiles_x, tiles_y=tiles_y, offsets=offsets, indices=indices,
                width=cam.width, height=cam.height)


def bin_entries(entry_kernel, depth, bbox, width, height):
    """Reference sort + bin (rasterizer.hpp:228-263) applied to externally
    supplied per-entry depth / bbox (the bit-exact binning contract)."""
    order = sorted(range(len(entry_kernel)), key=lambda i: (depth[i], entry_kernel[i]))
    tiles_x = (width + K_TILE - 1) // K_TILE
    tiles_y = (height + K_TILE - 1) // K_TILE
    bins = [[] for _ in range(tiles_x * tiles_y)]
    for rank, i in enumerate(order):
        x0, y0, x1, y1 = bbox[i]
        if x1 < 0 or x0 >= width or y1 < 0 or y0 >= height:
            continue
        tx0 = int(np.clip(math.floor(x0 / K_TILE), 0, tiles_x - 1))
        tx1 = int(np.clip(math.floor(x1 / K_TILE), 0, tiles_x - 1))
        ty0 = int(np.clip(math.floor(y0 / K_TILE), 0, tiles_y - 1))
        ty1 = int(np.clip(math.floor(y1 / K_TILE), 0, tiles_y - 1))
        for ty in range(ty0, ty1 + 1):
            for tx in range(tx0, tx1 + 1):
                bins[ty * tiles_x + tx].append(rank)
    offsets = np.zeros(len(bins) + 1, np.int32)
    for t, b in enumerate(bins):
        offsets[t + 1] = offsets[t] + len(b)
    return [entry_kernel[i] for i in order], offsets, np.array([i for b in bins for i in b], np.int32)


def composite(sl, background, raster):
    """composite_forward + composite_pixel with capture, rasterizer.hpp:274-442."""
    W, H = sl["width"], sl["height"]
    img = np.zeros((H, W, 3))
    capture = {}
    ents = sl["entries"]
    for ty in range(sl["tiles_y"]):
        for tx in range(sl["tiles_x"]):
            t = ty * sl["tiles_x"] + tx
            order = sl["indices"][sl["offsets"][t]:sl["offsets"][t + 1]]
            for y in range(ty * K_TILE, min((ty + 1) * K_TILE, H)):
                for x in range(tx * K_TILE, min((tx + 1) * K_TILE, W)):
                    pc = np.array([x + 0.5, y + 0.5])
                    T = 1.0
                    c = np.zeros(3)
                    recs = []
                    for idx in order:
                        e = ents[idx]
                        d = e["proj"]["pixel"] - pc
                        g = math.exp(-0.5 * d @ (e["proj"]["cov_inv"] @ d))
                        a = g * e["sigma"]
                        if a < raster["alpha_cutoff"]:
                            continue
                        recs.append((idx, g, a, T))
                        c += T * a * e["color"]
                        T *= 1 - a
                        if raster["t_min"] > 0 and T < raster["t_min"]:
                            break
                    img[y, x] = c + T * background
                    capture[(x, y)] = recs
    return img, capture


def invert_capture(sl, capture, background, n):
    """rasterizer.hpp:489-524: kernel-major records with the 'behind' colour."""
    ents = sl["entries"]
    out = {k: [] for k in range(n)}
    for (x, y), recs in sorted(capture.items(), key=lambda kv: (kv[0][1], kv[0][0])):
        if not recs:
            continue
        behind = [np.array(background, np.float64)] * len(recs)
        for i in range(len(recs) - 2, -1, -1):
            nxt = recs[i + 1]
            behind[i] = nxt[2] * ents[nxt[0]]["color"] + (1 - nxt[2]) * behind[i + 1]
        for i, (idx, g, a, T) in enumerate(recs):
            out[ents[idx]["kernel"]].append(dict(px=x, py=y, g=g, alpha=a, T=T, color=ents[idx]["color"],
                                                 behind=behind[i]))
    return out


# ---------------------------------------------------------------------------
# loss.hpp
# ---------------------------------------------------------------------------

def gaussian_window(window, sigma):
    """loss.hpp:66-77."""
    half = window // 2
    w = np.exp(-((np.arange(window) - half) ** 2) / (2 * sigma * sigma))
    return w / w.sum()


def sep_conv(field2d, kx):
    """SeparableConv::run with valid taps, loss.hpp:81-115 (x then y)."""
    H, W = field2d.shape
    half = len(kx) // 2
    tmp = np.zeros_like(field2d)
    for x in range(W):
        for i in range(max(-half, -x), min(half, W - 1 - x) + 1):
            tmp[:, x] += kx[i + half] * field2d[:, x + i]
    out = np.zeros_like(field2d)
    for y in range(H):
        for j in range(max(-half, -y), min(half, H - 1 - y) + 1):
            out[y, :] += kx[j + half] * tmp[y + j, :]
    return out


def axis_norms(n, k):
    """loss.hpp:117-128."""
    half = len(k) // 2
    return np.array([k[max(-half, -x) + half:min(half, n - 1 - x) + half + 1].sum() for x in range(n)])


def total_loss_derivs(img, tgt, cfg):
    """total_loss_derivs (loss.hpp:342-356) = L2 (138-156) + lambda * SSIM (162-335)."""
    H, W, _ = img.shape
    n = H * W
    inv = 1.0 / (3.0 * n)
    d = img - tgt
    grad = inv * d
    hess = np.full_like(img, inv)
    value = 0.5 * inv * float((d * d).sum())
    if cfg["lambda"] == 0.0:
        return value, grad, hess
    if W < cfg["window"] or H < cfg["window"]:
        raise InvalidInput("ssim stats: image smaller than the filter window")
    w = gaussian_window(cfg["window"], cfg["window_sigma"])
    w2 = w * w
    inv_norm = 1.0 / np.outer(axis_norms(H, w), axis_norms(W, w))
    c1, c2 = cfg["c1"], cfg["c2"]
    ssim_sum = 0.0
    gs = np.zeros_like(img)
    hs = np.zeros_like(img)
    for ch in range(3):
        c, t = img[:, :, ch], tgt[:, :, ch]
        mu = sep_conv(c, w) * inv_norm
        mu_t = sep_conv(t, w) * inv_norm
        var = np.maximum(0.0, sep_conv(c * c, w) * inv_norm - mu * mu)
        var_t = np.maximum(0.0, sep_conv(t * t, w) * inv_norm - mu_t * mu_t)
        cov = sep_conv(c * t, w) * inv_norm - mu * mu_t
        f0 = 2 * mu * mu_t + c1
        f1 = 2 * cov + c2
        f2 = mu * mu + mu_t * mu_t + c1
        f3 = var + var_t + c2
        nn, dd = f0 * f1, f2 * f3
        ssim_sum += float((nn / dd).sum())
        inv_d = 1.0 / dd
        fp = (2 * mu_t * (f1 - f0) * inv_d - 2 * mu * nn * inv_d / f2 + 2 * mu * nn * inv_d / f3) * inv_norm
        fq = 2 * f0 * inv_d * inv_norm
        fr = -2 * nn * inv_d / f3 * inv_norm
        a0, a1, b1 = 2 * mu_t, -2 * mu_t, 2.0
        a2, a3, b3 = 2 * mu, -2 * mu, 2.0
        A, B, Cc, E = a0 * f1 + f0 * a1, f0 * b1, a2 * f3 + f2 * a3, f2 * b3
        n2 = inv_norm * inv_norm
        fkw = -2 * nn / (f2 * f3 * f3) * inv_norm
        ft0 = (2 * a0 * a1 * inv_d - 2 * A * Cc * inv_d ** 2 - nn * (2 * a2 * a3 + 2 * f3 - 2 * f2) * inv_d ** 2 +
               2 * nn * Cc * Cc * inv_d ** 3) * n2
        ftc = (-2 * A * E * inv_d ** 2 - 2 * nn * a2 * b3 * inv_d ** 2 + 4 * nn * Cc * E * inv_d ** 3) * n2
        ftct = (2 * a0 * b1 * inv_d - 2 * B * Cc * inv_d ** 2) * n2
        ftcct = -2 * B * E * inv_d ** 2 * n2
        ftc2 = 2 * nn * E * E * inv_d ** 3 * n2
        gs[:, :, ch] = -inv * (sep_conv(fp, w) + t * sep_conv(fq, w) + c * sep_conv(fr, w))
        hs[:, :, ch] = -inv * (sep_conv(fkw, w) + sep_conv(ft0, w2) + c * sep_conv(ftc, w2) + t * sep_conv(ftct, w2) +
                               c * t * sep_conv(ftcct, w2) + c * c * sep_conv(ftc2, w2))
    lam = cfg["lambda"]
    value += lam * (1.0 - ssim_sum * inv)
    return value, grad + lam * gs, hess + lam * hs


def ssim_mean_value(img, tgt, cfg):
    """ssim_mean_value (loss.hpp:378-382): mean SSIM map over channels and pixels."""
    H, W, _ = img.shape
    if W < cfg["window"] or H < cfg["window"]:
        raise InvalidInput("ssim stats: image smaller than the filter window")
    w = gaussian_window(cfg["window"], cfg["window_sigma"])
    inv_norm = 1.0 / np.outer(axis_norms(H, w), axis_norms(W, w))
    c1, c2 = cfg["c1"], cfg["c2"]
    total = 0.0
    for ch in range(3):
        c, t = img[:, :, ch], tgt[:, :, ch]
        mu = sep_conv(c, w) * inv_norm
        mu_t = sep_conv(t, w) * inv_norm
        var = np.maximum(0.0, sep_conv(c * c, w) * inv_norm - mu * mu)
        var_t = np.maximum(0.0, sep_conv(t * t, w) * inv_norm - mu_t * mu_t)
        cov = sep_conv(c * t, w) * inv_norm - mu * mu_t
        total += float(((2 * mu * mu_t + c1) * (2 * cov + c2) / ((mu * mu + mu_t * mu_t + c1) * (var + var_t + c2))).sum())
    return total / (3.0 * H * W)


def total_loss_value(img, tgt, cfg):
    """total_loss_value (loss.hpp:359-375): value-only L2 + lambda (1 - mean SSIM)."""
    d = img - tgt
    value = 0.5 * float((d * d).sum()) / (3.0 * img.shape[0] * img.shape[1])
    if cfg["lambda"] != 0.0:
        value += cfg["lambda"] * (1.0 - ssim_mean_value(img, tgt, cfg))
    return value


def psnr(img, tgt):
    """psnr (metrics.hpp:14-24): dB over all pixels and channels, +inf if identical."""
    d = img - tgt
    mse = float((d * d).sum()) / d.size
    return math.inf if mse == 0.0 else -10.0 * math.log10(mse)


class Rng:
    """ngs::Rng (core.hpp:52-81): std::mt19937_64 (restated: MT19937-64 of the
    C++ standard, [rand.eng.mers]) with the reference's uniform/index/shuffle."""

    N, M = 312, 156
    MASK = (1 << 64) - 1

    def __init__(self, seed=5489):
        self.mt = [0] * self.N
        self.mt[0] = seed & self.MASK
        for i in range(1, self.N):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & self.MASK
        self.i = self.N

    def _twist(self):
        up, lo = 0xFFFFFFFF80000000, 0x7FFFFFFF
        for k in range(self.N):
            x = (self.mt[k] & up) | (self.mt[(k + 1) % self.N] & lo)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            self.mt[k] = self.mt[(k + self.M) % self.N] ^ xa
        self.i = 0

    def next(self):
        if self.i >= self.N:
            self._twist()
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & self.MASK

    def shuffle(self, v):
        """core.hpp:76-81: for i = n..2: swap(v[i-1], v[engine() % i])."""
        for i in range(len(v), 1, -1):
            j = self.next() % i
            v[i - 1], v[j] = v[j], v[i - 1]
        return v


# ---------------------------------------------------------------------------
# newton.hpp
# ---------------------------------------------------------------------------

def sym2_eigen(m):
    """newton.hpp:41-56."""
    a, b, c = m[0, 0], 0.5 * (m[0, 1] + m[1, 0]), m[1, 1]
    ht = 0.5 * (a + c)
    disc = math.sqrt(max(0.0, 0.25 * (a - c) ** 2 + b * b))
    vals = np.array([ht - disc, ht + disc])
    vecs = np.eye(2)
    if disc < 1e-300:
        return vals, vecs
    v1 = np.array([b, vals[1] - a])
    if v1 @ v1 < 1e-300:
        v1 = np.array([vals[1] - c, b])
    if v1 @ v1 < 1e-300:
        v1 = np.array([1.0, 0.0])
    v1 = v1 / np.linalg.norm(v1)
    vecs[:, 1] = v1
    vecs[:, 0] = [-v1[1], v1[0]]
    return vals, vecs


def psd_safeguard(Hm, mu_min=K_RIDGE_MIN, rel=0.0):
    """newton.hpp:205-238 (saddle-free |lambda| floored at mu)."""
    Hm = np.atleast_2d(Hm)
    n = Hm.shape[0]
    if n == 1:
        a = Hm[0, 0]
        return np.array([[max(abs(a), max(mu_min, rel * abs(a)))]])
    if n == 2:
        vals, vecs = sym2_eigen(0.5 * (Hm + Hm.T))
    else:
        vals, vecs = np.linalg.eigh(0.5 * (Hm + Hm.T))
    mu = max(mu_min, rel * float(np.max(np.abs(vals))))
    if vals.min() >= mu:
        return Hm
    return (vecs * np.maximum(np.abs(vals), mu)) @ vecs.T


def solve_safeguarded(Hm, g, opts):
    """newton.hpp:240-244."""
    Hs = psd_safeguard(Hm, opts["mu_min"], opts["eig_floor_rel"])
    return np.linalg.solve(Hs, -np.atleast_1d(g))


def position_subspace(r):
    """newton.hpp:130-139."""
    seed = np.array([0.0, 1.0, 0.0])
    if abs(r @ seed) > 0.99:
        seed = np.array([0.0, 0.0, 1.0])
    uy = seed - r * (r @ seed)
    uy /= np.linalg.norm(uy)
    return np.stack([np.cross(r, uy), uy], axis=1)


def scaling_subspace(entry, kern, cam: Cam, eigengap_rel):
    """build_scaling_subspace, newton.hpp:152-184."""
    vals, vecs = sym2_eigen(entry["proj"]["cov"])
    degenerate = (vals[1] - vals[0]) <= eigengap_rel * abs(vals[1])
    n = entry["proj"]["J"] @ cam.rot @ quaternion_to_rotation(kern["q"])
    T = np.zeros((2, 3))
    for i in range(2):
        for c in range(3):
            T[i, c] = 2 * kern["s"][c] * (vecs[:, i] @ n[:, c]) ** 2
    gv, ge = sym2_eigen(T @ T.T)
    cutoff = max(1e-30, 1e-12 * abs(gv[1]))
    gp = sum((1.0 / gv[i]) * np.outer(ge[:, i], ge[:, i]) for i in range(2) if gv[i] > cutoff) \
        if any(gv[i] > cutoff for i in range(2)) else np.zeros((2, 2))
    return dict(vals=vals, vecs=vecs, T=T, t_pinv=T.T @ gp, degenerate=degenerate)


def kernel_of(scene, k):
    return dict(p=scene["p"][k], s=scene["s"][k], q=scene["q"][k], sigma=scene["sigma"][k], sh=scene["sh"][k])


@dataclass
class View:
    """ViewContext (newton.hpp:86-118), capture-based like the reference."""
    scene: dict
    cam: Cam
    target: np.ndarray
    sl: dict
    image: np.ndarray
    records: dict
    entry_of: dict
    loss_value: float
    grad: np.ndarray
    hess: np.ndarray


def build_view(scene, cam: Cam, target, raster, loss_cfg) -> View:
    sl = build_splat_list(scene, cam, raster)
    img, cap = composite(sl, scene["bg"], raster)
    recs = invert_capture(sl, cap, scene["bg"], scene["n"])
    value, g, h = total_loss_derivs(img, np.asarray(target, np.float64), loss_cfg)
    entry_of = {e["kernel"]: i for i, e in enumerate(sl["entries"])}
    return View(scene, cam, target, sl, img, recs, entry_of, value, g, h)


def position_terms(k, v: View):
    """newton.hpp:266-343."""
    g = np.zeros(3)
    Hm = np.zeros((3, 3))
    recs = v.records[k]
    if k not in v.entry_of or not recs:
        return g, Hm, False
    kern = kernel_of(v.scene, k)
    e = v.sl["entries"][v.entry_of[k]]
    J, Hp = projection_derivatives(v.cam, kern["p"])
    dS, d2S = cov2d_derivatives(v.cam, kern)
    cj, chs = sh_color_derivs(v.cam, kern, v.scene["deg"])
    for rec in recs:
        gl = v.grad[rec["py"], rec["px"]]
        hl = v.hess[rec["py"], rec["px"]]
        gw = gaussian_weight(e["proj"]["cov"], e["proj"]["pixel"], np.array([rec["px"] + 0.5, rec["py"] + 0.5]))
        dg = J.T @ gw["d_pi"] + np.array([(gw["d_sigma"] * dS[c]).sum() for c in range(3)])
        d2g = J.T @ gw["d2_pi"] @ J + sum(gw["d_pi"][i] * Hp[i] for i in range(2))
        y = [sum(dS[c][p, l] * gw["d2_sigma"][p, l] for p in range(2) for l in range(2)) for c in range(3)]
        mixed = np.array([[(gw["d2_pi_sigma"][a] * dS[c]).sum() for c in range(3)] for a in range(2)])
        for c in range(3):
            for d in range(3):
                val = (y[c] * dS[d]).sum() + (gw["d_sigma"] * d2S[c, d]).sum()
                val += sum(J[a, c] * mixed[a, d] + J[a, d] * mixed[a, c] for a in range(2))
                d2g[c, d] += val
        wa = e["sigma"] * rec["T"]
        for ch in range(3):
            a_ch = rec["color"][ch] - rec["behind"][ch]
            dc = wa * (a_ch * dg + rec["g"] * cj[ch])
            g += gl[ch] * dc
            d2c = a_ch * d2g + rec["g"] * chs[ch] + np.outer(dg, cj[ch]) + np.outer(cj[ch], dg)
            Hm += hl[ch] * np.outer(dc, dc) + gl[ch] * wa * d2c
    return g, Hm, True


def rotation_terms(k, axis, v: View):
    """newton.hpp:353-404."""
    recs = v.records[k]
    if k not in v.entry_of or not recs:
        return 0.0, 0.0, False
    kern = kernel_of(v.scene, k)
    e = v.sl["entries"][v.entry_of[k]]
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    A = covariance_3d(kern["q"], kern["s"])
    dA = 2 * (K @ A - A @ K)
    d2A = 4 * (K @ K @ A + A @ K @ K) - 8 * K @ A @ K
    jw = e["proj"]["J"] @ v.cam.rot
    s1, s2 = jw @ dA @ jw.T, jw @ d2A @ jw.T
    g = h = 0.0
    for rec in recs:
        gl, hl = v.grad[rec["py"], rec["px"]], v.hess[rec["py"], rec["px"]]
        gw = gaussian_weight(e["proj"]["cov"], e["proj"]["pixel"], np.array([rec["px"] + 0.5, rec["py"] + 0.5]))
        dg = (gw["d_sigma"] * s1).sum()
        d2g = sum(s1[p, l] * (gw["d2_sigma"][p, l] * s1).sum() for p in range(2) for l in range(2))
        d2g += (gw["d_sigma"] * s2).sum()
        wa = e["sigma"] * rec["T"]
        for ch in range(3):
            a_ch = rec["color"][ch] - rec["behind"][ch]
            dc = wa * a_ch * dg
            g += gl[ch] * dc
            h += hl[ch] * dc * dc + gl[ch] * wa * a_ch * d2g
    return g, h, True


def scaling_terms(k, v: View, eigengap_rel):
    """newton.hpp:415-469."""
    g = np.zeros(2)
    Hm = np.zeros((2, 2))
    recs = v.records[k]
    if k not in v.entry_of or not recs:
        return g, Hm, False
    kern = kernel_of(v.scene, k)
    e = v.sl["entries"][v.entry_of[k]]
    sub = scaling_subspace(e, kern, v.cam, eigengap_rel)
    dirs = [np.outer(sub["vecs"][:, i], sub["vecs"][:, i]) for i in range(2)]
    for rec in recs:
        gl, hl = v.grad[rec["py"], rec["px"]], v.hess[rec["py"], rec["px"]]
        gw = gaussian_weight(e["proj"]["cov"], e["proj"]["pixel"], np.array([rec["px"] + 0.5, rec["py"] + 0.5]))
        dg = np.array([(gw["d_sigma"] * dirs[i]).sum() for i in range(2)])
        d2g = np.array([[sum(dirs[i][p, l] * (gw["d2_sigma"][p, l] * dirs[j]).sum() for p in range(2)
                             for l in range(2)) for j in range(2)] for i in range(2)])
        wa = e["sigma"] * rec["T"]
        for ch in range(3):
            a_ch = rec["color"][ch] - rec["behind"][ch]
            dc = wa * a_ch * dg
            g += gl[ch] * dc
            Hm += hl[ch] * np.outer(dc, dc) + gl[ch] * wa * a_ch * d2g
    return g, Hm, True


def scaling_gradient_s(k, v: View):
    """newton.hpp:472-503: 3-dof scale-space gradient (first-order baselines)."""
    grad = np.zeros(3)
    recs = v.records[k]
    if k not in v.entry_of or not recs:
        return grad
    kern = kernel_of(v.scene, k)
    e = v.sl["entries"][v.entry_of[k]]
    n = e["proj"]["J"] @ v.cam.rot @ quaternion_to_rotation(kern["q"])
    dsig = [2.0 * kern["s"][c] * np.outer(n[:, c], n[:, c]) for c in range(3)]
    for rec in recs:
        gl = v.grad[rec["py"], rec["px"]]
        gw = gaussian_weight(e["proj"]["cov"], e["proj"]["pixel"], np.array([rec["px"] + 0.5, rec["py"] + 0.5]))
        dg = np.array([(gw["d_sigma"] * dsig[c]).sum() for c in range(3)])
        wa = e["sigma"] * rec["T"]
        for ch in range(3):
            grad += gl[ch] * wa * (rec["color"][ch] - rec["behind"][ch]) * dg
    return grad


def opacity_terms(k, v: View):
    """newton.hpp:507-526."""
    recs = v.records[k]
    if k not in v.entry_of or not recs:
        return 0.0, 0.0, False
    g = h = 0.0
    for rec in recs:
        gl, hl = v.grad[rec["py"], rec["px"]], v.hess[rec["py"], rec["px"]]
        for ch in range(3):
            dc = rec["g"] * rec["T"] * (rec["color"][ch] - rec["behind"][ch])
            g += gl[ch] * dc
            h += hl[ch] * dc * dc
    return g, h, True


def color_terms(k, v: View):
    """newton.hpp:538-574 (dense n-vector / n x n per channel, zero-padded to 16)."""
    n = (v.scene["deg"] + 1) ** 2
    g = np.zeros((3, 16))
    Hm = np.zeros((3, 16, 16))
    recs = v.records[k]
    if k not in v.entry_of or not recs:
        return g, Hm, False
    e = v.sl["entries"][v.entry_of[k]]
    phi = sh_basis(e["proj"]["view_dir"], v.scene["deg"])[0][:n]
    ga = np.zeros(3)
    ha = np.zeros(3)
    for rec in recs:
        w = rec["alpha"] * rec["T"]
        ga += v.grad[rec["py"], rec["px"]] * w
        ha += v.hess[rec["py"], rec["px"]] * w * w
    for ch in range(3):
        if e["clamped"][ch]:
            continue
        g[ch, :n] = ga[ch] * phi
        Hm[ch, :n, :n] = ha[ch] * np.outer(phi, phi)
    return g, Hm, True


def solve(attr, scene, k, primary: View, secs, opts):
    """solve_* (newton.hpp:588-811); returns the reference's committed delta."""
    kern = kernel_of(scene, k)
    views = [primary] + list(secs)
    if attr == 0:
        g = sum(position_terms(k, v)[0] for v in views)
        Hm = sum(position_terms(k, v)[1] for v in views)
        r, _, _ = view_direction_derivs(primary.cam, kern["p"])
        U = position_subspace(r)
        d = solve_safeguarded(U.T @ Hm @ U, U.T @ g, opts)
        dp = U @ d
        if opts["step_cap_factor"] > 0:
            cap = opts["step_cap_factor"] * np.max(kern["s"])
            nrm = np.linalg.norm(dp)
            if nrm > cap:
                dp *= cap / nrm
        return dict(delta=dp, accepted=True, degenerate=False)
    if attr == 1:
        axis, _, _ = view_direction_derivs(primary.cam, kern["p"])
        t = [rotation_terms(k, axis, v) for v in views]
        th = solve_safeguarded(np.array([[sum(x[1] for x in t)]]), np.array([sum(x[0] for x in t)]), opts)[0]
        if opts["theta_cap"] > 0:
            th = float(np.clip(th, -opts["theta_cap"], opts["theta_cap"]))
        return dict(delta=np.array([th]), accepted=True, degenerate=False, axis=axis)
    if attr == 2:
        if k in primary.entry_of:
            sub = scaling_subspace(primary.sl["entries"][primary.entry_of[k]], kern, primary.cam, opts["eigengap_rel"])
        else:
            sub = dict(degenerate=True, t_pinv=np.zeros((3, 2)))
        t = [scaling_terms(k, v, opts["eigengap_rel"]) for v in views]
        g = sum(x[0] for x in t)
        Hm = sum(x[1] for x in t)
        if sub["degenerate"]:
            d = solve_safeguarded(np.array([[Hm.sum()]]), np.array([g.sum()]), opts)[0]
            dl = np.array([d, d])
        else:
            dl = solve_safeguarded(Hm, g, opts)
        ds = sub["t_pinv"] @ dl
        s = kern["s"]
        if opts["scale_cap_factor"] > 1:
            shrink = 1.0
            for c in range(3):
                lo = s[c] / opts["scale_cap_factor"] - s[c]
                hi = s[c] * opts["scale_cap_factor"] - s[c]
                if ds[c] > hi:
                    shrink = min(shrink, hi / ds[c])
                if ds[c] < lo:
                    shrink = min(shrink, lo / ds[c])
            ds = ds * shrink
        ok = False
        for _ in range(opts["max_backtrack"] + 1):
            if np.all(s + ds > 0):
                ok = True
                break
            ds = ds * 0.5
        if not ok:
            ds = np.zeros(3)
        return dict(delta=ds, accepted=ok, degenerate=bool(sub["degenerate"]))
    if attr == 3:
        t = [opacity_terms(k, v) for v in views]
        sg = kern["sigma"]
        w = opts["barrier_weight"]
        hb = w * (1 / sg ** 2 + 1 / (1 - sg) ** 2)
        gb = -w * (1 / sg - 1 / (1 - sg))
        d = solve_safeguarded(np.array([[sum(x[1] for x in t) + hb]]), np.array([sum(x[0] for x in t) + gb]), opts)[0]
        lo, hi = np.nextafter(K_SIGMA_MARGIN, 1.0), np.nextafter(1 - K_SIGMA_MARGIN, 0.0)
        return dict(delta=np.array([min(max(sg + d, lo), hi)]), accepted=True, degenerate=False)
    n = (scene["deg"] + 1) ** 2
    t = [color_terms(k, v) for v in views]
    g = sum(x[0] for x in t)
    Hm = sum(x[1] for x in t)
    out = np.zeros((3, 16))
    for ch in range(3):
        d = solve_safeguarded(Hm[ch, :n, :n], g[ch, :n], opts)
        if opts["color_cap"] > 0 and np.linalg.norm(d) > opts["color_cap"]:
            d = d * opts["color_cap"] / np.linalg.norm(d)
        out[ch, :n] = d
    return dict(delta=out.reshape(-1), accepted=True, degenerate=False)


def commit(attr, scene, k, res):
    """commit_* (newton.hpp:817-844)."""
    if not res["accepted"]:
        return
    if attr == 0:
        scene["p"][k] = scene["p"][k] + res["delta"]
    elif attr == 1:
        th, ax = res["delta"][0], res["axis"]
        dq = np.array([math.cos(th), math.sin(th) * ax[0], math.sin(th) * ax[1], math.sin(th) * ax[2]])
        q = quaternion_multiply(dq, scene["q"][k])
        scene["q"][k] = q / np.linalg.norm(q)
    elif attr == 2:
        scene["s"][k] = scene["s"][k] + res["delta"]
    elif attr == 3:
        scene["sigma"][k] = res["delta"][0]
    else:
        n = (scene["deg"] + 1) ** 2
        d = res["delta"].reshape(3, 16)
        scene["sh"][k][:, :n] += d[:, :n]


# ---------------------------------------------------------------------------
# Context mirroring the C-ABI binding
# ---------------------------------------------------------------------------

DEFAULT_RASTER = dict(lambda_lp=K_LOWPASS, alpha_cutoff=1e-4, t_min=1e-4)
REFERENCE_RASTER = dict(lambda_lp=K_LOWPASS, alpha_cutoff=0.0, t_min=0.0)
DEFAULT_LOSS = {"lambda": 0.2, "c1": 1e-4, "c2": 9e-4, "window": 11, "window_sigma": 1.5}
DEFAULT_NEWTON = dict(mu_min=1e-8, eig_floor_rel=5e-2, step_cap_factor=1.0, scale_cap_factor=2.0, color_cap=1.0,
                      theta_cap=math.pi / 2, barrier_weight=1e-4, max_backtrack=8, eigengap_rel=1e-6)


def _opts(o, defaults):
    if o is None:
        return dict(defaults)
    if isinstance(o, dict):
        return dict(o)
    out = dict(defaults)
    for k in out:
        attr = "lambda_" if k == "lambda" else k
        if hasattr(o, attr):
            out[k] = getattr(o, attr)
    return out


class OracleContext:
    """Same surface as paper_2501_13975_b200.capi.Context (subset used by parity tests)."""

    def __init__(self):
        self.scene = None
        self.views = {}

    def set_scene(self, s):
        self.scene = dict(n=s.count, deg=int(s.sh_degree), bg=np.array(s.background, np.float64),
                          p=[np.array(x, np.float64) for x in s.position], s=[np.array(x, np.float64) for x in s.scale],
                          q=[np.array(x, np.float64) for x in s.quaternion], sigma=[float(x) for x in s.sigma],
                          sh=[np.array(x, np.float64).reshape(3, 16) for x in s.sh])
        self.views = {}

    def get_scene_arrays(self):
        sc = self.scene
        return dict(position=np.array(sc["p"]).reshape(-1, 3), scale=np.array(sc["s"]).reshape(-1, 3),
                    quaternion=np.array(sc["q"]).reshape(-1, 4), sigma=np.array(sc["sigma"]),
                    sh=np.array(sc["sh"]).reshape(-1, 3, 16))

    def _snapshot(self):
        sc = self.scene
        return dict(sc, p=[x.copy() for x in sc["p"]], s=[x.copy() for x in sc["s"]], q=[x.copy() for x in sc["q"]],
                    sigma=list(sc["sigma"]), sh=[x.copy() for x in sc["sh"]])

    def render(self, camera, options=None):
        ro = _opts(options, DEFAULT_RASTER)
        sl = build_splat_list(self.scene, Cam.of(camera), ro)
        return composite(sl, self.scene["bg"], ro)[0]

    def build_view(self, slot, camera, target, raster=None, loss=None):
        v = build_view(self._snapshot(), Cam.of(camera), target, _opts(raster, DEFAULT_RASTER), _opts(loss, DEFAULT_LOSS))
        self.views[slot] = v
        return v.loss_value

    def view_image(self, slot):
        return self.views[slot].image

    def view_loss_derivs(self, slot):
        return self.views[slot].grad, self.views[slot].hess

    def view_splats(self, slot):
        sl = self.views[slot].sl
        return dict(kernel=np.array([e["kernel"] for e in sl["entries"]], np.int32), tile_offsets=sl["offsets"],
                    tile_indices=sl["indices"])

    def accumulate(self, attr, primary, secondaries=(), options=None):
        opts = _opts(options, DEFAULT_NEWTON)
        views = [self.views[primary]] + [self.views[s] for s in secondaries]
        n = self.scene["n"]
        width = {0: 3, 1: 1, 2: 2, 3: 1, 4: 48}[attr]
        hw = {0: 9, 1: 1, 2: 4, 3: 1, 4: 768}[attr]
        G = np.zeros((n, width))
        H = np.zeros((n, hw))
        vis = np.zeros(n, bool)
        for k in range(n):
            for v in views:
                if attr == 0:
                    g, h, ok = position_terms(k, v)
                elif attr == 1:
                    axis, _, _ = view_direction_derivs(views[0].cam, self.scene["p"][k])
                    g, h, ok = rotation_terms(k, axis, v)
                elif attr == 2:
                    g, h, ok = scaling_terms(k, v, opts["eigengap_rel"])
                elif attr == 3:
                    g, h, ok = opacity_terms(k, v)
                else:
                    g, h, ok = color_terms(k, v)
                G[k] += np.ravel(g)
                H[k] += np.ravel(h)
                vis[k] |= ok
        return G, H, vis

    def newton_step(self, attr, primary, secondaries=(), options=None, commit_=True):
        opts = _opts(options, DEFAULT_NEWTON)
        pv = self.views[primary]
        secs = [self.views[s] for s in secondaries]
        res = [solve(attr, self.scene, k, pv, secs, opts) for k in range(self.scene["n"])]
        nsq = 0.0
        for k, r in enumerate(res):
            if attr == 3:
                nsq += (r["delta"][0] - self.scene["sigma"][k]) ** 2
            else:
                nsq += float(np.sum(np.asarray(r["delta"]) ** 2))
        if commit_:
            for k, r in enumerate(res):
                commit(attr, self.scene, k, r)
        width = {0: 3, 1: 1, 2: 3, 3: 1, 4: 48}[attr]
        return dict(delta=np.array([np.ravel(r["delta"]) for r in res]).reshape(-1, width),
                    accepted=np.array([r["accepted"] for r in res]), degenerate=np.array([r["degenerate"] for r in res]),
                    delta_norm_sq=nsq)


# ---------------------------------------------------------------------------
# secondary.hpp + trainer.hpp (Trainer setup and newton_step)
# ---------------------------------------------------------------------------

def knn_views(cams, positions, k):
    """fit_bounding_sphere + knn_views, secondary.hpp:24-81 (ties -> lower id)."""
    pts = np.asarray(positions, np.float64)
    ctr = pts.mean(axis=0)
    maxd = float(np.max(np.linalg.norm(pts - ctr, axis=1)))
    radius = 1.05 * maxd if maxd > 0 else 1.0
    dirs = []
    for c in cams:
        d = c.center - ctr
        n = np.linalg.norm(d)
        if not n > 1e-12:
            raise DegenerateGeometry("sphere_direction: camera at the sphere center")
        dirs.append(d / n)
    out = []
    for t in range(len(cams)):
        dist = sorted((radius * math.acos(float(np.clip(dirs[t] @ dirs[j], -1.0, 1.0))), j)
                      for j in range(len(cams)) if j != t)
        out.append([j for _, j in dist[:k]] if k > 0 and len(cams) >= 2 else [])
    return out


def clamp_downsample_factor(w, h, f):
    """secondary.hpp:85-89."""
    f = max(1, f)
    while f > 1 and (w // f < 16 or h // f < 16):
        f -= 1
    return f


def downsample_box(img, f):
    """image.hpp:39-62."""
    H, W, _ = img.shape
    ow, oh = max(1, W // f), max(1, H // f)
    out = np.zeros((oh, ow, 3))
    for y in range(oh):
        for x in range(ow):
            out[y, x] = img[y * f:min(y * f + f, H), x * f:min(x * f + f, W)].reshape(-1, 3).mean(axis=0)
    return out


class OracleTrainer:
    """Trainer (trainer.hpp:130-175) + newton_step (trainer.hpp:299-417), Newton optimiser only."""

    def __init__(self, ctx: OracleContext, cameras, targets, train_ids, secondary_targets=None,
                 secondary_downsample=0, knn=3, downsample=4, order=(0, 1, 2, 3, 4), raster=None, loss=None,
                 newton=None):
        self.ctx = ctx
        self.train_ids = list(train_ids)
        self.cams = [Cam.of(c) for c in cameras]
        self.targets = [np.asarray(t, np.float64) for t in targets]
        self.raster = _opts(raster, DEFAULT_RASTER)
        self.loss = _opts(loss, DEFAULT_LOSS)
        self.newton = _opts(newton, DEFAULT_NEWTON)
        self.order = list(order)
        self.barrier = self.newton["barrier_weight"]
        train = [self.cams[i] for i in train_ids]
        local = knn_views(train, ctx.scene["p"], knn)
        self.neighbors = [[] for _ in self.cams]
        for i, nb in enumerate(local):
            self.neighbors[train_ids[i]] = [train_ids[j] for j in nb]
        self.down_cams, self.down_targets = [], []
        exact = secondary_targets is not None and secondary_downsample == downsample
        for i, c in enumerate(self.cams):
            f = clamp_downsample_factor(c.width, c.height, downsample)
            dc = Cam(c.view, c.proj, c.width // f, c.height // f)
            self.down_cams.append(dc)
            st = np.asarray(secondary_targets[i], np.float64) if exact else None
            if st is not None and st.shape[:2] == (dc.height, dc.width):
                self.down_targets.append(st)
            else:
                self.down_targets.append(downsample_box(self.targets[i], f))

    def probe_metrics(self, probe_ids=()):
        """Trainer::probe_metrics (trainer.hpp:215-233)."""
        ids = list(probe_ids) if len(probe_ids) else list(self.train_ids)
        loss = ps = ss = 0.0
        for i in ids:
            img = self.ctx.render(self.cams[i], self.raster)
            loss += total_loss_value(img, self.targets[i], self.loss)
            p = psnr(img, self.targets[i])
            ps += 99.0 if math.isinf(p) else p
            ss += ssim_mean_value(img, self.targets[i], self.loss)
        n = float(len(ids))
        return loss / n, ps / n, ss / n

    def run(self, epochs=1, seed=0, probe_cadence=1, probe_ids=(), barrier_decay=0.5, barrier_floor=1e-6):
        """Trainer::run (trainer.hpp:238-277): [(step, image_id, probe metrics, delta norms)]."""
        rng = Rng(seed)
        last = self.probe_metrics(probe_ids)
        rows = [(0, -1, last, np.zeros(5))]
        step = 0
        for _ in range(epochs):
            order = rng.shuffle(list(self.train_ids))
            for vid in order:
                norms = self.step(vid)
                step += 1
                if probe_cadence > 0 and step % probe_cadence == 0:
                    last = self.probe_metrics(probe_ids)
                rows.append((step, vid, last, norms))
            self.barrier = max(barrier_floor, self.barrier * barrier_decay)
        return rows

    def first_order_step(self, view_id, adam, lr, state):
        """first_order_step (trainer.hpp:419-509); lr = (position, rotation, scaling,
        opacity, color); state = dict(t, m, v) Adam moments (56 per kernel)."""
        sc = self.ctx.scene
        n = sc["n"]
        prim = build_view(self.ctx._snapshot(), self.cams[view_id], self.targets[view_id], self.raster, self.loss)
        if adam:
            state["t"] += 1
        grads = []
        for k in range(n):
            kern = kernel_of(sc, k)
            axis = self.cams[view_id].center
            r = kern["p"] - axis
            axis = r / np.linalg.norm(r)
            grads.append(dict(p=position_terms(k, prim)[0], axis=axis, th=rotation_terms(k, axis, prim)[0],
                              s=scaling_gradient_s(k, prim), sig=opacity_terms(k, prim)[0],
                              col=color_terms(k, prim)[0]))
        b1, b2, eps, t = 0.9, 0.999, 1e-8, state["t"]

        def upd(k, slot, g, rate):
            if not adam:
                return -rate * g
            m = state["m"][k, slot] = b1 * state["m"][k, slot] + (1 - b1) * g
            v = state["v"][k, slot] = b2 * state["v"][k, slot] + (1 - b2) * g * g
            return -rate * (m / (1 - b1 ** t)) / (math.sqrt(v / (1 - b2 ** t)) + eps)

        nsq = np.zeros(5)
        nsh = (sc["deg"] + 1) ** 2
        lo, hi = np.nextafter(1e-4, 1.0), np.nextafter(1.0 - 1e-4, 0.0)
        for k in range(n):
            g = grads[k]
            dp = np.array([upd(k, c, g["p"][c], lr[0]) for c in range(3)])
            ds = np.array([upd(k, 4 + c, g["s"][c], lr[2]) for c in range(3)])
            dth = upd(k, 3, g["th"], lr[1])
            dsg = upd(k, 7, g["sig"], lr[3])
            sc["p"][k] = sc["p"][k] + dp
            nsq[0] += dp @ dp
            dq = np.array([math.cos(dth), *(math.sin(dth) * g["axis"])])
            q = quaternion_multiply(dq, sc["q"][k])
            sc["q"][k] = q / np.linalg.norm(q)
            nsq[1] += dth * dth
            sc["s"][k] = np.maximum(1e-8, sc["s"][k] + ds)
            nsq[2] += ds @ ds
            before = sc["sigma"][k]
            sc["sigma"][k] = min(max(before + dsg, lo), hi)
            nsq[3] += (sc["sigma"][k] - before) ** 2
            for ch in range(3):
                for c in range(nsh):
                    d = upd(k, 8 + 16 * ch + c, g["col"][ch, c], lr[4])
                    sc["sh"][k][ch, c] += d
                    nsq[4] += d * d
        return np.sqrt(nsq)

    def _views(self, view_id):
        snap = self.ctx._snapshot()
        secs = [build_view(snap, self.down_cams[j], self.down_targets[j], self.raster, self.loss)
                for j in self.neighbors[view_id]]
        prim = build_view(self.ctx._snapshot(), self.cams[view_id], self.targets[view_id], self.raster, self.loss)
        return prim, secs

    def step(self, view_id):
        opts = dict(self.newton, barrier_weight=self.barrier)
        prim, secs = self._views(view_id)
        norms = np.zeros(5)
        sc = self.ctx.scene
        for pi, attr in enumerate(self.order):
            res = [solve(attr, sc, k, prim, secs, opts) for k in range(sc["n"])]
            nsq = 0.0
            for k, r in enumerate(res):
                if attr == 3:
                    before = sc["sigma"][k]
                    commit(attr, sc, k, r)
                    nsq += (sc["sigma"][k] - before) ** 2
                else:
                    commit(attr, sc, k, r)
                    nsq += float(np.sum(np.asarray(r["delta"]) ** 2))
            norms[attr] = math.sqrt(nsq)
            if attr in (0, 1, 2) and pi + 1 < len(self.order):
                prim, secs = self._views(view_id)
        return norms
