// geometry.cuh — FP64 per-kernel geometry on the device.
//
// O(N) work per view (projection, analytic derivative constants, local
// solves) runs in FP64: B200 keeps a full-rate-class FP64 pipe, these stages
// are a small fraction of the step, and they carry the ill-conditioned pieces
// (Sigma^-1 of anisotropic kernels, eigenvectors of near-isotropic Sigma) that
// FP32 cannot reproduce against the float64 reference. The per-(pixel,splat)
// hot loops run in FP32 (raster.cu, backward.cu).
//
// Every function cites the reference routine it restates.
#pragma once

#include <math.h>

#include "common.cuh"

namespace ngsb {

struct D3 {
    double x, y, z;
};

__device__ __forceinline__ D3 d3(double x, double y, double z) { return {x, y, z}; }
__device__ __forceinline__ double dot3(const D3& a, const D3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ D3 sub3(const D3& a, const D3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ D3 scale3(const D3& a, double s) { return {a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ D3 cross3(const D3& a, const D3& b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ double comp(const D3& a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }

// Symmetric 3x3 packed (xx, xy, xz, yy, yz, zz).
__device__ __forceinline__ int sym3(int i, int j) {
    const int a = i < j ? i : j, b = i < j ? j : i;
    return a == 0 ? b : (a == 1 ? 2 + b : 5);
}

// quaternion_to_rotation, scene.hpp:40-53 (renormalise if off the unit sphere by > 1e-12).
__device__ inline void quat_to_rot(double w, double x, double y, double z, double r[9]) {
    const double n = sqrt(w * w + x * x + y * y + z * z);
    if (fabs(n - 1.0) > 1e-12) {
        w /= n;
        x /= n;
        y /= n;
        z /= n;
    }
    r[0] = 1 - 2 * (y * y + z * z);
    r[1] = 2 * (x * y - w * z);
    r[2] = 2 * (x * z + w * y);
    r[3] = 2 * (x * y + w * z);
    r[4] = 1 - 2 * (x * x + z * z);
    r[5] = 2 * (y * z - w * x);
    r[6] = 2 * (x * z - w * y);
    r[7] = 2 * (y * z + w * x);
    r[8] = 1 - 2 * (x * x + y * y);
}

// A = R S S^T R^T, scene.hpp:56-63 (row-major 3x3).
__device__ inline void covariance_3d(const float4 q, const float4 s, double a[9]) {
    double r[9];
    quat_to_rot(q.x, q.y, q.z, q.w, r);
    const double sc[3] = {s.x, s.y, s.z};
    double rs[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) rs[3 * i + j] = r[3 * i + j] * sc[j];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double v = 0;
            for (int k = 0; k < 3; ++k) v += rs[3 * i + k] * rs[3 * j + k];
            a[3 * i + j] = v;
        }
}

// M = W3 A W3^T with W3 = view rotation (camera.hpp:226).
__device__ inline void rotate_cov(const CameraDev& cam, const double a[9], double m[9]) {
    double wa[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double v = 0;
            for (int k = 0; k < 3; ++k) v += mrow(cam.view, i, k) * a[3 * k + j];
            wa[3 * i + j] = v;
        }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double v = 0;
            for (int k = 0; k < 3; ++k) v += wa[3 * i + k] * mrow(cam.view, j, k);
            m[3 * i + j] = v;
        }
}

__device__ inline D3 to_camera_space(const CameraDev& cam, const D3& p) {
    return {mrow(cam.view, 0, 0) * p.x + mrow(cam.view, 0, 1) * p.y + mrow(cam.view, 0, 2) * p.z + mrow(cam.view, 0, 3),
            mrow(cam.view, 1, 0) * p.x + mrow(cam.view, 1, 1) * p.y + mrow(cam.view, 1, 2) * p.z + mrow(cam.view, 1, 3),
            mrow(cam.view, 2, 0) * p.x + mrow(cam.view, 2, 1) * p.y + mrow(cam.view, 2, 2) * p.z + mrow(cam.view, 2, 3)};
}

// detail::project_camera_space, camera.hpp:163-208 — pixel Jacobian J = dpi/dt of
// a camera-space point through `proj`, optionally with dJ/dt_e and d2J/dt_e dt_f.
struct CamProj {
    double hw;
    double J[6];         // 2x3 row-major
    double dJ[3][6];     // dJ/dt_e
    double d2J[3][3][6]; // d2J/dt_e dt_f
};

template <bool kFirst, bool kSecond>
__device__ inline bool project_camera_space(const CameraDev& cam, const D3& t, CamProj& out) {
    const double* P = cam.proj;
    const double hx = mrow(P, 0, 0) * t.x + mrow(P, 0, 1) * t.y + mrow(P, 0, 2) * t.z + mrow(P, 0, 3);
    const double hy = mrow(P, 1, 0) * t.x + mrow(P, 1, 1) * t.y + mrow(P, 1, 2) * t.z + mrow(P, 1, 3);
    const double hw = mrow(P, 3, 0) * t.x + mrow(P, 3, 1) * t.y + mrow(P, 3, 2) * t.z + mrow(P, 3, 3);
    if (!(hw > kNearPlaneEps)) return false;
    const double a[3] = {mrow(P, 0, 0), mrow(P, 0, 1), mrow(P, 0, 2)};
    const double b[3] = {mrow(P, 1, 0), mrow(P, 1, 1), mrow(P, 1, 2)};
    const double w[3] = {mrow(P, 3, 0), mrow(P, 3, 1), mrow(P, 3, 2)};
    const double i1 = 1.0 / hw, i2 = i1 * i1, i3 = i2 * i1, i4 = i2 * i2;
    const double sx = 0.5 * cam.width, sy = 0.5 * cam.height;
    out.hw = hw;
    for (int j = 0; j < 3; ++j) {
        out.J[j] = sx * (a[j] * i1 - hx * i2 * w[j]);
        out.J[3 + j] = sy * (b[j] * i1 - hy * i2 * w[j]);
    }
    if (kFirst) {
        for (int e = 0; e < 3; ++e)
            for (int j = 0; j < 3; ++j) {
                out.dJ[e][j] = sx * (-(w[e] * a[j] + a[e] * w[j]) * i2 + 2.0 * hx * w[e] * i3 * w[j]);
                out.dJ[e][3 + j] = sy * (-(w[e] * b[j] + b[e] * w[j]) * i2 + 2.0 * hy * w[e] * i3 * w[j]);
            }
    }
    if (kSecond) {
        for (int e = 0; e < 3; ++e)
            for (int f = 0; f < 3; ++f)
                for (int j = 0; j < 3; ++j) {
                    out.d2J[e][f][j] = sx * (2.0 * ((w[e] * a[j] + a[e] * w[j]) * w[f] + a[f] * w[e] * w[j]) * i3 -
                                             6.0 * hx * w[e] * w[f] * i4 * w[j]);
                    out.d2J[e][f][3 + j] = sy * (2.0 * ((w[e] * b[j] + b[e] * w[j]) * w[f] + b[f] * w[e] * w[j]) * i3 -
                                                 6.0 * hy * w[e] * w[f] * i4 * w[j]);
                }
    }
    return true;
}

// Sigma = J M J^T + lp I, symmetrised (camera.hpp:219-232). Returns (s00, s01, s11).
__device__ inline void ewa_sigma(const double J[6], const double m[9], double lp, double& s00, double& s01,
                                 double& s11) {
    double jm[6];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j) jm[3 * i + j] = J[3 * i] * m[j] + J[3 * i + 1] * m[3 + j] + J[3 * i + 2] * m[6 + j];
    double s[4];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j)
            s[2 * i + j] = jm[3 * i] * J[3 * j] + jm[3 * i + 1] * J[3 * j + 1] + jm[3 * i + 2] * J[3 * j + 2];
    s[0] += lp;
    s[3] += lp;
    s00 = s[0];
    s11 = s[3];
    s01 = 0.5 * (s[1] + s[2]);
}

// Full per-kernel projection (camera.hpp:319-339 project_kernel): pixel, depth,
// Sigma (low-pass included), EWA Jacobian. Returns false if culled.
struct Projected {
    double px, py, depth;
    double s00, s01, s11;
    double J[6];
    double m[9];  // W A W^T
};

__device__ inline bool project_kernel(const CameraDev& cam, const D3& p, const float4 q, const float4 s,
                                      double lambda_lp, Projected& out) {
    const double* VP = cam.view_proj;
    const double hx = mrow(VP, 0, 0) * p.x + mrow(VP, 0, 1) * p.y + mrow(VP, 0, 2) * p.z + mrow(VP, 0, 3);
    const double hy = mrow(VP, 1, 0) * p.x + mrow(VP, 1, 1) * p.y + mrow(VP, 1, 2) * p.z + mrow(VP, 1, 3);
    const double hw = mrow(VP, 3, 0) * p.x + mrow(VP, 3, 1) * p.y + mrow(VP, 3, 2) * p.z + mrow(VP, 3, 3);
    if (!(hw > kNearPlaneEps)) return false;
    out.px = 0.5 * cam.width * (hx / hw + 1.0);
    out.py = 0.5 * cam.height * (hy / hw + 1.0);
    out.depth = mrow(cam.view, 2, 0) * p.x + mrow(cam.view, 2, 1) * p.y + mrow(cam.view, 2, 2) * p.z +
                mrow(cam.view, 2, 3);
    const D3 t = to_camera_space(cam, p);
    CamProj cp;
    if (!project_camera_space<false, false>(cam, t, cp)) return false;
    double a[9];
    covariance_3d(q, s, a);
    rotate_cov(cam, a, out.m);
    for (int i = 0; i < 6; ++i) out.J[i] = cp.J[i];
    ewa_sigma(cp.J, out.m, lambda_lp, out.s00, out.s01, out.s11);
    return true;
}

// sym2_eigen, newton.hpp:41-56: ascending eigenvalues, orthonormal columns.
struct Eig2 {
    double l0, l1;
    double v0x, v0y, v1x, v1y;  // columns
};

__device__ inline Eig2 sym2_eigen(double a, double b, double c) {
    Eig2 e;
    const double half_tr = 0.5 * (a + c);
    const double disc = sqrt(fmax(0.0, 0.25 * (a - c) * (a - c) + b * b));
    e.l0 = half_tr - disc;
    e.l1 = half_tr + disc;
    e.v0x = 1;
    e.v0y = 0;
    e.v1x = 0;
    e.v1y = 1;
    if (disc < 1e-300) return e;
    double vx = b, vy = e.l1 - a;
    if (vx * vx + vy * vy < 1e-300) {
        vx = e.l1 - c;
        vy = b;
    }
    if (vx * vx + vy * vy < 1e-300) {
        vx = 1;
        vy = 0;
    }
    const double n = sqrt(vx * vx + vy * vy);
    vx /= n;
    vy /= n;
    e.v1x = vx;
    e.v1y = vy;
    e.v0x = -vy;
    e.v0y = vx;
    return e;
}

// ---- spherical harmonics (sh.hpp:13-123) ------------------------------------

constexpr double kSH0 = 0.28209479177387814;
constexpr double kSH1 = 0.4886025119029199;
constexpr double kSH2_0 = 1.0925484305920792, kSH2_1 = -1.0925484305920792, kSH2_2 = 0.31539156525252005,
                 kSH2_3 = -1.0925484305920792, kSH2_4 = 0.5462742152960396;
constexpr double kSH3_0 = -0.5900435899266435, kSH3_1 = 2.890611442640554, kSH3_2 = -0.4570457994644658,
                 kSH3_3 = 0.3731763325901154, kSH3_4 = -0.4570457994644658, kSH3_5 = 1.445305721320277,
                 kSH3_6 = -0.5900435899266435;

// eval_sh_basis values only (sh.hpp:35-105).
__device__ inline void sh_basis(const D3& r, int degree, double v[16]) {
    for (int i = 0; i < 16; ++i) v[i] = 0.0;
    const double x = r.x, y = r.y, z = r.z;
    v[0] = kSH0;
    if (degree < 1) return;
    v[1] = -kSH1 * y;
    v[2] = kSH1 * z;
    v[3] = -kSH1 * x;
    if (degree < 2) return;
    const double xx = x * x, yy = y * y, zz = z * z;
    v[4] = kSH2_0 * x * y;
    v[5] = kSH2_1 * y * z;
    v[6] = kSH2_2 * (2 * zz - xx - yy);
    v[7] = kSH2_3 * x * z;
    v[8] = kSH2_4 * (xx - yy);
    if (degree < 3) return;
    v[9] = kSH3_0 * y * (3 * xx - yy);
    v[10] = kSH3_1 * x * y * z;
    v[11] = kSH3_2 * y * (4 * zz - xx - yy);
    v[12] = kSH3_3 * z * (2 * zz - 3 * xx - 3 * yy);
    v[13] = kSH3_4 * x * (4 * zz - xx - yy);
    v[14] = kSH3_5 * z * (xx - yy);
    v[15] = kSH3_6 * x * (xx - 3 * yy);
}

// d c~/dr and d2 c~/dr2 for one channel: sum_i c_i grad Phi_i, sum_i c_i hess Phi_i
// (sh.hpp:61-104 basis derivatives contracted as in sh.hpp:149-155).
__device__ inline void sh_contract_derivs(const D3& r, int degree, const double c[16], double g[3], double h[6]) {
    const double x = r.x, y = r.y, z = r.z;
    for (int i = 0; i < 3; ++i) g[i] = 0;
    for (int i = 0; i < 6; ++i) h[i] = 0;
    if (degree < 1) return;
    g[1] += -kSH1 * c[1];
    g[2] += kSH1 * c[2];
    g[0] += -kSH1 * c[3];
    if (degree < 2) return;
    const double xx = x * x, yy = y * y, zz = z * z;
    // jacobian rows 4..8
    g[0] += c[4] * kSH2_0 * y;
    g[1] += c[4] * kSH2_0 * x;
    g[1] += c[5] * kSH2_1 * z;
    g[2] += c[5] * kSH2_1 * y;
    g[0] += c[6] * kSH2_2 * (-2 * x);
    g[1] += c[6] * kSH2_2 * (-2 * y);
    g[2] += c[6] * kSH2_2 * (4 * z);
    g[0] += c[7] * kSH2_3 * z;
    g[2] += c[7] * kSH2_3 * x;
    g[0] += c[8] * kSH2_4 * (2 * x);
    g[1] += c[8] * kSH2_4 * (-2 * y);
    // hessians 4..8 (packed xx, xy, xz, yy, yz, zz)
    h[1] += c[4] * kSH2_0;
    h[4] += c[5] * kSH2_1;
    h[0] += c[6] * kSH2_2 * -2;
    h[3] += c[6] * kSH2_2 * -2;
    h[5] += c[6] * kSH2_2 * 4;
    h[2] += c[7] * kSH2_3;
    h[0] += c[8] * kSH2_4 * 2;
    h[3] += c[8] * kSH2_4 * -2;
    if (degree < 3) return;
    // jacobian rows 9..15
    g[0] += c[9] * kSH3_0 * (6 * x * y);
    g[1] += c[9] * kSH3_0 * (3 * xx - 3 * yy);
    g[0] += c[10] * kSH3_1 * (y * z);
    g[1] += c[10] * kSH3_1 * (x * z);
    g[2] += c[10] * kSH3_1 * (x * y);
    g[0] += c[11] * kSH3_2 * (-2 * x * y);
    g[1] += c[11] * kSH3_2 * (4 * zz - xx - 3 * yy);
    g[2] += c[11] * kSH3_2 * (8 * y * z);
    g[0] += c[12] * kSH3_3 * (-6 * x * z);
    g[1] += c[12] * kSH3_3 * (-6 * y * z);
    g[2] += c[12] * kSH3_3 * (6 * zz - 3 * xx - 3 * yy);
    g[0] += c[13] * kSH3_4 * (4 * zz - 3 * xx - yy);
    g[1] += c[13] * kSH3_4 * (-2 * x * y);
    g[2] += c[13] * kSH3_4 * (8 * x * z);
    g[0] += c[14] * kSH3_5 * (2 * x * z);
    g[1] += c[14] * kSH3_5 * (-2 * y * z);
    g[2] += c[14] * kSH3_5 * (xx - yy);
    g[0] += c[15] * kSH3_6 * (3 * xx - 3 * yy);
    g[1] += c[15] * kSH3_6 * (-6 * x * y);
    // hessians 9..15 (sh.hpp:90-103)
    {
        const double k = c[9] * kSH3_0;
        h[0] += k * 6 * y;
        h[1] += k * 6 * x;
        h[3] += k * -6 * y;
    }
    {
        const double k = c[10] * kSH3_1;
        h[1] += k * z;
        h[2] += k * y;
        h[4] += k * x;
    }
    {
        const double k = c[11] * kSH3_2;
        h[0] += k * -2 * y;
        h[1] += k * -2 * x;
        h[3] += k * -6 * y;
        h[4] += k * 8 * z;
        h[5] += k * 8 * y;
    }
    {
        const double k = c[12] * kSH3_3;
        h[0] += k * -6 * z;
        h[2] += k * -6 * x;
        h[3] += k * -6 * z;
        h[4] += k * -6 * y;
        h[5] += k * 12 * z;
    }
    {
        const double k = c[13] * kSH3_4;
        h[0] += k * -6 * x;
        h[1] += k * -2 * y;
        h[2] += k * 8 * z;
        h[3] += k * -2 * x;
        h[5] += k * 8 * x;
    }
    {
        const double k = c[14] * kSH3_5;
        h[0] += k * 2 * z;
        h[2] += k * 2 * x;
        h[3] += k * -2 * z;
        h[4] += k * -2 * y;
    }
    {
        const double k = c[15] * kSH3_6;
        h[0] += k * 6 * x;
        h[1] += k * -6 * y;
        h[3] += k * -6 * x;
    }
}

// view_direction, camera.hpp:63-70. Returns false when degenerate.
__device__ inline bool view_direction(const CameraDev& cam, const D3& p, D3& r, double& n) {
    const D3 u = {p.x - cam.center[0], p.y - cam.center[1], p.z - cam.center[2]};
    n = sqrt(dot3(u, u));
    if (!(n > 1e-12)) return false;
    r = scale3(u, 1.0 / n);
    return true;
}

// build_position_subspace (newton.hpp:130-139): u_y = Gram-Schmidt of the world
// up axis (z near the poles) against the ray r, u_x = r x u_y.
__device__ inline void position_subspace(const D3& r, D3& ux, D3& uy) {
    D3 seed = d3(0, 1, 0);
    if (fabs(dot3(r, seed)) > 0.99) seed = d3(0, 0, 1);
    uy = sub3(seed, scale3(r, dot3(r, seed)));
    uy = scale3(uy, 1.0 / sqrt(dot3(uy, uy)));
    ux = cross3(r, uy);
}

__device__ inline D3 load_pos(const SceneDev& s, int k) {
    const float4 v = s.pos_sigma[k];
    return {v.x, v.y, v.z};
}

}  // namespace ngsb
