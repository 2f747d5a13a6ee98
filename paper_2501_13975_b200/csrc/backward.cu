// backward.cu — K8: per-Gaussian gradient / Hessian accumulation for one view.
//
// Replaces invert_capture (rasterizer.hpp:489-524) + <attr>_terms
// (newton.hpp:266-574). No capture buffer is materialised: each 16x16 tile
// block re-traverses its depth-ordered splat list front to back, recomputing
// G, alpha and T bit-identically to the forward pass (splat.cuh), and derives
// the reference's "behind" colour from the final pixel colour:
//     T_{i+1} * behind_i = C_final - sum_{j<=i} T_j alpha_j c_j   (behind_last = bg)
// which is the closed form of the back-to-front recurrence at
// rasterizer.hpp:509-514.
//
// Per (pixel, splat) work is FP32. Contributions are pre-reduced across the
// warp with shuffles, across the block in shared memory, and flushed once per
// (tile, splat) into FP64 per-Gaussian accumulators with global atomics.
//
// Per-(Gaussian, view) chain-rule constants are computed once per pass in FP64
// by the *_consts kernels and staged through shared memory per batch.
#include <algorithm>

#include <cstdio>

#include "backward.h"
#include "geometry.cuh"
#include "splat.cuh"

namespace ngsb {

namespace {

inline int blocks_for(int n, int b = 256) { return (n + b - 1) / b; }

// ---------------------------------------------------------------------------
// Per-(Gaussian, view) constants (FP64 -> FP32)
// ---------------------------------------------------------------------------

// Position: M (5x3) = d(pi_x, pi_y, S00, S01, S11)/dp, Hu (5 x sym3) second
// derivatives, Jc (3x3) = dc~/dp per channel, Hc (3 x sym3) = d2c~/dp2.
// projection_derivatives camera.hpp:124-148; cov2d_derivatives_wrt_position
// camera.hpp:241-284; sh_color_derivs_wrt_position sh.hpp:134-161.
// Two blocks per 128 Gaussians (blockIdx.y): 0 = pixel / Sigma derivatives
// (JS, HPI, SCD), 1 = SH colour derivatives (JC, HC); halves the FP64 live
// state per thread. Rows are staged in shared memory and stored coalesced.
// Resident blocks per SM of the position constants (the FP64 chain is latency-bound: 6
// blocks at 80 registers, with a little spill, beat 1 block-bound 124 registers: c3 consts
// 4.26 -> 3.43 ms per step).
#ifndef NGS_PCONST_MINB
#define NGS_PCONST_MINB 6
#endif
template <int ND, int PART>
__global__ void __launch_bounds__(128, NGS_PCONST_MINB) position_consts_k(SceneDev s, CameraDev cam, CameraDev primary,
                                                         const uint8_t* flags, float* out) {
    using L = PosLayout<ND>;
    constexpr int RS = (L::JC > L::N - L::JC ? L::JC : L::N - L::JC) + 1;  // staged row stride (floats)
    __shared__ float s_o[128 * RS];
    constexpr int part = PART;
    const int lo = part == 0 ? 0 : L::JC, hi = part == 0 ? L::JC : L::N;
    const int k0 = blockIdx.x * 128, k = k0 + threadIdx.x;
    float* o = s_o + threadIdx.x * RS;  // staged row: entries [lo, hi) at [0, hi - lo)
    for (int i = 0; i < hi - lo; ++i) o[i] = 0.f;
    if (k < s.n && (flags[k] & kProjected)) {
        const D3 p = load_pos(s, k);
        // Directional derivatives along D[a] (world axes, or the primary view's
        // position subspace for kPassPositionUV): first order x . D[a], second order
        // D[a]^T X D[b]. With the identity directions the values pass through exactly.
        double D[ND][3];
        if constexpr (ND == 3) {
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int c = 0; c < 3; ++c) D[a][c] = a == c ? 1.0 : 0.0;
        } else {
            D3 rp, ux, uy;
            double np;
            if (!view_direction(primary, p, rp, np)) rp = d3(0, 0, 1);  // as solve_position_k (error flagged there)
            position_subspace(rp, ux, uy);
            D[0][0] = ux.x, D[0][1] = ux.y, D[0][2] = ux.z;
            D[1][0] = uy.x, D[1][1] = uy.y, D[1][2] = uy.z;
        }
        auto d1 = [&](const double* x, int st, int a) {  // sum_c x[c * st] D[a][c]
            return x[0] * D[a][0] + x[st] * D[a][1] + x[2 * st] * D[a][2];
        };
        auto d2 = [&](const double* h, int st, int a, int b) {  // D[a]^T H D[b], H packed sym3 with stride st
            double acc = 0.0;
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int d = 0; d < 3; ++d) acc += h[sym3(c, d) * st] * D[a][c] * D[b][d];
            return acc;
        };

        if constexpr (PART == 0) {
            // All derivatives are taken directly along the ND directions D[a]: the
            // first-order formulas are linear and the second-order ones bilinear in
            // the per-axis direction vectors, so contracting those vectors first
            // (x_a = x . D[a]) gives the directional values without the 3-axis tensors.
            auto dirv = [&](const double (&x)[3], double (&xa)[ND]) {
#pragma unroll
                for (int q = 0; q < ND; ++q) xa[q] = x[0] * D[q][0] + x[1] * D[q][1] + x[2] * D[q][2];
            };
            // pi(p) through view_proj (projection_derivatives camera.hpp:124-148).
            {
                const double* VP = cam.view_proj;
                const double hx = mrow(VP, 0, 0) * p.x + mrow(VP, 0, 1) * p.y + mrow(VP, 0, 2) * p.z + mrow(VP, 0, 3);
                const double hy = mrow(VP, 1, 0) * p.x + mrow(VP, 1, 1) * p.y + mrow(VP, 1, 2) * p.z + mrow(VP, 1, 3);
                const double hw = mrow(VP, 3, 0) * p.x + mrow(VP, 3, 1) * p.y + mrow(VP, 3, 2) * p.z + mrow(VP, 3, 3);
                double av[ND], bv[ND], wv[ND];
                dirv({mrow(VP, 0, 0), mrow(VP, 0, 1), mrow(VP, 0, 2)}, av);
                dirv({mrow(VP, 1, 0), mrow(VP, 1, 1), mrow(VP, 1, 2)}, bv);
                dirv({mrow(VP, 3, 0), mrow(VP, 3, 1), mrow(VP, 3, 2)}, wv);
                const double i1 = 1.0 / hw, i2 = i1 * i1, i3 = i2 * i1;
                const double sx = 0.5 * cam.width, sy = 0.5 * cam.height;
#pragma unroll
                for (int q = 0; q < ND; ++q) {
                    o[L::jx(q)] = static_cast<float>(sx * (av[q] * i1 - hx * i2 * wv[q]));
                    o[L::jy(q)] = static_cast<float>(sy * (bv[q] * i1 - hy * i2 * wv[q]));
                }
                int pp = 0;
#pragma unroll
                for (int q = 0; q < ND; ++q)
#pragma unroll
                    for (int r = q; r < ND; ++r, ++pp) {
                        o[L::hpi(pp, 0)] = static_cast<float>(
                            sx * (-(av[q] * wv[r] + wv[q] * av[r]) * i2 + 2.0 * hx * wv[q] * wv[r] * i3));
                        o[L::hpi(pp, 1)] = static_cast<float>(
                            sy * (-(bv[q] * wv[r] + wv[q] * bv[r]) * i2 + 2.0 * hy * wv[q] * wv[r] * i3));
                    }
            }
            // Sigma(p) through the EWA Jacobian (cov2d_derivatives_wrt_position,
            // camera.hpp:241-284). With t = W p + t_w, the chain of dJ/dt_e and
            // d2J/dt_e dt_f (camera.hpp:185-206) through W contracts to the 3-vectors
            // a~ = W^T a, w~ = W^T w (a, b, w = rows 0, 1, 3 of proj), here along D:
            //   dJ/dp_q   row0 = sx (-(w~_q a + a~_q w) / hw^2 + 2 hx w~_q w / hw^3)
            //   d2J/dp_qr row0 = sx (2 ((w~_q a + a~_q w) w~_r + a~_r w~_q w) / hw^3 - 6 hx w~_q w~_r w / hw^4)
            // (row1 with b, hy, sy), which avoids materialising the 3x3x2x3 tensors.
            {
                const D3 t = to_camera_space(cam, p);
                const double* P = cam.proj;
                const double a[3] = {mrow(P, 0, 0), mrow(P, 0, 1), mrow(P, 0, 2)};
                const double bb[3] = {mrow(P, 1, 0), mrow(P, 1, 1), mrow(P, 1, 2)};
                const double w[3] = {mrow(P, 3, 0), mrow(P, 3, 1), mrow(P, 3, 2)};
                const double hx = a[0] * t.x + a[1] * t.y + a[2] * t.z + mrow(P, 0, 3);
                const double hy = bb[0] * t.x + bb[1] * t.y + bb[2] * t.z + mrow(P, 1, 3);
                const double hw = w[0] * t.x + w[1] * t.y + w[2] * t.z + mrow(P, 3, 3);
                const double i1 = 1.0 / hw, i2 = i1 * i1, i3 = i2 * i1, i4 = i2 * i2;
                const double sx = 0.5 * cam.width, sy = 0.5 * cam.height;
                double J[6];
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    J[j] = sx * (a[j] * i1 - hx * i2 * w[j]);
                    J[3 + j] = sy * (bb[j] * i1 - hy * i2 * w[j]);
                }
                double at[ND], bt[ND], wt[ND];
                {
                    double a3[3], b3[3], w3[3];
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        a3[c] = a[0] * mrow(cam.view, 0, c) + a[1] * mrow(cam.view, 1, c) + a[2] * mrow(cam.view, 2, c);
                        b3[c] = bb[0] * mrow(cam.view, 0, c) + bb[1] * mrow(cam.view, 1, c) + bb[2] * mrow(cam.view, 2, c);
                        w3[c] = w[0] * mrow(cam.view, 0, c) + w[1] * mrow(cam.view, 1, c) + w[2] * mrow(cam.view, 2, c);
                    }
                    dirv(a3, at);
                    dirv(b3, bt);
                    dirv(w3, wt);
                }
                double A[9], m[9];
                covariance_3d(s.quat[k], s.scale[k], A);
                rotate_cov(cam, A, m);
                // mjt = m J^T (3x2)
                double mjt[6];
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj)
                        mjt[2 * i + jj] = m[3 * i] * J[3 * jj] + m[3 * i + 1] * J[3 * jj + 1] + m[3 * i + 2] * J[3 * jj + 2];
                double dj[ND][6];
#pragma unroll
                for (int q = 0; q < ND; ++q)
#pragma unroll
                    for (int j = 0; j < 3; ++j) {
                        dj[q][j] = sx * (-(wt[q] * a[j] + at[q] * w[j]) * i2 + 2.0 * hx * wt[q] * i3 * w[j]);
                        dj[q][3 + j] = sy * (-(wt[q] * bb[j] + bt[q] * w[j]) * i2 + 2.0 * hy * wt[q] * i3 * w[j]);
                    }
                auto mul23_32 = [](const double* a23, const double* b32, double out4[4]) {
#pragma unroll
                    for (int i = 0; i < 2; ++i)
#pragma unroll
                        for (int j = 0; j < 2; ++j)
                            out4[2 * i + j] = a23[3 * i] * b32[j] + a23[3 * i + 1] * b32[2 + j] + a23[3 * i + 2] * b32[4 + j];
                };
#pragma unroll
                for (int q = 0; q < ND; ++q) {
                    double tm[4];
                    mul23_32(dj[q], mjt, tm);
                    o[L::sg(q, 0)] = static_cast<float>(2.0 * tm[0]);
                    o[L::sg(q, 1)] = static_cast<float>(tm[1] + tm[2]);
                    o[L::sg(q, 2)] = static_cast<float>(2.0 * tm[3]);
                }
                int pp = 0;
#pragma unroll
                for (int q = 0; q < ND; ++q)
#pragma unroll
                    for (int r = q; r < ND; ++r, ++pp) {
                        double d2j[6];
#pragma unroll
                        for (int j = 0; j < 3; ++j) {
                            d2j[j] = sx * (2.0 * ((wt[q] * a[j] + at[q] * w[j]) * wt[r] + at[r] * wt[q] * w[j]) * i3 -
                                           6.0 * hx * wt[q] * wt[r] * i4 * w[j]);
                            d2j[3 + j] = sy * (2.0 * ((wt[q] * bb[j] + bt[q] * w[j]) * wt[r] + bt[r] * wt[q] * w[j]) * i3 -
                                               6.0 * hy * wt[q] * wt[r] * i4 * w[j]);
                        }
                        double t1[4], t2[4], md[6];
                        mul23_32(d2j, mjt, t1);
#pragma unroll
                        for (int i = 0; i < 3; ++i)
#pragma unroll
                            for (int jj = 0; jj < 2; ++jj)
                                md[2 * i + jj] = m[3 * i] * dj[r][3 * jj] + m[3 * i + 1] * dj[r][3 * jj + 1] +
                                                 m[3 * i + 2] * dj[r][3 * jj + 2];
                        mul23_32(dj[q], md, t2);
                        o[L::scd(pp, 0)] = static_cast<float>(2.0 * t1[0] + 2.0 * t2[0]);
                        o[L::scd(pp, 1)] = static_cast<float>(t1[1] + t1[2] + t2[1] + t2[2]);
                        o[L::scd(pp, 2)] = static_cast<float>(2.0 * t1[3] + 2.0 * t2[3]);
                    }
            }
        } else {
            // SH colour derivatives through r(p) (view_direction_derivatives camera.hpp:79-104,
            // sh_color_derivs_wrt_position sh.hpp:134-161), taken directly along the ND
            // directions: with u_a = (dr/dp) D[a] = (D[a] - r (r . D[a])) / n,
            //   dc/dp . D[a]        = g . u_a,
            //   D[a]^T d2c/dp2 D[b] = u_a^T H u_b + g . v_ab / n^2,
            //   v_ab = 3 r (r.D[a])(r.D[b]) - D[a] (r.D[b]) - D[b] (r.D[a]) - r (D[a].D[b]),
            // where (g, H) are the gradient / Hessian of sum_i c_i Phi_i(r) in r. v_ab and u_a
            // do not depend on the channel; the clamp of each channel is the projection's
            // (flags: zero subgradient when clamped, sh.hpp:144-147).
            D3 r;
            double n;
            double jdir[3][ND] = {}, hdir[3][ND * (ND + 1) / 2] = {};
            if (view_direction(cam, p, r, n)) {
                const double rv[3] = {r.x, r.y, r.z};
                const double inv_n = 1.0 / n, inv_n2 = inv_n * inv_n;
                double rd[ND], ua[ND][3];
#pragma unroll
                for (int a = 0; a < ND; ++a) {
                    rd[a] = rv[0] * D[a][0] + rv[1] * D[a][1] + rv[2] * D[a][2];
#pragma unroll
                    for (int i = 0; i < 3; ++i) ua[a][i] = (D[a][i] - rv[i] * rd[a]) * inv_n;
                }
                double vab[ND * (ND + 1) / 2][3];
                {
                    int pp = 0;
#pragma unroll
                    for (int a = 0; a < ND; ++a)
#pragma unroll
                        for (int b = a; b < ND; ++b, ++pp) {
                            const double dd = D[a][0] * D[b][0] + D[a][1] * D[b][1] + D[a][2] * D[b][2];
#pragma unroll
                            for (int i = 0; i < 3; ++i)
                                vab[pp][i] = (3.0 * rv[i] * rd[a] * rd[b] - D[a][i] * rd[b] - D[b][i] * rd[a] -
                                              rv[i] * dd) * inv_n2;
                        }
                }
                const uint8_t fl = flags[k];
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    if (fl & (kClamp0 << ch)) continue;
                    double c[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) c[i] = i < s.n_coeffs ? static_cast<double>(s.sh[(16 * ch + i) * s.n + k]) : 0.0;
                    double gr[3], hr[6];
                    sh_contract_derivs(r, s.sh_degree, c, gr, hr);
#pragma unroll
                    for (int a = 0; a < ND; ++a) jdir[ch][a] = gr[0] * ua[a][0] + gr[1] * ua[a][1] + gr[2] * ua[a][2];
                    int pp = 0;
#pragma unroll
                    for (int a = 0; a < ND; ++a) {
                        double hu[3];  // H u_a
#pragma unroll
                        for (int i = 0; i < 3; ++i)
                            hu[i] = hr[sym3(i, 0)] * ua[a][0] + hr[sym3(i, 1)] * ua[a][1] + hr[sym3(i, 2)] * ua[a][2];
#pragma unroll
                        for (int b = a; b < ND; ++b, ++pp)
                            hdir[ch][pp] = hu[0] * ua[b][0] + hu[1] * ua[b][1] + hu[2] * ua[b][2] +
                                           gr[0] * vab[pp][0] + gr[1] * vab[pp][1] + gr[2] * vab[pp][2];
                    }
                }
            }
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
#pragma unroll
                for (int a = 0; a < ND; ++a) o[L::jc(ch, a) - L::JC] = static_cast<float>(jdir[ch][a]);
#pragma unroll
                for (int pp = 0; pp < ND * (ND + 1) / 2; ++pp) o[L::hc(ch, pp) - L::JC] = static_cast<float>(hdir[ch][pp]);
            }
        }
    }
    __syncthreads();
    const int w = hi - lo;
    const int rows = min(128, s.n - k0);
    for (int i = threadIdx.x; i < rows * w; i += 128) {
        const int r = i / w, c = i - r * w;
        out[static_cast<size_t>(k0 + r) * L::N + lo + c] = s_o[r * RS + c];
    }
}

// Rotation: s1 = JW dA (JW)^T, s2 = JW d2A (JW)^T with the axis = primary view
// ray (newton.hpp:366-375, 638).
__global__ void __launch_bounds__(128) rotation_consts_k(SceneDev s, CameraDev cam, CameraDev primary,
                                                         const uint8_t* flags, float* out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= s.n) return;
    float* o = out + static_cast<size_t>(k) * kRotConsts;
    if (!(flags[k] & kProjected)) return;
    const D3 p = load_pos(s, k);
    D3 ax;
    double n;
    if (!view_direction(primary, p, ax, n)) ax = d3(0, 0, 1);
    const double K[9] = {0, -ax.z, ax.y, ax.z, 0, -ax.x, -ax.y, ax.x, 0};
    double A[9];
    covariance_3d(s.quat[k], s.scale[k], A);
    auto mm = [](const double* a, const double* b, double* c) {
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) c[3 * i + j] = a[3 * i] * b[j] + a[3 * i + 1] * b[3 + j] + a[3 * i + 2] * b[6 + j];
    };
    double KA[9], AK[9], KK[9], KKA[9], AKK[9], KAK[9], dA[9], d2A[9];
    mm(K, A, KA);
    mm(A, K, AK);
    mm(K, K, KK);
    mm(KK, A, KKA);
    mm(A, KK, AKK);
    mm(KA, K, KAK);
    for (int i = 0; i < 9; ++i) {
        dA[i] = 2.0 * (KA[i] - AK[i]);
        d2A[i] = 4.0 * (KKA[i] + AKK[i]) - 8.0 * KAK[i];
    }
    const D3 t = to_camera_space(cam, p);
    CamProj cp;
    project_camera_space<false, false>(cam, t, cp);
    double jw[6];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j)
            jw[3 * i + j] = cp.J[3 * i] * mrow(cam.view, 0, j) + cp.J[3 * i + 1] * mrow(cam.view, 1, j) +
                            cp.J[3 * i + 2] * mrow(cam.view, 2, j);
    auto sandwich = [&](const double* X, double out3[3]) {
        double xj[6];  // X jw^T (3x2)
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 2; ++j) xj[2 * i + j] = X[3 * i] * jw[3 * j] + X[3 * i + 1] * jw[3 * j + 1] + X[3 * i + 2] * jw[3 * j + 2];
        double r4[4];
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j) r4[2 * i + j] = jw[3 * i] * xj[j] + jw[3 * i + 1] * xj[2 + j] + jw[3 * i + 2] * xj[4 + j];
        out3[0] = r4[0];
        out3[1] = 0.5 * (r4[1] + r4[2]);
        out3[2] = r4[3];
    };
    double s1[3], s2[3];
    sandwich(dA, s1);
    sandwich(d2A, s2);
    for (int i = 0; i < 3; ++i) {
        o[i] = static_cast<float>(s1[i]);
        o[3 + i] = static_cast<float>(s2[i]);
    }
    o[6] = 0.f;
    o[7] = 0.f;
}

// Scaling: this view's Sigma eigenframe (newton.hpp:152-160, 426-432) and
// m_ij = v_i^T Q v_j.
__global__ void __launch_bounds__(128) scaling_consts_k(SceneDev s, CameraDev cam, double lambda_lp,
                                                        const uint8_t* flags, float* out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= s.n) return;
    float* o = out + static_cast<size_t>(k) * kScaleConsts;
    if (!(flags[k] & kProjected)) return;
    Projected pr;
    project_kernel(cam, load_pos(s, k), s.quat[k], s.scale[k], lambda_lp, pr);
    const Eig2 e = sym2_eigen(pr.s00, pr.s01, pr.s11);
    const double det = pr.s00 * pr.s11 - pr.s01 * pr.s01;
    const double qa = pr.s11 / det, qb = -pr.s01 / det, qc = pr.s00 / det;
    auto quad = [&](double ux, double uy, double vx, double vy) {
        return ux * (qa * vx + qb * vy) + uy * (qb * vx + qc * vy);
    };
    o[0] = static_cast<float>(e.v0x);
    o[1] = static_cast<float>(e.v0y);
    o[2] = static_cast<float>(e.v1x);
    o[3] = static_cast<float>(e.v1y);
    o[4] = static_cast<float>(quad(e.v0x, e.v0y, e.v0x, e.v0y));
    o[5] = static_cast<float>(quad(e.v0x, e.v0y, e.v1x, e.v1y));
    o[6] = static_cast<float>(quad(e.v1x, e.v1y, e.v1x, e.v1y));
    o[7] = 0.f;
}

// ---------------------------------------------------------------------------
// Tile backward kernel
// ---------------------------------------------------------------------------

// 16x16-tile batch sizes and register caps (build-time knobs for A/B runs). The
// shared-memory footprint scales with the batch: rotation / scaling at 64 splats
// and <= 64 registers fit 4 resident blocks per SM instead of 3 (c2 97.9 -> 99.8
// views/s, A/B on one box); the position (UV) pass at 32 splats / 64 registers
// also fits 4 but measured slower (97.9 -> 97.5).
#ifndef NGS_B16_UV
#define NGS_B16_UV 64
#endif
#ifndef NGS_B16_ROT
#define NGS_B16_ROT 64
#endif
#ifndef NGS_B16_SCL
#define NGS_B16_SCL 64
#endif
#ifndef NGS_B8_ROT
#define NGS_B8_ROT 64
#endif
#ifndef NGS_B8_SCL
#define NGS_B8_SCL 64
#endif
#ifndef NGS_B16_OC
#define NGS_B16_OC 64
#endif
#ifndef NGS_MAXREG16
#define NGS_MAXREG16 72
#endif
#ifndef NGS_R16_UV
#define NGS_R16_UV NGS_MAXREG16
#endif
#ifndef NGS_R16_ROT
#define NGS_R16_ROT 64
#endif
#ifndef NGS_R16_SCL
#define NGS_R16_SCL 64
#endif
#ifndef NGS_R16_OC
#define NGS_R16_OC NGS_MAXREG16
#endif
template <int PASS>
struct PassTraits;
template <>
struct PassTraits<kPassPosition> {
    static constexpr int NC = kPosConsts, NA = 9, BATCH = 32, BATCH8 = 32, R16 = NGS_MAXREG16;
};
template <>
struct PassTraits<kPassPositionUV> {
    static constexpr int NC = kPosUVConsts, NA = 5, BATCH = NGS_B16_UV, BATCH8 = 32, R16 = NGS_R16_UV;
};
template <>
struct PassTraits<kPassGrad> {
    static constexpr int NC = 0, NA = kAccGrad, BATCH = 64, BATCH8 = 64, R16 = NGS_MAXREG16;
};
template <>
struct PassTraits<kPassRotation> {
    static constexpr int NC = kRotConsts, NA = 2, BATCH = NGS_B16_ROT, BATCH8 = NGS_B8_ROT, R16 = NGS_R16_ROT;
};
template <>
struct PassTraits<kPassScaling> {
    static constexpr int NC = kScaleConsts, NA = 5, BATCH = NGS_B16_SCL, BATCH8 = NGS_B8_SCL, R16 = NGS_R16_SCL;
};
template <>
struct PassTraits<kPassOpacityColor> {
    static constexpr int NC = 0, NA = 8, BATCH = NGS_B16_OC, BATCH8 = 64, R16 = NGS_R16_OC;
};

// Copies N float4 from shared memory into a register array.
template <int N>
__device__ __forceinline__ void ld4(float (&dst)[4 * N], const float4* src) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const float4 v = src[i];
        dst[4 * i] = v.x;
        dst[4 * i + 1] = v.y;
        dst[4 * i + 2] = v.z;
        dst[4 * i + 3] = v.w;
    }
}

// One contributing (pixel, splat) record, as phase 1 hands it to phase 2.
struct Rec {
    float G, q0, q1;   // Gaussian weight and Q d at the pixel
    float Ti;          // transmittance before this splat
    float wa;          // w_alpha = sigma * T_i
    float ac[3];       // c~ - behind per channel
    float gl[3], hl[3];
};

// Position record (newton.hpp:285-340) via derivatives of the quadratic form
// q = d^T Sigma^-1 d along p (G = exp(-q/2)):
//   r_c  = J_c - S_c qd,   q_c = qd . (J_c + r_c),
//   q_cd = 2 r_c^T Q r_d + 2 qd . Hpi_cd - qd^T S_cd qd,
//   dG_c = -G q_c / 2,     d2G_cd = G (q_c q_d / 4 - q_cd / 2),
// with J = dpi/dp, S_c = dSigma/dp_c, Hpi / S_cd the second derivatives. The
// three-channel Gauss-Newton and curvature sums are regrouped so each output
// entry costs a handful of FMAs (DESIGN.md §5 "K8 position").
template <int ND>
__device__ __forceinline__ void position_record(const float4* K4, const Rec& r, float qa, float qb, float qc,
                                                float (&v)[ND + ND * (ND + 1) / 2]) {
    using L = PosLayout<ND>;
    constexpr int NP = L::NP;
    const float G = r.G, q0 = r.q0, q1 = r.q1, wa = r.wa;
    float A[L::a4(5 * ND)];
    ld4<L::a4(5 * ND) / 4>(A, K4 + L::JS / 4);
    float r0[ND], r1[ND], qcv[ND], t0[ND], t1[ND];
#pragma unroll
    for (int c = 0; c < ND; ++c) {
        const float Jx = A[2 * c], Jy = A[2 * c + 1];
        const float Sa = A[2 * ND + 3 * c], Sb = A[2 * ND + 3 * c + 1], Sc = A[2 * ND + 3 * c + 2];
        r0[c] = Jx - (Sa * q0 + Sb * q1);
        r1[c] = Jy - (Sb * q0 + Sc * q1);
        qcv[c] = q0 * (Jx + r0[c]) + q1 * (Jy + r1[c]);
        t0[c] = qa * r0[c] + qb * r1[c];
        t1[c] = qb * r0[c] + qc * r1[c];
    }
    float dG[ND], d2G[NP];
#pragma unroll
    for (int c = 0; c < ND; ++c) dG[c] = -0.5f * G * qcv[c];
    {
        float Hp[L::a4(2 * NP)], Sd[L::a4(3 * NP)];
        ld4<L::a4(2 * NP) / 4>(Hp, K4 + L::HPI / 4);
        ld4<L::a4(3 * NP) / 4>(Sd, K4 + L::SCD / 4);
        const float m00 = q0 * q0, m01 = 2.f * q0 * q1, m11 = q1 * q1;
        int p = 0;
#pragma unroll
        for (int c = 0; c < ND; ++c)
#pragma unroll
            for (int d = c; d < ND; ++d, ++p) {
                const float qcd = 2.f * (r0[c] * t0[d] + r1[c] * t1[d]) + 2.f * (q0 * Hp[2 * p] + q1 * Hp[2 * p + 1]) -
                                  (Sd[3 * p] * m00 + Sd[3 * p + 1] * m01 + Sd[3 * p + 2] * m11);
                d2G[p] = G * (0.25f * qcv[c] * qcv[d] - 0.5f * qcd);
            }
    }
    float Jc[L::a4(3 * ND)];
    ld4<L::a4(3 * ND) / 4>(Jc, K4 + L::JC / 4);
    float sgl = 0.f, A2 = 0.f, vgl[ND], vh[ND], ga[3], ha[3];
#pragma unroll
    for (int i = 0; i < ND; ++i) vgl[i] = vh[i] = 0.f;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        ga[ch] = r.gl[ch] * wa;
        ha[ch] = r.hl[ch] * wa * wa;
        sgl += ga[ch] * r.ac[ch];
        const float hac = ha[ch] * r.ac[ch];
        A2 += hac * r.ac[ch];
#pragma unroll
        for (int i = 0; i < ND; ++i) {
            vgl[i] += ga[ch] * Jc[ND * ch + i];
            vh[i] += hac * Jc[ND * ch + i];
        }
    }
    // Gauss-Newton block sum_ch hl wa^2 Jc Jc^T from the loaded Jc (not stored).
    float Hc[L::a4(3 * NP)];
    ld4<L::a4(3 * NP) / 4>(Hc, K4 + L::HC / 4);
    float JJ[NP], hc[NP];
    {
        int q = 0;
#pragma unroll
        for (int c = 0; c < ND; ++c)
#pragma unroll
            for (int d = c; d < ND; ++d, ++q) {
                JJ[q] = ha[0] * Jc[c] * Jc[d] + ha[1] * Jc[ND + c] * Jc[ND + d] + ha[2] * Jc[2 * ND + c] * Jc[2 * ND + d];
                hc[q] = ga[0] * Hc[q] + ga[1] * Hc[NP + q] + ga[2] * Hc[2 * NP + q];
            }
    }
    const float GG = G * G;
#pragma unroll
    for (int c = 0; c < ND; ++c) v[c] = sgl * dG[c] + G * vgl[c];
    int p = 0;
#pragma unroll
    for (int c = 0; c < ND; ++c)
#pragma unroll
        for (int d = c; d < ND; ++d, ++p)
            v[ND + p] = sgl * d2G[p] + G * hc[p] + dG[c] * vgl[d] + vgl[c] * dG[d] + A2 * dG[c] * dG[d] +
                        G * (dG[c] * vh[d] + vh[c] * dG[d]) + GG * JJ[p];
}

// Packed FP32 pairs (f32x2): one FFMA2/FMUL2/FADD2 issue evaluates two lanes of
// work; a scalar operand is broadcast for free (.F32 operand form).
struct f2 {
    unsigned long long u;
};
__device__ __forceinline__ f2 pk(float a, float b) {
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r.u) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ f2 bc(float a) { return pk(a, a); }
__device__ __forceinline__ void unpk(f2 v, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v.u)); }
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
    f2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.u) : "l"(a.u), "l"(b.u), "l"(c.u));
    return r;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
    f2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.u) : "l"(a.u), "l"(b.u));
    return r;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
    f2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.u) : "l"(a.u), "l"(b.u));
    return r;
}
__device__ __forceinline__ f2 lo2(float4 v) { return pk(v.x, v.y); }
__device__ __forceinline__ f2 hi2(float4 v) { return pk(v.z, v.w); }

// position_record<2> on packed pairs: every per-direction quantity (r, t, q_c, dG_c,
// the gradient) is a (u_x, u_y) pair and every diagonal second-order quantity a
// (00, 11) pair (PosLayout<2> stores the constants that way); the (01) entries stay
// scalar. Same formulas as position_record, ~40 % fewer FP32 issues.
__device__ __forceinline__ void position_record_uv(const float4* K4, const Rec& r, float qa, float qb, float qc,
                                                   float (&v)[5]) {
    using L = PosLayout<2>;
    static_assert(L::JS == 0 && L::HPI == 12 && L::SCD == 20 && L::JC == 32 && L::HC == 40, "PosLayout<2>");
    const float G = r.G, q0 = r.q0, q1 = r.q1, wa = r.wa;
    const float4 k0 = K4[0], k1 = K4[1], k2 = K4[2];      // [Jx Jy] [Sa Sb] [Sc -]
    const f2 Jx = lo2(k0), Jy = hi2(k0), Sa = lo2(k1), Sb = hi2(k1), Sc = lo2(k2);
    const f2 r0 = fma2(Sb, bc(-q1), fma2(Sa, bc(-q0), Jx));  // J_c - S_c qd (x row)
    const f2 r1 = fma2(Sc, bc(-q1), fma2(Sb, bc(-q0), Jy));  // (y row)
    const f2 qcv = fma2(bc(q1), add2(Jy, r1), mul2(bc(q0), add2(Jx, r0)));
    const f2 t0 = fma2(bc(qb), r1, mul2(bc(qa), r0));       // Q r_c
    const f2 t1 = fma2(bc(qc), r1, mul2(bc(qb), r0));
    const f2 dG = mul2(bc(-0.5f * G), qcv);
    float r00, r01, r10, r11, t00, t01, t10, t11, qc0, qc1, dG0, dG1;
    unpk(r0, r00, r01);
    unpk(r1, r10, r11);
    unpk(t0, t00, t01);
    unpk(t1, t10, t11);
    unpk(qcv, qc0, qc1);
    unpk(dG, dG0, dG1);
    const float m00 = q0 * q0, m01 = 2.f * q0 * q1, m11 = q1 * q1;
    const float4 h0 = K4[3], h1 = K4[4];                    // [Hx(00,11) Hy(00,11)] [Hx01 Hy01 - -]
    const float4 s0 = K4[5], s1 = K4[6], s2 = K4[7];        // [Sa(00,11) Sb(00,11)] [Sc(00,11) Sa01 Sb01] [Sc01 ...]
    // Diagonal (00, 11) pair of q_cd and d2G.
    const f2 rt = fma2(r1, t1, mul2(r0, t0));
    const f2 hq = fma2(bc(q1), hi2(h0), mul2(bc(q0), lo2(h0)));
    const f2 sdn = fma2(bc(-m11), lo2(s1), fma2(bc(-m01), hi2(s0), mul2(bc(-m00), lo2(s0))));
    const f2 qcd = fma2(bc(2.f), add2(rt, hq), sdn);
    const f2 d2G = fma2(bc(0.25f * G), mul2(qcv, qcv), mul2(bc(-0.5f * G), qcd));
    // Off-diagonal (01) entry.
    const float qcd01 = 2.f * (r00 * t01 + r10 * t11) + 2.f * (q0 * h1.x + q1 * h1.y) -
                        (s1.z * m00 + s1.w * m01 + s2.x * m11);
    const float d2G01 = G * (0.25f * qc0 * qc1 - 0.5f * qcd01);
    // Colour: Jc per channel is a (u_x, u_y) pair, Hc per channel a (00, 11) pair + (01).
    const float4 j0 = K4[8], j1 = K4[9];                    // [Jc0 Jc1] [Jc2 -]
    const float4 c0 = K4[10], c1 = K4[11], c2 = K4[12];     // [Hc0 Hc1] [Hc2 Hc0_01 Hc1_01] [Hc2_01 ...]
    const f2 Jc[3] = {lo2(j0), hi2(j0), lo2(j1)};
    const f2 Hd[3] = {lo2(c0), hi2(c0), lo2(c1)};
    const float Ho[3] = {c1.z, c1.w, c2.x};
    const float wa2 = wa * wa;
    float ga[3], ha[3], hac[3], sgl = 0.f, A2 = 0.f;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        ga[ch] = r.gl[ch] * wa;
        ha[ch] = r.hl[ch] * wa2;
        hac[ch] = ha[ch] * r.ac[ch];
        sgl += ga[ch] * r.ac[ch];
        A2 += hac[ch] * r.ac[ch];
    }
    f2 vgl = mul2(bc(ga[0]), Jc[0]), vh = mul2(bc(hac[0]), Jc[0]), JJ = mul2(bc(ha[0]), mul2(Jc[0], Jc[0]));
    f2 hcd = mul2(bc(ga[0]), Hd[0]);
#pragma unroll
    for (int ch = 1; ch < 3; ++ch) {
        vgl = fma2(bc(ga[ch]), Jc[ch], vgl);
        vh = fma2(bc(hac[ch]), Jc[ch], vh);
        JJ = fma2(bc(ha[ch]), mul2(Jc[ch], Jc[ch]), JJ);
        hcd = fma2(bc(ga[ch]), Hd[ch], hcd);
    }
    float JJ01 = 0.f, hc01 = 0.f;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        float ja, jb;
        unpk(Jc[ch], ja, jb);
        JJ01 += ha[ch] * ja * jb;
        hc01 += ga[ch] * Ho[ch];
    }
    const float GG = G * G;
    const f2 g = fma2(bc(sgl), dG, mul2(bc(G), vgl));
    unpk(g, v[0], v[1]);
    // diag: sgl d2G + G hc + dG (2 vgl + A2 dG + 2 G vh) + GG JJ
    const f2 w = fma2(bc(2.f * G), vh, fma2(bc(A2), dG, add2(vgl, vgl)));
    const f2 hd = fma2(dG, w, fma2(bc(GG), JJ, fma2(bc(G), hcd, mul2(bc(sgl), d2G))));
    unpk(hd, v[2], v[4]);
    float vgl0, vgl1, vh0, vh1;
    unpk(vgl, vgl0, vgl1);
    unpk(vh, vh0, vh1);
    v[3] = sgl * d2G01 + G * hc01 + dG0 * vgl1 + vgl0 * dG1 + A2 * dG0 * dG1 + G * (dG0 * vh1 + vh0 * dG1) + GG * JJ01;
}

// Rotation (newton.hpp:366-401): directional derivatives along
// dSigma/dtheta = S1, d2Sigma/dtheta2 = S2: w = S1 qd, dq = -qd.w,
// d2q = 2 w^T Q w - qd^T S2 qd.
__device__ __forceinline__ void rotation_record(const float4* K4, const Rec& r, float qa, float qb, float qc,
                                                float (&v)[2]) {
    const float4 k0 = K4[0], k1 = K4[1];
    const float q0 = r.q0, q1 = r.q1, G = r.G;
    const float w0 = k0.x * q0 + k0.y * q1, w1 = k0.y * q0 + k0.z * q1;
    const float dq = -(q0 * w0 + q1 * w1);
    const float d2q = 2.f * (w0 * (qa * w0 + qb * w1) + w1 * (qb * w0 + qc * w1)) -
                      (q0 * (k0.w * q0 + k1.x * q1) + q1 * (k1.x * q0 + k1.y * q1));
    const float dg = -0.5f * G * dq;
    const float d2g = G * (0.25f * dq * dq - 0.5f * d2q);
    float sg = 0.f, sh = 0.f;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        const float s = r.wa * r.ac[ch];
        sg += r.gl[ch] * s;
        sh += r.hl[ch] * s * s;
    }
    v[0] = sg * dg;
    v[1] = sh * dg * dg + sg * d2g;
}

// Scaling (newton.hpp:426-465): z_i = v_i . qd, dG_i = G z_i^2 / 2,
// d2G_ij = G (z_i^2 z_j^2 / 4 - z_i z_j v_i^T Q v_j).
__device__ __forceinline__ void scaling_record(const float4* K4, const Rec& r, float (&v)[5]) {
    const float4 k0 = K4[0], k1 = K4[1];
    const float G = r.G;
    const float z0 = k0.x * r.q0 + k0.y * r.q1;
    const float z1 = k0.z * r.q0 + k0.w * r.q1;
    const float zz0 = z0 * z0, zz1 = z1 * z1;
    const float dg0 = 0.5f * G * zz0, dg1 = 0.5f * G * zz1;
    const float h00 = G * (0.25f * zz0 * zz0 - zz0 * k1.x);
    const float h01 = G * (0.25f * zz0 * zz1 - z0 * z1 * k1.y);
    const float h11 = G * (0.25f * zz1 * zz1 - zz1 * k1.z);
    float sg = 0.f, sh = 0.f;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        const float s = r.wa * r.ac[ch];
        sg += r.gl[ch] * s;
        sh += r.hl[ch] * s * s;
    }
    v[0] = sg * dg0;
    v[1] = sg * dg1;
    v[2] = sh * dg0 * dg0 + sg * h00;
    v[3] = sh * dg0 * dg1 + sg * h01;
    v[4] = sh * dg1 * dg1 + sg * h11;
}

// Opacity data terms + colour accumulators (newton.hpp:516-567):
// dc/dsigma = G T a, colour weight w = alpha T = G wa.
__device__ __forceinline__ void opacity_color_record(const Rec& r, float sigma, float (&v)[8]) {
    const float GT = r.G * r.Ti;
    const float w = blend_weight(r.Ti, __fmul_rn(r.G, sigma));  // alpha T, as composited
    v[0] = 0.f;
    v[1] = 0.f;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        const float dc = GT * r.ac[ch];
        v[0] += r.gl[ch] * dc;
        v[1] += r.hl[ch] * dc * dc;
        v[2 + ch] = r.gl[ch] * w;
        v[5 + ch] = r.hl[ch] * w * w;
    }
}

// First-order record (image space): with qd = Sigma^-1 d, dG/dpi = -G qd and
// dG/dSigma = G qd qd^T / 2; sgl = sum_ch gl wa (c~ - behind) (rasterizer.hpp:116-176,
// newton.hpp:266-343 first-order parts, 472-503, 507-526, 538-574).
__device__ __forceinline__ void grad_record(const Rec& r, float sigma, float (&v)[kAccGrad]) {
    float sgl = 0.f, sgo = 0.f;
    const float w = blend_weight(r.Ti, __fmul_rn(r.G, sigma));  // alpha T, as composited
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        sgl += r.gl[ch] * r.ac[ch];
        v[5 + ch] = r.gl[ch] * w;
    }
    sgo = sgl * r.G * r.Ti;  // dL/dsigma: sum gl G T (c~ - behind)
    sgl *= r.wa;
    const float gq = sgl * r.G;
    v[0] = -gq * r.q0;
    v[1] = -gq * r.q1;
    const float h = 0.5f * gq;
    v[2] = h * r.q0 * r.q0;
    v[3] = h * r.q0 * r.q1;
    v[4] = h * r.q1 * r.q1;
    v[8] = sgo;
}

// Exact, order-independent accumulation of x * 2^kLimbShift (see backward.h).
__device__ __forceinline__ void add_fixed128(unsigned long long* limbs, float x, int* err) {
    // Non-finite partials (the FP64 path's "non-finite update" abort) and |x| >= 2^38 (the
    // 128-bit sum, binary point 2^-88, keeps 2^39 of headroom for the accumulation) raise
    // the device error flag instead of wrapping the fixed-point sum.
    if (!(fabsf(x) < 0x1p38f)) {
        atomicOr(err, kErrFixedRange);
        return;
    }
    int e;
    const float m = frexpf(x, &e);                                  // x = m 2^e, 0.5 <= |m| < 1
    const long long mi = static_cast<long long>(ldexpf(m, 24));      // exact: |mi| < 2^24
    const int sh = e - 24 + kLimbShift;                              // <= 102 for |x| < 2^38
    __int128 v = static_cast<__int128>(mi);
    v = sh >= 0 ? (v << sh) : (sh > -64 ? (v >> (-sh)) : (mi < 0 ? -1 : 0));  // truncation below 2^-88
    const unsigned __int128 u = static_cast<unsigned __int128>(v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const unsigned long long chunk = static_cast<unsigned long long>((u >> (32 * i)) & 0xffffffffull);
        if (chunk) atomicAdd(limbs + i, chunk);
    }
}

// Sum of the four 32-bit-weighted limbs as a two's-complement 128-bit integer, rounded
// ONCE to the nearest FP64 (top 64 significant bits with a sticky bit for the rest, then
// one __ull2double_rn; 64 > 53 + 2 so the sticky bit makes the single rounding exact).
__device__ __forceinline__ double fixed128_to_double(unsigned __int128 u) {
    const bool neg = static_cast<__int128>(u) < 0;
    if (neg) u = ~u + 1;
    const unsigned long long hi = static_cast<unsigned long long>(u >> 64);
    const unsigned long long lo = static_cast<unsigned long long>(u);
    if (hi == 0 && lo == 0) return 0.0;
    const int lead = hi ? 127 - __clzll(hi) : 63 - __clzll(lo);   // index of the leading 1
    unsigned long long top;
    int shift;  // value = top * 2^shift (before the sticky bit)
    if (lead <= 63) {
        top = lo;
        shift = 0;
    } else {
        shift = lead - 63;
        top = static_cast<unsigned long long>(u >> shift);
        const unsigned __int128 rest = u & ((static_cast<unsigned __int128>(1) << shift) - 1);
        if (rest) top |= 1ull;
    }
    const double d = ldexp(__ull2double_rn(top), shift - kLimbShift);
    return neg ? -d : d;
}

__global__ void limbs_to_double_k(const unsigned long long* __restrict__ limbs, double* __restrict__ acc, size_t count) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        unsigned __int128 u = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) u += static_cast<unsigned __int128>(limbs[4 * i + q]) << (32 * q);
        acc[i] = fixed128_to_double(u);
    }
}

// Stage the per-view constant rows with TMA bulk copies (cp.async.bulk + mbarrier) instead
// of 16-byte cp.async (LDGSTS) chunks spread over the block (A/B knob).
#ifndef NGS_BWD_TMA
#define NGS_BWD_TMA 0
#endif
constexpr bool kBwdTma = NGS_BWD_TMA != 0;

#ifdef NGS_COUNT_CANDIDATES
__device__ unsigned long long g_cand[6][6];
#endif

// Per-warp record queue (ring of 64 entries) between the two phases.
constexpr int kQ = 64;
// Two float4 per record (one STS.128 / LDS.128 each, consecutive slots: conflict-free)
// and the (splat, pixel) byte pair in one u16: 3 shared-memory instructions per record
// instead of 10 on each side of the queue.
struct WarpQueue {
    float4 r0[kQ];            // G, q0, q1, T_i
    float4 r1[kQ];            // w_alpha, ac0, ac1, ac2
    unsigned short jp[kQ];    // splat index in the batch | lane << 8
};

// Backward over one tile (16x16 pixels, 8 warps of 2 rows).
//  Phase 1 (per pixel, front to back over the depth-ordered splats): recompute
//    alpha and T bit-identically to the forward, derive behind, and append each
//    contributing record to the warp's queue (records end up sorted by splat).
//  Phase 2 (whenever >= 32 records are queued, and at batch end): every lane
//    evaluates one record's terms, then a segmented warp scan keyed by splat
//    reduces them and each segment tail adds into the block's per-splat sums.
//  Batch end: per-splat block sums -> FP64 global accumulators (one atomic per
//    (tile, splat, component)).
// Shared memory of one backward block (dynamic: > 48 KB for the position passes).
template <int PASS, int TILE>
struct BackwardSmem {
    using TR = PassTraits<PASS>;
    static constexpr int NT = TILE * TILE, NW = NT / 32;
    static constexpr int B = TILE == 16 ? TR::BATCH : TR::BATCH8, NA = TR::NA, NC4 = TR::NC / 4;
    static constexpr int CST = (NC4 % 8 == 0 && NC4 > 0) ? NC4 + 1 : NC4;  // float4 stride, avoids bank conflicts
    float4 raw[2][4][B];                   // staged records (pix as double2, ra, rb, rc), double-buffered
    float4 cst[2][(CST > 0 ? CST : 1) * B];  // staged per-view constants, double-buffered
    SplatSh sp[B];                         // staged splats of the batch
    double cold[3][B];                     // their colours widened to FP64 once (the FP64 prefix operand)
    unsigned char wmask[B];                // bit w: the splat's cutoff ellipse reaches warp w's pixel rows
    // Per-warp sums (segment tails are unique within a drain), as NA / 4 float4 planes
    // plus a float2 and / or a float plane for the remainder: a segment tail adds its NA
    // components with ceil-ish(NA / 4) vector read-modify-writes; lane-indexed flush
    // reads stay conflict-free; same size as [NA][B].
    static constexpr int NQ = NA / 4, R2 = (NA % 4) / 2, R1 = NA % 2;
    float4 acc4[NW][NQ > 0 ? NQ * B : 1];
    float2 acc2[NW][R2 > 0 ? B : 1];
    float acc1[NW][R1 > 0 ? B : 1];
    int kid[2][B];
    unsigned char vis[NW][B];              // per warp: the splat had >= 1 record in this warp
    float4 lg[NT];                         // per-pixel loss derivatives (gl0, gl1, gl2, hl0)
    float2 lh[NT];                         // (hl1, hl2): two loads per record instead of six
    WarpQueue q[NW];
    unsigned long long cst_bar[2];         // NGS_BWD_TMA: mbarriers of the bulk-copied constant rows
    int maxlast;
};

template <int PASS, int TILE>
__device__ __forceinline__ void backward_body(const BackwardArgs& a, const int block) {
    using TR = PassTraits<PASS>;
    using SM = BackwardSmem<PASS, TILE>;
    constexpr int NT = TILE * TILE, NW = NT / 32;
    constexpr int B = SM::B, NA = TR::NA, NC4 = SM::NC4, CST = SM::CST;
    static_assert(B <= NT && B % 32 == 0, "one loader thread per splat of a batch");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SM& S = *reinterpret_cast<SM*>(smem_raw);
    auto& s_sp = S.sp;
    constexpr int NQ = SM::NQ, R2 = SM::R2, R1 = SM::R1;
    // Component c of splat j in warp w's sums.
    auto acc_at = [&](int w, int c, int j) -> float& {
        if (c < 4 * NQ) return reinterpret_cast<float*>(&S.acc4[w][(c >> 2) * B + j])[c & 3];
        if (R2 && c < 4 * NQ + 2) return reinterpret_cast<float*>(&S.acc2[w][j])[c - 4 * NQ];
        return S.acc1[w][j];
    };
    auto& s_vis = S.vis;
    auto& s_q = S.q;
    auto& s_maxlast = S.maxlast;
    unsigned long long block_pairs = 0;

    const int chunk = a.chunks > 1 ? block % a.chunks : 0;
    const int tile = a.tile0 + (a.chunks > 1 ? block / a.chunks : block);  // owned tile rows only (multi-GPU shard)
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    int lx, ly;
    WarpBox<TILE>::pixel(threadIdx.x, lx, ly);
    const int x = tx * TILE + lx, y = ty * TILE + ly;
    const bool inside = x < a.W && y < a.H;
    const float fx = lx + 0.5f, fy = ly + 0.5f;
    const double ox = tx * TILE, oy = ty * TILE;
    const int2 range_all = a.ranges[tile];
    // this block's part of the tile's list (the whole list when chunks == 1)
    const int2 range = a.chunks > 1 ? make_int2(chunk_begin(range_all, chunk, a.chunks),
                                                chunk_begin(range_all, chunk + 1, a.chunks))
                                    : range_all;
    const size_t plane = static_cast<size_t>(a.W) * a.H;
    const size_t pidx = static_cast<size_t>(y) * a.W + x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    WarpQueue& Q = s_q[warp];

    int last = -1;
    // Final colour (the forward's FP64 image) and the FP64 colour prefix, re-accumulated with
    // exactly the forward's operations (raster_forward_k: C = fma((double)w, (double)c, C)), so
    // C_final - prefix is the exact FP64 suffix sum: behind = suffix / T_next keeps ~1e-16
    // relative error even where T_next is ~1e-4 (an FP32 prefix loses ~n*eps/T_next there).
    double Cf[3] = {0.0, 0.0, 0.0};
    float gl[3] = {0.f, 0.f, 0.f}, hl[3] = {0.f, 0.f, 0.f};
    if (inside) {
        last = a.last[pidx];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            Cf[c] = a.image[c * plane + pidx];
            gl[c] = a.loss_grad[c * plane + pidx];
            hl[c] = a.loss_hess[c * plane + pidx];
        }
    }
    S.lg[threadIdx.x] = make_float4(gl[0], gl[1], gl[2], hl[0]);
    S.lh[threadIdx.x] = make_float2(hl[1], hl[2]);
    if (threadIdx.x == 0) s_maxlast = -1;
    for (int i = threadIdx.x; i < NW * (NQ > 0 ? NQ * B : 1); i += NT) (&S.acc4[0][0])[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i = threadIdx.x; i < NW * (R2 > 0 ? B : 1); i += NT) (&S.acc2[0][0])[i] = make_float2(0.f, 0.f);
    for (int i = threadIdx.x; i < NW * (R1 > 0 ? B : 1); i += NT) (&S.acc1[0][0])[i] = 0.f;
    for (int i = threadIdx.x; i < NW * B; i += NT) (&s_vis[0][0])[i] = 0;
    __syncthreads();
    if (last >= 0) atomicMax(&s_maxlast, last);
    __syncthreads();
    const int end = min(range.y, s_maxlast + 1);
    const int wlast = __reduce_max_sync(0xffffffffu, last);  // the warp's last contributing list entry

    float T = 1.0f;
    double P[3] = {0.0, 0.0, 0.0};
    if (chunk > 0 && inside) {  // the forward's state before list entry range.x
        T = a.ck_t[(chunk - 1) * plane + pidx];
#pragma unroll
        for (int c = 0; c < 3; ++c) P[c] = a.ck_p[(3 * (chunk - 1) + c) * plane + pidx];
    }
    int qhead = 0, qcount = 0;  // warp-uniform ring state

    const float4* s_const = S.cst[0];  // constants of the batch being traversed

    // Phase 2 over queue entries [qhead, qhead + n), n <= 32.
    auto drain = [&](int n) {
#ifdef NGS_SKIP_PHASE2  // debug A/B only: phase-1 cost alone (results are wrong)
        if (lane == 0) block_pairs += n;
        qhead = (qhead + n) & (kQ - 1);
        qcount -= n;
        return;
#endif
        const bool valid = lane < n;
        const int e = (qhead + lane) & (kQ - 1);
        const unsigned jp = valid ? Q.jp[e] : 0xFFFFu;
        const int jj = valid ? static_cast<int>(jp & 0xFFu) : -1;
        float v[NA];
#pragma unroll
        for (int c = 0; c < NA; ++c) v[c] = 0.f;
        if (valid) {
            Rec r;
            const float4 r0 = Q.r0[e], r1 = Q.r1[e];
            r.G = r0.x;
            r.q0 = r0.y;
            r.q1 = r0.z;
            r.Ti = r0.w;
            r.wa = r1.x;
            r.ac[0] = r1.y;
            r.ac[1] = r1.z;
            r.ac[2] = r1.w;
            const int px = warp * 32 + static_cast<int>(jp >> 8);
            const float4 lg = S.lg[px];
            const float2 lh = S.lh[px];
            r.gl[0] = lg.x;
            r.gl[1] = lg.y;
            r.gl[2] = lg.z;
            r.hl[0] = lg.w;
            r.hl[1] = lh.x;
            r.hl[2] = lh.y;
            if constexpr (PASS == kPassPosition || PASS == kPassPositionUV) {
                const float4 g0 = s_sp[jj].g0;
                if constexpr (PASS == kPassPosition)
                    position_record<3>(s_const + jj * CST, r, g0.z, g0.w, s_sp[jj].g1.x, v);
                else
                    position_record_uv(s_const + jj * CST, r, g0.z, g0.w, s_sp[jj].g1.x, v);
            } else if constexpr (PASS == kPassRotation) {
                const float4 g0 = s_sp[jj].g0;
                rotation_record(s_const + jj * CST, r, g0.z, g0.w, s_sp[jj].g1.x, v);
            } else if constexpr (PASS == kPassScaling) {
                scaling_record(s_const + jj * CST, r, v);
            } else if constexpr (PASS == kPassGrad) {
                grad_record(r, s_sp[jj].g1.y, v);
            } else {
                opacity_color_record(r, s_sp[jj].g1.y, v);
            }
        }
        // Segmented inclusive scan keyed by splat (entries are sorted by splat, so
        // each splat is one segment and its tail lane is unique in this drain).
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int kj = __shfl_up_sync(0xffffffffu, jj, d);
            const bool take = lane >= d && kj == jj;
#pragma unroll
            for (int c = 0; c < NA; ++c) {
                const float t = __shfl_up_sync(0xffffffffu, v[c], d);
                if (take) v[c] += t;
            }
        }
        const int next = __shfl_down_sync(0xffffffffu, jj, 1);
        const bool tail = valid && (lane == 31 || next != jj);
        if (tail) {
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                float4& t = S.acc4[warp][q * B + jj];
                float4 u = t;
                u.x += v[4 * q], u.y += v[4 * q + 1], u.z += v[4 * q + 2], u.w += v[4 * q + 3];
                t = u;
            }
            if constexpr (R2 > 0) {
                float2& t = S.acc2[warp][jj];
                float2 u = t;
                u.x += v[4 * NQ];
                u.y += v[4 * NQ + 1];
                t = u;
            }
            if constexpr (R1 > 0) S.acc1[warp][jj] += v[NA - 1];
            s_vis[warp][jj] = 1;
        }
        if (lane == 0) block_pairs += n;
        qhead = (qhead + n) & (kQ - 1);
        qcount -= n;
    };

    // Software pipeline: while batch `it` is traversed, the records and constants
    // of batch it+1 are in flight (cp.async) and the list entries of batch it+2
    // are being loaded into a register.
    const int tid = threadIdx.x;
    auto issue = [&](int buf, int b0) {
        const int n = min(B, end - b0);
        for (int i = tid; i < 4 * n; i += NT) {
            const int j = i >> 2, r = i & 3;
            const int k = S.kid[buf][j];
            const void* src = r == 0 ? static_cast<const void*>(a.pix + k)
                                     : static_cast<const void*>((r == 1 ? a.ra : r == 2 ? a.rb : a.rc) + k);
            cp_async16(&S.raw[buf][r][j], src);
        }
        if constexpr (NC4 > 0) {
            const float4* src = reinterpret_cast<const float4*>(a.consts);
            if constexpr (kBwdTma) {
                // One TMA bulk copy (UBLKCP) per splat: its contiguous row of NC4 float4s.
                if (tid == 0) mbar_expect_tx(&S.cst_bar[buf], static_cast<unsigned>(n * NC4 * 16));
                if (tid < n) {
                    fence_proxy_async();  // the generic-proxy reads of this buffer (two batches ago) are done
                    bulk_copy_g2s(&S.cst[buf][tid * CST], src + static_cast<size_t>(S.kid[buf][tid]) * NC4,
                                  NC4 * 16, &S.cst_bar[buf]);
                }
            } else {
                for (int i = tid; i < n * NC4; i += NT) {
                    const int j = i / NC4, c = i - j * NC4;
                    cp_async16(&S.cst[buf][j * CST + c], src + static_cast<size_t>(S.kid[buf][j]) * NC4 + c);
                }
            }
        }
    };
    int kid_next = 0;
    if (tid < B) {
        if (range.x + tid < end) S.kid[0][tid] = a.vals[range.x + tid];
        if (range.x + B + tid < end) kid_next = a.vals[range.x + B + tid];
    }
    if constexpr (kBwdTma && NC4 > 0) {
        if (tid == 0) {
            mbar_init(&S.cst_bar[0], 1);
            mbar_init(&S.cst_bar[1], 1);
            mbar_fence_init();
        }
    }
    __syncthreads();
    if (range.x < end) issue(0, range.x);
    cp_async_commit();
    int it = 0;
    for (int base = range.x; base < end; base += B, ++it) {
        const int buf = it & 1;
        const int cnt = min(B, end - base);
        s_const = S.cst[buf];
        cp_async_wait_all();
        if constexpr (kBwdTma && NC4 > 0) mbar_wait(&S.cst_bar[buf], (it >> 1) & 1);
        __syncthreads();  // batch `it` staged by every thread; the previous batch's readers are done
        if (tid < B) {
            if (tid < cnt) {
                const double2 p = reinterpret_cast<const double2*>(S.raw[buf][0])[tid];
                const float4 ra = S.raw[buf][1][tid], rb = S.raw[buf][2][tid], rc = S.raw[buf][3][tid];
                const float qmax = reject_bound(rb.y, a.cutoff);
                const float py = static_cast<float>(p.y - oy);
                const float px = static_cast<float>(p.x - ox);
                SplatSh sp;
                sp.g0 = make_float4(px, py, ra.z, ra.w);
                sp.g1 = make_float4(rb.x, rb.y, qmax, rb.z);
                sp.g2 = make_float2(rb.w, rc.x);
                sp.pad = make_float2(0.f, 0.f);
                s_sp[tid] = sp;
                S.cold[0][tid] = rb.z;
                S.cold[1][tid] = rb.w;
                S.cold[2][tid] = rc.x;
                S.wmask[tid] = static_cast<unsigned char>(
                    WarpBox<TILE>::mask_exact(px, py, ellipse_half_extent(qmax, rc.y), ellipse_half_extent(qmax, rc.w),
                                              ra.z, ra.w, rb.x, qmax));
            } else {
                S.wmask[tid] = 0;
            }
            S.kid[buf ^ 1][tid] = kid_next;
            const int nx = base + 2 * B + tid;
            kid_next = nx < end ? a.vals[nx] : 0;
        }
        __syncthreads();
        if (base + B < end) issue(buf ^ 1, base + B);
        cp_async_commit();
        // Phase 1: only the splats whose cutoff ellipse reaches this warp's rows
        // (per-warp bit masks, increasing j), up to the warp's last contributor.
#pragma unroll 1
        for (int c32 = 0; c32 < cnt; c32 += 32) {
            unsigned m = __ballot_sync(0xffffffffu, ((S.wmask[c32 + lane] >> warp) & 1u) && base + c32 + lane <= wlast);
            while (m) {
                const int j = c32 + __ffs(m) - 1;
                m &= m - 1;
                const SplatSh sp = s_sp[j];
                SplatEval ev;
                const bool contrib = eval_splat_bf(sp, fx, fy, a.cutoff, ev) && base + j <= last;
                const unsigned ballot = __ballot_sync(0xffffffffu, contrib);
#ifdef NGS_COUNT_CANDIDATES
                if (lane == 0) {  // debug: [PASS][0] candidates, [1] with >= 1 record, [2] records; [3] = TILE 8
                    const int t = TILE == 8 ? 3 : 0;
                    atomicAdd(&g_cand[PASS][t + 0], 1ull);
                    if (ballot) atomicAdd(&g_cand[PASS][t + 1], 1ull);
                    atomicAdd(&g_cand[PASS][t + 2], static_cast<unsigned long long>(__popc(ballot)));
                }
#endif
                if (ballot) {
                    if (contrib) {  // the record, straight into the warp's queue
                        const float col[3] = {sp.g1.w, sp.g2.x, sp.g2.y};
                        const float Ti = T;
                        const float w = blend_weight(Ti, ev.alpha);
                        const float Tn = next_transmittance(Ti, ev.alpha);
                        const bool is_last = (base + j == last);
                        float inv_tn;  // behind is a derived quantity (not re-composited): approximate 1/T is enough
                        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv_tn) : "f"(Tn));
                        const double wd = static_cast<double>(w);
                        float ac[3];  // c~ - behind, behind = (C_final - prefix) / T_next (bg for the last record)
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            // colours widened once per splat at staging (S.cold), not per record
                            const double Pn = __fma_rn(wd, S.cold[c][j], P[c]);
                            const float behind =
                                is_last ? a.bg[c] : __double2float_rn(__dsub_rn(Cf[c], Pn)) * inv_tn;
                            ac[c] = col[c] - behind;
                            P[c] = Pn;
                        }
                        T = Tn;
                        const int slot = (qhead + qcount + __popc(ballot & ((1u << lane) - 1u))) & (kQ - 1);
                        Q.r0[slot] = make_float4(ev.g, ev.qd0, ev.qd1, Ti);
                        Q.r1[slot] = make_float4(sp.g1.y * Ti, ac[0], ac[1], ac[2]);
                        Q.jp[slot] = static_cast<unsigned short>(j | (lane << 8));
                    }
                    qcount += __popc(ballot);
                    __syncwarp();
                    if (qcount >= 32) {
                        drain(32);
                        __syncwarp();
                    }
                }
            }
        }
        if (qcount > 0) {
            __syncwarp();
            drain(qcount);
        }
        __syncwarp();
        // Each warp flushes its own per-splat sums (FP64 global atomics, zeros
        // skipped) and clears them: no block-wide barrier at the batch end.
        for (int i = lane; i < cnt; i += 32) {
            if (!s_vis[warp][i]) continue;
            s_vis[warp][i] = 0;
            const int k = S.kid[buf][i];
            if (a.visible) a.visible[k] = 1;
            float vals[NA];
#pragma unroll
            for (int c = 0; c < NA; ++c) {
                vals[c] = acc_at(warp, c, i);
                acc_at(warp, c, i) = 0.f;
            }
#pragma unroll
            for (int c = 0; c < NA; ++c) {
                const float val = vals[c];
                if (val == 0.f) continue;
                if (a.acc_limbs) {
                    add_fixed128(a.acc_limbs + (static_cast<size_t>(c) * a.acc_stride + k) * 4, val, a.err);
                } else {
                    atomicAdd(&a.acc[static_cast<size_t>(c) * a.acc_stride + k], static_cast<double>(val));
                }
            }
        }
    }
    if (a.contrib_pairs && lane == 0 && block_pairs) atomicAdd(a.contrib_pairs, block_pairs);
}

template <int PASS, int TILE>
__global__ void __maxnreg__(TILE == 16 ? PassTraits<PASS>::R16 : 128) backward_k(BackwardArgs a) {
    backward_body<PASS, TILE>(a, blockIdx.x);
}

// The small (8x8-tile) secondary views of a pass in ONE launch: a view's blocks follow the
// previous view's (block_end: inclusive prefix of the per-view block counts). Each view alone
// is 625 blocks of 2 warps at c2 (~10 % occupancy, latency-bound); together they fill the SMs.
template <int PASS, int TILE>
__global__ void __maxnreg__(TILE == 16 ? PassTraits<PASS>::R16 : 128) backward_batch_k(BackwardBatch b) {
    const int bid = blockIdx.x;
    int v = 0;
#pragma unroll
    for (int i = 0; i < kBackwardBatch - 1; ++i)
        if (i + 1 < b.nv && bid >= b.block_end[i]) v = i + 1;
    const int first = v == 0 ? 0 : b.block_end[v == 1 ? 0 : v == 2 ? 1 : 2];
    // static-index selects (a dynamic index into the kernel parameters would copy them to local memory)
    const BackwardArgs& a = v == 0 ? b.a[0] : v == 1 ? b.a[1] : v == 2 ? b.a[2] : b.a[3];
    backward_body<PASS, TILE>(a, bid - first);
}

}  // namespace

void compute_pass_consts(int pass, const SceneDev& scene, ViewSlot& v, const CameraDev& primary, cudaStream_t s,
                         float* out) {
    const int n = scene.n;
    if (n == 0 || pass == kPassOpacityColor || pass == kPassGrad) return;
    StageScope st(NGS_STAGE_CONSTS, s, pass == kPassPosition || pass == kPassPositionUV ? 2 : 1);
    switch (pass) {
        case kPassPosition:
            if (!out) {
                v.consts.ensure(static_cast<size_t>(n) * kPosConsts);
                out = v.consts.ptr;
            }
            position_consts_k<3, 0><<<blocks_for(n, 128), 128, 0, s>>>(scene, v.cam, primary, v.flags.ptr, out);
            position_consts_k<3, 1><<<blocks_for(n, 128), 128, 0, s>>>(scene, v.cam, primary, v.flags.ptr, out);
            break;
        case kPassPositionUV:
            if (!out) {
                v.consts.ensure(static_cast<size_t>(n) * kPosUVConsts);
                out = v.consts.ptr;
            }
            position_consts_k<2, 0><<<blocks_for(n, 128), 128, 0, s>>>(scene, v.cam, primary, v.flags.ptr, out);
            position_consts_k<2, 1><<<blocks_for(n, 128), 128, 0, s>>>(scene, v.cam, primary, v.flags.ptr, out);
            break;
        case kPassRotation:
            if (!out) {
                v.consts.ensure(static_cast<size_t>(n) * kRotConsts);
                out = v.consts.ptr;
            }
            rotation_consts_k<<<blocks_for(n, 128), 128, 0, s>>>(scene, v.cam, primary, v.flags.ptr, out);
            break;
        case kPassScaling:
            if (!out) {
                v.consts.ensure(static_cast<size_t>(n) * kScaleConsts);
                out = v.consts.ptr;
            }
            scaling_consts_k<<<blocks_for(n, 128), 128, 0, s>>>(scene, v.cam, v.raster.lambda_lp, v.flags.ptr,
                                                                 out);
            break;
        default:
            return;
    }
    CUDA_LAUNCH_CHECK();
}

template <class T>
struct SmemTag {
    using type = T;
};

namespace {
__global__ void acc_to_f32_k(const double* __restrict__ a, float* __restrict__ f, size_t count) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        f[i] = __double2float_rn(a[i]);
}
__global__ void acc_from_f32_k(const float* __restrict__ f, double* __restrict__ a, size_t count) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        a[i] = static_cast<double>(f[i]);
}
}  // namespace

void acc_to_f32(const double* acc, float* out, size_t count, cudaStream_t s) {
    if (count == 0) return;
    acc_to_f32_k<<<static_cast<int>(std::min<size_t>((count + 255) / 256, 8 * 148)), 256, 0, s>>>(acc, out, count);
    CUDA_LAUNCH_CHECK();
}

void acc_from_f32(const float* in, double* acc, size_t count, cudaStream_t s) {
    if (count == 0) return;
    acc_from_f32_k<<<static_cast<int>(std::min<size_t>((count + 255) / 256, 8 * 148)), 256, 0, s>>>(in, acc, count);
    CUDA_LAUNCH_CHECK();
}

void limbs_to_double(const unsigned long long* limbs, double* acc, size_t count, cudaStream_t s) {
    if (count == 0) return;
    limbs_to_double_k<<<static_cast<int>(std::min<size_t>((count + 255) / 256, 8 * 148)), 256, 0, s>>>(limbs, acc, count);
    CUDA_LAUNCH_CHECK();
}

namespace {

// Kernel arguments of one view's backward; false when the view has nothing to traverse.
bool make_backward_args(const SceneDev& scene, ViewSlot& v, double* acc, size_t acc_stride, uint8_t* visible,
                        unsigned long long* contrib_pairs, unsigned long long* acc_limbs, int* err, BackwardArgs& a,
                        int& blocks) {
    if (v.pairs == 0 || v.n == 0) return false;
    a.tiles_x = v.cam.tiles_x;
    a.W = v.W;
    a.H = v.H;
    a.ranges = v.ranges.ptr;
    a.vals = v.pair_val.ptr;
    a.pix = v.pix.ptr;
    a.ra = v.rec_a.ptr;
    a.rb = v.rec_b.ptr;
    a.rc = v.rec_c.ptr;
    a.image = v.image.ptr;
    a.last = v.last.ptr;
    a.loss_grad = v.loss_grad.ptr;
    a.loss_hess = v.loss_hess.ptr;
    a.consts = v.consts.ptr;
    a.cutoff = v.raster.alpha_cutoff;
    for (int c = 0; c < 3; ++c) a.bg[c] = scene.bg[c];
    a.acc = acc;
    a.acc_stride = acc_stride;
    a.acc_limbs = acc_limbs;
    a.visible = visible;
    a.contrib_pairs = contrib_pairs;
    a.err = err;
    const int own0 = std::max(0, v.raster.own_y0), own1 = std::min(v.cam.tiles_y, v.raster.own_y1);
    if (own1 <= own0) return false;
    a.tile0 = own0 * v.cam.tiles_x;
    a.chunks = v.cam.tile == 8 ? std::max(1, v.ck_chunks) : 1;
    a.ck_t = v.ck_t.ptr;
    a.ck_p = v.ck_p.ptr;
    blocks = (own1 - own0) * v.cam.tiles_x * a.chunks;
    return true;
}

template <int PASS, int TILE>
struct BackwardKernels {
    using SM = BackwardSmem<PASS, TILE>;
    static void single(const BackwardArgs& a, int blocks, cudaStream_t s) {
        ensure_dynamic_smem(reinterpret_cast<const void*>(backward_k<PASS, TILE>), sizeof(SM));
        backward_k<PASS, TILE><<<blocks, TILE * TILE, sizeof(SM), s>>>(a);
    }
    static void batch(const BackwardBatch& b, int blocks, cudaStream_t s) {
        ensure_dynamic_smem(reinterpret_cast<const void*>(backward_batch_k<PASS, TILE>), sizeof(SM));
        backward_batch_k<PASS, TILE><<<blocks, TILE * TILE, sizeof(SM), s>>>(b);
    }
};

template <template <int, int> class K, typename F>
void dispatch_pass(int pass, bool small, F&& f) {
    switch (pass) {
        case kPassPosition: small ? f(K<kPassPosition, 8>{}) : f(K<kPassPosition, 16>{}); break;
        case kPassPositionUV: small ? f(K<kPassPositionUV, 8>{}) : f(K<kPassPositionUV, 16>{}); break;
        case kPassGrad: small ? f(K<kPassGrad, 8>{}) : f(K<kPassGrad, 16>{}); break;
        case kPassRotation: small ? f(K<kPassRotation, 8>{}) : f(K<kPassRotation, 16>{}); break;
        case kPassScaling: small ? f(K<kPassScaling, 8>{}) : f(K<kPassScaling, 16>{}); break;
        default: small ? f(K<kPassOpacityColor, 8>{}) : f(K<kPassOpacityColor, 16>{}); break;
    }
}

int stage_of(int pass) {
    return NGS_STAGE_BWD_POSITION + (pass == kPassPositionUV || pass == kPassGrad ? kPassPosition : pass);
}

}  // namespace

#ifdef NGS_COUNT_CANDIDATES
void dump_candidates() {
    unsigned long long h[6][6];
    cudaMemcpyFromSymbol(h, g_cand, sizeof(h));
    for (int p = 0; p < 6; ++p)
        fprintf(stderr, "[candidates] pass %d: 16x16 iters %llu with-record %llu records %llu | 8x8 iters %llu with-record %llu records %llu\n",
                p, h[p][0], h[p][1], h[p][2], h[p][3], h[p][4], h[p][5]);
    unsigned long long z[6][6] = {};
    cudaMemcpyToSymbol(g_cand, z, sizeof(z));
}
#endif

void launch_backward(int pass, const SceneDev& scene, ViewSlot& v, double* acc, size_t acc_stride, uint8_t* visible,
                     unsigned long long* contrib_pairs, cudaStream_t s, unsigned long long* acc_limbs, int* err,
                     int primary_tag) {
    if (acc_limbs && !err) throw Error(NGS_ERR_INTERNAL, "launch_backward: deterministic mode needs the error flag");
    BackwardArgs a;
    int blocks = 0;
    if (!make_backward_args(scene, v, acc, acc_stride, visible, contrib_pairs, acc_limbs, err, a, blocks)) return;
    StageScope st(stage_of(pass), s, 1, primary_tag);
    dispatch_pass<BackwardKernels>(pass, v.cam.tile == 8, [&](auto k) { decltype(k)::single(a, blocks, s); });
    CUDA_LAUNCH_CHECK();
}

void launch_backward_batch(int pass, const SceneDev& scene, ViewSlot* const* views, int nv, double* const* acc,
                           size_t acc_stride, uint8_t* visible, unsigned long long* contrib_pairs, cudaStream_t s,
                           unsigned long long* const* acc_limbs, int* err) {
    if (nv > kBackwardBatch) throw Error(NGS_ERR_INTERNAL, "launch_backward_batch: too many views");
    BackwardBatch b{};
    int total = 0, tile = 0;
    for (int i = 0; i < nv; ++i) {
        if (acc_limbs && acc_limbs[i] && !err)
            throw Error(NGS_ERR_INTERNAL, "launch_backward: deterministic mode needs the error flag");
        int blocks = 0;
        if (!make_backward_args(scene, *views[i], acc[i], acc_stride, visible, contrib_pairs,
                                acc_limbs ? acc_limbs[i] : nullptr, err, b.a[b.nv], blocks))
            continue;
        if (tile != 0 && views[i]->cam.tile != tile) throw Error(NGS_ERR_INTERNAL, "backward batch: mixed tile sizes");
        tile = views[i]->cam.tile;
        total += blocks;
        b.block_end[b.nv++] = total;
    }
    if (b.nv == 0) return;
    for (int i = b.nv; i < kBackwardBatch; ++i) b.block_end[i] = total;
    StageScope st(stage_of(pass), s, 1);
    dispatch_pass<BackwardKernels>(pass, tile == 8, [&](auto k) { decltype(k)::batch(b, total, s); });
    CUDA_LAUNCH_CHECK();
}

}  // namespace ngsb
