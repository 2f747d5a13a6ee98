// solve.cu — K9: one-thread-per-Gaussian safeguarded local Newton solves and
// commits (solve_* newton.hpp:588-811, commit_* newton.hpp:817-844).
//
// FP64 in registers. Each thread reads only its own kernel's accumulators and
// parameters and writes only its own parameters, so solve+commit in one
// kernel has exactly the reference's Jacobi semantics (trainer.hpp:331-343).
// The spectrum repair is psd_safeguard (newton.hpp:205-238): closed-form 1x1 /
// 2x2, and for SH colour an exact low-rank eigen-decomposition of
// H = sum_v h_v phi_v phi_v^T (rank <= views) instead of a dense n x n Jacobi.
#include "backward.h"
#include "geometry.cuh"
#include "solve.h"

// Minimum resident blocks per SM of the 4-view colour solve (build-time knob for A/B runs).
#ifndef NGS_COLOR4_MINB
#define NGS_COLOR4_MINB 5
#endif
#ifndef NGS_COLORF4_MINB  // ... and of the fused one-launch colour solve
#define NGS_COLORF4_MINB 3
#endif

constexpr double kJacobiTol = 1e-28;  // (1e-20 / 1e-16 measured: c4 colour 7.18 -> 7.10 / 7.27 ms, kept)

namespace ngsb {

namespace {

inline int blocks_for(int n, int b = 256) { return (n + b - 1) / b; }

__device__ __forceinline__ void block_add(double v, unsigned long long* target) {
    __shared__ double red[8];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // a previous block_add's thread 0 may still be reading red[] (first_order_k calls this
    // once per attribute back to back): overwrite only after it is done
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0;
        for (int i = 0; i < (blockDim.x >> 5); ++i) t += red[i];
        exact_add(target, t);  // order-independent: the report's norms are bitwise reproducible
    }
}

// psd_safeguard + LDLT solve for n = 1 (newton.hpp:208-214, 240-244).
__device__ __forceinline__ double solve1(double h, double g, const SolveParams& p) {
    const double mu = fmax(p.mu_min, p.eig_floor_rel * fabs(h));
    const double hs = fmax(fabs(h), mu);
    return -g / hs;
}

// psd_safeguard n = 2 (newton.hpp:215-227) + solve.
__device__ __forceinline__ void solve2(double h00, double h01, double h11, double g0, double g1, const SolveParams& p,
                                       double& d0, double& d1) {
    const Eig2 e = sym2_eigen(h00, h01, h11);
    const double lam_max = fmax(fabs(e.l0), fabs(e.l1));
    const double mu = fmax(p.mu_min, p.eig_floor_rel * lam_max);
    double a = h00, b = h01, c = h11;
    if (!(e.l0 >= mu)) {
        const double l0 = fmax(fabs(e.l0), mu), l1 = fmax(fabs(e.l1), mu);
        a = l0 * e.v0x * e.v0x + l1 * e.v1x * e.v1x;
        b = l0 * e.v0x * e.v0y + l1 * e.v1x * e.v1y;
        c = l0 * e.v0y * e.v0y + l1 * e.v1y * e.v1y;
    }
    const double det = a * c - b * b;
    d0 = -(c * g0 - b * g1) / det;
    d1 = -(-b * g0 + a * g1) / det;
}

__device__ inline bool primary_dir(const CameraDev& cam, const D3& p, D3& r, int* err) {
    double n;
    if (!view_direction(cam, p, r, n)) {
        atomicOr(err, 2);
        r = d3(0, 0, 1);
        return false;
    }
    return true;
}

__global__ void __launch_bounds__(256) solve_position_k(SceneDev s, CameraDev primary, SolveParams sp,
                                                        const double* __restrict__ acc, size_t stride,
                                                        SolveOutputs out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    double nsq = 0.0;
    if (k < s.n) {
        const float4 ps = s.pos_sigma[k];
        const D3 p = {ps.x, ps.y, ps.z};
        // Accumulators of kPassPositionUV: already U^T g and U^T H U (newton.hpp:604-606).
        D3 r;
        primary_dir(primary, p, r, out.err);
        D3 ux, uy;
        position_subspace(r, ux, uy);
        const double U[3][2] = {{ux.x, uy.x}, {ux.y, uy.y}, {ux.z, uy.z}};
        const double g2[2] = {acc[k], acc[stride + k]};
        const double H2[2][2] = {{acc[2 * stride + k], acc[3 * stride + k]},
                                 {acc[3 * stride + k], acc[4 * stride + k]}};
        double d0, d1;
        solve2(H2[0][0], 0.5 * (H2[0][1] + H2[1][0]), H2[1][1], g2[0], g2[1], sp, d0, d1);
        double dp[3];
        for (int i = 0; i < 3; ++i) dp[i] = U[i][0] * d0 + U[i][1] * d1;
        if (sp.step_cap_factor > 0.0) {  // newton.hpp:612-620
            const float4 sc = s.scale[k];
            const double cap = sp.step_cap_factor * fmax(fmax((double)sc.x, (double)sc.y), (double)sc.z);
            const double nrm = sqrt(dp[0] * dp[0] + dp[1] * dp[1] + dp[2] * dp[2]);
            if (nrm > cap)
                for (int i = 0; i < 3; ++i) dp[i] *= cap / nrm;
        }
        if (out.delta)
            for (int i = 0; i < 3; ++i) out.delta[3 * k + i] = dp[i];
        if (out.accepted) out.accepted[k] = 1;
        nsq = dp[0] * dp[0] + dp[1] * dp[1] + dp[2] * dp[2];
        if (sp.commit) s.pos_sigma[k] = make_float4((float)(p.x + dp[0]), (float)(p.y + dp[1]), (float)(p.z + dp[2]), ps.w);
    }
    block_add(nsq, out.norm_sq);
}

__global__ void __launch_bounds__(256) solve_rotation_k(SceneDev s, CameraDev primary, SolveParams sp,
                                                        const double* __restrict__ acc, size_t stride,
                                                        SolveOutputs out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    double nsq = 0.0;
    if (k < s.n) {
        const float4 ps = s.pos_sigma[k];
        D3 r;
        primary_dir(primary, d3(ps.x, ps.y, ps.z), r, out.err);
        double theta = solve1(acc[stride + k], acc[k], sp);
        if (sp.theta_cap > 0.0) theta = fmin(fmax(theta, -sp.theta_cap), sp.theta_cap);
        if (out.delta) out.delta[k] = theta;
        if (out.accepted) out.accepted[k] = 1;
        nsq = theta * theta;
        // commit_rotation newton.hpp:822-826: q <- normalize(dq (x) q). A rotation too small to
        // move the FP32-stored quaternion (dq (x) q rounds back to q, e.g. theta ~ 1e-14 at a fixed
        // point) leaves it bit for bit: renormalising the FP32-rounded q alone would move it by an
        // ulp, which the reference's FP64 q (unit to 1e-16) never sees.
        if (sp.commit) {
            const double c = cos(theta), sn = sin(theta);
            const double a0 = c, a1 = sn * r.x, a2 = sn * r.y, a3 = sn * r.z;
            const float4 q = s.quat[k];
            const double b0 = q.x, b1 = q.y, b2 = q.z, b3 = q.w;
            double w = a0 * b0 - a1 * b1 - a2 * b2 - a3 * b3;
            double x = a0 * b1 + a1 * b0 + a2 * b3 - a3 * b2;
            double y = a0 * b2 - a1 * b3 + a2 * b0 + a3 * b1;
            double z = a0 * b3 + a1 * b2 - a2 * b1 + a3 * b0;
            const bool moved = (float)w != q.x || (float)x != q.y || (float)y != q.z || (float)z != q.w;
            const double nq = sqrt(w * w + x * x + y * y + z * z);
            if (!(nq > 0.0) || !isfinite(nq)) {
                atomicOr(out.err, 4);
            } else {
                w /= nq;
                x /= nq;
                y /= nq;
                z /= nq;
            }
            if (moved || !(nq > 0.0) || !isfinite(nq))
                s.quat[k] = make_float4((float)w, (float)x, (float)y, (float)z);
        }
    }
    block_add(nsq, out.norm_sq);
}

__global__ void __launch_bounds__(256) solve_scaling_k(SceneDev s, CameraDev primary, double lambda_lp,
                                                       const uint8_t* __restrict__ primary_flags, SolveParams sp,
                                                       const double* __restrict__ acc, size_t stride,
                                                       SolveOutputs out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    double nsq = 0.0;
    if (k < s.n) {
        const float4 ps = s.pos_sigma[k];
        const D3 p = {ps.x, ps.y, ps.z};
        const float4 sc = s.scale[k];
        const double sv[3] = {sc.x, sc.y, sc.z};
        // build_scaling_subspace (newton.hpp:152-184) on the primary entry.
        bool degenerate = true;
        double tp[3][2] = {};
        if (primary_flags[k] & kProjected) {
            Projected pr;
            project_kernel(primary, p, s.quat[k], sc, lambda_lp, pr);
            const Eig2 e = sym2_eigen(pr.s00, pr.s01, pr.s11);
            degenerate = (e.l1 - e.l0) <= sp.eigengap_rel * fabs(e.l1);
            double R[9];
            const float4 q = s.quat[k];
            quat_to_rot(q.x, q.y, q.z, q.w, R);
            double JW[6];
            for (int i = 0; i < 2; ++i)
                for (int j = 0; j < 3; ++j)
                    JW[3 * i + j] = pr.J[3 * i] * mrow(primary.view, 0, j) + pr.J[3 * i + 1] * mrow(primary.view, 1, j) +
                                    pr.J[3 * i + 2] * mrow(primary.view, 2, j);
            double nm[6];  // n = J W R (2x3)
            for (int i = 0; i < 2; ++i)
                for (int j = 0; j < 3; ++j) nm[3 * i + j] = JW[3 * i] * R[j] + JW[3 * i + 1] * R[3 + j] + JW[3 * i + 2] * R[6 + j];
            const double vx[2] = {e.v0x, e.v1x}, vy[2] = {e.v0y, e.v1y};
            double t[2][3];
            for (int i = 0; i < 2; ++i)
                for (int c = 0; c < 3; ++c) {
                    const double vn = vx[i] * nm[c] + vy[i] * nm[3 + c];
                    t[i][c] = 2.0 * sv[c] * vn * vn;
                }
            const double g00 = t[0][0] * t[0][0] + t[0][1] * t[0][1] + t[0][2] * t[0][2];
            const double g01 = t[0][0] * t[1][0] + t[0][1] * t[1][1] + t[0][2] * t[1][2];
            const double g11 = t[1][0] * t[1][0] + t[1][1] * t[1][1] + t[1][2] * t[1][2];
            const Eig2 ge = sym2_eigen(g00, g01, g11);
            const double cutoff = fmax(1e-30, 1e-12 * fabs(ge.l1));
            double gp[2][2] = {};
            const double gl[2] = {ge.l0, ge.l1};
            const double gvx[2] = {ge.v0x, ge.v1x}, gvy[2] = {ge.v0y, ge.v1y};
            for (int i = 0; i < 2; ++i)
                if (gl[i] > cutoff) {
                    const double inv = 1.0 / gl[i];
                    gp[0][0] += inv * gvx[i] * gvx[i];
                    gp[0][1] += inv * gvx[i] * gvy[i];
                    gp[1][0] += inv * gvy[i] * gvx[i];
                    gp[1][1] += inv * gvy[i] * gvy[i];
                }
            for (int c = 0; c < 3; ++c)
                for (int j = 0; j < 2; ++j) tp[c][j] = t[0][c] * gp[0][j] + t[1][c] * gp[1][j];
        }
        const double g0 = acc[k], g1 = acc[stride + k];
        const double h00 = acc[2 * stride + k], h01 = acc[3 * stride + k], h11 = acc[4 * stride + k];
        double dl0, dl1;
        if (degenerate) {  // newton.hpp:691-703
            const double d = solve1(h00 + 2.0 * h01 + h11, g0 + g1, sp);
            dl0 = dl1 = d;
        } else {
            solve2(h00, h01, h11, g0, g1, sp, dl0, dl1);
        }
        double ds[3];
        for (int c = 0; c < 3; ++c) ds[c] = tp[c][0] * dl0 + tp[c][1] * dl1;
        if (sp.scale_cap_factor > 1.0) {  // newton.hpp:717-726
            double shrink = 1.0;
            for (int c = 0; c < 3; ++c) {
                const double lo = sv[c] / sp.scale_cap_factor - sv[c];
                const double hi = sv[c] * sp.scale_cap_factor - sv[c];
                if (ds[c] > hi) shrink = fmin(shrink, hi / ds[c]);
                if (ds[c] < lo) shrink = fmin(shrink, lo / ds[c]);
            }
            for (int c = 0; c < 3; ++c) ds[c] *= shrink;
        }
        bool feasible = false;  // newton.hpp:727-738
        for (int i = 0; i <= sp.max_backtrack; ++i) {
            if (sv[0] + ds[0] > 0.0 && sv[1] + ds[1] > 0.0 && sv[2] + ds[2] > 0.0) {
                feasible = true;
                break;
            }
            for (int c = 0; c < 3; ++c) ds[c] *= 0.5;
        }
        if (!feasible) ds[0] = ds[1] = ds[2] = 0.0;
        if (out.delta)
            for (int c = 0; c < 3; ++c) out.delta[3 * k + c] = ds[c];
        if (out.accepted) out.accepted[k] = feasible ? 1 : 0;
        if (out.degenerate) out.degenerate[k] = degenerate ? 1 : 0;
        nsq = ds[0] * ds[0] + ds[1] * ds[1] + ds[2] * ds[2];
        if (sp.commit && feasible) {
            float nx = (float)(sv[0] + ds[0]), ny = (float)(sv[1] + ds[1]), nz = (float)(sv[2] + ds[2]);
            // FP32 storage must keep the reference's strict positivity invariant.
            if (!(nx > 0.f)) nx = sc.x;
            if (!(ny > 0.f)) ny = sc.y;
            if (!(nz > 0.f)) nz = sc.z;
            s.scale[k] = make_float4(nx, ny, nz, 0.f);
        }
    }
    block_add(nsq, out.norm_sq);
}

__global__ void __launch_bounds__(256) solve_opacity_k(SceneDev s, SolveParams sp, const double* __restrict__ acc,
                                                       size_t stride, int n_views, SolveOutputs out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    double nsq = 0.0;
    if (k < s.n) {
        const float4 ps = s.pos_sigma[k];
        const double sig = ps.w;
        double g = 0, h = 0;
        for (int v = 0; v < n_views; ++v) {
            g += acc[(static_cast<size_t>(v) * kAccOpColor + 0) * stride + k];
            h += acc[(static_cast<size_t>(v) * kAccOpColor + 1) * stride + k];
        }
        // OpacityBarrier, newton.hpp:187-195
        const double w = sp.barrier_weight;
        const double bh = w * (1.0 / (sig * sig) + 1.0 / ((1.0 - sig) * (1.0 - sig)));
        const double bg = -w * (1.0 / sig - 1.0 / (1.0 - sig));
        const double d = solve1(h + bh, g + bg, sp);
        float ns = (float)(sig + d);
        ns = fminf(fmaxf(ns, sp.sigma_lo), sp.sigma_hi);
        if (out.delta) out.delta[k] = ns;
        if (out.accepted) out.accepted[k] = 1;
        const double dd = (double)ns - sig;
        nsq = dd * dd;
        if (sp.commit) s.pos_sigma[k].w = ns;
    }
    block_add(nsq, out.norm_sq);
}

// Rotation (c, s, t = s / c) that zeroes a_pq (Numerical Recipes convention); identity
// when a_pq is zero or negligible against both diagonals.
// 1/sqrt(x) for normal x > 0: the MUFU seed refined by two Newton steps (same
// role as the reciprocal below: accurate, not correctly rounded).
__device__ __forceinline__ double rsqrt_pos(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double hx = 0.5 * x;
    y = y * fma(-hx * y, y, 1.5);
    y = y * fma(-hx * y, y, 1.5);
    return y;
}

__device__ __forceinline__ void jacobi_rot(double app, double aqq, double apq, double& c, double& s, double& t) {
    const double g = 100.0 * fabs(apq);
    if (fabs(app) + g == fabs(app) && fabs(aqq) + g == fabs(aqq)) {
        c = 1.0, s = 0.0, t = 0.0;
        return;
    }
    // t = sgn(theta) / (|theta| + sqrt(theta^2 + 1)) with theta = d / e, d = aqq - app,
    // e = 2 apq, multiplied through by |e|: one FP64 division instead of two.
    // The reciprocal is the MUFU seed refined by two Newton steps (~full FP64
    // precision; a Jacobi angle only needs to be accurate, not correctly rounded).
    const double d = aqq - app, e = 2 * apq;
    const double h2 = d * d + e * e;
    const double den = fabs(d) + h2 * rsqrt_pos(h2);
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(den));
    r = fma(r, fma(-den, r, 1.0), r);
    r = fma(r, fma(-den, r, 1.0), r);
    t = (d * e >= 0 ? 1.0 : -1.0) * fabs(e) * r;
    c = rsqrt_pos(t * t + 1), s = t * c;
}

// One round of the 4x4 parallel-order Jacobi: the disjoint rotations (P1, Q1) and
// (P2, Q2) are computed from the same matrix (neither changes the other's 2x2
// block) and applied together; symmetric updates only (diagonal blocks by the
// t-formulas, the cross block B' = R1^T B R2), two independent dependency chains.
template <int P1, int Q1, int P2, int Q2>
__device__ __forceinline__ void jacobi4_round(double (&a)[4][4], double (&v)[4][4]) {
    double c1, s1, t1, c2, s2, t2;
    jacobi_rot(a[P1][P1], a[Q1][Q1], a[P1][Q1], c1, s1, t1);
    jacobi_rot(a[P2][P2], a[Q2][Q2], a[P2][Q2], c2, s2, t2);
    const double a1 = a[P1][Q1], a2 = a[P2][Q2];
    a[P1][P1] -= t1 * a1;
    a[Q1][Q1] += t1 * a1;
    a[P1][Q1] = a[Q1][P1] = 0.0;
    a[P2][P2] -= t2 * a2;
    a[Q2][Q2] += t2 * a2;
    a[P2][Q2] = a[Q2][P2] = 0.0;
    const double x00 = a[P2][P1], x01 = a[P2][Q1], x10 = a[Q2][P1], x11 = a[Q2][Q1];
    const double y00 = c1 * x00 - s1 * x01, y01 = s1 * x00 + c1 * x01;  // columns (P1, Q1)
    const double y10 = c1 * x10 - s1 * x11, y11 = s1 * x10 + c1 * x11;
    a[P2][P1] = a[P1][P2] = c2 * y00 - s2 * y10;                         // rows (P2, Q2)
    a[Q2][P1] = a[P1][Q2] = s2 * y00 + c2 * y10;
    a[P2][Q1] = a[Q1][P2] = c2 * y01 - s2 * y11;
    a[Q2][Q1] = a[Q1][Q2] = s2 * y01 + c2 * y11;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const double vp1 = v[r][P1], vq1 = v[r][Q1], vp2 = v[r][P2], vq2 = v[r][Q2];
        v[r][P1] = c1 * vp1 - s1 * vq1;
        v[r][Q1] = s1 * vp1 + c1 * vq1;
        v[r][P2] = c2 * vp2 - s2 * vq2;
        v[r][Q2] = s2 * vp2 + c2 * vq2;
    }
}

// Cyclic Jacobi for a small symmetric MAXM x MAXM matrix, fully unrolled so
// the matrices stay in registers (zero rows/columns are inert). Eigenvalues
// end on the diagonal of `a`, eigenvectors in the columns of `v`.
template <int MAXM>
__device__ inline void jacobi_eig(double (&a)[MAXM][MAXM], double (&v)[MAXM][MAXM]) {
#pragma unroll
    for (int i = 0; i < MAXM; ++i)
#pragma unroll
        for (int j = 0; j < MAXM; ++j) v[i][j] = (i == j) ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 24; ++sweep) {
        double off = 0, diag = 0;
#pragma unroll
        for (int i = 0; i < MAXM; ++i) {
            diag += a[i][i] * a[i][i];
#pragma unroll
            for (int j = i + 1; j < MAXM; ++j) off += a[i][j] * a[i][j];
        }
        // Converged when the off-diagonal mass is ~1e-14 of the diagonal: eigenvalues are then
        // within ~1e-14 ||A|| (Weyl), far below the FP32 accumulation error of the inputs.
        if (off == 0.0 || off <= kJacobiTol * diag) break;
        if constexpr (MAXM == 4) {  // parallel ordering: 3 rounds of 2 disjoint rotations
            jacobi4_round<0, 1, 2, 3>(a, v);
            jacobi4_round<0, 2, 1, 3>(a, v);
            jacobi4_round<0, 3, 1, 2>(a, v);
        } else {
#pragma unroll
            for (int p = 0; p < MAXM; ++p)
#pragma unroll
                for (int q = p + 1; q < MAXM; ++q) {
                    // Negligible off-diagonal (cannot change either diagonal in FP64): zero it
                    // and skip the rotation (the classical cyclic-Jacobi threshold test).
                    const double g = 100.0 * fabs(a[p][q]);
                    if (fabs(a[p][p]) + g == fabs(a[p][p]) && fabs(a[q][q]) + g == fabs(a[q][q])) {
                        a[p][q] = a[q][p] = 0.0;
                        continue;
                    }
                    const double theta = (a[q][q] - a[p][p]) / (2 * a[p][q]);
                    const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1));
                    const double c = rsqrt(t * t + 1), sn = t * c;
#pragma unroll
                    for (int kk = 0; kk < MAXM; ++kk) {
                        const double akp = a[kk][p], akq = a[kk][q];
                        a[kk][p] = c * akp - sn * akq;
                        a[kk][q] = sn * akp + c * akq;
                    }
#pragma unroll
                    for (int kk = 0; kk < MAXM; ++kk) {
                        const double apk = a[p][kk], aqk = a[q][kk];
                        a[p][kk] = c * apk - sn * aqk;
                        a[q][kk] = sn * apk + c * aqk;
                    }
#pragma unroll
                    for (int kk = 0; kk < MAXM; ++kk) {
                        const double vkp = v[kk][p], vkq = v[kk][q];
                        v[kk][p] = c * vkp - sn * vkq;
                        v[kk][q] = sn * vkp + c * vkq;
                    }
                }
        }
    }
}

// solve_color (newton.hpp:783-811) from per-view compact accumulators
// (color_terms, newton.hpp:538-574): grad_ch = sum_v g_v phi_v = Phi g,
// hess_ch = sum_v h_v phi_v phi_v^T = Phi D Phi^T. Exact psd_safeguard
// spectrum repair through the thin SVD of Phi, carried out entirely in the
// m-dimensional view space: with G = Phi^T Phi = E L E^T, the non-trivial
// eigenpairs of H are those of K = L^1/2 E^T D E L^1/2 = W Theta W^T, the
// eigenvectors are y_i = Phi c_i with c_i = E L^-1/2 W_i, and the solution is
// delta = Phi beta. Directions of range(Phi) whose Gram eigenvalue vanishes
// (near-collinear view directions) carry eigenvalue ~0 and are floored to mu;
// the null space of Phi^T carries no gradient. Nothing n-dimensional is
// stored: phi_v is re-evaluated when beta is committed.
// Colour solve, stage 1 (per Gaussian): the Gram matrix G = Phi^T Phi of the
// views' SH bases and its eigen-decomposition G = E L E^T (stored: E, diag L),
// shared by the three channels of stage 2.
// Gram matrix of the visible views' SH bases (phi_a . phi_b; absent views are zero) and its
// eigen-decomposition G = E diag(L) E^T (eigenvalues on the diagonal of L).
template <int MV>
__device__ __forceinline__ void color_gram_matrix(const SceneDev& s, const ColorViews& cv, int k, double (&L)[MV][MV]) {
    const float4 ps = s.pos_sigma[k];
    const D3 p = {ps.x, ps.y, ps.z};
    const int nv = cv.n_views;
    D3 dir[MV];
    uint8_t fl[MV];
#pragma unroll
    for (int v = 0; v < MV; ++v) {
        fl[v] = 0;
        dir[v] = d3(0, 0, 1);
        if (v < nv) {
            fl[v] = cv.flags[v][k];
            double nr;
            if (!view_direction(cv.cam[v], p, dir[v], nr)) dir[v] = d3(0, 0, 1);
        }
    }
#pragma unroll
    for (int a = 0; a < MV; ++a) {
        double pa[16];
        sh_basis(dir[a], s.sh_degree, pa);
#pragma unroll
        for (int b = 0; b <= a; ++b) {
            double pb[16];
            sh_basis(dir[b], s.sh_degree, pb);
            double t = 0;
#pragma unroll
            for (int i = 0; i < 16; ++i) t += pa[i] * pb[i];
            const bool on = (fl[a] & kProjected) && (fl[b] & kProjected);
            L[a][b] = on ? t : 0.0;
            L[b][a] = L[a][b];
        }
    }
}

// The same Gram matrix from the addition theorem of the orthonormal real SH basis
// (sum_m Y_lm(a) Y_lm(b) = (2l+1)/(4 pi) P_l(a.b)): G_ab = sum_{l <= degree}
// (2l+1)/(4 pi) P_l(d_a . d_b), equal to the explicit dot products up to rounding, from
// the view directions alone (also returned, for the commit).
template <int MV>
__device__ __forceinline__ void color_gram_addition(const SceneDev& s, const ColorViews& cv, int k,
                                                    const uint8_t (&fl)[MV], double (&G)[MV][MV], D3 (&dir)[MV]) {
    const float4 ps = s.pos_sigma[k];
    const D3 p = {ps.x, ps.y, ps.z};
    const int nv = cv.n_views, deg = s.sh_degree;
    constexpr double k4pi = 0.07957747154594767;  // 1 / (4 pi)
#pragma unroll
    for (int v = 0; v < MV; ++v) {
        dir[v] = d3(0, 0, 1);
        double nr;
        if (v < nv && !view_direction(cv.cam[v], p, dir[v], nr)) dir[v] = d3(0, 0, 1);
    }
#pragma unroll
    for (int a = 0; a < MV; ++a)
#pragma unroll
        for (int b = 0; b <= a; ++b) {
            const double t = dir[a].x * dir[b].x + dir[a].y * dir[b].y + dir[a].z * dir[b].z;
            double g = 1.0;                                  // l = 0
            if (deg >= 1) g += 3.0 * t;                      // l = 1
            if (deg >= 2) g += 5.0 * (1.5 * t * t - 0.5);    // l = 2
            if (deg >= 3) g += 7.0 * (2.5 * t * t - 1.5) * t;  // l = 3
            const bool on = (fl[a] & kProjected) && (fl[b] & kProjected);
            G[a][b] = G[b][a] = on ? g * k4pi : 0.0;
        }
}

template <int MV>
__device__ __forceinline__ void color_gram(const SceneDev& s, const ColorViews& cv, int k, double (&L)[MV][MV],
                                           double (&E)[MV][MV]) {
    color_gram_matrix<MV>(s, cv, k, L);
    jacobi_eig<MV>(L, E);
}

template <int MV>
__global__ void __launch_bounds__(128) solve_color_gram_k(SceneDev s, ColorViews cv, double* __restrict__ eig,
                                                          size_t stride) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < s.n) {
        double L[MV][MV], E[MV][MV];
        color_gram<MV>(s, cv, k, L, E);
#pragma unroll
        for (int a = 0; a < MV; ++a) {
            eig[static_cast<size_t>(MV * MV + a) * stride + k] = L[a][a];
#pragma unroll
            for (int b = 0; b < MV; ++b) eig[static_cast<size_t>(MV * a + b) * stride + k] = E[a][b];
        }
    }
}

// This channel's per-view compact accumulators (colour_terms): views that are projected
// and not colour-clamped in the channel; false when no view contributes.
template <int MV>
__device__ __forceinline__ bool color_channel_terms(const double* __restrict__ acc, size_t stride, int k, int nv,
                                                    const uint8_t (&fl)[MV], int ch, double (&gv)[MV],
                                                    double (&hv)[MV]) {
    bool any = false;
#pragma unroll
    for (int v = 0; v < MV; ++v) {
        gv[v] = 0.0;
        hv[v] = 0.0;
        if (v < nv && (fl[v] & kProjected) && !(fl[v] & (kClamp0 << ch))) {
            const double* a = acc + static_cast<size_t>(v) * kAccOpColor * stride;
            gv[v] = a[(2 + ch) * stride + k];
            hv[v] = a[(5 + ch) * stride + k];
            any = true;
        }
    }
    return any;
}

// The exact psd_safeguard solve of one channel in view space from the Gram
// eigen-decomposition G = E diag(L) E^T (n > 1): beta and |delta|^2 = beta^T G beta.
template <int MV>
__device__ __forceinline__ void color_channel_eigen(int n, const double (&L)[MV][MV], const double (&E)[MV][MV],
                                                    const double (&gv)[MV], const double (&hv)[MV],
                                                    const SolveParams& sp, double (&beta)[MV], double& nrm2) {
    double lmax = 0;
#pragma unroll
    for (int a = 0; a < MV; ++a) lmax = fmax(lmax, L[a][a]);
    bool kept[MV];
    double isq[MV], sq[MV];  // L^-1/2 on kept directions
    int r = 0;
#pragma unroll
    for (int a = 0; a < MV; ++a) {
        kept[a] = L[a][a] > 1e-13 * lmax && L[a][a] > 0.0;
        isq[a] = kept[a] ? rsqrt_pos(L[a][a]) : 0.0;
        sq[a] = L[a][a] * isq[a];  // L^1/2 on kept directions, 0 elsewhere
        r += kept[a] ? 1 : 0;
    }
#pragma unroll
    for (int a = 0; a < MV; ++a) beta[a] = 0.0;
    nrm2 = 0;
    // K = L^1/2 E^T D E L^1/2 on the kept directions.
    double K[MV][MV], W[MV][MV];
#pragma unroll
    for (int i = 0; i < MV; ++i)
#pragma unroll
        for (int j = i; j < MV; ++j) {
            double t = 0;
#pragma unroll
            for (int v = 0; v < MV; ++v) t += E[v][i] * hv[v] * E[v][j];
            K[i][j] = K[j][i] = t * sq[i] * sq[j];  // 0 unless both directions are kept
        }
    jacobi_eig<MV>(K, W);
    // Eigenvectors y_e = Phi c_e with c_e = E L^-1/2 W_e; those living in the
    // dropped subspace have c_e = 0.
    double c[MV][MV];
    bool live[MV];
    double lam_abs_max = 0, lam_min = 1e300;
#pragma unroll
    for (int e = 0; e < MV; ++e) {
        double wk = 0;
#pragma unroll
        for (int j = 0; j < MV; ++j) wk += kept[j] ? W[j][e] * W[j][e] : 0.0;
        live[e] = wk > 0.5;
#pragma unroll
        for (int v = 0; v < MV; ++v) {
            double t = 0;
#pragma unroll
            for (int j = 0; j < MV; ++j) t += E[v][j] * isq[j] * W[j][e];
            c[e][v] = live[e] ? t : 0.0;
        }
        if (live[e]) {
            lam_abs_max = fmax(lam_abs_max, fabs(K[e][e]));
            lam_min = fmin(lam_min, K[e][e]);
        }
    }
    if (r < n) lam_min = fmin(lam_min, 0.0);  // zero eigenvalues outside range(Phi)
    const double mu = fmax(sp.mu_min, sp.eig_floor_rel * lam_abs_max);
    const bool keep_h = lam_min >= mu;  // newton.hpp:231: PD input solved unmodified
    double Gg[MV], Etg[MV];
#pragma unroll
    for (int j = 0; j < MV; ++j) {
        double t = 0;
#pragma unroll
        for (int v = 0; v < MV; ++v) t += E[v][j] * gv[v];
        Etg[j] = L[j][j] * t;
    }
#pragma unroll
    for (int a = 0; a < MV; ++a) {
        double t = 0;
#pragma unroll
        for (int j = 0; j < MV; ++j) t += E[a][j] * Etg[j];
        Gg[a] = t;
    }
#pragma unroll
    for (int e = 0; e < MV; ++e) {
        if (!live[e]) continue;
        double yg = 0;
#pragma unroll
        for (int v = 0; v < MV; ++v) yg += c[e][v] * Gg[v];
        const double lam = K[e][e];
        const double l = keep_h ? lam : fmax(fabs(lam), mu);
#pragma unroll
        for (int v = 0; v < MV; ++v) beta[v] -= (yg / l) * c[e][v];
    }
    if (!keep_h) {
        // range(Phi) directions with a vanishing Gram eigenvalue: eigenvalue ~0 -> mu.
#pragma unroll
        for (int a = 0; a < MV; ++a) {
            if (kept[a] || !(L[a][a] > 0.0)) continue;
            double eg = 0;
#pragma unroll
            for (int v = 0; v < MV; ++v) eg += E[v][a] * gv[v];
#pragma unroll
            for (int v = 0; v < MV; ++v) beta[v] -= E[v][a] * eg / mu;
        }
    }
#pragma unroll
    for (int j = 0; j < MV; ++j) {
        double t = 0;
#pragma unroll
        for (int a = 0; a < MV; ++a) t += E[a][j] * beta[a];
        nrm2 += L[j][j] * t * t;
    }
}

// In-place lower Cholesky factor of a symmetric MV x MV matrix; false unless every pivot
// is positive (the matrix is numerically positive definite).
template <int MV>
__device__ __forceinline__ bool cholesky(double (&a)[MV][MV]) {
#pragma unroll
    for (int j = 0; j < MV; ++j) {
        double d = a[j][j];
#pragma unroll
        for (int q = 0; q < j; ++q) d -= a[j][q] * a[j][q];
        if (!(d > 0.0)) return false;
        const double inv = rsqrt_pos(d);
        a[j][j] = d * inv;
#pragma unroll
        for (int i = j + 1; i < MV; ++i) {
            double t = a[i][j];
#pragma unroll
            for (int q = 0; q < j; ++q) t -= a[i][q] * a[j][q];
            a[i][j] = t * inv;
        }
    }
    return true;
}

// Fast path of color_channel_eigen when the safeguard provably leaves the spectrum
// alone. On the views P that carry terms (the rest have zero Gram rows and beta_v = 0):
// if every Gram eigenvalue is kept (G_P - 1e-13 |G_P|_F I is PD, |G_P|_F >= lambda_max)
// and every eigenvalue of K ~ M = D^1/2 G_P D^1/2 (D = diag h_v > 0) is at least
// mu = max(mu_min, rel * lambda_max) (M - max(mu_min, rel |M|_F) I is PD), the repaired
// system is the unmodified one and the solution collapses to
// beta_P = -G_P^-1 (g_v / h_v): two Cholesky tests and one Cholesky solve, no Jacobi.
// Otherwise false (the caller runs the eigen path).
template <int MV>
__device__ __forceinline__ bool color_channel_fast(const double (&G)[MV][MV], const double (&gv)[MV],
                                                   const double (&hv)[MV], const bool (&in)[MV],
                                                   const SolveParams& sp, double (&beta)[MV], double& nrm2) {
    double gf = 0, mf = 0;
#pragma unroll
    for (int a = 0; a < MV; ++a) {
        if (in[a] && !(hv[a] > 0.0)) return false;
#pragma unroll
        for (int b = 0; b < MV; ++b)
            if (in[a] && in[b]) {
                gf += G[a][b] * G[a][b];
                mf += (hv[a] * G[a][b] * hv[b]) * G[a][b];  // M_ab^2 = h_a h_b G_ab^2
            }
    }
    gf = sqrt(gf);
    const double mu_hi = fmax(sp.mu_min, sp.eig_floor_rel * sqrt(mf));
    double A[MV][MV], C[MV][MV], F[MV][MV];
    double sh[MV];
#pragma unroll
    for (int a = 0; a < MV; ++a) sh[a] = in[a] ? sqrt(hv[a]) : 1.0;
#pragma unroll
    for (int a = 0; a < MV; ++a)
#pragma unroll
        for (int b = 0; b < MV; ++b) {
            const bool on = in[a] && in[b];
            const double off = a == b ? 1.0 : 0.0;  // identity outside P
            A[a][b] = on ? G[a][b] - (a == b ? 1e-13 * gf : 0.0) : off * (gf + 1.0);
            C[a][b] = on ? sh[a] * G[a][b] * sh[b] - (a == b ? mu_hi : 0.0) : off * (mu_hi + 1.0);
            F[a][b] = on ? G[a][b] : off;
        }
    if (!cholesky<MV>(A) || !cholesky<MV>(C) || !cholesky<MV>(F)) return false;
    // F F^T beta = -(g / h) on P (zero right-hand side outside P: beta_v = 0 there)
    double y[MV];
#pragma unroll
    for (int i = 0; i < MV; ++i) {
        double t = in[i] ? -gv[i] / hv[i] : 0.0;
#pragma unroll
        for (int q = 0; q < i; ++q) t -= F[i][q] * y[q];
        y[i] = t / F[i][i];
    }
#pragma unroll
    for (int i = MV - 1; i >= 0; --i) {
        double t = y[i];
#pragma unroll
        for (int q = i + 1; q < MV; ++q) t -= F[q][i] * beta[q];
        beta[i] = t / F[i][i];
    }
    // |delta|^2 = beta^T G beta = |F^T beta|^2
    nrm2 = 0;
#pragma unroll
    for (int j = 0; j < MV; ++j) {
        double t = 0;
#pragma unroll
        for (int i = j; i < MV; ++i) t += F[i][j] * beta[i];
        nrm2 += t * t;
    }
    return true;
}

// Colour cap (newton.hpp:801-804), then delta_ch = sum_v beta_v phi_v (SH0: beta_0);
// written to out.delta and / or committed.
template <int MV>
__device__ __forceinline__ void color_channel_commit(const SceneDev& s, const ColorViews& cv, const SolveParams& sp,
                                                     const SolveOutputs& out, int k, int ch, bool any,
                                                     const double (&beta)[MV], double nrm2, double& nsq,
                                                     const D3* dirs = nullptr) {
    const int n = s.n_coeffs, nv = cv.n_views;
    double beta_all[MV];
    double scale = 1.0;
    if (any && sp.color_cap > 0.0 && sqrt(nrm2) > sp.color_cap) scale = sp.color_cap / sqrt(nrm2);
    if (any) nsq += nrm2 * scale * scale;
#pragma unroll
    for (int a = 0; a < MV; ++a) beta_all[a] = any ? beta[a] * scale : 0.0;
    double delta[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) delta[i] = 0.0;
    if (n == 1) {
        delta[0] = beta_all[0];
    } else {
        const float4 ps = s.pos_sigma[k];
        const D3 p = {ps.x, ps.y, ps.z};
#pragma unroll
        for (int v = 0; v < MV; ++v) {
            D3 dir = d3(0, 0, 1);
            if (dirs) {
                dir = dirs[v];
            } else {
                double nr;
                if (v < nv && !view_direction(cv.cam[v], p, dir, nr)) dir = d3(0, 0, 1);
            }
            double ph[16];
            sh_basis(dir, s.sh_degree, ph);
#pragma unroll
            for (int i = 0; i < 16; ++i) delta[i] += beta_all[v] * ph[i];
        }
    }
    if (out.delta)
#pragma unroll
        for (int i = 0; i < 16; ++i) out.delta[48 * static_cast<size_t>(k) + 16 * ch + i] = i < n ? delta[i] : 0.0;
    if (sp.commit) {  // all loads of the channel first, then the stores (no load-store serialisation)
        float cur[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) cur[i] = i < n ? s.sh[(static_cast<size_t>(16 * ch + i)) * s.n + k] : 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i)
            if (i < n) s.sh[(static_cast<size_t>(16 * ch + i)) * s.n + k] = (float)((double)cur[i] + delta[i]);
    }
    if (out.accepted && ch == 0) out.accepted[k] = 1;
}

// Scalar system (psd_safeguard n = 1, SH0): phi = kSH0 for every view.
template <int MV>
__device__ __forceinline__ void color_channel_sh0(const double (&gv)[MV], const double (&hv)[MV],
                                                  const SolveParams& sp, double (&beta)[MV], double& nrm2) {
    double g = 0, h = 0;
#pragma unroll
    for (int a = 0; a < MV; ++a) {
        g += gv[a] * kSH0;
        h += hv[a] * kSH0 * kSH0;
        beta[a] = 0.0;
    }
    const double d = solve1(h, g, sp);  // coefficient delta
    beta[0] = d;
    nrm2 = d * d;
}

// Colour solve, stage 2 (one thread per Gaussian and channel, blockIdx.y = channel), from
// stage 1's Gram eigen-decomposition in the eig scratch.
// (One thread per Gaussian with stage 1 in registers and the channels in turn, no eigen
// scratch in HBM, measured slower: C4 colour 7.3 -> 8.9 ms.)
template <int MV>
__global__ void __launch_bounds__(128, MV == 4 ? NGS_COLOR4_MINB : 2)
    solve_color_k(SceneDev s, ColorViews cv, SolveParams sp, const double* __restrict__ acc, size_t stride,
                  const double* __restrict__ eig, SolveOutputs out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    double nsq = 0.0;
    if (k < s.n) {
        const int n = s.n_coeffs;
        const int nv = cv.n_views;
        const int ch = blockIdx.y;
        uint8_t fl[MV];
#pragma unroll
        for (int v = 0; v < MV; ++v) fl[v] = v < nv ? cv.flags[v][k] : 0;
        double gv[MV], hv[MV], beta[MV], nrm2 = 0.0;
        const bool any = color_channel_terms<MV>(acc, stride, k, nv, fl, ch, gv, hv);
        if (any) {
            if (n == 1) {
                color_channel_sh0<MV>(gv, hv, sp, beta, nrm2);
            } else {
                // Stage 1's G = E L E^T. G itself is not re-formed: G g = E L E^T g and
                // beta^T G beta = sum_j L_j (E^T beta)_j^2.
                double L[MV][MV], E[MV][MV];
#pragma unroll
                for (int a = 0; a < MV; ++a)
#pragma unroll
                    for (int b = 0; b < MV; ++b) {
                        L[a][b] = a == b ? eig[static_cast<size_t>(MV * MV + a) * stride + k] : 0.0;
                        E[a][b] = eig[static_cast<size_t>(MV * a + b) * stride + k];
                    }
                color_channel_eigen<MV>(n, L, E, gv, hv, sp, beta, nrm2);
            }
        }
        color_channel_commit<MV>(s, cv, sp, out, k, ch, any, beta, nrm2, nsq);
    }
    block_add(nsq, out.norm_sq);
}

// Colour solve in ONE launch (one thread per Gaussian and channel): the Gram matrix of
// the views' SH bases is formed in registers; the fast path (color_channel_fast) solves
// without any eigen-decomposition, and only the channels that fail its tests
// eigen-decompose G themselves and run the exact repair. No eig scratch in HBM.
template <int MV>
__global__ void __launch_bounds__(128, MV == 4 ? NGS_COLORF4_MINB : 2)
    solve_color_fused_k(SceneDev s, ColorViews cv, SolveParams sp, const double* __restrict__ acc, size_t stride,
                        SolveOutputs out, unsigned long long* __restrict__ fast_count) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    double nsq = 0.0;
    bool fast = false;
    if (k < s.n) {
        const int n = s.n_coeffs;
        const int nv = cv.n_views;
        const int ch = blockIdx.y;
        uint8_t fl[MV];
#pragma unroll
        for (int v = 0; v < MV; ++v) fl[v] = v < nv ? cv.flags[v][k] : 0;
        double gv[MV], hv[MV], beta[MV], nrm2 = 0.0;
        D3 dir[MV];
        const bool any = color_channel_terms<MV>(acc, stride, k, nv, fl, ch, gv, hv);
        if (any) {
            if (n == 1) {
                color_channel_sh0<MV>(gv, hv, sp, beta, nrm2);
            } else {
                double L[MV][MV], E[MV][MV];
                color_gram_addition<MV>(s, cv, k, fl, L, dir);
                // P = the projected views (the nonzero Gram rows); a projected view whose
                // colour is clamped in this channel carries h_v = 0 (a zero eigenvalue the
                // repair floors): eigen path.
                bool in[MV], clamped = false;
#pragma unroll
                for (int v = 0; v < MV; ++v) {
                    in[v] = v < nv && (fl[v] & kProjected);
                    clamped |= in[v] && (fl[v] & (kClamp0 << ch));
                }
                fast = !clamped && color_channel_fast<MV>(L, gv, hv, in, sp, beta, nrm2);
                if (!fast) {  // the explicit Gram (as the two-stage kernels) and the exact repair
                    color_gram_matrix<MV>(s, cv, k, L);
                    jacobi_eig<MV>(L, E);
                    color_channel_eigen<MV>(n, L, E, gv, hv, sp, beta, nrm2);
                }
            }
        }
        color_channel_commit<MV>(s, cv, sp, out, k, ch, any, beta, nrm2, nsq, any && n > 1 ? dir : nullptr);
    }
    if (fast_count) {
        const unsigned b = __ballot_sync(0xffffffffu, fast);
        if ((threadIdx.x & 31) == 0 && b) atomicAdd(fast_count, static_cast<unsigned long long>(__popc(b)));
    }
    block_add(nsq, out.norm_sq);
}

// first_order_step (trainer.hpp:419-509) for one Gaussian per thread.
__global__ void __launch_bounds__(128) first_order_k(SceneDev s, CameraDev cam, const uint8_t* __restrict__ flags,
                                                     const float* __restrict__ pcst, const float* __restrict__ rcst,
                                                     const double* __restrict__ acc, size_t stride, FirstOrderParams p,
                                                     double* __restrict__ am, double* __restrict__ av,
                                                     unsigned long long* __restrict__ norms, int* err) {
    using L = PosLayout<3>;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    double nsq[5] = {0, 0, 0, 0, 0};
    if (k < s.n) {
        const float4 ps = s.pos_sigma[k];
        const D3 p3 = {ps.x, ps.y, ps.z};
        const uint8_t fl = flags[k];
        // Gradients (zero for kernels without an entry in this view, newton.hpp:271-275 etc.).
        double gp[3] = {0, 0, 0}, gth = 0, gs[3] = {0, 0, 0}, gsig = 0, gc[3] = {0, 0, 0};
        D3 axis;
        double nr;
        if (!view_direction(cam, p3, axis, nr)) {
            atomicOr(err, 2);
            axis = d3(0, 0, 1);
        }
        if (fl & kProjected) {
            double A[kAccGrad];
#pragma unroll
            for (int c = 0; c < kAccGrad; ++c) A[c] = acc[c * stride + k];
            const float* pc = pcst + static_cast<size_t>(k) * L::N;
            auto sym = [&](double m00, double m01, double m11) { return A[2] * m00 + 2.0 * A[3] * m01 + A[4] * m11; };
#pragma unroll
            for (int c = 0; c < 3; ++c) {  // position_terms grad via dG/dpi, dG/dSigma, dc~/dp
                gp[c] = pc[L::JS + 2 * c] * A[0] + pc[L::JS + 2 * c + 1] * A[1] +
                        sym(pc[L::JS + 6 + 3 * c], pc[L::JS + 6 + 3 * c + 1], pc[L::JS + 6 + 3 * c + 2]);
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) gp[c] += pc[L::JC + 3 * ch + c] * A[5 + ch];
            }
            const float* rc = rcst + static_cast<size_t>(k) * kRotConsts;
            gth = sym(rc[0], rc[1], rc[2]);  // rotation_terms grad: dG/dSigma : s1
            // scaling_gradient_s (newton.hpp:472-503): dSigma/ds_c = 2 s_c n_c n_c^T, n = J W R.
            const D3 t = to_camera_space(cam, p3);
            CamProj cp;
            project_camera_space<false, false>(cam, t, cp);
            double jw[6];
            for (int i = 0; i < 2; ++i)
                for (int j = 0; j < 3; ++j)
                    jw[3 * i + j] = cp.J[3 * i] * mrow(cam.view, 0, j) + cp.J[3 * i + 1] * mrow(cam.view, 1, j) +
                                    cp.J[3 * i + 2] * mrow(cam.view, 2, j);
            const float4 q = s.quat[k];
            double R[9];
            quat_to_rot(q.x, q.y, q.z, q.w, R);
            const float4 sc = s.scale[k];
            const double sv[3] = {sc.x, sc.y, sc.z};
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double n0 = jw[0] * R[c] + jw[1] * R[3 + c] + jw[2] * R[6 + c];
                const double n1 = jw[3] * R[c] + jw[4] * R[3 + c] + jw[5] * R[6 + c];
                gs[c] = 2.0 * sv[c] * sym(n0 * n0, n0 * n1, n1 * n1);
            }
            gsig = A[8];  // opacity_data_terms grad
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) gc[ch] = (fl & (kClamp0 << ch)) ? 0.0 : A[5 + ch];  // color_terms g_acc
        }
        // Adam moments slot-major ([56][stride]) so a warp's accesses coalesce.
        const double bc1 = 1.0 - pow(p.beta1, (double)p.t), bc2 = 1.0 - pow(p.beta2, (double)p.t);
        auto upd = [&](int slot, double g, double lr) {
            if (!p.adam) return -lr * g;  // gd_update
            const size_t i = static_cast<size_t>(slot) * stride + k;
            const double m = p.beta1 * am[i] + (1.0 - p.beta1) * g;
            const double v = p.beta2 * av[i] + (1.0 - p.beta2) * g * g;
            am[i] = m;
            av[i] = v;
            return -lr * (m / bc1) / (sqrt(v / bc2) + p.eps);
        };
        double dp[3], ds[3];
        for (int c = 0; c < 3; ++c) dp[c] = upd(c, gp[c], p.lr[NGS_POSITION]);
        for (int c = 0; c < 3; ++c) ds[c] = upd(4 + c, gs[c], p.lr[NGS_SCALING]);
        const double dth = upd(3, gth, p.lr[NGS_ROTATION]);
        const double dsg = upd(7, gsig, p.lr[NGS_OPACITY]);
        // Commit (trainer.hpp:480-505).
        s.pos_sigma[k] = make_float4((float)(p3.x + dp[0]), (float)(p3.y + dp[1]), (float)(p3.z + dp[2]), ps.w);
        nsq[NGS_POSITION] = dp[0] * dp[0] + dp[1] * dp[1] + dp[2] * dp[2];
        {
            const double c = cos(dth), sn = sin(dth);
            const double a0 = c, a1 = sn * axis.x, a2 = sn * axis.y, a3 = sn * axis.z;
            const float4 qq = s.quat[k];
            const double b0 = qq.x, b1 = qq.y, b2 = qq.z, b3 = qq.w;
            double w = a0 * b0 - a1 * b1 - a2 * b2 - a3 * b3;
            double x = a0 * b1 + a1 * b0 + a2 * b3 - a3 * b2;
            double y = a0 * b2 - a1 * b3 + a2 * b0 + a3 * b1;
            double z = a0 * b3 + a1 * b2 - a2 * b1 + a3 * b0;
            const bool moved = (float)w != qq.x || (float)x != qq.y || (float)y != qq.z || (float)z != qq.w;
            const double nq = sqrt(w * w + x * x + y * y + z * z);
            if (!(nq > 0.0) || !isfinite(nq)) {
                atomicOr(err, 4);
            } else {
                w /= nq;
                x /= nq;
                y /= nq;
                z /= nq;
            }
            if (moved || !(nq > 0.0) || !isfinite(nq))  // see solve_rotation_k
                s.quat[k] = make_float4((float)w, (float)x, (float)y, (float)z);
        }
        nsq[NGS_ROTATION] = dth * dth;
        {
            const float4 sc = s.scale[k];
            s.scale[k] = make_float4((float)fmax(1e-8, (double)sc.x + ds[0]), (float)fmax(1e-8, (double)sc.y + ds[1]),
                                     (float)fmax(1e-8, (double)sc.z + ds[2]), 0.f);
        }
        nsq[NGS_SCALING] = ds[0] * ds[0] + ds[1] * ds[1] + ds[2] * ds[2];
        {
            float ns = (float)((double)ps.w + dsg);
            ns = fminf(fmaxf(ns, p.sigma_lo), p.sigma_hi);
            s.pos_sigma[k].w = ns;
            const double applied = (double)ns - (double)ps.w;
            nsq[NGS_OPACITY] = applied * applied;
        }
        if (s.n_coeffs > 0) {
            double basis[16];
            sh_basis(axis, s.sh_degree, basis);
#pragma unroll
            for (int ch = 0; ch < 3; ++ch)
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    if (i >= s.n_coeffs) continue;
                    const double d = upd(8 + 16 * ch + i, gc[ch] * basis[i], p.lr[NGS_COLOR]);
                    float* cc = s.sh + static_cast<size_t>(16 * ch + i) * s.n + k;
                    *cc = (float)((double)*cc + d);
                    nsq[NGS_COLOR] += d * d;
                }
        }
    }
#pragma unroll
    for (int a = 0; a < 5; ++a) block_add(nsq[a], norms + a * kExactWords);
}

}  // namespace

void launch_first_order(const SceneDev& scene, const CameraDev& cam, const uint8_t* flags, const float* pos_consts,
                        const float* rot_consts, const double* acc, size_t stride, const FirstOrderParams& p,
                        double* adam_m, double* adam_v, unsigned long long* norms, int* err, cudaStream_t s) {
    const int n = scene.n;
    if (n == 0) return;
    StageScope st(NGS_STAGE_SOLVE, s);
    first_order_k<<<blocks_for(n, 128), 128, 0, s>>>(scene, cam, flags, pos_consts, rot_consts, acc, stride, p, adam_m,
                                                      adam_v, norms, err);
    CUDA_LAUNCH_CHECK();
}

void launch_solve(int attr, const SceneDev& scene, const CameraDev& primary, double lambda_lp,
                  const uint8_t* primary_flags, const ColorViews& cv, const SolveParams& sp, const double* acc,
                  size_t stride, const SolveOutputs& out, cudaStream_t s) {
    const int n = scene.n;
    if (n == 0) return;
    StageScope st(NGS_STAGE_SOLVE, s, attr == NGS_COLOR && scene.n_coeffs > 1 && !cv.fused ? 2 : 1);
    switch (attr) {
        case NGS_POSITION:
            solve_position_k<<<blocks_for(n), 256, 0, s>>>(scene, primary, sp, acc, stride, out);
            break;
        case NGS_ROTATION:
            solve_rotation_k<<<blocks_for(n), 256, 0, s>>>(scene, primary, sp, acc, stride, out);
            break;
        case NGS_SCALING:
            solve_scaling_k<<<blocks_for(n), 256, 0, s>>>(scene, primary, lambda_lp, primary_flags, sp, acc, stride,
                                                          out);
            break;
        case NGS_OPACITY:
            solve_opacity_k<<<blocks_for(n), 256, 0, s>>>(scene, sp, acc, stride, cv.n_views, out);
            break;
        case NGS_COLOR: {
            // fused: one launch, Gram in registers, fast path / in-thread eigen repair;
            // otherwise stage 1 (Gram eigen-decomposition, only with higher SH bands) +
            // stage 2 per channel
            auto run = [&](auto gram_kernel, auto ch_kernel, auto fused_kernel) {
                if (cv.fused) {
                    fused_kernel<<<dim3(blocks_for(n, 128), 3), 128, 0, s>>>(scene, cv, sp, acc, stride, out,
                                                                              cv.fast_count);
                    return;
                }
                if (scene.n_coeffs > 1) gram_kernel<<<blocks_for(n, 128), 128, 0, s>>>(scene, cv, cv.eig, stride);
                ch_kernel<<<dim3(blocks_for(n, 128), 3), 128, 0, s>>>(scene, cv, sp, acc, stride, cv.eig, out);
            };
            if (cv.n_views <= 1) {
                run(solve_color_gram_k<1>, solve_color_k<1>, solve_color_fused_k<1>);
            } else if (cv.n_views <= 2) {
                run(solve_color_gram_k<2>, solve_color_k<2>, solve_color_fused_k<2>);
            } else if (cv.n_views <= 4) {
                run(solve_color_gram_k<4>, solve_color_k<4>, solve_color_fused_k<4>);
            } else if (cv.n_views <= 8) {
                run(solve_color_gram_k<8>, solve_color_k<8>, solve_color_fused_k<8>);
            } else {  // knn 8..15 (the reference's overshoot ablation uses knn = 8): spills, rarely used
                run(solve_color_gram_k<16>, solve_color_k<16>, solve_color_fused_k<16>);
            }
            break;
        }
    }
    CUDA_LAUNCH_CHECK();
}

}  // namespace ngsb
