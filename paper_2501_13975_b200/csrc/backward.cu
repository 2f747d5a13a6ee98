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
__global__ void __launch_bounds__(128) position_consts_k(SceneDev s, CameraDev cam, const uint8_t* flags,
                                                         float* out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= s.n) return;
    float* o = out + static_cast<size_t>(k) * kPosConsts;
    if (!(flags[k] & kProjected)) return;
    const D3 p = load_pos(s, k);
    double M[5][3], Hu[5][6];
    // pi(p) through view_proj.
    {
        const double* VP = cam.view_proj;
        const double hx = mrow(VP, 0, 0) * p.x + mrow(VP, 0, 1) * p.y + mrow(VP, 0, 2) * p.z + mrow(VP, 0, 3);
        const double hy = mrow(VP, 1, 0) * p.x + mrow(VP, 1, 1) * p.y + mrow(VP, 1, 2) * p.z + mrow(VP, 1, 3);
        const double hw = mrow(VP, 3, 0) * p.x + mrow(VP, 3, 1) * p.y + mrow(VP, 3, 2) * p.z + mrow(VP, 3, 3);
        const double a[3] = {mrow(VP, 0, 0), mrow(VP, 0, 1), mrow(VP, 0, 2)};
        const double b[3] = {mrow(VP, 1, 0), mrow(VP, 1, 1), mrow(VP, 1, 2)};
        const double w[3] = {mrow(VP, 3, 0), mrow(VP, 3, 1), mrow(VP, 3, 2)};
        const double i1 = 1.0 / hw, i2 = i1 * i1, i3 = i2 * i1;
        const double sx = 0.5 * cam.width, sy = 0.5 * cam.height;
        for (int j = 0; j < 3; ++j) {
            M[0][j] = sx * (a[j] * i1 - hx * i2 * w[j]);
            M[1][j] = sy * (b[j] * i1 - hy * i2 * w[j]);
        }
        for (int i = 0; i < 3; ++i)
            for (int j = i; j < 3; ++j) {
                Hu[0][sym3(i, j)] = sx * (-(a[i] * w[j] + w[i] * a[j]) * i2 + 2.0 * hx * w[i] * w[j] * i3);
                Hu[1][sym3(i, j)] = sy * (-(b[i] * w[j] + w[i] * b[j]) * i2 + 2.0 * hy * w[i] * w[j] * i3);
            }
    }
    // Sigma(p) through the EWA Jacobian.
    {
        const D3 t = to_camera_space(cam, p);
        CamProj cp;
        project_camera_space<true, true>(cam, t, cp);
        double A[9], m[9];
        covariance_3d(s.quat[k], s.scale[k], A);
        rotate_cov(cam, A, m);
        double dj[3][6], d2j[3][3][6];
        for (int c = 0; c < 3; ++c)
            for (int q = 0; q < 6; ++q) {
                double v = 0;
                for (int e = 0; e < 3; ++e) v += cp.dJ[e][q] * mrow(cam.view, e, c);
                dj[c][q] = v;
            }
        for (int c = 0; c < 3; ++c)
            for (int d = 0; d < 3; ++d)
                for (int q = 0; q < 6; ++q) {
                    double v = 0;
                    for (int e = 0; e < 3; ++e)
                        for (int f = 0; f < 3; ++f) v += cp.d2J[e][f][q] * (mrow(cam.view, e, c) * mrow(cam.view, f, d));
                    d2j[c][d][q] = v;
                }
        // mjt = m J^T (3x2)
        double mjt[6];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 2; ++j)
                mjt[2 * i + j] = m[3 * i] * cp.J[3 * j] + m[3 * i + 1] * cp.J[3 * j + 1] + m[3 * i + 2] * cp.J[3 * j + 2];
        auto mul23_32 = [](const double* a23, const double* b32, double out[4]) {
            for (int i = 0; i < 2; ++i)
                for (int j = 0; j < 2; ++j)
                    out[2 * i + j] = a23[3 * i] * b32[j] + a23[3 * i + 1] * b32[2 + j] + a23[3 * i + 2] * b32[4 + j];
        };
        for (int c = 0; c < 3; ++c) {
            double tm[4];
            mul23_32(dj[c], mjt, tm);
            M[2][c] = 2.0 * tm[0];
            M[3][c] = tm[1] + tm[2];
            M[4][c] = 2.0 * tm[3];
        }
        for (int c = 0; c < 3; ++c)
            for (int d = c; d < 3; ++d) {
                double t1[4], t2[4], md[6];
                mul23_32(d2j[c][d], mjt, t1);
                // dj_c m dj_d^T
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 2; ++j)
                        md[2 * i + j] = m[3 * i] * dj[d][3 * j] + m[3 * i + 1] * dj[d][3 * j + 1] + m[3 * i + 2] * dj[d][3 * j + 2];
                mul23_32(dj[c], md, t2);
                Hu[2][sym3(c, d)] = 2.0 * t1[0] + 2.0 * t2[0];
                Hu[3][sym3(c, d)] = t1[1] + t1[2] + t2[1] + t2[2];
                Hu[4][sym3(c, d)] = 2.0 * t1[3] + 2.0 * t2[3];
            }
    }
    for (int i = 0; i < 5; ++i)
        for (int j = 0; j < 3; ++j) o[kPosM + 3 * i + j] = static_cast<float>(M[i][j]);
    for (int i = 0; i < 5; ++i)
        for (int j = 0; j < 6; ++j) o[kPosHu + 6 * i + j] = static_cast<float>(Hu[i][j]);
    // SH colour derivatives through r(p) (view_direction_derivatives camera.hpp:79-104).
    D3 r;
    double n;
    double Jc[3][3] = {}, Hc[3][6] = {};
    if (view_direction(cam, p, r, n)) {
        const double rv[3] = {r.x, r.y, r.z};
        double jac[3][3];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) jac[i][j] = ((i == j ? 1.0 : 0.0) - rv[i] * rv[j]) / n;
        const double inv_n2 = 1.0 / (n * n);
        double basis[16];
        sh_basis(r, s.sh_degree, basis);
        for (int ch = 0; ch < 3; ++ch) {
            double c[16] = {};
            double v = 0;
            for (int i = 0; i < s.n_coeffs; ++i) {
                c[i] = s.sh[(16 * ch + i) * s.n + k];
                v += basis[i] * c[i];
            }
            v += kColorOffset;
            if (v <= 0.0) continue;  // clamped: zero subgradient (sh.hpp:144-147)
            double gr[3], hr[6];
            sh_contract_derivs(r, s.sh_degree, c, gr, hr);
            for (int j = 0; j < 3; ++j) Jc[ch][j] = jac[0][j] * gr[0] + jac[1][j] * gr[1] + jac[2][j] * gr[2];
            for (int a = 0; a < 3; ++a)
                for (int b = a; b < 3; ++b) {
                    double acc = 0;
                    for (int i = 0; i < 3; ++i)
                        for (int j = 0; j < 3; ++j) acc += jac[i][a] * hr[sym3(i, j)] * jac[j][b];
                    for (int i = 0; i < 3; ++i) {
                        double hv = 3.0 * rv[i] * rv[a] * rv[b];
                        if (i == a) hv -= rv[b];
                        if (i == b) hv -= rv[a];
                        if (a == b) hv -= rv[i];
                        acc += gr[i] * hv * inv_n2;
                    }
                    Hc[ch][sym3(a, b)] = acc;
                }
        }
    }
    for (int ch = 0; ch < 3; ++ch) {
        for (int j = 0; j < 3; ++j) o[kPosJc + 3 * ch + j] = static_cast<float>(Jc[ch][j]);
        for (int j = 0; j < 6; ++j) o[kPosHc + 6 * ch + j] = static_cast<float>(Hc[ch][j]);
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
}

// ---------------------------------------------------------------------------
// Tile backward kernel
// ---------------------------------------------------------------------------

template <int PASS>
struct PassTraits;
template <>
struct PassTraits<kPassPosition> {
    static constexpr int NC = kPosConsts, NACC = 9, BATCH = 64;
};
template <>
struct PassTraits<kPassRotation> {
    static constexpr int NC = kRotConsts, NACC = 2, BATCH = 128;
};
template <>
struct PassTraits<kPassScaling> {
    static constexpr int NC = kScaleConsts, NACC = 5, BATCH = 128;
};
template <>
struct PassTraits<kPassOpacityColor> {
    static constexpr int NC = 0, NACC = 8, BATCH = 128;
};

// d(G)/du and d2G/du2 for u = (pi_x, pi_y, S00, S01, S11), off-diagonal S01
// moving both symmetric entries (equivalent to the symmetrised tensors of
// gaussian_weight, rasterizer.hpp:116-176).
struct GDerivs {
    float g[5];
    float h[15];  // packed upper triangle, row-major over 5x5
};

__device__ __forceinline__ int s5(int i, int j) {
    const int a = i < j ? i : j, b = i < j ? j : i;
    return a * 5 - a * (a - 1) / 2 + (b - a);
}

__device__ __forceinline__ void sigma_second(float G, float qd0, float qd1, float qa, float qb, float qc, float hss[6]) {
    // u_E = E qd for E in {a, b, c}; d2q_EF = 2 u_E^T Q u_F; dq = (-qd0^2, -2 qd0 qd1, -qd1^2)
    const float ux[3] = {qd0, qd1, 0.f};
    const float uy[3] = {0.f, qd0, qd1};
    const float dq[3] = {-qd0 * qd0, -2.f * qd0 * qd1, -qd1 * qd1};
    int idx = 0;
    for (int e = 0; e < 3; ++e)
        for (int f = e; f < 3; ++f) {
            const float quad = ux[e] * (qa * ux[f] + qb * uy[f]) + uy[e] * (qb * ux[f] + qc * uy[f]);
            hss[idx++] = G * (0.25f * dq[e] * dq[f] - quad);
        }
}

__device__ __forceinline__ void g_derivs(const SplatEval& ev, float qa, float qb, float qc, GDerivs& d) {
    const float G = ev.g, q0 = ev.qd0, q1 = ev.qd1;
    d.g[0] = -G * q0;
    d.g[1] = -G * q1;
    d.g[2] = 0.5f * G * q0 * q0;
    d.g[3] = G * q0 * q1;
    d.g[4] = 0.5f * G * q1 * q1;
    // pi-pi block: G (qd qd^T - Q)
    d.h[s5(0, 0)] = G * (q0 * q0 - qa);
    d.h[s5(0, 1)] = G * (q0 * q1 - qb);
    d.h[s5(1, 1)] = G * (q1 * q1 - qc);
    // pi-Sigma block: -g_k qd_a + G (Q E_k qd)_a
    const float QEa[2] = {q0 * qa, q0 * qb};
    const float QEb[2] = {qa * q1 + qb * q0, qb * q1 + qc * q0};
    const float QEc[2] = {q1 * qb, q1 * qc};
    const float qdv[2] = {q0, q1};
    for (int a = 0; a < 2; ++a) {
        d.h[s5(a, 2)] = -d.g[2] * qdv[a] + G * QEa[a];
        d.h[s5(a, 3)] = -d.g[3] * qdv[a] + G * QEb[a];
        d.h[s5(a, 4)] = -d.g[4] * qdv[a] + G * QEc[a];
    }
    float hss[6];
    sigma_second(G, q0, q1, qa, qb, qc, hss);
    d.h[s5(2, 2)] = hss[0];
    d.h[s5(2, 3)] = hss[1];
    d.h[s5(2, 4)] = hss[2];
    d.h[s5(3, 3)] = hss[3];
    d.h[s5(3, 4)] = hss[4];
    d.h[s5(4, 4)] = hss[5];
}

template <int PASS>
__global__ void __launch_bounds__(256) backward_k(BackwardArgs a) {
    using TR = PassTraits<PASS>;
    constexpr int B = TR::BATCH, NC = TR::NC, NA = TR::NACC;
    __shared__ float s_px[B], s_py[B], s_qa[B], s_qb[B], s_qc[B], s_sig[B], s_c[3][B], s_qmax[B];
    __shared__ float s_const[(NC > 0 ? NC : 1) * B];
    __shared__ float s_acc[NA][B];
    __shared__ int s_kid[B];
    __shared__ int s_cnt[B];
    __shared__ int s_maxlast;
    unsigned long long block_pairs = 0;

    const int tile = blockIdx.x;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;
    const int x = tx * kTile + lx, y = ty * kTile + ly;
    const bool inside = x < a.W && y < a.H;
    const float fx = lx + 0.5f, fy = ly + 0.5f;
    const double ox = tx * kTile, oy = ty * kTile;
    const int2 range = a.ranges[tile];
    const size_t plane = static_cast<size_t>(a.W) * a.H;
    const size_t pidx = static_cast<size_t>(y) * a.W + x;

    int last = -1;
    double Cf[3] = {0, 0, 0};
    float gl[3] = {0, 0, 0}, hl[3] = {0, 0, 0};
    if (inside) {
        last = a.last[pidx];
        for (int c = 0; c < 3; ++c) {
            Cf[c] = a.image[c * plane + pidx];
            gl[c] = a.loss_grad[c * plane + pidx];
            hl[c] = a.loss_hess[c * plane + pidx];
        }
    }
    if (threadIdx.x == 0) s_maxlast = -1;
    __syncthreads();
    if (last >= 0) atomicMax(&s_maxlast, last);
    __syncthreads();
    const int end = min(range.y, s_maxlast + 1);

    float T = 1.0f;
    double P[3] = {0, 0, 0};  // FP64 prefix sums, identical to the forward's colour sums
    const int lane = threadIdx.x & 31;

    for (int base = range.x; base < end; base += B) {
        const int cnt = min(B, end - base);
        __syncthreads();
        for (int i = threadIdx.x; i < B; i += blockDim.x) {
            if (i < cnt) {
                const int k = a.vals[base + i];
                s_kid[i] = k;
                const double2 p = a.pix[k];
                const float4 ra = a.ra[k], rb = a.rb[k], rc = a.rc[k];
                s_px[i] = static_cast<float>(p.x - ox);
                s_py[i] = static_cast<float>(p.y - oy);
                s_qa[i] = ra.z;
                s_qb[i] = ra.w;
                s_qc[i] = rb.x;
                s_sig[i] = rb.y;
                s_c[0][i] = rb.z;
                s_c[1][i] = rb.w;
                s_c[2][i] = rc.x;
                s_qmax[i] = reject_bound(rb.y, a.cutoff);
            }
            for (int c = 0; c < NA; ++c) s_acc[c][i] = 0.f;
            s_cnt[i] = 0;
        }
        if constexpr (NC > 0) {
            for (int i = threadIdx.x; i < cnt * NC; i += blockDim.x) {
                const int j = i / NC, c = i - j * NC;
                s_const[i] = a.consts[static_cast<size_t>(a.vals[base + j]) * NC + c];
            }
        }
        __syncthreads();
        for (int j = 0; j < cnt; ++j) {
            float v[NA];
#pragma unroll
            for (int c = 0; c < NA; ++c) v[c] = 0.f;
            bool contrib = false;
            if (base + j <= last) {
                const float qa = s_qa[j], qb = s_qb[j], qc = s_qc[j], sig = s_sig[j];
                SplatEval ev;
                if (eval_splat(s_px[j], s_py[j], qa, qb, qc, sig, fx, fy, s_qmax[j], ev) && !(ev.alpha < a.cutoff)) {
                    contrib = true;
                    const float Ti = T;
                    const float w = blend_weight(Ti, ev.alpha);
                    const float Tn = next_transmittance(Ti, ev.alpha);
                    float acol[3];  // c~ - behind
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const float cc = s_c[c][j];
                        const double Pn = __fma_rn(static_cast<double>(w), cc, P[c]);
                        const float behind =
                            (base + j == last) ? a.bg[c] : static_cast<float>(Cf[c] - Pn) * __frcp_rn(Tn);
                        acol[c] = cc - behind;
                        P[c] = Pn;
                    }
                    T = Tn;
                    const float wa = sig * Ti;  // w_alpha = sigma * T
                    if constexpr (PASS == kPassPosition) {
                        const float* K = s_const + j * NC;
                        GDerivs d;
                        g_derivs(ev, qa, qb, qc, d);
                        // dG/dp = M^T g
                        float dG[3];
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            float t = 0.f;
#pragma unroll
                            for (int u = 0; u < 5; ++u) t += K[kPosM + 3 * u + c] * d.g[u];
                            dG[c] = t;
                        }
                        // V = H M (5x3)
                        float V[5][3];
#pragma unroll
                        for (int u = 0; u < 5; ++u)
#pragma unroll
                            for (int c = 0; c < 3; ++c) {
                                float t = 0.f;
#pragma unroll
                                for (int l = 0; l < 5; ++l) t += d.h[s5(u, l)] * K[kPosM + 3 * l + c];
                                V[u][c] = t;
                            }
                        // d2G/dp2 (sym 6) = M^T V + sum_u g_u Hu_u
                        float d2G[6];
#pragma unroll
                        for (int c = 0; c < 3; ++c)
#pragma unroll
                            for (int e = c; e < 3; ++e) {
                                float t = 0.f;
#pragma unroll
                                for (int u = 0; u < 5; ++u) t += K[kPosM + 3 * u + c] * V[u][e] + d.g[u] * K[kPosHu + 6 * u + sym3(c, e)];
                                d2G[sym3(c, e)] = t;
                            }
                        // Channel sums (newton.hpp:329-340)
                        float sgl = 0.f, vgl[3] = {0.f, 0.f, 0.f}, hc[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
                        for (int ch = 0; ch < 3; ++ch) {
                            const float gw = gl[ch] * wa;
                            sgl += gw * acol[ch];
#pragma unroll
                            for (int c = 0; c < 3; ++c) vgl[c] += gw * K[kPosJc + 3 * ch + c];
#pragma unroll
                            for (int q = 0; q < 6; ++q) hc[q] += gw * K[kPosHc + 6 * ch + q];
                        }
                        const float G = ev.g;
#pragma unroll
                        for (int c = 0; c < 3; ++c) v[c] = sgl * dG[c] + G * vgl[c];
#pragma unroll
                        for (int c = 0; c < 3; ++c)
#pragma unroll
                            for (int e = c; e < 3; ++e) {
                                const int q = sym3(c, e);
                                float t = sgl * d2G[q] + G * hc[q] + dG[c] * vgl[e] + vgl[c] * dG[e];
#pragma unroll
                                for (int ch = 0; ch < 3; ++ch) {
                                    const float dcc = wa * (acol[ch] * dG[c] + G * K[kPosJc + 3 * ch + c]);
                                    const float dce = wa * (acol[ch] * dG[e] + G * K[kPosJc + 3 * ch + e]);
                                    t += hl[ch] * dcc * dce;
                                }
                                v[3 + q] = t;
                            }
                    } else if constexpr (PASS == kPassRotation) {
                        const float* K = s_const + j * NC;
                        const float G = ev.g, q0 = ev.qd0, q1 = ev.qd1;
                        const float gs[3] = {0.5f * G * q0 * q0, G * q0 * q1, 0.5f * G * q1 * q1};
                        float hss[6];
                        sigma_second(G, q0, q1, qa, qb, qc, hss);
                        const float s1[3] = {K[0], K[1], K[2]};
                        const float dg = gs[0] * K[0] + gs[1] * K[1] + gs[2] * K[2];
                        float d2g = gs[0] * K[3] + gs[1] * K[4] + gs[2] * K[5];
                        d2g += s1[0] * (hss[0] * s1[0] + 2.f * hss[1] * s1[1] + 2.f * hss[2] * s1[2]) +
                               s1[1] * (hss[3] * s1[1] + 2.f * hss[4] * s1[2]) + s1[2] * hss[5] * s1[2];
#pragma unroll
                        for (int ch = 0; ch < 3; ++ch) {
                            const float dc = wa * acol[ch] * dg;
                            v[0] += gl[ch] * dc;
                            v[1] += hl[ch] * dc * dc + gl[ch] * wa * acol[ch] * d2g;
                        }
                    } else if constexpr (PASS == kPassScaling) {
                        const float* K = s_const + j * NC;
                        const float G = ev.g;
                        const float z0 = K[0] * ev.qd0 + K[1] * ev.qd1;
                        const float z1 = K[2] * ev.qd0 + K[3] * ev.qd1;
                        const float dg0 = 0.5f * G * z0 * z0, dg1 = 0.5f * G * z1 * z1;
                        const float h00 = G * (0.25f * z0 * z0 * z0 * z0 - z0 * z0 * K[4]);
                        const float h01 = G * (0.25f * z0 * z0 * z1 * z1 - z0 * z1 * K[5]);
                        const float h11 = G * (0.25f * z1 * z1 * z1 * z1 - z1 * z1 * K[6]);
#pragma unroll
                        for (int ch = 0; ch < 3; ++ch) {
                            const float s = wa * acol[ch];
                            const float dc0 = s * dg0, dc1 = s * dg1;
                            const float gs = gl[ch] * s;
                            v[0] += gl[ch] * dc0;
                            v[1] += gl[ch] * dc1;
                            v[2] += hl[ch] * dc0 * dc0 + gs * h00;
                            v[3] += hl[ch] * dc0 * dc1 + gs * h01;
                            v[4] += hl[ch] * dc1 * dc1 + gs * h11;
                        }
                    } else {  // opacity data terms + colour accumulators (newton.hpp:516-567)
                        const float GT = ev.g * Ti;
#pragma unroll
                        for (int ch = 0; ch < 3; ++ch) {
                            const float dc = GT * acol[ch];
                            v[0] += gl[ch] * dc;
                            v[1] += hl[ch] * dc * dc;
                            v[2 + ch] = gl[ch] * w;
                            v[5 + ch] = hl[ch] * w * w;
                        }
                    }
                }
            }
            const unsigned ballot = __ballot_sync(0xffffffffu, contrib);
            if (ballot) {
                const float sum = warp_reduce_scatter<NA>(v, lane);
                const int idx = reduce_index<NA>(lane);
                if (reduce_representative<NA>(lane) && idx < NA) atomicAdd(&s_acc[idx][j], sum);
                if (lane == 0) {
                    atomicAdd(&s_cnt[j], __popc(ballot));
                    block_pairs += __popc(ballot);
                }
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
            const int k = s_kid[i];
            if (a.visible && s_cnt[i] > 0) a.visible[k] = 1;
#pragma unroll
            for (int c = 0; c < NA; ++c) {
                const float val = s_acc[c][i];
                if (val != 0.f) atomicAdd(&a.acc[static_cast<size_t>(c) * a.acc_stride + k], static_cast<double>(val));
            }
        }
    }
    if (a.contrib_pairs && lane == 0 && block_pairs) atomicAdd(a.contrib_pairs, block_pairs);
}

}  // namespace

void compute_pass_consts(int pass, const SceneDev& scene, ViewSlot& v, const CameraDev& primary, cudaStream_t s) {
    const int n = scene.n;
    if (n == 0 || pass == kPassOpacityColor) return;
    StageScope st(NGS_STAGE_CONSTS, s);
    switch (pass) {
        case kPassPosition:
            v.consts.ensure(static_cast<size_t>(n) * kPosConsts);
            position_consts_k<<<blocks_for(n, 128), 128, 0, s>>>(scene, v.cam, v.flags.ptr, v.consts.ptr);
            break;
        case kPassRotation:
            v.consts.ensure(static_cast<size_t>(n) * kRotConsts);
            rotation_consts_k<<<blocks_for(n, 128), 128, 0, s>>>(scene, v.cam, primary, v.flags.ptr, v.consts.ptr);
            break;
        case kPassScaling:
            v.consts.ensure(static_cast<size_t>(n) * kScaleConsts);
            scaling_consts_k<<<blocks_for(n, 128), 128, 0, s>>>(scene, v.cam, v.raster.lambda_lp, v.flags.ptr,
                                                                 v.consts.ptr);
            break;
        default:
            return;
    }
    CUDA_LAUNCH_CHECK();
}

void launch_backward(int pass, const SceneDev& scene, ViewSlot& v, double* acc, size_t acc_stride, uint8_t* visible,
                     unsigned long long* contrib_pairs, cudaStream_t s) {
    if (v.pairs == 0 || v.n == 0) return;
    BackwardArgs a;
    a.tiles_x = v.cam.tiles_x;
    a.W = v.W;
    a.H = v.H;
    a.ranges = v.ranges.ptr;
    a.vals = v.pair_val_sorted.ptr;
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
    a.visible = visible;
    a.contrib_pairs = contrib_pairs;
    StageScope st(NGS_STAGE_BWD_POSITION + pass, s);
    switch (pass) {
        case kPassPosition: backward_k<kPassPosition><<<v.T, 256, 0, s>>>(a); break;
        case kPassRotation: backward_k<kPassRotation><<<v.T, 256, 0, s>>>(a); break;
        case kPassScaling: backward_k<kPassScaling><<<v.T, 256, 0, s>>>(a); break;
        case kPassOpacityColor: backward_k<kPassOpacityColor><<<v.T, 256, 0, s>>>(a); break;
    }
    CUDA_LAUNCH_CHECK();
}

}  // namespace ngsb
