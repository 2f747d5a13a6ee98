// loss.cu — K7: L2 + SSIM loss value and per-pixel gradient / diagonal Hessian
// fields (total_loss_derivs, loss.hpp:342-356).
//
// FP64 throughout: SSIM variance/covariance are E[x^2]-E[x]^2 differences of
// O(1) quantities whose result is O(1e-6) in flat regions; FP32 loses them
// entirely (SURVEY.md §7 hard part 1). Two kernels, each a separable valid-tap
// convolution (loss.hpp:81-115) with a halo of window/2 on every side:
//   A: 5 window statistics -> 9 window-centre fields (loss.hpp:162-214, 262-305)
//   B: 9 field convolutions (w for grad/kw, w^2 for the rest) -> grad, hess
//      (loss.hpp:309-329) plus the L2 terms (loss.hpp:138-156).
// The default 11-tap window runs the 32x32-tile register-blocked kernels
// (ssim_fields32_k / ssim_derivs32_k); other windows the generic 16x16 ones.
// compute_loss_value is the value-only variant used by the metrics.
#include <algorithm>

#include "context.h"
#include "splat.cuh"

// Minimum resident blocks per SM of the 32-bit SSIM kernels (build-time knobs for A/B runs).
#ifndef NGS_SSIMD_MINB
#define NGS_SSIMD_MINB 3
#endif
#ifndef NGS_SSIMF_MINB
#define NGS_SSIMF_MINB 3
#endif

namespace ngsb {

namespace {

constexpr int kLT = 16;       // output tile edge
constexpr int kMaxHalf = 10;  // window <= 21

struct Window {
    double w[2 * kMaxHalf + 1];
    double w2[2 * kMaxHalf + 1];
    double full;  // sum of all taps in the device loop's order (window wholly inside the image)
    int half;
};

__device__ __forceinline__ double axis_norm(int x, int n, const Window& win) {
    if (x >= win.half && x + win.half < n) return win.full;  // same sum, no loop
    const int i0 = max(-win.half, -x), i1 = min(win.half, n - 1 - x);
    double s = 0;
    for (int i = i0; i <= i1; ++i) s += win.w[i + win.half];
    return s;
}

__device__ __forceinline__ double block_sum(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double t = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (blockDim.x >> 5); ++i) t += red[i];
    return t;
}

// SSIM and its 9 window-centre derivative fields from the 5 filtered window
// statistics (loss.hpp:262-305); reciprocals of f2, f3 hoisted (two divisions).
__device__ __forceinline__ double ssim_centre_fields(const double (&st)[5], double inv_norm, double c1, double c2,
                                                     double (&out)[9]) {
    const double mu = st[0] * inv_norm, mu_t = st[2] * inv_norm;
    const double var = fmax(0.0, st[1] * inv_norm - mu * mu);
    const double var_t = fmax(0.0, st[3] * inv_norm - mu_t * mu_t);
    const double cov = st[4] * inv_norm - mu * mu_t;
    // loss.hpp:266-303 (reciprocals of f2, f3 hoisted: two divisions per pixel)
    const double f0 = 2.0 * mu * mu_t + c1;
    const double f1 = 2.0 * cov + c2;
    const double f2 = mu * mu + mu_t * mu_t + c1;
    const double f3 = var + var_t + c2;
    const double inv_f2 = 1.0 / f2, inv_f3 = 1.0 / f3;
    const double nn = f0 * f1;
    const double inv_d = inv_f2 * inv_f3;
    const double ssim = nn * inv_d;
    const double a0 = 2.0 * mu_t, a1 = -2.0 * mu_t, b1 = 2.0;
    const double a2 = 2.0 * mu, a3 = -2.0 * mu, b3 = 2.0;
    const double A = a0 * f1 + f0 * a1, B = f0 * b1, C = a2 * f3 + f2 * a3, E = f2 * b3;
    const double inv_d2 = inv_d * inv_d, inv_d3 = inv_d2 * inv_d, inv_norm2 = inv_norm * inv_norm;
    const double nnd = nn * inv_d;
    out[0] = (2.0 * mu_t * (f1 - f0) * inv_d - 2.0 * mu * nnd * inv_f2 + 2.0 * mu * nnd * inv_f3) * inv_norm;
    out[1] = 2.0 * f0 * inv_d * inv_norm;
    out[2] = -2.0 * nnd * inv_f3 * inv_norm;
    out[3] = -2.0 * nn * inv_f2 * inv_f3 * inv_f3 * inv_norm;
    out[4] = (2.0 * a0 * a1 * inv_d - 2.0 * A * C * inv_d2 - nn * (2.0 * a2 * a3 + 2.0 * f3 - 2.0 * f2) * inv_d2 +
              2.0 * nn * C * C * inv_d3) *
             inv_norm2;
    out[5] = (-2.0 * A * E * inv_d2 - 2.0 * nn * a2 * b3 * inv_d2 + 4.0 * nn * C * E * inv_d3) * inv_norm2;
    out[6] = (2.0 * a0 * b1 * inv_d - 2.0 * B * C * inv_d2) * inv_norm2;
    out[7] = -2.0 * B * E * inv_d2 * inv_norm2;
    out[8] = 2.0 * nn * E * E * inv_d3 * inv_norm2;
    return ssim;
}

// SSIM value alone (ssim_value_and_derivs with want_derivs = false, loss.hpp:262-277).
__device__ __forceinline__ double ssim_value_only(const double (&st)[5], double inv_norm, double c1, double c2) {
    const double mu = st[0] * inv_norm, mu_t = st[2] * inv_norm;
    const double var = fmax(0.0, st[1] * inv_norm - mu * mu);
    const double var_t = fmax(0.0, st[3] * inv_norm - mu_t * mu_t);
    const double cov = st[4] * inv_norm - mu * mu_t;
    const double f0 = 2.0 * mu * mu_t + c1, f1 = 2.0 * cov + c2;
    const double f2 = mu * mu + mu_t * mu_t + c1, f3 = var + var_t + c2;
    return (f0 * f1) / (f2 * f3);
}

// Sum of squared differences of two planar images (the L2 part of
// total_loss_value and the PSNR numerator, loss.hpp:363-368, metrics.hpp:16-20).
__global__ void __launch_bounds__(256) l2_sum_k(const double* __restrict__ a, const double* __restrict__ b, size_t n,
                                                unsigned long long* __restrict__ sum) {
    __shared__ double red[8];
    double acc = 0.0;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const double d = a[i] - b[i];
        acc += d * d;
    }
    const double tot = block_sum(acc, red);
    if (threadIdx.x == 0) exact_add(sum, tot);
}

// Separable valid-tap convolutions over a (kLT + 2h)^2 shared-memory halo tile.
// HT > 0 fixes the window half-width at compile time (the default 11-tap
// window: fully unrolled, register-blocked two outputs per horizontal task);
// HT == 0 is the generic path for any window <= 21.
template <int HT>
struct SsimGeom {
    static constexpr int HMAX = HT > 0 ? HT : kMaxHalf;
    static constexpr int SP = kLT + 2 * HMAX;  // halo tile edge
};

// Horizontal pass of `nf` planes: out[f][r][c] = sum_k w_f[k] in[f][r][c + k],
// rows r < span, two adjacent outputs per task (each input loaded once).
template <int HT, int NF, class In, class Out, class WSel>
__device__ __forceinline__ void hpass(int h, int span, In in, Out out, WSel wsel) {
    constexpr int HALF = kLT / 2;
    for (int task = threadIdx.x; task < NF * span * HALF; task += blockDim.x) {
        const int f = task / (span * HALF);
        const int rem = task - f * span * HALF;
        const int r = rem / HALF, c0 = (rem - r * HALF) * 2;
        const double* w = wsel(f);
        double a0 = 0.0, a1 = 0.0;
        if constexpr (HT > 0) {
#pragma unroll
            for (int k = 0; k <= 2 * HT + 1; ++k) {
                const double v = in(f, r, c0 + k);
                if (k <= 2 * HT) a0 += w[k] * v;
                if (k >= 1) a1 += w[k - 1] * v;
            }
        } else {
            for (int k = 0; k <= 2 * h + 1; ++k) {
                const double v = in(f, r, c0 + k);
                if (k <= 2 * h) a0 += w[k] * v;
                if (k >= 1) a1 += w[k - 1] * v;
            }
        }
        out(f, r, c0) = a0;
        out(f, r, c0 + 1) = a1;
    }
}

// Kernel A: window statistics and the 9 window-centre fields for one channel.
template <int HT>
__global__ void __launch_bounds__(256) ssim_fields_k(int W, int H, const double* __restrict__ image,
                                                     const double* __restrict__ target, Window win, double c1, double c2,
                                                     double* __restrict__ fields, unsigned long long* __restrict__ sums, int row0,
                                                     int own_y0, int own_y1) {
    constexpr int SP = SsimGeom<HT>::SP;
    __shared__ double s_x[SP][SP + 1], s_t[SP][SP + 1];
    __shared__ double s_h[5][SP][kLT + 1];
    __shared__ double red[8];
    const int ch = blockIdx.z;
    const int ox = blockIdx.x * kLT, oy = (row0 + blockIdx.y) * kLT;
    const int h = HT > 0 ? HT : win.half, span = kLT + 2 * h;
    const size_t plane = static_cast<size_t>(W) * H;
    const double* img = image + ch * plane;
    const double* tgt = target + ch * plane;
    for (int i = threadIdx.x; i < span * span; i += blockDim.x) {
        const int r = i / span, c = i - r * span;
        const int gx = ox - h + c, gy = oy - h + r;
        const bool in = gx >= 0 && gx < W && gy >= 0 && gy < H;
        const size_t idx = static_cast<size_t>(gy) * W + gx;
        s_x[r][c] = in ? img[idx] : 0.0;
        s_t[r][c] = in ? tgt[idx] : 0.0;
    }
    __syncthreads();
    // Horizontal pass of the 5 statistics (out-of-image taps are zero == skipped taps):
    // two outputs per task, 5 products per loaded tap.
    {
        constexpr int HALF = kLT / 2;
        for (int task = threadIdx.x; task < span * HALF; task += blockDim.x) {
            const int r = task / HALF, c0 = (task - r * HALF) * 2;
            double a[2][5] = {};
            auto tap = [&](int k) {
                const double xv = s_x[r][c0 + k], tv = s_t[r][c0 + k];
                const double p[5] = {xv, xv * xv, tv, tv * tv, xv * tv};
                const int hh = HT > 0 ? HT : h;
                if (k <= 2 * hh) {
                    const double wk = win.w[k];
#pragma unroll
                    for (int f = 0; f < 5; ++f) a[0][f] += wk * p[f];
                }
                if (k >= 1) {
                    const double wk = win.w[k - 1];
#pragma unroll
                    for (int f = 0; f < 5; ++f) a[1][f] += wk * p[f];
                }
            };
            if constexpr (HT > 0) {
#pragma unroll
                for (int k = 0; k <= 2 * HT + 1; ++k) tap(k);
            } else {
                for (int k = 0; k <= 2 * h + 1; ++k) tap(k);
            }
#pragma unroll
            for (int f = 0; f < 5; ++f) {
                s_h[f][r][c0] = a[0][f];
                s_h[f][r][c0 + 1] = a[1][f];
            }
        }
    }
    __syncthreads();
    const int lx = threadIdx.x % kLT, ly = threadIdx.x / kLT;
    const int x = ox + lx, y = oy + ly;
    double ssim = 0.0;
    if (x < W && y < H) {
        double st[5] = {};
        if constexpr (HT > 0) {
#pragma unroll
            for (int k = 0; k <= 2 * HT; ++k)
#pragma unroll
                for (int f = 0; f < 5; ++f) st[f] += win.w[k] * s_h[f][ly + k][lx];
        } else {
            for (int k = 0; k <= 2 * h; ++k)
#pragma unroll
                for (int f = 0; f < 5; ++f) st[f] += win.w[k] * s_h[f][ly + k][lx];
        }
        const double inv_norm = 1.0 / (axis_norm(x, W, win) * axis_norm(y, H, win));
        if (fields) {
            double out[9];
            ssim = ssim_centre_fields(st, inv_norm, c1, c2, out);
            const size_t idx = static_cast<size_t>(y) * W + x;
#pragma unroll
            for (int f = 0; f < 9; ++f) fields[(static_cast<size_t>(f) * 3 + ch) * plane + idx] = out[f];
        } else {
            ssim = ssim_value_only(st, inv_norm, c1, c2);  // value-only path (metrics)
        }
    }
    const bool own = y >= own_y0 && y < own_y1;  // owned pixel rows (multi-GPU shard)
    const double tot = block_sum(own ? ssim : 0.0, red);
    if (threadIdx.x == 0) exact_add(sums + kExactWords, tot);
}

// Kernel B: convolve the 9 centre fields (three per shared-memory round) and
// combine into grad / hess (loss.hpp:309-329); also the L2 part (loss.hpp:138-156).
// lambda == 0 skips the SSIM fields entirely (loss.hpp:345).
template <int HT>
__global__ void __launch_bounds__(256) ssim_derivs_k(int W, int H, const double* __restrict__ image,
                                                     const double* __restrict__ target, Window win, double lambda,
                                                     const double* __restrict__ fields, float* __restrict__ grad,
                                                     float* __restrict__ hess, unsigned long long* __restrict__ sums, int row0,
                                                     int own_y0, int own_y1) {
    constexpr int SP = SsimGeom<HT>::SP;
    __shared__ double s_f[3][SP][SP + 1];
    __shared__ double s_h[3][SP][kLT + 1];
    __shared__ double red[8];
    const int ch = blockIdx.z;
    const int ox = blockIdx.x * kLT, oy = (row0 + blockIdx.y) * kLT;
    const int h = HT > 0 ? HT : win.half, span = kLT + 2 * h;
    const size_t plane = static_cast<size_t>(W) * H;
    const int lx = threadIdx.x % kLT, ly = threadIdx.x / kLT;
    const int x = ox + lx, y = oy + ly;
    const bool valid = x < W && y < H;
    const size_t idx = static_cast<size_t>(y) * W + x;
    const double inv3n = 1.0 / (3.0 * static_cast<double>(plane));
    double c = 0, ct = 0;
    if (valid) {
        c = image[ch * plane + idx];
        ct = target[ch * plane + idx];
    }
    double g_ssim = 0, h_ssim = 0;
    if (lambda != 0.0) {
#pragma unroll 1
        for (int g = 0; g < 3; ++g) {
            __syncthreads();
            for (int i = threadIdx.x; i < 3 * span * span; i += blockDim.x) {
                const int f = i / (span * span);
                const int rem = i - f * span * span;
                const int r = rem / span, cc = rem - r * span;
                const int gx = ox - h + cc, gy = oy - h + r;
                const bool in = gx >= 0 && gx < W && gy >= 0 && gy < H;
                const double* field = fields + (static_cast<size_t>(3 * g + f) * 3 + ch) * plane;
                s_f[f][r][cc] = in ? field[static_cast<size_t>(gy) * W + gx] : 0.0;
            }
            __syncthreads();
            // fp, fq, fr, fkw (fields 0-3) use w; the rest w^2
            auto wsel = [&](int f) { return (3 * g + f) <= 3 ? win.w : win.w2; };
            hpass<HT, 3>(h, span, [&](int f, int r, int cc) -> const double& { return s_f[f][r][cc]; },
                         [&](int f, int r, int cc) -> double& { return s_h[f][r][cc]; }, wsel);
            __syncthreads();
            double sv[3] = {};
#pragma unroll
            for (int f = 0; f < 3; ++f) {
                const double* wk = wsel(f);
                if constexpr (HT > 0) {
#pragma unroll
                    for (int k = 0; k <= 2 * HT; ++k) sv[f] += wk[k] * s_h[f][ly + k][lx];
                } else {
                    for (int k = 0; k <= 2 * h; ++k) sv[f] += wk[k] * s_h[f][ly + k][lx];
                }
            }
            if (g == 0) {  // loss.hpp:323-327
                g_ssim += sv[0] + ct * sv[1] + c * sv[2];
            } else if (g == 1) {
                h_ssim += sv[0] + sv[1] + c * sv[2];
            } else {
                h_ssim += ct * sv[0] + c * ct * sv[1] + c * c * sv[2];
            }
        }
    }
    double dsq = 0;
    if (valid) {
        const double d = c - ct;
        dsq = d * d;
        double gg = inv3n * d, hh = inv3n;
        if (lambda != 0.0) {
            gg += lambda * (-inv3n * g_ssim);
            hh += lambda * (-inv3n * h_ssim);
        }
        grad[ch * plane + idx] = static_cast<float>(gg);
        hess[ch * plane + idx] = static_cast<float>(hh);
    }
    const bool own = y >= own_y0 && y < own_y1;
    const double tot = block_sum(own ? dsq : 0.0, red);
    if (threadIdx.x == 0) exact_add(sums, tot);
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit_l() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all_l() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// ---------------------------------------------------------------------------
// 11-tap fast path: 32x32 output tiles, 256 threads. The horizontal pass reads
// its 14-column input windows straight from global memory (L1-resident tile)
// and writes 4 outputs per task to shared memory; the vertical pass gives each
// thread one column x 4 rows and slides the 11 taps over 14 loaded rows, so
// every shared-memory load feeds ~3 FMAs. Thread t owns pixels
// (ox + t % 32, oy + 4 (t / 32) + i), i < 4.
// ---------------------------------------------------------------------------
constexpr int kFT = 32;              // output tile edge
constexpr int kFH = 5;               // window half-width (11 taps)
constexpr int kFS = kFT + 2 * kFH;   // 42 rows / columns incl. halo
constexpr int kFR = 4;               // outputs per task (both passes)
// Derivative-field halo tiles: rows of kFS + 2 doubles from global column ox - kFH - 1
// (16-byte aligned when W is even), row stride kBS (16-byte aligned rows); logical column
// cc (global ox - kFH + cc) lives at index cc + 1.
constexpr int kBS = kFS + 4;
constexpr int kHW = 6;                          // derivative horizontal pass: outputs per task
constexpr int kHG = (kFT + kHW - 1) / kHW;      // ... and tasks per row
constexpr unsigned kBulkRow = sizeof(double) * (kFS + 2);

template <int NF, class Load>
__device__ __forceinline__ void hpass32(const Window& win, unsigned w2mask, Load load, double (*s_h)[kFS][kFT + 1]) {
    // task = (f, r, column group of kFR); inputs c0 .. c0 + kFR + 9
    for (int task = threadIdx.x; task < NF * kFS * (kFT / kFR); task += blockDim.x) {
        const int f = task / (kFS * (kFT / kFR));
        const int rem = task - f * kFS * (kFT / kFR);
        const int r = rem / (kFT / kFR), c0 = (rem - r * (kFT / kFR)) * kFR;
        const bool w2 = (w2mask >> f) & 1u;  // weights selected by value (no parameter-space pointers)
        double acc[kFR] = {};
#pragma unroll
        for (int k = 0; k < kFR + 2 * kFH; ++k) {
            const double v = load(f, r, c0 + k);
#pragma unroll
            for (int o = 0; o < kFR; ++o)
                if (k - o >= 0 && k - o <= 2 * kFH) acc[o] += (w2 ? win.w2[k - o] : win.w[k - o]) * v;
        }
#pragma unroll
        for (int o = 0; o < kFR; ++o) s_h[f][r][c0 + o] = acc[o];
    }
}

// Vertical pass for the calling thread's column and 4 rows: out[o] = sum_k w[k] s_h[r0 + o + k][c].
__device__ __forceinline__ void vpass32(const Window& win, bool w2, const double (*s_hf)[kFT + 1], int c, int r0,
                                        double (&out)[kFR]) {
#pragma unroll
    for (int o = 0; o < kFR; ++o) out[o] = 0.0;
#pragma unroll
    for (int k = 0; k < kFR + 2 * kFH; ++k) {
        const double v = s_hf[r0 + k][c];
#pragma unroll
        for (int o = 0; o < kFR; ++o)
            if (k - o >= 0 && k - o <= 2 * kFH) out[o] += (w2 ? win.w2[k - o] : win.w[k - o]) * v;
    }
}

__global__ void __launch_bounds__(256, NGS_SSIMF_MINB) ssim_fields32_k(int W, int H, const double* __restrict__ image,
                                                       const double* __restrict__ target, Window win, double c1,
                                                       double c2, double* __restrict__ fields,
                                                       unsigned long long* __restrict__ sums, int row0, int own_y0, int own_y1) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    auto s_h = reinterpret_cast<double (*)[kFS][kFT + 1]>(smem_raw);  // [5][kFS][kFT + 1]
    __shared__ double red[8];
    const int ch = blockIdx.z;
    const int ox = blockIdx.x * kFT, oy = (row0 + blockIdx.y) * kFT;
    const size_t plane = static_cast<size_t>(W) * H;
    const double* img = image + ch * plane;
    const double* tgt = target + ch * plane;
    const bool interior = ox >= kFH && oy >= kFH && ox + kFT + kFH <= W && oy + kFT + kFH <= H;
    // Horizontal pass of the 5 statistics (out-of-image taps are zero == skipped taps).
    for (int task = threadIdx.x; task < kFS * (kFT / kFR); task += blockDim.x) {
        const int r = task / (kFT / kFR), c0 = (task - r * (kFT / kFR)) * kFR;
        const int gy = oy - kFH + r;
        const bool row_in = gy >= 0 && gy < H;
        double acc[kFR][5] = {};
#pragma unroll
        for (int k = 0; k < kFR + 2 * kFH; ++k) {
            const int gx = ox - kFH + c0 + k;
            double xv = 0.0, tv = 0.0;
            if (interior || (row_in && gx >= 0 && gx < W)) {
                const size_t idx = static_cast<size_t>(gy) * W + gx;
                xv = __ldg(img + idx);
                tv = __ldg(tgt + idx);
            }
            const double p[5] = {xv, xv * xv, tv, tv * tv, xv * tv};
#pragma unroll
            for (int o = 0; o < kFR; ++o)
                if (k - o >= 0 && k - o <= 2 * kFH) {
                    const double wk = win.w[k - o];
#pragma unroll
                    for (int f = 0; f < 5; ++f) acc[o][f] += wk * p[f];
                }
        }
#pragma unroll
        for (int o = 0; o < kFR; ++o)
#pragma unroll
            for (int f = 0; f < 5; ++f) s_h[f][r][c0 + o] = acc[o][f];
    }
    __syncthreads();
    const int c = threadIdx.x % kFT, r0 = (threadIdx.x / kFT) * kFR;
    const int x = ox + c;
    double st[kFR][5];
#pragma unroll
    for (int f = 0; f < 5; ++f) {
        double o4[kFR];
        vpass32(win, false, s_h[f], c, r0, o4);
#pragma unroll
        for (int o = 0; o < kFR; ++o) st[o][f] = o4[o];
    }
    double ssim_own = 0.0;
    if (x < W) {
        const double nx = axis_norm(x, W, win);
#pragma unroll
        for (int o = 0; o < kFR; ++o) {
            const int y = oy + r0 + o;
            if (y >= H) break;
            const double inv_norm = 1.0 / (nx * axis_norm(y, H, win));
            if (!fields) {  // value-only path (metrics)
                if (y >= own_y0 && y < own_y1) ssim_own += ssim_value_only(st[o], inv_norm, c1, c2);
                continue;
            }
            double out[9];
            const double ss = ssim_centre_fields(st[o], inv_norm, c1, c2, out);
            if (y >= own_y0 && y < own_y1) ssim_own += ss;  // owned pixel rows (multi-GPU shard)
            const size_t idx = static_cast<size_t>(y) * W + x;
#pragma unroll
            for (int f = 0; f < 9; ++f) fields[(static_cast<size_t>(f) * 3 + ch) * plane + idx] = out[f];
        }
    }
    const double tot = block_sum(ssim_own, red);
    if (threadIdx.x == 0) exact_add(sums + kExactWords, tot);
}

// Horizontal pass of one staged derivative field: kFS rows x kHG groups of kHW outputs
// (252 tasks, one per thread; the last group overlaps its neighbour and both write the
// same values). W2 selects the weights at compile time (constant-bank operands).
template <bool W2>
__device__ __forceinline__ void hpass_field(const Window& win, const double (*s_fb)[kBS], double (*s_h0)[kFT + 1]) {
    for (int task = threadIdx.x; task < kFS * kHG; task += blockDim.x) {
        const int cg = task / kFS, r = task - cg * kFS, c0 = min(cg * kHW, kFT - kHW);
        double acc[kHW] = {};
#pragma unroll
        for (int k = 0; k < kHW + 2 * kFH; ++k) {
            const double v = s_fb[r][c0 + k + 1];
#pragma unroll
            for (int o = 0; o < kHW; ++o)
                if (k - o >= 0 && k - o <= 2 * kFH) acc[o] += (W2 ? win.w2[k - o] : win.w[k - o]) * v;
        }
#pragma unroll
        for (int o = 0; o < kHW; ++o) s_h0[r][c0 + o] = acc[o];
    }
}

__global__ void __launch_bounds__(256, NGS_SSIMD_MINB) ssim_derivs32_k(int W, int H, const double* __restrict__ image,
                                                       const double* __restrict__ target, Window win, double lambda,
                                                       const double* __restrict__ fields, float* __restrict__ grad,
                                                       float* __restrict__ hess, unsigned long long* __restrict__ sums, int row0,
                                                       int own_y0, int own_y1) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    auto s_h = reinterpret_cast<double (*)[kFS][kFT + 1]>(smem_raw);  // [1][kFS][kFT + 1], then s_f [2][kFS][kBS]
    __shared__ double red[8];
    __shared__ unsigned long long fbar[2];
    const int ch = blockIdx.z;
    const int ox = blockIdx.x * kFT, oy = (row0 + blockIdx.y) * kFT;
    const size_t plane = static_cast<size_t>(W) * H;
    const int c = threadIdx.x % kFT, r0 = (threadIdx.x / kFT) * kFR;
    const int x = ox + c;
    const double inv3n = 1.0 / (3.0 * static_cast<double>(plane));
    // The thread's own pixels are re-read where needed (L1) rather than held across the
    // nine rounds: registers go to the horizontal pass.
    auto pix = [&](const double* a, int o) {
        const int y = oy + r0 + o;
        return (x < W && y < H) ? __ldg(a + ch * plane + static_cast<size_t>(y) * W + x) : 0.0;
    };
    double g_ssim[kFR] = {}, h_ssim[kFR] = {};
    if (lambda != 0.0) {
        // One field per round, double-buffered: the halo tile of field f+1 streams in
        // while field f is convolved. Interior tiles (W even) move it as one TMA bulk copy
        // per row completing on an mbarrier; edge tiles per element (cp.async, zeros
        // outside the image). Horizontal tasks are row-major so a warp's lanes read
        // different rows.
        auto s_f = reinterpret_cast<double (*)[kFS][kBS]>(smem_raw + sizeof(double) * kFS * (kFT + 1));
        const bool bulk = (W % 2 == 0) && ox >= kFH + 1 && ox + kFT + kFH + 1 <= W && oy >= kFH &&
                          oy + kFT + kFH <= H;
        if (bulk) {
            if (threadIdx.x == 0) {
                mbar_init(&fbar[0], 1);
                mbar_init(&fbar[1], 1);
                mbar_fence_init();
            }
            __syncthreads();
        }
        auto issue = [&](int f, int buf) {
            const double* field = fields + (static_cast<size_t>(f) * 3 + ch) * plane;
            if (bulk) {
                if (threadIdx.x == 0) mbar_expect_tx(&fbar[buf], kFS * kBulkRow);
                if (threadIdx.x < kFS)
                    bulk_copy_g2s(&s_f[buf][threadIdx.x][0],
                                  field + static_cast<size_t>(oy - kFH + threadIdx.x) * W + (ox - kFH - 1), kBulkRow,
                                  &fbar[buf]);
                return;
            }
            for (int i = threadIdx.x; i < kFS * kFS; i += blockDim.x) {
                const int r = i / kFS, cc = i - r * kFS;
                const int gx = ox - kFH + cc, gy = oy - kFH + r;
                if (gx >= 0 && gx < W && gy >= 0 && gy < H)
                    cp_async8(&s_f[buf][r][cc + 1], field + static_cast<size_t>(gy) * W + gx);
                else
                    s_f[buf][r][cc + 1] = 0.0;
            }
            cp_async_commit_l();
        };
        issue(0, 0);
#pragma unroll 1
        for (int f = 0; f < 9; ++f) {
            const int buf = f & 1;
            if (bulk)
                mbar_wait(&fbar[buf], (f >> 1) & 1);
            else
                cp_async_wait_all_l();
            __syncthreads();  // tile f visible; previous round's readers of s_h and s_f[buf ^ 1] done
            if (f + 1 < 9) issue(f + 1, buf ^ 1);
            const bool w2 = f >= 4;  // fp, fq, fr, fkw use w; the rest w^2
            if (w2)
                hpass_field<true>(win, s_f[buf], s_h[0]);
            else
                hpass_field<false>(win, s_f[buf], s_h[0]);
            __syncthreads();
            const bool need_c = f == 2 || f == 5 || f == 7 || f == 8, need_t = f == 1 || f == 6 || f == 7;
            double cv[kFR], ctv[kFR];
#pragma unroll
            for (int o = 0; o < kFR; ++o) {
                cv[o] = need_c ? pix(image, o) : 0.0;
                ctv[o] = need_t ? pix(target, o) : 0.0;
            }
            double sv[kFR];
            if (w2)
                vpass32(win, true, s_h[0], c, r0, sv);
            else
                vpass32(win, false, s_h[0], c, r0, sv);
#pragma unroll
            for (int o = 0; o < kFR; ++o) {  // loss.hpp:323-327
                const double cf = f == 1 ? ctv[o] : f == 2 ? cv[o] : f == 5 ? cv[o] : f == 6 ? ctv[o]
                                : f == 7 ? cv[o] * ctv[o] : f == 8 ? cv[o] * cv[o] : 1.0;
                if (f < 3) g_ssim[o] += cf * sv[o];
                else h_ssim[o] += cf * sv[o];
            }
        }
    }
    double dsq_own = 0.0;
#pragma unroll
    for (int o = 0; o < kFR; ++o) {
        const int y = oy + r0 + o;
        if (x >= W || y >= H) continue;
        const double d = pix(image, o) - pix(target, o);
        if (y >= own_y0 && y < own_y1) dsq_own += d * d;
        double gg = inv3n * d, hh = inv3n;
        if (lambda != 0.0) {
            gg += lambda * (-inv3n * g_ssim[o]);
            hh += lambda * (-inv3n * h_ssim[o]);
        }
        const size_t idx = ch * plane + static_cast<size_t>(y) * W + x;
        grad[idx] = static_cast<float>(gg);
        hess[idx] = static_cast<float>(hh);
    }
    const double tot = block_sum(dsq_own, red);
    if (threadIdx.x == 0) exact_add(sums, tot);
}

// gaussian_window_1d, loss.hpp:66-77
Window make_window(const LossParams& L) {
    Window win{};
    win.half = L.window / 2;
    double sum = 0;
    for (int i = 0; i < L.window; ++i) {
        const double d = i - win.half;
        win.w[i] = std::exp(-d * d / (2.0 * L.window_sigma * L.window_sigma));
        sum += win.w[i];
    }
    for (int i = 0; i < L.window; ++i) {
        win.w[i] /= sum;
        win.w2[i] = win.w[i] * win.w[i];
    }
    win.full = 0;
    for (int i = 0; i < L.window; ++i) win.full += win.w[i];  // axis_norm's order: i0 = -half .. half
    return win;
}

}  // namespace

void compute_loss(ViewSlot& v, cudaStream_t s) {
    const LossParams& L = v.loss;
    if (L.lambda < 0.0) throw Error(NGS_ERR_INVALID_INPUT, "loss: lambda must be >= 0");
    if (L.window < 3 || L.window % 2 == 0) throw Error(NGS_ERR_INVALID_INPUT, "loss: window must be odd and >= 3");
    if (L.window > 2 * kMaxHalf + 1) throw Error(NGS_ERR_INVALID_INPUT, "loss: window larger than 21 unsupported");
    const bool ssim = L.lambda != 0.0;
    if (ssim && (v.W < L.window || v.H < L.window))
        throw Error(NGS_ERR_INVALID_INPUT, "ssim stats: image smaller than the filter window");
    const Window win = make_window(L);
    const size_t npx = static_cast<size_t>(v.W) * v.H;
    v.loss_grad.ensure(3 * npx);
    v.loss_hess.ensure(3 * npx);
    v.loss_sums.ensure(2 * kExactWords);
    CUDA_CHECK(cudaMemsetAsync(v.loss_sums.ptr, 0, 2 * kExactWords * sizeof(unsigned long long), s));
    // Shard bands are in tile rows of the view's tile size; the loss grid uses 16-row blocks.
    const int t = v.cam.tile;
    const int band_px0 = std::max(0, v.raster.band_y0) * t, band_px1 = std::min(v.H, v.raster.band_y1 * t);
    const int own0 = std::max(0, v.raster.own_y0) * t, own1 = std::min(v.H, v.raster.own_y1 * t);
    const int row0 = band_px0 / kLT, row1 = (band_px1 + kLT - 1) / kLT;
    if (row1 <= row0) return;
    const dim3 grid((v.W + kLT - 1) / kLT, row1 - row0, 3);
    StageScope st(NGS_STAGE_LOSS, s, ssim ? 2 : 1);
    auto run = [&](auto fields_kernel, auto derivs_kernel) {
        if (ssim) {
            v.fields.ensure(27 * npx);
            fields_kernel<<<grid, 256, 0, s>>>(v.W, v.H, v.image.ptr, v.target_ptr(), win, L.c1, L.c2, v.fields.ptr,
                                               v.loss_sums.ptr, row0, own0, own1);
            CUDA_LAUNCH_CHECK();
        }
        derivs_kernel<<<grid, 256, 0, s>>>(v.W, v.H, v.image.ptr, v.target_ptr(), win, L.lambda,
                                           ssim ? v.fields.ptr : nullptr, v.loss_grad.ptr, v.loss_hess.ptr,
                                           v.loss_sums.ptr, row0, own0, own1);
        CUDA_LAUNCH_CHECK();
    };
    if (win.half == kFH) {  // the reference default (window 11): 32x32 register-blocked tiles
        const int r32a = band_px0 / kFT, r32b = (band_px1 + kFT - 1) / kFT;
        const dim3 g32((v.W + kFT - 1) / kFT, r32b - r32a, 3);
        const size_t sm_f = sizeof(double) * 5 * kFS * (kFT + 1), sm_d = sizeof(double) * kFS * (kFT + 1 + 2 * kBS);
        ensure_dynamic_smem(reinterpret_cast<const void*>(ssim_fields32_k), sm_f);
        ensure_dynamic_smem(reinterpret_cast<const void*>(ssim_derivs32_k), sm_d);
        if (ssim) {
            v.fields.ensure(27 * npx);
            ssim_fields32_k<<<g32, 256, sm_f, s>>>(v.W, v.H, v.image.ptr, v.target_ptr(), win, L.c1, L.c2, v.fields.ptr,
                                                   v.loss_sums.ptr, r32a, own0, own1);
            CUDA_LAUNCH_CHECK();
        }
        ssim_derivs32_k<<<g32, 256, ssim ? sm_d : 0, s>>>(v.W, v.H, v.image.ptr, v.target_ptr(), win, L.lambda,
                                                           ssim ? v.fields.ptr : nullptr, v.loss_grad.ptr,
                                                           v.loss_hess.ptr, v.loss_sums.ptr, r32a, own0, own1);
        CUDA_LAUNCH_CHECK();
    } else {
        run(ssim_fields_k<0>, ssim_derivs_k<0>);
    }
}

void compute_loss_value(ViewSlot& v, cudaStream_t s) {
    // Value-only evaluation of the whole image: sums[0] = sum (c - c^t)^2, sums[1] =
    // sum of the per-pixel SSIM over channels (always, for ssim_metric).
    const LossParams& L = v.loss;
    if (L.window < 3 || L.window % 2 == 0) throw Error(NGS_ERR_INVALID_INPUT, "loss: window must be odd and >= 3");
    if (L.window > 2 * kMaxHalf + 1) throw Error(NGS_ERR_INVALID_INPUT, "loss: window larger than 21 unsupported");
    if (v.W < L.window || v.H < L.window)
        throw Error(NGS_ERR_INVALID_INPUT, "ssim stats: image smaller than the filter window");
    const Window win = make_window(L);
    const size_t npx = static_cast<size_t>(v.W) * v.H;
    v.loss_sums.ensure(2 * kExactWords);
    CUDA_CHECK(cudaMemsetAsync(v.loss_sums.ptr, 0, 2 * kExactWords * sizeof(unsigned long long), s));
    StageScope st(NGS_STAGE_LOSS, s, 2);
    l2_sum_k<<<std::min<size_t>((3 * npx + 255) / 256, 4 * 148), 256, 0, s>>>(v.image.ptr, v.target_ptr(), 3 * npx,
                                                                           v.loss_sums.ptr);
    CUDA_LAUNCH_CHECK();
    if (win.half == kFH) {
        const dim3 g32((v.W + kFT - 1) / kFT, (v.H + kFT - 1) / kFT, 3);
        const size_t sm_f = sizeof(double) * 5 * kFS * (kFT + 1);
        ensure_dynamic_smem(reinterpret_cast<const void*>(ssim_fields32_k), sm_f);
        ssim_fields32_k<<<g32, 256, sm_f, s>>>(v.W, v.H, v.image.ptr, v.target_ptr(), win, L.c1, L.c2, nullptr,
                                               v.loss_sums.ptr, 0, 0, v.H);
    } else {
        const dim3 grid((v.W + kLT - 1) / kLT, (v.H + kLT - 1) / kLT, 3);
        ssim_fields_k<0><<<grid, 256, 0, s>>>(v.W, v.H, v.image.ptr, v.target_ptr(), win, L.c1, L.c2, nullptr,
                                              v.loss_sums.ptr, 0, 0, v.H);
    }
    CUDA_LAUNCH_CHECK();
}

}  // namespace ngsb
