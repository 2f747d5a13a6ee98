// splat.cuh — the FP32 per-(pixel, splat) Gaussian evaluation shared by the
// forward rasterizer and every backward pass.
//
// The backward passes re-traverse each tile's depth-ordered list and must make
// exactly the same alpha-cutoff / transmittance decisions as the forward pass
// (rasterizer.hpp:274-292). All arithmetic here therefore uses explicit
// round-to-nearest intrinsics, so the compiler cannot contract the two call
// sites differently and the recomputed alpha and T are bit-identical.
#pragma once

#include "common.cuh"

namespace ngsb {

struct SplatEval {
    float dx, dy;    // d = pi - x
    float qd0, qd1;  // Q d
    float g;         // G = exp(-1/2 d^T Q d)      (rasterizer.hpp:108-110)
    float alpha;     // G * sigma
};

// Quadratic-form bound beyond which alpha = sigma * exp(-q/2) is certainly
// below the cutoff: q > 2 ln(sigma / cutoff) + margin. The margin absorbs the
// rounding of logf/expf, so rejecting on it never changes a decision the full
// evaluation would make (forward and backward stay bit-identical).
// Pixel <-> thread map of a tile block: each warp owns an 8x4 pixel box (two
// boxes across a 16-wide tile), tighter than a 16x2 strip for the warp-level
// overlap masks built below.
template <int TILE, int BH_ = 4>
struct WarpBoxT {
    static constexpr int BW = 8, BH = BH_, ACROSS = TILE / BW, NW = TILE * TILE / (BW * BH);
    __device__ static void pixel(int tid, int& lx, int& ly) {
        const int warp = tid >> 5, lane = tid & 31;
        lx = (warp % ACROSS) * BW + (lane % BW);
        ly = (warp / ACROSS) * BH + lane / BW;
    }
    // Bit w set when the cutoff ellipse's bounding box [px -+ ex] x [py -+ ey] (tile
    // coordinates) reaches a pixel centre of warp w's box.
    __device__ static unsigned mask(float px, float py, float ex, float ey) {
        unsigned m = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const float x0 = (w % ACROSS) * BW + 0.5f, y0 = (w / ACROSS) * BH + 0.5f;
            if (!(px + ex < x0 || px - ex > x0 + (BW - 1) || py + ey < y0 || py - ey > y0 + (BH - 1))) m |= 1u << w;
        }
        return m;
    }
    // As mask(), then refined by the exact minimum of the quadratic form q over the
    // box: q(d) = qa dx^2 + 2 qb dx dy + qc dy^2 is convex, so unless the centre lies
    // in the box its minimum is on one of the four edges (1-D minimisation, clamped).
    // qmax already carries the reject bound's margin (> 1e-3 in q, far above the FP32
    // rounding here), so a dropped box never holds a pixel with alpha >= cutoff.
    __device__ static unsigned mask_exact(float px, float py, float ex, float ey, float qa, float qb, float qc,
                                          float qmax) {
        const unsigned m0 = mask(px, py, ex, ey);
        if (!(qmax < 3.0e38f)) return m0;  // no cutoff (reference mode): keep the bounding-box test
        const float ia = 1.0f / qa, ic = 1.0f / qc;
        unsigned m = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            if (!((m0 >> w) & 1u)) continue;
            const float x0 = (w % ACROSS) * BW + 0.5f - px, x1 = x0 + (BW - 1);
            const float y0 = (w / ACROSS) * BH + 0.5f - py, y1 = y0 + (BH - 1);
            if (x0 <= 0.f && x1 >= 0.f && y0 <= 0.f && y1 >= 0.f) {
                m |= 1u << w;
                continue;
            }
            auto qf = [&](float dx, float dy) { return qa * dx * dx + 2.f * qb * dx * dy + qc * dy * dy; };
            auto ex_ = [&](float dx) { return qf(dx, fminf(fmaxf(-qb * dx * ic, y0), y1)); };
            auto ey_ = [&](float dy) { return qf(fminf(fmaxf(-qb * dy * ia, x0), x1), dy); };
            const float qmin = fminf(fminf(ex_(x0), ex_(x1)), fminf(ey_(y0), ey_(y1)));
            if (qmin <= qmax) m |= 1u << w;
        }
        return m;
    }
};

template <int TILE>
using WarpBox = WarpBoxT<TILE, 4>;

// Half-extents of the cutoff ellipse {q <= qmax}: |dx| <= sqrt(qmax Sigma00),
// |dy| <= sqrt(qmax Sigma11); widened so the warp-level skip never drops a
// splat the per-pixel test would keep.
__device__ __forceinline__ float ellipse_half_extent(float qmax, float var) {
    return sqrtf(fmaxf(qmax, 0.f) * var) * 1.0001f + 1e-3f;
}

// cp.async (LDGSTS): 16-byte global -> shared copies without register staging.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// TMA bulk copies (cp.async.bulk, UBLKCP) completing on an mbarrier: one instruction
// moves a whole contiguous row (16-byte aligned, size a multiple of 16).
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile(
        "{\n .reg .pred P;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared.b64 P, [%0], %1;\n"
        " @!P bra WAIT_%=;\n}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_copy_g2s(void* smem, const void* gmem, unsigned bytes, unsigned long long* bar) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(d),
                 "l"(gmem), "r"(bytes), "r"(b)
                 : "memory");
}

__device__ __forceinline__ float reject_bound(float sigma, float cutoff) {
    return cutoff > 0.f ? 2.0f * logf(sigma / cutoff) + 1e-2f : __int_as_float(0x7f800000);
}

// A splat as staged in shared memory for a tile batch: one 48-byte record so
// every visit is a single broadcast base address.
// First list index of chunk c of a tile's list [range.x, range.y) split into `chunks`
// near-equal parts (c = chunks gives range.y): the chunked backward's block split.
__device__ __forceinline__ int chunk_begin(int2 range, int c, int chunks) {
    return range.x + static_cast<int>(static_cast<long long>(range.y - range.x) * c / chunks);
}

struct SplatSh {
    float4 g0;  // (px, py, Q00, Q01) in tile coordinates
    float4 g1;  // (Q11, sigma, qmax, c0)
    float2 g2;  // (c1, c2)
    float2 pad;
};

// exp(-q/2) = 2^(-q log2(e) / 2) on the SFU (MUFU.EX2, ~2 ulp). Forward and
// backward call the same instruction sequence, so alpha stays bit-identical.
__device__ __forceinline__ float exp_neg_half(float q) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__fmul_rn(q, -0.72134752044448170368f)));
    return r;
}

// Branch-free evaluation: every lane computes G and alpha; returns whether the
// (pixel, splat) pair composites (q within the reject bound and alpha >= cutoff).
__device__ __forceinline__ bool eval_splat_bf(const SplatSh& sp, float x, float y, float cutoff, SplatEval& e) {
    e.dx = __fsub_rn(sp.g0.x, x);
    e.dy = __fsub_rn(sp.g0.y, y);
    e.qd0 = __fmaf_rn(sp.g0.z, e.dx, __fmul_rn(sp.g0.w, e.dy));
    e.qd1 = __fmaf_rn(sp.g0.w, e.dx, __fmul_rn(sp.g1.x, e.dy));
    const float q = __fmaf_rn(e.dx, e.qd0, __fmul_rn(e.dy, e.qd1));
    e.g = exp_neg_half(q);
    e.alpha = __fmul_rn(e.g, sp.g1.y);
    return q <= sp.g1.z && !(e.alpha < cutoff);
}

// eval_splat_bf for two pixels of one column (x, y0) and (x, y1) on packed f32x2
// arithmetic: each half of FFMA2 / FMUL2 / FADD2 rounds exactly like the scalar op, so
// both results are bit-identical to eval_splat_bf (the backward recomputes them that way).
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void unpk2(unsigned long long v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ unsigned long long fma2rn(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ unsigned long long mul2rn(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ void eval_splat_bf2(const SplatSh& sp, float x, float y0, float y1, float cutoff,
                                               SplatEval& e0, SplatEval& e1, bool& c0, bool& c1) {
    const float dx = __fsub_rn(sp.g0.x, x);
    const float dy0 = __fsub_rn(sp.g0.y, y0), dy1 = __fsub_rn(sp.g0.y, y1);
    const unsigned long long DX = pk2(dx, dx), DY = pk2(dy0, dy1);
    const unsigned long long qd0 = fma2rn(pk2(sp.g0.z, sp.g0.z), DX, mul2rn(pk2(sp.g0.w, sp.g0.w), DY));
    const unsigned long long qd1 = fma2rn(pk2(sp.g0.w, sp.g0.w), DX, mul2rn(pk2(sp.g1.x, sp.g1.x), DY));
    const unsigned long long q = fma2rn(DX, qd0, mul2rn(DY, qd1));
    float q0, q1;
    unpk2(q, q0, q1);
    e0.dx = e1.dx = dx;
    e0.dy = dy0;
    e1.dy = dy1;
    unpk2(qd0, e0.qd0, e1.qd0);
    unpk2(qd1, e0.qd1, e1.qd1);
    e0.g = exp_neg_half(q0);
    e1.g = exp_neg_half(q1);
    e0.alpha = __fmul_rn(e0.g, sp.g1.y);
    e1.alpha = __fmul_rn(e1.g, sp.g1.y);
    c0 = q0 <= sp.g1.z && !(e0.alpha < cutoff);
    c1 = q1 <= sp.g1.z && !(e1.alpha < cutoff);
}

// T <- T * (1 - alpha), C <- C + T * alpha * c (rasterizer.hpp:287-288).
__device__ __forceinline__ float blend_weight(float t, float alpha) { return __fmul_rn(t, alpha); }
__device__ __forceinline__ float next_transmittance(float t, float alpha) {
    return __fmul_rn(t, __fsub_rn(1.0f, alpha));
}

}  // namespace ngsb
