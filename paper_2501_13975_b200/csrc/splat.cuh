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

__device__ __forceinline__ SplatEval eval_splat(float px, float py, float qa, float qb, float qc, float sigma,
                                                float x, float y) {
    SplatEval e;
    e.dx = __fsub_rn(px, x);
    e.dy = __fsub_rn(py, y);
    e.qd0 = __fmaf_rn(qa, e.dx, __fmul_rn(qb, e.dy));
    e.qd1 = __fmaf_rn(qb, e.dx, __fmul_rn(qc, e.dy));
    const float q = __fmaf_rn(e.dx, e.qd0, __fmul_rn(e.dy, e.qd1));
    e.g = expf(__fmul_rn(-0.5f, q));  // full-accuracy exp: the image feeds cancelling (c - c^t) terms
    e.alpha = __fmul_rn(e.g, sigma);
    return e;
}

// T <- T * (1 - alpha), C <- C + T * alpha * c (rasterizer.hpp:287-288).
__device__ __forceinline__ float blend_weight(float t, float alpha) { return __fmul_rn(t, alpha); }
__device__ __forceinline__ float next_transmittance(float t, float alpha) {
    return __fmul_rn(t, __fsub_rn(1.0f, alpha));
}

}  // namespace ngsb
