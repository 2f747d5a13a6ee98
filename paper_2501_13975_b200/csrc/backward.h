// backward.h — K8 backward-pass interface shared by backward.cu and the host.
#pragma once

#include "context.h"

namespace ngsb {

// kPassPositionUV is the position pass the solvers use: derivatives are taken
// along the two in-plane directions u_x, u_y of build_position_subspace
// (newton.hpp:130-139) instead of the world axes. The 2x2 system
// U^T (sum_v H_v) U = sum_v U^T H_v U is linear in the per-record terms, so the
// accumulators hold the projected system directly (5 instead of 9 components).
// kPassPosition (world axes) serves ngs_accumulate, which returns the 3x3 terms.
// kPassGrad: first-order baselines (first_order_step, trainer.hpp:419-509): per
// record only image-space quantities are accumulated (dL/dpi, dL/dSigma, dL/dc~,
// dL/dsigma); the per-Gaussian chain to (p, theta, s, sigma, SH) runs once in
// the update kernel.
enum PassId { kPassPosition = 0, kPassRotation = 1, kPassScaling = 2, kPassOpacityColor = 3, kPassPositionUV = 4,
              kPassGrad = 5 };

// Accumulator components per pass (FP64, component-major [c][N]).
constexpr int kAccPosition = 9;  // grad 3, hess sym (xx, xy, xz, yy, yz, zz)
constexpr int kAccPositionUV = 5;  // grad (u_x, u_y), hess (xx, xy, yy) in the subspace
constexpr int kAccRotation = 2;  // grad, hess
constexpr int kAccScaling = 5;   // grad 2, hess (00, 01, 11)
constexpr int kAccOpColor = 8;   // opacity grad, hess; colour g_acc[3], h_acc[3] (per view)
constexpr int kAccGrad = 9;      // dL/dpi (2), dL/dSigma (00, 01, 11), dL/dc~ (3), dL/dsigma

// Per-(Gaussian, view) constant layouts (floats, AoS per Gaussian, float4-aligned
// groups). ND derivative directions (3 world axes, or the 2 subspace directions);
// symmetric pairs (c, d), c <= d, packed row by row ((00, 01, 02, 11, 12, 22) for ND = 3).
template <int ND>
struct PosLayout {
    static constexpr int NP = ND * (ND + 1) / 2;
    __host__ __device__ static constexpr int a4(int x) { return (x + 3) & ~3; }
    static constexpr int JS = 0;                  // J columns (Jx_c, Jy_c) xND, then dSigma/dp_c (a, b, c) xND
    static constexpr int HPI = JS + a4(5 * ND);   // d2pi/dp_c dp_d: (x, y) per pair
    static constexpr int SCD = HPI + a4(2 * NP);  // d2Sigma/dp_c dp_d: (a, b, c) per pair
    static constexpr int JC = SCD + a4(3 * NP);   // dc~_ch/dp: ND per channel (channel-major)
    static constexpr int HC = JC + a4(3 * ND);    // d2c~_ch/dp2: NP per channel
    static constexpr int N = HC + a4(3 * NP);
    // Entry indices. ND = 3 keeps the natural order; ND = 2 stores each quantity as
    // a (direction 0, direction 1) or (00, 11) pair in adjacent floats so the record
    // evaluation runs on packed f32x2 arithmetic (position_record_uv).
    __host__ __device__ static constexpr int jx(int q) { return ND == 2 ? JS + q : JS + 2 * q; }
    __host__ __device__ static constexpr int jy(int q) { return ND == 2 ? JS + 2 + q : JS + 2 * q + 1; }
    __host__ __device__ static constexpr int sg(int q, int e) { return ND == 2 ? JS + 4 + 2 * e + q : JS + 2 * ND + 3 * q + e; }
    __host__ __device__ static constexpr int hpi(int pp, int e) {
        return ND == 2 ? (pp == 1 ? HPI + 4 + e : HPI + 2 * e + (pp == 2)) : HPI + 2 * pp + e;
    }
    __host__ __device__ static constexpr int scd(int pp, int e) {
        return ND == 2 ? (pp == 1 ? SCD + 6 + e : SCD + 2 * e + (pp == 2)) : SCD + 3 * pp + e;
    }
    __host__ __device__ static constexpr int jc(int ch, int q) { return JC + ND * ch + q; }
    __host__ __device__ static constexpr int hc(int ch, int pp) {
        return ND == 2 ? (pp == 1 ? HC + 6 + ch : HC + 2 * ch + (pp == 2)) : HC + NP * ch + pp;
    }
};
constexpr int kPosConsts = PosLayout<3>::N;    // 80
constexpr int kPosUVConsts = PosLayout<2>::N;  // 52
static_assert(kPosConsts == 80 && kPosUVConsts == 52, "position constant layout");
constexpr int kRotConsts = 8;    // s1 (00, 01, 11), s2 (00, 01, 11), pad 2
constexpr int kScaleConsts = 8;  // v0 (2), v1 (2), m00, m01, m11, pad

struct BackwardArgs {
    int tiles_x, W, H;
    int tile0;  // first tile of the owned band
    const int2* ranges;
    const int* vals;
    const double2* pix;
    const float4* ra;
    const float4* rb;
    const float4* rc;
    const double* image;
    const int* last;
    const float* loss_grad;
    const float* loss_hess;
    const float* consts;
    // Chunked traversal (8x8 tiles): block = (tile, chunk); chunk c > 0 starts from the
    // forward's checkpoint c (ck_t / ck_p, see ViewSlot). chunks == 1: whole lists.
    int chunks;
    const float* ck_t;
    const double* ck_p;
    float cutoff;
    float bg[3];
    double* acc;
    size_t acc_stride;
    unsigned long long* acc_limbs;  // deterministic mode: exact fixed-point limbs [comp][stride][4] (acc unused)
    uint8_t* visible;                    // optional: set to 1 for kernels with >= 1 record
    unsigned long long* contrib_pairs;   // optional: count of contributing (pixel, splat) records
    int* err;                            // device error flag (kErrFixedRange in deterministic mode)
};

#ifdef NGS_COUNT_CANDIDATES
void dump_candidates();  // debug build: phase-1 candidate statistics
#endif

// Up to kBackwardBatch views of one pass in one launch (launch_backward_batch).
constexpr int kBackwardBatch = 4;
struct BackwardBatch {
    int nv;
    int block_end[kBackwardBatch];
    BackwardArgs a[kBackwardBatch];
};

void compute_pass_consts(int pass, const SceneDev& scene, ViewSlot& v, const CameraDev& primary, cudaStream_t s,
                         float* out = nullptr);  // out: destination (default v.consts)
// Deterministic accumulation: each FP32 partial is converted exactly to a 128-bit
// two's-complement fixed-point number (binary point 2^-88) and added as four
// 32-bit chunks into four 64-bit counters with integer atomics. Integer addition
// is associative, so the sums do not depend on the order in which blocks finish;
// limbs_to_double normalises the carries and rounds once (correctly) to FP64.
// Non-finite or |x| >= 2^38 partials set kErrFixedRange instead of being added.
constexpr int kLimbShift = 88;
void limbs_to_double(const unsigned long long* limbs, double* acc, size_t count, cudaStream_t s);
// Multi-GPU exchange payload: the FP64 accumulators travel as FP32 (half the bytes; the
// cross-rank sum of world FP32-rounded partials stays ~1e-7 relative).
void acc_to_f32(const double* acc, float* out, size_t count, cudaStream_t s);
void acc_from_f32(const float* in, double* acc, size_t count, cudaStream_t s);

void launch_backward(int pass, const SceneDev& scene, ViewSlot& v, double* acc, size_t acc_stride, uint8_t* visible,
                     unsigned long long* contrib_pairs, cudaStream_t s, unsigned long long* acc_limbs = nullptr,
                     int* err = nullptr, int primary_tag = -1);
// The same for nv <= kBackwardBatch views with the same tile size in ONE launch (the small
// secondary views of a pass); per-view accumulator and counter pointers.
void launch_backward_batch(int pass, const SceneDev& scene, ViewSlot* const* views, int nv, double* const* acc,
                           size_t acc_stride, uint8_t* visible, unsigned long long* contrib_pairs, cudaStream_t s,
                           unsigned long long* const* acc_limbs, int* err);

}  // namespace ngsb
