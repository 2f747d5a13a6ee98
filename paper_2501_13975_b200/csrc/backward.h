// backward.h — K8 backward-pass interface shared by backward.cu and the host.
#pragma once

#include "context.h"

namespace ngsb {

enum PassId { kPassPosition = 0, kPassRotation = 1, kPassScaling = 2, kPassOpacityColor = 3 };

// Accumulator components per pass (FP64, component-major [c][N]).
constexpr int kAccPosition = 9;  // grad 3, hess sym (xx, xy, xz, yy, yz, zz)
constexpr int kAccRotation = 2;  // grad, hess
constexpr int kAccScaling = 5;   // grad 2, hess (00, 01, 11)
constexpr int kAccOpColor = 8;   // opacity grad, hess; colour g_acc[3], h_acc[3] (per view)

// Per-(Gaussian, view) constant layouts (floats, AoS per Gaussian, float4-aligned
// groups). Symmetric 3x3 pairs (c, d) are packed (00, 01, 02, 11, 12, 22).
constexpr int kPosJS = 0;    // J columns (Jx_c, Jy_c) x3, then dSigma/dp_c (a, b, c) x3   [15 + 1 pad]
constexpr int kPosHpi = 16;  // d2pi/dp_c dp_d: (x, y) per pair                            [12]
constexpr int kPosScd = 28;  // d2Sigma/dp_c dp_d: (a, b, c) per pair                      [18 + 2 pad]
constexpr int kPosJc = 48;   // dc~_ch/dp: 3 per channel, padded to 4                       [12]
constexpr int kPosJJ = 60;   // Jc_ch Jc_ch^T: 6 per channel                                [18]
constexpr int kPosHc = 78;   // d2c~_ch/dp2: 6 per channel                                  [18]
constexpr int kPosConsts = 96;
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
    float cutoff;
    float bg[3];
    double* acc;
    size_t acc_stride;
    uint8_t* visible;                    // optional: set to 1 for kernels with >= 1 record
    unsigned long long* contrib_pairs;   // optional: count of contributing (pixel, splat) records
};

void compute_pass_consts(int pass, const SceneDev& scene, ViewSlot& v, const CameraDev& primary, cudaStream_t s);
void launch_backward(int pass, const SceneDev& scene, ViewSlot& v, double* acc, size_t acc_stride, uint8_t* visible,
                     unsigned long long* contrib_pairs, cudaStream_t s);

}  // namespace ngsb
