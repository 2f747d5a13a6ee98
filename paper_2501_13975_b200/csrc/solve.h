// solve.h — K9 solve + commit interface.
#pragma once

#include "context.h"

namespace ngsb {

constexpr int kMaxSolveViews = 16;  // primary + up to 15 secondary views per step (reference knn has no cap)

// NewtonOptions (newton.hpp:58-68) plus commit flag and FP32 opacity bounds.
struct SolveParams {
    double mu_min, eig_floor_rel, step_cap_factor, scale_cap_factor, color_cap, theta_cap, barrier_weight;
    int max_backtrack;
    double eigengap_rel;
    int commit;
    float sigma_lo, sigma_hi;  // FP32 images of nextafter(1e-4, 1), nextafter(1 - 1e-4, 0)
};

struct SolveOutputs {
    double* delta;        // optional, layout of ngs_solve_result::delta
    uint8_t* accepted;    // optional
    uint8_t* degenerate;  // optional
    unsigned long long* norm_sq;  // required: exact (kExactWords) accumulator of the report's delta norm
    int* err;             // device error bits
};

// Per-view data the colour solve needs (views of the current step).
struct ColorViews {
    int n_views;
    CameraDev cam[kMaxSolveViews];
    const uint8_t* flags[kMaxSolveViews];
    double* eig;  // colour-solve scratch: (MV^2 + MV) doubles per Gaussian (Gram eigen-decomposition)
    int fused;    // 1: one-launch colour solve with the no-repair fast path (no eig scratch)
    unsigned long long* fast_count;  // optional: channel solves that took the fast path
};

// First-order baselines (first_order_step, trainer.hpp:419-509).
struct FirstOrderParams {
    int adam;               // 0: gd_update (trainer.hpp:104), 1: AdamState::update (trainer.hpp:106-122)
    double lr[5];           // indexed by ngs_attribute
    int t;                  // Adam step count after begin_step
    double beta1, beta2, eps;
    float sigma_lo, sigma_hi;
};
// Chains the image-space accumulators (kPassGrad) of the primary view to
// (p, theta, s, sigma, SH) gradients and applies GD or Adam to every Gaussian.
// pos_consts: PosLayout<3> constants of the view; rot_consts: rotation constants
// with this view's ray as axis; adam_m / adam_v: [56][stride] doubles (slot-major).
void launch_first_order(const SceneDev& scene, const CameraDev& cam, const uint8_t* flags, const float* pos_consts,
                        const float* rot_consts, const double* acc, size_t stride, const FirstOrderParams& p,
                        double* adam_m, double* adam_v, unsigned long long* norms, int* err, cudaStream_t s);

void launch_solve(int attr, const SceneDev& scene, const CameraDev& primary, double lambda_lp,
                  const uint8_t* primary_flags, const ColorViews& cv, const SolveParams& sp, const double* acc,
                  size_t stride, const SolveOutputs& out, cudaStream_t s);

}  // namespace ngsb
