// solve.h — K9 solve + commit interface.
#pragma once

#include "context.h"

namespace ngsb {

constexpr int kMaxSolveViews = 8;  // primary + up to 7 secondary views per step

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
    double* norm_sq;      // required: device accumulator of the report's delta norm
    int* err;             // device error bits
};

// Per-view data the colour solve needs (views of the current step).
struct ColorViews {
    int n_views;
    CameraDev cam[kMaxSolveViews];
    const uint8_t* flags[kMaxSolveViews];
};

void launch_solve(int attr, const SceneDev& scene, const CameraDev& primary, double lambda_lp,
                  const uint8_t* primary_flags, const ColorViews& cv, const SolveParams& sp, const double* acc,
                  size_t stride, const SolveOutputs& out, cudaStream_t s);

}  // namespace ngsb
