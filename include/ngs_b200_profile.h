/*
 * ngs_b200_profile.h — measurement hooks of libngs_b200.so (not part of the
 * reference-facing boundary in ngs_b200.h; used by bench.py).
 *
 * When profiling is enabled every kernel launch of the context is bracketed by
 * CUDA events on the context's stream and the 1+K views of a step run
 * serialised (so per-launch times do not overlap); ngs_profile_read resolves
 * them into per-stage device time. Counters (launches, contributing pairs)
 * are always on.
 */
#ifndef NGS_B200_PROFILE_H
#define NGS_B200_PROFILE_H

#include <stdint.h>

#include "ngs_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

enum {
    NGS_STAGE_PROJECT = 0,     /* K1 */
    NGS_STAGE_SORT = 1,        /* K2-K5: depth sort, pair emission, tile sort, ranges */
    NGS_STAGE_RASTER = 2,      /* K6 forward */
    NGS_STAGE_LOSS = 3,        /* K7 */
    NGS_STAGE_CONSTS = 4,      /* per-pass per-Gaussian constants */
    NGS_STAGE_BWD_POSITION = 5,/* K8 */
    NGS_STAGE_BWD_ROTATION = 6,
    NGS_STAGE_BWD_SCALING = 7,
    NGS_STAGE_BWD_OPACITY_COLOR = 8,
    NGS_STAGE_SOLVE = 9,       /* K9 solves + commits (all attributes) */
    NGS_STAGE_OTHER = 10,      /* memsets, copies */
    NGS_STAGE_COUNT = 11
};

typedef struct {
    double ms[NGS_STAGE_COUNT];             /* summed device time per stage (profiling on) */
    int64_t launches[NGS_STAGE_COUNT];      /* kernel launches per stage */
    int64_t total_launches;                 /* all kernel launches (always counted) */
    int64_t contrib_pairs[4];               /* contributing (pixel, splat) records per backward pass */
    int64_t raster_pairs;                   /* (tile, splat) pairs binned, summed over renders */
    int64_t renders;                        /* view renders */
    /* Trainer steps only, always on: wall time of each stage group on the
     * context stream as executed (views concurrent): render+loss of all
     * views, the four backward passes (incl. constants and all-reduce), solves. */
    double group_ms[6];
    /* Multi-GPU exchange (always counted): NCCL all-reduce calls issued by this rank
     * and their payload bytes (accumulators, overflow votes). */
    int64_t allreduce_calls;
    int64_t allreduce_bytes;
    /* The primary view's backward launch of each pass alone (the dominant kernel of the
     * step): summed device time (profiling on) and contributing records (always). */
    double primary_bwd_ms[4];
    int64_t primary_contrib_pairs[4];
    /* Colour solves (SH degree >= 1, always counted): channel systems solved, and those
     * that took the no-repair fast path (no eigen-decomposition, solve.cu). */
    int64_t color_channels;
    int64_t color_fast_channels;
} ngs_profile_stats;

/* Timeline of the concurrent schedule (views NOT serialised): one row per stage
 * bracket (a kernel or a short kernel sequence) with its stream and device times in
 * ms relative to the first bracket recorded after ngs_profile_timeline(ctx, 1). */
typedef struct {
    int32_t stage;
    int32_t stream;  /* opaque stream id */
    float start_ms, end_ms;
} ngs_timeline_row;
int32_t ngs_profile_timeline(ngs_context* ctx, int32_t on);
int32_t ngs_profile_read_timeline(ngs_context* ctx, ngs_timeline_row* rows, int32_t capacity, int32_t* n_rows);

int32_t ngs_profile_enable(ngs_context* ctx, int32_t on);
int32_t ngs_profile_reset(ngs_context* ctx);
int32_t ngs_profile_read(ngs_context* ctx, ngs_profile_stats* out);

/* Tile-size policy: 0 = auto (8x8 tiles for views with < 592 16x16 tiles in
 * the trainer, 16x16 elsewhere), 8 or 16 = forced. Results do not depend on it. */
int32_t ngs_set_tile_size(ngs_context* ctx, int32_t tile);

/* FP32 FFMA throughput microbenchmark on the context's device (TFLOP/s). */
int32_t ngs_microbench_fp32(ngs_context* ctx, double* tflops);
/* FP64 DFMA throughput microbenchmark (TFLOP/s). */
int32_t ngs_microbench_fp64(ngs_context* ctx, double* tflops);
/* Newton-solve microbenchmark (BASELINE config 4): n synthetic
 * Gaussians (SH degree sh_degree) with random SPD accumulator blocks for every
 * attribute group (position/scaling 2x2, rotation/opacity 1x1, colour rank-`views`
 * per channel), solved AND committed `reps` times (parameters restored between the
 * timed launches); ms_out[attr] = mean device time of solve_<attr> over all n
 * Gaussians; color_fast_frac (nullable) = fraction of the colour channel solves that
 * took the no-repair fast path. Scratch buffers only (the context's scene is untouched). */
int32_t ngs_microbench_solve(ngs_context* ctx, int32_t n, int32_t sh_degree, int32_t views, int32_t reps,
                             double ms_out[5], double* color_fast_frac);

#ifdef __cplusplus
}
#endif

#endif /* NGS_B200_PROFILE_H */
