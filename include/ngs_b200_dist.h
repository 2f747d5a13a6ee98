/*
 * ngs_b200_dist.h — multi-GPU sharding of the Newton step.
 *
 * Not part of the reference interface (the reference is single-process,
 * SURVEY.md §5; the natural sum point is the view loop of every solve_*,
 * newton.hpp:591-597). One process per GPU; every rank holds the full scene.
 * The 1+K views of a trainer step are partitioned (ngs_dist_plan): secondary
 * views go whole to ranks, the primary is split into tile-row bands that
 * water-fill the remaining load. A rank projects every view (the replicated
 * solve needs each view's flags) but sorts, rasterises, evaluates the loss and
 * back-propagates only its owned views/rows (+ a halo of
 * ceil((window - 1) / tile) tile rows for the SSIM support). After each backward
 * pass the per-Gaussian accumulators are summed across ranks (one NCCL
 * all-reduce, FP32 payload; exact uint64 limbs in deterministic mode) and every
 * rank runs the identical solve. The pair-capacity overflow vote is all-reduced
 * (MAX) too, so every rank takes the same retry decision.
 */
#ifndef NGS_B200_DIST_H
#define NGS_B200_DIST_H

#include <stdint.h>

#include "ngs_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

#define NGS_DIST_ID_BYTES 128

/* ncclGetUniqueId (rank 0); the caller broadcasts the bytes to every rank. */
int32_t ngs_dist_unique_id(uint8_t out[NGS_DIST_ID_BYTES]);
/* Joins the NCCL communicator and sets the context's shard to (rank, world). */
int32_t ngs_dist_init(ngs_context* ctx, const uint8_t id[NGS_DIST_ID_BYTES], int32_t rank, int32_t world);
/* Rows of each view owned by `rank` (tile rows of that view's tile size, 8 or 16):
 * [band_y0, band_y1) rendered (owned + halo), [own_y0, own_y1) owned. Empty band:
 * projection only. View 0 is the primary. Pure host function (no device needed). */
typedef struct {
    int32_t band_y0, band_y1, own_y0, own_y1;
} ngs_shard_rows;
int32_t ngs_dist_plan(int32_t world, int32_t rank, int32_t n_views, const int32_t* width, const int32_t* height,
                      const int32_t* tile, int32_t loss_window, ngs_shard_rows* out);
/* Shard without a communicator: accumulate/solve see this rank's partial sums
 * only (the caller reduces). Used to validate sharding on one device. */
int32_t ngs_set_shard(ngs_context* ctx, int32_t rank, int32_t world);

#ifdef __cplusplus
}
#endif

#endif /* NGS_B200_DIST_H */
