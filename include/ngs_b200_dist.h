/*
 * ngs_b200_dist.h — multi-GPU sharding of the Newton step.
 *
 * Not part of the reference interface (the reference is single-process,
 * SURVEY.md §5). One process per GPU; every rank holds the full scene. Each
 * view of a step is split into `world` tile-row bands: a rank projects and
 * bins only its band (+ a one-tile-row halo), rasterises it, evaluates the loss
 * fields for it and back-propagates its owned rows; the FP64 per-Gaussian
 * accumulators of every pass are then summed across ranks (NCCL all-reduce on
 * the context stream) and every rank runs the identical replicated solve.
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
/* Shard without a communicator: accumulate/solve see this rank's partial sums
 * only (the caller reduces). Used to validate sharding on one device. */
int32_t ngs_set_shard(ngs_context* ctx, int32_t rank, int32_t world);

#ifdef __cplusplus
}
#endif

#endif /* NGS_B200_DIST_H */
