/*
 * ngs_b200_ext.h — product-only extensions of the C-ABI (libngs_b200.so), used by
 * the drop-in C++ trainer (include/ngs_ref/ngs/trainer.hpp). Not part of the
 * interface the test oracle implements.
 */
#ifndef NGS_B200_EXT_H
#define NGS_B200_EXT_H

#include <stdint.h>

#include "ngs_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Sets the opacity-barrier weight the next Newton steps use (the reference Trainer
 * decays it once per epoch inside run(), trainer.hpp:264-265; a caller that drives
 * the epochs itself applies the same decay through this). */
int32_t ngs_trainer_set_barrier_weight(ngs_context* ctx, double weight);

#ifdef __cplusplus
}
#endif

#endif /* NGS_B200_EXT_H */
