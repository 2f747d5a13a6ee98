// sort.h — hand-written radix sort / scan interface (sort.cu).
#pragma once

#include <algorithm>

#include "context.h"

namespace ngsb {

struct SortScratch {
    DevBuf<unsigned> onesweep, dstart;  // histograms + tickets + look-back status; digit starts
    DevBuf<int> sums;
    void ensure(int n_max);
    void release() {
        onesweep.release();
        dstart.release();
        sums.release();
    }
};

// Stable LSD radix sort of (key, value) pairs on the low `bits` bits; the item
// count is read from device memory (*d_n <= n_max). Result in (keys, vals).
void radix_sort_pairs(uint32_t* keys, int* vals, uint32_t* keys_alt, int* vals_alt, const int* d_n, int n_max,
                      int bits, SortScratch& sc, cudaStream_t s);
// Exclusive prefix sum of n ints; optionally writes the total to *d_total (device).
void exclusive_scan(const int* in, int* out, int n, int* d_total, SortScratch& sc, cudaStream_t s);
// Re-orders runs of equal 32-bit depth keys by (FP64 depth, kernel id).
void depth_tie_fixup(const uint32_t* keys, int* ids, const double* depth, int n, cudaStream_t s);

}  // namespace ngsb
