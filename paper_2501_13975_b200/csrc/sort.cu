// sort.cu — hand-written stable LSD radix sort and exclusive scan (K2, K4).
//
// Replaces std::sort by (depth, kernel id) and the per-tile bins of
// build_splat_list (rasterizer.hpp:228-263). Item counts are read from device
// memory, so the binning never synchronises with the host.
//
// Each 8-bit pass is three kernels: per-block digit histograms, a per-digit
// scan over blocks, and a stable scatter (items ranked in index order inside a
// block with warp match_any + cross-warp prefix counts). 2048 items per block.
#include "sort.h"

namespace ngsb {

namespace {

constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kTileItems = kThreads * kItems;  // 2048
constexpr int kDigits = 256;

__global__ void __launch_bounds__(kThreads) radix_hist_k(const uint32_t* __restrict__ keys, const int* __restrict__ d_n,
                                                         int shift, int nblocks, int* __restrict__ counts) {
    __shared__ int s_hist[kDigits];
    const int n = *d_n;
    s_hist[threadIdx.x] = 0;
    __syncthreads();
    const int base = blockIdx.x * kTileItems;
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const int i = base + r * kThreads + threadIdx.x;
        if (i < n) atomicAdd(&s_hist[(keys[i] >> shift) & 0xFF], 1);
    }
    __syncthreads();
    counts[threadIdx.x * nblocks + blockIdx.x] = s_hist[threadIdx.x];
}

// One block per digit: exclusive scan of counts[digit][0..nblocks) in place;
// the digit total goes to totals[digit].
__global__ void __launch_bounds__(kThreads) radix_scan_digit_k(int* __restrict__ counts, int nblocks,
                                                               int* __restrict__ totals) {
    __shared__ int s_warp[kThreads / 32];
    __shared__ int s_carry;
    int* row = counts + blockIdx.x * nblocks;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int start = 0; start < nblocks; start += kThreads) {
        const int i = start + threadIdx.x;
        const int v = i < nblocks ? row[i] : 0;
        int x = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += t;
        }
        if (lane == 31) s_warp[warp] = x;
        __syncthreads();
        int wbase = 0;
        for (int w = 0; w < warp; ++w) wbase += s_warp[w];
        const int carry = s_carry;
        if (i < nblocks) row[i] = carry + wbase + x - v;
        __syncthreads();
        if (threadIdx.x == kThreads - 1) s_carry = carry + wbase + x;
        __syncthreads();
    }
    if (threadIdx.x == 0) totals[blockIdx.x] = s_carry;
}

__global__ void __launch_bounds__(kThreads) radix_scatter_k(const uint32_t* __restrict__ keys_in,
                                                            const int* __restrict__ vals_in, uint32_t* __restrict__ keys_out,
                                                            int* __restrict__ vals_out, const int* __restrict__ d_n,
                                                            int shift, int nblocks, const int* __restrict__ counts,
                                                            const int* __restrict__ totals) {
    __shared__ int s_base[kDigits];               // running output position per digit
    __shared__ int s_wcount[kThreads / 32][kDigits];
    const int n = *d_n;
    const int base = blockIdx.x * kTileItems;
    if (base >= n) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    {
        // digit start = sum of totals of smaller digits + this block's scanned offset
        __shared__ int s_tot[kDigits];
        s_tot[threadIdx.x] = totals[threadIdx.x];
        __syncthreads();
        int acc = 0;
        for (int d = 0; d < static_cast<int>(threadIdx.x); ++d) acc += s_tot[d];
        s_base[threadIdx.x] = acc + counts[threadIdx.x * nblocks + blockIdx.x];
    }
    for (int w = 0; w < kThreads / 32; ++w) s_wcount[w][threadIdx.x] = 0;
    __syncthreads();
#pragma unroll 1
    for (int r = 0; r < kItems; ++r) {
        const int i = base + r * kThreads + threadIdx.x;
        const bool valid = i < n;
        uint32_t key = 0;
        int val = 0, digit = -1;
        if (valid) {
            key = keys_in[i];
            val = vals_in[i];
            digit = static_cast<int>((key >> shift) & 0xFF);
        }
        const unsigned active = __ballot_sync(0xffffffffu, valid);
        const unsigned peers = __match_any_sync(0xffffffffu, digit) & active;
        const int wrank = __popc(peers & ((1u << lane) - 1u));
        const bool leader = valid && wrank == 0;
        if (leader) s_wcount[warp][digit] = __popc(peers);
        __syncthreads();
        if (valid) {
            int pos = s_base[digit] + wrank;
            for (int w = 0; w < warp; ++w) pos += s_wcount[w][digit];
            keys_out[pos] = key;
            vals_out[pos] = val;
        }
        __syncthreads();
        // advance the per-digit bases by this round's counts and clear them
        int add = 0;
#pragma unroll
        for (int w = 0; w < kThreads / 32; ++w) {
            add += s_wcount[w][threadIdx.x];
            s_wcount[w][threadIdx.x] = 0;
        }
        s_base[threadIdx.x] += add;
        __syncthreads();
    }
}

// Block-level exclusive scan helpers (two-level: per-block sums, then a
// single-block scan of the sums, then add).
__global__ void __launch_bounds__(kThreads) scan_blocks_k(const int* __restrict__ in, int* __restrict__ out, int n,
                                                          int* __restrict__ block_sums) {
    __shared__ int s_warp[kThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int base = blockIdx.x * kTileItems + threadIdx.x * kItems;
    int v[kItems];
    int tsum = 0;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        const int i = base + k;
        v[k] = i < n ? in[i] : 0;
        tsum += v[k];
    }
    int x = tsum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += t;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    int wbase = 0;
    for (int w = 0; w < warp; ++w) wbase += s_warp[w];
    int run = wbase + x - tsum;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        const int i = base + k;
        if (i < n) out[i] = run;
        run += v[k];
    }
    if (threadIdx.x == kThreads - 1) block_sums[blockIdx.x] = wbase + x;
}

__global__ void __launch_bounds__(kThreads) scan_sums_k(int* __restrict__ sums, int nblocks, int* __restrict__ total) {
    __shared__ int s_warp[kThreads / 32];
    __shared__ int s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int start = 0; start < nblocks; start += kThreads) {
        const int i = start + threadIdx.x;
        const int v = i < nblocks ? sums[i] : 0;
        int x = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += t;
        }
        if (lane == 31) s_warp[warp] = x;
        __syncthreads();
        int wbase = 0;
        for (int w = 0; w < warp; ++w) wbase += s_warp[w];
        const int carry = s_carry;
        if (i < nblocks) sums[i] = carry + wbase + x - v;
        __syncthreads();
        if (threadIdx.x == kThreads - 1) s_carry = carry + wbase + x;
        __syncthreads();
    }
    if (threadIdx.x == 0 && total) *total = s_carry;
}

__global__ void scan_add_k(int* __restrict__ out, int n, const int* __restrict__ sums) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] += sums[i / kTileItems];
}

// Runs of equal 32-bit (float) depth keys are re-ordered by (FP64 depth,
// kernel id) — the exact reference order (rasterizer.hpp:228-232). Runs are
// short (float rounding of nearby depths); the run head sorts it.
__global__ void depth_tie_fixup_k(const uint32_t* __restrict__ keys, int* __restrict__ ids, const double* __restrict__ depth,
                                  int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || keys[i] == 0xFFFFFFFFu) return;         // culled entries sort last, unused
    if (i > 0 && keys[i - 1] == keys[i]) return;          // not a run head
    int e = i + 1;
    while (e < n && keys[e] == keys[i]) ++e;
    if (e - i < 2) return;
    for (int a = i + 1; a < e; ++a) {  // insertion sort by (depth, id)
        const int id = ids[a];
        const double d = depth[id];
        int b = a - 1;
        while (b >= i) {
            const int ib = ids[b];
            const double db = depth[ib];
            if (db < d || (db == d && ib < id)) break;
            ids[b + 1] = ib;
            --b;
        }
        ids[b + 1] = id;
    }
}

inline int cdiv(int a, int b) { return (a + b - 1) / b; }

}  // namespace

void SortScratch::ensure(int n_max) {
    const int nb = cdiv(std::max(n_max, 1), kTileItems);
    counts.ensure(static_cast<size_t>(kDigits) * nb);
    totals.ensure(kDigits);
    sums.ensure(nb + 1);
}

void radix_sort_pairs(uint32_t* keys, int* vals, uint32_t* keys_alt, int* vals_alt, const int* d_n, int n_max,
                      int bits, SortScratch& sc, cudaStream_t s) {
    if (n_max <= 0) return;
    sc.ensure(n_max);
    const int nb = cdiv(n_max, kTileItems);
    const int passes = cdiv(bits, 8);
    uint32_t* kin = keys;
    int* vin = vals;
    uint32_t* kout = keys_alt;
    int* vout = vals_alt;
    for (int p = 0; p < passes; ++p) {
        const int shift = 8 * p;
        radix_hist_k<<<nb, kThreads, 0, s>>>(kin, d_n, shift, nb, sc.counts.ptr);
        radix_scan_digit_k<<<kDigits, kThreads, 0, s>>>(sc.counts.ptr, nb, sc.totals.ptr);
        radix_scatter_k<<<nb, kThreads, 0, s>>>(kin, vin, kout, vout, d_n, shift, nb, sc.counts.ptr, sc.totals.ptr);
        std::swap(kin, kout);
        std::swap(vin, vout);
    }
    CUDA_LAUNCH_CHECK();
    if (kin != keys) {  // odd pass count: result is in the alternate buffers
        CUDA_CHECK(cudaMemcpyAsync(keys, kin, sizeof(uint32_t) * n_max, cudaMemcpyDeviceToDevice, s));
        CUDA_CHECK(cudaMemcpyAsync(vals, vin, sizeof(int) * n_max, cudaMemcpyDeviceToDevice, s));
    }
}

void exclusive_scan(const int* in, int* out, int n, int* d_total, SortScratch& sc, cudaStream_t s) {
    if (n <= 0) return;
    sc.ensure(n);
    const int nb = cdiv(n, kTileItems);
    scan_blocks_k<<<nb, kThreads, 0, s>>>(in, out, n, sc.sums.ptr);
    scan_sums_k<<<1, kThreads, 0, s>>>(sc.sums.ptr, nb, d_total);
    scan_add_k<<<cdiv(n, 256), 256, 0, s>>>(out, n, sc.sums.ptr);
    CUDA_LAUNCH_CHECK();
}

void depth_tie_fixup(const uint32_t* keys, int* ids, const double* depth, int n, cudaStream_t s) {
    if (n <= 0) return;
    depth_tie_fixup_k<<<cdiv(n, 256), 256, 0, s>>>(keys, ids, depth, n);
    CUDA_LAUNCH_CHECK();
}

}  // namespace ngsb
