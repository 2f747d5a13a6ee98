// sort.cu — hand-written stable LSD radix sort and exclusive scan (K2, K4).
//
// Replaces std::sort by (depth, kernel id) and the per-tile bins of
// build_splat_list (rasterizer.hpp:228-263). Item counts are read from device
// memory, so the binning never synchronises with the host.
//
// One global histogram kernel for all passes, then one onesweep kernel per
// 8-bit pass (stable in-tile ranks + decoupled look-back across tiles).
// 2048 items per block.
#include "sort.h"

namespace ngsb {

namespace {

constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kTileItems = kThreads * kItems;  // 2048 (scan tiles)
constexpr int kSItems = 16;                      // onesweep items per thread
constexpr int kSTile = kThreads * kSItems;       // 4096 keys per onesweep tile
constexpr int kDigits = 256;

// ---------------------------------------------------------------------------
// Onesweep-style LSD radix sort: one global histogram kernel for all passes,
// then ONE kernel per 8-bit pass. Each block takes a 2048-item tile in ticket
// order, ranks its items stably (warp-contiguous ranges, match_any per round),
// obtains the exclusive prefix of every digit over earlier tiles by decoupled
// look-back on per-(tile, digit) status words, and writes through shared memory
// so that runs of equal digits are stored contiguously.
// ---------------------------------------------------------------------------

constexpr int kMaxPasses = 4;
#ifndef NGS_LOOKBACK
#define NGS_LOOKBACK 4
#endif
constexpr int kLookBack = NGS_LOOKBACK;  // predecessors loaded per look-back round
constexpr uint32_t kFlagAgg = 1u << 30, kFlagInc = 2u << 30, kCountMask = (1u << 30) - 1;

__global__ void __launch_bounds__(kThreads) radix_global_hist_k(const uint32_t* __restrict__ keys,
                                                                const int* __restrict__ d_n, int passes,
                                                                unsigned* __restrict__ hist) {
    __shared__ unsigned s_hist[kMaxPasses][kDigits];
    const int n = *d_n;
    for (int p = 0; p < passes; ++p) s_hist[p][threadIdx.x] = 0;
    __syncthreads();
    const int base = blockIdx.x * kSTile;
    if (base < n) {
#pragma unroll
        for (int r = 0; r < kSItems; ++r) {
            const int i = base + r * kThreads + threadIdx.x;
            if (i < n) {
                const uint32_t k = keys[i];
                for (int p = 0; p < passes; ++p) atomicAdd(&s_hist[p][(k >> (8 * p)) & 0xFF], 1u);
            }
        }
    }
    __syncthreads();
    for (int p = 0; p < passes; ++p) {
        const unsigned v = s_hist[p][threadIdx.x];
        if (v) atomicAdd(&hist[p * kDigits + threadIdx.x], v);
    }
}

// Block-wide exclusive scan of one value per thread (256 threads); returns the total in *total.
__device__ __forceinline__ unsigned block_exclusive_scan(unsigned v, unsigned* s_warp, unsigned* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += t;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    unsigned wbase = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
        const unsigned sw = s_warp[w];
        if (w < warp) wbase += sw;
        tot += sw;
    }
    if (total) *total = tot;
    __syncthreads();
    return wbase + x - v;
}

// Exclusive digit starts per pass: dstart[p][d] = sum of hist[p][d' < d].
__global__ void __launch_bounds__(kThreads) radix_digit_starts_k(const unsigned* __restrict__ hist, int passes,
                                                                 unsigned* __restrict__ dstart) {
    __shared__ unsigned s_warp[kThreads / 32];
    for (int p = 0; p < passes; ++p)
        dstart[p * kDigits + threadIdx.x] = block_exclusive_scan(hist[p * kDigits + threadIdx.x], s_warp, nullptr);
}

__global__ void __launch_bounds__(kThreads) radix_onesweep_k(const uint32_t* __restrict__ keys_in,
                                                             const int* __restrict__ vals_in,
                                                             uint32_t* __restrict__ keys_out, int* __restrict__ vals_out,
                                                             const int* __restrict__ d_n, int shift,
                                                             const unsigned* __restrict__ dstart,
                                                             unsigned* __restrict__ status, unsigned* __restrict__ ticket) {
    __shared__ unsigned s_wc[kThreads / 32][kDigits];  // per-warp digit counts -> per-warp exclusive prefix
    __shared__ unsigned s_bstart[kDigits];             // block-local digit starts
    __shared__ unsigned s_gbase[kDigits];              // global position of the block's first item of each digit
    __shared__ uint32_t s_k[kSTile];
    __shared__ int s_v[kSTile];
    __shared__ unsigned s_warp[kThreads / 32];
    __shared__ int s_tile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = static_cast<int>(atomicAdd(ticket, 1u));  // in-order tile ids for the look-back
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) s_wc[w][threadIdx.x] = 0;
    __syncthreads();
    const int tile = s_tile;
    const int n = *d_n;
    const int base = tile * kSTile;
    if (base >= n) return;

    // 1. Stable ranks inside each warp's contiguous 256-item range.
    uint32_t key[kSItems];
    int val[kSItems];
    unsigned wrank[kSItems];
#pragma unroll
    for (int r = 0; r < kSItems; ++r) {  // all loads first: 2 x kSItems in flight per thread
        const int i = base + warp * (kSItems * 32) + r * 32 + lane;
        key[r] = i < n ? keys_in[i] : 0u;
        val[r] = i < n ? vals_in[i] : 0;
    }
#pragma unroll
    for (int r = 0; r < kSItems; ++r) {
        const int i = base + warp * (kSItems * 32) + r * 32 + lane;
        const bool valid = i < n;
        const int digit = valid ? static_cast<int>((key[r] >> shift) & 0xFF) : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, digit);
        const unsigned before = __popc(peers & ((1u << lane) - 1u));
        unsigned old = 0;
        if (valid) old = s_wc[warp][digit];
        __syncwarp();
        if (valid && before == 0) s_wc[warp][digit] = old + __popc(peers);
        __syncwarp();
        wrank[r] = old + before;
    }
    __syncthreads();
    // 2. Per digit (thread d): exclusive prefix over warps, block count, block-local start.
    const int d = threadIdx.x;
    unsigned bc = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
        const unsigned c = s_wc[w][d];
        s_wc[w][d] = bc;
        bc += c;
    }
    // 3. Decoupled look-back for digit d over earlier tiles.
    unsigned* st = status + static_cast<size_t>(tile) * kDigits + d;
    unsigned excl = 0;
    if (tile == 0) {
        atomicExch(st, kFlagInc | bc);
    } else {
        atomicExch(st, kFlagAgg | bc);
        // Walk back kLookBack predecessors per round (independent loads in flight), in order,
        // re-polling only a status that is not published yet. All tiles of a pass start in
        // one wave, so early in the pass a tile sums many aggregates before it meets an
        // inclusive prefix: the round count, not the load count, sets the latency.
        bool found = false;
        for (int t = tile - 1; t >= 0 && !found; t -= kLookBack) {
            unsigned v[kLookBack];
#pragma unroll
            for (int q = 0; q < kLookBack; ++q)
                v[q] = t - q >= 0 ? *(const volatile unsigned*)(status + static_cast<size_t>(t - q) * kDigits + d) : 0u;
#pragma unroll
            for (int q = 0; q < kLookBack; ++q) {
                if (found || t - q < 0) break;
                const volatile unsigned* sp = status + static_cast<size_t>(t - q) * kDigits + d;
                while ((v[q] & ~kCountMask) == 0) v[q] = *sp;
                excl += v[q] & kCountMask;
                if ((v[q] & ~kCountMask) == kFlagInc) found = true;
            }
        }
        atomicExch(st, kFlagInc | (excl + bc));
    }
    const unsigned bstart = block_exclusive_scan(bc, s_warp, nullptr);
    s_bstart[d] = bstart;
    s_gbase[d] = dstart[d] + excl;
    __syncthreads();
    // 4. Local placement in digit order, then contiguous global stores.
#pragma unroll
    for (int r = 0; r < kSItems; ++r) {
        const int i = base + warp * (kSItems * 32) + r * 32 + lane;
        if (i < n) {
            const int digit = static_cast<int>((key[r] >> shift) & 0xFF);
            const unsigned lpos = s_bstart[digit] + s_wc[warp][digit] + wrank[r];
            s_k[lpos] = key[r];
            s_v[lpos] = val[r];
        }
    }
    __syncthreads();
    const int cnt = min(kSTile, n - base);
    for (int i = threadIdx.x; i < cnt; i += kThreads) {
        const uint32_t k = s_k[i];
        const int digit = static_cast<int>((k >> shift) & 0xFF);
        const unsigned g = s_gbase[digit] + (static_cast<unsigned>(i) - s_bstart[digit]);
        keys_out[g] = k;
        vals_out[g] = s_v[i];
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
    const int nb = cdiv(std::max(n_max, 1), kSTile);
    const int nbs = cdiv(std::max(n_max, 1), kTileItems);
    // one memset clears: hist [passes][256], tickets [passes], status [passes][nb][256]
    onesweep.ensure(static_cast<size_t>(kMaxPasses) * kDigits + kMaxPasses +
                    static_cast<size_t>(kMaxPasses) * nb * kDigits);
    dstart.ensure(static_cast<size_t>(kMaxPasses) * kDigits);
    sums.ensure(nbs + 1);
}

void radix_sort_pairs(uint32_t* keys, int* vals, uint32_t* keys_alt, int* vals_alt, const int* d_n, int n_max,
                      int bits, SortScratch& sc, cudaStream_t s) {
    if (n_max <= 0) return;
    sc.ensure(n_max);
    const int nb = cdiv(n_max, kSTile);
    const int passes = cdiv(bits, 8);
    if (passes > kMaxPasses) throw Error(NGS_ERR_INTERNAL, "radix sort: more than 32 key bits");
    unsigned* hist = sc.onesweep.ptr;
    unsigned* tickets = hist + kMaxPasses * kDigits;
    unsigned* status = tickets + kMaxPasses;
    CUDA_CHECK(cudaMemsetAsync(hist, 0,
                               sizeof(unsigned) * (kMaxPasses * kDigits + kMaxPasses + static_cast<size_t>(passes) * nb * kDigits),
                               s));
    radix_global_hist_k<<<nb, kThreads, 0, s>>>(keys, d_n, passes, hist);
    radix_digit_starts_k<<<1, kThreads, 0, s>>>(hist, passes, sc.dstart.ptr);
    uint32_t* kin = keys;
    int* vin = vals;
    uint32_t* kout = keys_alt;
    int* vout = vals_alt;
    for (int p = 0; p < passes; ++p) {
        radix_onesweep_k<<<nb, kThreads, 0, s>>>(kin, vin, kout, vout, d_n, 8 * p, sc.dstart.ptr + p * kDigits,
                                                 status + static_cast<size_t>(p) * nb * kDigits, tickets + p);
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
