// render.cu — K1 projection, K2-K5 depth sort + tile binning, K6 forward raster.
//
// Reference semantics: build_splat_list (rasterizer.hpp:182-265) and
// composite_forward / composite_pixel (rasterizer.hpp:274-442).
#include <cmath>
#include <cstring>

#include "context.h"
#include "solve.h"
#include "geometry.cuh"
#include "sort.h"
#include "splat.cuh"

namespace ngsb {

void ViewSlot::release_all() {
    rec_a.release();
    rec_b.release();
    rec_c.release();
    pix.release();
    depth.release();
    rect.release();
    tiles_touched.release();
    flags.release();
    entry64.release();
    depth_key.release();
    depth_key_alt.release();
    order.release();
    order_alt.release();
    counts_sorted.release();
    offsets.release();
    pair_key.release();
    pair_key_alt.release();
    pair_val.release();
    pair_val_alt.release();
    ranges.release();
    counters.release();
    if (sort_scratch) {
        auto* sc = static_cast<SortScratch*>(sort_scratch);
        sc->release();
        delete sc;
        sort_scratch = nullptr;
    }
    image.release();
    t_final.release();
    last.release();
    target.release();
    fields.release();
    loss_grad.release();
    loss_hess.release();
    loss_sums.release();
    consts.release();
    valid = false;
}

// Camera(view, proj, w, h), camera.hpp:30-42.
void upload_camera(const ngs_camera& c, CameraDev& out, int tile) {
    if (c.width < 16 || c.height < 16) throw Error(NGS_ERR_INVALID_INPUT, "camera: width and height must be >= 16");
    for (int i = 0; i < 16; ++i) {
        out.view[i] = c.view[i];
        out.proj[i] = c.proj[i];
    }
    for (int r = 0; r < 4; ++r)
        for (int col = 0; col < 4; ++col) {
            double v = 0;
            for (int k = 0; k < 4; ++k) v += c.proj[4 * r + k] * c.view[4 * k + col];
            out.view_proj[4 * r + col] = v;
        }
    const double* m = c.view;
    auto R = [&](int i, int j) { return m[4 * i + j]; };
    const double det = R(0, 0) * (R(1, 1) * R(2, 2) - R(2, 1) * R(1, 2)) -
                       R(1, 0) * (R(0, 1) * R(2, 2) - R(2, 1) * R(0, 2)) +
                       R(2, 0) * (R(0, 1) * R(1, 2) - R(1, 1) * R(0, 2));
    if (std::abs(det) < 1e-12) throw Error(NGS_ERR_INVALID_INPUT, "camera: view rotation block is singular");
    double inv[9];
    inv[0] = (R(1, 1) * R(2, 2) - R(1, 2) * R(2, 1)) / det;
    inv[1] = (R(0, 2) * R(2, 1) - R(0, 1) * R(2, 2)) / det;
    inv[2] = (R(0, 1) * R(1, 2) - R(0, 2) * R(1, 1)) / det;
    inv[3] = (R(1, 2) * R(2, 0) - R(1, 0) * R(2, 2)) / det;
    inv[4] = (R(0, 0) * R(2, 2) - R(0, 2) * R(2, 0)) / det;
    inv[5] = (R(0, 2) * R(1, 0) - R(0, 0) * R(1, 2)) / det;
    inv[6] = (R(1, 0) * R(2, 1) - R(1, 1) * R(2, 0)) / det;
    inv[7] = (R(0, 1) * R(2, 0) - R(0, 0) * R(2, 1)) / det;
    inv[8] = (R(0, 0) * R(1, 1) - R(0, 1) * R(1, 0)) / det;
    const double t[3] = {R(0, 3), R(1, 3), R(2, 3)};
    for (int i = 0; i < 3; ++i) out.center[i] = -(inv[3 * i] * t[0] + inv[3 * i + 1] * t[1] + inv[3 * i + 2] * t[2]);
    out.width = c.width;
    out.height = c.height;
    out.tile = tile;
    out.tiles_x = (c.width + tile - 1) / tile;
    out.tiles_y = (c.height + tile - 1) / tile;
}

namespace {

// Order-preserving 32-bit key of the FP32-rounded depth; equal-key runs are
// re-ordered by the FP64 depth afterwards (depth_tie_fixup), so the final
// order is exactly (FP64 depth, kernel id).
__device__ __forceinline__ unsigned int depth_sort_key(double d) {
    const unsigned int b = __float_as_uint(static_cast<float>(d));
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// Outputs of one view's projection (K1); `depth_key`/`ids` null when the slot keeps its
// sorted depth order (same positions and camera), `entry64` only for parity read-back.
struct ProjOut {
    float4 *ra, *rb, *rc;
    double2* pix;
    double* depth;
    int4* rect;
    int* tiles_touched;
    uint8_t* flags;
    unsigned int* depth_key;
    int* ids;
    double* entry64;
    // The slot's view colours (c~ in rb.zw / rc.x) and clamp flags are still those of the
    // current positions, SH coefficients and camera (ProjOut-level cache, prepare_view):
    // skip the SH evaluation and leave them in place.
    bool keep_color;
};

// K1: per-kernel projection, SH colour and tile extent (FP64 math, coalesced
// float4 SoA loads; build_splat_list per-entry block rasterizer.hpp:192-226).
__device__ __forceinline__ void project_one(const SceneDev& s, int k, const CameraDev& cam, const RasterParams& rp,
                                            const ProjOut& o, int* err) {
    if (o.ids) o.ids[k] = k;  // null: the slot keeps its sorted depth order (same positions and camera)
    const float4 ps = s.pos_sigma[k];
    const D3 p = {ps.x, ps.y, ps.z};
    Projected pr;
    const bool ok = project_kernel(cam, p, s.quat[k], s.scale[k], rp.lambda_lp, pr);
    double det = 0;
    if (ok) det = pr.s00 * pr.s11 - pr.s01 * pr.s01;
    if (!ok || !(det > 0.0)) {
        if (ok) atomicOr(err, kErrNonPD);  // project_kernel: projected covariance is not positive definite
        o.tiles_touched[k] = 0;
        o.flags[k] = 0;
        o.rect[k] = make_int4(1, 1, 0, 0);
        if (o.depth_key) o.depth_key[k] = 0xFFFFFFFFu;
        o.depth[k] = 0;
        return;
    }
    double col[3] = {0.0, 0.0, 0.0};
    uint8_t f = kProjected;
    if (!o.keep_color) {
        D3 r;
        double rn;
        if (!view_direction(cam, p, r, rn)) {
            atomicOr(err, kErrDegenerate);  // DegenerateGeometry
            r = d3(0, 0, 1);
        }
        double basis[16];
        sh_basis(r, s.sh_degree, basis);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            double v = 0;
#pragma unroll
            for (int i = 0; i < 16; ++i)  // fully unrolled (basis in registers, loads issued together)
                if (i < s.n_coeffs) v += basis[i] * static_cast<double>(s.sh[(16 * ch + i) * s.n + k]);
            v += kColorOffset;
            const bool clamped = v <= 0.0;
            col[ch] = clamped ? 0.0 : v;
            if (clamped) f |= static_cast<uint8_t>(kClamp0 << ch);
        }
    }
    const double qa = pr.s11 / det, qb = -pr.s01 / det, qc = pr.s00 / det;
    double x0, y0, x1, y1;
    if (rp.cutoff_enabled) {
        const double rx = rp.radius * sqrt(fmax(pr.s00, 0.0));
        const double ry = rp.radius * sqrt(fmax(pr.s11, 0.0));
        x0 = pr.px - rx;
        y0 = pr.py - ry;
        x1 = pr.px + rx;
        y1 = pr.py + ry;
    } else {
        x0 = 0.0;
        y0 = 0.0;
        x1 = cam.width - 1.0;
        y1 = cam.height - 1.0;
    }
    auto clampi = [](int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); };
    const double ts = cam.tile;
    const int tx0 = clampi(static_cast<int>(floor(x0 / ts)), 0, cam.tiles_x - 1);
    const int tx1 = clampi(static_cast<int>(floor(x1 / ts)), 0, cam.tiles_x - 1);
    int ty0 = clampi(static_cast<int>(floor(y0 / ts)), 0, cam.tiles_y - 1);
    int ty1 = clampi(static_cast<int>(floor(y1 / ts)), 0, cam.tiles_y - 1);
    bool off = x1 < 0 || x0 >= cam.width || y1 < 0 || y0 >= cam.height;
    // Multi-GPU shard: bin only into this rank's tile rows (band incl. halo).
    ty0 = max(ty0, rp.band_y0);
    ty1 = min(ty1, rp.band_y1 - 1);
    off = off || ty0 > ty1;
    o.rect[k] = off ? make_int4(1, 1, 0, 0) : make_int4(tx0, ty0, tx1, ty1);
    o.tiles_touched[k] = off ? 0 : (tx1 - tx0 + 1) * (ty1 - ty0 + 1);
    o.depth[k] = pr.depth;
    if (o.depth_key) o.depth_key[k] = depth_sort_key(pr.depth);
    o.pix[k] = make_double2(pr.px, pr.py);
    o.ra[k] = make_float4(0.f, 0.f, static_cast<float>(qa), static_cast<float>(qb));
    if (o.keep_color) {  // colours and clamp flags stay; the geometry halves are rewritten
        reinterpret_cast<float2*>(o.rb)[2 * static_cast<size_t>(k)] = make_float2(static_cast<float>(qc), ps.w);
        float* rc = reinterpret_cast<float*>(o.rc + k);
        rc[1] = static_cast<float>(pr.s00);
        rc[2] = static_cast<float>(pr.s01);
        rc[3] = static_cast<float>(pr.s11);
    } else {
        o.flags[k] = f;
        o.rb[k] = make_float4(static_cast<float>(qc), ps.w, static_cast<float>(col[0]), static_cast<float>(col[1]));
        o.rc[k] = make_float4(static_cast<float>(col[2]), static_cast<float>(pr.s00), static_cast<float>(pr.s01),
                              static_cast<float>(pr.s11));
    }
    if (o.entry64) {
        double* e = o.entry64 + kEntry64 * static_cast<size_t>(k);
        e[0] = pr.px;
        e[1] = pr.py;
        e[2] = pr.s00;
        e[3] = pr.s01;
        e[4] = pr.s11;
        e[5] = x0;
        e[6] = y0;
        e[7] = x1;
        e[8] = y1;
        e[9] = col[0];
        e[10] = col[1];
        e[11] = col[2];
    }
}

// One launch per view (a fused all-views launch measured slower: DESIGN.md §6).
// Also publishes the entry count for the device-side sort (`n_out`, the slot's counters[0]):
// no host->device copy per render.
__global__ void __launch_bounds__(256) project_view_k(SceneDev s, CameraDev cam, RasterParams rp, ProjOut o, int* err,
                                                      int* n_out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k == 0) *n_out = s.n;
    if (k < s.n) project_one(s, k, cam, rp, o, err);
}

// Also sums the pair count exactly in 64 bits (`total64`, zeroed by the caller): the int
// scan below and the onesweep status words (30-bit counts, sort.cu) are only valid up to
// kMaxPairs, and emit_pairs_k refuses to emit past that instead of corrupting the lists.
__global__ void gather_counts_k(int n, const int* order, const int* tiles_touched, int* counts_sorted,
                                unsigned long long* total64) {
    // grid-stride over a bounded grid: one atomic per block (a per-warp or per-256-item atomic
    // on one address serialises in L2: 11.7K of them took ~50 us at 3M Gaussians)
    unsigned long long w = 0;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        const int c = tiles_touched[order[r]];
        counts_sorted[r] = c;
        w += static_cast<unsigned long long>(c);
    }
    __shared__ unsigned long long red[8];
    for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = w;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int i = 0; i < (blockDim.x >> 5); ++i) t += red[i];
        if (t) atomicAdd(total64, t);
    }
}

// K3: emit (tile, kernel) pairs in depth order; a later stable sort on the
// tile key alone keeps depth order (ties by kernel id) inside every tile.
__global__ void emit_pairs_k(int n, int tiles_x, int cap, const int* order, const int* offsets, const int4* rect,
                             const int* tiles_touched, unsigned int* keys, int* vals, int* overflow,
                             unsigned long long* pair_counter, int* counters, int* d_err) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned long long total64 = *reinterpret_cast<const unsigned long long*>(counters + 4);
    if (total64 > static_cast<unsigned long long>(kMaxPairs)) {  // beyond the sort's 30-bit counts: error, no lists
        if (r == 0) {
            atomicOr(d_err, kErrPairLimit);
            counters[2] = 0;
        }
        return;
    }
    if (r == 0) {
        const int total = counters[1];
        if (total > cap && overflow) atomicOr(overflow, 1);
        if (pair_counter) atomicAdd(pair_counter, static_cast<unsigned long long>(total));
        counters[2] = total < cap ? total : cap;
    }
    // Warp-cooperative emission: the warp's 32 Gaussians (consecutive in depth order) own one
    // contiguous run of pairs starting at offsets[r0]; lane l writes items l, l + 32, ... of
    // that run, so every key / value store instruction is coalesced (one thread looping over
    // its own rect wrote 32 scattered streams). Item e belongs to the first lane whose
    // inclusive count exceeds e (5-step search over the shuffled counts).
    const int lane = threadIdx.x & 31;
    const int k = r < n ? order[r] : 0;
    const int cnt = r < n ? tiles_touched[k] : 0;
    int incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += t;
    }
    const int warp_total = __shfl_sync(0xffffffffu, incl, 31);
    if (warp_total == 0) return;
    const int r0 = r - lane;
    const int base = offsets[r0];
    const int4 rc = cnt ? rect[k] : make_int4(0, 0, 0, 0);
    const int rw = rc.z - rc.x + 1;
    for (int e0 = 0; e0 < warp_total; e0 += 32) {
        const int e = e0 + lane;
        // owner = number of lanes whose inclusive count is <= e
        int owner = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const int probe = __shfl_sync(0xffffffffu, incl, owner + step - 1);
            if (probe <= e) owner += step;
        }
        const int own_incl = __shfl_sync(0xffffffffu, incl, owner);
        const int own_cnt = __shfl_sync(0xffffffffu, cnt, owner);
        const int own_k = __shfl_sync(0xffffffffu, k, owner);
        const int own_x0 = __shfl_sync(0xffffffffu, rc.x, owner);
        const int own_y0 = __shfl_sync(0xffffffffu, rc.y, owner);
        const int own_w = __shfl_sync(0xffffffffu, rw, owner);
        if (e < warp_total) {
            const int i = e - (own_incl - own_cnt);  // index inside the owner's rect, row-major
            const int dy = i / own_w, dx = i - dy * own_w;
            const int o = base + e;
            if (o < cap) {
                keys[o] = static_cast<unsigned int>((own_y0 + dy) * tiles_x + own_x0 + dx);
                vals[o] = own_k;
            }
        }
    }
}

// K5: per-tile [start, end) ranges from the tile-sorted key array.
__global__ void tile_ranges_k(const int* d_pairs, int T, const unsigned int* keys, int2* ranges) {
    const int pairs = *d_pairs;  // grid-stride: the grid is sized for the capacity, the count is on the device
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < pairs; i += gridDim.x * blockDim.x) {
        const unsigned int t = keys[i];
        if (t >= static_cast<unsigned int>(T)) continue;
        if (i == 0 || keys[i - 1] != t) ranges[t].x = i;
        if (i == pairs - 1 || keys[i + 1] != t) ranges[t].y = i + 1;
    }
}

// K6: forward alpha-blend rasterizer. One 16x16 tile per 256-thread block;
// the tile's depth-ordered splats are staged through shared memory in
// batches; the block retires as soon as every pixel saturated
// (__syncthreads_count = block-wide ballot). Pixel centres and splat centres
// are expressed relative to the tile origin so the FP32 offsets carry
// full precision at 4K resolutions.
template <int N_>
struct RasterSmemB {
    static constexpr int N = N_;
    float4 raw[2][4][N];  // staged records (pix as double2, ra, rb, rc), double-buffered
    double col[3][N];
    SplatSh sp[N];
    unsigned char wmask[N];
};
template <int TILE>
using RasterSmem = RasterSmemB<TILE * TILE>;
#ifndef NGS_RASTER2_BATCH
#define NGS_RASTER2_BATCH 128
#endif

// CK: also write each pixel's compositing state (T, FP64 colour prefix) at the chunk
// boundaries chunk_begin(range, c, chunks), c = 1 .. chunks-1, of its tile's list: the
// backward of deep small-tile lists then runs one block per (tile, chunk) from there.
template <int TILE, bool CK>
__global__ void __launch_bounds__(TILE * TILE) raster_forward_k(int tiles_x, int W, int H, const int2* __restrict__ ranges,
                                                        const int* __restrict__ vals, const double2* __restrict__ pix,
                                                        const float4* __restrict__ ra, const float4* __restrict__ rb,
                                                        const float4* __restrict__ rc, float bg0, float bg1, float bg2,
                                                        float cutoff, float tmin, double* __restrict__ image,
                                                        float* __restrict__ t_final, int* __restrict__ last_out,
                                                        int chunks, float* __restrict__ ck_t, double* __restrict__ ck_p) {
    constexpr int kRasterBatch = TILE * TILE;  // one splat per thread per batch
    // Dynamic shared memory (> 48 KB for 16x16 tiles): RasterSmem<TILE>.
    extern __shared__ __align__(16) unsigned char smem_raw[];
    RasterSmem<TILE>& S = *reinterpret_cast<RasterSmem<TILE>*>(smem_raw);
    auto& s_sp = S.sp;
    auto& s_col = S.col;    // colours widened once per splat (no per-pixel F2F)
    auto& s_wmask = S.wmask;  // bit w: the cutoff ellipse reaches warp w's box
    auto& s_raw = S.raw;
    const int tile = blockIdx.x;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    int lx, ly;
    WarpBox<TILE>::pixel(threadIdx.x, lx, ly);
    const int x = tx * TILE + lx, y = ty * TILE + ly;
    const bool inside = x < W && y < H;
    const float fx = lx + 0.5f, fy = ly + 0.5f;
    const double ox = tx * TILE, oy = ty * TILE;
    const int2 range = ranges[tile];
    float T = 1.0f;
    double C0 = 0.0, C1 = 0.0, C2 = 0.0;  // FP64 colour sums: the image feeds the cancelling (c - c^t) loss terms
    int last = -1;
    bool done = !inside;
    const size_t npx = static_cast<size_t>(W) * H, pidx = static_cast<size_t>(y) * W + x;
    int nc = 1, bnd = CK ? chunk_begin(range, 1, chunks) : 0;  // next checkpoint and its list index
    auto save = [&](int c) {
        if (inside) {
            ck_t[(c - 1) * npx + pidx] = T;
            ck_p[(3 * (c - 1) + 0) * npx + pidx] = C0;
            ck_p[(3 * (c - 1) + 1) * npx + pidx] = C1;
            ck_p[(3 * (c - 1) + 2) * npx + pidx] = C2;
        }
    };
    const float tmin_eff = tmin > 0.f ? tmin : -1.0f;  // T < tmin_eff: early termination (none when tmin = 0)
    // Software pipeline: thread t stages splat t of the next batch with cp.async
    // (into its own slot, so only its own wait is needed) while the current batch
    // is composited; the list entry of the batch after that is loaded meanwhile.
    const int t = threadIdx.x;
    auto issue = [&](int buf, int k) {
        cp_async16(&s_raw[buf][0][t], pix + k);
        cp_async16(&s_raw[buf][1][t], ra + k);
        cp_async16(&s_raw[buf][2][t], rb + k);
        cp_async16(&s_raw[buf][3][t], rc + k);
    };
    if (range.x + t < range.y) issue(0, vals[range.x + t]);
    cp_async_commit();
    int kn = range.x + kRasterBatch + t < range.y ? vals[range.x + kRasterBatch + t] : 0;
    int it = 0;
    for (int base = range.x; base < range.y; base += kRasterBatch, ++it) {
        const int buf = it & 1;
        if (__syncthreads_count(done) == blockDim.x) break;
        cp_async_wait_all();
        const int i = base + t;
        if (i < range.y) {
            const double2 p = reinterpret_cast<const double2*>(s_raw[buf][0])[t];
            const float4 a = s_raw[buf][1][t], b = s_raw[buf][2][t], c = s_raw[buf][3][t];
            const float qmax = reject_bound(b.y, cutoff);
            const float py = static_cast<float>(p.y - oy);
            const float px = static_cast<float>(p.x - ox);
            SplatSh sp;
            sp.g0 = make_float4(px, py, a.z, a.w);
            sp.g1 = make_float4(b.x, b.y, qmax, b.z);
            sp.g2 = make_float2(b.w, c.x);
            sp.pad = make_float2(0.f, 0.f);
            s_sp[threadIdx.x] = sp;
            s_col[0][threadIdx.x] = b.z;
            s_col[1][threadIdx.x] = b.w;
            s_col[2][threadIdx.x] = c.x;
            s_wmask[threadIdx.x] = static_cast<unsigned char>(
                WarpBox<TILE>::mask_exact(px, py, ellipse_half_extent(qmax, c.y), ellipse_half_extent(qmax, c.w), a.z,
                                          a.w, b.x, qmax));
        } else {
            s_wmask[threadIdx.x] = 0;
        }
        if (i + kRasterBatch < range.y) issue(buf ^ 1, kn);
        cp_async_commit();
        kn = i + 2 * kRasterBatch < range.y ? vals[i + 2 * kRasterBatch] : 0;
        __syncthreads();
        const int cnt = min(kRasterBatch, range.y - base);
        // Only the splats whose cutoff ellipse reaches this warp's rows (per-warp bit
        // masks, increasing j); lanes that terminated skip the body.
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int c32 = 0; c32 < cnt && !__all_sync(0xffffffffu, done); c32 += 32) {
            unsigned m = __ballot_sync(0xffffffffu, (s_wmask[c32 + lane] >> warp) & 1u);
            while (m) {
                const int j = c32 + __ffs(m) - 1;
                m &= m - 1;
                if constexpr (CK) {
                    while (nc < chunks && base + j >= bnd) {  // state before list entry bnd
                        save(nc);
                        bnd = chunk_begin(range, ++nc, chunks);
                    }
                }
                const SplatSh sp = s_sp[j];
                SplatEval e;
                if (eval_splat_bf(sp, fx, fy, cutoff, e) && !done) {
                    const double w = blend_weight(T, e.alpha);
                    C0 = __fma_rn(w, s_col[0][j], C0);
                    C1 = __fma_rn(w, s_col[1][j], C1);
                    C2 = __fma_rn(w, s_col[2][j], C2);
                    T = next_transmittance(T, e.alpha);
                    last = base + j;
                    if (T < tmin_eff) done = true;
                }
            }
        }
    }
    cp_async_wait_all();
    if constexpr (CK)
        for (; nc < chunks; ++nc) save(nc);  // boundaries past the last entry this warp saw
    if (inside) {
        const size_t plane = static_cast<size_t>(W) * H;
        const size_t idx = static_cast<size_t>(y) * W + x;
        image[idx] = __fma_rn(T, bg0, C0);
        image[plane + idx] = __fma_rn(T, bg1, C1);
        image[2 * plane + idx] = __fma_rn(T, bg2, C2);
        t_final[idx] = T;
        last_out[idx] = last;
    }
}

// The 16x16-tile forward with TWO pixels per lane: 4 warps, each an 8x8 box, lane l
// owning pixels (l % 8, l / 8) and (l % 8, l / 8 + 4) of it. Per splat a warp loads the
// record and walks the mask loop once for 64 pixels and evaluates both on packed f32x2
// (eval_splat_bf2: bit-identical to the scalar evaluation), so the per-pixel results —
// image, T and last contributor — are the one-pixel-per-lane kernel's, bit for bit.
template <int TILE, int B>
__global__ void __launch_bounds__(TILE * TILE / 2) raster_forward2_k(
    int tiles_x, int W, int H, const int2* __restrict__ ranges, const int* __restrict__ vals,
    const double2* __restrict__ pix, const float4* __restrict__ ra, const float4* __restrict__ rb,
    const float4* __restrict__ rc, float bg0, float bg1, float bg2, float cutoff, float tmin,
    double* __restrict__ image, float* __restrict__ t_final, int* __restrict__ last_out) {
    using WB = WarpBoxT<TILE, 8>;
    constexpr int NT = TILE * TILE / 2, HPT = B / NT;  // B staged splats per batch, HPT per thread
    static_assert(B % NT == 0, "whole splats per thread");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    RasterSmemB<B>& S = *reinterpret_cast<RasterSmemB<B>*>(smem_raw);
    const int tile = blockIdx.x;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int lx = (warp % WB::ACROSS) * WB::BW + (lane & 7), ly = (warp / WB::ACROSS) * WB::BH + (lane >> 3);
    const int x = tx * TILE + lx, y0 = ty * TILE + ly, y1 = y0 + 4;
    const bool in0 = x < W && y0 < H, in1 = x < W && y1 < H;
    const float fx = lx + 0.5f, fy0 = ly + 0.5f, fy1 = ly + 4.5f;
    const double ox = tx * TILE, oy = ty * TILE;
    const int2 range = ranges[tile];
    float T0 = 1.0f, T1 = 1.0f;
    double C0[3] = {0.0, 0.0, 0.0}, C1[3] = {0.0, 0.0, 0.0};
    int last0 = -1, last1 = -1;
    bool done0 = !in0, done1 = !in1;
    const float tmin_eff = tmin > 0.f ? tmin : -1.0f;
    auto issue = [&](int buf, int slot, int k) {
        cp_async16(&S.raw[buf][0][slot], pix + k);
        cp_async16(&S.raw[buf][1][slot], ra + k);
        cp_async16(&S.raw[buf][2][slot], rb + k);
        cp_async16(&S.raw[buf][3][slot], rc + k);
    };
#pragma unroll
    for (int h = 0; h < HPT; ++h)
        if (range.x + t + h * NT < range.y) issue(0, t + h * NT, vals[range.x + t + h * NT]);
    cp_async_commit();
    int kn[HPT];
#pragma unroll
    for (int h = 0; h < HPT; ++h) kn[h] = range.x + B + t + h * NT < range.y ? vals[range.x + B + t + h * NT] : 0;
    int it = 0;
    for (int base = range.x; base < range.y; base += B, ++it) {
        const int buf = it & 1;
        if (__syncthreads_count(done0 && done1) == NT) break;
        cp_async_wait_all();
#pragma unroll
        for (int h = 0; h < HPT; ++h) {
            const int slot = t + h * NT, i = base + slot;
            if (i < range.y) {
                const double2 p = reinterpret_cast<const double2*>(S.raw[buf][0])[slot];
                const float4 a = S.raw[buf][1][slot], b = S.raw[buf][2][slot], c = S.raw[buf][3][slot];
                const float qmax = reject_bound(b.y, cutoff);
                const float py = static_cast<float>(p.y - oy);
                const float px = static_cast<float>(p.x - ox);
                SplatSh sp;
                sp.g0 = make_float4(px, py, a.z, a.w);
                sp.g1 = make_float4(b.x, b.y, qmax, b.z);
                sp.g2 = make_float2(b.w, c.x);
                sp.pad = make_float2(0.f, 0.f);
                S.sp[slot] = sp;
                S.col[0][slot] = b.z;
                S.col[1][slot] = b.w;
                S.col[2][slot] = c.x;
                S.wmask[slot] = static_cast<unsigned char>(WB::mask_exact(
                    px, py, ellipse_half_extent(qmax, c.y), ellipse_half_extent(qmax, c.w), a.z, a.w, b.x, qmax));
            } else {
                S.wmask[slot] = 0;
            }
            if (i + B < range.y) issue(buf ^ 1, slot, kn[h]);
        }
        cp_async_commit();
#pragma unroll
        for (int h = 0; h < HPT; ++h) {
            const int i2 = base + t + h * NT + 2 * B;
            kn[h] = i2 < range.y ? vals[i2] : 0;
        }
        __syncthreads();
        const int cnt = min(B, range.y - base);
        for (int c32 = 0; c32 < cnt && !__all_sync(0xffffffffu, done0 && done1); c32 += 32) {
            unsigned m = __ballot_sync(0xffffffffu, (S.wmask[c32 + lane] >> warp) & 1u);
            while (m) {
                const int j = c32 + __ffs(m) - 1;
                m &= m - 1;
                const SplatSh sp = S.sp[j];
                SplatEval e0, e1;
                bool k0, k1;
                eval_splat_bf2(sp, fx, fy0, fy1, cutoff, e0, e1, k0, k1);
                if (k0 && !done0) {
                    const double w = blend_weight(T0, e0.alpha);
#pragma unroll
                    for (int q = 0; q < 3; ++q) C0[q] = __fma_rn(w, S.col[q][j], C0[q]);
                    T0 = next_transmittance(T0, e0.alpha);
                    last0 = base + j;
                    if (T0 < tmin_eff) done0 = true;
                }
                if (k1 && !done1) {
                    const double w = blend_weight(T1, e1.alpha);
#pragma unroll
                    for (int q = 0; q < 3; ++q) C1[q] = __fma_rn(w, S.col[q][j], C1[q]);
                    T1 = next_transmittance(T1, e1.alpha);
                    last1 = base + j;
                    if (T1 < tmin_eff) done1 = true;
                }
            }
        }
    }
    cp_async_wait_all();
    const size_t plane = static_cast<size_t>(W) * H;
    if (in0) {
        const size_t idx = static_cast<size_t>(y0) * W + x;
        image[idx] = __fma_rn(T0, bg0, C0[0]);
        image[plane + idx] = __fma_rn(T0, bg1, C0[1]);
        image[2 * plane + idx] = __fma_rn(T0, bg2, C0[2]);
        t_final[idx] = T0;
        last_out[idx] = last0;
    }
    if (in1) {
        const size_t idx = static_cast<size_t>(y1) * W + x;
        image[idx] = __fma_rn(T1, bg0, C1[0]);
        image[plane + idx] = __fma_rn(T1, bg1, C1[1]);
        image[2 * plane + idx] = __fma_rn(T1, bg2, C1[2]);
        t_final[idx] = T1;
        last_out[idx] = last1;
    }
}

inline int blocks_for(int n, int b = 256) { return (n + b - 1) / b; }

}  // namespace

// 16x16 tiles: two pixels per lane in the forward (NGS_RASTER2=0: one pixel per lane, A/B).
static const bool g_raster2 = [] {
    const char* e = getenv("NGS_RASTER2");
    return !e || atoi(e) != 0;
}();

// Allocations of one view and the depth-order reuse decision (host only).
bool prepare_view(const SceneDev& scene, ViewSlot& v, bool want_debug, const RenderSync& sync) {
    const int n = scene.n;
    v.n = n;
    v.W = v.cam.width;
    v.H = v.cam.height;
    v.T = v.cam.tiles_x * v.cam.tiles_y;
    v.rec_a.ensure(n);
    v.rec_b.ensure(n);
    v.rec_c.ensure(n);
    v.pix.ensure(n);
    v.depth.ensure(n);
    v.rect.ensure(n);
    v.tiles_touched.ensure(n);
    v.flags.ensure(n);
    v.depth_key.ensure(n);
    v.order.ensure(n);
    v.counts_sorted.ensure(n + 1);
    v.offsets.ensure(n + 1);
    v.ranges.ensure(v.T);
    const size_t npx = static_cast<size_t>(v.W) * v.H;
    v.image.ensure(3 * npx);
    v.t_final.ensure(npx);
    v.last.ensure(npx);
    if (want_debug) v.entry64.ensure(kEntry64 * static_cast<size_t>(n));
    if (!v.sort_scratch) v.sort_scratch = new SortScratch();
    v.depth_key_alt.ensure(n);
    v.order_alt.ensure(n);
    v.counters.ensure(6);  // [0] n, [1] P (int scan), [2] min(P, cap), [4..5] P as u64
    // The culled set (key 0xFFFFFFFF: behind the near plane) and the depth keys depend on the
    // positions and the camera only; a non-PD projected covariance is a step error.
    const bool keep_order = sync.pos_version != 0 && v.order_version == sync.pos_version && v.order_n == n &&
                            std::memcmp(&v.order_cam, &v.cam, sizeof(CameraDev)) == 0;
    v.order_version = sync.pos_version;
    v.order_cam = v.cam;
    v.order_n = n;
    v.keep_order = keep_order;
    // View colours depend on the positions, the camera and the SH coefficients only.
    v.keep_color = keep_order && !want_debug && sync.sh_version != 0 && v.color_sh_version == sync.sh_version;
    v.color_sh_version = sync.sh_version;
    return keep_order;
}

void project_views(const SceneDev& scene, ViewSlot* const* views, int nv, bool want_debug, int* d_err,
                   cudaStream_t s) {
    const int n = scene.n;
    if (n == 0 || nv == 0) return;
    if (nv > kMaxSolveViews) throw Error(NGS_ERR_INTERNAL, "project_views: too many views");
    for (int i = 0; i < nv; ++i) {
        ViewSlot& v = *views[i];
        const ProjOut o{v.rec_a.ptr, v.rec_b.ptr, v.rec_c.ptr, v.pix.ptr, v.depth.ptr, v.rect.ptr,
                        v.tiles_touched.ptr, v.flags.ptr, v.keep_order ? nullptr : v.depth_key.ptr,
                        v.keep_order ? nullptr : v.order.ptr, want_debug ? v.entry64.ptr : nullptr, v.keep_color};
        StageScope st(NGS_STAGE_PROJECT, s);
        project_view_k<<<blocks_for(n), 256, 0, s>>>(scene, v.cam, v.raster, o, d_err, v.counters.ptr);
        CUDA_LAUNCH_CHECK();
    }
}

void render_view(const SceneDev& scene, ViewSlot& v, bool want_debug, int* d_err, cudaStream_t s,
                 const RenderSync& sync) {
    prepare_view(scene, v, want_debug, sync);
    ViewSlot* one = &v;
    project_views(scene, &one, 1, want_debug, d_err, s);
    if (sync.projected) CUDA_CHECK(cudaEventRecord(sync.projected, s));
    bin_and_raster(scene, v, d_err, s, sync);
}

// K2-K6 of one view after its projection: depth order, tile binning, forward raster.
void bin_and_raster(const SceneDev& scene, ViewSlot& v, int* d_err, cudaStream_t s, const RenderSync& sync) {
    const int n = scene.n;
    const bool keep_order = v.keep_order;
    int bits = 1;
    while ((1 << bits) < v.T) ++bits;
    SortScratch& sc = *static_cast<SortScratch*>(v.sort_scratch);
    if (!v.raster.owns_rows()) {
        // Multi-GPU: another rank owns this view; only its projection (flags for the
        // replicated colour solve) is needed here. The depth order was not sorted.
        v.order_version = 0;
        v.color_sh_version = 0;
        v.pairs = 0;
        v.valid = true;
        return;
    }
    if (n > 0) {
        StageScope st(NGS_STAGE_SORT, s, keep_order ? 4 : 11);  // sort 2 + 4 passes, fix-up, gather, scan 3
        // K2: global depth order, exactly (FP64 depth, kernel id): 4-pass radix sort of the
        // FP32 depth key (stable over the id-ordered input) + fix-up of equal-key runs.
        if (!keep_order) {
            radix_sort_pairs(v.depth_key.ptr, v.order.ptr, v.depth_key_alt.ptr, v.order_alt.ptr, v.counters.ptr, n, 32,
                             sc, s);
            depth_tie_fixup(v.depth_key.ptr, v.order.ptr, v.depth.ptr, n, s);
        }
        CUDA_CHECK(cudaMemsetAsync(v.counters.ptr + 4, 0, sizeof(unsigned long long), s));
        gather_counts_k<<<std::min(blocks_for(n), 8 * 148), 256, 0, s>>>(
            n, v.order.ptr, v.tiles_touched.ptr, v.counts_sorted.ptr,
            reinterpret_cast<unsigned long long*>(v.counters.ptr + 4));
        CUDA_LAUNCH_CHECK();
        exclusive_scan(v.counts_sorted.ptr, v.offsets.ptr, n, v.counters.ptr + 1, sc, s);
    } else {
        CUDA_CHECK(cudaMemsetAsync(v.counters.ptr, 0, 6 * sizeof(int), s));
    }
    // Pair capacity: exact (one host sync) or the slot's running capacity with a
    // device-side overflow flag (sync-free; the caller re-runs on overflow).
    size_t cap;
    if (sync.exact) {
        unsigned long long pairs = 0;
        if (n > 0) {
            CUDA_CHECK(cudaMemcpyAsync(&pairs, v.counters.ptr + 4, sizeof(pairs), cudaMemcpyDeviceToHost, s));
            CUDA_CHECK(cudaStreamSynchronize(s));
        }
        if (pairs > static_cast<unsigned long long>(kMaxPairs))
            throw Error(NGS_ERR_INVALID_INPUT, "render: (tile, splat) pair count exceeds 2^30 - 1 (sort limit)");
        v.pairs = static_cast<int>(pairs);
        cap = static_cast<size_t>(pairs);
        v.pair_cap = std::max(v.pair_cap, cap + cap / 4 + 4096);
    } else {
        v.pairs = -1;
        if (v.pair_cap == 0) v.pair_cap = static_cast<size_t>(n) * 4 + 4096;
        cap = v.pair_cap;
    }
    if (v.pairs > kMaxPairs)
        throw Error(NGS_ERR_INVALID_INPUT, "render: (tile, splat) pair count exceeds 2^30 - 1 (sort limit)");
    cap = std::min<size_t>(cap, static_cast<size_t>(kMaxPairs));
    CUDA_CHECK(cudaMemsetAsync(v.ranges.ptr, 0, sizeof(int2) * v.T, s));
    if (cap > 0 && n > 0) {
        StageScope st(NGS_STAGE_SORT, s, 4 + (bits + 7) / 8);  // emit, sort 2 + passes, ranges
        v.pair_key.ensure(cap);
        v.pair_key_alt.ensure(cap);
        v.pair_val.ensure(cap);
        v.pair_val_alt.ensure(cap);
        emit_pairs_k<<<blocks_for(n), 256, 0, s>>>(n, v.cam.tiles_x, static_cast<int>(cap), v.order.ptr,
                                                   v.offsets.ptr, v.rect.ptr, v.tiles_touched.ptr, v.pair_key.ptr,
                                                   v.pair_val.ptr, sync.overflow, sync.pair_counter, v.counters.ptr,
                                                   d_err);
        CUDA_LAUNCH_CHECK();
        // K4: stable sort of the depth-ordered pairs by tile key -> per-tile depth order.
        radix_sort_pairs(v.pair_key.ptr, v.pair_val.ptr, v.pair_key_alt.ptr, v.pair_val_alt.ptr, v.counters.ptr + 2,
                         static_cast<int>(cap), bits, sc, s);
        tile_ranges_k<<<std::min(blocks_for(static_cast<int>(cap)), 8 * 148), 256, 0, s>>>(
            v.counters.ptr + 2, v.T, v.pair_key.ptr, v.ranges.ptr);
        CUDA_LAUNCH_CHECK();
    }
    if (g_prof) g_prof->stats.renders += 1;
    StageScope st(NGS_STAGE_RASTER, s);
    // Chunked backward (8x8 tiles): checkpoints of the compositing state at the chunk starts.
    const int chunks = v.cam.tile == 8 ? std::max(1, v.chunks) : 1;
    v.ck_chunks = chunks;
    if (chunks > 1) {
        const size_t npx = static_cast<size_t>(v.W) * v.H;
        v.ck_t.ensure(static_cast<size_t>(chunks - 1) * npx);
        v.ck_p.ensure(static_cast<size_t>(chunks - 1) * 3 * npx);
    }
    auto launch = [&](auto kernel, int threads, size_t smem) {
        ensure_dynamic_smem(reinterpret_cast<const void*>(kernel), smem);
        kernel<<<v.T, threads, smem, s>>>(v.cam.tiles_x, v.W, v.H, v.ranges.ptr, cap > 0 ? v.pair_val.ptr : nullptr,
                                       v.pix.ptr, v.rec_a.ptr, v.rec_b.ptr, v.rec_c.ptr, scene.bg[0], scene.bg[1],
                                       scene.bg[2], v.raster.alpha_cutoff, v.raster.t_min, v.image.ptr, v.t_final.ptr,
                                       v.last.ptr, chunks, v.ck_t.ptr, v.ck_p.ptr);
    };
    if (v.cam.tile == 8 && chunks > 1) {
        launch(raster_forward_k<8, true>, 64, sizeof(RasterSmem<8>));
    } else if (v.cam.tile == 8) {
        launch(raster_forward_k<8, false>, 64, sizeof(RasterSmem<8>));
    } else if (g_raster2) {
        constexpr int B2 = NGS_RASTER2_BATCH;
        ensure_dynamic_smem(reinterpret_cast<const void*>(raster_forward2_k<16, B2>), sizeof(RasterSmemB<B2>));
        raster_forward2_k<16, B2><<<v.T, 128, sizeof(RasterSmemB<B2>), s>>>(
            v.cam.tiles_x, v.W, v.H, v.ranges.ptr, cap > 0 ? v.pair_val.ptr : nullptr, v.pix.ptr, v.rec_a.ptr,
            v.rec_b.ptr, v.rec_c.ptr, scene.bg[0], scene.bg[1], scene.bg[2], v.raster.alpha_cutoff, v.raster.t_min,
            v.image.ptr, v.t_final.ptr, v.last.ptr);
    } else {
        launch(raster_forward_k<16, false>, 256, sizeof(RasterSmem<16>));
    }
    CUDA_LAUNCH_CHECK();
    v.valid = true;
}

}  // namespace ngsb
