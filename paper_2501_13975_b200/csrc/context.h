// context.h — host-side state of one ngs_context (one device, one stream).
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <vector>
#include <string>
#include <vector>

#include "common.cuh"
#include "ngs_b200_profile.h"

namespace ngsb {

constexpr int kEntry64 = 12;

// Raster/loss options as the kernels consume them (FP32/FP64 copies of the
// reference structs, rasterizer.hpp:25-40, loss.hpp:11-22).
struct RasterParams {
    double lambda_lp;
    float alpha_cutoff;
    float t_min;
    bool cutoff_enabled;  // alpha_cutoff > 0: AABB binning, else every splat in every tile
    double radius;        // max(3, sqrt(2 ln(1/alpha_cutoff)))  rasterizer.hpp:215-216
    // Multi-GPU shard of this view (plan_step_shards), in tile rows of the
    // view's tile size: rows [band_y0, band_y1) are projected, binned, rasterised and get
    // SSIM statistics (owned rows plus a halo of ceil((window - 1) / tile) rows: the loss
    // derivatives at a pixel read statistics +-window/2 away, which read pixels
    // +-window/2 further); loss fields and the backward cover the owned rows
    // [own_y0, own_y1) only. An empty band (band_y0 == band_y1) is a view this rank
    // does not own: it is only projected (its flags feed the replicated colour solve).
    // Full frame when unsharded.
    int band_y0 = 0, band_y1 = 1 << 30;
    int own_y0 = 0, own_y1 = 1 << 30;
    bool owns_rows() const { return own_y0 < own_y1; }
};

struct ShardRows {
    int band_y0, band_y1, own_y0, own_y1;
};

// Partition of the views of one Newton step over `world` ranks (SURVEY.md
// §8(e) parity mode). View 0 is the primary; views 1..nv-1 are the secondaries.
//   * Secondaries go whole to ranks, largest first, each to the least-loaded rank
//     (load = pixels; ties: lowest rank).
//   * The primary's tile rows are then water-filled: rank r gets a contiguous share
//     proportional to max(0, L - load_r), L chosen so the shares cover the primary, in
//     rank order. With nv == 1 the single view is split evenly.
//   * Halo: ceil((window - 1) / tile) tile rows on each side of an owned range.
// Identical on every rank (pure function of its arguments). world <= 1: full frames.
void plan_step_shards(int world, int rank, int nv, const int* width, const int* height, const int* tile,
                      int window, ShardRows* out);
inline void apply_shard(const ShardRows& r, RasterParams& rp) {
    rp.band_y0 = r.band_y0;
    rp.band_y1 = r.band_y1;
    rp.own_y0 = r.own_y0;
    rp.own_y1 = r.own_y1;
}

// Views with fewer 16x16 tiles than this render with 8x8 tiles: their per-tile
// lists are deep (secondaries at 1/4 resolution) and 16x16 leaves the GPU idle.
constexpr int kSmallViewTiles = 4 * 148;
// Secondary views: 8x8 tiles only below this many 16x16 tiles (tile_for).
constexpr int kTinyViewTiles = 64;

struct LossParams {
    double lambda, c1, c2;
    int window;
    double window_sigma;
};

template <typename T>
struct DevBuf {
    T* ptr = nullptr;
    size_t cap = 0;
    void ensure(size_t n) {
        if (n <= cap) return;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
        const size_t want = n + n / 4 + 64;
        CUDA_CHECK(cudaMalloc(&ptr, want * sizeof(T)));
        cap = want;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
    }
};

// One rendered view: the device-resident equivalent of ViewContext
// (newton.hpp:86-96) without the capture buffers (SURVEY.md §7 design stance).
struct ViewSlot {
    bool valid = false;
    CameraDev cam{};
    unsigned long long order_version = 0;  // RenderSync::pos_version of the last depth sort (0: not reusable)
    bool keep_order = false;               // this render reuses the sorted depth order (prepare_view)
    unsigned long long color_sh_version = 0;  // RenderSync::sh_version of the slot's view colours
    bool keep_color = false;               // this render reuses the view colours (same positions, camera, SH)
    CameraDev order_cam{};
    int order_n = -1;
    int W = 0, H = 0, T = 0;
    int n = 0;         // kernels projected
    int entries = 0;   // projected (non-culled) kernels
    int pairs = 0;          // exact count when known on the host, else -1
    size_t pair_cap = 0;    // capacity of the pair buffers (sync-free renders)
    RasterParams raster{};
    LossParams loss{};
    double loss_value = 0.0;
    double loss_l2 = 0.0, loss_ssim_sum = 0.0;

    // K1 projection outputs (per kernel)
    DevBuf<float4> rec_a, rec_b, rec_c;
    DevBuf<double2> pix;     // splat centre in pixels (FP64: re-based per tile in FP32)
    DevBuf<double> depth;
    DevBuf<int4> rect;
    DevBuf<int> tiles_touched;
    DevBuf<uint8_t> flags;
    DevBuf<double> entry64;  // parity read-back: px, py, s00, s01, s11, bbox x0,y0,x1,y1, colour (kEntry64 per kernel)
    // K2-K5 binning (hand-written radix sort, sort.cu)
    DevBuf<unsigned int> depth_key, depth_key_alt;
    DevBuf<int> order, order_alt;
    DevBuf<int> counts_sorted, offsets;
    DevBuf<unsigned int> pair_key, pair_key_alt;
    DevBuf<int> pair_val, pair_val_alt;
    DevBuf<int2> ranges;
    DevBuf<int> counters;    // [0] entries n, [1] pairs P, [2] min(P, capacity)
    void* sort_scratch = nullptr;
    // K6 forward raster outputs (planar [3][H][W])
    DevBuf<double> image;   // FP64 (see raster_forward_k)
    DevBuf<float> t_final;
    DevBuf<int> last;       // index into the tile list of the last contributing splat, -1 if none
    // Chunked backward of 8x8-tile views: per-pixel compositing state at the chunk starts
    // ([chunk-1][H][W] T, [chunk-1][3][H][W] FP64 colour prefix), written by the forward.
    int chunks = 1;         // requested for the next render (trainer secondaries)
    int ck_chunks = 1;      // what the last render wrote (the backward's block split)
    DevBuf<float> ck_t;
    DevBuf<double> ck_p;
    // K7 loss fields
    DevBuf<double> target;  // planar [3][H][W], FP64 like the reference Image
    // Device-resident trainer targets are read in place (no per-step D2D copy into `target`).
    const double* target_ext = nullptr;
    const double* target_ptr() const { return target_ext ? target_ext : target.ptr; }
    DevBuf<double> fields;  // 9 center fields x 3 channels x H x W
    DevBuf<float> loss_grad, loss_hess;  // planar [3][H][W]
    DevBuf<unsigned long long> loss_sums;  // exact sums (kExactWords each): [0] sum d^2, [1] sum ssim
    // Per-pass backward constants (per kernel, AoS)
    DevBuf<float> consts;

    void release_all();
};

// Per-context measurement state (ngs_b200_profile.h). The active profiler of
// the calling thread is installed by each C-ABI entry point.
struct Profiler {
    bool enabled = false;
    // Timeline mode: per-launch events WITHOUT serialising the views (the concurrent
    // schedule as executed); resolve() also keeps (stage, stream, start, end) rows,
    // relative to `origin`, for ngs_profile_timeline.
    bool timeline = false;
    cudaEvent_t origin = nullptr;
    struct Rec {
        int stage;
        cudaEvent_t a, b;
        cudaStream_t s;
        int tag;  // >= 0: the primary view's backward of pass `tag` (also summed into primary_bwd_ms)
    };
    std::vector<Rec> pending;
    std::vector<ngs_timeline_row> rows;
    std::vector<cudaEvent_t> pool;
    ngs_profile_stats stats{};

    cudaEvent_t get() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        CUDA_CHECK(cudaEventCreate(&e));
        return e;
    }
    void resolve() {
        for (auto& r : pending) {
            CUDA_CHECK(cudaEventSynchronize(r.b));
            float ms = 0;
            CUDA_CHECK(cudaEventElapsedTime(&ms, r.a, r.b));
            stats.ms[r.stage] += ms;
            if (r.tag >= 0 && r.tag < 4) stats.primary_bwd_ms[r.tag] += ms;
            if (timeline && origin) {
                float t0 = 0, t1 = 0;
                CUDA_CHECK(cudaEventElapsedTime(&t0, origin, r.a));
                CUDA_CHECK(cudaEventElapsedTime(&t1, origin, r.b));
                rows.push_back(ngs_timeline_row{r.stage, static_cast<int32_t>(reinterpret_cast<uintptr_t>(r.s) & 0x7fffffff),
                                                t0, t1});
            }
            pool.push_back(r.a);
            pool.push_back(r.b);
        }
        pending.clear();
    }
    void reset() {
        resolve();
        stats = ngs_profile_stats{};
        rows.clear();
        if (origin) cudaEventDestroy(origin);
        origin = nullptr;
    }
    ~Profiler() {
        for (auto& r : pending) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        for (auto e : pool) cudaEventDestroy(e);
    }
};

extern thread_local Profiler* g_prof;

// Brackets the kernel launches of one stage; counts `launches` kernels.
struct StageScope {
    Profiler* p;
    int stage;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    int tag;
    StageScope(int stage_, cudaStream_t s_, int launches = 1, int tag_ = -1) : p(g_prof), stage(stage_), s(s_), tag(tag_) {
        if (!p) return;
        p->stats.launches[stage] += launches;
        p->stats.total_launches += launches;
        if (p->enabled || p->timeline) {
            a = p->get();
            CUDA_CHECK(cudaEventRecord(a, s));
        }
    }
    ~StageScope() {
        if (!p || !a) return;
        cudaEvent_t b = p->get();
        if (cudaEventRecord(b, s) == cudaSuccess) p->pending.push_back({stage, a, b, s, tag});
    }
};

// Launch wrappers (render.cu, loss.cu, backward.cu, solve.cu).
void upload_camera(const ngs_camera& c, CameraDev& out, int tile = kTile);
struct RenderSync {
    bool exact = true;                            // read the pair count back (one host sync)
    int* overflow = nullptr;                      // sync-free: set when the pair capacity was exceeded
    unsigned long long* pair_counter = nullptr;   // optional: adds the (tile, splat) pair count
    cudaEvent_t projected = nullptr;              // optional: recorded after the projection (flags ready)
    // Position version of the scene (0 = unknown). The depth order (and the culled set) is a
    // function of the positions and the camera only, so a slot re-rendered with the same
    // camera and version keeps its sorted order and skips K2.
    unsigned long long pos_version = 0;
    // SH version of the scene (0 = unknown): with the same position version and camera as well,
    // the view colours (SH evaluation, clamp flags) of the slot's last projection still hold.
    unsigned long long sh_version = 0;
};
void render_view(const SceneDev& scene, ViewSlot& v, bool want_debug, int* d_err, cudaStream_t s,
                 const RenderSync& sync = RenderSync{});
// render_view in three parts, so the 1+K views of a step share ONE projection launch:
// prepare_view (allocations, order reuse) per view, project_views for all of them, then
// bin_and_raster per view on its own stream.
bool prepare_view(const SceneDev& scene, ViewSlot& v, bool want_debug, const RenderSync& sync);
void project_views(const SceneDev& scene, ViewSlot* const* views, int nv, bool want_debug, int* d_err,
                   cudaStream_t s);
void bin_and_raster(const SceneDev& scene, ViewSlot& v, int* d_err, cudaStream_t s, const RenderSync& sync);
void compute_loss(ViewSlot& v, cudaStream_t s);
void compute_loss_value(ViewSlot& v, cudaStream_t s);  // sums only (metrics)

}  // namespace ngsb
