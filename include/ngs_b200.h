/*
 * ngs_b200.h — C-ABI drop-in boundary for the 3DGS² local-Newton training path.
 *
 * Plain C: pointers, sizes and POD structs only (no torch / CUDA types), so
 * the same header is implemented by
 *   - libngs_b200.so   (paper_2501_13975_b200/csrc, CUDA sm_100a — the product)
 *   - oracle/_ref/libngs_ref.so (the UNMODIFIED reference headers compiled
 *     against a test-only Eigen shim — the parity oracle / CPU baseline)
 * and parity tests drive both through one binding.
 *
 * Every entry point cites the reference interface it replaces
 * (/root/reference/proj/include/ngs/<file>:<line>). Host data is float64, the
 * reference's type (core.hpp:15-24); the CUDA implementation converts to its
 * FP32 device layout on upload and back on download.
 *
 * Errors: every function returns an ngs_status; the message of the last
 * failure on the calling thread is available from ngs_last_error(). The
 * status codes map 1:1 onto the reference exception types (core.hpp:30-48).
 */
#ifndef NGS_B200_H
#define NGS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NGS_ABI_VERSION 2
#define NGS_SH_COEFFS 16        /* scene.hpp:11 kShCoeffsPerChannel */
#define NGS_MAX_VIEW_SLOTS 16   /* primary + up to 15 secondary view contexts */

typedef enum {
    NGS_OK = 0,
    NGS_ERR_INVALID_INPUT = 1, /* ngs::InvalidInput       core.hpp:30-33 */
    NGS_ERR_DEGENERATE = 2,    /* ngs::DegenerateGeometry core.hpp:35-38 */
    NGS_ERR_NUMERICAL = 3,     /* ngs::NumericalError     core.hpp:40-43 */
    NGS_ERR_IO = 4,            /* ngs::IoError            core.hpp:45-48 */
    NGS_ERR_CUDA = 5,          /* device / driver failure (no reference analogue) */
    NGS_ERR_NCCL = 6,          /* collective failure (no reference analogue) */
    NGS_ERR_INTERNAL = 7
} ngs_status;

/* newton.hpp:21 enum class Attribute */
typedef enum {
    NGS_POSITION = 0,
    NGS_ROTATION = 1,
    NGS_SCALING = 2,
    NGS_OPACITY = 3,
    NGS_COLOR = 4
} ngs_attribute;

/* scene.hpp:16-28 GaussianKernel / Scene, as per-field arrays over kernels.
 * position[3n] xyz, scale[3n] (linear std-devs), quaternion[4n] (w,x,y,z),
 * sigma[n] (linear opacity), sh[48n] (per kernel: R0..R15,G0..G15,B0..B15). */
typedef struct {
    int32_t count;
    int32_t sh_degree;
    double background[3];
    double* position;
    double* scale;
    double* quaternion;
    double* sigma;
    double* sh;
} ngs_scene;

/* camera.hpp:17-45 Camera(view, proj, w, h); matrices row-major as in the
 * dataset manifest (scene_io.hpp:93-95). */
typedef struct {
    double view[16];
    double proj[16];
    int32_t width;
    int32_t height;
} ngs_camera;

/* rasterizer.hpp:25-40 RasterOptions */
typedef struct {
    double lambda_lp;
    double alpha_cutoff;
    double t_min;
    int32_t tiled;
    int32_t threads;
} ngs_raster_options;

/* loss.hpp:11-22 LossConfig */
typedef struct {
    double lambda;
    double c1;
    double c2;
    int32_t window;
    double window_sigma;
} ngs_loss_config;

/* newton.hpp:58-68 NewtonOptions */
typedef struct {
    double mu_min;
    double eig_floor_rel;
    double step_cap_factor;
    double scale_cap_factor;
    double color_cap;
    double theta_cap;
    double barrier_weight;
    int32_t max_backtrack;
    double eigengap_rel;
} ngs_newton_options;

/* trainer.hpp:24 OptimizerKind */
typedef enum { NGS_OPT_NEWTON = 0, NGS_OPT_GD = 1, NGS_OPT_ADAM = 2 } ngs_optimizer;

/* trainer.hpp:40-56 LearningRates (first-order baselines) */
typedef struct {
    double position;
    double rotation;
    double scaling;
    double opacity;
    double color;
} ngs_learning_rates;

/* trainer.hpp:58-88 TrainConfig. */
typedef struct {
    int32_t order[5];        /* permutation of ngs_attribute */
    int32_t epochs;
    uint64_t seed;
    int32_t knn;
    int32_t secondary_downsample;
    int32_t threads;         /* CPU implementations only */
    double barrier_decay;
    double barrier_floor;
    ngs_newton_options newton;
    ngs_raster_options raster;
    ngs_loss_config loss;
    int32_t host_targets;    /* CUDA: keep targets in pinned host memory and
                                upload the step's 1+K images inside each step */
    int32_t probe_cadence;   /* TrainConfig::probe_cadence: probe every N steps in run() */
    int32_t optimizer;       /* ngs_optimizer: Newton (the hot path) or the GD / Adam baselines
                                (first_order_step, trainer.hpp:419-509) */
    ngs_learning_rates gd_lr;
    ngs_learning_rates adam_lr;
} ngs_train_config;

/* Trainer::ProbeMetrics (trainer.hpp:209-213); also one view's
 * total_loss_value / psnr / ssim_metric (loss.hpp:359-375, metrics.hpp:14-30). */
typedef struct {
    double loss;
    double psnr;
    double ssim;
} ngs_metrics;

/* trainer.hpp:90-98 IterationReport */
typedef struct {
    int32_t step;
    int32_t image_id;
    double probe_loss;
    double probe_psnr;
    double probe_ssim;
    double delta_norms[5];   /* indexed by ngs_attribute */
    double dt_ms;
} ngs_iteration_report;

/* Sizes of one view context (rasterizer.hpp:59-67 SplatList). */
typedef struct {
    int32_t width;
    int32_t height;
    int32_t tiles_x;
    int32_t tiles_y;
    int32_t entries;   /* projected (non-culled) kernels */
    int32_t pairs;     /* (tile, entry) pairs == tile_indices length */
} ngs_view_info;

/* Splat list read-back (rasterizer.hpp:49-67), entries in sorted order
 * (ascending depth, ties by kernel id). Any pointer may be NULL. */
typedef struct {
    int32_t* kernel;        /* [entries] */
    double* pixel;          /* [2*entries] */
    double* depth;          /* [entries] */
    double* cov2d;          /* [4*entries] row-major 2x2 (low-pass included) */
    double* view_color;     /* [3*entries] */
    uint8_t* clamped;       /* [3*entries] */
    double* bbox;           /* [4*entries] min.x, min.y, max.x, max.y */
    int32_t* tile_offsets;  /* [tiles+1] */
    int32_t* tile_indices;  /* [pairs] */
} ngs_splat_list;

/* Per-kernel assembled terms of one attribute, summed over primary and
 * secondary views (the accumulation inside solve_*, newton.hpp:591-597 …).
 * Layout per kernel k (NULL pointers are skipped):
 *   position: grad[3k..], hess[9k..] (3x3 row-major)        newton.hpp:256-260
 *   rotation: grad[k], hess[k]                              newton.hpp:345-349
 *   scaling:  grad[2k..], hess[4k..] (each view's eigenbasis) newton.hpp:406-410
 *   opacity:  grad[k], hess[k] (data terms, no barrier)     newton.hpp:507-526
 *   color:    grad[3*16*k + 16*ch + i],
 *             hess[3*256*k + 256*ch + 16*i + j]              newton.hpp:528-532 */
typedef struct {
    double* grad;
    double* hess;
    uint8_t* visible;
} ngs_terms;

/* Per-kernel solve results (newton.hpp:582-811). NULL pointers are skipped.
 *   delta:  position dp[3k], rotation theta[k], scaling ds[3k],
 *           opacity new_sigma[k], color delta[3*16*k + 16*ch + i]
 *   accepted[k]: LocalNewtonSystem::accepted (scaling backtrack failure)
 *   degenerate[k]: scaling subspace degenerate flag (newton.hpp:149)
 *   delta_norm_sq: the trainer's per-pass report sum (trainer.hpp:339-411) */
typedef struct {
    double* delta;
    uint8_t* accepted;
    uint8_t* degenerate;
    double delta_norm_sq;
} ngs_solve_result;

/* ---- library ---------------------------------------------------------- */
int32_t ngs_abi_version(void);
const char* ngs_backend(void);          /* "cuda-sm_100a" | "reference-cpu" */
const char* ngs_last_error(void);

void ngs_raster_options_default(ngs_raster_options* out);   /* RasterOptions{}            */
void ngs_raster_options_reference(ngs_raster_options* out); /* RasterOptions::reference() */
void ngs_loss_config_default(ngs_loss_config* out);
void ngs_newton_options_default(ngs_newton_options* out);
void ngs_train_config_default(ngs_train_config* out);

/* ---- context: owns the scene, view contexts and trainer state --------- */
typedef struct ngs_context ngs_context;

int32_t ngs_context_create(int32_t device, ngs_context** out);
int32_t ngs_context_destroy(ngs_context* ctx);
/* Determinism (SURVEY.md §8(b) threading row; the reference is deterministic for a
 * fixed seed and thread count): on != 0 makes every per-Gaussian accumulation an
 * exact integer fixed-point sum (no floating-point atomics), so repeated runs give
 * bitwise-identical parameters. Off by default (FP64 atomics, same results up to
 * summation-order rounding). */
int32_t ngs_set_deterministic(ngs_context* ctx, int32_t on);

/* Scene upload / download (validate_scene, scene.hpp:209-217). */
int32_t ngs_set_scene(ngs_context* ctx, const ngs_scene* scene);
int32_t ngs_get_scene_info(ngs_context* ctx, int32_t* count, int32_t* sh_degree);
int32_t ngs_get_scene(ngs_context* ctx, ngs_scene* out); /* caller-allocated arrays */

/* render(scene, camera, options).image — rasterizer.hpp:444-449.
 * rgb_out: 3*width*height doubles, row-major, channel-interleaved. */
int32_t ngs_render(ngs_context* ctx, const ngs_camera* camera, const ngs_raster_options* options,
                   double* rgb_out);

/* build_view_context(scene, camera, target, raster, loss) — newton.hpp:101-118.
 * Renders the context's current scene into view slot `slot`, evaluates the
 * per-pixel loss derivative fields, and returns the loss value. */
int32_t ngs_build_view(ngs_context* ctx, int32_t slot, const ngs_camera* camera,
                       const double* target_rgb, const ngs_raster_options* raster,
                       const ngs_loss_config* loss, double* loss_value);
int32_t ngs_get_view_info(ngs_context* ctx, int32_t slot, ngs_view_info* out);
int32_t ngs_view_splats(ngs_context* ctx, int32_t slot, ngs_splat_list* out);
int32_t ngs_view_image(ngs_context* ctx, int32_t slot, double* rgb_out);
/* PixelLossDerivatives (loss.hpp:41-55): grad/hess 3 per pixel. */
int32_t ngs_view_loss_derivs(ngs_context* ctx, int32_t slot, double* grad_out, double* hess_out);

/* Accumulate-Hessian: `<attr>_terms(k, view)` summed over primary + secondary
 * slots for ALL kernels (newton.hpp:266-574, 591-597 …). Rotation uses the
 * primary view direction as axis (newton.hpp:638). */
int32_t ngs_accumulate(ngs_context* ctx, ngs_attribute attr, int32_t primary_slot,
                       const int32_t* secondary_slots, int32_t n_secondary,
                       const ngs_newton_options* options, ngs_terms* out);

/* Newton step: solve_<attr> for ALL kernels (newton.hpp:588-811) and, if
 * `commit`, commit_<attr> (newton.hpp:817-844) with Jacobi semantics. */
int32_t ngs_newton_step(ngs_context* ctx, ngs_attribute attr, int32_t primary_slot,
                        const int32_t* secondary_slots, int32_t n_secondary,
                        const ngs_newton_options* options, int32_t commit,
                        ngs_solve_result* out);

/* ---- trainer (trainer.hpp:128-175, 185-207, 299-417) ------------------ */
/* Dataset (scene_io.hpp:114-121): targets[i] is 3*w*h doubles for camera i;
 * secondary_targets may be NULL (then box-filtered, image.hpp:39-62). */
int32_t ngs_trainer_configure(ngs_context* ctx, const ngs_train_config* config,
                              int32_t n_cameras, const ngs_camera* cameras,
                              const double* const* targets, int32_t n_train,
                              const int32_t* train_ids, int32_t n_probe,
                              const int32_t* probe_ids,
                              const double* const* secondary_targets,
                              int32_t secondary_targets_downsample);
int32_t ngs_trainer_neighbors(ngs_context* ctx, int32_t view_id, int32_t* out, int32_t capacity,
                              int32_t* n_out);
/* Trainer::step(view_id) — one step on one training view: newton_step
 * (trainer.hpp:299-417), or first_order_step (GD / Adam, trainer.hpp:419-509)
 * when config.optimizer selects a baseline. */
int32_t ngs_trainer_step(ngs_context* ctx, int32_t view_id, ngs_iteration_report* report);
int32_t ngs_trainer_barrier_weight(ngs_context* ctx, double* out);
/* Trainer::probe_metrics (trainer.hpp:215-233): render every probe view (the
 * training views when there are none), mean total_loss_value / psnr (inf
 * counted as 99) / ssim_metric. */
int32_t ngs_trainer_probe(ngs_context* ctx, ngs_metrics* out);
/* Trainer::run (trainer.hpp:238-277) without the CSV / checkpoint I/O: rows[0]
 * is the initial probe row (step 0), then one row per step over `epochs`
 * epochs of the train ids shuffled by the config-seeded Rng (core.hpp:52-81),
 * re-probing every probe_cadence steps and decaying the barrier weight per
 * epoch. *n_rows = 1 + epochs * n_train (capacity must be at least that). */
int32_t ngs_trainer_run(ngs_context* ctx, ngs_iteration_report* rows, int32_t capacity, int32_t* n_rows);

/* ---- evaluation (metrics.hpp, loss.hpp:359-375) ------------------------ */
/* render(scene, camera, raster) against target_rgb (3*w*h doubles,
 * interleaved): total_loss_value, psnr (+inf for identical images) and
 * ssim_metric (mean SSIM over channels with the loss config's window). */
int32_t ngs_view_metrics(ngs_context* ctx, const ngs_camera* camera, const double* target_rgb,
                         const ngs_raster_options* raster, const ngs_loss_config* loss, ngs_metrics* out);

#ifdef __cplusplus
}
#endif

#endif /* NGS_B200_H */
