// include/ngs_ref/ngs/trainer.hpp — drop-in replacement of the reference's
// proj/include/ngs/trainer.hpp whose Trainer runs on the B200 (libngs_b200.so).
//
// Put this directory ahead of the reference's include directory:
//
//   g++ -std=c++20 -I <repo>/include/ngs_ref -I <repo>/include -I <reference>/proj/include ...
//       -L <repo>/paper_2501_13975_b200/lib -lngs_b200
//
// and every `#include "ngs/trainer.hpp"` of an unmodified reference translation
// unit (its tests, bench.hpp, the CLI) binds to the GPU trainer, while all the
// other reference headers (Scene, Camera, Image, Dataset, RasterOptions,
// LossConfig, NewtonOptions, Rng, save_scene, the exception types) stay the
// reference's own. The public surface below follows trainer.hpp: TrainConfig /
// IterationReport / LearningRates / OptimizerKind / AdamState / gd_update with the
// same fields, defaults and validation, and Trainer(scene, dataset, config) with
// scene(), dataset(), neighbors(), step_count(), barrier_weight(), step(view),
// probe_metrics() and run(csv). Errors are the reference's exception types
// (core.hpp:30-48), mapped from the C-ABI status codes.
//
// Differences a caller can observe:
//  * parameters live on the device in FP32 (scene() converts back to FP64 and
//    renormalises the quaternions, as renormalize_quaternion does);
//  * the trainer runs in the library's deterministic mode (exact fixed-point
//    accumulation), so the reference's "same seed -> same curve" contract holds;
//  * `threads` is ignored; `dump_hessian_path` is not supported (the per-kernel
//    systems stay on the device).
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <filesystem>
#include <optional>
#include <ostream>
#include <string>
#include <vector>

#include "ngs/camera.hpp"
#include "ngs/core.hpp"
#include "ngs/loss.hpp"
#include "ngs/metrics.hpp"
#include "ngs/newton.hpp"
#include "ngs/rasterizer.hpp"
#include "ngs/scene.hpp"
#include "ngs/scene_io.hpp"
#include "ngs/secondary.hpp"
#include "ngs_b200.h"
#include "ngs_b200_ext.h"

namespace ngs {

enum class OptimizerKind { newton, gd, adam };

inline const char* optimizer_name(OptimizerKind k) {
    return k == OptimizerKind::newton ? "newton" : k == OptimizerKind::gd ? "gd" : k == OptimizerKind::adam ? "adam" : "?";
}

/// First-order baseline learning rates (trainer.hpp: LearningRates).
struct LearningRates {
    double position = 2.0;
    double rotation = 40.0;
    double scaling = 1.0;
    double opacity = 24.0;
    double color = 60.0;

    static LearningRates adam_defaults() {
        LearningRates r;
        r.position = 1.6e-4;
        r.rotation = 1.0e-3;
        r.scaling = 5.0e-3;
        r.opacity = 2.5e-2;
        r.color = 2.5e-3;
        return r;
    }
};

struct TrainConfig {
    OptimizerKind optimizer = OptimizerKind::newton;
    std::array<Attribute, 5> order = {Attribute::position, Attribute::rotation, Attribute::scaling,
                                      Attribute::opacity, Attribute::color};
    int epochs = 1;
    std::uint64_t seed = 0;
    LossConfig loss;
    int knn = kDefaultKnn;
    int secondary_downsample = kDefaultSecondaryDownsample;
    LearningRates gd_lr;
    LearningRates adam_lr = LearningRates::adam_defaults();
    int probe_cadence = 1;
    int threads = 1;  // CPU thread count of the reference; the device ignores it
    NewtonOptions newton;
    double barrier_decay = 0.5;
    double barrier_floor = 1e-6;
    RasterOptions raster;
    std::string checkpoint_dir;
    std::string dump_hessian_path;  // not supported on the device (must stay empty)

    void validate() const {
        loss.validate();
        std::array<bool, 5> seen{};
        for (Attribute a : order) seen[static_cast<int>(a)] = true;
        if (!std::all_of(seen.begin(), seen.end(), [](bool b) { return b; }))
            throw InvalidInput("train config: order must be a permutation of all five");
        if (epochs < 0) throw InvalidInput("train config: epochs must be >= 0");
        if (knn < 0) throw InvalidInput("train config: knn must be >= 0");
    }
};

struct IterationReport {
    int step = 0;
    int image_id = -1;
    double probe_loss = 0.0;
    double probe_psnr = 0.0;
    double probe_ssim = 1.0;
    std::array<double, 5> delta_norms{};  // indexed by Attribute
    double dt_ms = 0.0;
};

inline double gd_update(double grad, double lr) { return -lr * grad; }

/// Host-side Adam moments (the device trainer keeps its own; this type is part of
/// the reference interface and its unit tests).
struct AdamState {
    VecX m, v;
    int t = 0;
    double beta1 = 0.9, beta2 = 0.999, eps = 1e-8;

    explicit AdamState(int n = 0) : m(VecX::Zero(n)), v(VecX::Zero(n)) {}
    void begin_step() { ++t; }
    double update(int i, double grad, double lr) {
        m[i] = beta1 * m[i] + (1.0 - beta1) * grad;
        v[i] = beta2 * v[i] + (1.0 - beta2) * grad * grad;
        const double mh = m[i] / (1.0 - std::pow(beta1, t));
        const double vh = v[i] / (1.0 - std::pow(beta2, t));
        return -lr * mh / (std::sqrt(vh) + eps);
    }
};

namespace b200_detail {

inline void check(int32_t st) {
    if (st == NGS_OK) return;
    const std::string msg = ngs_last_error();
    switch (st) {
        case NGS_ERR_INVALID_INPUT: throw InvalidInput(msg);
        case NGS_ERR_DEGENERATE: throw DegenerateGeometry(msg);
        case NGS_ERR_NUMERICAL: throw NumericalError(msg);
        case NGS_ERR_IO: throw IoError(msg);
        default: throw std::runtime_error("libngs_b200: " + msg);
    }
}

inline ngs_camera to_c(const Camera& c) {
    ngs_camera o{};
    for (int r = 0; r < 4; ++r)
        for (int k = 0; k < 4; ++k) {
            o.view[4 * r + k] = c.view(r, k);
            o.proj[4 * r + k] = c.proj(r, k);
        }
    o.width = c.width;
    o.height = c.height;
    return o;
}

inline ngs_learning_rates to_c(const LearningRates& l) {
    return ngs_learning_rates{l.position, l.rotation, l.scaling, l.opacity, l.color};
}

}  // namespace b200_detail

/// Trainer with the reference's public interface (trainer.hpp), executing every
/// step on the B200 through the C-ABI.
class Trainer {
public:
    struct ProbeMetrics {
        double loss = 0.0;
        double psnr = 0.0;
        double ssim = 1.0;
    };

    Trainer(Scene scene, Dataset dataset, TrainConfig config)
        : scene_(std::move(scene)), dataset_(std::move(dataset)), config_(std::move(config)), rng_(config_.seed) {
        using b200_detail::check;
        config_.validate();
        if (dataset_.cameras.empty()) throw InvalidInput("trainer: dataset has no cameras");
        if (dataset_.train_ids.empty()) throw InvalidInput("trainer: no training views");
        if (!config_.dump_hessian_path.empty())
            throw InvalidInput("trainer (B200): dump_hessian_path is not supported on the device");
        validate_scene(scene_);
        barrier_weight_ = config_.newton.barrier_weight;
        check(ngs_context_create(0, &ctx_));
        check(ngs_set_deterministic(ctx_, 1));
        upload_scene();
        configure();
        neighbors_.assign(dataset_.cameras.size(), {});
        for (std::size_t v = 0; v < dataset_.cameras.size(); ++v) {
            int32_t buf[NGS_MAX_VIEW_SLOTS], n = 0;
            check(ngs_trainer_neighbors(ctx_, static_cast<int32_t>(v), buf, NGS_MAX_VIEW_SLOTS, &n));
            neighbors_[v].assign(buf, buf + std::min<int32_t>(n, NGS_MAX_VIEW_SLOTS));
        }
    }
    Trainer(const Trainer&) = delete;
    Trainer& operator=(const Trainer&) = delete;
    ~Trainer() {
        if (ctx_) ngs_context_destroy(ctx_);
    }

    /// The current parameters (downloaded from the device on demand).
    const Scene& scene() const {
        if (dirty_) download_scene();
        return scene_;
    }
    const Dataset& dataset() const { return dataset_; }
    const std::vector<std::vector<int>>& neighbors() const { return neighbors_; }
    int step_count() const { return step_count_; }
    double barrier_weight() const { return barrier_weight_; }

    IterationReport step(int view_id) {
        if (!std::isfinite(probe_loss_cache_)) throw NumericalError("trainer: non-finite probe loss, aborting");
        ngs_iteration_report r{};
        dirty_ = true;
        b200_detail::check(ngs_trainer_step(ctx_, view_id, &r));
        IterationReport out;
        out.step = ++step_count_;
        out.image_id = r.image_id;
        for (int i = 0; i < 5; ++i) out.delta_norms[i] = r.delta_norms[i];
        out.dt_ms = r.dt_ms;
        return out;
    }

    ProbeMetrics probe_metrics() {
        ngs_metrics m{};
        b200_detail::check(ngs_trainer_probe(ctx_, &m));
        probe_loss_cache_ = m.loss;
        return ProbeMetrics{m.loss, m.psnr, m.ssim};
    }

    /// Epochs of shuffled training views (the reference Rng, seeded with config.seed),
    /// probes every probe_cadence steps, barrier decay per epoch, optional per-epoch
    /// checkpoints (save_scene) and CSV rows in the reference's column layout.
    std::vector<IterationReport> run(std::ostream* csv = nullptr) {
        std::vector<IterationReport> rows;
        if (csv) *csv << "step,image_id,probe_loss,psnr,ssim,dt_ms\n";
        IterationReport initial;
        ProbeMetrics last = probe_metrics();
        initial.probe_loss = last.loss;
        initial.probe_psnr = last.psnr;
        initial.probe_ssim = last.ssim;
        rows.push_back(initial);
        if (csv) csv_row(*csv, initial);
        for (int epoch = 0; epoch < config_.epochs; ++epoch) {
            std::vector<int> order = dataset_.train_ids;
            rng_.shuffle(order);
            for (int view_id : order) {
                IterationReport report = step(view_id);
                if (config_.probe_cadence > 0 && step_count_ % config_.probe_cadence == 0) last = probe_metrics();
                report.probe_loss = last.loss;
                report.probe_psnr = last.psnr;
                report.probe_ssim = last.ssim;
                rows.push_back(report);
                if (csv) csv_row(*csv, report);
            }
            barrier_weight_ = std::max(config_.barrier_floor, barrier_weight_ * config_.barrier_decay);
            b200_detail::check(ngs_trainer_set_barrier_weight(ctx_, barrier_weight_));
            if (!config_.checkpoint_dir.empty()) {
                namespace fs = std::filesystem;
                fs::create_directories(config_.checkpoint_dir);
                save_scene((fs::path(config_.checkpoint_dir) / ("epoch_" + std::to_string(epoch) + ".json")).string(),
                           scene());
            }
        }
        return rows;
    }

private:
    static void csv_row(std::ostream& os, const IterationReport& r) {
        os << r.step << ',' << r.image_id << ',';
        const auto prec = os.precision(17);
        os << r.probe_loss << ',' << r.probe_psnr << ',' << r.probe_ssim;
        os.precision(prec);
        os << ',' << r.dt_ms << '\n';
    }

    void upload_scene() {
        const std::size_t n = scene_.kernels.size();
        std::vector<double> p(3 * n), s(3 * n), q(4 * n), sig(n), sh(48 * n);
        for (std::size_t k = 0; k < n; ++k) {
            const GaussianKernel& g = scene_.kernels[k];
            for (int i = 0; i < 3; ++i) {
                p[3 * k + i] = g.position[i];
                s[3 * k + i] = g.scale[i];
            }
            for (int i = 0; i < 4; ++i) q[4 * k + i] = g.quaternion[i];
            sig[k] = g.sigma;
            for (int ch = 0; ch < 3; ++ch)
                for (int i = 0; i < 16; ++i) sh[48 * k + 16 * ch + i] = g.sh[ch][i];
        }
        ngs_scene cs{};
        cs.count = static_cast<int32_t>(n);
        cs.sh_degree = scene_.sh_degree;
        for (int i = 0; i < 3; ++i) cs.background[i] = scene_.background[i];
        cs.position = p.data();
        cs.scale = s.data();
        cs.quaternion = q.data();
        cs.sigma = sig.data();
        cs.sh = sh.data();
        b200_detail::check(ngs_set_scene(ctx_, &cs));
    }

    void download_scene() const {
        const std::size_t n = scene_.kernels.size();
        std::vector<double> p(3 * n), s(3 * n), q(4 * n), sig(n), sh(48 * n);
        ngs_scene cs{};
        cs.count = static_cast<int32_t>(n);
        cs.position = p.data();
        cs.scale = s.data();
        cs.quaternion = q.data();
        cs.sigma = sig.data();
        cs.sh = sh.data();
        b200_detail::check(ngs_get_scene(ctx_, &cs));
        for (std::size_t k = 0; k < n; ++k) {
            GaussianKernel& g = scene_.kernels[k];
            g.position = Vec3(p[3 * k], p[3 * k + 1], p[3 * k + 2]);
            g.scale = Vec3(s[3 * k], s[3 * k + 1], s[3 * k + 2]);
            g.quaternion = renormalize_quaternion(Vec4(q[4 * k], q[4 * k + 1], q[4 * k + 2], q[4 * k + 3]));
            g.sigma = sig[k];
            for (int ch = 0; ch < 3; ++ch)
                for (int i = 0; i < 16; ++i) g.sh[ch][i] = sh[48 * k + 16 * ch + i];
        }
        dirty_ = false;
    }

    void configure() {
        ngs_train_config c{};
        ngs_train_config_default(&c);
        for (int i = 0; i < 5; ++i) c.order[i] = static_cast<int32_t>(config_.order[i]);
        c.epochs = config_.epochs;
        c.seed = config_.seed;
        c.knn = config_.knn;
        c.secondary_downsample = config_.secondary_downsample;
        c.threads = config_.threads;
        c.barrier_decay = config_.barrier_decay;
        c.barrier_floor = config_.barrier_floor;
        const NewtonOptions& nw = config_.newton;
        c.newton = ngs_newton_options{nw.mu_min,        nw.eig_floor_rel, nw.step_cap_factor,
                                      nw.scale_cap_factor, nw.color_cap,  nw.theta_cap,
                                      nw.barrier_weight,  nw.max_backtrack, nw.eigengap_rel};
        const RasterOptions& ro = config_.raster;
        c.raster = ngs_raster_options{ro.lambda_lp, ro.alpha_cutoff, ro.t_min, ro.tiled ? 1 : 0, config_.threads};
        const LossConfig& lc = config_.loss;
        c.loss = ngs_loss_config{lc.lambda, lc.c1, lc.c2, lc.window, lc.window_sigma};
        c.probe_cadence = config_.probe_cadence;
        c.optimizer = config_.optimizer == OptimizerKind::newton ? NGS_OPT_NEWTON
                      : config_.optimizer == OptimizerKind::gd   ? NGS_OPT_GD
                                                                 : NGS_OPT_ADAM;
        c.gd_lr = b200_detail::to_c(config_.gd_lr);
        c.adam_lr = b200_detail::to_c(config_.adam_lr);
        std::vector<ngs_camera> cams;
        std::vector<const double*> targets;
        for (std::size_t i = 0; i < dataset_.cameras.size(); ++i) {
            cams.push_back(b200_detail::to_c(dataset_.cameras[i]));
            targets.push_back(dataset_.targets.at(i).data.data());
        }
        std::vector<const double*> sec;
        const bool have_sec = dataset_.secondary_targets.size() == dataset_.cameras.size();
        if (have_sec)
            for (const Image& im : dataset_.secondary_targets) sec.push_back(im.data.data());
        std::vector<int32_t> train(dataset_.train_ids.begin(), dataset_.train_ids.end());
        std::vector<int32_t> probe(dataset_.probe_ids.begin(), dataset_.probe_ids.end());
        b200_detail::check(ngs_trainer_configure(
            ctx_, &c, static_cast<int32_t>(cams.size()), cams.data(), targets.data(), static_cast<int32_t>(train.size()),
            train.data(), static_cast<int32_t>(probe.size()), probe.empty() ? nullptr : probe.data(),
            have_sec ? sec.data() : nullptr, have_sec ? dataset_.secondary_downsample : 0));
    }

    ngs_context* ctx_ = nullptr;
    mutable Scene scene_;
    mutable bool dirty_ = false;
    Dataset dataset_;
    TrainConfig config_;
    Rng rng_;
    std::vector<std::vector<int>> neighbors_;
    int step_count_ = 0;
    double barrier_weight_ = 1e-4;
    double probe_loss_cache_ = 0.0;
};

}  // namespace ngs
