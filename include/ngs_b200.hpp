// ngs_b200.hpp — C++ host interface mirroring the reference's proj/include/ngs
// API for the Newton training path, implemented over the C-ABI (ngs_b200.h)
// by libngs_b200.so (CUDA, sm_100a).
//
// A reference user switches by replacing the ngs:: types/calls below with
// ngs::b200:: ones (same names, argument meaning and exception types):
//
//   reference (float64 CPU)                      this header (CUDA)
//   ngs::Scene / GaussianKernel  scene.hpp:16-28  ngs::b200::Scene / GaussianKernel
//   ngs::Camera(view, proj, w, h) camera.hpp:30   ngs::b200::Camera(view, proj, w, h)
//   ngs::render(...)             rasterizer.hpp:444  Context::render(...)
//   ngs::build_view_context(...) newton.hpp:101   Context::build_view(slot, ...)
//   ngs::<attr>_terms(...)       newton.hpp:266   Context::accumulate(attr, ...) (all kernels)
//   ngs::solve_<attr> + commit   newton.hpp:588   Context::newton_step(attr, ...) (all kernels)
//   ngs::Trainer(scene, dataset, config).step(v)  ngs::b200::Trainer(...).step(v)
//   InvalidInput / DegenerateGeometry / NumericalError / IoError (core.hpp:30-48): same names.
//
// Header-only; no Eigen, no CUDA headers. Link: -lngs_b200 (rpath to the
// package's lib/ directory).
#pragma once

#include <array>
#include <memory>
#include <ostream>
#include <stdexcept>
#include <string>
#include <vector>

#include "ngs_b200.h"

namespace ngs::b200 {

// ---- exceptions (core.hpp:30-48) --------------------------------------------
struct InvalidInput : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DegenerateGeometry : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int32_t status) {
    if (status == NGS_OK) return;
    const std::string msg = ngs_last_error();
    switch (status) {
        case NGS_ERR_INVALID_INPUT: throw InvalidInput(msg);
        case NGS_ERR_DEGENERATE: throw DegenerateGeometry(msg);
        case NGS_ERR_NUMERICAL: throw NumericalError(msg);
        case NGS_ERR_IO: throw IoError(msg);
        default: throw DeviceError(msg);
    }
}

enum class Attribute { position = NGS_POSITION, rotation = NGS_ROTATION, scaling = NGS_SCALING,
                       opacity = NGS_OPACITY, color = NGS_COLOR };

// ---- scene.hpp:16-28 ---------------------------------------------------------
struct GaussianKernel {
    std::array<double, 3> position{0, 0, 0};
    std::array<double, 3> scale{1, 1, 1};
    std::array<double, 4> quaternion{1, 0, 0, 0};  // (w, x, y, z)
    double sigma = 0.5;
    std::array<std::array<double, 16>, 3> sh{};    // channel-major
};

struct Scene {
    std::vector<GaussianKernel> kernels;
    std::array<double, 3> background{0, 0, 0};
    int sh_degree = 3;
};

// ---- camera.hpp:17-45 (row-major 4x4) ----------------------------------------
struct Camera {
    std::array<double, 16> view{1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1};
    std::array<double, 16> proj{1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1};
    int width = 0;
    int height = 0;
    Camera() = default;
    Camera(const std::array<double, 16>& v, const std::array<double, 16>& p, int w, int h)
        : view(v), proj(p), width(w), height(h) {
        if (w < 16 || h < 16) throw InvalidInput("camera: width and height must be >= 16");
    }
    ngs_camera c() const {
        ngs_camera out{};
        for (int i = 0; i < 16; ++i) {
            out.view[i] = view[i];
            out.proj[i] = proj[i];
        }
        out.width = width;
        out.height = height;
        return out;
    }
};

// ---- image.hpp:11-35: RGB float64, row-major, channel-interleaved ------------
struct Image {
    int width = 0, height = 0;
    std::vector<double> data;
    Image() = default;
    Image(int w, int h, double fill = 0.0) : width(w), height(h), data(3u * w * h, fill) {}
};

// ---- option structs with the reference defaults ------------------------------
inline ngs_raster_options raster_defaults() { ngs_raster_options o; ngs_raster_options_default(&o); return o; }
inline ngs_raster_options raster_reference() { ngs_raster_options o; ngs_raster_options_reference(&o); return o; }
inline ngs_loss_config loss_defaults() { ngs_loss_config o; ngs_loss_config_default(&o); return o; }
inline ngs_newton_options newton_defaults() { ngs_newton_options o; ngs_newton_options_default(&o); return o; }
inline ngs_train_config train_defaults() { ngs_train_config o; ngs_train_config_default(&o); return o; }

using IterationReport = ngs_iteration_report;  // trainer.hpp:90-98
using ProbeMetrics = ngs_metrics;             // trainer.hpp:209-213 (loss, psnr, ssim)

// Per-field host arrays for the C-ABI scene (scene.hpp layout -> ngs_scene).
struct SceneArrays {
    std::vector<double> p, s, q, sigma, sh;
    ngs_scene view{};
    explicit SceneArrays(const Scene& sc) {
        const size_t n = sc.kernels.size();
        p.resize(3 * n); s.resize(3 * n); q.resize(4 * n); sigma.resize(n); sh.resize(48 * n);
        for (size_t k = 0; k < n; ++k) {
            const auto& g = sc.kernels[k];
            for (int i = 0; i < 3; ++i) { p[3 * k + i] = g.position[i]; s[3 * k + i] = g.scale[i]; }
            for (int i = 0; i < 4; ++i) q[4 * k + i] = g.quaternion[i];
            sigma[k] = g.sigma;
            for (int ch = 0; ch < 3; ++ch)
                for (int i = 0; i < 16; ++i) sh[48 * k + 16 * ch + i] = g.sh[ch][i];
        }
        view.count = static_cast<int32_t>(n);
        view.sh_degree = sc.sh_degree;
        for (int i = 0; i < 3; ++i) view.background[i] = sc.background[i];
        view.position = p.data(); view.scale = s.data(); view.quaternion = q.data();
        view.sigma = sigma.data(); view.sh = sh.data();
    }
};

// Terms of one attribute for all kernels (layout: ngs_b200.h ngs_terms).
struct Terms {
    std::vector<double> grad, hess;
    std::vector<uint8_t> visible;
};
// Solve results for all kernels (layout: ngs_b200.h ngs_solve_result).
struct SolveResults {
    std::vector<double> delta;
    std::vector<uint8_t> accepted, degenerate;
    double delta_norm_sq = 0.0;
};

// One device context: scene + view contexts (ViewContext, newton.hpp:86-118).
class Context {
public:
    explicit Context(int device = 0) {
        ngs_context* c = nullptr;
        check(ngs_context_create(device, &c));
        ctx_.reset(c);
    }
    ngs_context* get() const { return ctx_.get(); }
    // Bitwise-reproducible accumulation (ngs_set_deterministic).
    void set_deterministic(bool on) { check(ngs_set_deterministic(get(), on ? 1 : 0)); }

    void set_scene(const Scene& s) {
        SceneArrays a(s);
        check(ngs_set_scene(get(), &a.view));
    }
    Scene scene() const {
        int32_t n = 0, deg = 0;
        check(ngs_get_scene_info(get(), &n, &deg));
        Scene sc;
        sc.sh_degree = deg;
        sc.kernels.resize(n);
        SceneArrays a(sc);
        check(ngs_get_scene(get(), &a.view));
        for (int k = 0; k < n; ++k) {
            auto& g = sc.kernels[k];
            for (int i = 0; i < 3; ++i) { g.position[i] = a.p[3 * k + i]; g.scale[i] = a.s[3 * k + i]; }
            for (int i = 0; i < 4; ++i) g.quaternion[i] = a.q[4 * k + i];
            g.sigma = a.sigma[k];
            for (int ch = 0; ch < 3; ++ch)
                for (int i = 0; i < 16; ++i) g.sh[ch][i] = a.sh[48 * k + 16 * ch + i];
        }
        for (int i = 0; i < 3; ++i) sc.background[i] = a.view.background[i];
        return sc;
    }

    // render(scene, camera, options).image — rasterizer.hpp:444-449
    Image render(const Camera& cam, const ngs_raster_options& o = raster_defaults()) const {
        Image img(cam.width, cam.height);
        const ngs_camera c = cam.c();
        check(ngs_render(get(), &c, &o, img.data.data()));
        return img;
    }

    // total_loss_value / psnr / ssim_metric of render(scene, cam) against target
    // (loss.hpp:359-375, metrics.hpp:14-30).
    ProbeMetrics view_metrics(const Camera& cam, const Image& target, const ngs_raster_options& ro = raster_defaults(),
                              const ngs_loss_config& lc = loss_defaults()) const {
        ProbeMetrics m{};
        const ngs_camera c = cam.c();
        check(ngs_view_metrics(get(), &c, target.data.data(), &ro, &lc, &m));
        return m;
    }

    // build_view_context — newton.hpp:101-118; returns the loss value.
    double build_view(int slot, const Camera& cam, const Image& target,
                      const ngs_raster_options& r = raster_defaults(), const ngs_loss_config& l = loss_defaults()) {
        if (target.width != cam.width || target.height != cam.height)
            throw InvalidInput("build_view: target size differs from the camera");
        double v = 0;
        const ngs_camera c = cam.c();
        check(ngs_build_view(get(), slot, &c, target.data.data(), &r, &l, &v));
        return v;
    }

    // <attr>_terms over primary + secondaries for all kernels — newton.hpp:266-574
    Terms accumulate(Attribute a, int primary, const std::vector<int32_t>& secondaries,
                     const ngs_newton_options& o = newton_defaults()) const {
        int32_t n = 0, deg = 0;
        check(ngs_get_scene_info(get(), &n, &deg));
        static constexpr int gw[5] = {3, 1, 2, 1, 48}, hw[5] = {9, 1, 4, 1, 768};
        Terms t;
        t.grad.resize(static_cast<size_t>(n) * gw[static_cast<int>(a)]);
        t.hess.resize(static_cast<size_t>(n) * hw[static_cast<int>(a)]);
        t.visible.resize(n);
        ngs_terms out{t.grad.data(), t.hess.data(), t.visible.data()};
        check(ngs_accumulate(get(), static_cast<ngs_attribute>(a), primary, secondaries.data(),
                             static_cast<int32_t>(secondaries.size()), &o, &out));
        return t;
    }

    // solve_<attr> (+ commit_<attr>) for all kernels — newton.hpp:588-844
    SolveResults newton_step(Attribute a, int primary, const std::vector<int32_t>& secondaries,
                             const ngs_newton_options& o = newton_defaults(), bool commit = true) {
        int32_t n = 0, deg = 0;
        check(ngs_get_scene_info(get(), &n, &deg));
        static constexpr int dw[5] = {3, 1, 3, 1, 48};
        SolveResults r;
        r.delta.resize(static_cast<size_t>(n) * dw[static_cast<int>(a)]);
        r.accepted.resize(n);
        r.degenerate.resize(n);
        ngs_solve_result out{r.delta.data(), r.accepted.data(), r.degenerate.data(), 0.0};
        check(ngs_newton_step(get(), static_cast<ngs_attribute>(a), primary, secondaries.data(),
                              static_cast<int32_t>(secondaries.size()), &o, commit ? 1 : 0, &out));
        r.delta_norm_sq = out.delta_norm_sq;
        return r;
    }

private:
    struct Deleter {
        void operator()(ngs_context* c) const { ngs_context_destroy(c); }
    };
    std::unique_ptr<ngs_context, Deleter> ctx_;
};

// Dataset (scene_io.hpp:114-121).
struct Dataset {
    std::vector<Camera> cameras;
    std::vector<Image> targets;
    std::vector<int> train_ids;
    std::vector<int> probe_ids;
    std::vector<Image> secondary_targets;  // optional
    int secondary_downsample = 0;
};

// Trainer(scene, dataset, config) / step(view_id) — trainer.hpp:130-207, 299-417.
class Trainer {
public:
    Trainer(const Scene& scene, const Dataset& ds, const ngs_train_config& cfg = train_defaults(), int device = 0)
        : ctx_(device), epochs_(cfg.epochs), n_train_(static_cast<int>(ds.train_ids.size())) {
        ctx_.set_scene(scene);
        std::vector<ngs_camera> cams;
        std::vector<const double*> tg, st;
        for (const auto& c : ds.cameras) cams.push_back(c.c());
        for (const auto& t : ds.targets) tg.push_back(t.data.data());
        for (const auto& t : ds.secondary_targets) st.push_back(t.data.data());
        if (tg.size() != cams.size()) throw InvalidInput("trainer: one target per camera required");
        check(ngs_trainer_configure(ctx_.get(), &cfg, static_cast<int32_t>(cams.size()), cams.data(), tg.data(),
                                    static_cast<int32_t>(ds.train_ids.size()), ds.train_ids.data(),
                                    static_cast<int32_t>(ds.probe_ids.size()), ds.probe_ids.data(),
                                    st.empty() ? nullptr : st.data(), ds.secondary_downsample));
    }
    IterationReport step(int view_id) {
        IterationReport r{};
        check(ngs_trainer_step(ctx_.get(), view_id, &r));
        return r;
    }
    std::vector<int> neighbors(int view_id) const {
        std::vector<int32_t> buf(64);
        int32_t n = 0;
        check(ngs_trainer_neighbors(ctx_.get(), view_id, buf.data(), 64, &n));
        return std::vector<int>(buf.begin(), buf.begin() + n);
    }
    double barrier_weight() const {
        double w = 0;
        check(ngs_trainer_barrier_weight(ctx_.get(), &w));
        return w;
    }
    // Trainer::probe_metrics — trainer.hpp:215-233.
    ProbeMetrics probe_metrics() {
        ProbeMetrics m{};
        check(ngs_trainer_probe(ctx_.get(), &m));
        return m;
    }
    // Trainer::run — trainer.hpp:238-277 (CSV rows as the reference writes them;
    // checkpoints are not part of this library).
    std::vector<IterationReport> run(std::ostream* csv = nullptr) {
        std::vector<IterationReport> rows(1 + static_cast<size_t>(epochs_ > 0 ? epochs_ : 0) * n_train_);
        int32_t n = 0;
        check(ngs_trainer_run(ctx_.get(), rows.data(), static_cast<int32_t>(rows.size()), &n));
        rows.resize(n);
        if (csv) {
            *csv << "step,image_id,probe_loss,psnr,ssim,dt_ms\n";
            for (const auto& r : rows) {
                *csv << r.step << ',' << r.image_id << ',';
                const auto old = csv->precision(17);
                *csv << r.probe_loss << ',' << r.probe_psnr << ',' << r.probe_ssim;
                csv->precision(old);
                *csv << ',' << r.dt_ms << '\n';
            }
        }
        return rows;
    }
    Scene scene() const { return ctx_.scene(); }
    Context& context() { return ctx_; }

private:
    Context ctx_;
    int epochs_ = 1, n_train_ = 0;
};

}  // namespace ngs::b200
