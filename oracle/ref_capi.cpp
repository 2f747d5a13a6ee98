// oracle/ref_capi.cpp — TEST INFRASTRUCTURE (parity oracle + CPU baseline).
//
// Implements include/ngs_b200.h on top of the UNMODIFIED reference headers in
// /root/reference/proj/include/ngs, compiled against the test-only Eigen shim
// (oracle/eigen_shim). Built by oracle/Makefile into oracle/_ref/libngs_ref.so
// (git-ignored, travels to the GPU box). Only tests/, __graft_entry__.smoke()
// and bench.py's reference / cpu_baseline legs load it — never the product.
//
// Each entry point forwards to the reference function named in the header.
#include <cstring>
#include <memory>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "ngs/metrics.hpp"
#include "ngs/newton.hpp"
#include "ngs/rasterizer.hpp"
#include "ngs/secondary.hpp"
#include "ngs/trainer.hpp"
#include "ngs_b200.h"

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return NGS_OK;
    } catch (const ngs::InvalidInput& e) {
        return fail(NGS_ERR_INVALID_INPUT, e.what());
    } catch (const ngs::DegenerateGeometry& e) {
        return fail(NGS_ERR_DEGENERATE, e.what());
    } catch (const ngs::NumericalError& e) {
        return fail(NGS_ERR_NUMERICAL, e.what());
    } catch (const ngs::IoError& e) {
        return fail(NGS_ERR_IO, e.what());
    } catch (const std::exception& e) {
        return fail(NGS_ERR_INTERNAL, e.what());
    }
}

int env_threads() {
    if (const char* s = std::getenv("NGS_THREADS")) {
        const int t = std::atoi(s);
        if (t > 0) return t;
    }
    return ngs::default_threads();
}

ngs::Mat4 mat4_rowmajor(const double* m) {
    ngs::Mat4 out;
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) out(r, c) = m[4 * r + c];
    return out;
}

ngs::Camera to_camera(const ngs_camera& c) {
    return ngs::Camera(mat4_rowmajor(c.view), mat4_rowmajor(c.proj), c.width, c.height);
}

ngs::RasterOptions to_raster(const ngs_raster_options* o) {
    ngs::RasterOptions r;
    if (!o) return r;
    r.lambda_lp = o->lambda_lp;
    r.alpha_cutoff = o->alpha_cutoff;
    r.t_min = o->t_min;
    r.tiled = o->tiled != 0;
    r.threads = o->threads;
    return r;
}

ngs::LossConfig to_loss(const ngs_loss_config* o) {
    ngs::LossConfig l;
    if (!o) return l;
    l.lambda = o->lambda;
    l.c1 = o->c1;
    l.c2 = o->c2;
    l.window = o->window;
    l.window_sigma = o->window_sigma;
    return l;
}

ngs::NewtonOptions to_newton(const ngs_newton_options* o) {
    ngs::NewtonOptions n;
    if (!o) return n;
    n.mu_min = o->mu_min;
    n.eig_floor_rel = o->eig_floor_rel;
    n.step_cap_factor = o->step_cap_factor;
    n.scale_cap_factor = o->scale_cap_factor;
    n.color_cap = o->color_cap;
    n.theta_cap = o->theta_cap;
    n.barrier_weight = o->barrier_weight;
    n.max_backtrack = o->max_backtrack;
    n.eigengap_rel = o->eigengap_rel;
    return n;
}

ngs::Image to_image(const double* rgb, int w, int h) {
    ngs::Image img(w, h);
    std::memcpy(img.data.data(), rgb, sizeof(double) * 3 * static_cast<std::size_t>(w) * h);
    return img;
}

}  // namespace

struct ngs_context {
    ngs::Scene scene;
    struct Slot {
        std::unique_ptr<ngs::Scene> snapshot;  // ViewContext keeps a raw Scene*
        std::optional<ngs::ViewContext> view;
    };
    std::array<Slot, NGS_MAX_VIEW_SLOTS> slots;
    std::optional<ngs::Trainer> trainer;

    const ngs::Scene& current() const { return trainer ? trainer->scene() : scene; }
    const ngs::ViewContext& view(int slot) const {
        if (slot < 0 || slot >= NGS_MAX_VIEW_SLOTS || !slots[slot].view) {
            throw ngs::InvalidInput("view slot " + std::to_string(slot) + " is empty");
        }
        return *slots[slot].view;
    }
    std::vector<const ngs::ViewContext*> views(const int32_t* ids, int n) const {
        std::vector<const ngs::ViewContext*> out;
        for (int i = 0; i < n; ++i) out.push_back(&view(ids[i]));
        return out;
    }
};

extern "C" {

int32_t ngs_abi_version(void) { return NGS_ABI_VERSION; }
const char* ngs_backend(void) { return "reference-cpu"; }
const char* ngs_last_error(void) { return g_last_error.c_str(); }

void ngs_raster_options_default(ngs_raster_options* out) {
    const ngs::RasterOptions r;
    *out = {r.lambda_lp, r.alpha_cutoff, r.t_min, r.tiled ? 1 : 0, r.threads};
}
void ngs_raster_options_reference(ngs_raster_options* out) {
    const ngs::RasterOptions r = ngs::RasterOptions::reference();
    *out = {r.lambda_lp, r.alpha_cutoff, r.t_min, r.tiled ? 1 : 0, r.threads};
}
void ngs_loss_config_default(ngs_loss_config* out) {
    const ngs::LossConfig l;
    *out = {l.lambda, l.c1, l.c2, l.window, l.window_sigma};
}
void ngs_newton_options_default(ngs_newton_options* out) {
    const ngs::NewtonOptions n;
    *out = {n.mu_min, n.eig_floor_rel, n.step_cap_factor, n.scale_cap_factor, n.color_cap,
            n.theta_cap, n.barrier_weight, n.max_backtrack, n.eigengap_rel};
}
void ngs_train_config_default(ngs_train_config* out) {
    const ngs::TrainConfig t;
    std::memset(out, 0, sizeof(*out));
    for (int i = 0; i < 5; ++i) out->order[i] = static_cast<int32_t>(t.order[i]);
    out->epochs = t.epochs;
    out->seed = t.seed;
    out->knn = t.knn;
    out->secondary_downsample = t.secondary_downsample;
    out->threads = t.threads;
    out->barrier_decay = t.barrier_decay;
    out->barrier_floor = t.barrier_floor;
    ngs_newton_options_default(&out->newton);
    ngs_raster_options_default(&out->raster);
    ngs_loss_config_default(&out->loss);
    out->host_targets = 0;
    out->probe_cadence = t.probe_cadence;
    out->optimizer = static_cast<int32_t>(t.optimizer);
    out->gd_lr = {t.gd_lr.position, t.gd_lr.rotation, t.gd_lr.scaling, t.gd_lr.opacity, t.gd_lr.color};
    out->adam_lr = {t.adam_lr.position, t.adam_lr.rotation, t.adam_lr.scaling, t.adam_lr.opacity, t.adam_lr.color};
}

int32_t ngs_context_create(int32_t /*device*/, ngs_context** out) {
    return guarded([&] { *out = new ngs_context(); });
}
int32_t ngs_context_destroy(ngs_context* ctx) {
    delete ctx;
    return NGS_OK;
}
int32_t ngs_set_deterministic(ngs_context*, int32_t) {
    return NGS_OK;  // the reference is deterministic for a fixed thread count (parallel_for, core.hpp:89-108)
}

int32_t ngs_set_scene(ngs_context* ctx, const ngs_scene* s) {
    return guarded([&] {
        ngs::Scene scene;
        scene.sh_degree = s->sh_degree;
        scene.background = ngs::Vec3(s->background[0], s->background[1], s->background[2]);
        scene.kernels.resize(s->count);
        for (int k = 0; k < s->count; ++k) {
            auto& g = scene.kernels[k];
            g.position = ngs::Vec3(s->position[3 * k], s->position[3 * k + 1], s->position[3 * k + 2]);
            g.scale = ngs::Vec3(s->scale[3 * k], s->scale[3 * k + 1], s->scale[3 * k + 2]);
            g.quaternion = ngs::Vec4(s->quaternion[4 * k], s->quaternion[4 * k + 1],
                                     s->quaternion[4 * k + 2], s->quaternion[4 * k + 3]);
            g.sigma = s->sigma[k];
            for (int ch = 0; ch < 3; ++ch)
                for (int i = 0; i < 16; ++i) g.sh[ch][i] = s->sh[48 * k + 16 * ch + i];
        }
        ngs::validate_scene(scene);
        ctx->scene = std::move(scene);
        ctx->trainer.reset();
    });
}

int32_t ngs_get_scene_info(ngs_context* ctx, int32_t* count, int32_t* sh_degree) {
    return guarded([&] {
        *count = static_cast<int32_t>(ctx->current().kernels.size());
        *sh_degree = ctx->current().sh_degree;
    });
}

int32_t ngs_get_scene(ngs_context* ctx, ngs_scene* s) {
    return guarded([&] {
        const ngs::Scene& scene = ctx->current();
        if (s->count != static_cast<int32_t>(scene.kernels.size())) {
            throw ngs::InvalidInput("ngs_get_scene: count mismatch");
        }
        s->sh_degree = scene.sh_degree;
        for (int i = 0; i < 3; ++i) s->background[i] = scene.background[i];
        for (int k = 0; k < s->count; ++k) {
            const auto& g = scene.kernels[k];
            for (int i = 0; i < 3; ++i) {
                if (s->position) s->position[3 * k + i] = g.position[i];
                if (s->scale) s->scale[3 * k + i] = g.scale[i];
            }
            for (int i = 0; i < 4; ++i)
                if (s->quaternion) s->quaternion[4 * k + i] = g.quaternion[i];
            if (s->sigma) s->sigma[k] = g.sigma;
            if (s->sh)
                for (int ch = 0; ch < 3; ++ch)
                    for (int i = 0; i < 16; ++i) s->sh[48 * k + 16 * ch + i] = g.sh[ch][i];
        }
    });
}

int32_t ngs_render(ngs_context* ctx, const ngs_camera* camera, const ngs_raster_options* options,
                   double* rgb_out) {
    return guarded([&] {
        const ngs::Camera cam = to_camera(*camera);
        const ngs::RenderTarget rt = ngs::render(ctx->current(), cam, to_raster(options));
        std::memcpy(rgb_out, rt.image.data.data(), sizeof(double) * rt.image.data.size());
    });
}

int32_t ngs_build_view(ngs_context* ctx, int32_t slot, const ngs_camera* camera,
                       const double* target_rgb, const ngs_raster_options* raster,
                       const ngs_loss_config* loss, double* loss_value) {
    return guarded([&] {
        if (slot < 0 || slot >= NGS_MAX_VIEW_SLOTS) throw ngs::InvalidInput("bad view slot");
        const ngs::Camera cam = to_camera(*camera);
        auto& s = ctx->slots[slot];
        s.view.reset();
        s.snapshot = std::make_unique<ngs::Scene>(ctx->current());
        s.view = ngs::build_view_context(*s.snapshot, cam, to_image(target_rgb, cam.width, cam.height),
                                         to_raster(raster), to_loss(loss), true);
        if (loss_value) *loss_value = s.view->loss_value;
    });
}

int32_t ngs_get_view_info(ngs_context* ctx, int32_t slot, ngs_view_info* out) {
    return guarded([&] {
        const auto& v = ctx->view(slot);
        out->width = v.list.width;
        out->height = v.list.height;
        out->tiles_x = v.list.tiles_x;
        out->tiles_y = v.list.tiles_y;
        out->entries = static_cast<int32_t>(v.list.entries.size());
        out->pairs = static_cast<int32_t>(v.list.tile_indices.size());
    });
}

int32_t ngs_view_splats(ngs_context* ctx, int32_t slot, ngs_splat_list* out) {
    return guarded([&] {
        const auto& v = ctx->view(slot);
        const auto& L = v.list;
        for (std::size_t i = 0; i < L.entries.size(); ++i) {
            const auto& e = L.entries[i];
            if (out->kernel) out->kernel[i] = e.kernel;
            if (out->pixel) {
                out->pixel[2 * i] = e.proj.pixel.x();
                out->pixel[2 * i + 1] = e.proj.pixel.y();
            }
            if (out->depth) out->depth[i] = e.proj.depth;
            if (out->cov2d)
                for (int r = 0; r < 2; ++r)
                    for (int c = 0; c < 2; ++c) out->cov2d[4 * i + 2 * r + c] = e.proj.cov2d(r, c);
            for (int ch = 0; ch < 3; ++ch) {
                if (out->view_color) out->view_color[3 * i + ch] = e.view_color[ch];
                if (out->clamped) out->clamped[3 * i + ch] = e.color_clamped[ch] ? 1 : 0;
            }
            if (out->bbox) {
                out->bbox[4 * i] = e.bbox_min.x();
                out->bbox[4 * i + 1] = e.bbox_min.y();
                out->bbox[4 * i + 2] = e.bbox_max.x();
                out->bbox[4 * i + 3] = e.bbox_max.y();
            }
        }
        if (out->tile_offsets)
            std::memcpy(out->tile_offsets, L.tile_offsets.data(), sizeof(int32_t) * L.tile_offsets.size());
        if (out->tile_indices)
            std::memcpy(out->tile_indices, L.tile_indices.data(), sizeof(int32_t) * L.tile_indices.size());
    });
}

int32_t ngs_view_image(ngs_context* ctx, int32_t slot, double* rgb_out) {
    return guarded([&] {
        const auto& v = ctx->view(slot);
        std::memcpy(rgb_out, v.rendered.data.data(), sizeof(double) * v.rendered.data.size());
    });
}

int32_t ngs_view_loss_derivs(ngs_context* ctx, int32_t slot, double* grad_out, double* hess_out) {
    return guarded([&] {
        const auto& v = ctx->view(slot);
        if (grad_out) std::memcpy(grad_out, v.loss.grad.data(), sizeof(double) * v.loss.grad.size());
        if (hess_out) std::memcpy(hess_out, v.loss.hess.data(), sizeof(double) * v.loss.hess.size());
    });
}

int32_t ngs_accumulate(ngs_context* ctx, ngs_attribute attr, int32_t primary_slot,
                       const int32_t* secondary_slots, int32_t n_secondary,
                       const ngs_newton_options* options, ngs_terms* out) {
    return guarded([&] {
        const ngs::Scene& scene = ctx->current();
        const auto& primary = ctx->view(primary_slot);
        std::vector<const ngs::ViewContext*> views{&primary};
        for (const auto* v : ctx->views(secondary_slots, n_secondary)) views.push_back(v);
        const ngs::NewtonOptions opts = to_newton(options);
        const int n = static_cast<int>(scene.kernels.size());
        const int nsh = ngs::sh_coeff_count(scene.sh_degree);
        ngs::parallel_for(n, env_threads(), [&](std::size_t lo, std::size_t hi) {
            for (std::size_t kk = lo; kk < hi; ++kk) {
                const int k = static_cast<int>(kk);
                bool visible = false;
                switch (attr) {
                    case NGS_POSITION: {
                        ngs::Vec3 g = ngs::Vec3::Zero();
                        ngs::Mat3 h = ngs::Mat3::Zero();
                        for (const auto* v : views) {
                            const auto t = ngs::position_terms(k, *v);
                            g += t.grad;
                            h += t.hess;
                            visible = visible || t.visible;
                        }
                        for (int i = 0; i < 3; ++i) {
                            if (out->grad) out->grad[3 * k + i] = g[i];
                            for (int j = 0; j < 3; ++j)
                                if (out->hess) out->hess[9 * k + 3 * i + j] = h(i, j);
                        }
                        break;
                    }
                    case NGS_ROTATION: {
                        const ngs::Vec3 axis = ngs::view_direction(primary.camera, scene.kernels[k].position);
                        double g = 0, h = 0;
                        for (const auto* v : views) {
                            const auto t = ngs::rotation_terms(k, axis, *v);
                            g += t.grad;
                            h += t.hess;
                            visible = visible || t.visible;
                        }
                        if (out->grad) out->grad[k] = g;
                        if (out->hess) out->hess[k] = h;
                        break;
                    }
                    case NGS_SCALING: {
                        ngs::Vec2 g = ngs::Vec2::Zero();
                        ngs::Mat2 h = ngs::Mat2::Zero();
                        for (const auto* v : views) {
                            const auto t = ngs::scaling_terms(k, *v, opts.eigengap_rel);
                            g += t.grad;
                            h += t.hess;
                            visible = visible || t.visible;
                        }
                        for (int i = 0; i < 2; ++i) {
                            if (out->grad) out->grad[2 * k + i] = g[i];
                            for (int j = 0; j < 2; ++j)
                                if (out->hess) out->hess[4 * k + 2 * i + j] = h(i, j);
                        }
                        break;
                    }
                    case NGS_OPACITY: {
                        double g = 0, h = 0;
                        for (const auto* v : views) {
                            const auto t = ngs::opacity_data_terms(k, *v);
                            g += t.grad;
                            h += t.hess;
                            visible = visible || t.visible;
                        }
                        if (out->grad) out->grad[k] = g;
                        if (out->hess) out->hess[k] = h;
                        break;
                    }
                    case NGS_COLOR: {
                        std::array<ngs::VecX, 3> g;
                        std::array<ngs::MatX, 3> h;
                        for (int ch = 0; ch < 3; ++ch) {
                            g[ch] = ngs::VecX::Zero(nsh);
                            h[ch] = ngs::MatX::Zero(nsh, nsh);
                        }
                        for (const auto* v : views) {
                            const auto t = ngs::color_terms(k, *v);
                            for (int ch = 0; ch < 3; ++ch) {
                                g[ch] += t.grad[ch];
                                h[ch] += t.hess[ch];
                            }
                            visible = visible || t.visible;
                        }
                        for (int ch = 0; ch < 3; ++ch)
                            for (int i = 0; i < 16; ++i) {
                                if (out->grad) out->grad[48 * k + 16 * ch + i] = i < nsh ? g[ch][i] : 0.0;
                                for (int j = 0; j < 16; ++j)
                                    if (out->hess)
                                        out->hess[768 * k + 256 * ch + 16 * i + j] =
                                            (i < nsh && j < nsh) ? h[ch](i, j) : 0.0;
                            }
                        break;
                    }
                }
                if (out->visible) out->visible[k] = visible ? 1 : 0;
            }
        });
    });
}

int32_t ngs_newton_step(ngs_context* ctx, ngs_attribute attr, int32_t primary_slot,
                        const int32_t* secondary_slots, int32_t n_secondary,
                        const ngs_newton_options* options, int32_t commit, ngs_solve_result* out) {
    return guarded([&] {
        if (ctx->trainer) throw ngs::InvalidInput("ngs_newton_step: context is owned by a trainer");
        ngs::Scene& scene = ctx->scene;
        const auto& primary = ctx->view(primary_slot);
        const auto secs = ctx->views(secondary_slots, n_secondary);
        const ngs::ViewSpan span(secs);
        const ngs::NewtonOptions opts = to_newton(options);
        const int n = static_cast<int>(scene.kernels.size());
        const int nsh = ngs::sh_coeff_count(scene.sh_degree);
        const int threads = env_threads();
        double norm_sq = 0.0;
        auto write_flags = [&](int k, bool accepted, bool degenerate) {
            if (out && out->accepted) out->accepted[k] = accepted ? 1 : 0;
            if (out && out->degenerate) out->degenerate[k] = degenerate ? 1 : 0;
        };
        switch (attr) {
            case NGS_POSITION: {
                std::vector<ngs::PositionSolve> solves(n);
                ngs::parallel_for(n, threads, [&](std::size_t lo, std::size_t hi) {
                    for (std::size_t k = lo; k < hi; ++k)
                        solves[k] = ngs::solve_position(scene, static_cast<int>(k), primary, span, opts);
                });
                for (int k = 0; k < n; ++k) {
                    if (out && out->delta)
                        for (int i = 0; i < 3; ++i) out->delta[3 * k + i] = solves[k].delta_position[i];
                    write_flags(k, solves[k].sys.accepted, false);
                    norm_sq += solves[k].delta_position.squaredNorm();
                    if (commit) ngs::commit_position(scene.kernels[k], solves[k]);
                }
                break;
            }
            case NGS_ROTATION: {
                std::vector<ngs::RotationSolve> solves(n);
                ngs::parallel_for(n, threads, [&](std::size_t lo, std::size_t hi) {
                    for (std::size_t k = lo; k < hi; ++k)
                        solves[k] = ngs::solve_rotation(scene, static_cast<int>(k), primary, span, opts);
                });
                for (int k = 0; k < n; ++k) {
                    if (out && out->delta) out->delta[k] = solves[k].theta;
                    write_flags(k, solves[k].sys.accepted, false);
                    norm_sq += solves[k].theta * solves[k].theta;
                    if (commit) ngs::commit_rotation(scene.kernels[k], solves[k]);
                }
                break;
            }
            case NGS_SCALING: {
                std::vector<ngs::ScalingSolve> solves(n);
                ngs::parallel_for(n, threads, [&](std::size_t lo, std::size_t hi) {
                    for (std::size_t k = lo; k < hi; ++k)
                        solves[k] = ngs::solve_scaling(scene, static_cast<int>(k), primary, span, opts);
                });
                for (int k = 0; k < n; ++k) {
                    if (out && out->delta)
                        for (int i = 0; i < 3; ++i) out->delta[3 * k + i] = solves[k].delta_scale[i];
                    write_flags(k, solves[k].sys.accepted, solves[k].subspace.degenerate);
                    norm_sq += solves[k].delta_scale.squaredNorm();
                    if (commit) ngs::commit_scaling(scene.kernels[k], solves[k]);
                }
                break;
            }
            case NGS_OPACITY: {
                std::vector<ngs::OpacitySolve> solves(n);
                ngs::parallel_for(n, threads, [&](std::size_t lo, std::size_t hi) {
                    for (std::size_t k = lo; k < hi; ++k)
                        solves[k] = ngs::solve_opacity(scene, static_cast<int>(k), primary, span, opts);
                });
                for (int k = 0; k < n; ++k) {
                    if (out && out->delta) out->delta[k] = solves[k].new_sigma;
                    write_flags(k, solves[k].sys.accepted, false);
                    const double d = solves[k].new_sigma - scene.kernels[k].sigma;
                    norm_sq += d * d;
                    if (commit) ngs::commit_opacity(scene.kernels[k], solves[k]);
                }
                break;
            }
            case NGS_COLOR: {
                std::vector<ngs::ColorSolve> solves(n);
                ngs::parallel_for(n, threads, [&](std::size_t lo, std::size_t hi) {
                    for (std::size_t k = lo; k < hi; ++k)
                        solves[k] = ngs::solve_color(scene, static_cast<int>(k), primary, span, opts);
                });
                for (int k = 0; k < n; ++k) {
                    for (int ch = 0; ch < 3; ++ch) {
                        if (out && out->delta)
                            for (int i = 0; i < 16; ++i)
                                out->delta[48 * k + 16 * ch + i] = i < nsh ? solves[k].delta[ch][i] : 0.0;
                        norm_sq += solves[k].delta[ch].squaredNorm();
                    }
                    write_flags(k, true, false);
                    if (commit) ngs::commit_color(scene.kernels[k], solves[k], scene.sh_degree);
                }
                break;
            }
        }
        if (out) out->delta_norm_sq = norm_sq;
    });
}

int32_t ngs_trainer_configure(ngs_context* ctx, const ngs_train_config* c, int32_t n_cameras,
                              const ngs_camera* cameras, const double* const* targets, int32_t n_train,
                              const int32_t* train_ids, int32_t n_probe, const int32_t* probe_ids,
                              const double* const* secondary_targets,
                              int32_t secondary_targets_downsample) {
    return guarded([&] {
        ngs::Dataset ds;
        for (int i = 0; i < n_cameras; ++i) {
            ds.cameras.push_back(to_camera(cameras[i]));
            ds.targets.push_back(to_image(targets[i], cameras[i].width, cameras[i].height));
        }
        ds.train_ids.assign(train_ids, train_ids + n_train);
        if (n_probe > 0) ds.probe_ids.assign(probe_ids, probe_ids + n_probe);
        if (secondary_targets) {
            ds.secondary_downsample = secondary_targets_downsample;
            for (int i = 0; i < n_cameras; ++i) {
                const ngs::Camera down =
                    ngs::make_downsampled_camera(ds.cameras[i], secondary_targets_downsample);
                ds.secondary_targets.push_back(to_image(secondary_targets[i], down.width, down.height));
            }
        }
        ngs::TrainConfig cfg;
        for (int i = 0; i < 5; ++i) cfg.order[i] = static_cast<ngs::Attribute>(c->order[i]);
        cfg.epochs = c->epochs;
        cfg.seed = c->seed;
        cfg.knn = c->knn;
        cfg.secondary_downsample = c->secondary_downsample;
        cfg.threads = c->threads > 0 ? c->threads : env_threads();
        cfg.barrier_decay = c->barrier_decay;
        cfg.barrier_floor = c->barrier_floor;
        cfg.newton = to_newton(&c->newton);
        cfg.raster = to_raster(&c->raster);
        cfg.loss = to_loss(&c->loss);
        cfg.probe_cadence = c->probe_cadence;
        cfg.optimizer = static_cast<ngs::OptimizerKind>(c->optimizer);
        auto lr = [](const ngs_learning_rates& l) {
            ngs::LearningRates r;
            r.position = l.position;
            r.rotation = l.rotation;
            r.scaling = l.scaling;
            r.opacity = l.opacity;
            r.color = l.color;
            return r;
        };
        cfg.gd_lr = lr(c->gd_lr);
        cfg.adam_lr = lr(c->adam_lr);
        ctx->trainer.reset();
        ctx->trainer.emplace(ctx->scene, std::move(ds), std::move(cfg));
    });
}

int32_t ngs_trainer_neighbors(ngs_context* ctx, int32_t view_id, int32_t* out, int32_t capacity,
                              int32_t* n_out) {
    return guarded([&] {
        if (!ctx->trainer) throw ngs::InvalidInput("trainer not configured");
        const auto& nb = ctx->trainer->neighbors().at(view_id);
        *n_out = static_cast<int32_t>(nb.size());
        for (int i = 0; i < std::min<int>(capacity, static_cast<int>(nb.size())); ++i) out[i] = nb[i];
    });
}

int32_t ngs_trainer_step(ngs_context* ctx, int32_t view_id, ngs_iteration_report* report) {
    return guarded([&] {
        if (!ctx->trainer) throw ngs::InvalidInput("trainer not configured");
        const ngs::IterationReport r = ctx->trainer->step(view_id);
        if (report) {
            report->step = r.step;
            report->image_id = r.image_id;
            report->probe_loss = r.probe_loss;
            report->probe_psnr = r.probe_psnr;
            report->probe_ssim = r.probe_ssim;
            for (int i = 0; i < 5; ++i) report->delta_norms[i] = r.delta_norms[i];
            report->dt_ms = r.dt_ms;
        }
    });
}

static void to_report(const ngs::IterationReport& r, ngs_iteration_report* report) {
    report->step = r.step;
    report->image_id = r.image_id;
    report->probe_loss = r.probe_loss;
    report->probe_psnr = r.probe_psnr;
    report->probe_ssim = r.probe_ssim;
    for (int i = 0; i < 5; ++i) report->delta_norms[i] = r.delta_norms[i];
    report->dt_ms = r.dt_ms;
}

int32_t ngs_trainer_probe(ngs_context* ctx, ngs_metrics* out) {
    return guarded([&] {
        if (!ctx->trainer) throw ngs::InvalidInput("trainer not configured");
        const auto m = ctx->trainer->probe_metrics();
        *out = {m.loss, m.psnr, m.ssim};
    });
}

int32_t ngs_trainer_run(ngs_context* ctx, ngs_iteration_report* rows, int32_t capacity, int32_t* n_rows) {
    return guarded([&] {
        if (!ctx->trainer) throw ngs::InvalidInput("trainer not configured");
        const std::vector<ngs::IterationReport> r = ctx->trainer->run(nullptr);
        if (static_cast<int32_t>(r.size()) > capacity) throw ngs::InvalidInput("trainer run: rows capacity too small");
        for (size_t i = 0; i < r.size(); ++i) to_report(r[i], rows + i);
        *n_rows = static_cast<int32_t>(r.size());
    });
}

int32_t ngs_view_metrics(ngs_context* ctx, const ngs_camera* camera, const double* target_rgb,
                         const ngs_raster_options* raster, const ngs_loss_config* loss, ngs_metrics* out) {
    return guarded([&] {
        const ngs::Camera cam = to_camera(*camera);
        const ngs::Image img = ngs::render(ctx->current(), cam, to_raster(raster)).image;
        const ngs::Image tgt = to_image(target_rgb, cam.width, cam.height);
        const ngs::LossConfig lc = to_loss(loss);
        *out = {ngs::total_loss_value(img, tgt, lc), ngs::psnr(img, tgt), ngs::ssim_metric(img, tgt, lc)};
    });
}

int32_t ngs_trainer_barrier_weight(ngs_context* ctx, double* out) {
    return guarded([&] {
        if (!ctx->trainer) throw ngs::InvalidInput("trainer not configured");
        *out = ctx->trainer->barrier_weight();
    });
}

}  // extern "C"
#include "ref_fixtures.inc"
