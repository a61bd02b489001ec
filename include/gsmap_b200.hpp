// C++ shim over the C-ABI (gsmap_b200.h) that re-exports the reference's hot-path interface
// (proj/include/gsmap/{core/types.hpp, core/gaussian.hpp, render/rasterizer.hpp,
// map/gaussian_map.hpp, map/mapper.hpp}) with the same names, argument meaning and exception
// types, so the mapping thread (proj/src/pipeline/pipeline.cpp:149-175) can call it in place of
// the CPU rasterizer. Eigen is not required: fixed-size vectors are std::array with the
// reference's component order. Header-only; link with libgsmap_b200.so.
#pragma once

#include <array>
#include <cmath>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "gsmap_b200.h"

namespace gsmap_b200 {

inline void check(int st) {
    if (st == GS_OK) return;
    const std::string msg = gs_last_error();
    if (st == GS_EINVAL) throw std::invalid_argument(msg);
    if (st == GS_ELOGIC) throw std::logic_error(msg);
    throw std::runtime_error(msg);
}

using Vec3 = std::array<double, 3>;
using Vec4 = std::array<double, 4>;

// core/types.hpp:15-45
struct CameraModel {
    double fx = 0, fy = 0, cx = 0, cy = 0;
    int width = 0, height = 0;
    gs_camera c() const { return gs_camera{fx, fy, cx, cy, width, height}; }
    void validate() const {
        const gs_camera g = c();
        check(gs_camera_validate(&g));
    }
    CameraModel scaled(int level) const {
        const gs_camera g = c();
        gs_camera o;
        check(gs_camera_scaled(&g, level, &o));
        return CameraModel{o.fx, o.fy, o.cx, o.cy, o.width, o.height};
    }
};

// core/types.hpp:48-64: stores q.normalized() (w, x, y, z) and t
struct Pose {
    Vec4 rotation{1, 0, 0, 0};
    Vec3 translation{0, 0, 0};
    Pose() = default;
    Pose(const Vec4& q, const Vec3& t) : translation(t) {
        const double n2 = ((q[1] * q[1] + q[2] * q[2]) + q[3] * q[3]) + q[0] * q[0];
        const double n = std::sqrt(n2);
        for (int i = 0; i < 4; ++i) rotation[i] = n2 > 0.0 ? q[i] / n : q[i];
    }
    gs_pose p() const {
        return gs_pose{rotation[0], rotation[1], rotation[2], rotation[3], translation[0], translation[1], translation[2]};
    }
};

// core/gaussian.hpp:16-26
struct Gaussian3D {
    Vec3 position{0, 0, 0};
    Vec4 rotation{1, 0, 0, 0};
    Vec3 log_scale{0, 0, 0};
    double opacity_logit = 0.0;
    std::array<Vec3, 16> sh_coeffs{};
    int active_degree = 0;

    gs_gaussian pack() const {
        gs_gaussian g{};
        for (int i = 0; i < 3; ++i) g.p[i] = position[i];
        for (int i = 0; i < 4; ++i) g.p[3 + i] = rotation[i];
        for (int i = 0; i < 3; ++i) g.p[7 + i] = log_scale[i];
        g.p[10] = opacity_logit;
        for (int k = 0; k < 16; ++k)
            for (int c = 0; c < 3; ++c) g.p[11 + 3 * k + c] = sh_coeffs[k][c];
        g.active_degree = active_degree;
        return g;
    }
    static Gaussian3D unpack(const gs_gaussian& g) {
        Gaussian3D o;
        for (int i = 0; i < 3; ++i) o.position[i] = g.p[i];
        for (int i = 0; i < 4; ++i) o.rotation[i] = g.p[3 + i];
        for (int i = 0; i < 3; ++i) o.log_scale[i] = g.p[7 + i];
        o.opacity_logit = g.p[10];
        for (int k = 0; k < 16; ++k)
            for (int c = 0; c < 3; ++c) o.sh_coeffs[k][c] = g.p[11 + 3 * k + c];
        o.active_degree = g.active_degree;
        return o;
    }
};

// core/gaussian.hpp:40-58 (flattened 59 scalars, same order as Gaussian3D)
struct GaussianGrad {
    std::array<double, 59> v{};
    Vec3 position() const { return {v[0], v[1], v[2]}; }
    double opacity_logit() const { return v[10]; }
};

// io/image.hpp: row-major HWC doubles
struct ImageD {
    int h = 0, w = 0, c = 0;
    std::vector<double> data;
    ImageD() = default;
    ImageD(int hh, int ww, int cc, double fill = 0.0) : h(hh), w(ww), c(cc), data(size_t(hh) * ww * cc, fill) {}
    double& at(int y, int x, int ch = 0) { return data[(size_t(y) * w + x) * c + ch]; }
    double at(int y, int x, int ch = 0) const { return data[(size_t(y) * w + x) * c + ch]; }
    int height() const { return h; }
    int width() const { return w; }
    int channels() const { return c; }
};

// map/gaussian_map.hpp:34-40
struct LearningRates {
    double position = 1.6e-4, rotation = 1e-3, log_scale = 5e-3, opacity = 5e-2, sh = 2.5e-3;
    gs_learning_rates l() const { return gs_learning_rates{position, rotation, log_scale, opacity, sh}; }
};

// One device + stream; every object below belongs to one context.
class Context {
public:
    explicit Context(int device = 0, void* stream = nullptr) { check(gs_context_create(device, stream, &h_)); }
    ~Context() { gs_context_destroy(h_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    gs_context* get() const { return h_; }
    static Context& default_context() {
        static Context c(0);
        return c;
    }

private:
    gs_context* h_ = nullptr;
};

struct RenderGradients {  // rasterizer.hpp:62-64, device-resident
    std::shared_ptr<gs_grads> h;
    int64_t n = 0;
    std::vector<GaussianGrad> per_gaussian() const {
        std::vector<double> flat(static_cast<size_t>(n) * 59);
        check(gs_grads_read(h.get(), flat.data(), n));
        std::vector<GaussianGrad> out(n);
        for (int64_t i = 0; i < n; ++i)
            for (int k = 0; k < 59; ++k) out[i].v[k] = flat[i * 59 + k];
        return out;
    }
};

// map/gaussian_map.hpp:44-96 — the map lives on the GPU (fp32 SoA + Adam state)
class GaussianMap {
public:
    explicit GaussianMap(Context& ctx = Context::default_context()) : ctx_(&ctx) { check(gs_map_create(ctx.get(), &h_)); }
    GaussianMap(Context& ctx, gs_map* adopt) : ctx_(&ctx), h_(adopt) {}  // takes ownership of a C-ABI handle
    ~GaussianMap() {
        if (h_) gs_map_destroy(h_);
    }
    GaussianMap(const GaussianMap&) = delete;
    GaussianMap& operator=(const GaussianMap&) = delete;
    GaussianMap(GaussianMap&& o) noexcept : ctx_(o.ctx_), h_(o.h_) { o.h_ = nullptr; }

    size_t size() const {
        int64_t n = 0;
        check(gs_map_size(h_, &n));
        return static_cast<size_t>(n);
    }
    bool empty() const { return size() == 0; }
    void append(const std::vector<Gaussian3D>& gs) {
        std::vector<gs_gaussian> p(gs.size());
        for (size_t i = 0; i < gs.size(); ++i) p[i] = gs[i].pack();
        check(gs_map_append(h_, p.data(), static_cast<int64_t>(p.size())));
    }
    std::vector<Gaussian3D> gaussians() const {  // snapshot (host copy)
        std::vector<gs_gaussian> p(size());
        check(gs_map_get_gaussians(h_, p.data(), static_cast<int64_t>(p.size())));
        std::vector<Gaussian3D> out(p.size());
        for (size_t i = 0; i < p.size(); ++i) out[i] = Gaussian3D::unpack(p[i]);
        return out;
    }
    void set_gaussians(const std::vector<Gaussian3D>& gs) {  // host edit, keeps Adam state
        std::vector<gs_gaussian> p(gs.size());
        for (size_t i = 0; i < gs.size(); ++i) p[i] = gs[i].pack();
        check(gs_map_set_gaussians(h_, p.data(), static_cast<int64_t>(p.size())));
    }
    void apply_gradients(const RenderGradients& g, const LearningRates& lr) {  // gaussian_map.cpp:37-54
        const gs_learning_rates l = lr.l();
        check(gs_apply_gradients(h_, g.h.get(), &l));
    }
    int64_t global_step() const {
        int64_t s = 0;
        check(gs_map_global_step(h_, &s));
        return s;
    }
    void set_global_step(int64_t s) { check(gs_map_set_global_step(h_, s)); }
    double scene_extent() const {
        double e = 0;
        check(gs_map_scene_extent(h_, &e));
        return e;
    }
    void raise_sh_degree(int d) { check(gs_map_raise_sh_degree(h_, d)); }
    int max_active_degree() const {  // gaussian_map.hpp:84
        int d = 0;
        check(gs_map_max_active_degree(h_, &d));
        return d;
    }
    std::size_t prune(double opacity_threshold) {  // gaussian_map.hpp:79
        int64_t removed = 0;
        check(gs_map_prune(h_, opacity_threshold, &removed));
        return static_cast<std::size_t>(removed);
    }
    gs_map* get() const { return h_; }
    Context& context() const { return *ctx_; }

private:
    Context* ctx_;
    gs_map* h_ = nullptr;
};

// rasterizer.hpp:43-59: images download lazily; the contributor table only on request
struct RenderOutput {
    std::shared_ptr<gs_frame> h;
    CameraModel cam;
    ImageD color() const {
        ImageD c(cam.height, cam.width, 3);
        check(gs_frame_read(h.get(), c.data.data(), nullptr, nullptr));
        return c;
    }
    ImageD depth() const {
        ImageD d(cam.height, cam.width, 1);
        check(gs_frame_read(h.get(), nullptr, d.data.data(), nullptr));
        return d;
    }
    ImageD visibility() const {
        ImageD v(cam.height, cam.width, 1);
        check(gs_frame_read(h.get(), nullptr, nullptr, v.data.data()));
        return v;
    }
    // contributors(y, x) as (map index, alpha), rasterizer.hpp:55-58
    std::vector<std::pair<int32_t, double>> contributors(int y, int x) const {
        gs_frame_stats s;
        check(gs_frame_stats_get(h.get(), &s));
        std::vector<uint32_t> off(static_cast<size_t>(s.width) * s.height + 1);
        std::vector<int32_t> g(s.n_contrib);
        std::vector<double> a(s.n_contrib);
        check(gs_frame_materialize(h.get(), off.data(), g.data(), a.data()));
        const size_t p = static_cast<size_t>(y) * s.width + x;
        std::vector<std::pair<int32_t, double>> out;
        for (uint32_t i = off[p]; i < off[p + 1]; ++i) out.emplace_back(g[i], a[i]);
        return out;
    }
};

struct ThreadPool;  // accepted for signature compatibility; the GPU path ignores it

inline std::shared_ptr<gs_frame> make_frame(Context& ctx) {
    gs_frame* f = nullptr;
    check(gs_frame_create(ctx.get(), &f));
    return std::shared_ptr<gs_frame>(f, [](gs_frame* p) { gs_frame_destroy(p); });
}

inline std::shared_ptr<gs_grads> make_grads(Context& ctx) {
    gs_grads* g = nullptr;
    check(gs_grads_create(ctx.get(), &g));
    return std::shared_ptr<gs_grads>(g, [](gs_grads* p) { gs_grads_destroy(p); });
}

// io/sequence.hpp:70 (sequence.cpp:246-259): ColoredPoint = position xyz + colour rgb (6 doubles)
struct ColoredPoint {
    Vec3 position{0, 0, 0};
    Vec3 color{0, 0, 0};
};

inline ImageD project_sparse_depth(Context& ctx, const std::vector<ColoredPoint>& points, const Pose& pose,
                                   const CameraModel& cam) {
    std::vector<double> flat(points.size() * 6);
    for (size_t i = 0; i < points.size(); ++i) {
        for (int k = 0; k < 3; ++k) flat[6 * i + k] = points[i].position[k];
        for (int k = 0; k < 3; ++k) flat[6 * i + 3 + k] = points[i].color[k];
    }
    ImageD depth(cam.height, cam.width, 1, 0.0);
    const gs_pose p = pose.p();
    const gs_camera c = cam.c();
    check(gs_project_sparse_depth(ctx.get(), flat.data(), static_cast<int64_t>(points.size()), 6, &p, &c,
                                  depth.data.data()));
    return depth;
}

// mapper.cpp:43-61 (device grid 3-NN); returns the number of Gaussians appended
inline std::size_t init_gaussians_from_points(GaussianMap& map, const std::vector<ColoredPoint>& points) {
    std::vector<double> flat(points.size() * 6);
    for (size_t i = 0; i < points.size(); ++i) {
        for (int k = 0; k < 3; ++k) flat[6 * i + k] = points[i].position[k];
        for (int k = 0; k < 3; ++k) flat[6 * i + 3 + k] = points[i].color[k];
    }
    int64_t added = 0;
    check(gs_map_init_from_points(map.get(), flat.data(), static_cast<int64_t>(points.size()), &added));
    return static_cast<std::size_t>(added);
}

class Keyframe;
// keyframe.cpp:49-74: the points (in order) behind the near plane, outside the image, or on a
// pixel whose rendered visibility is <= tau_alpha
inline std::vector<ColoredPoint> filter_points_by_visibility(const std::vector<ColoredPoint>& points,
                                                             const Keyframe& kf, const GaussianMap& map,
                                                             const CameraModel& cam, double tau_alpha,
                                                             ThreadPool* = nullptr);

// mapper.cpp:240-246 (sh_interval = TrainConfig::sh_interval in the reference); returns the degree
inline int maybe_upgrade_sh(GaussianMap& map, int sh_interval) {
    int d = 0;
    check(gs_maybe_upgrade_sh(map.get(), sh_interval, &d));
    return d;
}

// io/checkpoint.hpp (checkpoint.cpp:17-73), format v1
inline void save_checkpoint(const std::string& path, const GaussianMap& map) {
    check(gs_save_checkpoint(map.get(), path.c_str()));
}
inline GaussianMap load_checkpoint(const std::string& path, Context& ctx = Context::default_context()) {
    gs_map* h = nullptr;
    check(gs_load_checkpoint(ctx.get(), path.c_str(), &h));
    return GaussianMap(ctx, h);
}

// rasterizer.hpp:69-70
inline RenderOutput render(const GaussianMap& map, const Pose& pose, const CameraModel& cam, ThreadPool* = nullptr) {
    RenderOutput out{make_frame(map.context()), cam};
    const gs_pose p = pose.p();
    const gs_camera c = cam.c();
    check(gs_render(map.get(), &p, &c, out.h.get()));
    return out;
}

// rasterizer.hpp:74-77
inline RenderGradients render_backward(const GaussianMap& map, const Pose& pose, const CameraModel& cam,
                                       const RenderOutput& out, const ImageD& dl_dcolor, const ImageD& dl_ddepth,
                                       ThreadPool* = nullptr) {
    if (dl_dcolor.h != cam.height || dl_dcolor.w != cam.width || dl_dcolor.c != 3)
        throw std::invalid_argument("render_backward: dl_dcolor dimensions mismatch");
    if (dl_ddepth.h != cam.height || dl_ddepth.w != cam.width || dl_ddepth.c != 1)
        throw std::invalid_argument("render_backward: dl_ddepth dimensions mismatch");
    RenderGradients g{make_grads(map.context()), static_cast<int64_t>(map.size())};
    const gs_pose p = pose.p();
    const gs_camera c = cam.c();
    check(gs_render_backward(map.get(), &p, &c, out.h.get(), dl_dcolor.data.data(), dl_ddepth.data.data(),
                             cam.height, cam.width, g.h.get()));
    return g;
}

// map/mapper.hpp:17-30 (hot-path fields)
struct TrainConfig {
    double lambda = 0.2, lambda_d = 0.5;
    int pyramid_levels = 2, iters_per_level = 0;
    LearningRates lr;
    gs_train_config c() const { return gs_train_config{lambda, lambda_d, pyramid_levels, iters_per_level, lr.l()}; }
};

// map/keyframe.hpp:23-34 (hot-path fields); the pyramid is built on the device
class Keyframe {
public:
    Keyframe(Context& ctx, const Pose& pose, const ImageD& color, const ImageD& sparse_depth, int initial_iters,
             int levels)
        : pose_(pose) {
        const gs_pose p = pose.p();
        check(gs_keyframe_create(ctx.get(), &p, color.data.data(), sparse_depth.data.data(), color.h, color.w,
                                 initial_iters, levels, &h_));
    }
    Keyframe(const Pose& pose, gs_keyframe* adopt) : pose_(pose), h_(adopt) {}  // owns a C-ABI handle
    ~Keyframe() {
        if (h_) gs_keyframe_destroy(h_);
    }
    Keyframe(const Keyframe&) = delete;
    Keyframe& operator=(const Keyframe&) = delete;
    Keyframe(Keyframe&& o) noexcept : pose_(o.pose_), h_(o.h_) { o.h_ = nullptr; }
    int consumed_iters() const {
        int32_t c = 0;
        check(gs_keyframe_consumed(h_, &c));
        return c;
    }
    const Pose& pose() const { return pose_; }
    gs_keyframe* get() const { return h_; }

private:
    Pose pose_;
    gs_keyframe* h_ = nullptr;
};

inline std::vector<ColoredPoint> filter_points_by_visibility(const std::vector<ColoredPoint>& points,
                                                             const Keyframe& kf, const GaussianMap& map,
                                                             const CameraModel& cam, double tau_alpha, ThreadPool*) {
    std::vector<double> flat(points.size() * 6), kept(points.size() * 6);
    for (size_t i = 0; i < points.size(); ++i) {
        for (int k = 0; k < 3; ++k) flat[6 * i + k] = points[i].position[k];
        for (int k = 0; k < 3; ++k) flat[6 * i + 3 + k] = points[i].color[k];
    }
    const gs_pose p = kf.pose().p();
    const gs_camera c = cam.c();
    int64_t n = 0;
    check(gs_filter_points_by_visibility(map.get(), flat.data(), static_cast<int64_t>(points.size()), &p, &c,
                                         tau_alpha, kept.data(), &n));
    std::vector<ColoredPoint> out(static_cast<size_t>(n));
    for (size_t i = 0; i < out.size(); ++i) {
        for (int k = 0; k < 3; ++k) out[i].position[k] = kept[6 * i + k];
        for (int k = 0; k < 3; ++k) out[i].color[k] = kept[6 * i + 3 + k];
    }
    return out;
}

// integrate_keyframe (pipeline.cpp:148-155) in one device call: filter the frame's cloud by the
// map's visibility, initialise Gaussians from the kept points, and build the keyframe (pyramid of
// `color` and of the cloud's project_sparse_depth). Returns the keyframe; *added = Gaussians added.
inline Keyframe integrate_keyframe(GaussianMap& map, const Pose& pose, const CameraModel& cam, const ImageD& color,
                                   const std::vector<ColoredPoint>& points, double tau_alpha, int initial_iters,
                                   int levels, std::size_t* added = nullptr) {
    std::vector<double> flat(points.size() * 6);
    for (size_t i = 0; i < points.size(); ++i) {
        for (int k = 0; k < 3; ++k) flat[6 * i + k] = points[i].position[k];
        for (int k = 0; k < 3; ++k) flat[6 * i + 3 + k] = points[i].color[k];
    }
    const gs_pose p = pose.p();
    const gs_camera c = cam.c();
    gs_keyframe* h = nullptr;
    int64_t n = 0;
    check(gs_integrate_keyframe(map.get(), &p, &c, color.data.data(), flat.data(), static_cast<int64_t>(points.size()),
                                tau_alpha, initial_iters, levels, &h, &n));
    if (added) *added = static_cast<std::size_t>(n);
    return Keyframe(pose, h);
}

// optimizer state beside a checkpoint (true resume; the v1 format has none)
inline void save_training_state(const std::string& path, const GaussianMap& map) {
    check(gs_save_training_state(map.get(), path.c_str()));
}
inline void load_training_state(const std::string& path, GaussianMap& map) {
    check(gs_load_training_state(map.get(), path.c_str()));
}

// evaluate_sequence (pipeline.cpp:41-64), one frame: EvalRecord's metric fields
struct EvalMetrics {
    double psnr = 0, ssim = 0, depth_rmse = 0;
};
inline EvalMetrics evaluate_view(const GaussianMap& map, const Pose& pose, const CameraModel& cam,
                                 const ImageD& gt_color, const ImageD* gt_depth) {
    const gs_pose p = pose.p();
    const gs_camera c = cam.c();
    gs_eval_metrics m{};
    check(gs_evaluate_view(map.get(), &p, &c, gt_color.data.data(), gt_depth ? gt_depth->data.data() : nullptr, &m));
    return EvalMetrics{m.psnr, m.ssim, m.depth_rmse};
}

struct LossResult {  // mapper.hpp:52-60
    double total = 0, color_loss = 0, depth_loss = 0, l1 = 0, ssim = 0;
    ImageD dl_dcolor, dl_ddepth;
};

// mapper.hpp:61-62
inline LossResult compute_loss(const RenderOutput& rendered, const Keyframe& kf, int level, const TrainConfig& cfg) {
    LossResult r;
    r.dl_dcolor = ImageD(rendered.cam.height, rendered.cam.width, 3);
    r.dl_ddepth = ImageD(rendered.cam.height, rendered.cam.width, 1);
    gs_loss_result s;
    const gs_train_config c = cfg.c();
    check(gs_compute_loss(rendered.h.get(), kf.get(), level, &c, &s, r.dl_dcolor.data.data(), r.dl_ddepth.data.data()));
    r.total = s.total;
    r.color_loss = s.color_loss;
    r.depth_loss = s.depth_loss;
    r.l1 = s.l1;
    r.ssim = s.ssim;
    return r;
}

struct StepReport {  // mapper.hpp:64-68
    int level = 0;
    double loss = 0, psnr = 0;
};

// mapper.hpp:74-76 — the fused hot step
inline std::optional<StepReport> train_keyframe_step(GaussianMap& map, Keyframe& kf, const TrainConfig& cfg,
                                                     const CameraModel& cam, ThreadPool* = nullptr) {
    gs_step_report r;
    const gs_train_config c = cfg.c();
    const gs_camera cm = cam.c();
    check(gs_train_step(map.get(), kf.get(), &c, &cm, &r));
    if (!r.ran) return std::nullopt;
    return StepReport{r.level, r.loss, r.psnr};
}

}  // namespace gsmap_b200
