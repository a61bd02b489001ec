// The reference-side binding a maintainer adds to run the reference's mapping back end on the
// B200 path: this translation unit DEFINES the reference's five hot-path entry points over the
// gsmap_b200 C-ABI, against the reference's own headers and types (Eigen, ImageD,
// GaussianMap, Keyframe, ...). integration/Makefile compiles the reference's sources unchanged
// and weakens exactly these five definitions in their objects (objcopy --weaken-symbol), so the
// strong definitions here win at link time and every unchanged caller — pipeline.cpp's mapping
// thread, keyframe.cpp, gradcheck.cpp and the reference's unit tests — runs on the GPU:
//
//   render                         proj/include/gsmap/render/rasterizer.hpp:69-70
//   render_backward                proj/include/gsmap/render/rasterizer.hpp:74-77
//   GaussianMap::apply_gradients   proj/include/gsmap/map/gaussian_map.hpp:75
//   compute_loss                   proj/include/gsmap/map/mapper.hpp:61-62
//   train_keyframe_step            proj/include/gsmap/map/mapper.hpp:74-76
//
// Residency: the reference's GaussianMap owns fp64 AoS parameters and Adam state on the host, so
// this binding mirrors them into one device map per call (upload, run, write back). That keeps
// the reference's semantics (callers may edit map.gaussians() between calls) at the cost of the
// host<->device copies; a caller that keeps the map resident uses the C-ABI directly.
// The device holds fp32 parameters: after an Adam step the host map holds the fp32-representable
// values the device computed. Errors come back as the reference's exception types.
#include <cstdlib>
#include <memory>
#include <mutex>  // (recursive: train_keyframe_step writes back through apply_gradients)
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "gsmap/core/projection.hpp"
#include "gsmap/core/sh.hpp"
#include "gsmap/map/gaussian_map.hpp"
#include "gsmap/map/mapper.hpp"
#include "gsmap/metrics/metrics.hpp"
#include "gsmap/render/rasterizer.hpp"
#include "gsmap_b200.h"

namespace {

void check(int st) {
    if (st == GS_OK) return;
    const std::string msg = gs_last_error();
    if (st == GS_EINVAL) throw std::invalid_argument(msg);
    if (st == GS_ELOGIC) throw std::logic_error(msg);
    throw std::runtime_error("gsmap_b200: " + msg);
}

// One context / map / frame / gradient set on device GSMAP_B200_DEVICE (default 0). The
// reference's API is synchronous; calls are serialised here.
struct Backend {
    gs_context* ctx = nullptr;
    gs_map* map = nullptr;
    gs_frame* frame = nullptr;
    gs_grads* grads = nullptr;
    std::recursive_mutex mu;
    Backend() {
        const char* d = std::getenv("GSMAP_B200_DEVICE");
        check(gs_context_create(d ? std::atoi(d) : 0, nullptr, &ctx));
        check(gs_map_create(ctx, &map));
        check(gs_frame_create(ctx, &frame));
        check(gs_grads_create(ctx, &grads));
    }
    static Backend& get() {
        static Backend b;
        return b;
    }
};

gs_pose to_pose(const gsmap::Pose& p) {
    const Eigen::Quaterniond& q = p.rotation;  // already normalised (types.hpp:53-54)
    return gs_pose{q.w(), q.x(), q.y(), q.z(), p.translation.x(), p.translation.y(), p.translation.z()};
}

gs_camera to_cam(const gsmap::CameraModel& c) { return gs_camera{c.fx, c.fy, c.cx, c.cy, c.width, c.height}; }

gs_gaussian pack(const gsmap::Gaussian3D& g) {
    gs_gaussian o{};
    for (int i = 0; i < 3; ++i) o.p[i] = g.position[i];
    for (int i = 0; i < 4; ++i) o.p[3 + i] = g.rotation[i];
    for (int i = 0; i < 3; ++i) o.p[7 + i] = g.log_scale[i];
    o.p[10] = g.opacity_logit;
    for (int k = 0; k < gsmap::kShCoeffCount; ++k)
        for (int c = 0; c < 3; ++c) o.p[11 + 3 * k + c] = g.sh_coeffs[k][c];
    o.active_degree = g.active_degree;
    return o;
}

void unpack(const gs_gaussian& o, gsmap::Gaussian3D& g) {
    for (int i = 0; i < 3; ++i) g.position[i] = o.p[i];
    for (int i = 0; i < 4; ++i) g.rotation[i] = o.p[3 + i];
    for (int i = 0; i < 3; ++i) g.log_scale[i] = o.p[7 + i];
    g.opacity_logit = o.p[10];
    for (int k = 0; k < gsmap::kShCoeffCount; ++k)
        for (int c = 0; c < 3; ++c) g.sh_coeffs[k][c] = o.p[11 + 3 * k + c];
    g.active_degree = o.active_degree;
}

// the device map := the host map's parameters (+ extent and step; Adam state on request)
void upload(Backend& b, const gsmap::GaussianMap& m) {
    std::vector<gs_gaussian> gs(m.size());
    for (size_t i = 0; i < m.size(); ++i) gs[i] = pack(m.gaussians()[i]);
    int64_t n = 0;
    check(gs_map_size(b.map, &n));
    if (n == static_cast<int64_t>(gs.size())) {
        check(gs_map_set_gaussians(b.map, gs.data(), n));
    } else {  // a map of another size: a fresh device map of this one
        check(gs_map_destroy(b.map));
        b.map = nullptr;
        check(gs_map_create(b.ctx, &b.map));
        if (!gs.empty()) check(gs_map_append(b.map, gs.data(), static_cast<int64_t>(gs.size())));
    }
    check(gs_map_set_scene_extent(b.map, m.scene_extent()));
    check(gs_map_set_global_step(b.map, m.global_step()));
}

void upload_adam(Backend& b, const gsmap::GaussianMap& m) {
    const size_t n = m.size();
    std::vector<double> mm(59 * n), vv(59 * n);
    std::vector<int64_t> step(n);
    for (size_t i = 0; i < n; ++i) {
        const gsmap::AdamState& s = m.optimizer_state()[i];
        double* a = &mm[59 * i];
        double* c = &vv[59 * i];
        for (int k = 0; k < 3; ++k) a[k] = s.m_position[k], c[k] = s.v_position[k];
        for (int k = 0; k < 4; ++k) a[3 + k] = s.m_rotation[k], c[3 + k] = s.v_rotation[k];
        for (int k = 0; k < 3; ++k) a[7 + k] = s.m_log_scale[k], c[7 + k] = s.v_log_scale[k];
        a[10] = s.m_opacity, c[10] = s.v_opacity;
        for (int j = 0; j < gsmap::kShCoeffCount; ++j)
            for (int k = 0; k < 3; ++k) a[11 + 3 * j + k] = s.m_sh[j][k], c[11 + 3 * j + k] = s.v_sh[j][k];
        step[i] = s.step;
    }
    check(gs_map_set_adam(b.map, mm.data(), vv.data(), step.data(), static_cast<int64_t>(n)));
}

// device -> host gaussians and Adam state (the reference's AdamState layout)
void download(Backend& b, std::vector<gsmap::Gaussian3D>& gs, std::vector<gsmap::AdamState>& opt) {
    const size_t n = gs.size();
    std::vector<gs_gaussian> raw(n);
    check(gs_map_get_gaussians(b.map, raw.data(), static_cast<int64_t>(n)));
    for (size_t i = 0; i < n; ++i) unpack(raw[i], gs[i]);
    std::vector<double> mm(59 * n), vv(59 * n);
    std::vector<int64_t> step(n);
    check(gs_map_get_adam(b.map, mm.data(), vv.data(), step.data(), static_cast<int64_t>(n)));
    opt.resize(n);
    for (size_t i = 0; i < n; ++i) {
        gsmap::AdamState& s = opt[i];
        const double* a = &mm[59 * i];
        const double* c = &vv[59 * i];
        for (int k = 0; k < 3; ++k) s.m_position[k] = a[k], s.v_position[k] = c[k];
        for (int k = 0; k < 4; ++k) s.m_rotation[k] = a[3 + k], s.v_rotation[k] = c[3 + k];
        for (int k = 0; k < 3; ++k) s.m_log_scale[k] = a[7 + k], s.v_log_scale[k] = c[7 + k];
        s.m_opacity = a[10], s.v_opacity = c[10];
        for (int j = 0; j < gsmap::kShCoeffCount; ++j)
            for (int k = 0; k < 3; ++k) s.m_sh[j][k] = a[11 + 3 * j + k], s.v_sh[j][k] = c[11 + 3 * j + k];
        s.step = step[i];
    }
}

// The Gaussian the device holds (fp32 storage of each parameter)
gsmap::Gaussian3D as_stored(const gsmap::Gaussian3D& g) {
    gs_gaussian p = pack(g);
    for (double& x : p.p) x = static_cast<double>(static_cast<float>(x));
    gsmap::Gaussian3D o;
    unpack(p, o);
    return o;
}

// RenderOutput of the frame: images, CSR contributor table and the projected set (the device's
// bit-exact (depth, index) order; each record's fields from the reference's own core functions
// on the stored parameters, as rasterizer.cpp:37-68 fills them)
gsmap::RenderOutput read_output(Backend& b, const gsmap::GaussianMap& m, const gsmap::Pose& pose,
                                const gsmap::CameraModel& cam) {
    gsmap::RenderOutput out;
    const int h = cam.height, w = cam.width;
    out.color = gsmap::ImageD(h, w, 3, 0.0);
    out.depth = gsmap::ImageD(h, w, 1, 0.0);
    out.visibility = gsmap::ImageD(h, w, 1, 0.0);
    check(gs_frame_read(b.frame, out.color.data(), out.depth.data(), out.visibility.data()));
    gs_frame_stats st{};
    check(gs_frame_stats_get(b.frame, &st));
    out.contrib_offsets.resize(static_cast<size_t>(h) * w + 1);
    std::vector<int32_t> gid(static_cast<size_t>(st.n_contrib));
    std::vector<double> alpha(static_cast<size_t>(st.n_contrib));
    check(gs_frame_materialize(b.frame, out.contrib_offsets.data(), gid.data(), alpha.data()));
    out.contribs.resize(gid.size());
    for (size_t i = 0; i < gid.size(); ++i) out.contribs[i] = gsmap::Contribution{gid[i], alpha[i]};
    std::vector<int32_t> index(static_cast<size_t>(st.n_visible));
    check(gs_frame_read_projected(b.frame, index.data(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr));
    const Eigen::Vector3d center = pose.camera_center();
    out.projected.reserve(index.size());
    for (const int32_t i : index) {
        const gsmap::Gaussian3D g = as_stored(m.gaussians()[static_cast<size_t>(i)]);
        const auto p2 = gsmap::project_gaussian(g, pose, cam);
        if (!p2) throw std::logic_error("gsmap_b200: projected set disagrees with the host projection");
        gsmap::ProjectedGaussian pg;
        pg.index = i;
        pg.mean = p2->mean;
        pg.cov2d = p2->cov2d;
        pg.cov_inv = p2->cov2d.inverse();
        pg.depth = p2->depth;
        pg.radius = p2->radius;
        pg.opacity = g.opacity();
        const Eigen::Vector3d v = g.position - center;
        pg.view_dist = v.norm();
        pg.view_dir = pg.view_dist > 0.0 ? Eigen::Vector3d(v / pg.view_dist) : Eigen::Vector3d(0, 0, 1);
        pg.color_raw = gsmap::eval_sh(g.sh_coeffs, g.active_degree, pg.view_dir);
        pg.color = pg.color_raw.cwiseMax(0.0).cwiseMin(1.0);
        out.projected.push_back(pg);
    }
    return out;
}

// the device keyframe of a host Keyframe: its pyramid (already built by the reference's
// build_keyframe_pyramid) uploaded level by level, and its consumed-iteration count
struct DeviceKeyframe {
    gs_keyframe* kf = nullptr;
    DeviceKeyframe(Backend& b, const gsmap::Keyframe& k) {
        const gsmap::PyramidLevel& l0 = k.pyramid.front();
        const gs_pose pose = to_pose(k.pose);
        const int levels = static_cast<int>(k.pyramid.size()) - 1;
        check(gs_keyframe_create(b.ctx, &pose, l0.color.data(), l0.depth.data(), l0.color.height(),
                                 l0.color.width(), k.initial_iters, levels, &kf));
        for (int l = 1; l <= levels; ++l)
            check(gs_keyframe_upload_level(kf, l, k.pyramid[l].color.data(), k.pyramid[l].depth.data()));
        check(gs_keyframe_set_consumed(kf, k.consumed_iters));
    }
    ~DeviceKeyframe() {
        if (kf) gs_keyframe_destroy(kf);
    }
};

// Internal marker passed to GaussianMap::apply_gradients by train_keyframe_step: "the device has
// already run this step's Adam update; write the device state back into this map". Its address
// is private to this file, so no caller can pass it.
const gsmap::RenderGradients kDeviceStepDone{};

gs_train_config to_cfg(const gsmap::TrainConfig& c) {
    gs_train_config o{};
    o.lambda = c.lambda;
    o.lambda_d = c.lambda_d;
    o.pyramid_levels = c.pyramid_levels;
    o.iters_per_level = c.iters_per_level;
    o.lr = gs_learning_rates{c.lr.position, c.lr.rotation, c.lr.log_scale, c.lr.opacity, c.lr.sh};
    return o;
}

}  // namespace

namespace gsmap {

RenderOutput render(const GaussianMap& map, const Pose& pose, const CameraModel& cam, ThreadPool*) {
    cam.validate();
    Backend& b = Backend::get();
    std::lock_guard<std::recursive_mutex> lk(b.mu);
    upload(b, map);
    const gs_pose p = to_pose(pose);
    const gs_camera c = to_cam(cam);
    check(gs_render(b.map, &p, &c, b.frame));
    return read_output(b, map, pose, cam);
}

RenderGradients render_backward(const GaussianMap& map, const Pose& pose, const CameraModel& cam,
                                const RenderOutput& out, const ImageD& dl_dcolor, const ImageD& dl_ddepth,
                                ThreadPool*) {
    // the reference's argument checks (rasterizer.cpp:229-237)
    if (dl_dcolor.height() != out.color.height() || dl_dcolor.width() != out.color.width() ||
        dl_dcolor.channels() != 3 || dl_ddepth.height() != out.color.height() ||
        dl_ddepth.width() != out.color.width() || dl_ddepth.channels() != 1)
        throw std::invalid_argument("render_backward: cotangent buffers do not match the render");
    if (out.contrib_offsets.size() != static_cast<size_t>(out.color.height()) * out.color.width() + 1)
        throw std::logic_error("render_backward: contributor lists missing or inconsistent");
    Backend& b = Backend::get();
    std::lock_guard<std::recursive_mutex> lk(b.mu);
    // the device replays the render it produced `out` with (deterministic: same map, pose and
    // camera give the same lists) and differentiates it
    upload(b, map);
    const gs_pose p = to_pose(pose);
    const gs_camera c = to_cam(cam);
    check(gs_render(b.map, &p, &c, b.frame));
    check(gs_render_backward(b.map, &p, &c, b.frame, dl_dcolor.data(), dl_ddepth.data(), cam.height, cam.width,
                             b.grads));
    const size_t n = map.size();
    std::vector<double> g59(59 * n);
    check(gs_grads_read(b.grads, g59.data(), static_cast<int64_t>(n)));
    RenderGradients rg;
    rg.per_gaussian.resize(n);
    for (size_t i = 0; i < n; ++i) {
        grad::GaussianGrad& d = rg.per_gaussian[i];
        const double* s = &g59[59 * i];
        for (int k = 0; k < 3; ++k) d.position[k] = s[k];
        for (int k = 0; k < 4; ++k) d.rotation[k] = s[3 + k];
        for (int k = 0; k < 3; ++k) d.log_scale[k] = s[7 + k];
        d.opacity_logit = s[10];
        for (int j = 0; j < kShCoeffCount; ++j)
            for (int k = 0; k < 3; ++k) d.sh_coeffs[j][k] = s[11 + 3 * j + k];
    }
    return rg;
}

void GaussianMap::apply_gradients(const RenderGradients& grads, const LearningRates& lr) {
    Backend& b = Backend::get();
    std::lock_guard<std::recursive_mutex> lk(b.mu);
    if (&grads == &kDeviceStepDone) {  // train_keyframe_step: the device map is this map, stepped
        download(b, gaussians_, opt_);
        check(gs_map_global_step(b.map, &global_step_));
        return;
    }
    if (grads.per_gaussian.size() != gaussians_.size())
        throw std::invalid_argument("apply_gradients: gradient count does not match map size");
    upload(b, *this);
    upload_adam(b, *this);
    const size_t n = gaussians_.size();
    std::vector<double> g59(59 * n);
    for (size_t i = 0; i < n; ++i) {
        const grad::GaussianGrad& d = grads.per_gaussian[i];
        double* s = &g59[59 * i];
        for (int k = 0; k < 3; ++k) s[k] = d.position[k];
        for (int k = 0; k < 4; ++k) s[3 + k] = d.rotation[k];
        for (int k = 0; k < 3; ++k) s[7 + k] = d.log_scale[k];
        s[10] = d.opacity_logit;
        for (int j = 0; j < kShCoeffCount; ++j)
            for (int k = 0; k < 3; ++k) s[11 + 3 * j + k] = d.sh_coeffs[j][k];
    }
    check(gs_grads_zero(b.grads, b.map));
    check(gs_grads_write(b.grads, g59.data(), static_cast<int64_t>(n)));
    const gs_learning_rates l{lr.position, lr.rotation, lr.log_scale, lr.opacity, lr.sh};
    check(gs_apply_gradients(b.map, b.grads, &l));
    download(b, gaussians_, opt_);
    check(gs_map_global_step(b.map, &global_step_));
}

LossResult compute_loss(const RenderOutput& rendered, const Keyframe& kf, int level, const TrainConfig& cfg) {
    // the reference's argument checks (mapper.cpp:148-153)
    if (level < 0 || level >= static_cast<int>(kf.pyramid.size()))
        throw std::invalid_argument("compute_loss: pyramid level out of range");
    if (!rendered.color.same_shape(kf.pyramid[level].color))
        throw std::invalid_argument("compute_loss: rendered resolution does not match level");
    Backend& b = Backend::get();
    std::lock_guard<std::recursive_mutex> lk(b.mu);
    const int h = rendered.color.height(), w = rendered.color.width();
    check(gs_frame_set_images(b.frame, rendered.color.data(), rendered.depth.data(), rendered.visibility.data(), h,
                              w));
    DeviceKeyframe dk(b, kf);
    const gs_train_config c = to_cfg(cfg);
    gs_loss_result r{};
    LossResult res;
    res.dl_dcolor = ImageD(h, w, 3, 0.0);
    res.dl_ddepth = ImageD(h, w, 1, 0.0);
    check(gs_compute_loss(b.frame, dk.kf, level, &c, &r, res.dl_dcolor.data(), res.dl_ddepth.data()));
    res.total = r.total;
    res.color_loss = r.color_loss;
    res.depth_loss = r.depth_loss;
    res.l1 = r.l1;
    res.ssim = r.ssim;
    return res;
}

std::optional<StepReport> train_keyframe_step(GaussianMap& map, Keyframe& kf, const TrainConfig& cfg,
                                              const CameraModel& cam, ThreadPool*) {
    // the reference's contract (mapper.cpp:217-219)
    if (kf.pyramid.empty()) throw std::invalid_argument("train_keyframe_step: keyframe pyramid not built");
    if (kf.consumed_iters >= kf.initial_iters) return std::nullopt;
    cam.validate();
    Backend& b = Backend::get();
    std::lock_guard<std::recursive_mutex> lk(b.mu);
    upload(b, map);
    upload_adam(b, map);
    DeviceKeyframe dk(b, kf);
    const gs_train_config c = to_cfg(cfg);
    const gs_camera gc = to_cam(cam);
    gs_step_report rep{};
    check(gs_train_step(b.map, dk.kf, &c, &gc, &rep));
    if (!rep.ran) return std::nullopt;
    // the fused device step (render -> loss -> backward -> Adam, gs_train_step) ran on this map:
    // write parameters, Adam state and step back (the optimizer state is private to GaussianMap;
    // apply_gradients is the member this binding defines)
    map.apply_gradients(kDeviceStepDone, cfg.lr);
    ++kf.consumed_iters;
    StepReport report;
    report.level = rep.level;
    report.loss = rep.loss;
    report.psnr = rep.psnr;
    return report;
}

}  // namespace gsmap
