// TEST INFRASTRUCTURE ONLY — the flat C-ABI of the oracle (same orc_* names and signatures as
// oracle/capi.cpp) implemented over the REFERENCE ITSELF: the reference's own sources under
// /root/reference/proj/src, compiled unchanged against oracle/ref_eigen (see oracle/ref/Makefile).
// Loaded by oracle/pyref.py as a second instance of the oracle wrappers, so every test can run
// the same calls against the restatement (liborc.so) and the reference (libgsref.so).
//
// Entry points the reference has no public equivalent for are omitted (the tile bins of
// rasterizer.cpp's anonymous bin_tiles, the optimizer-state setters); the Python side skips them.
#include <cstring>
#include <memory>
#include <random>
#include <span>

#include "gsmap/core/covariance.hpp"
#include "gsmap/core/projection.hpp"
#include "gsmap/core/sh.hpp"
#include "gsmap/io/checkpoint.hpp"
#include "gsmap/io/sequence.hpp"
#include "gsmap/io/synthetic.hpp"
#include "gsmap/map/gaussian_map.hpp"
#include "gsmap/map/keyframe.hpp"
#include "gsmap/map/mapper.hpp"
#include "gsmap/metrics/metrics.hpp"
#include "gsmap/pipeline/gradcheck.hpp"
#include "gsmap/render/rasterizer.hpp"
#include "support/brute_force.hpp"  // /root/reference/proj/tests/support

using namespace gsmap;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

struct orc_camera_t { double fx, fy, cx, cy; int32_t width, height; };
struct orc_pose_t { double qw, qx, qy, qz, tx, ty, tz; };
struct orc_gaussian_t { double p[59]; int32_t degree; int32_t pad; };
struct orc_lr_t { double position, rotation, log_scale, opacity, sh; };
struct orc_cfg_t {
    double lambda, lambda_d;
    int32_t pyramid_levels, iters_per_level;
    orc_lr_t lr;
};

CameraModel cam_of(const orc_camera_t* c) {
    CameraModel m;
    m.fx = c->fx; m.fy = c->fy; m.cx = c->cx; m.cy = c->cy;
    m.width = c->width; m.height = c->height;
    return m;
}
// the C-ABI pose carries the already-normalised quaternion: set the members directly (the
// Pose(q, t) constructor would normalise a second time)
Pose pose_of(const orc_pose_t* p) {
    Pose q;
    q.rotation = Eigen::Quaterniond(p->qw, p->qx, p->qy, p->qz);
    q.translation = Eigen::Vector3d(p->tx, p->ty, p->tz);
    return q;
}
LearningRates lr_of(const orc_lr_t* l) {
    LearningRates r;
    r.position = l->position; r.rotation = l->rotation; r.log_scale = l->log_scale;
    r.opacity = l->opacity; r.sh = l->sh;
    return r;
}
TrainConfig cfg_of(const orc_cfg_t* c) {
    TrainConfig t;
    t.lambda = c->lambda; t.lambda_d = c->lambda_d;
    t.pyramid_levels = c->pyramid_levels; t.iters_per_level = c->iters_per_level;
    t.lr = lr_of(&c->lr);
    return t;
}
// 59 scalars in gaussian.hpp:16-26 order
void unpack(const double* p, Gaussian3D& g) {
    g.position = Eigen::Vector3d(p[0], p[1], p[2]);
    g.rotation = Eigen::Vector4d(p[3], p[4], p[5], p[6]);
    g.log_scale = Eigen::Vector3d(p[7], p[8], p[9]);
    g.opacity_logit = p[10];
    for (int k = 0; k < kShCoeffCount; ++k) g.sh_coeffs[k] = Eigen::Vector3d(p[11 + 3 * k], p[12 + 3 * k], p[13 + 3 * k]);
}
void pack(const Gaussian3D& g, double* p) {
    for (int i = 0; i < 3; ++i) p[i] = g.position[i];
    for (int i = 0; i < 4; ++i) p[3 + i] = g.rotation[i];
    for (int i = 0; i < 3; ++i) p[7 + i] = g.log_scale[i];
    p[10] = g.opacity_logit;
    for (int k = 0; k < kShCoeffCount; ++k)
        for (int c = 0; c < 3; ++c) p[11 + 3 * k + c] = g.sh_coeffs[k][c];
}
void pack_grad(const grad::GaussianGrad& g, double* p) {
    for (int i = 0; i < 3; ++i) p[i] = g.position[i];
    for (int i = 0; i < 4; ++i) p[3 + i] = g.rotation[i];
    for (int i = 0; i < 3; ++i) p[7 + i] = g.log_scale[i];
    p[10] = g.opacity_logit;
    for (int k = 0; k < kShCoeffCount; ++k)
        for (int c = 0; c < 3; ++c) p[11 + 3 * k + c] = g.sh_coeffs[k][c];
}
std::vector<Gaussian3D> gaussians_of(const orc_gaussian_t* g, int64_t n) {
    std::vector<Gaussian3D> out(n);
    for (int64_t i = 0; i < n; ++i) {
        unpack(g[i].p, out[i]);
        out[i].active_degree = g[i].degree;
    }
    return out;
}
ImageD image_of(const double* d, int h, int w, int c) {
    ImageD im(h, w, c);
    std::memcpy(im.data(), d, sizeof(double) * im.size());
    return im;
}
void store(const ImageD& im, double* d) { std::memcpy(d, im.data(), sizeof(double) * im.size()); }
std::unique_ptr<ThreadPool> pool_of(int threads) {
    return threads > 1 ? std::make_unique<ThreadPool>(threads) : nullptr;
}
std::vector<ColoredPoint> points_of(const double* pts6, int64_t n) {
    std::vector<ColoredPoint> pts(n);
    for (int64_t i = 0; i < n; ++i) {
        pts[i].position = Eigen::Vector3d(pts6[6 * i], pts6[6 * i + 1], pts6[6 * i + 2]);
        pts[i].color = Eigen::Vector3d(pts6[6 * i + 3], pts6[6 * i + 4], pts6[6 * i + 5]);
    }
    return pts;
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }
// identifies this build (the Python side asserts it loaded the reference, not the restatement)
const char* orc_build_kind() { return "reference (/root/reference/proj/src, unchanged, oracle/ref_eigen)"; }

int orc_pose_make(double w, double x, double y, double z, double tx, double ty, double tz, orc_pose_t* out) {
    return guard([&] {
        const Pose p(Eigen::Quaterniond(w, x, y, z), Eigen::Vector3d(tx, ty, tz));
        *out = {p.rotation.w(), p.rotation.x(), p.rotation.y(), p.rotation.z(), p.translation.x(),
                p.translation.y(), p.translation.z()};
    });
}
int orc_pose_camera_center(const orc_pose_t* p, double* out3) {
    return guard([&] {
        const Eigen::Vector3d c = pose_of(p).camera_center();
        for (int i = 0; i < 3; ++i) out3[i] = c[i];
    });
}
int orc_camera_scaled(const orc_camera_t* c, int level, orc_camera_t* out) {
    return guard([&] {
        const CameraModel s = cam_of(c).scaled(level);
        *out = {s.fx, s.fy, s.cx, s.cy, s.width, s.height};
    });
}
int orc_camera_validate(const orc_camera_t* c) { return guard([&] { cam_of(c).validate(); }); }

int orc_build_covariance(const double* q4, const double* ls3, double* out9) {
    return guard([&] {
        const Eigen::Matrix3d s = build_covariance(Eigen::Vector4d(q4[0], q4[1], q4[2], q4[3]),
                                                   Eigen::Vector3d(ls3[0], ls3[1], ls3[2]));
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) out9[3 * i + j] = s(i, j);
    });
}
int orc_project_gaussian(const orc_gaussian_t* g, const orc_pose_t* pose, const orc_camera_t* cam,
                         int32_t* visible, double* mean2, double* cov4, double* depth, int32_t* radius) {
    return guard([&] {
        const auto gs = gaussians_of(g, 1);
        const auto p = project_gaussian(gs[0], pose_of(pose), cam_of(cam));
        *visible = p.has_value();
        if (!p) return;
        mean2[0] = p->mean.x(); mean2[1] = p->mean.y();
        cov4[0] = p->cov2d(0, 0); cov4[1] = p->cov2d(0, 1); cov4[2] = p->cov2d(1, 0); cov4[3] = p->cov2d(1, 1);
        *depth = p->depth;
        *radius = p->radius;
    });
}
int orc_eval_gaussian_2d(const double* mean2, const double* cov4, const double* x2, double* out) {
    return guard([&] {
        Eigen::Matrix2d c;
        c(0, 0) = cov4[0]; c(0, 1) = cov4[1]; c(1, 0) = cov4[2]; c(1, 1) = cov4[3];
        *out = eval_gaussian_2d_conic(Eigen::Vector2d(mean2[0], mean2[1]), c.inverse(), Eigen::Vector2d(x2[0], x2[1]));
    });
}
int orc_eval_sh(const double* coeffs48, int degree, const double* dir3, double* out3) {
    return guard([&] {
        std::array<Eigen::Vector3d, kShCoeffCount> c;
        for (int k = 0; k < kShCoeffCount; ++k) c[k] = Eigen::Vector3d(coeffs48[3 * k], coeffs48[3 * k + 1], coeffs48[3 * k + 2]);
        const Eigen::Vector3d r = eval_sh(c, degree, Eigen::Vector3d(dir3[0], dir3[1], dir3[2]));
        for (int i = 0; i < 3; ++i) out3[i] = r[i];
    });
}

// ---------------------------------------------------------------- map
void* orc_map_create(const orc_gaussian_t* g, int64_t n) {
    auto* m = new GaussianMap();
    if (n > 0) m->append(gaussians_of(g, n));
    return m;
}
void orc_map_free(void* m) { delete static_cast<GaussianMap*>(m); }
int64_t orc_map_size(void* m) { return static_cast<int64_t>(static_cast<GaussianMap*>(m)->size()); }
int orc_map_append(void* m, const orc_gaussian_t* g, int64_t n) {
    return guard([&] { static_cast<GaussianMap*>(m)->append(gaussians_of(g, n)); });
}
void orc_map_get(void* mp, orc_gaussian_t* out) {
    const auto& gs = static_cast<GaussianMap*>(mp)->gaussians();
    for (size_t i = 0; i < gs.size(); ++i) {
        pack(gs[i], out[i].p);
        out[i].degree = gs[i].active_degree;
        out[i].pad = 0;
    }
}
void orc_map_set(void* mp, const orc_gaussian_t* in) {  // non-const gaussians() (gaussian_map.hpp:62)
    auto& gs = static_cast<GaussianMap*>(mp)->gaussians();
    for (size_t i = 0; i < gs.size(); ++i) {
        unpack(in[i].p, gs[i]);
        gs[i].active_degree = in[i].degree;
    }
}
void orc_map_get_adam(void* mp, double* m, double* v, int64_t* step) {
    const auto& st = static_cast<GaussianMap*>(mp)->optimizer_state();
    for (size_t i = 0; i < st.size(); ++i) {
        const AdamState& a = st[i];
        double* pm = m + 59 * i;
        double* pv = v + 59 * i;
        for (int k = 0; k < 3; ++k) { pm[k] = a.m_position[k]; pv[k] = a.v_position[k]; }
        for (int k = 0; k < 4; ++k) { pm[3 + k] = a.m_rotation[k]; pv[3 + k] = a.v_rotation[k]; }
        for (int k = 0; k < 3; ++k) { pm[7 + k] = a.m_log_scale[k]; pv[7 + k] = a.v_log_scale[k]; }
        pm[10] = a.m_opacity; pv[10] = a.v_opacity;
        for (int s = 0; s < kShCoeffCount; ++s)
            for (int c = 0; c < 3; ++c) { pm[11 + 3 * s + c] = a.m_sh[s][c]; pv[11 + 3 * s + c] = a.v_sh[s][c]; }
        step[i] = a.step;
    }
}
double orc_map_scene_extent(void* m) { return static_cast<GaussianMap*>(m)->scene_extent(); }
int64_t orc_map_global_step(void* m) { return static_cast<GaussianMap*>(m)->global_step(); }
void orc_map_set_global_step(void* m, int64_t s) { static_cast<GaussianMap*>(m)->set_global_step(s); }
int64_t orc_map_prune(void* m, double thr, int* status) {
    int64_t removed = 0;
    *status = guard([&] { removed = static_cast<int64_t>(static_cast<GaussianMap*>(m)->prune(thr)); });
    return removed;
}
void orc_map_raise_sh_degree(void* m, int d) { static_cast<GaussianMap*>(m)->raise_sh_degree(d); }
int orc_map_max_active_degree(void* m) { return static_cast<GaussianMap*>(m)->max_active_degree(); }
int orc_maybe_upgrade_sh(void* m, int sh_interval) {
    TrainConfig c;
    c.sh_interval = sh_interval;
    return maybe_upgrade_sh(*static_cast<GaussianMap*>(m), c);
}
int orc_apply_gradients(void* mp, const double* grads59, int64_t n, const orc_lr_t* lr) {
    return guard([&] {
        RenderGradients rg;
        rg.per_gaussian.resize(n);
        for (int64_t i = 0; i < n; ++i) {
            const double* g = grads59 + 59 * i;
            grad::GaussianGrad& d = rg.per_gaussian[i];
            d.position = Eigen::Vector3d(g[0], g[1], g[2]);
            d.rotation = Eigen::Vector4d(g[3], g[4], g[5], g[6]);
            d.log_scale = Eigen::Vector3d(g[7], g[8], g[9]);
            d.opacity_logit = g[10];
            for (int k = 0; k < kShCoeffCount; ++k) d.sh_coeffs[k] = Eigen::Vector3d(g[11 + 3 * k], g[12 + 3 * k], g[13 + 3 * k]);
        }
        static_cast<GaussianMap*>(mp)->apply_gradients(rg, lr_of(lr));
    });
}

// ---------------------------------------------------------------- render / backward
int orc_render(void* mp, const orc_pose_t* pose, const orc_camera_t* cam, int threads, void** out) {
    return guard([&] {
        auto pool = pool_of(threads);
        *out = new RenderOutput(render(*static_cast<GaussianMap*>(mp), pose_of(pose), cam_of(cam), pool.get()));
    });
}
void orc_out_free(void* o) { delete static_cast<RenderOutput*>(o); }
void orc_out_images(void* op, double* color, double* depth, double* vis) {
    const auto* o = static_cast<RenderOutput*>(op);
    store(o->color, color);
    store(o->depth, depth);
    store(o->visibility, vis);
}
int64_t orc_out_num_contribs(void* op) { return static_cast<int64_t>(static_cast<RenderOutput*>(op)->contribs.size()); }
void orc_out_csr(void* op, uint32_t* offsets, int32_t* gauss, double* alpha) {
    const auto* o = static_cast<RenderOutput*>(op);
    std::memcpy(offsets, o->contrib_offsets.data(), o->contrib_offsets.size() * sizeof(uint32_t));
    for (size_t i = 0; i < o->contribs.size(); ++i) {
        gauss[i] = o->contribs[i].gaussian;
        alpha[i] = o->contribs[i].alpha;
    }
}
int64_t orc_out_num_projected(void* op) { return static_cast<int64_t>(static_cast<RenderOutput*>(op)->projected.size()); }
void orc_out_projected(void* op, int32_t* index, double* mean2, double* cov4, double* cinv4, double* depth,
                       int32_t* radius, double* opacity, double* color3, double* color_raw3) {
    const auto* o = static_cast<RenderOutput*>(op);
    for (size_t i = 0; i < o->projected.size(); ++i) {
        const ProjectedGaussian& p = o->projected[i];
        index[i] = p.index;
        mean2[2 * i] = p.mean.x();
        mean2[2 * i + 1] = p.mean.y();
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) {
                cov4[4 * i + 2 * a + b] = p.cov2d(a, b);
                cinv4[4 * i + 2 * a + b] = p.cov_inv(a, b);
            }
        depth[i] = p.depth;
        radius[i] = p.radius;
        opacity[i] = p.opacity;
        for (int c = 0; c < 3; ++c) {
            color3[3 * i + c] = p.color[c];
            color_raw3[3 * i + c] = p.color_raw[c];
        }
    }
}
int orc_render_backward(void* mp, const orc_pose_t* pose, const orc_camera_t* cam, void* op, const double* dcolor,
                        const double* ddepth, int dh, int dw, int threads, double* grads59) {
    return guard([&] {
        auto pool = pool_of(threads);
        const auto g = render_backward(*static_cast<GaussianMap*>(mp), pose_of(pose), cam_of(cam),
                                       *static_cast<RenderOutput*>(op), image_of(dcolor, dh, dw, 3),
                                       image_of(ddepth, dh, dw, 1), pool.get());
        for (size_t i = 0; i < g.per_gaussian.size(); ++i) pack_grad(g.per_gaussian[i], grads59 + 59 * i);
    });
}
int orc_brute_force(void* mp, const orc_pose_t* pose, const orc_camera_t* cam, double* color, double* depth,
                    double* vis) {
    return guard([&] {
        const auto o = testing::brute_force_render(*static_cast<GaussianMap*>(mp), pose_of(pose), cam_of(cam));
        store(o.color, color);
        store(o.depth, depth);
        store(o.visibility, vis);
    });
}

// ---------------------------------------------------------------- metrics / loss
int orc_psnr(const double* a, const double* b, int h, int w, int c, double* out) {
    return guard([&] { *out = psnr(image_of(a, h, w, c), image_of(b, h, w, c)); });
}
int orc_ssim(const double* a, const double* b, int h, int w, int c, double* out, double* grad) {
    return guard([&] {
        if (grad) {
            ImageD g;
            *out = ssim_with_gradient(image_of(a, h, w, c), image_of(b, h, w, c), g);
            store(g, grad);
        } else {
            *out = ssim(image_of(a, h, w, c), image_of(b, h, w, c));
        }
    });
}
int orc_depth_rmse(const double* r, const double* g, int h, int w, double* out, int* empty) {
    return guard([&] {
        bool e = false;
        *out = depth_rmse(image_of(r, h, w, 1), image_of(g, h, w, 1), &e);
        *empty = e;
    });
}
int orc_compute_loss(const double* color, const double* depth, const double* vis, const double* gt_color,
                     const double* gt_depth, int h, int w, const orc_cfg_t* cfg, double* dl_dcolor,
                     double* dl_ddepth, double* scalars5) {
    return guard([&] {
        RenderOutput r;
        r.color = image_of(color, h, w, 3);
        r.depth = image_of(depth, h, w, 1);
        r.visibility = image_of(vis, h, w, 1);
        Keyframe kf;
        kf.pyramid.push_back({image_of(gt_color, h, w, 3), image_of(gt_depth, h, w, 1)});
        const LossResult res = compute_loss(r, kf, 0, cfg_of(cfg));
        store(res.dl_dcolor, dl_dcolor);
        store(res.dl_ddepth, dl_ddepth);
        scalars5[0] = res.total; scalars5[1] = res.color_loss; scalars5[2] = res.depth_loss;
        scalars5[3] = res.l1; scalars5[4] = res.ssim;
    });
}
int orc_build_pyramid(const double* img, int h, int w, int c, int levels, int is_depth, double* out) {
    return guard([&] {
        const auto v = is_depth ? build_depth_pyramid(image_of(img, h, w, 1), levels)
                                : build_pyramid(image_of(img, h, w, c), levels);
        size_t off = 0;
        for (const auto& im : v) {
            std::memcpy(out + off, im.data(), im.size() * sizeof(double));
            off += im.size();
        }
    });
}

// ---------------------------------------------------------------- keyframes / train step
void* orc_keyframe_create(const orc_pose_t* pose, const double* color, const double* sparse_depth, int h, int w,
                          int initial_iters, int levels, int* status) {
    auto* kf = new Keyframe();
    *status = guard([&] {
        kf->pose = pose_of(pose);
        kf->color_image = image_of(color, h, w, 3);
        kf->sparse_depth = image_of(sparse_depth, h, w, 1);
        kf->initial_iters = kf->remaining_iters = initial_iters;
        if (levels >= 0) build_keyframe_pyramid(*kf, levels);
    });
    return kf;
}
void orc_keyframe_free(void* k) { delete static_cast<Keyframe*>(k); }
int orc_keyframe_consumed(void* k) { return static_cast<Keyframe*>(k)->consumed_iters; }
void orc_keyframe_set_consumed(void* k, int c) { static_cast<Keyframe*>(k)->consumed_iters = c; }
int orc_train_step(void* mp, void* kp, const orc_cfg_t* cfg, const orc_camera_t* cam, void* pool, int* ran,
                   int* level, double* loss, double* psnr_out) {
    return guard([&] {
        const auto r = train_keyframe_step(*static_cast<GaussianMap*>(mp), *static_cast<Keyframe*>(kp), cfg_of(cfg),
                                           cam_of(cam), static_cast<ThreadPool*>(pool));
        *ran = r.has_value();
        if (r) {
            *level = r->level;
            *loss = r->loss;
            *psnr_out = r->psnr;
        }
    });
}
void* orc_pool_create(int threads) { return new ThreadPool(threads); }
void orc_pool_free(void* p) { delete static_cast<ThreadPool*>(p); }
int orc_pool_threads(void* p) { return static_cast<ThreadPool*>(p)->thread_count(); }

int orc_init_from_points(void* mp, const double* pts6, int64_t n, int64_t* added) {
    return guard([&] {
        const auto pts = points_of(pts6, n);
        *added = static_cast<int64_t>(init_gaussians_from_points(*static_cast<GaussianMap*>(mp), pts));
    });
}
int orc_project_sparse_depth(const double* pts6, int64_t n, const orc_pose_t* pose, const orc_camera_t* cam,
                             double* out) {
    return guard([&] { store(project_sparse_depth(points_of(pts6, n), pose_of(pose), cam_of(cam)), out); });
}
// kept: indices of the kept points (the reference returns the kept points in input order)
int orc_filter_points_by_visibility(void* mp, const double* pts6, int64_t n, const orc_pose_t* pose,
                                    const orc_camera_t* cam, double tau_alpha, int64_t* kept, int64_t* n_kept) {
    return guard([&] {
        const auto pts = points_of(pts6, n);
        Keyframe kf;
        kf.pose = pose_of(pose);
        const auto k = filter_points_by_visibility(pts, kf, *static_cast<GaussianMap*>(mp), cam_of(cam), tau_alpha);
        int64_t j = 0, m = 0;
        for (const ColoredPoint& p : k) {
            while (j < n && !(pts[j].position == p.position)) ++j;
            if (j == n) throw std::logic_error("filter_points_by_visibility: kept point not found");
            kept[m++] = j++;
        }
        *n_kept = m;
    });
}
int orc_save_checkpoint(void* mp, const char* path) {
    return guard([&] { save_checkpoint(path, *static_cast<GaussianMap*>(mp)); });
}
int orc_load_checkpoint(const char* path, void** out) {
    return guard([&] { *out = new GaussianMap(load_checkpoint(path)); });
}

// ---------------------------------------------------------------- fixtures
void* orc_rng_create(uint32_t seed) { return new std::mt19937(seed); }
void orc_rng_free(void* r) { delete static_cast<std::mt19937*>(r); }
double orc_rng_uniform(void* r, double lo, double hi) {
    return std::uniform_real_distribution<double>(lo, hi)(*static_cast<std::mt19937*>(r));
}
void* orc_random_scene(void* r, int n, const orc_camera_t* cam, const orc_pose_t* pose, double lo, double hi) {
    return new GaussianMap(testing::random_scene(*static_cast<std::mt19937*>(r), n, cam_of(cam), pose_of(pose), lo, hi));
}
int orc_run_gradcheck(uint32_t seed, int configs, int core_configs, int n_gaussians, int image_size,
                      int params_per_config, double* res4) {
    return guard([&] {
        GradCheckOptions o;
        o.seed = seed; o.configs = configs; o.core_configs = core_configs;
        o.n_gaussians = n_gaussians; o.image_size = image_size; o.params_per_config = params_per_config;
        const auto r = run_gradcheck(o);
        res4[0] = r.max_rel_err_core; res4[1] = r.max_rel_err_render;
        res4[2] = r.configs_run; res4[3] = r.configs_resampled;
    });
}

// generate_synthetic_scene (io/synthetic.cpp:48-187): the GT map, camera and per-frame poses +
// clouds (points [n][6]); the caller passes capacities from the _sizes call
void* orc_synthetic_scene(int n_gaussians, double extent, int n_frames, uint32_t seed, int width, int height,
                          double focal, double lidar_noise, int orbit, int* status) {
    SyntheticScene* s = nullptr;
    *status = guard([&] {
        SyntheticSpec spec;
        spec.n_gaussians = n_gaussians; spec.extent = extent; spec.n_frames = n_frames; spec.seed = seed;
        spec.width = width; spec.height = height; spec.focal = focal; spec.lidar_noise = lidar_noise;
        spec.trajectory = orbit ? "orbit" : "line";
        s = new SyntheticScene(generate_synthetic_scene(spec));
    });
    return s;
}
void orc_synthetic_free(void* s) { delete static_cast<SyntheticScene*>(s); }
void* orc_synthetic_map(void* s) { return &static_cast<SyntheticScene*>(s)->map; }  // owned by the scene
void orc_synthetic_camera(void* s, orc_camera_t* out) {
    const CameraModel& c = static_cast<SyntheticScene*>(s)->camera;
    *out = {c.fx, c.fy, c.cx, c.cy, c.width, c.height};
}
void orc_synthetic_frame(void* s, int f, orc_pose_t* pose, int64_t* n_points) {
    const Frame& fr = static_cast<SyntheticScene*>(s)->frames.at(f);
    *pose = {fr.pose.rotation.w(), fr.pose.rotation.x(), fr.pose.rotation.y(), fr.pose.rotation.z(),
             fr.pose.translation.x(), fr.pose.translation.y(), fr.pose.translation.z()};
    *n_points = static_cast<int64_t>(fr.cloud.size());
}
void orc_synthetic_cloud(void* s, int f, double* pts6) {
    const Frame& fr = static_cast<SyntheticScene*>(s)->frames.at(f);
    for (size_t i = 0; i < fr.cloud.size(); ++i) {
        for (int k = 0; k < 3; ++k) {
            pts6[6 * i + k] = fr.cloud[i].position[k];
            pts6[6 * i + 3 + k] = fr.cloud[i].color[k];
        }
    }
}
void orc_synthetic_images(void* s, int f, double* color, double* depth) {
    const SyntheticScene* sc = static_cast<SyntheticScene*>(s);
    store(sc->frames.at(f).color, color);
    store(sc->gt_depths.at(f), depth);
}

}  // extern "C"
