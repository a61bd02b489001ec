// TEST INFRASTRUCTURE ONLY — flat C-ABI over the oracle so pytest (ctypes) and bench.py's
// cpu_baseline leg can drive it. Exceptions never cross the boundary: every entry point returns
// an int status (0 ok, 1 std::invalid_argument, 2 std::logic_error, 9 other) and the message is
// kept in a thread-local buffer (orc_last_error).
#include <cstring>
#include <memory>

#include "oracle.hpp"

using namespace orc;

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

CameraModel to_cam(const orc_camera_t* c) {
    CameraModel m;
    m.fx = c->fx; m.fy = c->fy; m.cx = c->cx; m.cy = c->cy;
    m.width = c->width; m.height = c->height;
    return m;
}
Pose to_pose(const orc_pose_t* p) {  // already normalised: copy bits verbatim
    Pose q;
    q.qw = p->qw; q.qx = p->qx; q.qy = p->qy; q.qz = p->qz;
    q.t = {p->tx, p->ty, p->tz};
    return q;
}
LearningRates to_lr(const orc_lr_t* l) {
    LearningRates r;
    r.position = l->position; r.rotation = l->rotation; r.log_scale = l->log_scale;
    r.opacity = l->opacity; r.sh = l->sh;
    return r;
}
TrainConfig to_cfg(const orc_cfg_t* c) {
    TrainConfig t;
    t.lambda = c->lambda; t.lambda_d = c->lambda_d;
    t.pyramid_levels = c->pyramid_levels; t.iters_per_level = c->iters_per_level;
    t.lr = to_lr(&c->lr);
    return t;
}
std::vector<Gaussian3D> to_gaussians(const orc_gaussian_t* g, int64_t n) {
    std::vector<Gaussian3D> out(n);
    for (int64_t i = 0; i < n; ++i) {
        flat_to_gaussian(g[i].p, out[i]);
        out[i].active_degree = g[i].degree;
    }
    return out;
}
ImageD to_image(const double* d, int h, int w, int c) {
    ImageD im(h, w, c);
    std::memcpy(im.data.data(), d, sizeof(double) * im.size());
    return im;
}
void from_image(const ImageD& im, double* d) {
    if (d) std::memcpy(d, im.data.data(), sizeof(double) * im.size());
}
std::unique_ptr<ThreadPool> make_pool(int threads) {
    if (threads == 1) return nullptr;
    return std::make_unique<ThreadPool>(threads);
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

int orc_pose_make(double w, double x, double y, double z, double tx, double ty, double tz,
                  orc_pose_t* out) {
    return guard([&] {
        const Pose p(w, x, y, z, {tx, ty, tz});
        *out = {p.qw, p.qx, p.qy, p.qz, p.t.x, p.t.y, p.t.z};
    });
}
int orc_pose_camera_center(const orc_pose_t* p, double* out3) {
    return guard([&] {
        const Vec3 c = to_pose(p).camera_center();
        out3[0] = c.x; out3[1] = c.y; out3[2] = c.z;
    });
}
int orc_camera_scaled(const orc_camera_t* c, int level, orc_camera_t* out) {
    return guard([&] {
        const CameraModel s = to_cam(c).scaled(level);
        *out = {s.fx, s.fy, s.cx, s.cy, s.width, s.height};
    });
}
int orc_camera_validate(const orc_camera_t* c) { return guard([&] { to_cam(c).validate(); }); }

// ---------------------------------------------------------------- core primitives
int orc_build_covariance(const double* q4, const double* ls3, double* out9) {
    return guard([&] {
        Vec4 q;
        for (int i = 0; i < 4; ++i) q[i] = q4[i];
        const Mat3 s = build_covariance(q, {ls3[0], ls3[1], ls3[2]});
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) out9[3 * i + j] = s.m[i][j];
    });
}
// returns 1 in *visible when not culled; mean2, cov4 (row-major), depth, radius
int orc_project_gaussian(const orc_gaussian_t* g, const orc_pose_t* pose, const orc_camera_t* cam,
                         int32_t* visible, double* mean2, double* cov4, double* depth, int32_t* radius) {
    return guard([&] {
        const auto gs = to_gaussians(g, 1);
        const auto p = project_gaussian(gs[0], to_pose(pose), to_cam(cam));
        *visible = p.has_value();
        if (!p) return;
        mean2[0] = p->mean.x; mean2[1] = p->mean.y;
        cov4[0] = p->cov2d.m[0][0]; cov4[1] = p->cov2d.m[0][1];
        cov4[2] = p->cov2d.m[1][0]; cov4[3] = p->cov2d.m[1][1];
        *depth = p->depth;
        *radius = p->radius;
    });
}
int orc_eval_gaussian_2d(const double* mean2, const double* cov4, const double* x2, double* out) {
    return guard([&] {
        Mat2 c;
        c.m[0][0] = cov4[0]; c.m[0][1] = cov4[1]; c.m[1][0] = cov4[2]; c.m[1][1] = cov4[3];
        *out = eval_gaussian_2d_conic({mean2[0], mean2[1]}, inverse2(c), {x2[0], x2[1]});
    });
}
int orc_eval_sh(const double* coeffs48, int degree, const double* dir3, double* out3) {
    return guard([&] {
        std::array<Vec3, 16> c;
        for (int k = 0; k < 16; ++k) c[k] = {coeffs48[3 * k], coeffs48[3 * k + 1], coeffs48[3 * k + 2]};
        const Vec3 r = eval_sh(c, degree, {dir3[0], dir3[1], dir3[2]});
        out3[0] = r.x; out3[1] = r.y; out3[2] = r.z;
    });
}

// ---------------------------------------------------------------- map
void* orc_map_create(const orc_gaussian_t* g, int64_t n) {
    auto* m = new GaussianMap();
    if (n > 0) m->append(to_gaussians(g, n));
    return m;
}
void orc_map_free(void* m) { delete static_cast<GaussianMap*>(m); }
int64_t orc_map_size(void* m) { return static_cast<int64_t>(static_cast<GaussianMap*>(m)->size()); }
int orc_map_append(void* m, const orc_gaussian_t* g, int64_t n) {
    return guard([&] { static_cast<GaussianMap*>(m)->append(to_gaussians(g, n)); });
}
void orc_map_get(void* mp, orc_gaussian_t* out) {
    const auto& gs = static_cast<GaussianMap*>(mp)->gaussians();
    for (size_t i = 0; i < gs.size(); ++i) {
        gaussian_to_flat(gs[i], out[i].p);
        out[i].degree = gs[i].active_degree;
        out[i].pad = 0;
    }
}
void orc_map_set(void* mp, const orc_gaussian_t* in) {  // in-place edit, like gaussians() non-const
    auto& gs = static_cast<GaussianMap*>(mp)->gaussians();
    for (size_t i = 0; i < gs.size(); ++i) {
        flat_to_gaussian(in[i].p, gs[i]);
        gs[i].active_degree = in[i].degree;
    }
}
void orc_map_get_adam(void* mp, double* m, double* v, int64_t* step) {
    const auto& st = static_cast<GaussianMap*>(mp)->optimizer_state();
    for (size_t i = 0; i < st.size(); ++i) {
        std::memcpy(m + 59 * i, st[i].m.data(), 59 * sizeof(double));
        std::memcpy(v + 59 * i, st[i].v.data(), 59 * sizeof(double));
        step[i] = st[i].step;
    }
}
void orc_map_set_adam(void* mp, const double* m, const double* v, const int64_t* step) {
    auto& st = static_cast<GaussianMap*>(mp)->optimizer_state();
    for (size_t i = 0; i < st.size(); ++i) {
        std::memcpy(st[i].m.data(), m + 59 * i, 59 * sizeof(double));
        std::memcpy(st[i].v.data(), v + 59 * i, 59 * sizeof(double));
        st[i].step = step[i];
    }
}
double orc_map_scene_extent(void* m) { return static_cast<GaussianMap*>(m)->scene_extent(); }
void orc_map_set_scene_extent(void* m, double e) { static_cast<GaussianMap*>(m)->set_scene_extent(e); }
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
            GaussianGrad& d = rg.per_gaussian[i];
            d.position = {g[0], g[1], g[2]};
            for (int k = 0; k < 4; ++k) d.rotation[k] = g[3 + k];
            d.log_scale = {g[7], g[8], g[9]};
            d.opacity_logit = g[10];
            for (int k = 0; k < 16; ++k) d.sh[k] = {g[11 + 3 * k], g[12 + 3 * k], g[13 + 3 * k]};
        }
        static_cast<GaussianMap*>(mp)->apply_gradients(rg, to_lr(lr));
    });
}

// ---------------------------------------------------------------- render / backward
int orc_render(void* mp, const orc_pose_t* pose, const orc_camera_t* cam, int threads, void** out) {
    return guard([&] {
        auto pool = make_pool(threads);
        auto* o = new RenderOutput(render(*static_cast<GaussianMap*>(mp), to_pose(pose), to_cam(cam), pool.get()));
        *out = o;
    });
}
void orc_out_free(void* o) { delete static_cast<RenderOutput*>(o); }
void orc_out_images(void* op, double* color, double* depth, double* vis) {
    const auto* o = static_cast<RenderOutput*>(op);
    from_image(o->color, color);
    from_image(o->depth, depth);
    from_image(o->visibility, vis);
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
// per projected (rank order): index, mean2, cov4, cov_inv4, depth, radius, opacity, color3, color_raw3
void orc_out_projected(void* op, int32_t* index, double* mean2, double* cov4, double* cinv4,
                       double* depth, int32_t* radius, double* opacity, double* color3,
                       double* color_raw3) {
    const auto* o = static_cast<RenderOutput*>(op);
    for (size_t i = 0; i < o->projected.size(); ++i) {
        const auto& p = o->projected[i];
        index[i] = p.index;
        mean2[2 * i] = p.mean.x; mean2[2 * i + 1] = p.mean.y;
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) {
                cov4[4 * i + 2 * a + b] = p.cov2d.m[a][b];
                cinv4[4 * i + 2 * a + b] = p.cov_inv.m[a][b];
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
int64_t orc_out_num_bin_entries(void* op) {
    int64_t k = 0;
    for (const auto& b : static_cast<RenderOutput*>(op)->bins) k += static_cast<int64_t>(b.size());
    return k;
}
// tile_offsets[T+1] and entries[K] (rank into projected) — bin_tiles order (rasterizer.cpp:76-91)
void orc_out_bins(void* op, int64_t* tile_offsets, int32_t* entries) {
    const auto* o = static_cast<RenderOutput*>(op);
    int64_t k = 0;
    tile_offsets[0] = 0;
    for (size_t t = 0; t < o->bins.size(); ++t) {
        for (int32_t e : o->bins[t]) entries[k++] = e;
        tile_offsets[t + 1] = k;
    }
}
int orc_out_is_smooth(void* mp, void* op) {
    return config_is_smooth(*static_cast<GaussianMap*>(mp), *static_cast<RenderOutput*>(op)) ? 1 : 0;
}

int orc_render_backward(void* mp, const orc_pose_t* pose, const orc_camera_t* cam, void* op,
                        const double* dcolor, const double* ddepth, int dh, int dw, int threads,
                        double* grads59) {
    return guard([&] {
        auto pool = make_pool(threads);
        const ImageD dc = to_image(dcolor, dh, dw, 3);
        const ImageD dd = to_image(ddepth, dh, dw, 1);
        const auto g = render_backward(*static_cast<GaussianMap*>(mp), to_pose(pose), to_cam(cam),
                                       *static_cast<RenderOutput*>(op), dc, dd, pool.get());
        for (size_t i = 0; i < g.per_gaussian.size(); ++i) grad_to_flat(g.per_gaussian[i], grads59 + 59 * i);
    });
}

int orc_brute_force(void* mp, const orc_pose_t* pose, const orc_camera_t* cam, double* color,
                    double* depth, double* vis) {
    return guard([&] {
        const auto o = brute_force_render(*static_cast<GaussianMap*>(mp), to_pose(pose), to_cam(cam));
        from_image(o.color, color);
        from_image(o.depth, depth);
        from_image(o.visibility, vis);
    });
}

// ---------------------------------------------------------------- metrics / loss
int orc_psnr(const double* a, const double* b, int h, int w, int c, double* out) {
    return guard([&] { *out = psnr(to_image(a, h, w, c), to_image(b, h, w, c)); });
}
int orc_ssim(const double* a, const double* b, int h, int w, int c, double* out, double* grad) {
    return guard([&] {
        if (grad) {
            ImageD g;
            *out = ssim_with_gradient(to_image(a, h, w, c), to_image(b, h, w, c), g);
            from_image(g, grad);
        } else {
            *out = ssim(to_image(a, h, w, c), to_image(b, h, w, c));
        }
    });
}
int orc_depth_rmse(const double* r, const double* g, int h, int w, double* out, int* empty) {
    return guard([&] {
        bool e = false;
        *out = depth_rmse(to_image(r, h, w, 1), to_image(g, h, w, 1), &e);
        *empty = e;
    });
}
// scalars5 = total, color_loss, depth_loss, l1, ssim
int orc_compute_loss(const double* color, const double* depth, const double* vis,
                     const double* gt_color, const double* gt_depth, int h, int w,
                     const orc_cfg_t* cfg, double* dl_dcolor, double* dl_ddepth, double* scalars5) {
    return guard([&] {
        RenderOutput r;
        r.color = to_image(color, h, w, 3);
        r.depth = to_image(depth, h, w, 1);
        r.visibility = to_image(vis, h, w, 1);
        Keyframe kf;
        kf.pyramid.push_back({to_image(gt_color, h, w, 3), to_image(gt_depth, h, w, 1)});
        const LossResult res = compute_loss(r, kf, 0, to_cfg(cfg));
        from_image(res.dl_dcolor, dl_dcolor);
        from_image(res.dl_ddepth, dl_ddepth);
        scalars5[0] = res.total; scalars5[1] = res.color_loss; scalars5[2] = res.depth_loss;
        scalars5[3] = res.l1; scalars5[4] = res.ssim;
    });
}
// out = concatenation of levels 0..levels (each h_l*w_l*c)
int orc_build_pyramid(const double* img, int h, int w, int c, int levels, int is_depth, double* out) {
    return guard([&] {
        const auto v = is_depth ? build_depth_pyramid(to_image(img, h, w, 1), levels)
                                : build_pyramid(to_image(img, h, w, c), levels);
        size_t off = 0;
        for (const auto& im : v) {
            std::memcpy(out + off, im.data.data(), im.size() * sizeof(double));
            off += im.size();
        }
    });
}

// ---------------------------------------------------------------- keyframes / train step
void* orc_keyframe_create(const orc_pose_t* pose, const double* color, const double* sparse_depth,
                          int h, int w, int initial_iters, int levels, int* status) {
    Keyframe* kf = new Keyframe();
    *status = guard([&] {
        kf->pose = to_pose(pose);
        kf->color_image = to_image(color, h, w, 3);
        kf->sparse_depth = to_image(sparse_depth, h, w, 1);
        kf->initial_iters = kf->remaining_iters = initial_iters;
        if (levels >= 0) build_keyframe_pyramid(*kf, levels);
    });
    return kf;
}
void orc_keyframe_free(void* k) { delete static_cast<Keyframe*>(k); }
int orc_keyframe_consumed(void* k) { return static_cast<Keyframe*>(k)->consumed_iters; }
void orc_keyframe_set_consumed(void* k, int c) { static_cast<Keyframe*>(k)->consumed_iters = c; }
// ran = 1 when a step happened (0 = budget exhausted, std::nullopt)
int orc_train_step(void* mp, void* kp, const orc_cfg_t* cfg, const orc_camera_t* cam, void* pool,
                   int* ran, int* level, double* loss, double* psnr_out) {
    return guard([&] {
        const auto r = train_keyframe_step(*static_cast<GaussianMap*>(mp), *static_cast<Keyframe*>(kp),
                                           to_cfg(cfg), to_cam(cam), static_cast<ThreadPool*>(pool));
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

// points: n x 6 (x, y, z, r, g, b)
int orc_init_from_points(void* mp, const double* pts6, int64_t n, int64_t* added) {
    return guard([&] {
        std::vector<ColoredPoint> pts(n);
        for (int64_t i = 0; i < n; ++i) {
            pts[i].position = {pts6[6 * i], pts6[6 * i + 1], pts6[6 * i + 2]};
            pts[i].color = {pts6[6 * i + 3], pts6[6 * i + 4], pts6[6 * i + 5]};
        }
        *added = static_cast<int64_t>(init_gaussians_from_points(*static_cast<GaussianMap*>(mp), pts));
    });
}
int orc_project_sparse_depth(const double* pts6, int64_t n, const orc_pose_t* pose,
                             const orc_camera_t* cam, double* out) {
    return guard([&] {
        std::vector<ColoredPoint> pts(n);
        for (int64_t i = 0; i < n; ++i) pts[i].position = {pts6[6 * i], pts6[6 * i + 1], pts6[6 * i + 2]};
        from_image(project_sparse_depth(pts, to_pose(pose), to_cam(cam)), out);
    });
}

// kept: indices of the kept points (n capacity)
int orc_filter_points_by_visibility(void* mp, const double* pts6, int64_t n, const orc_pose_t* pose,
                                    const orc_camera_t* cam, double tau_alpha, int64_t* kept, int64_t* n_kept) {
    return guard([&] {
        std::vector<ColoredPoint> pts(n);
        for (int64_t i = 0; i < n; ++i) pts[i].position = {pts6[6 * i], pts6[6 * i + 1], pts6[6 * i + 2]};
        const auto k = filter_points_by_visibility(pts, to_pose(pose), *static_cast<GaussianMap*>(mp), to_cam(cam),
                                                   tau_alpha);
        for (size_t i = 0; i < k.size(); ++i) kept[i] = static_cast<int64_t>(k[i]);
        *n_kept = static_cast<int64_t>(k.size());
    });
}

int orc_save_checkpoint(void* mp, const char* path) {
    return guard([&] { save_checkpoint(path, *static_cast<GaussianMap*>(mp)); });
}
int orc_load_checkpoint(const char* path, void** out) {
    return guard([&] { *out = new GaussianMap(load_checkpoint(path)); });
}
// res3 = psnr, ssim, depth_rmse (gt_depth may be NULL)
int orc_evaluate_view(void* mp, const orc_pose_t* pose, const orc_camera_t* cam, const double* gt_color,
                      const double* gt_depth, double* res3) {
    return guard([&] {
        const ImageD gc = to_image(gt_color, cam->height, cam->width, 3);
        const ImageD gd = gt_depth ? to_image(gt_depth, cam->height, cam->width, 1) : ImageD();
        const EvalMetrics m = evaluate_view(*static_cast<GaussianMap*>(mp), to_pose(pose), to_cam(cam), gc,
                                            gt_depth ? &gd : nullptr);
        res3[0] = m.psnr;
        res3[1] = m.ssim;
        res3[2] = m.depth_rmse;
    });
}

// ---------------------------------------------------------------- fixtures
void* orc_rng_create(uint32_t seed) { return new std::mt19937(seed); }
void orc_rng_free(void* r) { delete static_cast<std::mt19937*>(r); }
double orc_rng_uniform(void* r, double lo, double hi) {
    return std::uniform_real_distribution<double>(lo, hi)(*static_cast<std::mt19937*>(r));
}
void* orc_random_scene(void* r, int n, const orc_camera_t* cam, const orc_pose_t* pose, double lo,
                       double hi) {
    return new GaussianMap(random_scene(*static_cast<std::mt19937*>(r), n, to_cam(cam), to_pose(pose), lo, hi));
}

// res4 = max_rel_err_core, max_rel_err_render, configs_run, configs_resampled
int orc_run_gradcheck(uint32_t seed, int configs, int core_configs, int n_gaussians,
                      int image_size, int params_per_config, double* res4) {
    return guard([&] {
        GradCheckOptions o;
        o.seed = seed; o.configs = configs; o.core_configs = core_configs;
        o.n_gaussians = n_gaussians; o.image_size = image_size; o.params_per_config = params_per_config;
        const auto r = run_gradcheck(o);
        res4[0] = r.max_rel_err_core; res4[1] = r.max_rel_err_render;
        res4[2] = r.configs_run; res4[3] = r.configs_resampled;
    });
}

}  // extern "C"
