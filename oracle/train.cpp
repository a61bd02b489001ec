// TEST INFRASTRUCTURE ONLY — oracle restatement of proj/src/map/gaussian_map.cpp (Adam),
// proj/src/metrics/metrics.cpp (SSIM/PSNR), proj/src/map/mapper.cpp (loss, pyramid, schedule,
// init), proj/src/io/sequence.cpp:246-259, proj/tests/support/brute_force.hpp:92-117 and
// proj/src/pipeline/gradcheck.cpp, io/checkpoint.cpp (format v1) and pipeline.cpp:34-64 (eval).
#include <algorithm>
#include <fstream>
#include <limits>
#include <sstream>
#include <unordered_map>

#include "oracle.hpp"

namespace orc {

// ------------------------------------------------------------------ gaussian_map.cpp
namespace {
constexpr double kBeta1 = 0.9, kBeta2 = 0.999, kEps = 1e-15;  // gaussian_map.cpp:11-13

inline double adam_step(double grad, double& m, double& v, int64_t t, double lr) {  // :15-21
    m = kBeta1 * m + (1.0 - kBeta1) * grad;
    v = kBeta2 * v + (1.0 - kBeta2) * grad * grad;
    const double m_hat = m / (1.0 - std::pow(kBeta1, static_cast<double>(t)));
    const double v_hat = v / (1.0 - std::pow(kBeta2, static_cast<double>(t)));
    return -lr * m_hat / (std::sqrt(v_hat) + kEps);
}
}  // namespace

void GaussianMap::append(const std::vector<Gaussian3D>& gs) {  // gaussian_map.cpp:31-35
    gaussians_.insert(gaussians_.end(), gs.begin(), gs.end());
    opt_.resize(gaussians_.size());
    refresh_extent();
}

void GaussianMap::apply_gradients(const RenderGradients& grads, const LearningRates& lr) {
    // gaussian_map.cpp:37-54 — every Gaussian, every one of the 59 scalars, eps = 1e-15.
    if (grads.per_gaussian.size() != gaussians_.size())
        throw std::invalid_argument("apply_gradients: gradient count does not match map size");
    const double lr_pos = lr.position * scene_extent_;
    double p[59], g[59];
    for (size_t i = 0; i < gaussians_.size(); ++i) {
        Gaussian3D& ga = gaussians_[i];
        AdamState& s = opt_[i];
        gaussian_to_flat(ga, p);
        grad_to_flat(grads.per_gaussian[i], g);
        const int64_t t = ++s.step;
        for (int k = 0; k < 59; ++k) {
            const double rate = k < 3 ? lr_pos : k < 7 ? lr.rotation : k < 10 ? lr.log_scale
                                : k < 11 ? lr.opacity : lr.sh;
            p[k] += adam_step(g[k], s.m[k], s.v[k], t, rate);
        }
        const int deg = ga.active_degree;
        flat_to_gaussian(p, ga);
        ga.active_degree = deg;
    }
    ++global_step_;
}

size_t GaussianMap::prune(double threshold) {  // gaussian_map.cpp:56-73
    if (threshold <= 0.0 || threshold >= 1.0)
        throw std::invalid_argument("prune: threshold must be in (0, 1)");
    size_t kept = 0;
    for (size_t i = 0; i < gaussians_.size(); ++i) {
        if (gaussians_[i].opacity() >= threshold) {
            if (kept != i) {
                gaussians_[kept] = gaussians_[i];
                opt_[kept] = opt_[i];
            }
            ++kept;
        }
    }
    const size_t removed = gaussians_.size() - kept;
    gaussians_.resize(kept);
    opt_.resize(kept);
    return removed;
}

void GaussianMap::raise_sh_degree(int degree) {  // gaussian_map.cpp:75-79
    const int d = std::clamp(degree, 0, kShMaxDegree);
    for (auto& g : gaussians_) g.active_degree = std::max(g.active_degree, d);
}

int GaussianMap::max_active_degree() const {
    int d = 0;
    for (const auto& g : gaussians_) d = std::max(d, g.active_degree);
    return d;
}

void GaussianMap::refresh_extent() {  // gaussian_map.cpp:87-99
    if (gaussians_.empty()) {
        scene_extent_ = 1.0;
        return;
    }
    Vec3 lo = gaussians_.front().position, hi = lo;
    for (const auto& g : gaussians_)
        for (int c = 0; c < 3; ++c) {
            lo[c] = std::min(lo[c], g.position[c]);
            hi[c] = std::max(hi[c], g.position[c]);
        }
    scene_extent_ = std::max(0.5 * norm(sub(hi, lo)), 1e-6);
}

// ------------------------------------------------------------------ metrics.cpp
namespace {
constexpr int kWindow = 11, kHalf = 5;
constexpr double kSsimC1 = 0.01 * 0.01, kSsimC2 = 0.03 * 0.03;

const std::array<double, kWindow>& gaussian_taps() {  // metrics.cpp:20-30
    static const std::array<double, kWindow> taps = [] {
        std::array<double, kWindow> g{};
        double sum = 0.0;
        for (int i = 0; i < kWindow; ++i) {
            const double d = i - kHalf;
            g[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
            sum += g[i];
        }
        for (double& v : g) v /= sum;
        return g;
    }();
    return taps;
}

void conv_valid(const std::vector<double>& in, int h, int w, std::vector<double>& out) {  // :34-52
    const auto& g = gaussian_taps();
    const int vw = w - kWindow + 1, vh = h - kWindow + 1;
    std::vector<double> tmp(size_t(h) * vw);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < vw; ++x) {
            double s = 0.0;
            for (int k = 0; k < kWindow; ++k) s += g[k] * in[size_t(y) * w + x + k];
            tmp[size_t(y) * vw + x] = s;
        }
    out.assign(size_t(vh) * vw, 0.0);
    for (int y = 0; y < vh; ++y)
        for (int x = 0; x < vw; ++x) {
            double s = 0.0;
            for (int k = 0; k < kWindow; ++k) s += g[k] * tmp[size_t(y + k) * vw + x];
            out[size_t(y) * vw + x] = s;
        }
}

void conv_valid_adjoint(const std::vector<double>& in, int h, int w, std::vector<double>& out) {
    // metrics.cpp:55-73
    const auto& g = gaussian_taps();
    const int vw = w - kWindow + 1, vh = h - kWindow + 1;
    std::vector<double> tmp(size_t(h) * vw, 0.0);
    for (int y = 0; y < vh; ++y)
        for (int x = 0; x < vw; ++x) {
            const double v = in[size_t(y) * vw + x];
            if (v == 0.0) continue;
            for (int k = 0; k < kWindow; ++k) tmp[size_t(y + k) * vw + x] += g[k] * v;
        }
    out.assign(size_t(h) * w, 0.0);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < vw; ++x) {
            const double v = tmp[size_t(y) * vw + x];
            if (v == 0.0) continue;
            for (int k = 0; k < kWindow; ++k) out[size_t(y) * w + x + k] += g[k] * v;
        }
}

double ssim_impl(const ImageD& a, const ImageD& b, ImageD* d_da) {  // metrics.cpp:82-161
    if (!a.same_shape(b)) throw std::invalid_argument("ssim: image dimensions mismatch");
    if (a.h < kWindow || a.w < kWindow)
        throw std::invalid_argument("ssim: image smaller than the 11x11 window");
    const int h = a.h, w = a.w, channels = a.c;
    const int vh = h - kWindow + 1, vw = w - kWindow + 1;
    const double inv_n = 1.0 / (static_cast<double>(vh) * vw * channels);
    if (d_da) *d_da = ImageD(h, w, channels, 0.0);
    std::vector<double> pa, pb, a2, b2, ab, mu_a, mu_b, m_a2, m_b2, m_ab, back;
    std::vector<double> w_mu(size_t(vh) * vw), w_a2(w_mu.size()), w_ab(w_mu.size());
    double total = 0.0;
    for (int c = 0; c < channels; ++c) {
        pa.resize(size_t(h) * w);
        pb.resize(pa.size());
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                pa[size_t(y) * w + x] = a.at(y, x, c);
                pb[size_t(y) * w + x] = b.at(y, x, c);
            }
        a2.resize(pa.size());
        b2.resize(pa.size());
        ab.resize(pa.size());
        for (size_t i = 0; i < pa.size(); ++i) {
            a2[i] = pa[i] * pa[i];
            b2[i] = pb[i] * pb[i];
            ab[i] = pa[i] * pb[i];
        }
        conv_valid(pa, h, w, mu_a);
        conv_valid(pb, h, w, mu_b);
        conv_valid(a2, h, w, m_a2);
        conv_valid(b2, h, w, m_b2);
        conv_valid(ab, h, w, m_ab);
        for (size_t i = 0; i < mu_a.size(); ++i) {
            const double ma = mu_a[i], mb = mu_b[i];
            const double sa = m_a2[i] - ma * ma;
            const double sb = m_b2[i] - mb * mb;
            const double sab = m_ab[i] - ma * mb;
            const double num1 = 2.0 * ma * mb + kSsimC1;
            const double num2 = 2.0 * sab + kSsimC2;
            const double den1 = ma * ma + mb * mb + kSsimC1;
            const double den2 = sa + sb + kSsimC2;
            const double s = (num1 * num2) / (den1 * den2);
            total += s;
            if (d_da) {
                const double inv_dd = 1.0 / (den1 * den2);
                const double ds_dsab = 2.0 * num1 * inv_dd;
                const double ds_dsa = -s / den2;
                const double ds_dmu_direct = (2.0 * mb * num2) * inv_dd - s * (2.0 * ma) / den1;
                const double ds_dmu = ds_dmu_direct + ds_dsa * (-2.0 * ma) + ds_dsab * (-mb);
                w_mu[i] = ds_dmu * inv_n;
                w_a2[i] = ds_dsa * inv_n;
                w_ab[i] = ds_dsab * inv_n;
            }
        }
        if (d_da) {
            conv_valid_adjoint(w_mu, h, w, back);
            for (int y = 0; y < h; ++y)
                for (int x = 0; x < w; ++x) d_da->at(y, x, c) += back[size_t(y) * w + x];
            conv_valid_adjoint(w_a2, h, w, back);
            for (int y = 0; y < h; ++y)
                for (int x = 0; x < w; ++x)
                    d_da->at(y, x, c) += 2.0 * pa[size_t(y) * w + x] * back[size_t(y) * w + x];
            conv_valid_adjoint(w_ab, h, w, back);
            for (int y = 0; y < h; ++y)
                for (int x = 0; x < w; ++x)
                    d_da->at(y, x, c) += pb[size_t(y) * w + x] * back[size_t(y) * w + x];
        }
    }
    return total * inv_n;
}
}  // namespace

double psnr(const ImageD& a, const ImageD& b) {  // metrics.cpp:165-175
    if (!a.same_shape(b)) throw std::invalid_argument("psnr: image dimensions mismatch");
    double mse = 0.0;
    for (size_t i = 0; i < a.size(); ++i) {
        const double d = a.data[i] - b.data[i];
        mse += d * d;
    }
    mse /= static_cast<double>(a.size());
    if (mse == 0.0) return 100.0;
    return 10.0 * std::log10(1.0 / mse);
}

double ssim(const ImageD& a, const ImageD& b) { return ssim_impl(a, b, nullptr); }
double ssim_with_gradient(const ImageD& a, const ImageD& b, ImageD& d) { return ssim_impl(a, b, &d); }

double depth_rmse(const ImageD& rendered, const ImageD& gt, bool* empty_mask) {  // :183-197
    if (!rendered.same_shape(gt)) throw std::invalid_argument("depth_rmse: dimensions mismatch");
    double sum = 0.0;
    size_t n = 0;
    for (size_t i = 0; i < gt.size(); ++i)
        if (gt.data[i] > 0.0) {
            const double d = rendered.data[i] - gt.data[i];
            sum += d * d;
            ++n;
        }
    if (empty_mask) *empty_mask = (n == 0);
    if (n == 0) return std::nan("");
    return std::sqrt(sum / static_cast<double>(n));
}

// ------------------------------------------------------------------ mapper.cpp
namespace {
ImageD downsample_color(const ImageD& in) {  // mapper.cpp:65-88
    const int h = (in.h + 1) / 2, w = (in.w + 1) / 2;
    ImageD out(h, w, in.c, 0.0);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x)
            for (int c = 0; c < in.c; ++c) {
                double sum = 0.0;
                int n = 0;
                for (int dy = 0; dy < 2; ++dy)
                    for (int dx = 0; dx < 2; ++dx) {
                        const int sy = 2 * y + dy, sx = 2 * x + dx;
                        if (sy < in.h && sx < in.w) {
                            sum += in.at(sy, sx, c);
                            ++n;
                        }
                    }
                out.at(y, x, c) = sum / n;
            }
    return out;
}

ImageD downsample_depth(const ImageD& in) {  // mapper.cpp:90-110
    const int h = (in.h + 1) / 2, w = (in.w + 1) / 2;
    ImageD out(h, w, 1, 0.0);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            double sum = 0.0;
            int n = 0;
            for (int dy = 0; dy < 2; ++dy)
                for (int dx = 0; dx < 2; ++dx) {
                    const int sy = 2 * y + dy, sx = 2 * x + dx;
                    if (sy < in.h && sx < in.w && in.at(sy, sx) > 0.0) {
                        sum += in.at(sy, sx);
                        ++n;
                    }
                }
            out.at(y, x) = n ? sum / n : 0.0;
        }
    return out;
}

void check_pyramid_size(int h, int w, int levels) {  // mapper.cpp:112-116
    if (levels < 0) throw std::invalid_argument("build_pyramid: levels must be >= 0");
    if (h < (1 << levels) || w < (1 << levels))
        throw std::invalid_argument("build_pyramid: image too small for requested levels");
}
}  // namespace

std::vector<ImageD> build_pyramid(const ImageD& image, int levels) {  // mapper.cpp:120-127
    check_pyramid_size(image.h, image.w, levels);
    std::vector<ImageD> out;
    out.push_back(image);
    for (int l = 0; l < levels; ++l) out.push_back(downsample_color(out.back()));
    return out;
}

std::vector<ImageD> build_depth_pyramid(const ImageD& depth, int levels) {  // :129-135
    check_pyramid_size(depth.h, depth.w, levels);
    std::vector<ImageD> out;
    out.push_back(depth);
    for (int l = 0; l < levels; ++l) out.push_back(downsample_depth(out.back()));
    return out;
}

void build_keyframe_pyramid(Keyframe& kf, int levels) {  // mapper.cpp:137-144
    auto colors = build_pyramid(kf.color_image, levels);
    auto depths = build_depth_pyramid(kf.sparse_depth, levels);
    kf.pyramid.clear();
    for (size_t i = 0; i < colors.size(); ++i)
        kf.pyramid.push_back({std::move(colors[i]), std::move(depths[i])});
}

LossResult compute_loss(const RenderOutput& rendered, const Keyframe& kf, int level,
                        const TrainConfig& cfg) {  // mapper.cpp:146-212
    if (level < 0 || level >= static_cast<int>(kf.pyramid.size()))
        throw std::invalid_argument("compute_loss: pyramid level out of range");
    const ImageD& gt_color = kf.pyramid[level].color;
    const ImageD& gt_depth = kf.pyramid[level].depth;
    if (!rendered.color.same_shape(gt_color))
        throw std::invalid_argument("compute_loss: rendered resolution does not match level");
    LossResult res;
    const int h = gt_color.h, w = gt_color.w;
    res.dl_dcolor = ImageD(h, w, 3, 0.0);
    const double inv_n = 1.0 / (static_cast<double>(h) * w * 3);
    double l1 = 0.0;
    for (size_t i = 0; i < gt_color.size(); ++i) {
        const double d = rendered.color.data[i] - gt_color.data[i];
        l1 += std::abs(d);
        res.dl_dcolor.data[i] = (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) * inv_n * (1.0 - cfg.lambda);
    }
    res.l1 = l1 * inv_n;
    if (cfg.lambda != 0.0) {
        ImageD d_ssim;
        res.ssim = ssim_with_gradient(rendered.color, gt_color, d_ssim);
        for (size_t i = 0; i < d_ssim.size(); ++i) res.dl_dcolor.data[i] += -cfg.lambda * d_ssim.data[i];
    } else {
        res.ssim = 0.0;
    }
    res.color_loss = (1.0 - cfg.lambda) * res.l1 + (cfg.lambda != 0.0 ? cfg.lambda * (1.0 - res.ssim) : 0.0);
    res.dl_ddepth = ImageD(h, w, 1, 0.0);
    double ld = 0.0;
    size_t n_valid = 0;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x)
            if (gt_depth.at(y, x) > 0.0 && rendered.visibility.at(y, x) > kDepthLossMinVisibility)
                ++n_valid;
    if (n_valid > 0) {
        const double inv_v = 1.0 / static_cast<double>(n_valid);
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                const double vis = rendered.visibility.at(y, x);
                if (gt_depth.at(y, x) > 0.0 && vis > kDepthLossMinVisibility) {
                    const double d = rendered.depth.at(y, x) / vis - gt_depth.at(y, x);
                    ld += std::abs(d);
                    res.dl_ddepth.at(y, x) =
                        (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) * inv_v * cfg.lambda_d / vis;
                }
            }
        ld *= inv_v;
    }
    res.depth_loss = ld;
    res.total = res.color_loss + cfg.lambda_d * res.depth_loss;
    return res;
}

std::optional<StepReport> train_keyframe_step(GaussianMap& map, Keyframe& kf,
                                              const TrainConfig& cfg, const CameraModel& cam,
                                              ThreadPool* pool) {  // mapper.cpp:214-238
    if (kf.pyramid.empty())
        throw std::invalid_argument("train_keyframe_step: keyframe pyramid not built");
    if (kf.consumed_iters >= kf.initial_iters) return std::nullopt;
    const int n = static_cast<int>(kf.pyramid.size()) - 1;
    const int ipl = cfg.effective_iters_per_level(kf.initial_iters);
    const int level = n - std::min(n, kf.consumed_iters / ipl);
    const CameraModel level_cam = cam.scaled(level);
    const RenderOutput out = render(map, kf.pose, level_cam, pool);
    const LossResult loss = compute_loss(out, kf, level, cfg);
    const RenderGradients grads =
        render_backward(map, kf.pose, level_cam, out, loss.dl_dcolor, loss.dl_ddepth, pool);
    map.apply_gradients(grads, cfg.lr);
    ++kf.consumed_iters;
    StepReport r;
    r.level = level;
    r.loss = loss.total;
    r.psnr = psnr(out.color, kf.pyramid[level].color);
    return r;
}

int maybe_upgrade_sh(GaussianMap& map, const TrainConfig& cfg) {  // mapper.cpp:240-246
    if (cfg.sh_interval <= 0) return map.max_active_degree();
    const int target = static_cast<int>(std::min<int64_t>(kShMaxDegree, map.global_step() / cfg.sh_interval));
    map.raise_sh_degree(target);
    return target;
}

namespace {
constexpr double kShC0 = 0.28209479177387814;
constexpr double kMinInitScale = 1e-4, kDefaultInitScale = 0.1, kInitOpacity = 0.1;

double mean_knn_distance(const std::vector<ColoredPoint>& pts, size_t i, int k) {  // mapper.cpp:19-39
    std::array<double, 3> best{};
    int found = 0;
    for (size_t j = 0; j < pts.size(); ++j) {
        if (j == i) continue;
        const Vec3 d = sub(pts[j].position, pts[i].position);
        const double d2 = (d.x * d.x + d.y * d.y) + d.z * d.z;
        if (found < k) {
            best[found++] = d2;
            std::push_heap(best.begin(), best.begin() + found);
        } else if (d2 < best.front()) {
            std::pop_heap(best.begin(), best.begin() + k);
            best[k - 1] = d2;
            std::push_heap(best.begin(), best.begin() + k);
        }
    }
    if (found == 0) return kDefaultInitScale;
    double sum = 0.0;
    for (int j = 0; j < found; ++j) sum += std::sqrt(best[j]);
    return sum / found;
}

Gaussian3D gaussian_from_point(const ColoredPoint& p, double s) {  // mapper.cpp:47-58
    Gaussian3D g;
    g.position = p.position;
    g.rotation = Vec4{{1, 0, 0, 0}};
    g.log_scale = {std::log(s), std::log(s), std::log(s)};
    g.opacity_logit = logit(kInitOpacity);
    for (auto& c : g.sh) c = {0, 0, 0};
    g.sh[0] = {(p.color.x - 0.5) / kShC0, (p.color.y - 0.5) / kShC0, (p.color.z - 0.5) / kShC0};
    g.active_degree = 0;
    return g;
}
}  // namespace

size_t init_gaussians_from_points(GaussianMap& map, const std::vector<ColoredPoint>& points) {
    // mapper.cpp:43-61 (O(n^2) brute-force 3-NN, as the reference)
    if (points.empty()) return 0;
    const int k = static_cast<int>(std::min<size_t>(3, points.size() - 1));
    std::vector<Gaussian3D> fresh(points.size());
    for (size_t i = 0; i < points.size(); ++i) {
        const double s = k > 0 ? std::max(mean_knn_distance(points, i, k), kMinInitScale)
                               : kDefaultInitScale;
        fresh[i] = gaussian_from_point(points[i], s);
    }
    map.append(fresh);
    return fresh.size();
}

ImageD project_sparse_depth(const std::vector<ColoredPoint>& points, const Pose& pose,
                            const CameraModel& cam) {  // io/sequence.cpp:246-259
    ImageD depth(cam.height, cam.width, 1, 0.0);
    for (const ColoredPoint& p : points) {
        const Vec3 pc = pose.world_to_camera(p.position);
        if (pc.z <= kNearClip) continue;
        const long px = std::lround(cam.fx * pc.x / pc.z + cam.cx);
        const long py = std::lround(cam.fy * pc.y / pc.z + cam.cy);
        if (px < 0 || px >= cam.width || py < 0 || py >= cam.height) continue;
        double& d = depth.at(static_cast<int>(py), static_cast<int>(px));
        if (d == 0.0 || pc.z < d) d = pc.z;
    }
    return depth;
}

std::vector<size_t> filter_points_by_visibility(const std::vector<ColoredPoint>& points, const Pose& pose,
                                                const GaussianMap& map, const CameraModel& cam,
                                                double tau_alpha) {  // keyframe.cpp:49-74 (kept indices)
    if (tau_alpha < 0.0 || tau_alpha > 1.0)
        throw std::invalid_argument("filter_points_by_visibility: tau_alpha must be in [0,1]");
    const RenderOutput out = render(map, pose, cam);
    std::vector<size_t> kept;
    for (size_t i = 0; i < points.size(); ++i) {
        const Vec3 pc = pose.world_to_camera(points[i].position);
        bool keep = true;
        if (pc.z > kNearClip) {
            const long px = std::lround(cam.fx * pc.x / pc.z + cam.cx);
            const long py = std::lround(cam.fy * pc.y / pc.z + cam.cy);
            if (px >= 0 && px < cam.width && py >= 0 && py < cam.height)
                keep = out.visibility.at(static_cast<int>(py), static_cast<int>(px)) <= tau_alpha;
        }
        if (keep) kept.push_back(i);
    }
    return kept;
}

// ------------------------------------------------------------------ io/checkpoint.cpp:17-73 (format v1)
void save_checkpoint(const std::string& path, const GaussianMap& map) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("save_checkpoint: cannot open " + path);
    out << "gsmap-checkpoint" << ' ' << 1 << '\n' << "count " << map.size() << '\n'
        << "sh_degree " << map.max_active_degree() << '\n' << "end_header\n";
    double rec[59];
    for (const Gaussian3D& g : map.gaussians()) {
        gaussian_to_flat(g, rec);  // position, rotation (w,x,y,z), log_scale, opacity, sh: the v1 order
        out.write(reinterpret_cast<const char*>(rec), sizeof(rec));
        const int32_t deg = g.active_degree;
        out.write(reinterpret_cast<const char*>(&deg), sizeof(deg));
    }
    if (!out) throw std::runtime_error("save_checkpoint: write failed for " + path);
}

GaussianMap load_checkpoint(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("load_checkpoint: cannot open " + path);
    std::string line, magic;
    std::getline(in, line);
    std::istringstream head(line);
    int version = 0;
    head >> magic >> version;
    if (magic != "gsmap-checkpoint") throw std::runtime_error("load_checkpoint: not a checkpoint file: " + path);
    if (version != 1) throw std::runtime_error("load_checkpoint: unsupported version in " + path);
    size_t count = 0;
    while (std::getline(in, line) && line != "end_header") {
        std::istringstream is(line);
        std::string key;
        is >> key;
        if (key == "count") is >> count;
    }
    std::vector<Gaussian3D> gs(count);
    double rec[59];
    for (Gaussian3D& g : gs) {
        in.read(reinterpret_cast<char*>(rec), sizeof(rec));
        flat_to_gaussian(rec, g);
        int32_t deg = 0;
        in.read(reinterpret_cast<char*>(&deg), sizeof(deg));
        g.active_degree = deg;
    }
    if (!in) throw std::runtime_error("load_checkpoint: truncated file " + path);
    GaussianMap map;
    map.append(gs);
    return map;
}

// ------------------------------------------------------------------ pipeline.cpp:34-64 (one frame)
ImageD quantize_8bit(const ImageD& image) {
    ImageD out = image;
    for (size_t i = 0; i < out.size(); ++i)
        out.data[i] = std::lround(std::clamp(out.data[i], 0.0, 1.0) * 255.0) / 255.0;
    return out;
}

EvalMetrics evaluate_view(const GaussianMap& map, const Pose& pose, const CameraModel& cam, const ImageD& gt_color,
                          const ImageD* gt_depth) {
    const RenderOutput out = render(map, pose, cam);
    const ImageD q = quantize_8bit(out.color);
    EvalMetrics m;
    m.psnr = psnr(q, gt_color);
    m.ssim = ssim(q, gt_color);
    m.depth_rmse = gt_depth ? depth_rmse(out.depth, *gt_depth) : std::numeric_limits<double>::quiet_NaN();
    return m;
}

// ------------------------------------------------------------------ tests/support/brute_force.hpp
GaussianMap random_scene(std::mt19937& rng, int n, const CameraModel& cam, const Pose& pose,
                         double lo, double hi) {  // brute_force.hpp:92-117
    (void)cam;
    auto uni = [&](double a, double b) { return std::uniform_real_distribution<double>(a, b)(rng); };
    std::vector<Gaussian3D> gs(n);
    for (auto& g : gs) {
        const double z = uni(1.5, 8.0);
        // Vector3d(uni(), uni(), z): GCC evaluates constructor arguments right to left.
        const double py = uni(-0.45, 0.45) * z;
        const double px = uni(-0.45, 0.45) * z;
        const Vec3 p_cam{px, py, z};
        g.position = pose.rotate_inverse(sub(p_cam, pose.t));
        do {
            for (int i = 0; i < 4; ++i) g.rotation[i] = uni(-1.0, 1.0);
        } while (norm4(g.rotation) < 0.3);
        for (int i = 0; i < 3; ++i) g.log_scale[i] = std::log(uni(0.03, 0.3));
        g.opacity_logit = uni(lo, hi);
        g.active_degree = static_cast<int>(uni(0.0, 3.999));
        for (auto& c : g.sh) c = {0, 0, 0};
        for (int c = 0; c < 3; ++c) g.sh[0][c] = uni(-1.2, 1.2);
        for (int k = 1; k < sh_basis_count(g.active_degree); ++k)
            for (int c = 0; c < 3; ++c) g.sh[k][c] = uni(-0.1, 0.1);
    }
    GaussianMap map;
    map.append(gs);
    return map;
}

// ------------------------------------------------------------------ gradcheck.cpp
namespace {
constexpr double kStep = 1e-4, kEdgeBand = 0.01, kErrFloor = 1e-6;  // gradcheck.cpp:17-19

double rel_err(double a, double fd) {  // gradcheck.cpp:21-24
    const double denom = std::max({std::abs(a), std::abs(fd), kErrFloor});
    return std::abs(a - fd) / denom;
}
double uni(std::mt19937& rng, double lo, double hi) {
    return std::uniform_real_distribution<double>(lo, hi)(rng);
}

double check_build_covariance(std::mt19937& rng) {  // gradcheck.cpp:32-64
    Vec4 q;
    do {
        for (int i = 0; i < 4; ++i) q[i] = uni(rng, -1.0, 1.0);
    } while (norm4(q) < 0.5);
    Vec3 s;
    for (int i = 0; i < 3; ++i) s[i] = uni(rng, -2.0, 0.5);
    Mat3 w;
    for (int i = 0; i < 9; ++i) w.m[i % 3][i / 3] = uni(rng, -1.0, 1.0);  // column-major fill
    Vec4 d_q;
    Vec3 d_s;
    build_covariance_vjp(q, s, w, d_q, d_s);
    auto loss = [&](const Vec4& qq, const Vec3& ss) {  // (w.array() * C.array()).sum()
        const Mat3 c = build_covariance(qq, ss);
        double e[9];
        for (int j = 0; j < 3; ++j)
            for (int i = 0; i < 3; ++i) e[3 * j + i] = w.m[i][j] * c.m[i][j];
        return esum9_vec(e);
    };
    double worst = 0.0;
    for (int i = 0; i < 4; ++i) {
        Vec4 hi = q, lo = q;
        hi[i] += kStep;
        lo[i] -= kStep;
        worst = std::max(worst, rel_err(d_q[i], (loss(hi, s) - loss(lo, s)) / (2 * kStep)));
    }
    for (int i = 0; i < 3; ++i) {
        Vec3 hi = s, lo = s;
        hi[i] += kStep;
        lo[i] -= kStep;
        worst = std::max(worst, rel_err(d_s[i], (loss(q, hi) - loss(q, lo)) / (2 * kStep)));
    }
    return worst;
}

Gaussian2D must_project(const Gaussian3D& g, const Pose& p, const CameraModel& c) {
    auto r = project_gaussian(g, p, c);
    return r ? *r : Gaussian2D{};
}

double check_project(std::mt19937& rng) {  // gradcheck.cpp:66-117
    Gaussian3D g;
    // Pose(Quaterniond(..).normalized(), Vector3d(..)): the call's arguments are evaluated
    // right to left (g++), the translation's draws before the rotation's
    const double tz = uni(rng, -1, 1), ty = uni(rng, -1, 1), tx = uni(rng, -1, 1);
    const double qz = uni(rng, -1, 1), qy = uni(rng, -1, 1), qx = uni(rng, -1, 1),
                 qw = uni(rng, -1, 1);
    const Pose n0(qw, qx, qy, qz, {0, 0, 0});
    const Pose pose(n0.qw, n0.qx, n0.qy, n0.qz, {tx, ty, tz});
    CameraModel cam{50.0, 55.0, 31.5, 31.5, 64, 64};
    const double pz = uni(rng, 1.0, 5.0), py = uni(rng, -1, 1), px = uni(rng, -1, 1);
    g.position = pose.rotate_inverse(sub({px, py, pz}, pose.t));
    do {
        for (int i = 0; i < 4; ++i) g.rotation[i] = uni(rng, -1.0, 1.0);
    } while (norm4(g.rotation) < 0.5);
    for (int i = 0; i < 3; ++i) g.log_scale[i] = uni(rng, -3.0, -0.5);
    const double wmy = uni(rng, -1, 1), wmx = uni(rng, -1, 1);
    const Vec2 w_mean{wmx, wmy};
    Mat2 w_cov;
    for (int i = 0; i < 4; ++i) w_cov.m[i % 2][i / 2] = uni(rng, -1, 1);
    const double w_depth = uni(rng, -1, 1);
    Vec3 d_pos, d_scale;
    Vec4 d_rot;
    project_gaussian_vjp(g, pose, cam, w_mean, w_cov, w_depth, d_pos, d_rot, d_scale);
    auto loss = [&](const Gaussian3D& gg) {
        const Gaussian2D p2 = must_project(gg, pose, cam);
        // w_mean.dot(mean) + (w_cov.array() * cov2d.array()).sum() + w_depth * depth
        const double cs = esum4_vec(w_cov.m[0][0] * p2.cov2d.m[0][0], w_cov.m[1][0] * p2.cov2d.m[1][0],
                                    w_cov.m[0][1] * p2.cov2d.m[0][1], w_cov.m[1][1] * p2.cov2d.m[1][1]);
        return ((w_mean.x * p2.mean.x + w_mean.y * p2.mean.y) + cs) + w_depth * p2.depth;
    };
    double worst = 0.0;
    for (int i = 0; i < 3; ++i) {
        Gaussian3D hi = g, lo = g;
        hi.position[i] += kStep;
        lo.position[i] -= kStep;
        worst = std::max(worst, rel_err(d_pos[i], (loss(hi) - loss(lo)) / (2 * kStep)));
    }
    for (int i = 0; i < 4; ++i) {
        Gaussian3D hi = g, lo = g;
        hi.rotation[i] += kStep;
        lo.rotation[i] -= kStep;
        worst = std::max(worst, rel_err(d_rot[i], (loss(hi) - loss(lo)) / (2 * kStep)));
    }
    for (int i = 0; i < 3; ++i) {
        Gaussian3D hi = g, lo = g;
        hi.log_scale[i] += kStep;
        lo.log_scale[i] -= kStep;
        worst = std::max(worst, rel_err(d_scale[i], (loss(hi) - loss(lo)) / (2 * kStep)));
    }
    return worst;
}

double check_eval2d(std::mt19937& rng) {  // gradcheck.cpp:119-160
    Mat2 a;
    for (int i = 0; i < 4; ++i) a.m[i % 2][i / 2] = uni(rng, -2, 2);
    Mat2 cov;
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) cov.m[i][j] = a.m[i][0] * a.m[j][0] + a.m[i][1] * a.m[j][1];
    cov.m[0][0] += kCovRegularization;
    cov.m[1][1] += kCovRegularization;
    const double my = uni(rng, -5, 5), mx = uni(rng, -5, 5);
    const Vec2 mean{mx, my};
    const double sigma = std::sqrt((cov.m[0][0] + cov.m[1][1]) / 2.0);
    const double oy = uni(rng, -2, 2), ox = uni(rng, -2, 2);
    const Vec2 x{mean.x + ox * sigma, mean.y + oy * sigma};
    const double w = uni(rng, -1, 1);
    const Mat2 ci = inverse2(cov);
    const double value = eval_gaussian_2d_conic(mean, ci, x);
    Vec2 d_mean, d_x;
    Mat2 d_cov;
    eval_gaussian_2d_vjp(mean, ci, x, value, w, d_mean, d_cov, d_x);
    auto loss = [&](const Vec2& m, const Mat2& c, const Vec2& xx) {
        return w * eval_gaussian_2d_conic(m, inverse2(c), xx);
    };
    double worst = 0.0;
    for (int i = 0; i < 2; ++i) {
        Vec2 hi = mean, lo = mean;
        (i ? hi.y : hi.x) += kStep;
        (i ? lo.y : lo.x) -= kStep;
        worst = std::max(worst, rel_err(i ? d_mean.y : d_mean.x,
                                        (loss(hi, cov, x) - loss(lo, cov, x)) / (2 * kStep)));
        hi = x;
        lo = x;
        (i ? hi.y : hi.x) += kStep;
        (i ? lo.y : lo.x) -= kStep;
        worst = std::max(worst, rel_err(i ? d_x.y : d_x.x,
                                        (loss(mean, cov, hi) - loss(mean, cov, lo)) / (2 * kStep)));
    }
    for (int i = 0; i < 2; ++i)
        for (int j = i; j < 2; ++j) {
            Mat2 hi = cov, lo = cov;
            hi.m[i][j] += kStep;
            hi.m[j][i] = hi.m[i][j];
            lo.m[i][j] -= kStep;
            lo.m[j][i] = lo.m[i][j];
            const double fd = (loss(mean, hi, x) - loss(mean, lo, x)) / (2 * kStep);
            const double an = i == j ? d_cov.m[i][i] : d_cov.m[i][j] + d_cov.m[j][i];
            worst = std::max(worst, rel_err(an, fd));
        }
    return worst;
}

double check_sh(std::mt19937& rng) {  // gradcheck.cpp:162-199
    std::array<Vec3, kShCoeffCount> coeffs;
    for (auto& c : coeffs) {
        const double z = uni(rng, -1, 1), y = uni(rng, -1, 1), x = uni(rng, -1, 1);
        c = {x, y, z};
    }
    Vec3 raw;
    do {
        const double z = uni(rng, -1, 1), y = uni(rng, -1, 1), x = uni(rng, -1, 1);
        raw = {x, y, z};
    } while (norm(raw) < 0.3);
    const double wz = uni(rng, -1, 1), wy = uni(rng, -1, 1), wx = uni(rng, -1, 1);
    const Vec3 w{wx, wy, wz};
    const int degree = 3;
    auto normalize = [](const Vec3& v) { const double n = norm(v); return Vec3{v.x / n, v.y / n, v.z / n}; };
    const Vec3 dir = normalize(raw);
    std::array<Vec3, kShCoeffCount> d_coeffs;
    Vec3 d_dir;
    eval_sh_vjp(coeffs, degree, dir, w, d_coeffs, d_dir);
    const double rn = norm(raw), dd = dot(dir, d_dir);
    const Vec3 d_raw{(d_dir.x - dir.x * dd) / rn, (d_dir.y - dir.y * dd) / rn, (d_dir.z - dir.z * dd) / rn};
    auto loss = [&](const std::array<Vec3, kShCoeffCount>& cc, const Vec3& rr) {
        return dot(w, eval_sh(cc, degree, normalize(rr)));
    };
    double worst = 0.0;
    for (int k = 0; k < kShCoeffCount; ++k)
        for (int c = 0; c < 3; ++c) {
            auto hi = coeffs, lo = coeffs;
            hi[k][c] += kStep;
            lo[k][c] -= kStep;
            worst = std::max(worst, rel_err(d_coeffs[k][c], (loss(hi, raw) - loss(lo, raw)) / (2 * kStep)));
        }
    for (int i = 0; i < 3; ++i) {
        Vec3 hi = raw, lo = raw;
        hi[i] += kStep;
        lo[i] -= kStep;
        worst = std::max(worst, rel_err(d_raw[i], (loss(coeffs, hi) - loss(coeffs, lo)) / (2 * kStep)));
    }
    return worst;
}

struct RenderConfig {  // gradcheck.cpp:205-211
    GaussianMap map;
    Pose pose;
    CameraModel cam;
    ImageD w_color, w_depth;
};

RenderConfig draw_render_config(std::mt19937& rng, int n_gaussians, int image_size) {  // :213-247
    RenderConfig rc;
    rc.cam = CameraModel{40.0, 42.0, (image_size - 1) / 2.0, (image_size - 1) / 2.0, image_size, image_size};
    const double tz = uni(rng, -0.5, 0.5), ty = uni(rng, -0.5, 0.5), tx = uni(rng, -0.5, 0.5);
    const double qz = uni(rng, -1, 1), qy = uni(rng, -1, 1), qx = uni(rng, -1, 1), qw = uni(rng, -1, 1);
    const Pose n0(qw, qx, qy, qz, {0, 0, 0});
    rc.pose = Pose(n0.qw, n0.qx, n0.qy, n0.qz, {tx, ty, tz});
    const int n = std::max(1, n_gaussians);
    std::vector<Gaussian3D> gs(n);
    for (auto& g : gs) {
        const double z = uni(rng, 1.5, 6.0);
        const double py = uni(rng, -0.35, 0.35) * z;
        const double px = uni(rng, -0.35, 0.35) * z;
        g.position = rc.pose.rotate_inverse(sub({px, py, z}, rc.pose.t));
        do {
            for (int i = 0; i < 4; ++i) g.rotation[i] = uni(rng, -1.0, 1.0);
        } while (norm4(g.rotation) < 0.5);
        for (int i = 0; i < 3; ++i) g.log_scale[i] = std::log(uni(rng, 0.05, 0.25));
        g.opacity_logit = uni(rng, -2.5, 1.5);
        g.active_degree = static_cast<int>(uni(rng, 0.0, 3.999));
        for (auto& c : g.sh) c = {0, 0, 0};
        for (int c = 0; c < 3; ++c) g.sh[0][c] = uni(rng, -0.7, 0.7);
        for (int k = 1; k < sh_basis_count(g.active_degree); ++k)
            for (int c = 0; c < 3; ++c) g.sh[k][c] = uni(rng, -0.04, 0.04);
    }
    rc.map.append(gs);
    rc.w_color = ImageD(image_size, image_size, 3);
    rc.w_depth = ImageD(image_size, image_size, 1);
    for (auto& v : rc.w_color.data) v = uni(rng, -1, 1);
    for (auto& v : rc.w_depth.data) v = uni(rng, -0.3, 0.3);
    return rc;
}

}  // namespace

bool config_is_smooth(const GaussianMap& map, const RenderOutput& out) {  // gradcheck.cpp:251-283
    if (out.projected.size() != map.size()) return false;
    for (const ProjectedGaussian& pg : out.projected) {
        if (pg.depth < 0.2) return false;
        const double fx_ = pg.mean.x - std::floor(pg.mean.x);
        const double fy_ = pg.mean.y - std::floor(pg.mean.y);
        if (fx_ < kEdgeBand || fx_ > 1.0 - kEdgeBand) return false;
        if (fy_ < kEdgeBand || fy_ > 1.0 - kEdgeBand) return false;
        const double half_trace = 0.5 * (pg.cov2d.m[0][0] + pg.cov2d.m[1][1]);
        const double det = det2(pg.cov2d);
        const double lmax = half_trace + std::sqrt(std::max(half_trace * half_trace - det, 0.0));
        const double r = 3.0 * std::sqrt(lmax);
        if (std::abs(r - std::round(r)) < kEdgeBand) return false;
        for (int c = 0; c < 3; ++c)
            if (pg.color_raw[c] < 0.03 || pg.color_raw[c] > 0.97) return false;
        if (pg.opacity > 0.95) return false;
    }
    const int h = out.color.h, w = out.color.w;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            double t = 1.0;
            const size_t p = size_t(y) * w + x;
            for (uint32_t i = out.contrib_offsets[p]; i < out.contrib_offsets[p + 1]; ++i) {
                t *= 1.0 - out.contribs[i].alpha;
                if (t > 2.0 * kTransmittanceMin) continue;
                if (t > 0.5 * kTransmittanceMin) return false;
                break;
            }
        }
    return true;
}

static double weighted_loss(const GaussianMap& map, const Pose& pose, const CameraModel& cam,
                            const ImageD& wc, const ImageD& wd) {  // gradcheck.cpp:285-293
    const RenderOutput out = render(map, pose, cam);
    double loss = 0.0;
    for (size_t i = 0; i < out.color.size(); ++i) loss += out.color.data[i] * wc.data[i];
    for (size_t i = 0; i < out.depth.size(); ++i) loss += out.depth.data[i] * wd.data[i];
    return loss;
}

GradCheckResult run_gradcheck(const GradCheckOptions& opts) {  // gradcheck.cpp:324-371
    GradCheckResult res;
    std::mt19937 rng(opts.seed);
    for (int i = 0; i < opts.core_configs; ++i) {
        res.max_rel_err_core = std::max(res.max_rel_err_core, check_build_covariance(rng));
        res.max_rel_err_core = std::max(res.max_rel_err_core, check_project(rng));
        res.max_rel_err_core = std::max(res.max_rel_err_core, check_eval2d(rng));
        res.max_rel_err_core = std::max(res.max_rel_err_core, check_sh(rng));
    }
    std::uniform_int_distribution<int> slot_pick(0, 4);
    for (int cfg = 0; cfg < opts.configs; ++cfg) {
        RenderConfig rc;
        RenderOutput out;
        for (;;) {
            rc = draw_render_config(rng, opts.n_gaussians, opts.image_size);
            out = render(rc.map, rc.pose, rc.cam);
            if (config_is_smooth(rc.map, out)) break;
            ++res.configs_resampled;
        }
        const RenderGradients grads = render_backward(rc.map, rc.pose, rc.cam, out, rc.w_color, rc.w_depth);
        std::uniform_int_distribution<size_t> g_pick(0, rc.map.size() - 1);
        for (int p = 0; p < opts.params_per_config; ++p) {
            const size_t gi = g_pick(rng);
            const int slot = p < 5 ? p : slot_pick(rng);
            const int idx = static_cast<int>(rng() % 14400);
            Gaussian3D& g = rc.map.gaussians()[gi];
            const GaussianGrad& gg = grads.per_gaussian[gi];
            double* target = nullptr;
            double analytic = 0.0;
            switch (slot) {  // gradcheck.cpp:296-314
                case 0: target = &g.position[idx % 3]; analytic = gg.position[idx % 3]; break;
                case 1: target = &g.rotation[idx % 4]; analytic = gg.rotation[idx % 4]; break;
                case 2: target = &g.log_scale[idx % 3]; analytic = gg.log_scale[idx % 3]; break;
                case 3: target = &g.opacity_logit; analytic = gg.opacity_logit; break;
                default: {
                    const int k = (idx / 3) % sh_basis_count(g.active_degree);
                    const int c = idx % 3;
                    target = &g.sh[k][c];
                    analytic = gg.sh[k][c];
                    break;
                }
            }
            const double saved = *target;
            *target = saved + kStep;
            const double hi = weighted_loss(rc.map, rc.pose, rc.cam, rc.w_color, rc.w_depth);
            *target = saved - kStep;
            const double lo = weighted_loss(rc.map, rc.pose, rc.cam, rc.w_color, rc.w_depth);
            *target = saved;
            const double fd = (hi - lo) / (2.0 * kStep);
            res.max_rel_err_render = std::max(res.max_rel_err_render, rel_err(analytic, fd));
        }
        ++res.configs_run;
    }
    res.passed = res.max_rel_err_core < opts.core_tolerance &&
                 res.max_rel_err_render < opts.render_tolerance;
    return res;
}

}  // namespace orc
