// TEST INFRASTRUCTURE ONLY — CPU fp64 restatement of the gsmap (LVI-GS) mapping hot path.
//
// This is the parity ORACLE for the B200 product in paper_2411_02703_b200/. It restates the
// reference C++ (/root/reference/proj, CPU-only, Eigen fp64) without Eigen, function by
// function; each function cites the reference file:line it follows. Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may load it.
// The product path never links or calls it.
//
// The reference itself cannot be compiled here (Eigen3 / libpng headers and the vendored
// doctest / CLI11 are absent, no network: proj/CMakeLists.txt:10-14). Parity of this
// restatement is pinned by porting the reference's own known-answer and property tests
// (proj/tests/test_{core,rasterizer,mapper,metrics}.cpp) onto it: tests/test_oracle_*.py.
//
// Floating-point operation order: where Eigen's evaluation order decides bits we follow the
// formulas Eigen uses (Quaternion::_transformVector, toRotationMatrix, 2x2 inverse/determinant)
// and otherwise a canonical left-to-right order (k = 0, 1, 2) for small products. The
// product's FP64 preprocess kernel follows the SAME canonical order, which is what makes
// mean / depth / radius / tile keys bit-exact between the two. Built with -ffp-contract=off.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <functional>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

// ---------------------------------------------------------------- small fixed-size algebra
struct Vec2 { double x = 0, y = 0; };
struct Vec3 {
    double x = 0, y = 0, z = 0;
    double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
    double& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
};
struct Vec4 {  // raw quaternion (w, x, y, z) — reference Eigen::Vector4d indices 0..3
    double v[4] = {1, 0, 0, 0};
    double operator[](int i) const { return v[i]; }
    double& operator[](int i) { return v[i]; }
};
struct Mat2 { double m[2][2] = {{0, 0}, {0, 0}}; };
struct Mat3 { double m[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}; };
struct Mat23 { double m[2][3] = {{0, 0, 0}, {0, 0, 0}}; };

inline Vec3 add(const Vec3& a, const Vec3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline Vec3 sub(const Vec3& a, const Vec3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline Vec3 scale(const Vec3& a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline double dot(const Vec3& a, const Vec3& b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
inline double norm(const Vec3& a) { return std::sqrt(dot(a, a)); }
// Eigen cross(): (a1 b2 - a2 b1, a2 b0 - a0 b2, a0 b1 - a1 b0)
inline Vec3 cross(const Vec3& a, const Vec3& b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

// Eigen 3.4 (SSE2) evaluation orders where they decide bits; oracle/ref_eigen/Eigen/EigenSubset.h
// restates the rules and oracle/_ref (the reference compiled against it) pins them:
//   - a reduction over contiguous storage (dot, squaredNorm, sum of a plain matrix) adds packets
//     of 2 as a tree: 4 terms (e0 + e2) + (e1 + e3), 9 terms ((e0+e2)+(e4+e6) + (e1+e3)+(e5+e7)) + e8;
//   - a 3x3 * 3x3 product of plain (column-major) matrices computes rows 0-1 as the sequential
//     sum over k (packets) and row 2 as a halving tree e0 + (e1 + e2) (strided redux).
inline double esum4_vec(double e0, double e1, double e2, double e3) { return (e0 + e2) + (e1 + e3); }
inline double esum9_vec(const double* e) {
    return (((e[0] + e[2]) + (e[4] + e[6])) + ((e[1] + e[3]) + (e[5] + e[7]))) + e[8];
}

inline double sigmoid(double x) { return 1.0 / (1.0 + std::exp(-x)); }  // core/types.hpp:11
inline double logit(double p) { return std::log(p / (1.0 - p)); }         // core/types.hpp:12

// ---------------------------------------------------------------- camera / pose (core/types.hpp)
struct CameraModel {  // core/types.hpp:15-45
    double fx = 0, fy = 0, cx = 0, cy = 0;
    int width = 0, height = 0;
    void validate() const;           // types.hpp:22-29
    CameraModel scaled(int level) const;  // types.hpp:34-44
};

struct Pose {  // core/types.hpp:48-64 ; q_cw stored normalised (w, x, y, z)
    double qw = 1, qx = 0, qy = 0, qz = 0;
    Vec3 t;
    Pose() = default;
    Pose(double w, double x, double y, double z, const Vec3& tr);  // normalises like q.normalized()
    Vec3 rotate(const Vec3& v) const;          // Eigen Quaternion * Vector3 (_transformVector)
    Vec3 rotate_inverse(const Vec3& v) const;  // conjugate() * v
    Vec3 world_to_camera(const Vec3& p) const { return add(rotate(p), t); }  // types.hpp:56-58
    Vec3 camera_center() const { return rotate_inverse({-t.x, -t.y, -t.z}); }  // types.hpp:61-63
    Mat3 rotation_matrix() const;              // Eigen toRotationMatrix
};

// ---------------------------------------------------------------- Gaussians (core/gaussian.hpp)
constexpr int kShMaxDegree = 3;
constexpr int kShCoeffCount = 16;
inline constexpr int sh_basis_count(int d) { return (d + 1) * (d + 1); }

struct Gaussian3D {  // core/gaussian.hpp:16-26
    Vec3 position;
    Vec4 rotation;  // (w, x, y, z), normalised on use
    Vec3 log_scale;
    double opacity_logit = 0.0;
    std::array<Vec3, kShCoeffCount> sh{};
    int active_degree = 0;
    double opacity() const { return sigmoid(opacity_logit); }
};

struct Gaussian2D {  // core/gaussian.hpp:30-35
    Vec2 mean;
    Mat2 cov2d;
    double depth = 0.0;
    int radius = 1;
};

struct GaussianGrad {  // core/gaussian.hpp:40-58
    Vec3 position;
    Vec4 rotation{{0, 0, 0, 0}};
    Vec3 log_scale;
    double opacity_logit = 0.0;
    std::array<Vec3, kShCoeffCount> sh{};
    void add(const GaussianGrad& o);
};

// ---------------------------------------------------------------- core math (src/core/*.cpp)
constexpr double kNearClip = 0.01;          // core/projection.hpp:11
constexpr double kCovRegularization = 0.3;  // core/projection.hpp:12

Mat3 rotation_from_unit(const Vec4& u);
Mat3 quat_to_rotation(const Vec4& q);
Vec4 normalized4(const Vec4& q);
double norm4(const Vec4& q);
Mat3 build_covariance(const Vec4& q, const Vec3& log_scale);
void build_covariance_vjp(const Vec4& q, const Vec3& log_scale, const Mat3& d_sigma, Vec4& d_q,
                          Vec3& d_log_scale);
Mat23 perspective_jacobian(const Vec3& p, const CameraModel& cam);
std::optional<Gaussian2D> project_gaussian(const Gaussian3D& g, const Pose& pose,
                                           const CameraModel& cam);
void project_gaussian_vjp(const Gaussian3D& g, const Pose& pose, const CameraModel& cam,
                          const Vec2& d_mean, const Mat2& d_cov2d, double d_depth, Vec3& d_position,
                          Vec4& d_rotation, Vec3& d_log_scale);
Mat2 inverse2(const Mat2& m);
double det2(const Mat2& m);
double eval_gaussian_2d_conic(const Vec2& mean, const Mat2& cov_inv, const Vec2& x);
void eval_gaussian_2d_vjp(const Vec2& mean, const Mat2& cov_inv, const Vec2& x, double value,
                          double d_value, Vec2& d_mean, Mat2& d_cov2d, Vec2& d_x);
void sh_basis(const Vec3& dir, int degree, std::array<double, kShCoeffCount>& out);
void sh_basis_jacobian(const Vec3& dir, int degree, std::array<double, kShCoeffCount>& basis,
                       std::array<Vec3, kShCoeffCount>& jac);
Vec3 eval_sh(const std::array<Vec3, kShCoeffCount>& coeffs, int degree, const Vec3& dir);
void eval_sh_vjp(const std::array<Vec3, kShCoeffCount>& coeffs, int degree, const Vec3& dir,
                 const Vec3& d_color, std::array<Vec3, kShCoeffCount>& d_coeffs, Vec3& d_dir);

// ---------------------------------------------------------------- util (util/thread_pool.hpp)
class ThreadPool {  // util/thread_pool.hpp:15-106 (restated with the same static partition)
public:
    explicit ThreadPool(int threads = 0);
    ~ThreadPool();
    ThreadPool(const ThreadPool&) = delete;
    ThreadPool& operator=(const ThreadPool&) = delete;
    int thread_count() const { return n_threads_; }
    void parallel_for(size_t n, const std::function<void(int, size_t, size_t)>& fn);

private:
    struct Impl;
    Impl* impl_;
    int n_threads_;
};

// ---------------------------------------------------------------- image (io/image.hpp)
struct ImageD {  // row-major HWC doubles, io/image.hpp:15-51
    int h = 0, w = 0, c = 0;
    std::vector<double> data;
    ImageD() = default;
    ImageD(int hh, int ww, int cc, double fill = 0.0)
        : h(hh), w(ww), c(cc), data(size_t(hh) * ww * cc, fill) {}
    double& at(int y, int x, int ch = 0) { return data[(size_t(y) * w + x) * c + ch]; }
    double at(int y, int x, int ch = 0) const { return data[(size_t(y) * w + x) * c + ch]; }
    size_t size() const { return data.size(); }
    bool same_shape(const ImageD& o) const { return h == o.h && w == o.w && c == o.c; }
};

// ---------------------------------------------------------------- map + Adam (map/gaussian_map.*)
struct AdamState {  // map/gaussian_map.hpp:13-30, flattened as 59 m + 59 v
    std::array<double, 59> m{};
    std::array<double, 59> v{};
    int64_t step = 0;
};

struct LearningRates {  // map/gaussian_map.hpp:34-40
    double position = 1.6e-4, rotation = 1e-3, log_scale = 5e-3, opacity = 5e-2, sh = 2.5e-3;
};

struct RenderGradients { std::vector<GaussianGrad> per_gaussian; };

class GaussianMap {  // map/gaussian_map.hpp:44-96
public:
    size_t size() const { return gaussians_.size(); }
    bool empty() const { return gaussians_.empty(); }
    const std::vector<Gaussian3D>& gaussians() const { return gaussians_; }
    std::vector<Gaussian3D>& gaussians() { return gaussians_; }
    const std::vector<AdamState>& optimizer_state() const { return opt_; }
    std::vector<AdamState>& optimizer_state() { return opt_; }
    int64_t global_step() const { return global_step_; }
    void set_global_step(int64_t s) { global_step_ = s; }
    double scene_extent() const { return scene_extent_; }
    void set_scene_extent(double e) { scene_extent_ = e; }
    void append(const std::vector<Gaussian3D>& gs);
    void apply_gradients(const RenderGradients& grads, const LearningRates& lr);
    size_t prune(double threshold);
    void raise_sh_degree(int degree);
    int max_active_degree() const;

private:
    void refresh_extent();
    std::vector<Gaussian3D> gaussians_;
    std::vector<AdamState> opt_;
    int64_t global_step_ = 0;
    double scene_extent_ = 1.0;
};

// Gaussian <-> flat 59-scalar view (position 3, rotation 4, log_scale 3, opacity 1, sh 48)
void gaussian_to_flat(const Gaussian3D& g, double* out59);
void flat_to_gaussian(const double* in59, Gaussian3D& g);
void grad_to_flat(const GaussianGrad& g, double* out59);

// ---------------------------------------------------------------- rasterizer (render/rasterizer.*)
constexpr int kTileSize = 16;              // rasterizer.hpp:17
constexpr double kAlphaMax = 0.99;         // rasterizer.hpp:18
constexpr double kTransmittanceMin = 1e-4; // rasterizer.hpp:19

struct Contribution { int32_t gaussian = 0; double alpha = 0.0; };  // rasterizer.hpp:22-25

struct ProjectedGaussian {  // rasterizer.hpp:28-40
    int32_t index = 0;
    Vec2 mean;
    Mat2 cov2d, cov_inv;
    double depth = 0.0;
    int radius = 1;
    double opacity = 0.0;
    Vec3 color, color_raw, view_dir;
    double view_dist = 0.0;
};

struct RenderOutput {  // rasterizer.hpp:43-59
    ImageD color, depth, visibility;
    std::vector<uint32_t> contrib_offsets;
    std::vector<Contribution> contribs;
    std::vector<ProjectedGaussian> projected;
    // Oracle extra (for bit-exact key parity): the per-tile bins exactly as bin_tiles built them
    // (each entry = rank into `projected`), rasterizer.cpp:76-91.
    std::vector<std::vector<int32_t>> bins;
    int tiles_x = 0, tiles_y = 0;
};

RenderOutput render(const GaussianMap& map, const Pose& pose, const CameraModel& cam,
                    ThreadPool* pool = nullptr);
RenderGradients render_backward(const GaussianMap& map, const Pose& pose, const CameraModel& cam,
                                const RenderOutput& out, const ImageD& dl_dcolor,
                                const ImageD& dl_ddepth, ThreadPool* pool = nullptr);

struct BruteForceOutput { ImageD color, depth, visibility; };
BruteForceOutput brute_force_render(const GaussianMap& map, const Pose& pose,
                                    const CameraModel& cam);  // tests/support/brute_force.hpp:26-89

// ---------------------------------------------------------------- metrics (metrics/metrics.cpp)
double psnr(const ImageD& a, const ImageD& b);
double ssim(const ImageD& a, const ImageD& b);
double ssim_with_gradient(const ImageD& a, const ImageD& b, ImageD& d_ssim_da);
double depth_rmse(const ImageD& rendered, const ImageD& gt, bool* empty_mask = nullptr);

// ---------------------------------------------------------------- trainer (map/mapper.*)
constexpr double kDepthLossMinVisibility = 0.98;  // mapper.hpp:15

struct TrainConfig {  // mapper.hpp:17-30
    double lambda = 0.2, lambda_d = 0.5;
    int pyramid_levels = 2, iters_per_level = 0;
    LearningRates lr;
    double prune_threshold = 0.005;
    int sh_interval = 300;
    int effective_iters_per_level(int budget) const {
        if (iters_per_level > 0) return iters_per_level;
        return std::max(1, budget / (pyramid_levels + 1));
    }
};

struct PyramidLevel { ImageD color, depth; };  // keyframe.hpp:18-21
struct Keyframe {                              // keyframe.hpp:23-34 (hot-path fields)
    Pose pose;
    ImageD color_image, sparse_depth;
    int initial_iters = 0, remaining_iters = 0, consumed_iters = 0;
    std::vector<PyramidLevel> pyramid;
};

struct ColoredPoint { Vec3 position, color; double timestamp = 0.0; };

struct LossResult {  // mapper.hpp:52-60
    double total = 0, color_loss = 0, depth_loss = 0, l1 = 0, ssim = 0;
    ImageD dl_dcolor, dl_ddepth;
};
struct StepReport { int level = 0; double loss = 0, psnr = 0; };

std::vector<ImageD> build_pyramid(const ImageD& image, int levels);
std::vector<ImageD> build_depth_pyramid(const ImageD& depth, int levels);
void build_keyframe_pyramid(Keyframe& kf, int levels);
LossResult compute_loss(const RenderOutput& rendered, const Keyframe& kf, int level,
                        const TrainConfig& cfg);
std::optional<StepReport> train_keyframe_step(GaussianMap& map, Keyframe& kf,
                                              const TrainConfig& cfg, const CameraModel& cam,
                                              ThreadPool* pool = nullptr);
int maybe_upgrade_sh(GaussianMap& map, const TrainConfig& cfg);
size_t init_gaussians_from_points(GaussianMap& map, const std::vector<ColoredPoint>& points);
ImageD project_sparse_depth(const std::vector<ColoredPoint>& points, const Pose& pose,
                            const CameraModel& cam);  // io/sequence.cpp:246-259
void save_checkpoint(const std::string& path, const GaussianMap& map);  // io/checkpoint.cpp:17-35
GaussianMap load_checkpoint(const std::string& path);                   // io/checkpoint.cpp:37-71
ImageD quantize_8bit(const ImageD& image);                              // pipeline.cpp:34-39
struct EvalMetrics {
    double psnr = 0.0, ssim = 0.0, depth_rmse = 0.0;
};
EvalMetrics evaluate_view(const GaussianMap& map, const Pose& pose, const CameraModel& cam, const ImageD& gt_color,
                          const ImageD* gt_depth);  // pipeline.cpp:46-60, one frame
std::vector<size_t> filter_points_by_visibility(const std::vector<ColoredPoint>& points, const Pose& pose,
                                                const GaussianMap& map, const CameraModel& cam,
                                                double tau_alpha);  // keyframe.cpp:49-74

// ---------------------------------------------------------------- fixtures
GaussianMap random_scene(std::mt19937& rng, int n, const CameraModel& cam, const Pose& pose,
                         double lo = -2.5, double hi = 1.5);  // tests/support/brute_force.hpp:92-117

struct GradCheckOptions {  // pipeline/gradcheck.hpp:8-19
    uint32_t seed = 1;
    int n_gaussians = 20, configs = 1000, core_configs = 1000, image_size = 32,
        params_per_config = 8;
    double core_tolerance = 1e-4, render_tolerance = 1e-3;
};
struct GradCheckResult {
    bool passed = false;
    double max_rel_err_core = 0, max_rel_err_render = 0;
    int configs_run = 0, configs_resampled = 0;
};
GradCheckResult run_gradcheck(const GradCheckOptions& opts);  // pipeline/gradcheck.cpp:324-371
bool config_is_smooth(const GaussianMap& map, const RenderOutput& out);  // gradcheck.cpp:251-283

}  // namespace orc
