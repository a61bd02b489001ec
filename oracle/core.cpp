// TEST INFRASTRUCTURE ONLY — oracle restatement of proj/src/core/{covariance,projection,sh}.cpp
// and proj/include/gsmap/core/types.hpp. See oracle.hpp for the operation-order contract.
#include <algorithm>
#include <condition_variable>
#include <mutex>
#include <thread>

#include "oracle.hpp"

namespace orc {

// ------------------------------------------------------------------ types.hpp
void CameraModel::validate() const {  // core/types.hpp:22-29
    if (fx <= 0.0 || fy <= 0.0)
        throw std::invalid_argument("CameraModel: focal lengths must be positive");
    if (width <= 0 || height <= 0)
        throw std::invalid_argument("CameraModel: image size must be positive");
    if (cx < 0.0 || cx >= width || cy < 0.0 || cy >= height)
        throw std::invalid_argument("CameraModel: principal point outside image");
}

CameraModel CameraModel::scaled(int level) const {  // core/types.hpp:34-44
    CameraModel c = *this;
    const double f = static_cast<double>(1 << level);
    c.fx = fx / f;
    c.fy = fy / f;
    c.cx = (cx + 0.5) / f - 0.5;
    c.cy = (cy + 0.5) / f - 0.5;
    c.width = (width + (1 << level) - 1) >> level;
    c.height = (height + (1 << level) - 1) >> level;
    return c;
}

Pose::Pose(double w, double x, double y, double z, const Vec3& tr) : t(tr) {
    // types.hpp:53-54 rotation(q.normalized()): q / sqrt(|q|^2), the squared norm over the
    // quaternion's coefficient storage (x, y, z, w)
    const double n2 = esum4_vec(x * x, y * y, z * z, w * w);
    const double n = std::sqrt(n2);
    if (n2 > 0.0) {
        qw = w / n; qx = x / n; qy = y / n; qz = z / n;
    } else {
        qw = w; qx = x; qy = y; qz = z;
    }
}

// Eigen QuaternionBase::_transformVector: uv = q.vec x v; uv += uv; v + w*uv + q.vec x uv
static Vec3 quat_rotate(double w, double x, double y, double z, const Vec3& v) {
    const Vec3 qv{x, y, z};
    Vec3 uv = cross(qv, v);
    uv = {uv.x + uv.x, uv.y + uv.y, uv.z + uv.z};
    const Vec3 c = cross(qv, uv);
    return {(v.x + w * uv.x) + c.x, (v.y + w * uv.y) + c.y, (v.z + w * uv.z) + c.z};
}

Vec3 Pose::rotate(const Vec3& v) const { return quat_rotate(qw, qx, qy, qz, v); }
Vec3 Pose::rotate_inverse(const Vec3& v) const { return quat_rotate(qw, -qx, -qy, -qz, v); }

Mat3 Pose::rotation_matrix() const {  // Eigen QuaternionBase::toRotationMatrix
    const double tx = 2.0 * qx, ty = 2.0 * qy, tz = 2.0 * qz;
    const double twx = tx * qw, twy = ty * qw, twz = tz * qw;
    const double txx = tx * qx, txy = ty * qx, txz = tz * qx;
    const double tyy = ty * qy, tyz = tz * qy, tzz = tz * qz;
    Mat3 r;
    r.m[0][0] = 1.0 - (tyy + tzz);
    r.m[0][1] = txy - twz;
    r.m[0][2] = txz + twy;
    r.m[1][0] = txy + twz;
    r.m[1][1] = 1.0 - (txx + tzz);
    r.m[1][2] = tyz - twx;
    r.m[2][0] = txz - twy;
    r.m[2][1] = tyz + twx;
    r.m[2][2] = 1.0 - (txx + tyy);
    return r;
}

// ------------------------------------------------------------------ covariance.cpp
Mat3 rotation_from_unit(const Vec4& u) {  // covariance.cpp:7-14
    const double w = u[0], x = u[1], y = u[2], z = u[3];
    Mat3 r;
    r.m[0][0] = 1 - 2 * (y * y + z * z);
    r.m[0][1] = 2 * (x * y - w * z);
    r.m[0][2] = 2 * (x * z + w * y);
    r.m[1][0] = 2 * (x * y + w * z);
    r.m[1][1] = 1 - 2 * (x * x + z * z);
    r.m[1][2] = 2 * (y * z - w * x);
    r.m[2][0] = 2 * (x * z - w * y);
    r.m[2][1] = 2 * (y * z + w * x);
    r.m[2][2] = 1 - 2 * (x * x + y * y);
    return r;
}

static Mat3 rotation_partial(const Vec4& u, int k) {  // covariance.cpp:17-43
    const double w = u[0], x = u[1], y = u[2], z = u[3];
    double d[3][3];
    switch (k) {
        case 0: { double t[3][3] = {{0, -z, y}, {z, 0, -x}, {-y, x, 0}}; std::copy(&t[0][0], &t[0][0] + 9, &d[0][0]); break; }
        case 1: { double t[3][3] = {{0, y, z}, {y, -2 * x, -w}, {z, w, -2 * x}}; std::copy(&t[0][0], &t[0][0] + 9, &d[0][0]); break; }
        case 2: { double t[3][3] = {{-2 * y, x, w}, {x, 0, z}, {-w, z, -2 * y}}; std::copy(&t[0][0], &t[0][0] + 9, &d[0][0]); break; }
        default: { double t[3][3] = {{-2 * z, -w, x}, {w, -2 * z, y}, {x, y, 0}}; std::copy(&t[0][0], &t[0][0] + 9, &d[0][0]); break; }
    }
    Mat3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.m[i][j] = 2.0 * d[i][j];
    return r;
}

double norm4(const Vec4& q) {  // Vector4d::norm
    return std::sqrt(esum4_vec(q[0] * q[0], q[1] * q[1], q[2] * q[2], q[3] * q[3]));
}

Vec4 normalized4(const Vec4& q) {  // Eigen normalized(): n / sqrt(squaredNorm) if > 0
    const double n2 = esum4_vec(q[0] * q[0], q[1] * q[1], q[2] * q[2], q[3] * q[3]);
    if (!(n2 > 0.0)) return q;
    const double n = std::sqrt(n2);
    Vec4 u;
    for (int i = 0; i < 4; ++i) u[i] = q[i] / n;
    return u;
}

Mat3 quat_to_rotation(const Vec4& q) { return rotation_from_unit(normalized4(q)); }  // :47-49

Mat3 build_covariance(const Vec4& q, const Vec3& ls) {  // covariance.cpp:51-56
    const Mat3 r = quat_to_rotation(q);
    const double s2[3] = {std::exp(2.0 * ls.x), std::exp(2.0 * ls.y), std::exp(2.0 * ls.z)};
    Mat3 rd, sigma, out;
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) rd.m[i][k] = r.m[i][k] * s2[k];
    for (int j = 0; j < 3; ++j) {  // (R D) R^T: rows 0-1 sequential, row 2 halving (Eigen)
        for (int i = 0; i < 2; ++i)
            sigma.m[i][j] = (rd.m[i][0] * r.m[j][0] + rd.m[i][1] * r.m[j][1]) + rd.m[i][2] * r.m[j][2];
        sigma.m[2][j] = rd.m[2][0] * r.m[j][0] + (rd.m[2][1] * r.m[j][1] + rd.m[2][2] * r.m[j][2]);
    }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) out.m[i][j] = 0.5 * (sigma.m[i][j] + sigma.m[j][i]);
    return out;
}

// A^T B (lhs a transpose: every coefficient is a contiguous redux, 3 terms sequential)
static Mat3 mul33_tn(const Mat3& a, const Mat3& b) {
    Mat3 c;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            c.m[i][j] = (a.m[0][i] * b.m[0][j] + a.m[1][i] * b.m[1][j]) + a.m[2][i] * b.m[2][j];
    return c;
}
// A B of plain matrices: rows 0-1 sequential (packets), row 2 halving (Eigen)
static Mat3 mul33(const Mat3& a, const Mat3& b) {
    Mat3 c;
    for (int j = 0; j < 3; ++j) {
        for (int i = 0; i < 2; ++i)
            c.m[i][j] = (a.m[i][0] * b.m[0][j] + a.m[i][1] * b.m[1][j]) + a.m[i][2] * b.m[2][j];
        c.m[2][j] = a.m[2][0] * b.m[0][j] + (a.m[2][1] * b.m[1][j] + a.m[2][2] * b.m[2][j]);
    }
    return c;
}
static Mat3 transpose3(const Mat3& a) {
    Mat3 t;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) t.m[i][j] = a.m[j][i];
    return t;
}

void build_covariance_vjp(const Vec4& q, const Vec3& ls, const Mat3& d_sigma, Vec4& d_q,
                          Vec3& d_ls) {  // covariance.cpp:58-79
    const double nrm = norm4(q);
    Vec4 u;
    for (int i = 0; i < 4; ++i) u[i] = q[i] / nrm;
    const Mat3 r = rotation_from_unit(u);
    const double s2[3] = {std::exp(2.0 * ls.x), std::exp(2.0 * ls.y), std::exp(2.0 * ls.z)};
    Mat3 g_sym;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) g_sym.m[i][j] = d_sigma.m[i][j] + d_sigma.m[j][i];
    const Mat3 rtgr = mul33(mul33_tn(r, d_sigma), r);
    for (int k = 0; k < 3; ++k) d_ls[k] = 2.0 * s2[k] * rtgr.m[k][k];
    Mat3 d_r = mul33(g_sym, r);
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) d_r.m[i][k] *= s2[k];
    Vec4 d_u;
    for (int k = 0; k < 4; ++k) {
        const Mat3 p = rotation_partial(u, k);
        double e[9];  // (d_r.array() * P.array()).sum(): column-major storage, packet tree
        for (int j = 0; j < 3; ++j)
            for (int i = 0; i < 3; ++i) e[3 * j + i] = d_r.m[i][j] * p.m[i][j];
        d_u[k] = esum9_vec(e);
    }
    const double ud = esum4_vec(u[0] * d_u[0], u[1] * d_u[1], u[2] * d_u[2], u[3] * d_u[3]);
    for (int k = 0; k < 4; ++k) d_q[k] = (d_u[k] - u[k] * ud) / nrm;
}

// ------------------------------------------------------------------ projection.cpp
Mat23 perspective_jacobian(const Vec3& p, const CameraModel& cam) {  // projection.cpp:9-15
    const double z = p.z;
    Mat23 j;
    j.m[0][0] = cam.fx / z; j.m[0][1] = 0.0; j.m[0][2] = -cam.fx * p.x / (z * z);
    j.m[1][0] = 0.0; j.m[1][1] = cam.fy / z; j.m[1][2] = -cam.fy * p.y / (z * z);
    return j;
}

double det2(const Mat2& m) { return m.m[0][0] * m.m[1][1] - m.m[1][0] * m.m[0][1]; }

Mat2 inverse2(const Mat2& m) {  // Eigen compute_inverse<2x2>: adj * (1/det)
    const double invdet = 1.0 / det2(m);
    Mat2 r;
    r.m[0][0] = m.m[1][1] * invdet;
    r.m[1][0] = -m.m[1][0] * invdet;
    r.m[0][1] = -m.m[0][1] * invdet;
    r.m[1][1] = m.m[0][0] * invdet;
    return r;
}

static Mat23 mul23_33(const Mat23& a, const Mat3& b) {
    Mat23 c;
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j)
            c.m[i][j] = (a.m[i][0] * b.m[0][j] + a.m[i][1] * b.m[1][j]) + a.m[i][2] * b.m[2][j];
    return c;
}

std::optional<Gaussian2D> project_gaussian(const Gaussian3D& g, const Pose& pose,
                                           const CameraModel& cam) {  // projection.cpp:17-40
    const Vec3 p = pose.world_to_camera(g.position);
    if (p.z <= kNearClip) return std::nullopt;
    Gaussian2D out;
    out.mean = {cam.fx * p.x / p.z + cam.cx, cam.fy * p.y / p.z + cam.cy};
    out.depth = p.z;
    const Mat3 w = pose.rotation_matrix();
    const Mat23 m = mul23_33(perspective_jacobian(p, cam), w);
    const Mat3 sw = build_covariance(g.rotation, g.log_scale);
    const Mat23 ms = mul23_33(m, sw);
    Mat2 cov;
    for (int i = 0; i < 2; ++i)
        for (int k = 0; k < 2; ++k)
            cov.m[i][k] = (ms.m[i][0] * m.m[k][0] + ms.m[i][1] * m.m[k][1]) + ms.m[i][2] * m.m[k][2];
    cov.m[0][0] += kCovRegularization;
    cov.m[1][1] += kCovRegularization;
    for (int i = 0; i < 2; ++i)
        for (int k = 0; k < 2; ++k) out.cov2d.m[i][k] = 0.5 * (cov.m[i][k] + cov.m[k][i]);
    const double half_trace = 0.5 * (out.cov2d.m[0][0] + out.cov2d.m[1][1]);
    const double det = det2(out.cov2d);
    const double disc = std::sqrt(std::max(half_trace * half_trace - det, 0.0));
    const double lambda_max = half_trace + disc;
    out.radius = std::max(1, static_cast<int>(std::ceil(3.0 * std::sqrt(lambda_max))));
    return out;
}

void project_gaussian_vjp(const Gaussian3D& g, const Pose& pose, const CameraModel& cam,
                          const Vec2& d_mean, const Mat2& d_cov, double d_depth, Vec3& d_position,
                          Vec4& d_rotation, Vec3& d_log_scale) {  // projection.cpp:42-74
    const Vec3 p = pose.world_to_camera(g.position);
    const Mat3 w = pose.rotation_matrix();
    const Mat23 j = perspective_jacobian(p, cam);
    const Mat23 m = mul23_33(j, w);
    const Mat3 sw = build_covariance(g.rotation, g.log_scale);
    // d_sigma_w = m^T d_cov m
    double mtd[3][2];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 2; ++b) mtd[a][b] = m.m[0][a] * d_cov.m[0][b] + m.m[1][a] * d_cov.m[1][b];
    Mat3 dsw;
    for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 3; ++c) dsw.m[a][c] = mtd[a][0] * m.m[0][c] + mtd[a][1] * m.m[1][c];
    // d_m = (d_cov + d_cov^T) m sigma_w
    Mat2 ds;
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) ds.m[a][b] = d_cov.m[a][b] + d_cov.m[b][a];
    Mat23 dsm;
    for (int a = 0; a < 2; ++a)
        for (int c = 0; c < 3; ++c) dsm.m[a][c] = ds.m[a][0] * m.m[0][c] + ds.m[a][1] * m.m[1][c];
    const Mat23 dm = mul23_33(dsm, sw);
    const Mat23 dj = mul23_33(dm, transpose3(w));
    build_covariance_vjp(g.rotation, g.log_scale, dsw, d_rotation, d_log_scale);
    Vec3 dp;
    for (int c = 0; c < 3; ++c) dp[c] = j.m[0][c] * d_mean.x + j.m[1][c] * d_mean.y;
    const double z = p.z, z2 = z * z, z3 = z2 * z;
    dp.x += dj.m[0][2] * (-cam.fx / z2);
    dp.y += dj.m[1][2] * (-cam.fy / z2);
    dp.z += dj.m[0][0] * (-cam.fx / z2) + dj.m[1][1] * (-cam.fy / z2) +
            dj.m[0][2] * (2.0 * cam.fx * p.x / z3) + dj.m[1][2] * (2.0 * cam.fy * p.y / z3);
    dp.z += d_depth;
    for (int c = 0; c < 3; ++c)
        d_position[c] = (w.m[0][c] * dp.x + w.m[1][c] * dp.y) + w.m[2][c] * dp.z;
}

double eval_gaussian_2d_conic(const Vec2& mean, const Mat2& ci, const Vec2& x) {  // :80-84
    const double dx = x.x - mean.x, dy = x.y - mean.y;
    const double u0 = ci.m[0][0] * dx + ci.m[0][1] * dy;
    const double u1 = ci.m[1][0] * dx + ci.m[1][1] * dy;
    return std::exp(-0.5 * (dx * u0 + dy * u1));
}

void eval_gaussian_2d_vjp(const Vec2& mean, const Mat2& ci, const Vec2& x, double value,
                          double d_value, Vec2& d_mean, Mat2& d_cov, Vec2& d_x) {  // :86-96
    const double dx = x.x - mean.x, dy = x.y - mean.y;
    const double u0 = ci.m[0][0] * dx + ci.m[0][1] * dy;
    const double u1 = ci.m[1][0] * dx + ci.m[1][1] * dy;
    const double s = value * d_value;
    d_mean = {s * u0, s * u1};
    d_x = {-s * u0, -s * u1};
    const double hs = 0.5 * s;
    d_cov.m[0][0] = hs * u0 * u0;
    d_cov.m[0][1] = hs * u0 * u1;
    d_cov.m[1][0] = hs * u1 * u0;
    d_cov.m[1][1] = hs * u1 * u1;
}

// ------------------------------------------------------------------ sh.cpp
namespace {
constexpr double kC0 = 0.28209479177387814;
constexpr double kC1 = 0.4886025119029199;
constexpr double kC2[5] = {1.0925484305920792, 1.0925484305920792, 0.31539156525252005,
                           1.0925484305920792, 0.5462742152960396};
constexpr double kC3[7] = {0.5900435899266435, 2.890611442640554, 0.4570457994644658,
                           0.3731763325901154, 0.4570457994644658, 1.445305721320277,
                           0.5900435899266435};
}  // namespace

void sh_basis(const Vec3& d, int degree, std::array<double, kShCoeffCount>& out) {  // sh.cpp:30-53
    const double x = d.x, y = d.y, z = d.z;
    out.fill(0.0);
    out[0] = kC0;
    if (degree < 1) return;
    out[1] = kC1 * y;
    out[2] = kC1 * z;
    out[3] = kC1 * x;
    if (degree < 2) return;
    const double xx = x * x, yy = y * y, zz = z * z;
    out[4] = kC2[0] * x * y;
    out[5] = kC2[1] * y * z;
    out[6] = kC2[2] * (2.0 * zz - xx - yy);
    out[7] = kC2[3] * x * z;
    out[8] = kC2[4] * (xx - yy);
    if (degree < 3) return;
    out[9] = kC3[0] * y * (3.0 * xx - yy);
    out[10] = kC3[1] * x * y * z;
    out[11] = kC3[2] * y * (4.0 * zz - xx - yy);
    out[12] = kC3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    out[13] = kC3[4] * x * (4.0 * zz - xx - yy);
    out[14] = kC3[5] * z * (xx - yy);
    out[15] = kC3[6] * x * (xx - 3.0 * yy);
}

void sh_basis_jacobian(const Vec3& d, int degree, std::array<double, kShCoeffCount>& basis,
                       std::array<Vec3, kShCoeffCount>& jac) {  // sh.cpp:55-80
    sh_basis(d, degree, basis);
    const double x = d.x, y = d.y, z = d.z;
    for (auto& j : jac) j = {0, 0, 0};
    if (degree < 1) return;
    jac[1] = {0, kC1, 0};
    jac[2] = {0, 0, kC1};
    jac[3] = {kC1, 0, 0};
    if (degree < 2) return;
    jac[4] = scale({y, x, 0}, kC2[0]);
    jac[5] = scale({0, z, y}, kC2[1]);
    jac[6] = scale({-2.0 * x, -2.0 * y, 4.0 * z}, kC2[2]);
    jac[7] = scale({z, 0, x}, kC2[3]);
    jac[8] = scale({2.0 * x, -2.0 * y, 0}, kC2[4]);
    if (degree < 3) return;
    const double xx = x * x, yy = y * y, zz = z * z;
    jac[9] = scale({6.0 * x * y, 3.0 * xx - 3.0 * yy, 0}, kC3[0]);
    jac[10] = scale({y * z, x * z, x * y}, kC3[1]);
    jac[11] = scale({-2.0 * x * y, 4.0 * zz - xx - 3.0 * yy, 8.0 * y * z}, kC3[2]);
    jac[12] = scale({-6.0 * x * z, -6.0 * y * z, 6.0 * zz - 3.0 * xx - 3.0 * yy}, kC3[3]);
    jac[13] = scale({4.0 * zz - 3.0 * xx - yy, -2.0 * x * y, 8.0 * x * z}, kC3[4]);
    jac[14] = scale({2.0 * x * z, -2.0 * y * z, xx - yy}, kC3[5]);
    jac[15] = scale({3.0 * xx - 3.0 * yy, -6.0 * x * y, 0}, kC3[6]);
}

Vec3 eval_sh(const std::array<Vec3, kShCoeffCount>& coeffs, int degree, const Vec3& dir) {
    // sh.cpp:82-92
    if (degree < 0 || degree > kShMaxDegree)
        throw std::invalid_argument("eval_sh: active_degree out of range");
    std::array<double, kShCoeffCount> basis;
    sh_basis(dir, degree, basis);
    Vec3 c{0.5, 0.5, 0.5};
    const int n = sh_basis_count(degree);
    for (int i = 0; i < n; ++i) c = add(c, scale(coeffs[i], basis[i]));
    return c;
}

void eval_sh_vjp(const std::array<Vec3, kShCoeffCount>& coeffs, int degree, const Vec3& dir,
                 const Vec3& d_color, std::array<Vec3, kShCoeffCount>& d_coeffs,
                 Vec3& d_dir) {  // sh.cpp:94-109
    std::array<double, kShCoeffCount> basis;
    std::array<Vec3, kShCoeffCount> jac;
    sh_basis_jacobian(dir, degree, basis, jac);
    for (auto& c : d_coeffs) c = {0, 0, 0};
    d_dir = {0, 0, 0};
    const int n = sh_basis_count(degree);
    for (int i = 0; i < n; ++i) {
        d_coeffs[i] = scale(d_color, basis[i]);
        d_dir = add(d_dir, scale(jac[i], dot(coeffs[i], d_color)));
    }
}

// ------------------------------------------------------------------ gaussian.hpp helpers
void GaussianGrad::add(const GaussianGrad& o) {  // gaussian.hpp:51-57
    position = orc::add(position, o.position);
    for (int i = 0; i < 4; ++i) rotation[i] += o.rotation[i];
    log_scale = orc::add(log_scale, o.log_scale);
    opacity_logit += o.opacity_logit;
    for (int i = 0; i < kShCoeffCount; ++i) sh[i] = orc::add(sh[i], o.sh[i]);
}

void gaussian_to_flat(const Gaussian3D& g, double* o) {
    o[0] = g.position.x; o[1] = g.position.y; o[2] = g.position.z;
    for (int i = 0; i < 4; ++i) o[3 + i] = g.rotation[i];
    o[7] = g.log_scale.x; o[8] = g.log_scale.y; o[9] = g.log_scale.z;
    o[10] = g.opacity_logit;
    for (int k = 0; k < 16; ++k)
        for (int c = 0; c < 3; ++c) o[11 + 3 * k + c] = g.sh[k][c];
}

void flat_to_gaussian(const double* o, Gaussian3D& g) {
    g.position = {o[0], o[1], o[2]};
    for (int i = 0; i < 4; ++i) g.rotation[i] = o[3 + i];
    g.log_scale = {o[7], o[8], o[9]};
    g.opacity_logit = o[10];
    for (int k = 0; k < 16; ++k)
        for (int c = 0; c < 3; ++c) g.sh[k][c] = o[11 + 3 * k + c];
}

void grad_to_flat(const GaussianGrad& g, double* o) {
    o[0] = g.position.x; o[1] = g.position.y; o[2] = g.position.z;
    for (int i = 0; i < 4; ++i) o[3 + i] = g.rotation[i];
    o[7] = g.log_scale.x; o[8] = g.log_scale.y; o[9] = g.log_scale.z;
    o[10] = g.opacity_logit;
    for (int k = 0; k < 16; ++k)
        for (int c = 0; c < 3; ++c) o[11 + 3 * k + c] = g.sh[k][c];
}

// ------------------------------------------------------------------ util/thread_pool.hpp
struct ThreadPool::Impl {  // fork-join pool, static contiguous chunking (thread_pool.hpp:15-106)
    std::vector<std::thread> workers;
    std::mutex mu;
    std::condition_variable cv_start, cv_done;
    const std::function<void(int, size_t, size_t)>* job = nullptr;
    size_t job_n = 0;
    int job_used = 0, pending = 0;
    uint64_t generation = 0;
    bool stop = false;
};

static void run_chunk(int idx, const std::function<void(int, size_t, size_t)>& fn, size_t n,
                      int used) {
    const size_t chunk = (n + used - 1) / used;
    const size_t begin = std::min(n, chunk * static_cast<size_t>(idx));
    const size_t end = std::min(n, begin + chunk);
    if (begin < end) fn(idx, begin, end);
}

ThreadPool::ThreadPool(int threads) : impl_(new Impl) {
    int n = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
    n_threads_ = std::max(1, n);
    for (int i = 1; i < n_threads_; ++i) {
        impl_->workers.emplace_back([this, i] {
            uint64_t seen = 0;
            for (;;) {
                const std::function<void(int, size_t, size_t)>* job = nullptr;
                size_t n = 0;
                int used = 0;
                {
                    std::unique_lock<std::mutex> lk(impl_->mu);
                    impl_->cv_start.wait(lk, [&] { return impl_->stop || impl_->generation != seen; });
                    if (impl_->stop) return;
                    seen = impl_->generation;
                    job = impl_->job;
                    n = impl_->job_n;
                    used = impl_->job_used;
                }
                if (i < used && job) run_chunk(i, *job, n, used);
                {
                    std::lock_guard<std::mutex> lk(impl_->mu);
                    if (--impl_->pending == 0) impl_->cv_done.notify_all();
                }
            }
        });
    }
}

ThreadPool::~ThreadPool() {
    {
        std::lock_guard<std::mutex> lk(impl_->mu);
        impl_->stop = true;
    }
    impl_->cv_start.notify_all();
    for (auto& t : impl_->workers) t.join();
    delete impl_;
}

void ThreadPool::parallel_for(size_t n, const std::function<void(int, size_t, size_t)>& fn) {
    if (n == 0) return;
    const int used = static_cast<int>(std::min<size_t>(n_threads_, n));
    if (used == 1) {
        fn(0, 0, n);
        return;
    }
    {
        std::lock_guard<std::mutex> lk(impl_->mu);
        impl_->job = &fn;
        impl_->job_n = n;
        impl_->job_used = used;
        impl_->pending = n_threads_ - 1;
        ++impl_->generation;
    }
    impl_->cv_start.notify_all();
    run_chunk(0, fn, n, used);
    std::unique_lock<std::mutex> lk(impl_->mu);
    impl_->cv_done.wait(lk, [this] { return impl_->pending == 0; });
    impl_->job = nullptr;
}

}  // namespace orc
