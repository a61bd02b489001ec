// K1 preprocess_fwd and K8 preprocess_bwd: per-Gaussian FP64 geometry.
//
// This translation unit is compiled with --fmad=false. The fp64 operation sequence for the
// camera transform, mean, depth, 2D covariance and radius follows the reference's order under
// Eigen 3.4 (proj/src/core/projection.cpp:17-40, covariance.cpp:51-56; the oracle restates it and
// oracle/_ref — the reference itself — pins it bitwise), so mean / depth / radius / pixel
// rect / tile keys come out bit-identical to the fp64 reference on the same inputs. Only the
// data the blend needs at fp32 (conic, opacity, colour, depth) is rounded after the fact.
#include "common.cuh"
#include "kernels.cuh"

namespace gsb {

namespace {

struct D3 { double x, y, z; };

__device__ __forceinline__ D3 cross3(const D3& a, const D3& b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

// Eigen QuaternionBase::_transformVector (uv = q.vec x v; uv += uv; v + w uv + q.vec x uv)
__device__ __forceinline__ D3 quat_rotate(double w, double x, double y, double z, const D3& v) {
    const D3 qv{x, y, z};
    D3 uv = cross3(qv, v);
    uv = {uv.x + uv.x, uv.y + uv.y, uv.z + uv.z};
    const D3 c = cross3(qv, uv);
    return {(v.x + w * uv.x) + c.x, (v.y + w * uv.y) + c.y, (v.z + w * uv.z) + c.z};
}

// Eigen QuaternionBase::toRotationMatrix
__device__ __forceinline__ void pose_matrix(const ViewParams& v, double W[3][3]) {
    const double tx = 2.0 * v.qx, ty = 2.0 * v.qy, tz = 2.0 * v.qz;
    const double twx = tx * v.qw, twy = ty * v.qw, twz = tz * v.qw;
    const double txx = tx * v.qx, txy = ty * v.qx, txz = tz * v.qx;
    const double tyy = ty * v.qy, tyz = tz * v.qy, tzz = tz * v.qz;
    W[0][0] = 1.0 - (tyy + tzz); W[0][1] = txy - twz; W[0][2] = txz + twy;
    W[1][0] = txy + twz; W[1][1] = 1.0 - (txx + tzz); W[1][2] = tyz - twx;
    W[2][0] = txz - twy; W[2][1] = tyz + twx; W[2][2] = 1.0 - (txx + tyy);
}

// covariance.cpp:7-14 on the normalised quaternion (Eigen normalized(): q / sqrt(|q|^2), the
// squared norm of a Vector4d summed as packets: (q0^2 + q2^2) + (q1^2 + q3^2), see
// oracle/ref_eigen/Eigen/EigenSubset.h)
__device__ __forceinline__ void unit_quat(const double q[4], double u[4], double* nrm) {
    const double n2 = (q[0] * q[0] + q[2] * q[2]) + (q[1] * q[1] + q[3] * q[3]);
    const double n = sqrt(n2);
    *nrm = n;
    if (n2 > 0.0) {
        for (int i = 0; i < 4; ++i) u[i] = q[i] / n;
    } else {
        for (int i = 0; i < 4; ++i) u[i] = q[i];
    }
}

__device__ __forceinline__ void rotation_from_unit(const double u[4], double r[3][3]) {
    const double w = u[0], x = u[1], y = u[2], z = u[3];
    r[0][0] = 1 - 2 * (y * y + z * z); r[0][1] = 2 * (x * y - w * z); r[0][2] = 2 * (x * z + w * y);
    r[1][0] = 2 * (x * y + w * z); r[1][1] = 1 - 2 * (x * x + z * z); r[1][2] = 2 * (y * z - w * x);
    r[2][0] = 2 * (x * z - w * y); r[2][1] = 2 * (y * z + w * x); r[2][2] = 1 - 2 * (x * x + y * y);
}

// covariance.cpp:51-56: Sigma = R diag(exp(2 ls)) R^T, then 0.5 (Sigma + Sigma^T)
__device__ __forceinline__ void build_covariance(const double q[4], const double ls[3],
                                                 double out[3][3]) {
    double u[4], nrm, r[3][3];
    unit_quat(q, u, &nrm);
    rotation_from_unit(u, r);
    const double s2[3] = {exp(2.0 * ls[0]), exp(2.0 * ls[1]), exp(2.0 * ls[2])};
    double rd[3][3], sg[3][3];
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) rd[i][k] = r[i][k] * s2[k];
    // Eigen's (R D) R^T: rows 0-1 are packet (sequential) sums, row 2 a halving-tree redux
    for (int j = 0; j < 3; ++j) {
        for (int i = 0; i < 2; ++i) sg[i][j] = (rd[i][0] * r[j][0] + rd[i][1] * r[j][1]) + rd[i][2] * r[j][2];
        sg[2][j] = rd[2][0] * r[j][0] + (rd[2][1] * r[j][1] + rd[2][2] * r[j][2]);
    }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) out[i][j] = 0.5 * (sg[i][j] + sg[j][i]);
}

__device__ __forceinline__ void mul23_33(const double a[2][3], const double b[3][3], double c[2][3]) {
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 3; ++j)
            c[i][j] = (a[i][0] * b[0][j] + a[i][1] * b[1][j]) + a[i][2] * b[2][j];
}

// projection.cpp:9-15
__device__ __forceinline__ void perspective_jacobian(const D3& p, const ViewParams& v, double j[2][3]) {
    const double z = p.z;
    j[0][0] = v.fx / z; j[0][1] = 0.0; j[0][2] = -v.fx * p.x / (z * z);
    j[1][0] = 0.0; j[1][1] = v.fy / z; j[1][2] = -v.fy * p.y / (z * z);
}

// sh.cpp constants
constexpr double kC0 = 0.28209479177387814;
constexpr double kC1 = 0.4886025119029199;
constexpr double kC2_0 = 1.0925484305920792, kC2_1 = 1.0925484305920792, kC2_2 = 0.31539156525252005,
                 kC2_3 = 1.0925484305920792, kC2_4 = 0.5462742152960396;
constexpr double kC3_0 = 0.5900435899266435, kC3_1 = 2.890611442640554, kC3_2 = 0.4570457994644658,
                 kC3_3 = 0.3731763325901154, kC3_4 = 0.4570457994644658, kC3_5 = 1.445305721320277,
                 kC3_6 = 0.5900435899266435;

// sh.cpp:30-53
__device__ __forceinline__ void sh_basis(const D3& d, int degree, double out[16]) {
    const double x = d.x, y = d.y, z = d.z;
#pragma unroll
    for (int i = 0; i < 16; ++i) out[i] = 0.0;
    out[0] = kC0;
    if (degree < 1) return;
    out[1] = kC1 * y; out[2] = kC1 * z; out[3] = kC1 * x;
    if (degree < 2) return;
    const double xx = x * x, yy = y * y, zz = z * z;
    out[4] = kC2_0 * x * y; out[5] = kC2_1 * y * z; out[6] = kC2_2 * (2.0 * zz - xx - yy);
    out[7] = kC2_3 * x * z; out[8] = kC2_4 * (xx - yy);
    if (degree < 3) return;
    out[9] = kC3_0 * y * (3.0 * xx - yy);
    out[10] = kC3_1 * x * y * z;
    out[11] = kC3_2 * y * (4.0 * zz - xx - yy);
    out[12] = kC3_3 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    out[13] = kC3_4 * x * (4.0 * zz - xx - yy);
    out[14] = kC3_5 * z * (xx - yy);
    out[15] = kC3_6 * x * (xx - 3.0 * yy);
}

// d(basis_k)/d(dir) . a  accumulated over k with weights wk = coeffs_k . d_color (sh.cpp:55-80)
__device__ __forceinline__ D3 sh_dir_grad(const D3& d, int degree, const double wk[16]) {
    D3 g{0.0, 0.0, 0.0};
    if (degree < 1) return g;
    const double x = d.x, y = d.y, z = d.z;
    auto acc = [&](double s, double jx, double jy, double jz, double w) {
        g.x += s * jx * w; g.y += s * jy * w; g.z += s * jz * w;
    };
    acc(1.0, 0.0, kC1, 0.0, wk[1]);
    acc(1.0, 0.0, 0.0, kC1, wk[2]);
    acc(1.0, kC1, 0.0, 0.0, wk[3]);
    if (degree < 2) return g;
    acc(kC2_0, y, x, 0.0, wk[4]);
    acc(kC2_1, 0.0, z, y, wk[5]);
    acc(kC2_2, -2.0 * x, -2.0 * y, 4.0 * z, wk[6]);
    acc(kC2_3, z, 0.0, x, wk[7]);
    acc(kC2_4, 2.0 * x, -2.0 * y, 0.0, wk[8]);
    if (degree < 3) return g;
    const double xx = x * x, yy = y * y, zz = z * z;
    acc(kC3_0, 6.0 * x * y, 3.0 * xx - 3.0 * yy, 0.0, wk[9]);
    acc(kC3_1, y * z, x * z, x * y, wk[10]);
    acc(kC3_2, -2.0 * x * y, 4.0 * zz - xx - 3.0 * yy, 8.0 * y * z, wk[11]);
    acc(kC3_3, -6.0 * x * z, -6.0 * y * z, 6.0 * zz - 3.0 * xx - 3.0 * yy, wk[12]);
    acc(kC3_4, 4.0 * zz - 3.0 * xx - yy, -2.0 * x * y, 8.0 * x * z, wk[13]);
    acc(kC3_5, 2.0 * x * z, -2.0 * y * z, xx - yy, wk[14]);
    acc(kC3_6, 3.0 * xx - 3.0 * yy, -6.0 * x * y, 0.0, wk[15]);
    return g;
}

__device__ __forceinline__ double ldp(const float* __restrict__ params, int64_t cap, int plane, int i) {
    return static_cast<double>(__ldg(params + plane * cap + i));
}

// Degree-specialised SH (sh.cpp:82-109): with D a compile-time constant every basis array is
// fully unrolled into registers (a runtime-bounded loop would spill it to local memory).
template <int D>
__device__ __forceinline__ void sh_raw_t(const D3& dir, const float* __restrict__ params, int64_t cap, int i,
                                         double raw[3]) {
    double basis[16];
    sh_basis(dir, D, basis);
    raw[0] = raw[1] = raw[2] = 0.5;
#pragma unroll
    for (int k = 0; k < (D + 1) * (D + 1); ++k)
#pragma unroll
        for (int c = 0; c < 3; ++c) raw[c] += basis[k] * ldp(params, cap, P_SH + 3 * k + c, i);
}

__device__ __forceinline__ void sh_raw(int deg, const D3& dir, const float* __restrict__ params, int64_t cap, int i,
                                       double raw[3]) {
    switch (deg) {
        case 0: sh_raw_t<0>(dir, params, cap, i, raw); break;
        case 1: sh_raw_t<1>(dir, params, cap, i, raw); break;
        case 2: sh_raw_t<2>(dir, params, cap, i, raw); break;
        default: sh_raw_t<3>(dir, params, cap, i, raw); break;
    }
}

__device__ __forceinline__ void gput(float* __restrict__ g, int64_t idx, double val, bool acc) {
    if (acc) g[idx] += static_cast<float>(val); else g[idx] = static_cast<float>(val);
}

template <int D>
__device__ __forceinline__ D3 sh_vjp_t(const D3& dir, const float* __restrict__ params, int64_t cap, int i,
                                       const double dr[3], float* __restrict__ grads, int64_t gcap, bool accum) {
    double basis[16], wk[16];
    sh_basis(dir, D, basis);
#pragma unroll
    for (int k = 0; k < 16; ++k) wk[k] = 0.0;
#pragma unroll
    for (int k = 0; k < (D + 1) * (D + 1); ++k) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c) s += ldp(params, cap, P_SH + 3 * k + c, i) * dr[c];
        wk[k] = s;
#pragma unroll
        for (int c = 0; c < 3; ++c) gput(grads, (P_SH + 3 * k + c) * gcap + i, basis[k] * dr[c], accum);
    }
    return sh_dir_grad(dir, D, wk);
}

__device__ __forceinline__ D3 sh_vjp(int deg, const D3& dir, const float* __restrict__ params, int64_t cap, int i,
                                     const double dr[3], float* __restrict__ grads, int64_t gcap, bool accum) {
    switch (deg) {
        case 0: return sh_vjp_t<0>(dir, params, cap, i, dr, grads, gcap, accum);
        case 1: return sh_vjp_t<1>(dir, params, cap, i, dr, grads, gcap, accum);
        case 2: return sh_vjp_t<2>(dir, params, cap, i, dr, grads, gcap, accum);
        default: return sh_vjp_t<3>(dir, params, cap, i, dr, grads, gcap, accum);
    }
}

// covariance.cpp:17-43 rotation_partial(u, k) (without the factor 2, applied by the caller)
__device__ __forceinline__ void rotation_partial(const double u[4], int k, double d[3][3]) {
    const double w = u[0], x = u[1], y = u[2], z = u[3];
    if (k == 0) {
        d[0][0] = 0; d[0][1] = -z; d[0][2] = y; d[1][0] = z; d[1][1] = 0; d[1][2] = -x;
        d[2][0] = -y; d[2][1] = x; d[2][2] = 0;
    } else if (k == 1) {
        d[0][0] = 0; d[0][1] = y; d[0][2] = z; d[1][0] = y; d[1][1] = -2 * x; d[1][2] = -w;
        d[2][0] = z; d[2][1] = w; d[2][2] = -2 * x;
    } else if (k == 2) {
        d[0][0] = -2 * y; d[0][1] = x; d[0][2] = w; d[1][0] = x; d[1][1] = 0; d[1][2] = z;
        d[2][0] = -w; d[2][1] = z; d[2][2] = -2 * y;
    } else {
        d[0][0] = -2 * z; d[0][1] = -w; d[0][2] = x; d[1][0] = w; d[1][1] = -2 * z; d[1][2] = y;
        d[2][0] = x; d[2][1] = y; d[2][2] = 0;
    }
}

}  // namespace

// ------------------------------------------------------------------------------------------
// K1 runs in two phases so the expensive exact projection only sees dense warps of likely
// survivors (about a third of the map in view).
//
// K1a: camera transform (exact fp64, as in K1b), near clip, and the off-screen test with a
// conservative radius bound R >= the exact radius: lambda_max(Sigma_I) <= ||J||_F^2
// max_k exp(2 ls_k) + 0.3 (W is a rotation). A Gaussian K1a culls is culled by the exact test
// too, so the candidate list is a superset of the visible set (the camera transform and near clip
// in fp64 as K1b; the bound itself in fp32 with margins). Candidates are appended with
// warp-aggregated atomics (their order does not matter: K1b writes by map index).
__global__ void __launch_bounds__(256) cull_kernel(const float* __restrict__ params, int64_t cap, int n,
                                                   ViewParams v, int32_t* __restrict__ cand,
                                                   unsigned long long* __restrict__ counters) {
    pdl_enter();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    bool keep = false;
    if (i < n) {
        const D3 pos{ldp(params, cap, P_POS, i), ldp(params, cap, P_POS + 1, i), ldp(params, cap, P_POS + 2, i)};
        D3 p = quat_rotate(v.qw, v.qx, v.qy, v.qz, pos);
        p = {p.x + v.tx, p.y + v.ty, p.z + v.tz};
        if (!(p.z <= kNearClip)) {  // the exact test's own near clip (same fp64 sequence)
            // the rest in fp32 with margins that cover its rounding (relative ~1e-6 against the
            // 1e-3 and 1e-4 |m| slack): the bound only has to stay conservative
            const float px = static_cast<float>(p.x), py = static_cast<float>(p.y), pz = static_cast<float>(p.z);
            const float fx = static_cast<float>(v.fx), fy = static_cast<float>(v.fy);
            const float iz = 1.0f / pz;
            const float ux = px * iz, uy = py * iz;
            const float mx = fx * ux + static_cast<float>(v.cx), my = fy * uy + static_cast<float>(v.cy);
            const float jf2 = (fx * iz) * (fx * iz) * (1.0f + ux * ux) + (fy * iz) * (fy * iz) * (1.0f + uy * uy);
            const float lsmax = fmaxf(fmaxf(params[P_LS * cap + i], params[(P_LS + 1) * cap + i]),
                                      params[(P_LS + 2) * cap + i]);
            const float lam = (jf2 * __expf(2.0f * lsmax) + static_cast<float>(kCovReg)) * 1.001f;
            const float R = ceilf(3.0f * sqrtf(lam)) + 2.0f + 1e-4f * (fabsf(mx) + fabsf(my));
            keep = !(mx + R < 0.0f || mx - R > static_cast<float>(v.width - 1) || my + R < 0.0f ||
                     my - R > static_cast<float>(v.height - 1)) ||
                   !(lam < 1e30f);  // non-finite bound: leave the decision to the exact test
        }
    }
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    if (mask) {
        const int lane = threadIdx.x & 31;
        const int leader = __ffs(mask) - 1;
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(counters + 2, static_cast<unsigned long long>(__popc(mask)));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (keep) cand[base + __popc(mask & ((1u << lane) - 1u))] = i;
    }
}

void launch_cull(const float* params, int64_t cap, int n, const ViewParams& v, int32_t* cand,
                 unsigned long long* counters, cudaStream_t st) {
    if (n > 0) launch_pdl(cull_kernel, div_up(n, 256), 256, st, params, cap, n, v, cand, counters);
}

// K1b: exact projection of the candidates (grid-stride over the device-side candidate count).
// Writes the 64 B Splat record at the map index and the fp64 depth bits (map-indexed), and
// appends visible Gaussians to the sort input: a 24-bit key from the fp32-rounded depth bits (a
// monotone non-decreasing function of the depth) and the map index. Counts the visible set and the (tile, gaussian) pairs.
// Reference: rasterizer.cpp:37-68 (project_visible) + projection.cpp:17-40 + sh.cpp:82-92 +
// rasterizer.cpp:81-88 (pixel rect -> tile rect).
// 3 CTAs per SM (80 registers, 80 B of L1-resident spills) beat the unconstrained 128-register
// build: the fp64 chain is latency-bound and the extra warps hide it (measured -6%)
#ifndef GSB_K1_MIN_BLOCKS
#define GSB_K1_MIN_BLOCKS 4  // 64 registers (small spill): -3% on K1 against 3 (diag/variant_levels.sh)
#endif
__global__ void __launch_bounds__(256, GSB_K1_MIN_BLOCKS) preprocess_fwd_kernel(
    const float* __restrict__ params, int64_t cap, const int8_t* __restrict__ degree,
    const int32_t* __restrict__ cand, ViewParams v, Splat* __restrict__ rec_by_gid,
    unsigned long long* __restrict__ depth_key, int32_t* __restrict__ vis_gid, uint32_t* __restrict__ key32,
    unsigned long long* __restrict__ counters) {
    pdl_enter();
    const int n_cand = static_cast<int>(counters[2]);
    const int stride = gridDim.x * blockDim.x;
    const int first = blockIdx.x * blockDim.x + threadIdx.x;
    for (int base_c = first - (threadIdx.x & 31); base_c < n_cand; base_c += stride) {
    const int c = base_c + (threadIdx.x & 31);
    const int i = c < n_cand ? cand[c] : 0;
    bool visible = false;
    uint32_t ntiles = 0;
    double depth = 0.0;
    if (c < n_cand) {
        const D3 pos{ldp(params, cap, P_POS, i), ldp(params, cap, P_POS + 1, i), ldp(params, cap, P_POS + 2, i)};
        D3 p = quat_rotate(v.qw, v.qx, v.qy, v.qz, pos);
        p = {p.x + v.tx, p.y + v.ty, p.z + v.tz};
        if (!(p.z <= kNearClip)) {  // projection.cpp:20 (culled, not clamped)
            const double mx = v.fx * p.x / p.z + v.cx;
            const double my = v.fy * p.y / p.z + v.cy;
            double W[3][3], J[2][3], M[2][3], S[3][3], MS[2][3];
            pose_matrix(v, W);
            perspective_jacobian(p, v, J);
            mul23_33(J, W, M);
            const double q[4] = {ldp(params, cap, P_ROT, i), ldp(params, cap, P_ROT + 1, i),
                                 ldp(params, cap, P_ROT + 2, i), ldp(params, cap, P_ROT + 3, i)};
            const double ls[3] = {ldp(params, cap, P_LS, i), ldp(params, cap, P_LS + 1, i),
                                  ldp(params, cap, P_LS + 2, i)};
            build_covariance(q, ls, S);
            mul23_33(M, S, MS);
            double cov[2][2];
            for (int a = 0; a < 2; ++a)
                for (int b = 0; b < 2; ++b)
                    cov[a][b] = (MS[a][0] * M[b][0] + MS[a][1] * M[b][1]) + MS[a][2] * M[b][2];
            cov[0][0] += kCovReg;
            cov[1][1] += kCovReg;
            double c2[2][2];
            for (int a = 0; a < 2; ++a)
                for (int b = 0; b < 2; ++b) c2[a][b] = 0.5 * (cov[a][b] + cov[b][a]);
            const double half_trace = 0.5 * (c2[0][0] + c2[1][1]);
            const double det = c2[0][0] * c2[1][1] - c2[1][0] * c2[0][1];
            const double disc = sqrt(fmax(half_trace * half_trace - det, 0.0));
            const double lmax = half_trace + disc;
            const double rr = fmin(ceil(3.0 * sqrt(lmax)), 1073741824.0);
            const int radius = max(1, static_cast<int>(rr));
            const double rd = static_cast<double>(radius);
            // rasterizer.cpp:48-50 off-screen cull
            if (!(mx + rd < 0.0 || mx - rd > static_cast<double>(v.width - 1) || my + rd < 0.0 ||
                  my - rd > static_cast<double>(v.height - 1))) {
                visible = true;
                // Eigen 2x2 inverse: adj * (1 / det)
                const double invdet = 1.0 / det;
                Splat s;
                s.mx = mx;
                s.my = my;
                s.ca = static_cast<float>(c2[1][1] * invdet);
                s.cb = static_cast<float>(-c2[0][1] * invdet);
                s.cc = static_cast<float>(c2[0][0] * invdet);
                s.opacity = static_cast<float>(1.0 / (1.0 + exp(-ldp(params, cap, P_OP, i))));
                // view direction from the camera centre (types.hpp:61-63, rasterizer.cpp:61-64)
                const D3 ctr = quat_rotate(v.qw, -v.qx, -v.qy, -v.qz, D3{-v.tx, -v.ty, -v.tz});
                const D3 vd{pos.x - ctr.x, pos.y - ctr.y, pos.z - ctr.z};
                const double dist = sqrt((vd.x * vd.x + vd.y * vd.y) + vd.z * vd.z);
                const D3 dir = dist > 0.0 ? D3{vd.x / dist, vd.y / dist, vd.z / dist} : D3{0.0, 0.0, 1.0};
                double col[3];
                sh_raw(degree[i], dir, params, cap, i, col);
                s.r = static_cast<float>(fmin(fmax(col[0], 0.0), 1.0));
                s.g = static_cast<float>(fmin(fmax(col[1], 0.0), 1.0));
                s.b = static_cast<float>(fmin(fmax(col[2], 0.0), 1.0));
                s.depth = static_cast<float>(p.z);
                // rasterizer.cpp:81-88: integer pixel rect of the 3-sigma box
                const int px0 = max(0, static_cast<int>(ceil(mx - rd)));
                const int px1 = min(v.width - 1, static_cast<int>(floor(mx + rd)));
                const int py0 = max(0, static_cast<int>(ceil(my - rd)));
                const int py1 = min(v.height - 1, static_cast<int>(floor(my + rd)));
                if (px0 <= px1 && py0 <= py1) {
                    ntiles = static_cast<uint32_t>((px1 / kTile - px0 / kTile + 1) * (py1 / kTile - py0 / kTile + 1));
                    s.x0 = static_cast<int16_t>(px0); s.x1 = static_cast<int16_t>(px1);
                    s.y0 = static_cast<int16_t>(py0); s.y1 = static_cast<int16_t>(py1);
                } else {
                    s.x0 = 1; s.x1 = 0; s.y0 = 1; s.y1 = 0;  // empty
                }
                s.gid = i;
                s.ntiles = ntiles;
                rec_by_gid[i] = s;
                depth_key[i] = static_cast<unsigned long long>(__double_as_longlong(p.z));
                depth = p.z;
            }
        }
    }
    // warp-aggregated: append visible (fp32 depth key, map index); count pairs
    const int lane = threadIdx.x & 31;
    const unsigned mask = __ballot_sync(0xffffffffu, visible);
    if (mask) {
        const int leader = __ffs(mask) - 1;
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(counters + 0, static_cast<unsigned long long>(__popc(mask)));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (visible) {
            const size_t slot = base + __popc(mask & ((1u << lane) - 1u));
            vis_gid[slot] = i;
            // 24-bit monotone depth key: fp32 bits above the near plane, 16 ulps per step,
            // clamped (ties, including the clamp, are ordered exactly by fix_ties)
            const uint32_t bits = __float_as_uint(__double2float_rn(depth)) - kDepthKeyBase;
            key32[slot] = min(bits >> 4, 0xffffffu);
        }
    }
    unsigned long long pairs = ntiles;
    for (int o = 16; o > 0; o >>= 1) pairs += __shfl_xor_sync(0xffffffffu, pairs, o);
    if (lane == 0 && pairs) atomicAdd(counters + 1, pairs);
    }
}

void launch_preprocess_fwd(const float* params, int64_t cap, const int8_t* degree, const int32_t* cand,
                           int max_cand, const ViewParams& v, Splat* rec_by_gid, unsigned long long* depth_key,
                           int32_t* vis_gid, uint32_t* key32, unsigned long long* counters, cudaStream_t st) {
    if (max_cand <= 0) return;
    const int blocks = std::min(div_up(max_cand, 256), 148 * 8);
    launch_pdl(preprocess_fwd_kernel, blocks, 256, st, params, cap, degree, cand, v, rec_by_gid, depth_key, vis_gid,
                                                  key32, counters);
}

// ------------------------------------------------------------------------------------------
// K8: per visible Gaussian, the fp64 sum of its (tile, gaussian) partial rows, then the VJP chain
// (rasterizer.cpp:323-353): colour clamp mask -> eval_sh_vjp -> view-direction chain, sigmoid,
// project_gaussian_vjp (projection.cpp:42-74) -> build_covariance_vjp (covariance.cpp:58-79).
// Accumulates into the gradient planes (batch semantics = GaussianGrad::add, gaussian.hpp:51-57).
// Two kernels: K8a reduces each rank's rows (streaming, low register count) into a rank-ordered
// fp32 [N_vis][10] buffer; K8b runs the fp64 VJP with threads over K1's visible list (runs of
// ascending map indices: the 14-59 parameter planes are read and the gradient planes written
// mostly coalesced), the rank looked up in rank_of (written by pack).
constexpr int kBwdThreads = 64;  // 2 warps per block: -9% on K8 against 128 (more resident blocks)

// K8a: a warp owns 32 consecutive ranks, whose partial rows are one contiguous range (rank
// order: the sums do not depend on K1's run-to-run append order). It streams them 32 rows at a
// time (lane l reads row base + l: 1280 B coalesced), finds each row's rank with a 5-step
// shuffle search over the 33 segment offsets, sums runs of equal rank
// with a segmented shuffle reduction (fixed tree: deterministic), and the owning lane adds the
// run total into its fp64 accumulator. No block barriers; load balance is per row, not per rank.
__global__ void __launch_bounds__(kBwdThreads) reduce_partials_kernel(const uint32_t* __restrict__ emit_off,
                                                                    const float* __restrict__ partials,
                                                                    const unsigned long long* __restrict__ cnt,
                                                                    float* __restrict__ sums) {
    pdl_enter();
    __shared__ float seg[kBwdThreads / 32][32][kNumPartials + 1];
    __shared__ int stamp[kBwdThreads / 32][32];  // pass in which rank l's run total was written
    const int n_vis = static_cast<int>(cnt[kCntVisible]);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q0 = blockIdx.x * kBwdThreads + warp * 32;
    if (q0 >= n_vis || overflowed(cnt)) return;  // warp-uniform; no block barrier below
    const int nr = min(32, n_vis - q0);
    const uint32_t off = emit_off[q0 + min(lane, nr)];  // lane l: first row of rank q0 + l
    const uint32_t end = __shfl_sync(0xffffffffu, emit_off[q0 + nr], 0);
    const uint32_t beg = __shfl_sync(0xffffffffu, off, 0);
    GSB_CHECK(beg <= end && end <= cnt[kCntPairs]);
    double acc[kNumPartials];
#pragma unroll
    for (int k = 0; k < kNumPartials; ++k) acc[k] = 0.0;
    stamp[warp][lane] = -1;
    __syncwarp();
    // the next pass's rows are loaded one pass ahead (their latency overlaps this pass's shuffles)
    auto load_row = [&](uint32_t e, float2 r[kNumPartials / 2]) {
        if (e < end) {
            const float2* row = reinterpret_cast<const float2*>(partials + static_cast<size_t>(e) * kNumPartials);
#pragma unroll
            for (int k = 0; k < kNumPartials / 2; ++k) r[k] = __ldg(row + k);
        }
    };
    float2 cur[kNumPartials / 2];
    load_row(beg + lane, cur);
    int pass = 0;
    for (uint32_t base = beg; base < end; base += 32, ++pass) {
        const uint32_t e = base + lane;
        const bool valid = e < end;
        float2 nxt[kNumPartials / 2];
        load_row(e + 32, nxt);
        // rank (0..nr-1) of row e: largest l with off_l <= e (offsets are non-decreasing)
        int rl = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const int c = rl + step;
            const uint32_t oc = __shfl_sync(0xffffffffu, off, c < nr ? c : 0);
            if (c < nr && oc <= e) rl = c;
        }
        float v[kNumPartials];
        if (valid) {
#pragma unroll
            for (int k = 0; k < kNumPartials / 2; ++k) {
                v[2 * k] = cur[k].x;
                v[2 * k + 1] = cur[k].y;
            }
        } else {
#pragma unroll
            for (int k = 0; k < kNumPartials; ++k) v[k] = 0.f;
            rl = -1;  // never matches a real run
        }
        // segmented suffix sums: lane ends up with the sum over [lane, end of its run]
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int ro = __shfl_down_sync(0xffffffffu, rl, d);
            const bool same = lane + d < 32 && ro == rl;
#pragma unroll
            for (int k = 0; k < kNumPartials; ++k) {
                const float o = __shfl_down_sync(0xffffffffu, v[k], d);
                if (same) v[k] += o;
            }
        }
        const int rprev = __shfl_up_sync(0xffffffffu, rl, 1);
        const bool head = valid && (lane == 0 || rprev != rl);
        if (head) {
#pragma unroll
            for (int k = 0; k < kNumPartials; ++k) seg[warp][rl][k] = v[k];
            stamp[warp][rl] = pass;
        }
        __syncwarp();
        if (stamp[warp][lane] == pass) {
#pragma unroll
            for (int k = 0; k < kNumPartials; ++k) acc[k] += static_cast<double>(seg[warp][lane][k]);
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < kNumPartials / 2; ++k) cur[k] = nxt[k];
    }
    if (lane >= nr) return;
    // stored as fp32 (half the round trip to K8b; the rounding, 2^-24 relative, is far below the
    // fp32 partials' own error)
    float2* out = reinterpret_cast<float2*>(sums + static_cast<size_t>(q0 + lane) * kNumPartials);
#pragma unroll
    for (int k = 0; k < kNumPartials / 2; ++k)
        out[k] = make_float2(static_cast<float>(acc[2 * k]), static_cast<float>(acc[2 * k + 1]));
}

template <bool ACC>
#ifndef GSB_K8B_MIN_BLOCKS
#define GSB_K8B_MIN_BLOCKS 12  // 85 registers: -3% on K8 against the unconstrained 128 (diag/variant_levels.sh)
#endif
__global__ void __launch_bounds__(kBwdThreads, GSB_K8B_MIN_BLOCKS) preprocess_bwd_kernel(
    const float* __restrict__ params, int64_t cap, const int8_t* __restrict__ degree, ViewParams v,
    const uint32_t* __restrict__ emit_off, const float* __restrict__ sums, const unsigned long long* __restrict__ cnt,
    float* __restrict__ grads, int64_t gcap, const int32_t* __restrict__ rank_of, const int32_t* __restrict__ vis_gid) {
    pdl_enter();
    const int t = blockIdx.x * kBwdThreads + threadIdx.x;
    if (t >= static_cast<int>(cnt[kCntVisible]) || overflowed(cnt)) return;
    const int i = vis_gid[t];
    GSB_CHECK(i >= 0 && i < gcap);
    const int r = rank_of[i];
    GSB_CHECK(r >= 0 && r < static_cast<int>(cnt[kCntVisible]));
    if (emit_off[r] == emit_off[r + 1]) return;  // no tile: never touched (rasterizer.cpp:327)
    float gp[kGeomParams];  // map-indexed: all loads in flight at once
#pragma unroll
    for (int k = 0; k < kGeomParams; ++k) gp[k] = __ldg(params + static_cast<int64_t>(k) * cap + i);
    const int deg = degree[i];
    double acc[kNumPartials];
    const float2* in = reinterpret_cast<const float2*>(sums + static_cast<size_t>(r) * kNumPartials);
#pragma unroll
    for (int k = 0; k < kNumPartials / 2; ++k) {
        const float2 q = in[k];
        acc[2 * k] = q.x;
        acc[2 * k + 1] = q.y;
    }
    // the opacity exactly as K1 rounded it into the record (same expression, same translation unit)
    const float opf = static_cast<float>(1.0 / (1.0 + exp(-static_cast<double>(gp[P_OP]))));
    bool any = false;
#pragma unroll
    for (int k = 0; k < kNumPartials; ++k) any |= (acc[k] != 0.0);
    if (!any) return;  // untouched (or all-zero cotangent): exact zero gradient
    // the blend evaluates u = Sigma^-1 d with the conic pre-scaled by k = -log2(e)/2 (exp2 form)
    // and accumulates the mean / covariance terms without the opacity factor (op and op / 2)
    const double inv_k = 1.0 / static_cast<double>(-0.72134752044448170368f);
    const double op = static_cast<double>(opf);
    acc[5] *= op * inv_k;
    acc[6] *= op * inv_k;
    acc[7] *= 0.5 * op * inv_k * inv_k;
    acc[8] *= 0.5 * op * inv_k * inv_k;
    acc[9] *= 0.5 * op * inv_k * inv_k;
    const D3 pos{gp[P_POS], gp[P_POS + 1], gp[P_POS + 2]};

    // ---- colour: clamp mask, SH, view direction (rasterizer.cpp:330-340)
    const D3 ctr = quat_rotate(v.qw, -v.qx, -v.qy, -v.qz, D3{-v.tx, -v.ty, -v.tz});
    const D3 vd{pos.x - ctr.x, pos.y - ctr.y, pos.z - ctr.z};
    const double dist = sqrt((vd.x * vd.x + vd.y * vd.y) + vd.z * vd.z);
    const D3 dir = dist > 0.0 ? D3{vd.x / dist, vd.y / dist, vd.z / dist} : D3{0.0, 0.0, 1.0};
    double raw[3];
    sh_raw(deg, dir, params, cap, i, raw);
    double dr[3];
    for (int c = 0; c < 3; ++c) dr[c] = (raw[c] <= 0.0 || raw[c] >= 1.0) ? 0.0 : acc[c];
    const D3 ddir = sh_vjp(deg, dir, params, cap, i, dr, grads, gcap, ACC);
    double gpos[3] = {0.0, 0.0, 0.0};
    if (dist > 0.0) {
        const double vdd = (dir.x * ddir.x + dir.y * ddir.y) + dir.z * ddir.z;
        gpos[0] = (ddir.x - dir.x * vdd) / dist;
        gpos[1] = (ddir.y - dir.y * vdd) / dist;
        gpos[2] = (ddir.z - dir.z * vdd) / dist;
    }

    // ---- opacity logit through the sigmoid (rasterizer.cpp:343)
    const double o = 1.0 / (1.0 + exp(-static_cast<double>(gp[P_OP])));
    gput(grads, P_OP * gcap + i, acc[4] * o * (1.0 - o), ACC);

    // ---- geometry (projection.cpp:42-74)
    D3 p = quat_rotate(v.qw, v.qx, v.qy, v.qz, pos);
    p = {p.x + v.tx, p.y + v.ty, p.z + v.tz};
    double W[3][3], J[2][3], M[2][3], S[3][3];
    pose_matrix(v, W);
    perspective_jacobian(p, v, J);
    mul23_33(J, W, M);
    const double q[4] = {gp[P_ROT], gp[P_ROT + 1], gp[P_ROT + 2], gp[P_ROT + 3]};
    const double ls[3] = {gp[P_LS], gp[P_LS + 1], gp[P_LS + 2]};
    build_covariance(q, ls, S);
    const double dcov[2][2] = {{acc[7], acc[8]}, {acc[8], acc[9]}};
    // d_sigma_w = M^T dcov M
    double dsw[3][3];
    for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 3; ++c) {
            const double t0 = M[0][a] * dcov[0][0] + M[1][a] * dcov[1][0];
            const double t1 = M[0][a] * dcov[0][1] + M[1][a] * dcov[1][1];
            dsw[a][c] = t0 * M[0][c] + t1 * M[1][c];
        }
    // d_m = (dcov + dcov^T) M Sigma_w ; d_j = d_m W^T
    double dsm[2][3], dm[2][3], dj[2][3];
    for (int a = 0; a < 2; ++a)
        for (int c = 0; c < 3; ++c) dsm[a][c] = (2.0 * dcov[a][0]) * M[0][c] + (2.0 * dcov[a][1]) * M[1][c];
    mul23_33(dsm, S, dm);
    for (int a = 0; a < 2; ++a)
        for (int c = 0; c < 3; ++c) dj[a][c] = (dm[a][0] * W[c][0] + dm[a][1] * W[c][1]) + dm[a][2] * W[c][2];
    // build_covariance_vjp (covariance.cpp:58-79)
    {
        double u[4], nrm, R[3][3];
        unit_quat(q, u, &nrm);
        rotation_from_unit(u, R);
        const double s2[3] = {exp(2.0 * ls[0]), exp(2.0 * ls[1]), exp(2.0 * ls[2])};
        double rtg[3][3], rtgr[3][3];
        for (int a = 0; a < 3; ++a)
            for (int c = 0; c < 3; ++c)
                rtg[a][c] = (R[0][a] * dsw[0][c] + R[1][a] * dsw[1][c]) + R[2][a] * dsw[2][c];
        for (int a = 0; a < 3; ++a)
            for (int c = 0; c < 3; ++c) rtgr[a][c] = (rtg[a][0] * R[0][c] + rtg[a][1] * R[1][c]) + rtg[a][2] * R[2][c];
        for (int k = 0; k < 3; ++k) gput(grads, (P_LS + k) * gcap + i, 2.0 * s2[k] * rtgr[k][k], ACC);
        double dR[3][3];
        for (int a = 0; a < 3; ++a)
            for (int c = 0; c < 3; ++c) {
                double s = 0.0;
                for (int b = 0; b < 3; ++b) s += (dsw[a][b] + dsw[b][a]) * R[b][c];
                dR[a][c] = s * s2[c];
            }
        double du[4];
        for (int k = 0; k < 4; ++k) {
            double d[3][3];
            rotation_partial(u, k, d);
            double s = 0.0;
            for (int c = 0; c < 3; ++c)
                for (int a = 0; a < 3; ++a) s += dR[a][c] * (2.0 * d[a][c]);
            du[k] = s;
        }
        const double ud = ((u[0] * du[0] + u[1] * du[1]) + u[2] * du[2]) + u[3] * du[3];
        for (int k = 0; k < 4; ++k) gput(grads, (P_ROT + k) * gcap + i, (du[k] - u[k] * ud) / nrm, ACC);
    }
    // position: J^T d_mean + J(p) terms + depth, then W^T
    double dp[3];
    for (int c = 0; c < 3; ++c) dp[c] = J[0][c] * acc[5] + J[1][c] * acc[6];
    const double z = p.z, z2 = z * z, z3 = z2 * z;
    dp[0] += dj[0][2] * (-v.fx / z2);
    dp[1] += dj[1][2] * (-v.fy / z2);
    dp[2] += dj[0][0] * (-v.fx / z2) + dj[1][1] * (-v.fy / z2) + dj[0][2] * (2.0 * v.fx * p.x / z3) +
             dj[1][2] * (2.0 * v.fy * p.y / z3);
    dp[2] += acc[3];
    for (int c = 0; c < 3; ++c) {
        const double dpos = (W[0][c] * dp[0] + W[1][c] * dp[1]) + W[2][c] * dp[2];
        gput(grads, (P_POS + c) * gcap + i, gpos[c] + dpos, ACC);
    }
}

// project_sparse_depth (sequence.cpp:246-259): LiDAR points -> per-pixel minimum camera z. The
// camera transform is K1's exact fp64 sequence; the pixel is lround(f x / z + c); the min rule is
// an atomicMin on the bits of the (positive) fp64 depths, so the result is order independent.
__global__ void sparse_depth_kernel(const double* __restrict__ pts, int stride, int64_t n, ViewParams v,
                                    unsigned long long* __restrict__ depth_bits) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double* q = pts + k * stride;
    D3 pc = quat_rotate(v.qw, v.qx, v.qy, v.qz, D3{q[0], q[1], q[2]});
    pc = {pc.x + v.tx, pc.y + v.ty, pc.z + v.tz};
    if (pc.z <= kNearClip) return;
    const long long px = llround(v.fx * pc.x / pc.z + v.cx);
    const long long py = llround(v.fy * pc.y / pc.z + v.cy);
    if (px < 0 || px >= v.width || py < 0 || py >= v.height) return;
    atomicMin(depth_bits + py * v.width + px, static_cast<unsigned long long>(__double_as_longlong(pc.z)));
}

__global__ void sparse_depth_finish_kernel(unsigned long long* __restrict__ bits, int P) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < P && bits[i] == 0x7ff0000000000000ull) bits[i] = 0ull;  // no point: 0.0 (the reference's empty)
}

__global__ void fill_u64_kernel(unsigned long long* __restrict__ out, int P, unsigned long long val) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < P) out[i] = val;
}

void launch_sparse_depth(const double* pts, int stride, int64_t n, const ViewParams& v, double* depth,
                         cudaStream_t st) {
    const int P = v.width * v.height;
    auto* bits = reinterpret_cast<unsigned long long*>(depth);
    fill_u64_kernel<<<div_up(P, 256), 256, 0, st>>>(bits, P, 0x7ff0000000000000ull);  // +inf
    if (n > 0)
        sparse_depth_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(pts, stride, n, v, bits);
    sparse_depth_finish_kernel<<<div_up(P, 256), 256, 0, st>>>(bits, P);
}

// ------------------------------------------------------------------------------------------
// init_gaussians_from_points (mapper.cpp:19-61) on the device. The isotropic scale is the mean
// distance to the k = min(3, n - 1) nearest other points (floored at 1e-4 m; 0.1 m with no
// neighbour), found exactly by expanding Chebyshev shells over a uniform grid whose occupied
// cells sit in an open-addressing hash table. Distances use the oracle's fp64 order
// ((dx^2 + dy^2) + dz^2, this file is --fmad=false); the k distances are summed in ascending
// order (the reference sums its heap's array order: at most 1 fp64 ulp apart).
namespace {
__device__ __forceinline__ uint64_t knn_pack(int64_t x, int64_t y, int64_t z) {
    return (static_cast<uint64_t>(x & 0x1fffff) << 42) | (static_cast<uint64_t>(y & 0x1fffff) << 21) |
           static_cast<uint64_t>(z & 0x1fffff);
}
__device__ __forceinline__ uint32_t knn_hash(uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return static_cast<uint32_t>(k);
}
constexpr uint64_t kKnnEmpty = ~0ull;
}  // namespace

__global__ void knn_keys_kernel(const double* __restrict__ pts, int64_t n, KnnGrid g, uint64_t* __restrict__ keys,
                                int32_t* __restrict__ idx) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* q = pts + 6 * i;
    const int64_t x = static_cast<int64_t>(floor((q[0] - g.lo[0]) / g.cell));
    const int64_t y = static_cast<int64_t>(floor((q[1] - g.lo[1]) / g.cell));
    const int64_t z = static_cast<int64_t>(floor((q[2] - g.lo[2]) / g.cell));
    keys[i] = knn_pack(x, y, z);
    idx[i] = static_cast<int32_t>(i);
}

// one thread per run of equal keys in the sorted order: insert (key -> [start, end))
__global__ void knn_table_kernel(const uint64_t* __restrict__ skeys, int64_t n, uint64_t* __restrict__ hkeys,
                                 int2* __restrict__ hvals, uint32_t hmask) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n || (i > 0 && skeys[i - 1] == skeys[i])) return;
    const uint64_t k = skeys[i];
    int64_t e = i + 1;
    while (e < n && skeys[e] == k) ++e;
    uint32_t h = knn_hash(k) & hmask;
    while (true) {
        const unsigned long long prev = atomicCAS(reinterpret_cast<unsigned long long*>(hkeys + h), kKnnEmpty, k);
        if (prev == kKnnEmpty || prev == k) break;
        h = (h + 1) & hmask;
    }
    hvals[h] = make_int2(static_cast<int>(i), static_cast<int>(e));
}

__device__ __forceinline__ int2 knn_lookup(const uint64_t* __restrict__ hkeys, const int2* __restrict__ hvals,
                                           uint32_t hmask, uint64_t k) {
    uint32_t h = knn_hash(k) & hmask;
    while (true) {
        const uint64_t c = hkeys[h];
        if (c == k) return hvals[h];
        if (c == kKnnEmpty) return make_int2(0, 0);
        h = (h + 1) & hmask;
    }
}

// writes the new Gaussians (fp32 SoA) at map index first + i (gaussian_from_point, mapper.cpp:47-58)
__global__ void knn_init_kernel(const double* __restrict__ pts, int64_t n, int k, KnnGrid g,
                                const uint64_t* __restrict__ hkeys, const int2* __restrict__ hvals, uint32_t hmask,
                                const int32_t* __restrict__ sidx, float* __restrict__ params, int64_t cap,
                                int64_t first) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* q = pts + 6 * i;
    const double px = q[0], py = q[1], pz = q[2];
    const int64_t cx = static_cast<int64_t>(floor((px - g.lo[0]) / g.cell));
    const int64_t cy = static_cast<int64_t>(floor((py - g.lo[1]) / g.cell));
    const int64_t cz = static_cast<int64_t>(floor((pz - g.lo[2]) / g.cell));
    double best[3] = {1e300, 1e300, 1e300};  // ascending
    int found = 0;
    for (int64_t r = 0; k > 0 && r <= g.max_ring; ++r) {
        for (int64_t dx = -r; dx <= r; ++dx)
            for (int64_t dy = -r; dy <= r; ++dy)
                for (int64_t dz = -r; dz <= r; ++dz) {
                    if (max(max(llabs(dx), llabs(dy)), llabs(dz)) != r) continue;
                    const int2 range = knn_lookup(hkeys, hvals, hmask, knn_pack(cx + dx, cy + dy, cz + dz));
                    for (int qq = range.x; qq < range.y; ++qq) {
                        const int64_t j = sidx[qq];
                        if (j == i) continue;
                        const double* o = pts + 6 * j;
                        const double ddx = o[0] - px, ddy = o[1] - py, ddz = o[2] - pz;
                        const double d2 = (ddx * ddx + ddy * ddy) + ddz * ddz;
                        int slot;
                        if (found < k) slot = found++;
                        else if (d2 < best[k - 1]) slot = k - 1;
                        else continue;
                        while (slot > 0 && best[slot - 1] > d2) {
                            best[slot] = best[slot - 1];
                            --slot;
                        }
                        best[slot] = d2;
                    }
                }
        if (found == k && sqrt(best[k - 1]) <= static_cast<double>(r) * g.cell) break;
    }
    double sc = 0.1;  // kDefaultInitScale
    if (k > 0 && found > 0) {
        double sum = 0.0;
        for (int j = 0; j < found; ++j) sum += sqrt(best[j]);
        sc = fmax(sum / found, 1e-4);  // kMinInitScale
    }
    const int64_t o = first + i;
    for (int pl = 0; pl < kNumParams; ++pl) params[pl * cap + o] = 0.f;
    params[P_POS * cap + o] = static_cast<float>(px);
    params[(P_POS + 1) * cap + o] = static_cast<float>(py);
    params[(P_POS + 2) * cap + o] = static_cast<float>(pz);
    params[P_ROT * cap + o] = 1.f;
    const float ls = static_cast<float>(log(sc));
    for (int a = 0; a < 3; ++a) params[(P_LS + a) * cap + o] = ls;
    params[P_OP * cap + o] = static_cast<float>(log(0.1 / (1.0 - 0.1)));  // logit(kInitOpacity)
    const double kShC0 = 0.28209479177387814;
    for (int c = 0; c < 3; ++c) params[(P_SH + c) * cap + o] = static_cast<float>((q[3 + c] - 0.5) / kShC0);
}

__global__ void knn_bbox_kernel(const double* __restrict__ pts, int64_t n, unsigned long long* __restrict__ out6) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int a = 0; a < 3; ++a) {
        const long long b = __double_as_longlong(pts[6 * i + a]);
        // order-preserving map of doubles onto unsigned integers
        const unsigned long long u = b < 0 ? ~static_cast<unsigned long long>(b)
                                           : static_cast<unsigned long long>(b) | 0x8000000000000000ull;
        atomicMin(out6 + a, u);
        atomicMax(out6 + 3 + a, u);
    }
}

__global__ void knn_count_runs_kernel(const uint64_t* __restrict__ skeys, int64_t n,
                                      unsigned long long* __restrict__ runs) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool start = i < n && (i == 0 || skeys[i - 1] != skeys[i]);
    const unsigned m = __ballot_sync(0xffffffffu, start);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(runs, static_cast<unsigned long long>(__popc(m)));
}

void launch_knn_count_runs(const uint64_t* skeys, int64_t n, unsigned long long* runs, cudaStream_t st) {
    cudaMemsetAsync(runs, 0, sizeof(unsigned long long), st);
    if (n > 0) knn_count_runs_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(skeys, n, runs);
}

// filter_points_by_visibility (keyframe.cpp:49-74): keep a point when it is behind the near
// plane, projects outside the image, or lands on a pixel whose rendered visibility is <= tau.
__global__ void vis_filter_kernel(const double* __restrict__ pts, int64_t n, ViewParams v,
                                  const float* __restrict__ vis, double tau, int32_t* __restrict__ keep) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double* q = pts + 6 * k;
    D3 pc = quat_rotate(v.qw, v.qx, v.qy, v.qz, D3{q[0], q[1], q[2]});
    pc = {pc.x + v.tx, pc.y + v.ty, pc.z + v.tz};
    int32_t kp = 1;
    if (pc.z > kNearClip) {
        const long long px = llround(v.fx * pc.x / pc.z + v.cx);
        const long long py = llround(v.fy * pc.y / pc.z + v.cy);
        if (px >= 0 && px < v.width && py >= 0 && py < v.height)
            kp = static_cast<double>(vis[py * v.width + px]) <= tau ? 1 : 0;
    }
    keep[k] = kp;
}

__global__ void compact_points_kernel(const double* __restrict__ src, int64_t n, const int32_t* __restrict__ keep,
                                      const int32_t* __restrict__ pos, double* __restrict__ dst) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n || !keep[k]) return;
#pragma unroll
    for (int c = 0; c < 6; ++c) dst[6 * static_cast<int64_t>(pos[k]) + c] = src[6 * k + c];
}

void launch_vis_filter(const double* pts6, int64_t n, const ViewParams& v, const float* vis, double tau,
                       int32_t* keep, cudaStream_t st) {
    if (n > 0) vis_filter_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(pts6, n, v, vis, tau, keep);
}

void launch_compact_points(const double* src6, int64_t n, const int32_t* keep, const int32_t* pos, double* dst6,
                           cudaStream_t st) {
    if (n > 0) compact_points_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(src6, n, keep, pos, dst6);
}

void launch_knn_bbox(const double* pts, int64_t n, unsigned long long* out6, cudaStream_t st) {
    cudaMemsetAsync(out6, 0xff, 3 * sizeof(unsigned long long), st);
    cudaMemsetAsync(out6 + 3, 0, 3 * sizeof(unsigned long long), st);
    if (n > 0) knn_bbox_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(pts, n, out6);
}

void launch_knn_keys(const double* pts, int64_t n, const KnnGrid& g, uint64_t* keys, int32_t* idx, cudaStream_t st) {
    if (n > 0) knn_keys_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(pts, n, g, keys, idx);
}

void launch_knn_table(const uint64_t* skeys, int64_t n, uint64_t* hkeys, int2* hvals, uint32_t hmask,
                      cudaStream_t st) {
    cudaMemsetAsync(hkeys, 0xff, sizeof(uint64_t) * (static_cast<size_t>(hmask) + 1), st);
    if (n > 0) knn_table_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(skeys, n, hkeys, hvals, hmask);
}

void launch_knn_init(const double* pts, int64_t n, int k, const KnnGrid& g, const uint64_t* hkeys, const int2* hvals,
                     uint32_t hmask, const int32_t* sidx, float* params, int64_t cap, int64_t first, cudaStream_t st) {
    if (n > 0)
        knn_init_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, st>>>(pts, n, k, g, hkeys, hvals, hmask,
                                                                                 sidx, params, cap, first);
}

void launch_preprocess_bwd(const float* params, int64_t cap, const int8_t* degree, const ViewParams& v,
                           const uint32_t* emit_off, const float* partials, float* sums, const unsigned long long* cnt,
                           int max_ranks, float* grads, int64_t gcap, bool accumulate, const int32_t* rank_of,
                           const int32_t* vis_gid, cudaStream_t st) {
    if (max_ranks <= 0) return;
    const int blocks = div_up(max_ranks, kBwdThreads);
    launch_pdl(reduce_partials_kernel, blocks, kBwdThreads, st, emit_off, partials, cnt, sums);
    // accumulate = false: the gradient planes were just zeroed, so plain stores replace the
    // read-modify-write of the gradient entries
    if (accumulate)
        launch_pdl(preprocess_bwd_kernel<true>, blocks, kBwdThreads, st, params, cap, degree, v, emit_off, sums, cnt,
                                                                   grads, gcap, rank_of, vis_gid);
    else
        launch_pdl(preprocess_bwd_kernel<false>, blocks, kBwdThreads, st, params, cap, degree, v, emit_off, sums, cnt,
                                                                    grads, gcap, rank_of, vis_gid);
}

}  // namespace gsb
