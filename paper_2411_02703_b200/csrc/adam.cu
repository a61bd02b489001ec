// K9 fused Adam over the Gaussian SoA (GaussianMap::apply_gradients, gaussian_map.cpp:37-54),
// the scene-extent reduction (refresh_extent, gaussian_map.cpp:87-99) and host-layout converters.
#include <cfloat>

#include "common.cuh"
#include "kernels.cuh"

namespace gsb {

// Step counts are stored as births: Gaussian i's Adam step after this update is
// t = t_common - birth[i] (birth = the map's update count when its state was reset), so the
// update only reads them. One thread per Gaussian; every Gaussian steps (even when unseen, so
// momentum keeps moving it, as in the reference). The per-Gaussian bias corrections are fp64;
// the per-scalar update is fp32 on fp32 m/v. Inactive SH coefficients are skipped: their m, v
// and gradient are exactly zero, so the reference's update there is -lr*0/(0+eps) = -0 (exact).
namespace {
struct AdamArgs {
    float lr[5];        // position (x scene_extent), rotation, log_scale, opacity, sh
    int32_t t_common;   // count + 1: the new step of every Gaussian with birth 0
    float a_common;     // 1 / (1 - 0.9^t_common)
    float b_common;     // 1 / (1 - 0.999^t_common)
};

__device__ __forceinline__ void adam_scalar(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                                            float g, float lr, float a, float b) {
    const float mk = fmaf(0.9f, *m, 0.1f * g);
    const float vk = fmaf(0.999f, *v, 0.001f * g * g);
    *m = mk;
    *v = vk;
    *p += -lr * (mk * a) / (sqrtf(vk * b) + 1e-15f);
}
}  // namespace

// The 11 geometry planes are unrolled so all their loads are in flight at once; SH planes
// follow per coefficient up to the Gaussian's active degree. The fp64 bias corrections come
// from the host for the common step count and are computed only for Gaussians appended later.
__global__ void __launch_bounds__(256) adam_kernel(float* __restrict__ params, float* __restrict__ m,
                                                   float* __restrict__ v, const int32_t* __restrict__ birth,
                                                   const int8_t* __restrict__ degree,
                                                   const float* __restrict__ grads, int64_t gcap, int64_t cap, int n,
                                                   AdamArgs args, const unsigned long long* __restrict__ cnt) {
    pdl_enter();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || overflowed(cnt)) return;
    const int t = args.t_common - birth[i];
    float a = args.a_common, b = args.b_common;
    if (t != args.t_common) {
        a = static_cast<float>(1.0 / (1.0 - pow(0.9, static_cast<double>(t))));
        b = static_cast<float>(1.0 / (1.0 - pow(0.999, static_cast<double>(t))));
    }
    float g[kGeomParams];
#pragma unroll
    for (int k = 0; k < kGeomParams; ++k) g[k] = __ldg(grads + static_cast<size_t>(k) * gcap + i);
#pragma unroll
    for (int k = 0; k < kGeomParams; ++k) {
        const float lr = k < 3 ? args.lr[0] : k < 7 ? args.lr[1] : k < 10 ? args.lr[2] : args.lr[3];
        const size_t o = static_cast<size_t>(k) * cap + i;
        adam_scalar(params + o, m + o, v + o, g[k], lr, a, b);
    }
    const int ncoef = (degree[i] + 1) * (degree[i] + 1);
    for (int c = 0; c < ncoef; ++c) {
        float gs[3];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) gs[ch] = __ldg(grads + static_cast<size_t>(P_SH + 3 * c + ch) * gcap + i);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            const size_t o = static_cast<size_t>(P_SH + 3 * c + ch) * cap + i;
            adam_scalar(params + o, m + o, v + o, gs[ch], args.lr[4], a, b);
        }
    }
}

// One thread per (parameter plane, 4 consecutive Gaussians): four independent 16-byte loads
// (gradient, value, m, v), the per-scalar update of adam_kernel, three 16-byte stores. Many
// small independent threads keep enough loads in flight to stream HBM (the per-Gaussian form
// serialises its planes). Every plane base is 16-byte aligned when both capacities are
// multiples of 4. SH planes past a Gaussian's degree are left untouched.
// 128-thread blocks: -5% (d = 0) / -6% (d = 3) against 256 (measured; more blocks in flight)
__global__ void __launch_bounds__(128) adam_plane_kernel(float* __restrict__ params, float* __restrict__ m,
                                                         float* __restrict__ v, const int32_t* __restrict__ birth,
                                                         const int8_t* __restrict__ degree,
                                                         const float* __restrict__ grads, int64_t gcap, int64_t cap,
                                                         int n, AdamArgs args,
                                                         const unsigned long long* __restrict__ cnt) {
    pdl_enter();
    const int i = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
    const int k = blockIdx.y;  // plane
    if (i >= n || overflowed(cnt)) return;
    const float4 g = __ldg(reinterpret_cast<const float4*>(grads + k * gcap + i));
    float4* pp = reinterpret_cast<float4*>(params + k * cap + i);
    float4* mp = reinterpret_cast<float4*>(m + k * cap + i);
    float4* vp = reinterpret_cast<float4*>(v + k * cap + i);
    float4 P = *pp, M = *mp, V = *vp;
    const int4 b4 = __ldg(reinterpret_cast<const int4*>(birth + i));
    const float lr = k < 3 ? args.lr[0] : k < 7 ? args.lr[1] : k < 10 ? args.lr[2] : k < 11 ? args.lr[3] : args.lr[4];
    const int ne = min(4, n - i);
    int live = (1 << ne) - 1;
    if (k >= P_SH) {  // coefficient c = (k - 11) / 3 exists up to the Gaussian's degree
        const int c = (k - P_SH) / 3;
        const char4 d4 = *reinterpret_cast<const char4*>(degree + i);
        const int d[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if ((d[e] + 1) * (d[e] + 1) <= c) live &= ~(1 << e);
        if (!live) return;
    }
    const int t[4] = {args.t_common - b4.x, args.t_common - b4.y, args.t_common - b4.z, args.t_common - b4.w};
    float* ps = &P.x;
    float* ms = &M.x;
    float* vs = &V.x;
    const float* gs = &g.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        if (!((live >> e) & 1)) continue;
        float a = args.a_common, b = args.b_common;
        if (t[e] != args.t_common) {
            a = static_cast<float>(1.0 / (1.0 - pow(0.9, static_cast<double>(t[e]))));
            b = static_cast<float>(1.0 / (1.0 - pow(0.999, static_cast<double>(t[e]))));
        }
        adam_scalar(ps + e, ms + e, vs + e, gs[e], lr, a, b);
    }
    *pp = P;
    *mp = M;
    *vp = V;
}

void launch_adam(float* params, float* m, float* v, const int32_t* birth, const int8_t* degree, const float* grads,
                 int64_t gcap, int64_t cap, int n, const double lr[5], double scene_extent, int64_t t_common,
                 const unsigned long long* cnt, int max_degree, cudaStream_t st) {
    if (n <= 0) return;
    AdamArgs args;
    args.lr[0] = static_cast<float>(lr[0] * scene_extent);
    for (int k = 1; k < 5; ++k) args.lr[k] = static_cast<float>(lr[k]);
    args.t_common = static_cast<int32_t>(t_common);
    args.a_common = static_cast<float>(1.0 / (1.0 - std::pow(0.9, static_cast<double>(t_common))));
    args.b_common = static_cast<float>(1.0 / (1.0 - std::pow(0.999, static_cast<double>(t_common))));
    if (cap % 4 == 0 && gcap % 4 == 0) {
        const dim3 grid(div_up(div_up(n, 4), 128), kGeomParams + 3 * (max_degree + 1) * (max_degree + 1));
        launch_pdl(adam_plane_kernel, grid, 128, st, params, m, v, birth, degree, grads, gcap, cap, n, args, cnt);
    } else
        launch_pdl(adam_kernel, div_up(n, 256), 256, st, params, m, v, birth, degree, grads, gcap, cap, n, args, cnt);
}

// GaussianMap::prune (gaussian_map.cpp:56-73): keep sigmoid(opacity_logit) >= threshold (fp64,
// types.hpp:10), then a stable compaction of every per-Gaussian array (parameters, Adam m / v,
// births, degrees) so the optimizer state stays aligned.
__global__ void prune_flags_kernel(const float* __restrict__ params, int64_t cap, int n, double thr,
                                   int32_t* __restrict__ keep) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double o = 1.0 / (1.0 + exp(-static_cast<double>(params[P_OP * cap + i])));
    keep[i] = o >= thr ? 1 : 0;
}

template <class T>
__global__ void compact_kernel(const T* __restrict__ src, T* __restrict__ dst, int64_t scap, int64_t dcap, int n,
                               const int32_t* __restrict__ keep, const int32_t* __restrict__ pos) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int plane = blockIdx.y;
    if (i >= n || !keep[i]) return;
    dst[plane * dcap + pos[i]] = src[plane * scap + i];
}

void launch_prune_flags(const float* params, int64_t cap, int n, double thr, int32_t* keep, cudaStream_t st) {
    if (n > 0) prune_flags_kernel<<<div_up(n, 256), 256, 0, st>>>(params, cap, n, thr, keep);
}

void launch_compact(const float* src, float* dst, int64_t scap, int64_t dcap, int planes, int n, const int32_t* keep,
                    const int32_t* pos, cudaStream_t st) {
    if (n > 0) compact_kernel<float><<<dim3(div_up(n, 256), planes), 256, 0, st>>>(src, dst, scap, dcap, n, keep, pos);
}

void launch_compact(const int32_t* src, int32_t* dst, int n, const int32_t* keep, const int32_t* pos, cudaStream_t st) {
    if (n > 0) compact_kernel<int32_t><<<div_up(n, 256), 256, 0, st>>>(src, dst, 0, 0, n, keep, pos);
}

void launch_compact(const int8_t* src, int8_t* dst, int n, const int32_t* keep, const int32_t* pos, cudaStream_t st) {
    if (n > 0) compact_kernel<int8_t><<<div_up(n, 256), 256, 0, st>>>(src, dst, 0, 0, n, keep, pos);
}

namespace {
__device__ __forceinline__ unsigned int ord(float f) {
    const unsigned int u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
}  // namespace

// out6 holds ordered-int encodings: min x,y,z then max x,y,z (host decodes)
__global__ void position_minmax_kernel(const float* __restrict__ params, int64_t cap, int n,
                                       unsigned int* __restrict__ out6) {
    unsigned int lo[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, hi[3] = {0u, 0u, 0u};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        for (int c = 0; c < 3; ++c) {
            const unsigned int o = ord(params[c * cap + i]);
            lo[c] = min(lo[c], o);
            hi[c] = max(hi[c], o);
        }
    for (int c = 0; c < 3; ++c) {
        for (int s = 16; s > 0; s >>= 1) {
            lo[c] = min(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], s));
            hi[c] = max(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], s));
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(out6 + c, lo[c]);
            atomicMax(out6 + 3 + c, hi[c]);
        }
    }
}

void launch_position_minmax(const float* params, int64_t cap, int n, float* out6, cudaStream_t st) {
    unsigned int init[6] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0u, 0u, 0u};
    cudaMemcpyAsync(out6, init, sizeof(init), cudaMemcpyHostToDevice, st);
    if (n > 0)
        position_minmax_kernel<<<std::min(div_up(n, 256), 148 * 4), 256, 0, st>>>(
            params, cap, n, reinterpret_cast<unsigned int*>(out6));
}

__global__ void to_hwc_kernel(const float* __restrict__ planes, int P, int channels, double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P * channels) return;
    const int p = i / channels, c = i % channels;
    out[i] = planes[static_cast<size_t>(c) * P + p];
}

void launch_to_hwc_double(const float* planes, int h, int w, int channels, double* out, cudaStream_t st) {
    const int total = h * w * channels;
    if (total > 0) to_hwc_kernel<<<div_up(total, 256), 256, 0, st>>>(planes, h * w, channels, out);
}

__global__ void from_hwc_kernel(const double* __restrict__ hwc, int P, int channels, float* __restrict__ planes) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P * channels) return;
    const int p = i / channels, c = i % channels;
    planes[static_cast<size_t>(c) * P + p] = static_cast<float>(hwc[i]);
}

void launch_from_hwc_double(const double* hwc, int h, int w, int channels, float* planes, cudaStream_t st) {
    const int total = h * w * channels;
    if (total > 0) from_hwc_kernel<<<div_up(total, 256), 256, 0, st>>>(hwc, h * w, channels, planes);
}

}  // namespace gsb
