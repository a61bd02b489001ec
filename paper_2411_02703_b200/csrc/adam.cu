// K9 fused Adam over the Gaussian SoA (GaussianMap::apply_gradients, gaussian_map.cpp:37-54),
// the scene-extent reduction (refresh_extent, gaussian_map.cpp:87-99) and host-layout converters.
#include <cfloat>

#include "common.cuh"
#include "kernels.cuh"

namespace gsb {

// One thread per Gaussian; every Gaussian steps (its counter increments even when unseen, so
// momentum keeps moving it, as in the reference). The per-Gaussian bias corrections are fp64;
// the per-scalar update is fp32 on fp32 m/v. Inactive SH coefficients are skipped: their m, v
// and gradient are exactly zero, so the reference's update there is -lr*0/(0+eps) = -0 (exact).
namespace {
struct AdamArgs {
    float lr[5];        // position (x scene_extent), rotation, log_scale, opacity, sh
    int32_t t_common;   // the new step of every Gaussian present since the last append
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
                                                   float* __restrict__ v, int32_t* __restrict__ step,
                                                   const int8_t* __restrict__ degree,
                                                   const float* __restrict__ grads, int64_t gcap, int64_t cap, int n,
                                                   AdamArgs args, const unsigned long long* __restrict__ cnt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || overflowed(cnt)) return;
    const int t = step[i] + 1;
    step[i] = t;
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

// Four consecutive Gaussians per thread with 16-byte loads and stores (every plane base is
// 16-byte aligned when both capacities are multiples of 4). Same per-scalar arithmetic as
// adam_kernel; SH coefficients past a Gaussian's degree are left untouched exactly as there.
__device__ __forceinline__ void adam_vec(float4* __restrict__ p, float4* __restrict__ m, float4* __restrict__ v,
                                         float4 g, float lr, const float (&a)[4], const float (&b)[4], int live) {
    float4 P = *p, Mv = *m, V = *v;
    float* pp = &P.x;
    float* mm = &Mv.x;
    float* vv = &V.x;
    const float* gg = &g.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        if (!((live >> e) & 1)) continue;
        adam_scalar(pp + e, mm + e, vv + e, gg[e], lr, a[e], b[e]);
    }
    *p = P;
    *m = Mv;
    *v = V;
}

__global__ void __launch_bounds__(256) adam4_kernel(float* __restrict__ params, float* __restrict__ m,
                                                    float* __restrict__ v, int32_t* __restrict__ step,
                                                    const int8_t* __restrict__ degree,
                                                    const float* __restrict__ grads, int64_t gcap, int64_t cap, int n,
                                                    AdamArgs args, const unsigned long long* __restrict__ cnt) {
    const int i = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (i >= n || overflowed(cnt)) return;
    const int ne = min(4, n - i);
    const int all = (1 << ne) - 1;
    int4 t4 = *reinterpret_cast<const int4*>(step + i);
    int* tt = &t4.x;
    float a[4], b[4];
    int deg[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        a[e] = args.a_common;
        b[e] = args.b_common;
        deg[e] = -1;
        if (e < ne) {
            const int t = tt[e] + 1;
            tt[e] = t;
            deg[e] = degree[i + e];
            if (t != args.t_common) {
                a[e] = static_cast<float>(1.0 / (1.0 - pow(0.9, static_cast<double>(t))));
                b[e] = static_cast<float>(1.0 / (1.0 - pow(0.999, static_cast<double>(t))));
            }
        }
    }
    *reinterpret_cast<int4*>(step + i) = t4;  // step entries past n are never read
    float4 g[kGeomParams];
#pragma unroll
    for (int k = 0; k < kGeomParams; ++k) g[k] = __ldg(reinterpret_cast<const float4*>(grads + k * gcap + i));
#pragma unroll
    for (int k = 0; k < kGeomParams; ++k) {
        const float lr = k < 3 ? args.lr[0] : k < 7 ? args.lr[1] : k < 10 ? args.lr[2] : args.lr[3];
        const int64_t o = k * cap + i;
        adam_vec(reinterpret_cast<float4*>(params + o), reinterpret_cast<float4*>(m + o),
                 reinterpret_cast<float4*>(v + o), g[k], lr, a, b, all);
    }
    const int dmax = max(max(deg[0], deg[1]), max(deg[2], deg[3]));
    const int ncoef = (dmax + 1) * (dmax + 1);
    for (int c = 0; c < ncoef; ++c) {
        int live = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) live |= ((deg[e] + 1) * (deg[e] + 1) > c) << e;
        float4 gs[3];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch)
            gs[ch] = __ldg(reinterpret_cast<const float4*>(grads + (P_SH + 3 * c + ch) * gcap + i));
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            const int64_t o = (P_SH + 3 * c + ch) * cap + i;
            adam_vec(reinterpret_cast<float4*>(params + o), reinterpret_cast<float4*>(m + o),
                     reinterpret_cast<float4*>(v + o), gs[ch], args.lr[4], a, b, live);
        }
    }
}

void launch_adam(float* params, float* m, float* v, int32_t* step, const int8_t* degree, const float* grads,
                 int64_t gcap, int64_t cap, int n, const double lr[5], double scene_extent, int64_t t_common,
                 const unsigned long long* cnt, cudaStream_t st) {
    if (n <= 0) return;
    AdamArgs args;
    args.lr[0] = static_cast<float>(lr[0] * scene_extent);
    for (int k = 1; k < 5; ++k) args.lr[k] = static_cast<float>(lr[k]);
    args.t_common = static_cast<int32_t>(t_common);
    args.a_common = static_cast<float>(1.0 / (1.0 - std::pow(0.9, static_cast<double>(t_common))));
    args.b_common = static_cast<float>(1.0 / (1.0 - std::pow(0.999, static_cast<double>(t_common))));
    if (cap % 4 == 0 && gcap % 4 == 0)
        adam4_kernel<<<div_up(div_up(n, 4), 256), 256, 0, st>>>(params, m, v, step, degree, grads, gcap, cap, n, args,
                                                                 cnt);
    else
        adam_kernel<<<div_up(n, 256), 256, 0, st>>>(params, m, v, step, degree, grads, gcap, cap, n, args, cnt);
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
