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
__global__ void __launch_bounds__(256) adam_kernel(float* __restrict__ params, float* __restrict__ m,
                                                   float* __restrict__ v, int32_t* __restrict__ step,
                                                   const int8_t* __restrict__ degree,
                                                   const float* __restrict__ grads, int64_t gcap, int64_t cap, int n,
                                                   float lr_pos, float lr_rot, float lr_ls, float lr_op,
                                                   float lr_sh) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int t = step[i] + 1;
    step[i] = t;
    const double bc1 = 1.0 - pow(0.9, static_cast<double>(t));
    const double bc2 = 1.0 - pow(0.999, static_cast<double>(t));
    const float a = static_cast<float>(1.0 / bc1);
    const float b = static_cast<float>(1.0 / bc2);
    const int deg = degree[i];
    const int nk = kGeomParams + 3 * (deg + 1) * (deg + 1);
    for (int k = 0; k < nk; ++k) {
        const float lr = k < 3 ? lr_pos : k < 7 ? lr_rot : k < 10 ? lr_ls : k < 11 ? lr_op : lr_sh;
        const size_t o = static_cast<size_t>(k) * cap + i;
        const float g = grads[static_cast<size_t>(k) * gcap + i];
        const float mk = fmaf(0.9f, m[o], 0.1f * g);
        const float vk = fmaf(0.999f, v[o], 0.001f * g * g);
        m[o] = mk;
        v[o] = vk;
        params[o] += -lr * (mk * a) / (sqrtf(vk * b) + 1e-15f);
    }
}

void launch_adam(float* params, float* m, float* v, int32_t* step, const int8_t* degree, const float* grads,
                 int64_t gcap, int64_t cap, int n, const double lr[5], double scene_extent, cudaStream_t st) {
    if (n <= 0) return;
    adam_kernel<<<div_up(n, 256), 256, 0, st>>>(params, m, v, step, degree, grads, gcap, cap, n,
                                                static_cast<float>(lr[0] * scene_extent), static_cast<float>(lr[1]),
                                                static_cast<float>(lr[2]), static_cast<float>(lr[3]),
                                                static_cast<float>(lr[4]));
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
