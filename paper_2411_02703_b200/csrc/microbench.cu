// Roofline denominators for the non-tensor kernels, measured on the box: FP32 FMA issue rate
// and MUFU.EX2 rate (MEASURED_PEAKS.json carries only HBM copy bandwidth and bf16 GEMM).
#include "../../include/gsmap_b200.h"
#include "common.cuh"

namespace gsb {

__global__ void __launch_bounds__(256) fma_peak_kernel(float* out, int iters) {
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-7f + k;
    const float b = 0.9999999f, c = 1e-7f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], b, c);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 12345.f) out[threadIdx.x] = s;  // keep the chains live
}

__global__ void __launch_bounds__(256) ex2_peak_kernel(float* out, int iters) {
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = -1e-3f * (threadIdx.x + k);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            float r;
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a[k]));
            a[k] = -r;
        }
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 12345.f) out[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) dfma_peak_kernel(float* out, int iters) {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-7 + k;
    const double b = 0.9999999, c = 1e-7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 12345.0) out[threadIdx.x] = static_cast<float>(s);
}

// f32 -> f64 -> f32 round trips (2 conversions per op counted as 1 "op")
__global__ void __launch_bounds__(256) f2f_peak_kernel(float* out, int iters) {
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-7f + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            double d = static_cast<double>(a[k]);
            asm volatile("" : "+d"(d));
            a[k] = static_cast<float>(d) * 0.9999999f;
        }
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 12345.f) out[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) shfl_peak_kernel(float* out, int iters) {
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-7f + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = __shfl_xor_sync(0xffffffffu, a[k], 1 + (k & 15));
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 12345.f) out[threadIdx.x] = s;
}

}  // namespace gsb

extern "C" int gs_microbench(int device, int kind, double* per_second) {
    using namespace gsb;
    if (cudaSetDevice(device) != cudaSuccess) return GS_ECUDA;
    float* out = nullptr;
    if (cudaMalloc(&out, 1024) != cudaSuccess) return GS_ECUDA;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int blocks = sms * 8, threads = 256, iters = kind == 0 ? 1 << 15 : 1 << 13;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a);
        if (kind == 0)
            fma_peak_kernel<<<blocks, threads>>>(out, iters);
        else if (kind == 1)
            ex2_peak_kernel<<<blocks, threads>>>(out, iters);
        else if (kind == 2)
            dfma_peak_kernel<<<blocks, threads>>>(out, iters);
        else if (kind == 3)
            f2f_peak_kernel<<<blocks, threads>>>(out, iters);
        else
            shfl_peak_kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        if (rep > 0) best = ms < best ? ms : best;
    }
    const double ops = static_cast<double>(blocks) * threads * iters * 8 * (kind == 0 || kind == 2 ? 2.0 : 1.0);
    *per_second = ops / (best * 1e-3);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    return cudaGetLastError() == cudaSuccess ? GS_OK : GS_ECUDA;
}
