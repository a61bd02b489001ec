// Shared device-side definitions for the gsmap_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

namespace gsb {

// Programmatic dependent launch along the training step's kernel chain: a kernel launched with
// launch_pdl first waits for its predecessor grid (griddepcontrol.wait: complete and its writes
// visible; a no-op for an ordinary launch), then lets its own dependent grid launch, so the
// next kernel's launch and CTA start-up overlap this one's work and tail. Only a kernel whose
// predecessor on the stream is a kernel (not a memset or copy) is launched this way.
#ifndef GSB_PDL
#define GSB_PDL 1
#endif
__device__ __forceinline__ void pdl_enter() {
#if GSB_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, Args... args) {
#if GSB_PDL
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
#else
    kernel<<<grid, block, 0, st>>>(static_cast<KArgs>(args)...);
    return cudaGetLastError();
#endif
}

// Device-side bounds assertions, compiled in only by the checked build (diag/build_variant.sh
// checked -DGSB_CHECKS): compute-sanitizer is closed on this GPU pool, so the index invariants
// of the hot kernels are asserted in-kernel instead and the GPU suite runs against that build.
#ifdef GSB_CHECKS
#define GSB_CHECK(cond)                                                                   \
    do {                                                                                  \
        if (!(cond)) {                                                                    \
            printf("GSB_CHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, \
                   static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x), #cond);   \
            __trap();                                                                     \
        }                                                                                 \
    } while (0)
#else
#define GSB_CHECK(cond) \
    do {                \
    } while (0)
#endif

constexpr int kTile = 16;                 // rasterizer.hpp:17 kTileSize
constexpr int kTileThreads = kTile * kTile;
constexpr double kNearClip = 0.01;        // projection.hpp:11
constexpr double kCovReg = 0.3;           // projection.hpp:12
constexpr float kAlphaMaxF = 0.99f;       // rasterizer.hpp:18 (fp32 compare)
constexpr double kAlphaMaxD = 0.99;       // rasterizer.hpp:18 (fp64 transmittance update)
constexpr double kTMin = 1e-4;            // rasterizer.hpp:19
constexpr int kNumParams = 59;            // gaussian.hpp:16-26 flattened
constexpr int kGeomParams = 11;           // position 3, rotation 4, log_scale 3, opacity 1
constexpr int kNumPartials = 10;          // per (tile, gaussian) backward partial sums
constexpr uint32_t kDepthKeyBase = 0x3C23D70Au;  // fp32 bits of 0.01f (visible depths are >= it)
constexpr int kDepthKeyBits = 24;

// Parameter planes ([59][capacity], fp32): same order as the reference's Gaussian3D.
enum Plane : int { P_POS = 0, P_ROT = 3, P_LS = 7, P_OP = 10, P_SH = 11 };

// 64-byte projected-Gaussian record, rank (depth) ordered after the sort. Everything the
// blend kernels need, fetched as 4 x 16 B.
struct __align__(16) Splat {
    double mx, my;           // fp64 image-plane mean (pixels)
    float ca, cb, cc;        // conic = inverse(cov2d) (00, 01, 11), rounded to fp32
    float opacity;           // sigmoid(opacity_logit)
    float r, g, b;           // SH colour clamped to [0, 1]
    float depth;             // camera-frame z
    int16_t x0, y0, x1, y1;  // clamped integer pixel rect (inclusive) = the per-pixel box test
    int32_t gid;             // map index
    uint32_t ntiles;         // tiles the rect touches (0 when the rect is empty)
};
static_assert(sizeof(Splat) == 64, "Splat must be 64 bytes");

// Per-view camera + pose in fp64, passed by value to kernels.
struct ViewParams {
    double qw, qx, qy, qz, tx, ty, tz;  // normalised q_cw, t_cw
    double fx, fy, cx, cy;
    int width, height, tiles_x, tiles_y;
};

struct LossScalars {       // device-side loss accumulators (fp64) for one compute_loss call
    double l1_sum;         // sum |C - I|
    double sq_sum;         // sum (C - I)^2   (psnr)
    double ssim_sum;       // sum of SSIM map values over valid windows and channels
    double depth_abs_sum;  // sum |D/V - gt| over valid pixels
    unsigned long long n_valid;
    float depth_scale;     // lambda_d / n_valid (written by finalize, read by blend_bwd)
    float pad;
};

// Per-frame device counters (u64). The step is enqueued without reading them on the host:
// kernels take their element counts from here, and the pair buffers are sized by a
// per-resolution capacity; a render whose pair count exceeds it raises kCntOverflow, every
// consumer (blend_bwd, preprocess_bwd, adam) then does nothing, and the host re-runs the step.
enum Counter : int { kCntVisible = 0, kCntPairs = 1, kCntCand = 2, kCntOverflow = 3, kNumCounters = 4 };

__device__ __forceinline__ bool overflowed(const unsigned long long* cnt) {
    return cnt != nullptr && *(volatile const unsigned long long*)(cnt + kCntOverflow) != 0ull;
}

__host__ __device__ inline int div_up(int a, int b) { return (a + b - 1) / b; }

}  // namespace gsb
