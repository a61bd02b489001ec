// K6: pyramid-level loss (compute_loss, mapper.cpp:146-212) — L1 + SSIM (metrics.cpp:82-161)
// + masked LiDAR depth on D/V — and the keyframe pyramid (mapper.cpp:65-144).
// Images are fp32 planes; all scalar reductions are fp64.
#include "common.cuh"
#include "kernels.cuh"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace gsb {

namespace {
// metrics.cpp:20-30: the normalised 11-tap Gaussian (sigma 1.5), exp(-d^2 / 4.5) / sum in fp64,
// rounded to fp32. A static initialiser: every device gets it when the module loads (a runtime
// cudaMemcpyToSymbol would reach only the device current at the first call).
__constant__ float c_taps[11] = {1.028380124e-03f, 7.598758209e-03f, 3.600077331e-02f, 1.093606874e-01f,
                                 2.130055428e-01f, 2.660117149e-01f, 2.130055428e-01f, 1.093606874e-01f,
                                 3.600077331e-02f, 7.598758209e-03f, 1.028380124e-03f};

// host check that the literals are the reference's taps (once per process)
void ensure_taps() {
    static const bool ok = [] {
        double g[11], sum = 0.0;
        for (int i = 0; i < 11; ++i) {
            const double d = i - 5;
            g[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
            sum += g[i];
        }
        const float lit[11] = {1.028380124e-03f, 7.598758209e-03f, 3.600077331e-02f, 1.093606874e-01f,
                               2.130055428e-01f, 2.660117149e-01f, 2.130055428e-01f, 1.093606874e-01f,
                               3.600077331e-02f, 7.598758209e-03f, 1.028380124e-03f};
        for (int i = 0; i < 11; ++i)
            if (static_cast<float>(g[i] / sum) != lit[i]) return false;
        return true;
    }();
    if (!ok) throw std::logic_error("ssim: tap table differs from metrics.cpp's window");
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic reductions: every block stores its total (a fixed butterfly over the warp, then
// over the warps) in its own slot of the frame's loss buffer, and loss_finalize_kernel sums the
// slots in a fixed order — no atomics, so the loss and psnr are bitwise reproducible run to run
// (the reference's are for a fixed thread count, test_rasterizer.cpp:137-176).
// Slot layout after the LossScalars header: field f, block b at slots[f * stride + b].
__device__ __forceinline__ int linear_block() {
    return static_cast<int>(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z));
}
__device__ __forceinline__ double* slot_base(LossScalars* acc) { return reinterpret_cast<double*>(acc + 1); }

// block of 256 threads: its sum of v (all threads call it) into slot b of field f
__device__ __forceinline__ void block_store(double v, LossScalars* acc, int f, int stride, int b, double* scratch) {
    v = warp_sum(v);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double t = lane < (blockDim.x >> 5) ? scratch[lane] : 0.0;
        t = warp_sum(t);
        if (lane == 0) slot_base(acc)[f * stride + b] = t;
    }
    __syncthreads();
}

__device__ __forceinline__ float sgnf(double d) { return d > 0.0 ? 1.f : (d < 0.0 ? -1.f : 0.f); }
}  // namespace

// L1 (+psnr MSE) on colour and the masked depth residual (mapper.cpp:156-208). Writes the L1
// part of dL/dC and sign(r)/V for depth (scaled by lambda_d / n_valid in blend_bwd).
__global__ void __launch_bounds__(256) loss_pixel_kernel(
    const float* __restrict__ color, const float* __restrict__ depth, const float* __restrict__ vis,
    const float* __restrict__ gt_color, const float* __restrict__ gt_depth, int P, float l1_grad,
    float* __restrict__ dl_dcolor, float* __restrict__ depth_cot, LossScalars* __restrict__ acc, int stride) {
    __shared__ double scratch[8];
    double l1 = 0.0, sq = 0.0, dabs = 0.0;
    unsigned long long nv = 0;
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double d = static_cast<double>(color[c * P + p]) - static_cast<double>(gt_color[c * P + p]);
            l1 += fabs(d);
            sq += d * d;
            dl_dcolor[c * P + p] = sgnf(d) * l1_grad;
        }
        const double gd = gt_depth[p];
        const double v = vis[p];
        float cot = 0.f;
        if (gd > 0.0 && v > 0.98) {  // kDepthLossMinVisibility (mapper.hpp:15)
            const double r = static_cast<double>(depth[p]) / v - gd;
            dabs += fabs(r);
            ++nv;
            cot = static_cast<float>(sgnf(r) / v);
        }
        depth_cot[p] = cot;
    }
    const int b = linear_block();
    block_store(l1, acc, kLossL1, stride, b, scratch);
    block_store(sq, acc, kLossSq, stride, b, scratch);
    block_store(dabs, acc, kLossDabs, stride, b, scratch);
    block_store(static_cast<double>(nv), acc, kLossNv, stride, b, scratch);
}

namespace {
int pixel_blocks(int P) { return std::min(div_up(P, 256), 148 * 8); }
}  // namespace

size_t loss_buffer_bytes(int h, int w) {
    return sizeof(LossScalars) + sizeof(double) * kLossFields * static_cast<size_t>(loss_slot_stride(h, w));
}

LossLayout launch_loss_pixel(const float* color, const float* depth, const float* vis, const float* gt_color,
                             const float* gt_depth, int h, int w, double lambda, float* dl_dcolor,
                             float* depth_cot, LossScalars* acc, cudaStream_t st) {
    const int P = h * w;
    const float l1_grad = static_cast<float>((1.0 / (static_cast<double>(h) * w * 3)) * (1.0 - lambda));
    const int blocks = pixel_blocks(P);
    LossLayout L{};
    L.stride = loss_slot_stride(h, w);
    loss_pixel_kernel<<<blocks, 256, 0, st>>>(color, depth, vis, gt_color, gt_depth, P, l1_grad, dl_dcolor,
                                              depth_cot, acc, L.stride);
    L.n[kLossL1] = L.n[kLossSq] = L.n[kLossDabs] = L.n[kLossNv] = blocks;
    return L;
}

// ---------------------------------------------------------------------------------- SSIM
// Tiles of 32x32 valid-window outputs, separable 11-tap passes through shared memory with
// register blocking (a thread slides its window over 4 consecutive outputs, so each staged
// value is read once per 4 outputs instead of once per tap). Moments use values shifted by
// 0.5 (variance and covariance are shift invariant) to cut fp32 cancellation in
// E[a^2] - mu^2; the gradient weights are re-expressed for the shifted moments.
constexpr int kSx = 32, kSy = 32, kHalo = 10, kRB = 4;  // kRB outputs per thread and pass
constexpr int kInX = kSx + kHalo, kInY = kSy + kHalo;   // 42 x 42 staged inputs
constexpr float kShift = 0.5f;

__global__ void __launch_bounds__(256) ssim_fwd_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                       int h, int w, float inv_n, float* __restrict__ wbuf,
                                                       LossScalars* __restrict__ acc, int stride) {
    pdl_enter();
    __shared__ float sa[kInY][kInX + 2], sb[kInY][kInX + 2];
    __shared__ float hs[5][kInY][kSx + 1];
    __shared__ double scratch[8];
    const int c = blockIdx.z;
    const int x0 = blockIdx.x * kSx, y0 = blockIdx.y * kSy;
    const int vh = h - kHalo, vw = w - kHalo;
    const size_t P = static_cast<size_t>(h) * w;
    const float* Ac = A + c * P;
    const float* Bc = B + c * P;
    for (int i = threadIdx.x; i < kInY * kInX; i += blockDim.x) {
        const int r = i / kInX, q = i % kInX;
        const int gy = y0 + r, gx = x0 + q;
        const bool ok = gy < h && gx < w;
        sa[r][q] = ok ? Ac[static_cast<size_t>(gy) * w + gx] - kShift : 0.f;
        sb[r][q] = ok ? Bc[static_cast<size_t>(gy) * w + gx] - kShift : 0.f;
    }
    __syncthreads();
    // horizontal: item = (row r, 4 consecutive output columns)
    for (int it = threadIdx.x; it < kInY * (kSx / kRB); it += blockDim.x) {
        const int r = it / (kSx / kRB), q0 = (it % (kSx / kRB)) * kRB;
        float va[kRB + 10], vb[kRB + 10];
#pragma unroll
        for (int l = 0; l < kRB + 10; ++l) {
            va[l] = sa[r][q0 + l];
            vb[l] = sb[r][q0 + l];
        }
#pragma unroll
        for (int o = 0; o < kRB; ++o) {
            float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f, m4 = 0.f;
#pragma unroll
            for (int l = 0; l < 11; ++l) {
                const float g = c_taps[l], a = va[o + l], b = vb[o + l];
                const float ga = g * a;
                m0 = fmaf(g, a, m0);
                m1 = fmaf(g, b, m1);
                m2 = fmaf(ga, a, m2);
                m3 = fmaf(g * b, b, m3);
                m4 = fmaf(ga, b, m4);
            }
            hs[0][r][q0 + o] = m0; hs[1][r][q0 + o] = m1; hs[2][r][q0 + o] = m2;
            hs[3][r][q0 + o] = m3; hs[4][r][q0 + o] = m4;
        }
    }
    __syncthreads();
    // vertical: item = (column q, 4 consecutive output rows) -> 256 items
    double ssum = 0.0;
    {
        const int q = threadIdx.x % kSx, r0 = (threadIdx.x / kSx) * kRB;
        float m[kRB][5];
#pragma unroll
        for (int o = 0; o < kRB; ++o)
#pragma unroll
            for (int t = 0; t < 5; ++t) m[o][t] = 0.f;
#pragma unroll
        for (int l = 0; l < kRB + 10; ++l) {
            float hv[5];
#pragma unroll
            for (int t = 0; t < 5; ++t) hv[t] = hs[t][r0 + l][q];
#pragma unroll
            for (int o = 0; o < kRB; ++o) {
                const int k = l - o;
                if (k < 0 || k > 10) continue;
                const float g = c_taps[k];
#pragma unroll
                for (int t = 0; t < 5; ++t) m[o][t] = fmaf(g, hv[t], m[o][t]);
            }
        }
        const size_t VP = static_cast<size_t>(vh) * vw;
        float* wc = wbuf + static_cast<size_t>(c) * 3 * VP;
        const int ox = x0 + q;
#pragma unroll
        for (int o = 0; o < kRB; ++o) {
            const int oy = y0 + r0 + o;
            if (oy >= vh || ox >= vw) continue;
            const float mas = m[o][0], mbs = m[o][1];  // shifted means
            const float ma = mas + kShift, mb = mbs + kShift;
            const float va = m[o][2] - mas * mas, vb = m[o][3] - mbs * mbs, cab = m[o][4] - mas * mbs;
            const float C1 = 1e-4f, C2 = 9e-4f;
            const float num1 = 2.f * ma * mb + C1, num2 = 2.f * cab + C2;
            const float den1 = ma * ma + mb * mb + C1, den2 = va + vb + C2;
            const float inv_dd = 1.f / (den1 * den2);
            const float s = num1 * num2 * inv_dd;
            ssum += s;
            const float ds_dsab = 2.f * num1 * inv_dd;
            const float ds_dsa = -s / den2;
            const float ds_dmu_direct = 2.f * mb * num2 * inv_dd - s * 2.f * ma / den1;
            const float ds_dmu = ds_dmu_direct + ds_dsa * (-2.f * mas) + ds_dsab * (-mbs);
            const size_t oo = static_cast<size_t>(oy) * vw + ox;
            wc[oo] = ds_dmu * inv_n;
            wc[VP + oo] = ds_dsa * inv_n;
            wc[2 * VP + oo] = ds_dsab * inv_n;
        }
    }
    block_store(ssum, acc, kLossSsim, stride, linear_block(), scratch);
}

// Adjoint of the valid correlation (metrics.cpp:55-73) for the three weight maps, combined as
// d/da = adj(w_mu) + 2 a' adj(w_a2) + b' adj(w_ab), then dL/dC += -lambda * d.
// PixelLoss: the per-pixel L1 / psnr / masked-depth terms of loss_pixel_kernel, fused here when
// SSIM runs (this kernel visits every pixel of every channel once with colour and target in
// hand): dL/dC = sign(C - I) l1_grad - lambda dSSIM is written without a read-modify-write.
struct PixelLoss {
    const float* depth;
    const float* vis;
    const float* gt_depth;
    float* depth_cot;
    float l1_grad;
    LossScalars* acc;
    int stride;
};

template <bool FUSED>
__global__ void __launch_bounds__(256) ssim_bwd_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                       int h, int w, const float* __restrict__ wbuf,
                                                       float neg_lambda, float* __restrict__ dl, PixelLoss pl) {
    pdl_enter();
    __shared__ float sw[3][kInY][kInX + 2];
    __shared__ float hx[3][kInY][kSx + 1];
    const int c = blockIdx.z;
    const int x0 = blockIdx.x * kSx, y0 = blockIdx.y * kSy;
    const int vh = h - kHalo, vw = w - kHalo;
    const size_t VP = static_cast<size_t>(vh) * vw;
    const float* wc = wbuf + static_cast<size_t>(c) * 3 * VP;
    for (int i = threadIdx.x; i < kInY * kInX; i += blockDim.x) {
        const int r = i / kInX, q = i % kInX;
        const int gy = y0 - kHalo + r, gx = x0 - kHalo + q;
        const bool ok = gy >= 0 && gx >= 0 && gy < vh && gx < vw;
        const size_t o = static_cast<size_t>(gy) * vw + gx;
        sw[0][r][q] = ok ? wc[o] : 0.f;
        sw[1][r][q] = ok ? wc[VP + o] : 0.f;
        sw[2][r][q] = ok ? wc[2 * VP + o] : 0.f;
    }
    __syncthreads();
    // horizontal adjoint: out[q] = sum_l g[l] w[q + 10 - l]
    for (int it = threadIdx.x; it < kInY * (kSx / kRB); it += blockDim.x) {
        const int r = it / (kSx / kRB), q0 = (it % (kSx / kRB)) * kRB;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            float vw_[kRB + 10];
#pragma unroll
            for (int l = 0; l < kRB + 10; ++l) vw_[l] = sw[t][r][q0 + l];
#pragma unroll
            for (int o = 0; o < kRB; ++o) {
                float a = 0.f;
#pragma unroll
                for (int l = 0; l < 11; ++l) a = fmaf(c_taps[l], vw_[o + kHalo - l], a);
                hx[t][r][q0 + o] = a;
            }
        }
    }
    __syncthreads();
    const int q = threadIdx.x % kSx, r0 = (threadIdx.x / kSx) * kRB;
    float bsum[kRB][3];
#pragma unroll
    for (int o = 0; o < kRB; ++o)
#pragma unroll
        for (int t = 0; t < 3; ++t) bsum[o][t] = 0.f;
#pragma unroll
    for (int l = 0; l < kRB + 10; ++l) {  // staged row r0 + l feeds output row r0 + o with tap 10 - (l - o)
        float hv[3];
#pragma unroll
        for (int t = 0; t < 3; ++t) hv[t] = hx[t][r0 + l][q];
#pragma unroll
        for (int o = 0; o < kRB; ++o) {
            const int k = kHalo - (l - o);
            if (k < 0 || k > 10) continue;
            const float g = c_taps[k];
#pragma unroll
            for (int t = 0; t < 3; ++t) bsum[o][t] = fmaf(g, hv[t], bsum[o][t]);
        }
    }
    const size_t P = static_cast<size_t>(h) * w;
    const int x = x0 + q;
    double l1 = 0.0, sq = 0.0, dabs = 0.0;
    unsigned long long nv = 0;
#pragma unroll
    for (int o = 0; o < kRB; ++o) {
        const int y = y0 + r0 + o;
        if (y >= h || x >= w) continue;
        const size_t p = c * P + static_cast<size_t>(y) * w + x;
        const float av = A[p], bv = B[p];
        const float as = av - kShift, bs = bv - kShift;
        const float d = bsum[o][0] + 2.f * as * bsum[o][1] + bs * bsum[o][2];
        if (FUSED) {  // loss_pixel_kernel's terms for this pixel and channel
            const double e = static_cast<double>(av) - static_cast<double>(bv);
            l1 += fabs(e);
            sq += e * e;
            dl[p] = fmaf(neg_lambda, d, sgnf(e) * pl.l1_grad);
            if (c == 0) {
                const size_t o2 = static_cast<size_t>(y) * w + x;
                const double gd = pl.gt_depth[o2];
                const double vv = pl.vis[o2];
                float cot = 0.f;
                if (gd > 0.0 && vv > 0.98) {  // kDepthLossMinVisibility (mapper.hpp:15)
                    const double r = static_cast<double>(pl.depth[o2]) / vv - gd;
                    dabs += fabs(r);
                    ++nv;
                    cot = static_cast<float>(sgnf(r) / vv);
                }
                pl.depth_cot[o2] = cot;
            }
        } else {
            dl[p] = fmaf(neg_lambda, d, dl[p]);
        }
    }
    if (FUSED) {
        __shared__ double scratch[8];
        const int b = linear_block();
        block_store(l1, pl.acc, kLossL1, pl.stride, b, scratch);
        block_store(sq, pl.acc, kLossSq, pl.stride, b, scratch);
        if (c == 0) {  // depth terms from the channel-0 blocks: slots [0, gridDim.x * gridDim.y)
            block_store(dabs, pl.acc, kLossDabs, pl.stride, b, scratch);
            block_store(static_cast<double>(nv), pl.acc, kLossNv, pl.stride, b, scratch);
        }
    }
}

LossLayout launch_ssim(const float* color, const float* gt_color, int h, int w, double lambda, float* wbuf,
                       float* dl_dcolor, LossScalars* acc, const float* depth, const float* vis,
                       const float* gt_depth, float* depth_cot, cudaStream_t st) {
    ensure_taps();
    LossLayout L{};
    L.stride = loss_slot_stride(h, w);
    const int vh = h - kHalo, vw = w - kHalo;
    const float inv_n = static_cast<float>(1.0 / (static_cast<double>(vh) * vw * 3));
    dim3 gf(div_up(vw, kSx), div_up(vh, kSy), 3);
    launch_pdl(ssim_fwd_kernel, gf, 256, st, color, gt_color, h, w, inv_n, wbuf, acc, L.stride);
    L.n[kLossSsim] = static_cast<int>(gf.x * gf.y * gf.z);
    dim3 gb(div_up(w, kSx), div_up(h, kSy), 3);
    if (depth) {  // fused pixel loss (loss_pixel_kernel is not launched)
        PixelLoss pl{depth, vis, gt_depth, depth_cot,
                     static_cast<float>((1.0 / (static_cast<double>(h) * w * 3)) * (1.0 - lambda)), acc, L.stride};
        launch_pdl(ssim_bwd_kernel<true>, gb, 256, st, color, gt_color, h, w, wbuf, static_cast<float>(-lambda), dl_dcolor,
                                                   pl);
        L.n[kLossL1] = L.n[kLossSq] = static_cast<int>(gb.x * gb.y * gb.z);
        L.n[kLossDabs] = L.n[kLossNv] = static_cast<int>(gb.x * gb.y);
    } else {
        launch_pdl(ssim_bwd_kernel<false>, gb, 256, st, color, gt_color, h, w, wbuf, static_cast<float>(-lambda),
                                                    dl_dcolor, PixelLoss{});
    }
    return L;
}

int loss_slot_stride(int h, int w) {
    const int fwd = h > kHalo && w > kHalo ? div_up(w - kHalo, kSx) * div_up(h - kHalo, kSy) * 3 : 0;
    const int bwd = div_up(w, kSx) * div_up(h, kSy) * 3;
    return std::max({pixel_blocks(h * w), fwd, bwd, 1});
}

// ---------------------------------------------------------------------------- evaluation
// evaluate_sequence (pipeline.cpp:41-64) per view: quantize_8bit of the render (pipeline.cpp:
// 34-39: lround(clamp(c, 0, 1) * 255) / 255), psnr's squared error (metrics.cpp:165-175) and
// depth_rmse over gt > 0 (metrics.cpp:183-197). The quantized planes feed the SSIM forward.
__global__ void __launch_bounds__(256) eval_pixel_kernel(
    const float* __restrict__ color, const float* __restrict__ depth, const float* __restrict__ gt_color,
    const float* __restrict__ gt_depth, int P, float* __restrict__ quant, LossScalars* __restrict__ acc, int stride) {
    __shared__ double scratch[8];
    double sq = 0.0, dsq = 0.0;
    unsigned long long nv = 0;
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double x = fmin(fmax(static_cast<double>(color[c * P + p]), 0.0), 1.0);
            const double q = static_cast<double>(llround(x * 255.0)) / 255.0;
            quant[c * P + p] = static_cast<float>(q);
            const double d = q - static_cast<double>(gt_color[c * P + p]);
            sq += d * d;
        }
        if (gt_depth) {
            const double gd = gt_depth[p];
            if (gd > 0.0) {
                const double d = static_cast<double>(depth[p]) - gd;
                dsq += d * d;
                ++nv;
            }
        }
    }
    const int b = linear_block();
    block_store(sq, acc, kLossSq, stride, b, scratch);
    block_store(dsq, acc, kLossDabs, stride, b, scratch);
    block_store(static_cast<double>(nv), acc, kLossNv, stride, b, scratch);
}

LossLayout launch_eval(const float* color, const float* depth, const float* gt_color, const float* gt_depth, int h,
                       int w, float* quant, float* wbuf, LossScalars* acc, cudaStream_t st) {
    const int P = h * w;
    LossLayout L{};
    L.stride = loss_slot_stride(h, w);
    const int blocks = pixel_blocks(P);
    eval_pixel_kernel<<<blocks, 256, 0, st>>>(color, depth, gt_color, gt_depth, P, quant, acc, L.stride);
    L.n[kLossSq] = L.n[kLossDabs] = L.n[kLossNv] = blocks;
    if (h >= 11 && w >= 11) {
        ensure_taps();
        const int vh = h - kHalo, vw = w - kHalo;
        const float inv_n = static_cast<float>(1.0 / (static_cast<double>(vh) * vw * 3));
        dim3 gf(div_up(vw, kSx), div_up(vh, kSy), 3);
        ssim_fwd_kernel<<<gf, 256, 0, st>>>(quant, gt_color, h, w, inv_n, wbuf, acc, L.stride);
        L.n[kLossSsim] = static_cast<int>(gf.x * gf.y * gf.z);
    }
    return L;
}

// Sums every field's block slots in a fixed order (thread t takes slots t, t + T, ... in turn,
// the five fields' loads of one slot index issued together; then a fixed tree over the lanes and
// a fixed sum over the warps) into the LossScalars header; then depth_scale. One block of 1024
// threads: ~4 dependent round trips at full resolution instead of ~75.
constexpr int kFinalizeThreads = 1024;

__global__ void __launch_bounds__(kFinalizeThreads) loss_finalize_kernel(LossScalars* acc, LossLayout L,
                                                                          double lambda_d) {
    pdl_enter();
    __shared__ double scratch[kLossFields][kFinalizeThreads / 32];
    const double* slots = slot_base(acc);
    int nmax = 0;
#pragma unroll
    for (int f = 0; f < kLossFields; ++f) nmax = max(nmax, L.n[f]);
    double s[kLossFields];
#pragma unroll
    for (int f = 0; f < kLossFields; ++f) s[f] = 0.0;
    for (int b = threadIdx.x; b < nmax; b += kFinalizeThreads) {
        double v[kLossFields];
#pragma unroll
        for (int f = 0; f < kLossFields; ++f) v[f] = b < L.n[f] ? slots[f * L.stride + b] : 0.0;
#pragma unroll
        for (int f = 0; f < kLossFields; ++f) s[f] += v[f];
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int f = 0; f < kLossFields; ++f) {
        const double t = warp_sum(s[f]);
        if (lane == 0) scratch[f][warp] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot[kLossFields];
        for (int f = 0; f < kLossFields; ++f) {
            double t = 0.0;
            for (int w = 0; w < kFinalizeThreads / 32; ++w) t += scratch[f][w];
            tot[f] = t;
        }
        acc->l1_sum = tot[kLossL1];
        acc->sq_sum = tot[kLossSq];
        acc->ssim_sum = tot[kLossSsim];
        acc->depth_abs_sum = tot[kLossDabs];
        const unsigned long long n = static_cast<unsigned long long>(tot[kLossNv]);
        acc->n_valid = n;
        acc->depth_scale = n > 0 ? static_cast<float>(lambda_d / static_cast<double>(n)) : 0.f;
    }
}

void launch_loss_finalize(LossScalars* acc, const LossLayout& L, double lambda_d, cudaStream_t st) {
    launch_pdl(loss_finalize_kernel, 1, kFinalizeThreads, st, acc, L, lambda_d);
}

// ---------------------------------------------------------------------------------- pyramid
// mapper.cpp:65-110: 2x2 box average (partial blocks average what exists); depth averages only
// the valid (> 0) samples, 0 if none. Planes in, planes out.
__global__ void downsample_kernel(const float* __restrict__ in, int h, int w, int channels, int depth_mode,
                                  float* __restrict__ out) {
    const int oh = (h + 1) / 2, ow = (w + 1) / 2;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= oh * ow * channels) return;
    const int c = i / (oh * ow), rem = i % (oh * ow), y = rem / ow, x = rem % ow;
    double sum = 0.0;
    int n = 0;
    for (int dy = 0; dy < 2; ++dy)
        for (int dx = 0; dx < 2; ++dx) {
            const int sy = 2 * y + dy, sx = 2 * x + dx;
            if (sy < h && sx < w) {
                const float v = in[static_cast<size_t>(c) * h * w + static_cast<size_t>(sy) * w + sx];
                if (!depth_mode || v > 0.f) {
                    sum += v;
                    ++n;
                }
            }
        }
    out[i] = n ? static_cast<float>(sum / n) : 0.f;
}

void launch_downsample(const float* in, int h, int w, int channels, bool depth, float* out, cudaStream_t st) {
    const int total = ((h + 1) / 2) * ((w + 1) / 2) * channels;
    downsample_kernel<<<div_up(total, 256), 256, 0, st>>>(in, h, w, channels, depth ? 1 : 0, out);
}

}  // namespace gsb
