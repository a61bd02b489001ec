// K6: pyramid-level loss (compute_loss, mapper.cpp:146-212) — L1 + SSIM (metrics.cpp:82-161)
// + masked LiDAR depth on D/V — and the keyframe pyramid (mapper.cpp:65-144).
// Images are fp32 planes; all scalar reductions are fp64.
#include "common.cuh"
#include "kernels.cuh"

namespace gsb {

namespace {
__constant__ float c_taps[11];  // metrics.cpp:20-30, normalised 11-tap Gaussian, sigma 1.5
bool g_taps_ready = false;

void ensure_taps() {
    if (g_taps_ready) return;
    double g[11], sum = 0.0;
    for (int i = 0; i < 11; ++i) {
        const double d = i - 5;
        g[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
        sum += g[i];
    }
    float f[11];
    for (int i = 0; i < 11; ++i) f[i] = static_cast<float>(g[i] / sum);
    cudaMemcpyToSymbol(c_taps, f, sizeof(f));
    g_taps_ready = true;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// block of 256 threads: sum a double into *dst with one atomic per block
__device__ __forceinline__ void block_add(double v, double* dst, double* scratch) {
    v = warp_sum(v);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double t = lane < (blockDim.x >> 5) ? scratch[lane] : 0.0;
        t = warp_sum(t);
        if (lane == 0 && t != 0.0) atomicAdd(dst, t);
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
    float* __restrict__ dl_dcolor, float* __restrict__ depth_cot, LossScalars* __restrict__ acc) {
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
    block_add(l1, &acc->l1_sum, scratch);
    block_add(sq, &acc->sq_sum, scratch);
    block_add(dabs, &acc->depth_abs_sum, scratch);
    nv = warp_sum(nv);
    if ((threadIdx.x & 31) == 0 && nv) atomicAdd(&acc->n_valid, nv);
}

void launch_loss_pixel(const float* color, const float* depth, const float* vis, const float* gt_color,
                       const float* gt_depth, int h, int w, double lambda, float* dl_dcolor,
                       float* depth_cot, LossScalars* acc, cudaStream_t st) {
    const int P = h * w;
    const float l1_grad = static_cast<float>((1.0 / (static_cast<double>(h) * w * 3)) * (1.0 - lambda));
    const int blocks = std::min(div_up(P, 256), 148 * 8);
    loss_pixel_kernel<<<blocks, 256, 0, st>>>(color, depth, vis, gt_color, gt_depth, P, l1_grad, dl_dcolor,
                                              depth_cot, acc);
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
                                                       LossScalars* __restrict__ acc) {
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
    block_add(ssum, &acc->ssim_sum, scratch);
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
};

template <bool FUSED>
__global__ void __launch_bounds__(256) ssim_bwd_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                       int h, int w, const float* __restrict__ wbuf,
                                                       float neg_lambda, float* __restrict__ dl, PixelLoss pl) {
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
        block_add(l1, &pl.acc->l1_sum, scratch);
        block_add(sq, &pl.acc->sq_sum, scratch);
        if (c == 0) {
            block_add(dabs, &pl.acc->depth_abs_sum, scratch);
            nv = warp_sum(nv);
            if ((threadIdx.x & 31) == 0 && nv) atomicAdd(&pl.acc->n_valid, nv);
        }
    }
}

void launch_ssim(const float* color, const float* gt_color, int h, int w, double lambda, float* wbuf,
                 float* dl_dcolor, LossScalars* acc, const float* depth, const float* vis, const float* gt_depth,
                 float* depth_cot, cudaStream_t st) {
    ensure_taps();
    const int vh = h - kHalo, vw = w - kHalo;
    const float inv_n = static_cast<float>(1.0 / (static_cast<double>(vh) * vw * 3));
    dim3 gf(div_up(vw, kSx), div_up(vh, kSy), 3);
    ssim_fwd_kernel<<<gf, 256, 0, st>>>(color, gt_color, h, w, inv_n, wbuf, acc);
    dim3 gb(div_up(w, kSx), div_up(h, kSy), 3);
    if (depth) {  // fused pixel loss (loss_pixel_kernel is not launched)
        PixelLoss pl{depth, vis, gt_depth, depth_cot,
                     static_cast<float>((1.0 / (static_cast<double>(h) * w * 3)) * (1.0 - lambda)), acc};
        ssim_bwd_kernel<true><<<gb, 256, 0, st>>>(color, gt_color, h, w, wbuf, static_cast<float>(-lambda), dl_dcolor,
                                                   pl);
    } else {
        ssim_bwd_kernel<false><<<gb, 256, 0, st>>>(color, gt_color, h, w, wbuf, static_cast<float>(-lambda),
                                                    dl_dcolor, PixelLoss{});
    }
}

// ---------------------------------------------------------------------------- evaluation
// evaluate_sequence (pipeline.cpp:41-64) per view: quantize_8bit of the render (pipeline.cpp:
// 34-39: lround(clamp(c, 0, 1) * 255) / 255), psnr's squared error (metrics.cpp:165-175) and
// depth_rmse over gt > 0 (metrics.cpp:183-197). The quantized planes feed the SSIM forward.
__global__ void __launch_bounds__(256) eval_pixel_kernel(
    const float* __restrict__ color, const float* __restrict__ depth, const float* __restrict__ gt_color,
    const float* __restrict__ gt_depth, int P, float* __restrict__ quant, LossScalars* __restrict__ acc) {
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
    block_add(sq, &acc->sq_sum, scratch);
    block_add(dsq, &acc->depth_abs_sum, scratch);
    nv = warp_sum(nv);
    if ((threadIdx.x & 31) == 0 && nv) atomicAdd(&acc->n_valid, nv);
}

void launch_eval(const float* color, const float* depth, const float* gt_color, const float* gt_depth, int h, int w,
                 float* quant, float* wbuf, LossScalars* acc, cudaStream_t st) {
    const int P = h * w;
    eval_pixel_kernel<<<std::min(div_up(P, 256), 148 * 8), 256, 0, st>>>(color, depth, gt_color, gt_depth, P, quant,
                                                                         acc);
    if (h >= 11 && w >= 11) {
        ensure_taps();
        const int vh = h - kHalo, vw = w - kHalo;
        const float inv_n = static_cast<float>(1.0 / (static_cast<double>(vh) * vw * 3));
        dim3 gf(div_up(vw, kSx), div_up(vh, kSy), 3);
        ssim_fwd_kernel<<<gf, 256, 0, st>>>(quant, gt_color, h, w, inv_n, wbuf, acc);
    }
}

__global__ void loss_finalize_kernel(LossScalars* acc, double lambda_d) {
    const unsigned long long n = acc->n_valid;
    acc->depth_scale = n > 0 ? static_cast<float>(lambda_d / static_cast<double>(n)) : 0.f;
}

void launch_loss_finalize(LossScalars* acc, double lambda_d, cudaStream_t st) {
    loss_finalize_kernel<<<1, 1, 0, st>>>(acc, lambda_d);
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
