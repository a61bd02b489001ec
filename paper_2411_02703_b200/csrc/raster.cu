// Tile binning (K2-K4 glue), front-to-back blend (K5), reverse blend (K7) and the on-request
// CSR materialisation. One 256-thread CTA per 16x16 tile; each warp owns an 8x4 pixel block.
#include "common.cuh"
#include "kernels.cuh"

namespace gsb {

namespace {

// Staged copy of one tile-list entry in shared memory (SoA to keep the broadcast reads of a
// warp conflict-free). Means are rebased to the tile origin in fp64 before rounding to fp32,
// which keeps ~1e-6 px precision at any image coordinate.
struct StageSoA {
    float2 mean[kTileThreads];
    float4 cop[kTileThreads];   // conic a, b, c, opacity
    float4 col[kTileThreads];   // r, g, b, depth
    int4 rect[kTileThreads];    // x0, y0, x1, y1 (absolute pixel coordinates, inclusive)
};

// The per-contributor alpha, pinned to explicit round-to-nearest intrinsics so the forward, the
// backward replay and the CSR materialisation produce bit-identical values (contraction cannot
// differ between kernels). eval_gaussian_2d_conic (projection.cpp:80-84) + rasterizer.cpp:142-143.
struct AlphaEval {
    float dx, dy, u0, u1, g, a_raw, alpha;
};

__device__ __forceinline__ AlphaEval eval_alpha(float2 m, float4 cop, float fx, float fy) {
    AlphaEval e;
    e.dx = __fsub_rn(fx, m.x);
    e.dy = __fsub_rn(fy, m.y);
    e.u0 = __fmaf_rn(cop.y, e.dy, __fmul_rn(cop.x, e.dx));  // (Sigma^-1 d).x
    e.u1 = __fmaf_rn(cop.z, e.dy, __fmul_rn(cop.y, e.dx));  // (Sigma^-1 d).y
    const float q = __fmaf_rn(e.dy, e.u1, __fmul_rn(e.dx, e.u0));
    e.g = __expf(__fmul_rn(-0.5f, q));
    e.a_raw = __fmul_rn(cop.w, e.g);
    e.alpha = fminf(e.a_raw, kAlphaMaxF);
    return e;
}

// fp64 transmittance step: the clamp substitutes the exact double 0.99 so two stacked clamped
// splats leave T = (1 - 0.99)^2 = 1.0000000000000018e-4 (no termination), as in the fp64
// reference (rasterizer.cpp:143-151).
__device__ __forceinline__ double alpha_d(const AlphaEval& e) {
    return e.a_raw >= kAlphaMaxF ? kAlphaMaxD : static_cast<double>(e.alpha);
}

__device__ __forceinline__ void stage_entry(StageSoA& s, int t, const Splat& sp, double ox, double oy) {
    s.mean[t] = make_float2(static_cast<float>(sp.mx - ox), static_cast<float>(sp.my - oy));
    s.cop[t] = make_float4(sp.ca, sp.cb, sp.cc, sp.opacity);
    s.col[t] = make_float4(sp.r, sp.g, sp.b, sp.depth);
    s.rect[t] = make_int4(sp.x0, sp.y0, sp.x1, sp.y1);
}

__device__ __forceinline__ uint32_t emission_index(const Splat& sp, uint32_t off, int tx, int ty) {
    const int tx0 = sp.x0 >> 4, ty0 = sp.y0 >> 4;
    const int ntx = (sp.x1 >> 4) - tx0 + 1;
    return off + static_cast<uint32_t>((ty - ty0) * ntx + (tx - tx0));
}

__device__ __forceinline__ void pixel_of(int tiles_x, int& tx, int& ty, int& lx, int& ly) {
    const int tile = blockIdx.x;
    tx = tile % tiles_x;
    ty = tile / tiles_x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    lx = (warp & 1) * 8 + (lane & 7);
    ly = (warp >> 1) * 4 + (lane >> 3);
}

}  // namespace

// ------------------------------------------------------------------------------------------ glue
__global__ void gather_keys_kernel(const int32_t* __restrict__ vis_gid,
                                   const unsigned long long* __restrict__ key_by_gid, int n,
                                   unsigned long long* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = key_by_gid[vis_gid[i]];
}

void launch_gather_keys(const int32_t* vis_gid, const unsigned long long* key_by_gid, int n,
                        unsigned long long* out, cudaStream_t st) {
    if (n > 0) gather_keys_kernel<<<div_up(n, 256), 256, 0, st>>>(vis_gid, key_by_gid, n, out);
}

// rank-ordered copy of the projected records (the reference's sorted `projected` vector)
__global__ void pack_kernel(const int32_t* __restrict__ gid_sorted, const Splat* __restrict__ rec_by_gid,
                            int n, Splat* __restrict__ rec_sorted, uint32_t* __restrict__ ntiles) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const Splat s = rec_by_gid[gid_sorted[r]];
    rec_sorted[r] = s;
    ntiles[r] = s.ntiles;
}

void launch_pack(const int32_t* gid_sorted, const Splat* rec_by_gid, int n, Splat* rec_sorted,
                 uint32_t* ntiles, cudaStream_t st) {
    if (n > 0) pack_kernel<<<div_up(n, 256), 256, 0, st>>>(gid_sorted, rec_by_gid, n, rec_sorted, ntiles);
}

// Duplicate-key emission (bin_tiles, rasterizer.cpp:76-91): one thread per (gaussian, tile)
// pair, owner rank found by binary search over the exclusive scan of tile counts. Keys are
// tile ids; values are depth ranks, so a stable sort by tile yields each tile's list in
// (depth, index) order, exactly the reference's push_back order.
__global__ void emit_pairs_kernel(const uint32_t* __restrict__ emit_off, const Splat* __restrict__ rec,
                                  int n_vis, uint32_t n_pairs, int tiles_x, uint32_t* __restrict__ keys,
                                  uint32_t* __restrict__ vals) {
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n_pairs) return;
    int lo = 0, hi = n_vis;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(emit_off + mid) <= e) lo = mid; else hi = mid;
    }
    const int r = lo;
    const uint32_t l = e - __ldg(emit_off + r);
    const Splat& s = rec[r];
    const int tx0 = s.x0 >> 4, ty0 = s.y0 >> 4;
    const int ntx = (s.x1 >> 4) - tx0 + 1;
    const int ty = ty0 + static_cast<int>(l) / ntx, tx = tx0 + static_cast<int>(l) % ntx;
    keys[e] = static_cast<uint32_t>(ty * tiles_x + tx);
    vals[e] = static_cast<uint32_t>(r);
}

void launch_emit_pairs(const uint32_t* emit_off, const Splat* rec, int n_vis, uint32_t n_pairs, int tiles_x,
                       uint32_t* keys, uint32_t* vals, cudaStream_t st) {
    if (n_pairs > 0)
        emit_pairs_kernel<<<div_up(static_cast<int>(n_pairs), 256), 256, 0, st>>>(emit_off, rec, n_vis, n_pairs,
                                                                                 tiles_x, keys, vals);
}

__global__ void tile_ranges_kernel(const uint32_t* __restrict__ keys, uint32_t n, uint2* __restrict__ ranges) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t k = keys[i];
    if (i == 0 || keys[i - 1] != k) ranges[k].x = i;
    if (i == n - 1 || keys[i + 1] != k) ranges[k].y = i + 1;
}

void launch_tile_ranges(const uint32_t* keys, uint32_t n, uint2* ranges, cudaStream_t st) {
    if (n > 0) tile_ranges_kernel<<<div_up(static_cast<int>(n), 256), 256, 0, st>>>(keys, n, ranges);
}

// ------------------------------------------------------------------------------------------ K5
// Front-to-back blend (rasterizer.cpp:118-162). Box test = integer pixel rect; alpha clamped
// at 0.99; the contributor is accumulated BEFORE the T < 1e-4 break; V = sum of weights.
// Per pixel it keeps n_proc (list position + 1 of the last contributor) and fp32 T_final for
// the backward replay instead of the reference's CSR table (rasterizer.cpp:164-197).
__global__ void __launch_bounds__(kTileThreads) blend_fwd_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals, const Splat* __restrict__ rec,
    ViewParams v, float* __restrict__ out_color, float* __restrict__ out_depth, float* __restrict__ out_vis,
    float* __restrict__ out_t, int32_t* __restrict__ out_nproc, int32_t* __restrict__ out_ncontrib) {
    __shared__ StageSoA s;
    int tx, ty, lx, ly;
    pixel_of(v.tiles_x, tx, ty, lx, ly);
    const int px = tx * kTile + lx, py = ty * kTile + ly;
    const bool inside = px < v.width && py < v.height;
    const uint2 range = ranges[blockIdx.x];
    const double ox = tx * kTile, oy = ty * kTile;
    const float fx = static_cast<float>(lx), fy = static_cast<float>(ly);

    double T = 1.0;
    float c0 = 0.f, c1 = 0.f, c2 = 0.f, d = 0.f, vis = 0.f;
    int nproc = 0, ncontrib = 0;
    bool done = !inside;
    for (uint32_t base = range.x; base < range.y; base += kTileThreads) {
        if (__syncthreads_count(!done) == 0) break;
        const uint32_t idx = base + threadIdx.x;
        if (idx < range.y) stage_entry(s, threadIdx.x, rec[vals[idx]], ox, oy);
        __syncthreads();
        const int cnt = min(kTileThreads, static_cast<int>(range.y - base));
        if (!done) {
            for (int j = 0; j < cnt; ++j) {
                const int4 rc = s.rect[j];
                if (px < rc.x || px > rc.z || py < rc.y || py > rc.w) continue;
                const AlphaEval e = eval_alpha(s.mean[j], s.cop[j], fx, fy);
                const float4 col = s.col[j];
                const float w = e.alpha * static_cast<float>(T);
                c0 = fmaf(w, col.x, c0);
                c1 = fmaf(w, col.y, c1);
                c2 = fmaf(w, col.z, c2);
                d = fmaf(w, col.w, d);
                vis += w;
                ++ncontrib;
                nproc = static_cast<int>(base - range.x) + j + 1;
                T = __dmul_rn(T, __dadd_rn(1.0, -alpha_d(e)));
                if (T < kTMin) {
                    done = true;
                    break;
                }
            }
        }
    }
    if (inside) {
        const size_t p = static_cast<size_t>(py) * v.width + px;
        const size_t P = static_cast<size_t>(v.width) * v.height;
        out_color[p] = c0;
        out_color[P + p] = c1;
        out_color[2 * P + p] = c2;
        out_depth[p] = d;
        out_vis[p] = vis;
        out_t[p] = static_cast<float>(T);
        out_nproc[p] = nproc;
        out_ncontrib[p] = ncontrib;
    }
}

void launch_blend_fwd(const uint2* ranges, const uint32_t* vals, const Splat* rec, const ViewParams& v,
                      float* color, float* depth, float* vis, float* t_final, int32_t* n_proc,
                      int32_t* n_contrib, cudaStream_t st) {
    const int n_tiles = v.tiles_x * v.tiles_y;
    blend_fwd_kernel<<<n_tiles, kTileThreads, 0, st>>>(ranges, vals, rec, v, color, depth, vis, t_final,
                                                       n_proc, n_contrib);
}

// ------------------------------------------------------------------------------------------ K7
// Reverse replay (rasterizer.cpp:253-315): per pixel, walk its contributors back to front,
// reconstructing T_i = T_{i+1} / (1 - alpha_i) from the forward's T_final, accumulating the
// colour/depth suffix sums. Each (tile, gaussian) pair's 10 cotangent sums are reduced in the
// warp by shuffles, across the CTA's 8 warps in shared memory, and written once to its
// emission slot -- deterministic, no global atomics; K8 sums a Gaussian's slots in fp64.
constexpr int kBwdBatch = 32;

struct BwdShared {
    float2 mean[kBwdBatch];
    float4 cop[kBwdBatch];
    float4 col[kBwdBatch];
    int4 rect[kBwdBatch];
    uint32_t slot[kBwdBatch];
    uint32_t mask[kTileThreads / 32];
    float red[kTileThreads / 32][kBwdBatch][kNumPartials];
    int max_last;
};

__global__ void __launch_bounds__(kTileThreads) blend_bwd_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals, const Splat* __restrict__ rec,
    const uint32_t* __restrict__ emit_off, ViewParams v, const float* __restrict__ t_final,
    const int32_t* __restrict__ n_proc, const float* __restrict__ dl_dcolor,
    const float* __restrict__ dl_ddepth, const float* __restrict__ depth_scale, float* __restrict__ partials) {
    __shared__ BwdShared s;
    int tx, ty, lx, ly;
    pixel_of(v.tiles_x, tx, ty, lx, ly);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int px = tx * kTile + lx, py = ty * kTile + ly;
    const bool inside = px < v.width && py < v.height;
    const uint2 range = ranges[blockIdx.x];
    const double ox = tx * kTile, oy = ty * kTile;
    const float fx = static_cast<float>(lx), fy = static_cast<float>(ly);
    // warp pixel block (for the warp-uniform rect cull)
    const int bx0 = tx * kTile + (warp & 1) * 8, by0 = ty * kTile + (warp >> 1) * 4;

    float T = 0.f, dc0 = 0.f, dc1 = 0.f, dc2 = 0.f, dd = 0.f;
    int last = 0;
    if (inside) {
        const size_t p = static_cast<size_t>(py) * v.width + px;
        const size_t P = static_cast<size_t>(v.width) * v.height;
        last = n_proc[p];
        T = t_final[p];
        dc0 = dl_dcolor[p];
        dc1 = dl_dcolor[P + p];
        dc2 = dl_dcolor[2 * P + p];
        dd = dl_ddepth ? dl_ddepth[p] * (depth_scale ? *depth_scale : 1.f) : 0.f;
        // rasterizer.cpp:264: a pixel with an all-zero cotangent contributes nothing
        if (dc0 == 0.f && dc1 == 0.f && dc2 == 0.f && dd == 0.f) last = 0;
    }
    if (threadIdx.x == 0) s.max_last = 0;
    __syncthreads();
    if (last > 0) atomicMax(&s.max_last, last);
    __syncthreads();
    const int max_last = s.max_last;
    const int n_list = static_cast<int>(range.y - range.x);

    // entries no pixel reached still own a partial slot: zero it
    for (int j = max_last + threadIdx.x; j < n_list; j += kTileThreads) {
        const uint32_t r = vals[range.x + j];
        const uint32_t slot = emission_index(rec[r], emit_off[r], tx, ty);
        float2* dst = reinterpret_cast<float2*>(partials + static_cast<size_t>(slot) * kNumPartials);
#pragma unroll
        for (int k = 0; k < kNumPartials / 2; ++k) dst[k] = make_float2(0.f, 0.f);
    }

    float sc0 = 0.f, sc1 = 0.f, sc2 = 0.f, sd = 0.f;
    for (int hi = max_last; hi > 0; hi -= kBwdBatch) {
        const int lo = max(0, hi - kBwdBatch);
        const int cnt = hi - lo;
        if (threadIdx.x < cnt) {
            const uint32_t r = vals[range.x + lo + threadIdx.x];
            const Splat sp = rec[r];
            s.mean[threadIdx.x] = make_float2(static_cast<float>(sp.mx - ox), static_cast<float>(sp.my - oy));
            s.cop[threadIdx.x] = make_float4(sp.ca, sp.cb, sp.cc, sp.opacity);
            s.col[threadIdx.x] = make_float4(sp.r, sp.g, sp.b, sp.depth);
            s.rect[threadIdx.x] = make_int4(sp.x0, sp.y0, sp.x1, sp.y1);
            s.slot[threadIdx.x] = emission_index(sp, emit_off[r], tx, ty);
        }
        if (lane == 0) s.mask[warp] = 0u;
        __syncthreads();
        for (int k = cnt - 1; k >= 0; --k) {
            const int j = lo + k;
            const int4 rc = s.rect[k];
            if (rc.x > bx0 + 7 || rc.z < bx0 || rc.y > by0 + 3 || rc.w < by0) continue;  // warp-uniform
            const bool act = j < last && px >= rc.x && px <= rc.z && py >= rc.y && py <= rc.w;
            if (!__any_sync(0xffffffffu, act)) continue;
            float g0 = 0.f, g1 = 0.f, g2 = 0.f, g3 = 0.f, g4 = 0.f, g5 = 0.f, g6 = 0.f, g7 = 0.f, g8 = 0.f, g9 = 0.f;
            if (act) {
                const float4 cop = s.cop[k];
                const AlphaEval e = eval_alpha(s.mean[k], cop, fx, fy);
                const float4 col = s.col[k];
                const float one_m = 1.f - e.alpha;
                const float inv = 1.f / one_m;
                const float ti = T * inv;
                const float w = e.alpha * ti;
                g0 = w * dc0;
                g1 = w * dc1;
                g2 = w * dc2;
                g3 = w * dd;
                const float dalpha = dc0 * (col.x * ti - sc0 * inv) + dc1 * (col.y * ti - sc1 * inv) +
                                     dc2 * (col.z * ti - sc2 * inv) + dd * (col.w * ti - sd * inv);
                sc0 = fmaf(w, col.x, sc0);
                sc1 = fmaf(w, col.y, sc1);
                sc2 = fmaf(w, col.z, sc2);
                sd = fmaf(w, col.w, sd);
                T = ti;
                if (e.a_raw < kAlphaMaxF) {  // rasterizer.cpp:297: the clamp is flat
                    g4 = dalpha * e.g;
                    const float sg = e.g * dalpha * cop.w;
                    g5 = sg * e.u0;
                    g6 = sg * e.u1;
                    const float hs = 0.5f * sg;
                    g7 = hs * e.u0 * e.u0;
                    g8 = hs * e.u0 * e.u1;
                    g9 = hs * e.u1 * e.u1;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                g0 += __shfl_xor_sync(0xffffffffu, g0, o);
                g1 += __shfl_xor_sync(0xffffffffu, g1, o);
                g2 += __shfl_xor_sync(0xffffffffu, g2, o);
                g3 += __shfl_xor_sync(0xffffffffu, g3, o);
                g4 += __shfl_xor_sync(0xffffffffu, g4, o);
                g5 += __shfl_xor_sync(0xffffffffu, g5, o);
                g6 += __shfl_xor_sync(0xffffffffu, g6, o);
                g7 += __shfl_xor_sync(0xffffffffu, g7, o);
                g8 += __shfl_xor_sync(0xffffffffu, g8, o);
                g9 += __shfl_xor_sync(0xffffffffu, g9, o);
            }
            if (lane == 0) {
                float* dst = s.red[warp][k];
                dst[0] = g0; dst[1] = g1; dst[2] = g2; dst[3] = g3; dst[4] = g4;
                dst[5] = g5; dst[6] = g6; dst[7] = g7; dst[8] = g8; dst[9] = g9;
                s.mask[warp] |= 1u << k;
            }
        }
        __syncthreads();
        for (int t = threadIdx.x; t < cnt * kNumPartials; t += kTileThreads) {
            const int k = t / kNumPartials, c = t - k * kNumPartials;
            float acc = 0.f;
#pragma unroll
            for (int w = 0; w < kTileThreads / 32; ++w)
                if (s.mask[w] & (1u << k)) acc += s.red[w][k][c];
            partials[static_cast<size_t>(s.slot[k]) * kNumPartials + c] = acc;
        }
        __syncthreads();
    }
}

void launch_blend_bwd(const uint2* ranges, const uint32_t* vals, const Splat* rec, const uint32_t* emit_off,
                      const ViewParams& v, const float* t_final, const int32_t* n_proc,
                      const float* dl_dcolor, const float* dl_ddepth, const float* depth_scale,
                      float* partials, cudaStream_t st) {
    const int n_tiles = v.tiles_x * v.tiles_y;
    blend_bwd_kernel<<<n_tiles, kTileThreads, 0, st>>>(ranges, vals, rec, emit_off, v, t_final, n_proc,
                                                       dl_dcolor, dl_ddepth, depth_scale, partials);
}

// ------------------------------------------------------------------------------------------ CSR
// RenderOutput::contribs materialised on request (tests, gradcheck): one thread per pixel
// replays the forward with the same alpha / fp64-T arithmetic, writing (map index, alpha).
__global__ void materialize_kernel(const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals,
                                   const Splat* __restrict__ rec, ViewParams v, const uint32_t* __restrict__ offsets,
                                   int32_t* __restrict__ out_gid, double* __restrict__ out_alpha) {
    int tx, ty, lx, ly;
    pixel_of(v.tiles_x, tx, ty, lx, ly);
    const int px = tx * kTile + lx, py = ty * kTile + ly;
    if (px >= v.width || py >= v.height) return;
    const uint2 range = ranges[blockIdx.x];
    const double ox = tx * kTile, oy = ty * kTile;
    const size_t p = static_cast<size_t>(py) * v.width + px;
    uint32_t w = offsets[p];
    double T = 1.0;
    for (uint32_t idx = range.x; idx < range.y; ++idx) {
        const Splat sp = rec[vals[idx]];
        if (px < sp.x0 || px > sp.x1 || py < sp.y0 || py > sp.y1) continue;
        const float2 m = make_float2(static_cast<float>(sp.mx - ox), static_cast<float>(sp.my - oy));
        const AlphaEval e = eval_alpha(m, make_float4(sp.ca, sp.cb, sp.cc, sp.opacity), static_cast<float>(lx),
                                       static_cast<float>(ly));
        const double ad = alpha_d(e);
        out_gid[w] = sp.gid;
        out_alpha[w] = ad;
        ++w;
        T = __dmul_rn(T, __dadd_rn(1.0, -ad));
        if (T < kTMin) break;
    }
}

void launch_materialize(const uint2* ranges, const uint32_t* vals, const Splat* rec, const ViewParams& v,
                        const uint32_t* offsets, int32_t* out_gid, double* out_alpha, cudaStream_t st) {
    const int n_tiles = v.tiles_x * v.tiles_y;
    materialize_kernel<<<n_tiles, kTileThreads, 0, st>>>(ranges, vals, rec, v, offsets, out_gid, out_alpha);
}

}  // namespace gsb
