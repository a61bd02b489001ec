// Shared device helpers of the blend kernels (forward, backward, CSR materialisation).
//
// Blend layout: one CTA per 16x16 tile with 256/PPT threads; each thread owns a vertical strip
// of PPT pixels (warp w: rows w*2*PPT .. +2*PPT-1; lane l: column l&15, rows +PPT*(l>>4)+p).
// Pixels are processed in vertically adjacent pairs with packed FP32x2 arithmetic (FFMA2 /
// FMUL2 / FADD2 on sm_100a), which halves the issue slots of the per-contributor math.
#pragma once

#include "common.cuh"

namespace gsb {

// exp(-q/2) = 2^(k q) with k = -log2(e)/2 folded into the staged conic.
constexpr float kExpScale = -0.72134752044448170368f;

__device__ __forceinline__ float ex2(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }

// Staged form of one tile-list entry. The mean is rebased to the tile origin in fp64 and then
// rounded (keeps ~1e-6 px precision anywhere in the image); the conic carries the exp2 scale.
struct Staged {
    float2 mean;
    float4 con;  // k*a, k*b, k*c, opacity
    float4 col;  // r, g, b, depth
    int4 rect;   // x0, y0, x1, y1 (absolute, inclusive)
};

__device__ __forceinline__ Staged stage_of(const Splat& sp, double ox, double oy) {
    Staged s;
    s.mean = make_float2(static_cast<float>(sp.mx - ox), static_cast<float>(sp.my - oy));
    s.con = make_float4(__fmul_rn(sp.ca, kExpScale), __fmul_rn(sp.cb, kExpScale), __fmul_rn(sp.cc, kExpScale),
                        sp.opacity);
    s.col = make_float4(sp.r, sp.g, sp.b, sp.depth);
    s.rect = make_int4(sp.x0, sp.y0, sp.x1, sp.y1);
    return s;
}

template <int N>
struct StageBuf {
    float2 mean[N];
    float4 con[N];
    float4 col[N];
    int4 rect[N];
    __device__ __forceinline__ void put(int t, const Staged& s) {
        mean[t] = s.mean;
        con[t] = s.con;
        col[t] = s.col;
        rect[t] = s.rect;
    }
};

// Per-contributor alpha (eval_gaussian_2d_conic, projection.cpp:80-84, and the 0.99 clamp,
// rasterizer.cpp:142-143). Every operation is an explicit round-to-nearest intrinsic, and the
// packed pair version performs the identical sequence lane by lane, so the forward, the
// backward replay and the CSR materialisation see bit-identical alphas.
struct AlphaS {
    float u0, u1, g, a_raw, alpha;
};

__device__ __forceinline__ AlphaS alpha_scalar(float2 m, float4 cn, float fx, float fy) {
    const float dx = __fadd_rn(fx, -m.x), dy = __fadd_rn(fy, -m.y);
    AlphaS a;
    a.u0 = __fmaf_rn(cn.y, dy, __fmul_rn(cn.x, dx));
    a.u1 = __fmaf_rn(cn.z, dy, __fmul_rn(cn.y, dx));
    const float q = __fmaf_rn(dy, a.u1, __fmul_rn(dx, a.u0));
    a.g = ex2(q);
    a.a_raw = __fmul_rn(cn.w, a.g);
    a.alpha = fminf(a.a_raw, kAlphaMaxF);
    return a;
}

struct AlphaP {
    float2 u0, u1, g, a_raw, alpha;
};

// CLAMP = false: the entry's opacity is below 0.99f, so o * g (g <= 1) never reaches the clamp
// and alpha = a_raw exactly (the blends pick the variant per entry, warp-uniformly)
template <bool CLAMP = true>
__device__ __forceinline__ AlphaP alpha_pair(float2 m, float4 cn, float fx, float2 fy) {
    const float dx = __fadd_rn(fx, -m.x);
    const float2 dy = __fadd2_rn(fy, f2(-m.y));
    const float adx = __fmul_rn(cn.x, dx), bdx = __fmul_rn(cn.y, dx);
    AlphaP a;
    a.u0 = __ffma2_rn(f2(cn.y), dy, f2(adx));
    a.u1 = __ffma2_rn(f2(cn.z), dy, f2(bdx));
    const float2 q = __ffma2_rn(dy, a.u1, __fmul2_rn(f2(dx), a.u0));
    a.g = make_float2(ex2(q.x), ex2(q.y));
    a.a_raw = __fmul2_rn(f2(cn.w), a.g);
    a.alpha = CLAMP ? make_float2(fminf(a.a_raw.x, kAlphaMaxF), fminf(a.a_raw.y, kAlphaMaxF)) : a.a_raw;
    return a;
}

// The same with a per-pixel opacity pair (the forward masks stopped pixels by opacity 0):
// op = cn.w * 1 is cn.w exactly, so a live pixel's alpha is bit-identical to alpha_pair's.
template <bool CLAMP = true>
__device__ __forceinline__ AlphaP alpha_pair_op(float2 m, float4 cn, float2 op, float fx, float2 fy) {
    const float dx = __fadd_rn(fx, -m.x);
    const float2 dy = __fadd2_rn(fy, f2(-m.y));
    const float adx = __fmul_rn(cn.x, dx), bdx = __fmul_rn(cn.y, dx);
    AlphaP a;
    a.u0 = __ffma2_rn(f2(cn.y), dy, f2(adx));
    a.u1 = __ffma2_rn(f2(cn.z), dy, f2(bdx));
    const float2 q = __ffma2_rn(dy, a.u1, __fmul2_rn(f2(dx), a.u0));
    a.g = make_float2(ex2(q.x), ex2(q.y));
    a.a_raw = __fmul2_rn(op, a.g);
    a.alpha = CLAMP ? make_float2(fminf(a.a_raw.x, kAlphaMaxF), fminf(a.a_raw.y, kAlphaMaxF)) : a.a_raw;
    return a;
}

// 64-byte record copy global -> shared without staging registers (cp.async, L2 only): the
// blends prefetch the next batch's records this way while walking the current one
__device__ __forceinline__ void cp_async_splat(Splat* dst, const Splat* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    const char* g = reinterpret_cast<const char*>(src);
#pragma unroll
    for (int i = 0; i < 4; ++i)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + 16 * i), "l"(g + 16 * i) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// fp64 transmittance factor (1 - alpha): the clamp substitutes the exact double 0.99, so two
// stacked clamped splats leave T = (1 - 0.99)^2 = 1.0000000000000018e-4 (no termination),
// exactly as the fp64 reference (rasterizer.cpp:143-151).
__device__ __forceinline__ double one_minus_alpha_d(float a_raw, float alpha) {
    return __dadd_rn(1.0, -(a_raw >= kAlphaMaxF ? kAlphaMaxD : static_cast<double>(alpha)));
}

__device__ __forceinline__ uint32_t emission_index(const Splat& sp, uint32_t off, int tx, int ty) {
    const int tx0 = sp.x0 >> 4, ty0 = sp.y0 >> 4;
    const int ntx = (sp.x1 >> 4) - tx0 + 1;
    return off + static_cast<uint32_t>((ty - ty0) * ntx + (tx - tx0));
}

// Each warp owns a compact kBW x kBH block of its tile (8x8 quadrants at PPT = 2, 8x16 halves
// at PPT = 4, 8x4 at PPT = 1, the whole tile at PPT = 8); lane l owns column l % kBW and the
// PPT rows starting at (l / kBW) * PPT.
template <int PPT>
struct Strip {
    static constexpr int kThreads = kTileThreads / PPT;
    static constexpr int kBW = PPT == 8 ? 16 : 8;
    static constexpr int kBH = 32 * PPT / kBW;
    static constexpr int kWarpsPerRow = kTile / kBW;
    int tx, ty, warp, lane, lx, ly0, px, py0, bx0, by0;
    __device__ __forceinline__ Strip(int tiles_x) : Strip(tiles_x, blockIdx.x, threadIdx.x >> 5) {}
    // tile `tile`, warp `w` of the tile's kThreads / 32 (a tile may be split over several CTAs)
    __device__ __forceinline__ Strip(int tiles_x, int tile, int w) {
        tx = tile % tiles_x;
        ty = tile / tiles_x;
        warp = w;
        lane = threadIdx.x & 31;
        const int wx = (warp % kWarpsPerRow) * kBW, wy = (warp / kWarpsPerRow) * kBH;
        lx = wx + lane % kBW;
        ly0 = wy + (lane / kBW) * PPT;
        px = tx * kTile + lx;
        py0 = ty * kTile + ly0;
        bx0 = tx * kTile + wx;
        by0 = ty * kTile + wy;
    }
    // the warp's block intersects the integer rect (x0, y0, x1, y1)
    __device__ __forceinline__ bool touches(const int4& rc) const {
        return !(rc.x > bx0 + kBW - 1 || rc.z < bx0 || rc.y > by0 + kBH - 1 || rc.w < by0);
    }
};

// Bounding box (x0, y0, x1, y1) of the warp's pixels flagged in `bits` (bit p = row py0 + p of
// this lane); empty (x0 > x1) when no lane has one. Entries whose rect misses it cannot touch
// any of those pixels, so the warp's ballot skips them: as pixels terminate (forward) or before
// they start (backward), the walk shrinks to the entries that can still matter.
template <int PPT>
__device__ __forceinline__ int4 warp_bbox(unsigned bits, const Strip<PPT>& sc) {
    const bool any = bits != 0u;
    const int x0 = any ? sc.px : 0x7fffffff, x1 = any ? sc.px : -1;
    const int y0 = any ? sc.py0 + __ffs(bits) - 1 : 0x7fffffff, y1 = any ? sc.py0 + 31 - __clz(bits) : -1;
    return make_int4(__reduce_min_sync(0xffffffffu, x0), __reduce_min_sync(0xffffffffu, y0),
                     __reduce_max_sync(0xffffffffu, x1), __reduce_max_sync(0xffffffffu, y1));
}

__device__ __forceinline__ bool rect_meets(const int4& rc, const int4& bb) {
    return !(rc.x > bb.z || rc.z < bb.x || rc.y > bb.w || rc.w < bb.y);
}

// Backward list segments. A tile's list is cut at multiples of L = seg_len(n, nseg) (a multiple
// of kSegAlign, itself a multiple of every forward staging batch); the forward stores each
// pixel's state before entry k L (k = 1 .. nseg - 1) as a checkpoint [k - 1][field][pixel] with
// fields T, C_r, C_g, C_b, D, and the backward runs one CTA per (tile, segment).
constexpr int kSegAlign = 256;
constexpr int kCkFields = 5;
__host__ __device__ inline int seg_len(int n_list, int nseg) {
    return nseg <= 1 ? n_list : div_up(div_up(n_list, nseg), kSegAlign) * kSegAlign;
}

// Tile launch order of the blends: tiles sorted by descending list length (longest first), so
// the longest tiles start in the first wave instead of forming the tail of the last one. The
// order sits behind the tile ranges in the same buffer (ranges[T], then order[T]).
#ifndef GSB_LPT
#define GSB_LPT 1
#endif
__host__ __device__ inline const uint32_t* tile_order(const uint2* ranges, int tiles) {
    return GSB_LPT ? reinterpret_cast<const uint32_t*>(ranges + tiles) : nullptr;
}
void launch_tile_order(const uint2* ranges, int tiles, cudaStream_t st);

// pixels-per-thread chosen per level (host override for experiments; 0 = automatic)
int blend_ppt(const ViewParams& v, bool backward);
// backward list segments per tile, chosen per level (host override; 0 = automatic)
int blend_segments(const ViewParams& v);

}  // namespace gsb
