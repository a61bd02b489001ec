// K5: front-to-back blend (rasterizer.cpp:118-162). Box test = integer pixel rect; alpha clamped
// at 0.99; the contributor is accumulated BEFORE the T < 1e-4 break; V = sum of weights. Per
// pixel it keeps n_proc (list position + 1 of the last contributor) and T_final for the
// backward instead of the reference's CSR table (rasterizer.cpp:164-197).
//
// Exact termination without fp64 arithmetic: the transmittance is carried as an unevaluated
// pair of floats (Th + Tl, "df32"). Each factor (1 - alpha) is split exactly (Fast2Sum) and the
// product uses the FMA-exact product error, so Th + Tl tracks the real product to ~2^-46 per
// step. The fp64 reference rounds by <= 2^-52 per step, so both decide T < 1e-4 identically
// unless T lies within ~k 2^-44 of the threshold; only then is the pixel replayed in fp64 with
// the reference's own operation order (never observed in practice; counted in g_blend_stats).
#include "blend_common.cuh"
#include "kernels.cuh"

namespace gsb {

__device__ unsigned long long g_blend_stats[2];  // [0] near-threshold checks, [1] fp64 replays

void read_blend_stats(unsigned long long out[2], bool reset) {
    cudaMemcpyFromSymbol(out, g_blend_stats, sizeof(unsigned long long) * 2);
    if (reset) {
        const unsigned long long z[2] = {0ull, 0ull};
        cudaMemcpyToSymbol(g_blend_stats, z, sizeof(z));
    }
}

namespace {

// 1 - 0.99 (fp64) = 0.010000000000000009 and 1e-4 (fp64) as exact float pairs
constexpr float kClampFacHi = 0.009999999776482582f, kClampFacLo = 2.2351742678949904e-10f;
constexpr float kTMinHi = 9.999999747378752e-05f, kTMinLo = 2.5262125290942405e-12f;
constexpr float kTNear = 1.0001e-4f;

// Exact fp64 transmittance of pixel (px, py) after the contributor at list position `upto`.
__device__ __noinline__ double replay_transmittance(const uint32_t* __restrict__ vals, const Splat* __restrict__ rec,
                                                     uint2 range, int upto, int px, int py, double ox, double oy,
                                                     float fx, float fy) {
    double T = 1.0;
    for (int j = 0; j <= upto; ++j) {
        const Splat sp = rec[vals[range.x + j]];
        if (px < sp.x0 || px > sp.x1 || py < sp.y0 || py > sp.y1) continue;
        const Staged s = stage_of(sp, ox, oy);
        const AlphaS e = alpha_scalar(s.mean, s.con, fx, fy);
        T = __dmul_rn(T, one_minus_alpha_d(e.a_raw, e.alpha));
    }
    return T;
}

}  // namespace

// Per-pixel blend state of one thread (NP packed pairs of vertically adjacent pixels).
template <int NP>
struct FwdState {
    float2 Th[NP], Tl[NP], c0[NP], c1[NP], c2[NP], dd[NP], vis[NP];
    int nproc[2 * NP], ncontrib[2 * NP];
    unsigned live;
};

// One tile-list entry over the thread's pixels. COVER: the entry's rect contains every live
// pixel of the warp (warp-uniform), so the per-pixel box test reduces to the live bits.
// STATS: maintain n_contrib (only the public render reports it).
template <int PPT, bool COVER, bool STATS>
__device__ __forceinline__ void fwd_entry(FwdState<(PPT + 1) / 2>& s, const Strip<PPT>& sc, const int4& rc,
                                          float2 m, float4 cn, float4 col, int pos, float fx,
                                          const uint32_t* __restrict__ vals, const Splat* __restrict__ rec,
                                          uint2 range, double ox, double oy) {
    constexpr int NP = (PPT + 1) / 2;
    const bool colin = COVER || (sc.px >= rc.x && sc.px <= rc.z);
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        const int p0 = 2 * q, y0 = sc.py0 + p0;
        bool a0 = (s.live >> p0) & 1u, a1 = (s.live >> (p0 + 1)) & 1u;
        if (!COVER) {
            a0 = a0 && colin && y0 >= rc.y && y0 <= rc.w;
            a1 = a1 && colin && y0 + 1 >= rc.y && y0 + 1 <= rc.w;
        }
        // no branch on (a0 || a1): an inactive half has al = 0 -> w = 0 and factor 1 + 0,
        // which leaves Th + Tl exactly unchanged (Fast2Sum renormalisation)
        const float fy = static_cast<float>(sc.ly0 + p0);
        const AlphaP e = alpha_pair(m, cn, fx, make_float2(fy, fy + 1.f));
        const float2 al = make_float2(a0 ? e.alpha.x : 0.f, a1 ? e.alpha.y : 0.f);
        const float2 w = __fmul2_rn(al, s.Th[q]);
        s.c0[q] = __ffma2_rn(w, f2(col.x), s.c0[q]);
        s.c1[q] = __ffma2_rn(w, f2(col.y), s.c1[q]);
        s.c2[q] = __ffma2_rn(w, f2(col.z), s.c2[q]);
        s.dd[q] = __ffma2_rn(w, f2(col.w), s.dd[q]);
        s.vis[q] = __fadd2_rn(s.vis[q], w);
        // exact factor 1 - alpha = fh + fl (Fast2Sum(1, -alpha)); clamp -> 1 - 0.99 (fp64)
        float2 fh = __fadd2_rn(f2(1.f), neg2(al));
        float2 fl = __fadd2_rn(neg2(al), neg2(__fadd2_rn(fh, f2(-1.f))));
        if (a0 && e.a_raw.x >= kAlphaMaxF) { fh.x = kClampFacHi; fl.x = kClampFacLo; }
        if (a1 && e.a_raw.y >= kAlphaMaxF) { fh.y = kClampFacHi; fl.y = kClampFacLo; }
        // (Th + Tl) * (fh + fl) with the exact product error of Th * fh
        const float2 pr = __fmul2_rn(s.Th[q], fh);
        const float2 er = __ffma2_rn(s.Th[q], fh, neg2(pr));
        const float2 t = __ffma2_rn(s.Th[q], fl, __ffma2_rn(s.Tl[q], fh, er));
        s.Th[q] = __fadd2_rn(pr, t);
        s.Tl[q] = __fadd2_rn(t, neg2(__fadd2_rn(s.Th[q], neg2(pr))));
        if (a0) s.nproc[p0] = pos + 1;
        if (a1) s.nproc[p0 + 1] = pos + 1;
        if (STATS) {
            s.ncontrib[p0] += a0;
            s.ncontrib[p0 + 1] += a1;
        }
        if ((a0 && s.Th[q].x < kTNear) || (a1 && s.Th[q].y < kTNear)) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int p = p0 + h;
                const float th = h ? s.Th[q].y : s.Th[q].x, tl = h ? s.Tl[q].y : s.Tl[q].x;
                if (!(h ? a1 : a0) || !(th < kTNear)) continue;
                atomicAdd(&g_blend_stats[0], 1ull);
                // sign of (Th + Tl) - 1e-4, with Th - kTMinHi exact (Sterbenz)
                const float d = __fadd_rn(th, -kTMinHi) + __fadd_rn(tl, -kTMinLo);
                const float tol = 1e-4f * 5.7e-14f * static_cast<float>(pos + 16);
                bool term = d < -tol;
                if (!(d < -tol) && !(d > tol)) {
                    atomicAdd(&g_blend_stats[1], 1ull);
                    term = replay_transmittance(vals, rec, range, pos, sc.px, sc.py0 + p, ox, oy, fx,
                                                static_cast<float>(sc.ly0 + p)) < kTMin;
                }
                if (term) s.live &= ~(1u << p);
            }
        }
    }
}

template <int PPT, bool STATS>
__global__ void __launch_bounds__(kTileThreads / PPT) blend_fwd_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals, const Splat* __restrict__ rec,
    ViewParams v, float* __restrict__ out_color, float* __restrict__ out_depth, float* __restrict__ out_vis,
    float* __restrict__ out_t, int32_t* __restrict__ out_nproc, int32_t* __restrict__ out_ncontrib) {
    using S = Strip<PPT>;
    // PPT = 1 runs one (real) pixel per lane in the low half of the pair; the high half is never
    // live, so its packed lane computes nothing that is kept.
    constexpr int NT = S::kThreads, NP = (PPT + 1) / 2;
    __shared__ StageBuf<NT> sb;
    const S sc(v.tiles_x);
    const uint2 range = ranges[blockIdx.x];
    const double ox = sc.tx * kTile, oy = sc.ty * kTile;
    const float fx = static_cast<float>(sc.lx);

    FwdState<NP> s;
    s.live = 0;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        s.Th[q] = f2(1.f);
        s.Tl[q] = s.c0[q] = s.c1[q] = s.c2[q] = s.dd[q] = s.vis[q] = f2(0.f);
    }
#pragma unroll
    for (int p = 0; p < 2 * NP; ++p) {
        s.nproc[p] = s.ncontrib[p] = 0;
        if (p < PPT && sc.px < v.width && sc.py0 + p < v.height) s.live |= 1u << p;
    }
    int4 lb = warp_bbox<PPT>(s.live, sc);
    unsigned seen = s.live;
    // the next batch's record is loaded one batch ahead (its latency overlaps the current walk)
    Splat nsp;
    if (range.x + threadIdx.x < range.y) nsp = rec[vals[range.x + threadIdx.x]];
    for (uint32_t base = range.x; base < range.y; base += NT) {
        if (__syncthreads_count(s.live != 0) == 0) break;
        const uint32_t idx = base + threadIdx.x;
        if (idx < range.y) sb.put(threadIdx.x, stage_of(nsp, ox, oy));
        if (idx + NT < range.y) nsp = rec[vals[idx + NT]];
        __syncthreads();
        const int cnt = min(NT, static_cast<int>(range.y - base));
        // the warp first ballots which staged entries meet the bounding box of its live pixels,
        // then walks only those (in list order)
        for (int b0 = 0; b0 < cnt; b0 += 32) {
            if (__any_sync(0xffffffffu, s.live != seen)) {
                seen = s.live;
                lb = warp_bbox<PPT>(s.live, sc);
            }
            if (lb.x > lb.z) break;  // no live pixel left in this warp
            const int jj = b0 + sc.lane;
            unsigned todo = __ballot_sync(0xffffffffu, jj < cnt && rect_meets(sb.rect[jj], lb));
            while (todo) {
                const int j = b0 + __ffs(todo) - 1;
                todo &= todo - 1;
                const int4 rc = sb.rect[j];
                const int pos = static_cast<int>(base - range.x) + j;
                if (rc.x <= lb.x && rc.z >= lb.z && rc.y <= lb.y && rc.w >= lb.w)
                    fwd_entry<PPT, true, STATS>(s, sc, rc, sb.mean[j], sb.con[j], sb.col[j], pos, fx, vals, rec,
                                                range, ox, oy);
                else
                    fwd_entry<PPT, false, STATS>(s, sc, rc, sb.mean[j], sb.con[j], sb.col[j], pos, fx, vals, rec,
                                                 range, ox, oy);
            }
        }
    }
    const size_t P = static_cast<size_t>(v.width) * v.height;
#pragma unroll
    for (int p = 0; p < PPT; ++p) {
        const int y = sc.py0 + p;
        if (sc.px >= v.width || y >= v.height) continue;
        const int q = p >> 1;
        const bool hi = p & 1;
        const size_t o = static_cast<size_t>(y) * v.width + sc.px;
        out_color[o] = hi ? s.c0[q].y : s.c0[q].x;
        out_color[P + o] = hi ? s.c1[q].y : s.c1[q].x;
        out_color[2 * P + o] = hi ? s.c2[q].y : s.c2[q].x;
        out_depth[o] = hi ? s.dd[q].y : s.dd[q].x;
        out_vis[o] = hi ? s.vis[q].y : s.vis[q].x;
        out_t[o] = hi ? s.Th[q].y + s.Tl[q].y : s.Th[q].x + s.Tl[q].x;
        out_nproc[o] = s.nproc[p];
        if (STATS) out_ncontrib[o] = s.ncontrib[p];
    }
}

static int g_ppt_override[2] = {0, 0};  // [forward, backward]; 0 = automatic

void set_blend_ppt(int fwd, int bwd) {
    g_ppt_override[0] = fwd;
    g_ppt_override[1] = bwd;
}

int blend_ppt(const ViewParams& v, bool backward) {
    const int o = g_ppt_override[backward ? 1 : 0];
    if (o == 1 || o == 2 || o == 4 || o == 8) return o;
    // measured on B200 (1M Gaussians, 1280x1024 pyramid, tests/diag_fwd.py): the forward wants
    // 2 pixels per thread at every level; the backward amortises its per-entry warp reduction
    // over 4 pixels once there are >= 1280 tiles (L1, L0) and keeps 2 (more warps per tile) at
    // the 320-tile level.
    const int tiles = v.tiles_x * v.tiles_y;
    if (!backward) return 2;
    return tiles >= 1024 ? 4 : 2;
}

void launch_blend_fwd(const uint2* ranges, const uint32_t* vals, const Splat* rec, const ViewParams& v,
                      float* color, float* depth, float* vis, float* t_final, int32_t* n_proc,
                      int32_t* n_contrib, bool stats, cudaStream_t st) {
    const int n_tiles = v.tiles_x * v.tiles_y;
#define GSB_FWD(P, S) \
    blend_fwd_kernel<P, S><<<n_tiles, kTileThreads / P, 0, st>>>(ranges, vals, rec, v, color, depth, vis, t_final, \
                                                               n_proc, n_contrib)
    switch (blend_ppt(v, false)) {
        case 4:
            if (stats) GSB_FWD(4, true); else GSB_FWD(4, false);
            break;
        case 1:
            if (stats) GSB_FWD(1, true); else GSB_FWD(1, false);
            break;
        default:
            if (stats) GSB_FWD(2, true); else GSB_FWD(2, false);
    }
#undef GSB_FWD
}

}  // namespace gsb
