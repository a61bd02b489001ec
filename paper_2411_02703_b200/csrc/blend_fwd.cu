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

template <int PPT>
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

    float2 Th[NP], Tl[NP], c0[NP], c1[NP], c2[NP], dd[NP], vis[NP];
    int nproc[2 * NP], ncontrib[2 * NP];
    unsigned live = 0;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        Th[q] = f2(1.f);
        Tl[q] = c0[q] = c1[q] = c2[q] = dd[q] = vis[q] = f2(0.f);
    }
#pragma unroll
    for (int p = 0; p < 2 * NP; ++p) {
        nproc[p] = ncontrib[p] = 0;
        if (p < PPT && sc.px < v.width && sc.py0 + p < v.height) live |= 1u << p;
    }
    int4 lb = warp_bbox<PPT>(live, sc);
    unsigned seen = live;
    // the next batch's record is loaded one batch ahead (its latency overlaps the current walk)
    Splat nsp;
    if (range.x + threadIdx.x < range.y) nsp = rec[vals[range.x + threadIdx.x]];
    for (uint32_t base = range.x; base < range.y; base += NT) {
        if (__syncthreads_count(live != 0) == 0) break;
        const uint32_t idx = base + threadIdx.x;
        if (idx < range.y) sb.put(threadIdx.x, stage_of(nsp, ox, oy));
        if (idx + NT < range.y) nsp = rec[vals[idx + NT]];
        __syncthreads();
        const int cnt = min(NT, static_cast<int>(range.y - base));
        // the warp first ballots which staged entries meet the bounding box of its live pixels,
        // then walks only those (in list order)
        for (int b0 = 0; b0 < cnt; b0 += 32) {
            if (__any_sync(0xffffffffu, live != seen)) {
                seen = live;
                lb = warp_bbox<PPT>(live, sc);
            }
            if (lb.x > lb.z) break;  // no live pixel left in this warp
            const int jj = b0 + sc.lane;
            unsigned todo = __ballot_sync(0xffffffffu, jj < cnt && rect_meets(sb.rect[jj], lb));
            while (todo) {
            const int j = b0 + __ffs(todo) - 1;
            todo &= todo - 1;
            const int4 rc = sb.rect[j];
            if (!live || sc.px < rc.x || sc.px > rc.z || sc.py0 + PPT - 1 < rc.y || sc.py0 > rc.w) continue;
            const float2 m = sb.mean[j];
            const float4 cn = sb.con[j];
            const float4 col = sb.col[j];
            const int pos = static_cast<int>(base - range.x) + j;
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                const int p0 = 2 * q, y0 = sc.py0 + p0;
                const bool a0 = ((live >> p0) & 1u) && y0 >= rc.y && y0 <= rc.w;
                const bool a1 = ((live >> (p0 + 1)) & 1u) && y0 + 1 >= rc.y && y0 + 1 <= rc.w;
                // no branch on (a0 || a1): an inactive half has al = 0 -> w = 0 and factor 1 + 0,
                // which leaves Th + Tl exactly unchanged (Fast2Sum renormalisation)
                const float fy = static_cast<float>(sc.ly0 + p0);
                const AlphaP e = alpha_pair(m, cn, fx, make_float2(fy, fy + 1.f));
                const float2 al = make_float2(a0 ? e.alpha.x : 0.f, a1 ? e.alpha.y : 0.f);
                const float2 w = __fmul2_rn(al, Th[q]);
                c0[q] = __ffma2_rn(w, f2(col.x), c0[q]);
                c1[q] = __ffma2_rn(w, f2(col.y), c1[q]);
                c2[q] = __ffma2_rn(w, f2(col.z), c2[q]);
                dd[q] = __ffma2_rn(w, f2(col.w), dd[q]);
                vis[q] = __fadd2_rn(vis[q], w);
                // exact factor 1 - alpha = fh + fl (Fast2Sum(1, -alpha)); clamp -> 1 - 0.99 (fp64)
                float2 fh = __fadd2_rn(f2(1.f), neg2(al));
                float2 fl = __fadd2_rn(neg2(al), neg2(__fadd2_rn(fh, f2(-1.f))));
                if (a0 && e.a_raw.x >= kAlphaMaxF) { fh.x = kClampFacHi; fl.x = kClampFacLo; }
                if (a1 && e.a_raw.y >= kAlphaMaxF) { fh.y = kClampFacHi; fl.y = kClampFacLo; }
                // (Th + Tl) * (fh + fl) with the exact product error of Th * fh
                const float2 pr = __fmul2_rn(Th[q], fh);
                const float2 er = __ffma2_rn(Th[q], fh, neg2(pr));
                const float2 t = __ffma2_rn(Th[q], fl, __ffma2_rn(Tl[q], fh, er));
                Th[q] = __fadd2_rn(pr, t);
                Tl[q] = __fadd2_rn(t, neg2(__fadd2_rn(Th[q], neg2(pr))));
                if (a0) {
                    ++ncontrib[p0];
                    nproc[p0] = pos + 1;
                }
                if (a1) {
                    ++ncontrib[p0 + 1];
                    nproc[p0 + 1] = pos + 1;
                }
                if ((a0 && Th[q].x < kTNear) || (a1 && Th[q].y < kTNear)) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int p = p0 + h;
                        const float th = h ? Th[q].y : Th[q].x, tl = h ? Tl[q].y : Tl[q].x;
                        if (!(h ? a1 : a0) || !(th < kTNear)) continue;
                        atomicAdd(&g_blend_stats[0], 1ull);
                        // sign of (Th + Tl) - 1e-4, with Th - kTMinHi exact (Sterbenz)
                        const float d = __fadd_rn(th, -kTMinHi) + __fadd_rn(tl, -kTMinLo);
                        const float tol = 1e-4f * 5.7e-14f * static_cast<float>(ncontrib[p] + 16);
                        bool term = d < -tol;
                        if (!(d < -tol) && !(d > tol)) {
                            atomicAdd(&g_blend_stats[1], 1ull);
                            term = replay_transmittance(vals, rec, range, pos, sc.px, sc.py0 + p, ox, oy, fx,
                                                        static_cast<float>(sc.ly0 + p)) < kTMin;
                        }
                        if (term) live &= ~(1u << p);
                    }
                }
            }
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
        out_color[o] = hi ? c0[q].y : c0[q].x;
        out_color[P + o] = hi ? c1[q].y : c1[q].x;
        out_color[2 * P + o] = hi ? c2[q].y : c2[q].x;
        out_depth[o] = hi ? dd[q].y : dd[q].x;
        out_vis[o] = hi ? vis[q].y : vis[q].x;
        out_t[o] = hi ? Th[q].y + Tl[q].y : Th[q].x + Tl[q].x;
        out_nproc[o] = nproc[p];
        out_ncontrib[o] = ncontrib[p];
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
    // 2 pixels per thread, and 1 at the coarsest level where only 320 tiles (long lists) exist;
    // the backward amortises its per-entry warp reduction over 4 pixels once there are >= 1280
    // tiles (L1, L0) and keeps 2 (more warps per tile) at the 320-tile level.
    const int tiles = v.tiles_x * v.tiles_y;
    if (!backward) return tiles >= 1024 ? 2 : 1;
    return tiles >= 1024 ? 4 : 2;
}

void launch_blend_fwd(const uint2* ranges, const uint32_t* vals, const Splat* rec, const ViewParams& v,
                      float* color, float* depth, float* vis, float* t_final, int32_t* n_proc,
                      int32_t* n_contrib, cudaStream_t st) {
    const int n_tiles = v.tiles_x * v.tiles_y;
    switch (blend_ppt(v, false)) {
        case 8:
            blend_fwd_kernel<8><<<n_tiles, 32, 0, st>>>(ranges, vals, rec, v, color, depth, vis, t_final, n_proc, n_contrib);
            break;
        case 4:
            blend_fwd_kernel<4><<<n_tiles, 64, 0, st>>>(ranges, vals, rec, v, color, depth, vis, t_final, n_proc, n_contrib);
            break;
        case 1:
            blend_fwd_kernel<1><<<n_tiles, 256, 0, st>>>(ranges, vals, rec, v, color, depth, vis, t_final, n_proc, n_contrib);
            break;
        default:
            blend_fwd_kernel<2><<<n_tiles, 128, 0, st>>>(ranges, vals, rec, v, color, depth, vis, t_final, n_proc, n_contrib);
    }
}

}  // namespace gsb
