// K5: front-to-back blend (rasterizer.cpp:118-162). Box test = integer pixel rect; alpha clamped
// at 0.99; the contributor is accumulated BEFORE the T < 1e-4 break; V = sum of weights. Per
// pixel it keeps n_proc (list position + 1 of the terminating contributor, the list length when
// the pixel never terminates) and T_final for the backward instead of the reference's CSR table
// (rasterizer.cpp:164-197).
//
// Exact termination with fp32 arithmetic: the transmittance is carried in fp32 together with a
// rigorous bound on its distance from the reference's fp64 product. Each fp32 factor
// fl(1 - alpha) (0.01f for a clamp) is within 2^-24 of the reference's fp64 factor and each
// product rounds by <= 2^-24, so after k factors |T32 / T64 - 1| <= beta(k) = 2k 2^-24 (+5%).
// Only when T32 lies inside [1e-4 (1 - beta), 1e-4 (1 + beta)] is the decision ambiguous; the
// warp then replays that pixel cooperatively in fp64 (32 entries per step, product tree), and
// only if even that lands within its own rounding bound of 1e-4 does one lane replay it
// sequentially in the reference's operation order. (Counted in g_blend_stats.)
#include "blend_common.cuh"
#include "kernels.cuh"

// build knobs (diag/build_variant.sh experiments; the defaults are the product build)
#ifndef GSB_FWD_MIN_BLOCKS
#define GSB_FWD_MIN_BLOCKS 6  // 80 registers, 6 CTAs per SM: -13% at full resolution (diag/variant_levels.sh)
#endif
// levels with more tiles than kFwdWideTiles run a 7-CTA build (72 registers): -2.5% on the
// full-resolution forward, +6% at 1280 tiles (diag/variant_levels.sh)
constexpr int kFwdWideTiles = 2048, kFwdWideBlocks = 7;
#ifdef GSB_NEAR_NOINLINE
#define GSB_NEAR_INLINE __noinline__
#else
#define GSB_NEAR_INLINE __forceinline__
#endif

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

constexpr float kClampFac = 0.01f;              // within 2^-24 of 1 - 0.99 (fp64) = 0.010000000000000009
// df32 mode: 1 - 0.99 (fp64) and 1e-4 (fp64) as exact float pairs
constexpr float kClampFacHi = 0.009999999776482582f, kClampFacLo = 2.2351742678949904e-10f;
constexpr float kTMinHi = 9.999999747378752e-05f, kTMinLo = 2.5262125290942405e-12f;
constexpr double kBetaPerFactor = 1.2517e-7;     // 2 * 2^-24 * 1.05

// Exact fp64 transmittance of pixel (px, py) after the contributor at list position `upto`, in
// the reference's sequential operation order (rasterizer.cpp:143-151).
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

// The same product computed by the whole warp (uniform arguments): lane l evaluates entry
// base + l, each chunk of 32 factors is multiplied as a butterfly tree. Differs from the
// sequential product by at most ~2 (upto + 1) 2^-53 relative.
__device__ __noinline__ double warp_replay(const uint32_t* __restrict__ vals, const Splat* __restrict__ rec,
                                           uint2 range, int upto, int px, int py, double ox, double oy, float fx,
                                           float fy) {
    const int lane = threadIdx.x & 31;
    double T = 1.0;
    for (int base = 0; base <= upto; base += 32) {
        const int j = base + lane;
        double f = 1.0;
        if (j <= upto) {
            const Splat sp = rec[vals[range.x + j]];
            if (!(px < sp.x0 || px > sp.x1 || py < sp.y0 || py > sp.y1)) {
                const Staged s = stage_of(sp, ox, oy);
                const AlphaS e = alpha_scalar(s.mean, s.con, fx, fy);
                f = one_minus_alpha_d(e.a_raw, e.alpha);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) f = __dmul_rn(f, __shfl_xor_sync(0xffffffffu, f, o));
        T = __dmul_rn(T, f);
    }
    return T;
}

}  // namespace

// Per-pixel blend state of one thread (NP packed pairs of vertically adjacent pixels).
template <int NP>
struct FwdState {
    float2 T[NP], Tl[NP], c0[NP], c1[NP], c2[NP], dd[NP], vis[NP];  // Tl: df32 low part (DF mode)
    // per pixel, as packed multipliers of the walk: on = 1 while the pixel is live, else 0 (it
    // scales the entry's opacity, so a stopped or absent pixel takes alpha = 0, weight 0, factor
    // 1); tn = on * t_near (a stopped pixel never asks for a termination check)
    float2 on[NP], tn[NP];
    int nproc[2 * NP], ncontrib[2 * NP];
    unsigned live;
    // pixel p stops after the entry at list position pos
    __device__ __forceinline__ void stop(int p, int pos) {
        live &= ~(1u << p);
#pragma unroll
        for (int q = 0; q < 2 * NP; ++q) {  // static indices: the arrays stay in registers
            if (q != p) continue;
            nproc[q] = pos + 1;
            if (q & 1) on[q >> 1].y = tn[q >> 1].y = 0.f;
            else on[q >> 1].x = tn[q >> 1].x = 0.f;
        }
    }
    __device__ __forceinline__ void arm(float t_near) {
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            on[q] = make_float2((live >> (2 * q)) & 1u ? 1.f : 0.f, (live >> (2 * q + 1)) & 1u ? 1.f : 0.f);
            tn[q] = make_float2(on[q].x * t_near, on[q].y * t_near);
        }
    }
};

// Pixels whose fp32 transmittance fell below t_near after the entry at `pos` (bits in `near`):
// decide T64 < 1e-4 exactly. Called by the whole warp; every pixel has taken at most pos + 1
// factors (the list entries up to pos).
template <int PPT>
__device__ GSB_NEAR_INLINE void resolve_near(FwdState<(PPT + 1) / 2>& s, unsigned near, const Strip<PPT>& sc, int pos,
                                          float fx, const uint32_t* __restrict__ vals,
                                          const Splat* __restrict__ rec, uint2 range, double ox, double oy) {
    const double beta = kBetaPerFactor * (pos + 1);
    unsigned amb = 0;
#pragma unroll
    for (int p = 0; p < 2 * ((PPT + 1) / 2); ++p) {
        if (!((near >> p) & 1u)) continue;
        atomicAdd(&g_blend_stats[0], 1ull);
        const double t = (p & 1) ? s.T[p >> 1].y : s.T[p >> 1].x;
        if (t / (1.0 - beta) < kTMin) {  // T64 <= T32 / (1 - beta) < 1e-4
            s.stop(p, pos);
        } else if (!(t / (1.0 + beta) >= kTMin)) {
            amb |= 1u << p;  // else T64 >= T32 / (1 + beta) >= 1e-4
        }
    }
    unsigned need = __ballot_sync(0xffffffffu, amb != 0u);
    while (need) {
        const int src = __ffs(need) - 1;
        need &= need - 1;
        const unsigned bits = __shfl_sync(0xffffffffu, amb, src);
        const int px = __shfl_sync(0xffffffffu, sc.px, src);
        const int py0 = __shfl_sync(0xffffffffu, sc.py0, src);
        const int ly0 = __shfl_sync(0xffffffffu, sc.ly0, src);
        const float sfx = __shfl_sync(0xffffffffu, fx, src);
        for (int p = 0; p < PPT; ++p) {
            if (!((bits >> p) & 1u)) continue;
            atomicAdd(&g_blend_stats[1], 1ull);
            const float fy = static_cast<float>(ly0 + p);
            double T = warp_replay(vals, rec, range, pos, px, py0 + p, ox, oy, sfx, fy);
            if (fabs(T / kTMin - 1.0) <= 2.5 * (pos + 1) * 1.1102230246251565e-16 && (threadIdx.x & 31) == src)
                T = replay_transmittance(vals, rec, range, pos, px, py0 + p, ox, oy, sfx, fy);
            if ((threadIdx.x & 31) == src && T < kTMin) s.stop(p, pos);
        }
    }
}

// DF mode: sign of (Th + Tl) - 1e-4 per near pixel; the sequential fp64 replay only if even the
// df32 value is within its rounding bound of the threshold (not observed in practice).
template <int PPT>
__device__ GSB_NEAR_INLINE void df_near(FwdState<(PPT + 1) / 2>& s, unsigned near, const Strip<PPT>& sc, int pos,
                                        float fx, const uint32_t* __restrict__ vals, const Splat* __restrict__ rec,
                                        uint2 range, double ox, double oy) {
#pragma unroll
    for (int p = 0; p < 2 * ((PPT + 1) / 2); ++p) {
        if (!((near >> p) & 1u)) continue;
        atomicAdd(&g_blend_stats[0], 1ull);
        const float th = (p & 1) ? s.T[p >> 1].y : s.T[p >> 1].x, tl = (p & 1) ? s.Tl[p >> 1].y : s.Tl[p >> 1].x;
        // Th - kTMinHi is exact (Sterbenz)
        const float d = __fadd_rn(th, -kTMinHi) + __fadd_rn(tl, -kTMinLo);
        const float tol = 1e-4f * 5.7e-14f * static_cast<float>(pos + 16);
        bool term = d < -tol;
        if (!(d < -tol) && !(d > tol)) {
            atomicAdd(&g_blend_stats[1], 1ull);
            term = replay_transmittance(vals, rec, range, pos, sc.px, sc.py0 + p, ox, oy, fx,
                                        static_cast<float>(sc.ly0 + p)) < kTMin;
        }
        if (term) s.stop(p, pos);
    }
}

// Transmittance modes of the forward walk.
//   kBand:  fp32 T + rigorous error band, warp-cooperative fp64 replay when ambiguous.
//   kDf:    df32 T (Th + Tl, exact to ~2^-46 per step), sequential replay only if even that is
//           ambiguous (not observed in practice).
//   kLocal: df32 T of one list segment started at T = 1 (segmented forward, pass 1): a pixel
//           stops only once its local T is certainly below 1e-4 (the global T is then too).
enum FwdMode : int { kBand = 0, kDf = 1, kLocal = 2 };

// One tile-list entry over the thread's pixels. COVER: the entry's rect contains every live
// pixel of the warp (warp-uniform), so no per-pixel box test (a stopped pixel has opacity 0).
// STATS: maintain n_contrib (only the public render reports it).
template <int PPT, bool COVER, bool STATS, int MODE, bool CLAMP>
__device__ __forceinline__ void fwd_entry(FwdState<(PPT + 1) / 2>& s, const Strip<PPT>& sc, const int4& rc,
                                          float2 m, float4 cn, float4 col, int pos, float fx,
                                          const uint32_t* __restrict__ vals, const Splat* __restrict__ rec,
                                          uint2 range, double ox, double oy) {
    constexpr int NP = (PPT + 1) / 2;
    const bool colin = COVER || (sc.px >= rc.x && sc.px <= rc.z);
    // pixels whose fp32 transmittance fell below t_near at this entry: kept as predicates, the
    // bitmask is built only on the (rare) slow path
    bool nb[2 * NP];
    bool anyn = false;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        const int p0 = 2 * q, y0 = sc.py0 + p0;
        // in the entry's rect (a stopped pixel is masked by its zero opacity instead)
        bool a0 = true, a1 = true;
        if (!COVER) {
            a0 = colin && y0 >= rc.y && y0 <= rc.w;
            a1 = colin && y0 + 1 >= rc.y && y0 + 1 <= rc.w;
        }
        // no branch on (a0 || a1): an inactive half has al = 0 -> w = 0 and factor exactly 1
        const float fy = static_cast<float>(sc.ly0 + p0);
        const AlphaP e = alpha_pair_op<CLAMP>(m, cn, __fmul2_rn(f2(cn.w), s.on[q]), fx, make_float2(fy, fy + 1.f));
        const float2 al = COVER ? e.alpha : make_float2(a0 ? e.alpha.x : 0.f, a1 ? e.alpha.y : 0.f);
        const float2 w = __fmul2_rn(al, s.T[q]);
        s.c0[q] = __ffma2_rn(w, f2(col.x), s.c0[q]);
        s.c1[q] = __ffma2_rn(w, f2(col.y), s.c1[q]);
        s.c2[q] = __ffma2_rn(w, f2(col.z), s.c2[q]);
        s.dd[q] = __ffma2_rn(w, f2(col.w), s.dd[q]);
        s.vis[q] = __fadd2_rn(s.vis[q], w);
        if (MODE != kBand) {
            // exact factor 1 - alpha = fh + fl (Fast2Sum(1, -alpha)); clamp -> 1 - 0.99 (fp64)
            float2 fh = __fadd2_rn(f2(1.f), neg2(al));
            float2 fl = __fadd2_rn(neg2(al), neg2(__fadd2_rn(fh, f2(-1.f))));
            if (CLAMP && a0 && e.a_raw.x >= kAlphaMaxF) { fh.x = kClampFacHi; fl.x = kClampFacLo; }
            if (CLAMP && a1 && e.a_raw.y >= kAlphaMaxF) { fh.y = kClampFacHi; fl.y = kClampFacLo; }
            // (Th + Tl) * (fh + fl) with the exact product error of Th * fh
            const float2 pr = __fmul2_rn(s.T[q], fh);
            const float2 er = __ffma2_rn(s.T[q], fh, neg2(pr));
            const float2 t = __ffma2_rn(s.T[q], fl, __ffma2_rn(s.Tl[q], fh, er));
            s.T[q] = __fadd2_rn(pr, t);
            s.Tl[q] = __fadd2_rn(t, neg2(__fadd2_rn(s.T[q], neg2(pr))));
        } else {
            // 1 - al, with a clamp (al = 0.99f, 1 - al = 0.0099999905f) replaced by 0.01f: every
            // unclamped al < 0.99f gives 1 - al >= 0.0100000501f, so a max does it (inactive: 1)
            const float2 f = __fadd2_rn(f2(1.f), neg2(al));
            s.T[q] = __fmul2_rn(s.T[q], CLAMP ? make_float2(fmaxf(f.x, kClampFac), fmaxf(f.y, kClampFac)) : f);
        }
        if (STATS) {
            s.ncontrib[p0] += a0 && ((s.live >> p0) & 1u);
            s.ncontrib[p0 + 1] += a1 && ((s.live >> (p0 + 1)) & 1u);
        }
        // a pixel outside the rect kept T (already decided at its last contributor): no check
        nb[p0] = a0 && s.T[q].x < s.tn[q].x;
        nb[p0 + 1] = a1 && s.T[q].y < s.tn[q].y;
        anyn = anyn || nb[p0] || nb[p0 + 1];
    }
    if (MODE == kDf) {
        if (anyn) {
            unsigned near = 0;
#pragma unroll
            for (int p = 0; p < 2 * NP; ++p) near |= static_cast<unsigned>(nb[p]) << p;
            df_near<PPT>(s, near, sc, pos, fx, vals, rec, range, ox, oy);
        }
    } else if (MODE == kLocal) {
#pragma unroll
        for (int p = 0; p < 2 * NP; ++p) {
            if (!nb[p]) continue;
            const float th = (p & 1) ? s.T[p >> 1].y : s.T[p >> 1].x, tl = (p & 1) ? s.Tl[p >> 1].y : s.Tl[p >> 1].x;
            const float d = __fadd_rn(th, -kTMinHi) + __fadd_rn(tl, -kTMinLo);
            if (d < -1e-4f * 5.7e-14f * static_cast<float>(pos + 16)) s.stop(p, pos);  // certainly below
        }
    } else if (__any_sync(0xffffffffu, anyn)) {
        unsigned near = 0;
#pragma unroll
        for (int p = 0; p < 2 * NP; ++p) near |= static_cast<unsigned>(nb[p]) << p;
        resolve_near<PPT>(s, near, sc, pos, fx, vals, rec, range, ox, oy);
    }
}

// Backward checkpoint k: this thread's pixel states before list entry k L (see seg_len).
template <int PPT>
__device__ __forceinline__ void write_checkpoint(const FwdState<(PPT + 1) / 2>& s, const Strip<PPT>& sc, float* ck,
                                                 int k, int width, int height) {
    const size_t P = static_cast<size_t>(width) * height;
    float* base = ck + static_cast<size_t>(k - 1) * kCkFields * P;
#pragma unroll
    for (int p = 0; p < PPT; ++p) {
        const int y = sc.py0 + p;
        if (sc.px >= width || y >= height) continue;
        const int q = p >> 1;
        const bool hi = p & 1;
        const size_t o = static_cast<size_t>(y) * width + sc.px;
        base[o] = hi ? s.T[q].y + s.Tl[q].y : s.T[q].x + s.Tl[q].x;
        base[P + o] = hi ? s.c0[q].y : s.c0[q].x;
        base[2 * P + o] = hi ? s.c1[q].y : s.c1[q].x;
        base[3 * P + o] = hi ? s.c2[q].y : s.c2[q].x;
        base[4 * P + o] = hi ? s.dd[q].y : s.dd[q].x;
    }
}

// The walk over entries [start, end) of one tile's list `full` (staging batches of NT entries,
// per-warp ballot against the live-pixel box, list order within the warp). Positions are
// relative to the list start; checkpoints are written only by a whole-list walk (start = 0).
// The next batch's records are copied into `raw` (cp.async, one 64-byte record per thread)
// while the current batch is walked; the list index of the batch after that is kept in a
// register so the copy's address is ready when it is issued.
template <int PPT, bool STATS, int MODE, int NT = kTileThreads / PPT>
__device__ __forceinline__ void blend_walk(FwdState<(PPT + 1) / 2>& s, StageBuf<NT>& sb, Splat* raw,
                                           const Strip<PPT>& sc, const uint32_t* __restrict__ vals,
                                           const Splat* __restrict__ rec, uint2 full, int start, int end, double ox,
                                           double oy, float fx, float* ck, int nseg, int width, int height,
                                           [[maybe_unused]] const unsigned long long* cnt) {
    GSB_CHECK(full.x <= full.y && full.y <= cnt[kCntPairs] && end <= static_cast<int>(full.y - full.x));
    // NT: threads of the CTA = the staging batch (a tile may be split over SUB CTAs)
    static_assert(kSegAlign % NT == 0, "segment boundaries must fall on staging batches");
    const int n_list = static_cast<int>(full.y - full.x);
    const int L = seg_len(n_list, nseg);
    int next_ck = (start == 0 && nseg > 1 && L > 0) ? 1 : nseg;  // next checkpoint to write
    // below t_near the termination needs a closer look: fp32 mode 1e-4 (1 + beta(list length)),
    // rounded up; df32 modes a fixed guard
    const float t_near = MODE != kBand ? 1.0001e-4f
                                       : __double2float_ru(kTMin * (1.0 + kBetaPerFactor * (n_list + 1)));
    s.arm(t_near);
    int4 lb = warp_bbox<PPT>(s.live, sc);
    unsigned seen = s.live;
    const uint32_t b_end = full.x + end;
    const uint32_t i0 = full.x + start + threadIdx.x;
    if (i0 < b_end) {
        GSB_CHECK(vals[i0] < cnt[kCntVisible]);
        cp_async_splat(&raw[threadIdx.x], &rec[vals[i0]]);
    }
    cp_async_commit();
    uint32_t nvi = i0 + NT < b_end ? vals[i0 + NT] : 0u;
    for (uint32_t base = full.x + start; base < b_end; base += NT) {
        if (next_ck < nseg && static_cast<int>(base - full.x) == next_ck * L)
            write_checkpoint<PPT>(s, sc, ck, next_ck++, width, height);
        if (__syncthreads_count(s.live != 0) == 0) break;
        const uint32_t idx = base + threadIdx.x;
        cp_async_wait_all();  // this thread's own record (each thread reads only its slot)
        if (idx < b_end) sb.put(threadIdx.x, stage_of(raw[threadIdx.x], ox, oy));
        if (idx + NT < b_end) {
            GSB_CHECK(nvi < cnt[kCntVisible]);
            cp_async_splat(&raw[threadIdx.x], &rec[nvi]);
            if (idx + 2 * NT < b_end) nvi = vals[idx + 2 * NT];
        }
        cp_async_commit();
        __syncthreads();
        const int cnt = min(NT, static_cast<int>(b_end - base));
        for (int b0 = 0; b0 < cnt; b0 += 32) {
            if (__any_sync(0xffffffffu, s.live != seen)) {
                seen = s.live;
                lb = warp_bbox<PPT>(s.live, sc);
            }
            if (lb.x > lb.z) break;  // no live pixel left in this warp
            // per chunk of 32 staged entries, lane l classifies entry b0 + l against the chunk's
            // live box: meets it (walked), covers it (no per-pixel box test), opacity >= 0.99f
            // (alpha may clamp). Pixels stopping inside the chunk only shrink the true box, so
            // the chunk-start classification stays valid.
            const int jj = b0 + sc.lane;
            bool meets = false, covers = false, clamps = false;
            if (jj < cnt) {
                const int4 r = sb.rect[jj];
                meets = rect_meets(r, lb);
                covers = r.x <= lb.x && r.z >= lb.z && r.y <= lb.y && r.w >= lb.w;
                clamps = sb.con[jj].w >= kAlphaMaxF;
            }
            unsigned todo = __ballot_sync(0xffffffffu, meets);
            const unsigned cov = __ballot_sync(0xffffffffu, meets && covers);
            const unsigned clp = __ballot_sync(0xffffffffu, meets && clamps);
            while (todo) {
                const int bit = __ffs(todo) - 1;
                todo &= todo - 1;
                const int j = b0 + bit;
                const int pos = static_cast<int>(base - full.x) + j;
                const float4 cn = sb.con[j];
                if (!((clp >> bit) & 1u)) {
                    if ((cov >> bit) & 1u)
                        fwd_entry<PPT, true, STATS, MODE, false>(s, sc, lb, sb.mean[j], cn, sb.col[j], pos, fx,
                                                                 vals, rec, full, ox, oy);
                    else
                        fwd_entry<PPT, false, STATS, MODE, false>(s, sc, sb.rect[j], sb.mean[j], cn, sb.col[j], pos,
                                                                  fx, vals, rec, full, ox, oy);
                } else if ((cov >> bit) & 1u) {
                    fwd_entry<PPT, true, STATS, MODE, true>(s, sc, lb, sb.mean[j], cn, sb.col[j], pos, fx, vals,
                                                            rec, full, ox, oy);
                } else {
                    fwd_entry<PPT, false, STATS, MODE, true>(s, sc, sb.rect[j], sb.mean[j], cn, sb.col[j], pos,
                                                             fx, vals, rec, full, ox, oy);
                }
            }
        }
    }
    cp_async_wait_all();  // no copy may land after the CTA's shared memory is reused
    // boundaries past an early exit (every pixel terminated) hold the final state
    for (; next_ck < nseg && next_ck * L < n_list; ++next_ck) write_checkpoint<PPT>(s, sc, ck, next_ck, width, height);
}

// SUB CTAs per tile, each with kThreads / SUB threads (its share of the tile's warps): finer work
// units for the block scheduler (a level whose tile count is not a multiple of the resident CTA
// slots leaves a part-empty last wave)
template <int PPT, bool STATS, int SUB, int MINB = GSB_FWD_MIN_BLOCKS>
__global__ void __launch_bounds__(kTileThreads / PPT / SUB, MINB * SUB) blend_fwd_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals, const Splat* __restrict__ rec,
    ViewParams v, float* __restrict__ out_color, float* __restrict__ out_depth, float* __restrict__ out_vis,
    float* __restrict__ out_t, int32_t* __restrict__ out_nproc, int32_t* __restrict__ out_ncontrib, int df_list,
    float* __restrict__ ck, int nseg, const uint32_t* __restrict__ order, const unsigned long long* __restrict__ cnt) {
    pdl_enter();
    using S = Strip<PPT>;
    // PPT = 1 runs one (real) pixel per lane in the low half of the pair; the high half is never
    // live, so its packed lane computes nothing that is kept.
    constexpr int NT = S::kThreads / SUB, NP = (PPT + 1) / 2;
    __shared__ StageBuf<NT> sb;
    __shared__ Splat raw[NT];
    const int tile = order ? static_cast<int>(order[blockIdx.x / SUB]) : static_cast<int>(blockIdx.x / SUB);
    const S sc(v.tiles_x, tile, (blockIdx.x % SUB) * (NT / 32) + (threadIdx.x >> 5));
    const uint2 range = ranges[tile];
    const double ox = sc.tx * kTile, oy = sc.ty * kTile;
    const float fx = static_cast<float>(sc.lx);

    FwdState<NP> s;
    s.live = 0;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        s.T[q] = f2(1.f);
        s.Tl[q] = s.c0[q] = s.c1[q] = s.c2[q] = s.dd[q] = s.vis[q] = f2(0.f);
    }
    // n_proc: list position + 1 of the terminating contributor; a pixel that never terminates
    // keeps the list length (its later entries do not contain it, so the backward's replay from
    // there is the same)
#pragma unroll
    for (int p = 0; p < 2 * NP; ++p) {
        s.nproc[p] = static_cast<int>(range.y - range.x);
        s.ncontrib[p] = 0;
        if (p < PPT && sc.px < v.width && sc.py0 + p < v.height) s.live |= 1u << p;
    }
    // fp32 + band for short lists; df32 for lists longer than df_list (wide band, long replays)
    if (static_cast<int>(range.y - range.x) > df_list)
        blend_walk<PPT, STATS, kDf, NT>(s, sb, raw, sc, vals, rec, range, 0, static_cast<int>(range.y - range.x), ox, oy,
                                        fx, ck, nseg, v.width, v.height, cnt);
    else
        blend_walk<PPT, STATS, kBand, NT>(s, sb, raw, sc, vals, rec, range, 0, static_cast<int>(range.y - range.x), ox,
                                          oy, fx, ck, nseg, v.width, v.height, cnt);
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
        out_t[o] = hi ? s.T[q].y + s.Tl[q].y : s.T[q].x + s.Tl[q].x;
        out_nproc[o] = s.nproc[p];
        if (STATS) out_ncontrib[o] = s.ncontrib[p];
    }
}

// ------------------------------------------------------------------------------------------
// Segmented forward (few tiles, long lists): the tile lists are cut at the backward's segment
// boundaries and walked in three passes, so the latency-bound sequential walk is spread over
// (tile, segment) CTAs. Exactness: every termination decision is taken either on a df32 product
// certainly above 1e-4 or by the exact df32 walk of pass 3.
constexpr int kSegFields = 9;  // Th, Tl, C_r, C_g, C_b, D, V, (unused), contributions

template <int PPT>
__device__ __forceinline__ void init_state(FwdState<(PPT + 1) / 2>& s, const Strip<PPT>& sc, int width, int height) {
    constexpr int NP = (PPT + 1) / 2;
    s.live = 0;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        s.T[q] = f2(1.f);
        s.Tl[q] = s.c0[q] = s.c1[q] = s.c2[q] = s.dd[q] = s.vis[q] = f2(0.f);
    }
#pragma unroll
    for (int p = 0; p < 2 * NP; ++p) {
        s.nproc[p] = s.ncontrib[p] = 0;
        if (p < PPT && sc.px < width && sc.py0 + p < height) s.live |= 1u << p;
    }
}

// pass 1: CTA (tile, segment) walks the segment from T = 1 (df32) and stores the local state
template <int PPT, bool STATS>
__global__ void __launch_bounds__(kTileThreads / PPT) fwd_seg_local_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals, const Splat* __restrict__ rec,
    ViewParams v, float* __restrict__ seg, int nseg, const unsigned long long* __restrict__ cnt) {
    pdl_enter();
    using S = Strip<PPT>;
    __shared__ StageBuf<S::kThreads> sb;
    __shared__ Splat raw[S::kThreads];
    const S sc(v.tiles_x);
    const uint2 range = ranges[blockIdx.x];
    const int n_list = static_cast<int>(range.y - range.x);
    const int L = seg_len(n_list, nseg);
    const int lo = static_cast<int>(blockIdx.y) * L;
    if (lo >= n_list) return;
    const double ox = sc.tx * kTile, oy = sc.ty * kTile;
    const float fx = static_cast<float>(sc.lx);
    FwdState<(PPT + 1) / 2> s;
    init_state<PPT>(s, sc, v.width, v.height);
    blend_walk<PPT, STATS, kLocal>(s, sb, raw, sc, vals, rec, range, lo, min(lo + L, n_list), ox, oy, fx, nullptr, 1,
                                   v.width, v.height, cnt);
    const size_t P = static_cast<size_t>(v.width) * v.height;
    float* base = seg + static_cast<size_t>(blockIdx.y) * kSegFields * P;
#pragma unroll
    for (int p = 0; p < PPT; ++p) {
        const int y = sc.py0 + p;
        if (sc.px >= v.width || y >= v.height) continue;
        const int q = p >> 1;
        const bool hi = p & 1;
        const size_t o = static_cast<size_t>(y) * v.width + sc.px;
        base[o] = hi ? s.T[q].y : s.T[q].x;
        base[P + o] = hi ? s.Tl[q].y : s.Tl[q].x;
        base[2 * P + o] = hi ? s.c0[q].y : s.c0[q].x;
        base[3 * P + o] = hi ? s.c1[q].y : s.c1[q].x;
        base[4 * P + o] = hi ? s.c2[q].y : s.c2[q].x;
        base[5 * P + o] = hi ? s.dd[q].y : s.dd[q].x;
        base[6 * P + o] = hi ? s.vis[q].y : s.vis[q].x;
        base[8 * P + o] = __int_as_float(s.ncontrib[p]);  // (field 7 unused: n_proc comes from pass 3)
    }
}

// pass 2: per pixel, chain the segments front to back; a segment is taken whole only if the
// df32 product after it is certainly >= 1e-4, else the pixel stops there (star) for pass 3.
// Writes the backward checkpoints at the segment boundaries it passes.
__global__ void fwd_seg_chain_kernel(const uint2* __restrict__ ranges, ViewParams v, const float* __restrict__ seg,
                                     int nseg, float* __restrict__ out_color, float* __restrict__ out_depth,
                                     float* __restrict__ out_vis, float* __restrict__ out_t,
                                     int32_t* __restrict__ out_nproc, int32_t* __restrict__ out_ncontrib,
                                     float* __restrict__ tl_plane, int32_t* __restrict__ star_plane,
                                     float* __restrict__ ck) {
    pdl_enter();
    const int P = v.width * v.height;
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= P) return;
    const int x = o % v.width, y = o / v.width;
    const uint2 range = ranges[(y / kTile) * v.tiles_x + x / kTile];
    const int n_list = static_cast<int>(range.y - range.x);
    const int L = seg_len(n_list, nseg);
    float th = 1.f, tl = 0.f, c0 = 0.f, c1 = 0.f, c2 = 0.f, dd = 0.f, vis = 0.f;
    // no termination before the stopping segment: n_proc = the list length unless pass 3 finds it
    const int nproc = n_list;
    int ncontrib = 0, star = -1;
    for (int s = 0; s < nseg && s * L < n_list; ++s) {
        if (s >= 1) {
            float* cp = ck + static_cast<size_t>(s - 1) * kCkFields * P;
            cp[o] = th + tl;
            cp[P + o] = c0;
            cp[2 * P + o] = c1;
            cp[3 * P + o] = c2;
            cp[4 * P + o] = dd;
        }
        const float* sg = seg + static_cast<size_t>(s) * kSegFields * P;
        const float lh = sg[o], ll = sg[P + o];
        // (th + tl) * (lh + ll) with the exact product error of th * lh
        const float pr = __fmul_rn(th, lh);
        const float er = __fmaf_rn(th, lh, -pr);
        const float t = __fmaf_rn(th, ll, __fmaf_rn(tl, lh, er));
        const float nh = __fadd_rn(pr, t);
        const float nl = __fadd_rn(t, -__fadd_rn(nh, -pr));
        const float d = __fadd_rn(nh, -kTMinHi) + __fadd_rn(nl, -kTMinLo);
        const float tol = 1e-4f * 1.2e-13f * static_cast<float>(min(n_list, (s + 1) * L) + 16);
        if (!(d > tol)) {
            star = s;
            break;
        }
        c0 = __fmaf_rn(th, sg[2 * P + o], c0);
        c1 = __fmaf_rn(th, sg[3 * P + o], c1);
        c2 = __fmaf_rn(th, sg[4 * P + o], c2);
        dd = __fmaf_rn(th, sg[5 * P + o], dd);
        vis = __fmaf_rn(th, sg[6 * P + o], vis);
        ncontrib += __float_as_int(sg[8 * P + o]);
        th = nh;
        tl = nl;
    }
    out_color[o] = c0;
    out_color[P + o] = c1;
    out_color[2 * P + o] = c2;
    out_depth[o] = dd;
    out_vis[o] = vis;
    out_t[o] = star < 0 ? th + tl : th;  // pass 3 continues from (th, tl)
    out_nproc[o] = nproc;
    if (out_ncontrib) out_ncontrib[o] = ncontrib;
    tl_plane[o] = tl;
    star_plane[o] = star;
}

// pass 3: CTA (tile, segment s) finishes the pixels that stopped at s with the exact df32 walk
template <int PPT, bool STATS>
__global__ void __launch_bounds__(kTileThreads / PPT) fwd_seg_finish_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals, const Splat* __restrict__ rec,
    ViewParams v, float* __restrict__ out_color, float* __restrict__ out_depth, float* __restrict__ out_vis,
    float* __restrict__ out_t, int32_t* __restrict__ out_nproc, int32_t* __restrict__ out_ncontrib,
    const float* __restrict__ tl_plane, const int32_t* __restrict__ star_plane, int nseg,
    const unsigned long long* __restrict__ cnt) {
    pdl_enter();
    using S = Strip<PPT>;
    constexpr int NP = (PPT + 1) / 2;
    __shared__ StageBuf<S::kThreads> sb;
    __shared__ Splat raw[S::kThreads];
    const S sc(v.tiles_x);
    const uint2 range = ranges[blockIdx.x];
    const int n_list = static_cast<int>(range.y - range.x);
    const int L = seg_len(n_list, nseg);
    const int lo = static_cast<int>(blockIdx.y) * L;
    if (lo >= n_list) return;
    const size_t P = static_cast<size_t>(v.width) * v.height;
    FwdState<NP> s;
    s.live = 0;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        float th[2] = {1.f, 1.f}, tl[2] = {0.f, 0.f}, a[2] = {0.f, 0.f}, b[2] = {0.f, 0.f}, c[2] = {0.f, 0.f};
        float d[2] = {0.f, 0.f}, w[2] = {0.f, 0.f};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int p = 2 * q + h, y = sc.py0 + p;
            s.nproc[p] = s.ncontrib[p] = 0;
            if (p < PPT && sc.px < v.width && y < v.height) {
                const size_t o = static_cast<size_t>(y) * v.width + sc.px;
                if (star_plane[o] == static_cast<int>(blockIdx.y)) {
                    s.live |= 1u << p;
                    th[h] = out_t[o];
                    tl[h] = tl_plane[o];
                    a[h] = out_color[o];
                    b[h] = out_color[P + o];
                    c[h] = out_color[2 * P + o];
                    d[h] = out_depth[o];
                    w[h] = out_vis[o];
                    s.nproc[p] = out_nproc[o];
                    if (STATS) s.ncontrib[p] = out_ncontrib[o];
                }
            }
        }
        s.T[q] = make_float2(th[0], th[1]);
        s.Tl[q] = make_float2(tl[0], tl[1]);
        s.c0[q] = make_float2(a[0], a[1]);
        s.c1[q] = make_float2(b[0], b[1]);
        s.c2[q] = make_float2(c[0], c[1]);
        s.dd[q] = make_float2(d[0], d[1]);
        s.vis[q] = make_float2(w[0], w[1]);
    }
    const unsigned mine = s.live;
    if (__syncthreads_count(mine != 0u) == 0) return;
    const double ox = sc.tx * kTile, oy = sc.ty * kTile;
    const float fx = static_cast<float>(sc.lx);
    blend_walk<PPT, STATS, kDf>(s, sb, raw, sc, vals, rec, range, lo, n_list, ox, oy, fx, nullptr, 1, v.width, v.height,
                                cnt);
#pragma unroll
    for (int p = 0; p < PPT; ++p) {
        if (!((mine >> p) & 1u)) continue;
        const int y = sc.py0 + p;
        const int q = p >> 1;
        const bool hi = p & 1;
        const size_t o = static_cast<size_t>(y) * v.width + sc.px;
        out_color[o] = hi ? s.c0[q].y : s.c0[q].x;
        out_color[P + o] = hi ? s.c1[q].y : s.c1[q].x;
        out_color[2 * P + o] = hi ? s.c2[q].y : s.c2[q].x;
        out_depth[o] = hi ? s.dd[q].y : s.dd[q].x;
        out_vis[o] = hi ? s.vis[q].y : s.vis[q].x;
        out_t[o] = hi ? s.T[q].y + s.Tl[q].y : s.T[q].x + s.Tl[q].x;
        out_nproc[o] = s.nproc[p];
        if (STATS) out_ncontrib[o] = s.ncontrib[p];
    }
}

static int g_ppt_override[2] = {0, 0};  // [forward, backward]; 0 = automatic
// tiles with longer lists use the df32 transmittance (measured crossover, diag/diag_fwd.py)
static int g_df_list = 1100;

void set_blend_df_list(int n) { g_df_list = n < 0 ? 1100 : n; }

static int g_nseg_override = 0;
void set_blend_segments(int n) { g_nseg_override = n; }
// segmented forward up to this many tiles (measured: it pays at the 320-tile level, where the
// sequential walk is latency-bound, and loses at 1280 tiles); 0 = never
static int g_seg_forward_tiles = 512;
void set_blend_seg_forward(int max_tiles) { g_seg_forward_tiles = max_tiles < 0 ? 512 : max_tiles; }

int blend_segments(const ViewParams& v) {
    if (g_nseg_override > 0) return g_nseg_override;
    // few tiles (long lists): split each list so the backward fills the GPU (measured with
    // diag/diag_fwd.py on the 1M-Gaussian 1280x1024 pyramid: 16 segments at the 320-tile level,
    // 8 at the 1280-tile level; none at full resolution)
    const int tiles = v.tiles_x * v.tiles_y;
    return tiles <= 512 ? 16 : tiles <= 2048 ? 8 : 1;
}

void set_blend_ppt(int fwd, int bwd) {
    g_ppt_override[0] = fwd;
    g_ppt_override[1] = bwd;
}

int blend_ppt(const ViewParams& v, bool backward) {
    const int o = g_ppt_override[backward ? 1 : 0];
    if (o == 1 || o == 2 || o == 4 || o == 8) return o;
    // measured on B200 (1M Gaussians, 1280x1024 pyramid, diag/diag_fwd.py): the forward wants
    // 2 pixels per thread at every level; the backward amortises its per-entry warp reduction
    // over 4 pixels (its parallelism at the coarse levels comes from the list segments)
    return backward ? 4 : 2;
}

int launch_blend_fwd(const uint2* ranges, const uint32_t* vals, const Splat* rec, const ViewParams& v,
                      float* color, float* depth, float* vis, float* t_final, int32_t* n_proc,
                      int32_t* n_contrib, bool stats, float* ck, int nseg, float* seg_scratch,
                      const unsigned long long* cnt, cudaStream_t st) {
    const int n_tiles = v.tiles_x * v.tiles_y;
    // the order is computed for every forward: the backward of the frame reads it too
    const uint32_t* order = tile_order(ranges, n_tiles);
    if (order) launch_tile_order(ranges, n_tiles, st);
    if (nseg > 1 && n_tiles <= g_seg_forward_tiles && seg_scratch) {
        const size_t P = static_cast<size_t>(v.width) * v.height;
        float* seg = seg_scratch;
        float* tl_plane = seg_scratch + static_cast<size_t>(nseg) * kSegFields * P;
        int32_t* star = reinterpret_cast<int32_t*>(tl_plane + P);
        const dim3 grid(n_tiles, nseg);
        if (stats) launch_pdl(fwd_seg_local_kernel<2, true>, grid, kTileThreads / 2, st, ranges, vals, rec, v, seg, nseg, cnt);
        else launch_pdl(fwd_seg_local_kernel<2, false>, grid, kTileThreads / 2, st, ranges, vals, rec, v, seg, nseg, cnt);
        launch_pdl(fwd_seg_chain_kernel, div_up(static_cast<int>(P), 256), 256, st, 
            ranges, v, seg, nseg, color, depth, vis, t_final, n_proc, stats ? n_contrib : nullptr, tl_plane, star, ck);
        if (stats)
            launch_pdl(fwd_seg_finish_kernel<2, true>, grid, kTileThreads / 2, st, 
                ranges, vals, rec, v, color, depth, vis, t_final, n_proc, n_contrib, tl_plane, star, nseg, cnt);
        else
            launch_pdl(fwd_seg_finish_kernel<2, false>, grid, kTileThreads / 2, st, 
                ranges, vals, rec, v, color, depth, vis, t_final, n_proc, n_contrib, tl_plane, star, nseg, cnt);
        return order ? 4 : 3;
    }
#ifndef GSB_FWD_SUB
#define GSB_FWD_SUB 1
#endif
#define GSB_FWD(P, S, B)                                                                                        \
    launch_pdl(blend_fwd_kernel<P, S, GSB_FWD_SUB, B>, n_tiles * GSB_FWD_SUB, kTileThreads / P / GSB_FWD_SUB, st,  \
               ranges, vals, rec, v, color, depth, vis, t_final, n_proc, n_contrib, g_df_list, ck, nseg, order, cnt)
    switch (blend_ppt(v, false)) {
        case 4:
            if (stats) GSB_FWD(4, true, GSB_FWD_MIN_BLOCKS); else GSB_FWD(4, false, GSB_FWD_MIN_BLOCKS);
            break;
        default:
            if (stats) GSB_FWD(2, true, GSB_FWD_MIN_BLOCKS);
            else if (n_tiles > kFwdWideTiles) GSB_FWD(2, false, kFwdWideBlocks);
            else GSB_FWD(2, false, GSB_FWD_MIN_BLOCKS);
    }
#undef GSB_FWD
    return order ? 2 : 1;  // launches
}

// Counting sort of the tiles by list length, descending, in buckets of 16 entries (ties in any
// order: the launch order does not change any tile's result). One CTA.
__global__ void __launch_bounds__(1024) tile_order_kernel(const uint2* __restrict__ ranges, int tiles,
                                                          uint32_t* __restrict__ order) {
    pdl_enter();
    constexpr int kBuckets = 1024;
    __shared__ uint32_t cnt[kBuckets];
    __shared__ uint32_t warp_tot[32];
    auto bucket = [&](int t) {
        const uint2 r = ranges[t];
        return kBuckets - 1 - static_cast<int>(min((r.y - r.x) >> 4, static_cast<uint32_t>(kBuckets - 1)));
    };
    cnt[threadIdx.x] = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < tiles; t += blockDim.x) atomicAdd(&cnt[bucket(t)], 1u);
    __syncthreads();
    // exclusive scan of the 1024 bucket counts (thread i owns bucket i)
    const uint32_t c = cnt[threadIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    uint32_t base = 0;
    for (int w = 0; w < warp; ++w) base += warp_tot[w];
    __syncthreads();
    cnt[threadIdx.x] = base + incl - c;
    __syncthreads();
    for (int t = threadIdx.x; t < tiles; t += blockDim.x) order[atomicAdd(&cnt[bucket(t)], 1u)] = static_cast<uint32_t>(t);
}

void launch_tile_order(const uint2* ranges, int tiles, cudaStream_t st) {
    launch_pdl(tile_order_kernel, 1, 1024, st, ranges, tiles,
               const_cast<uint32_t*>(reinterpret_cast<const uint32_t*>(ranges + tiles)));
}

}  // namespace gsb
