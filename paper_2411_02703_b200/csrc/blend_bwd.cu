// K7: reverse replay of the blend (rasterizer.cpp:253-315). Per pixel, walk its contributors
// back to front, reconstructing T_i = T_{i+1} / (1 - alpha_i) from the forward's T_final. The
// suffix sums enter dalpha only through B = dC.S_c + dD.S_d, so one running scalar replaces the
// four suffix sums:
//   dalpha_i = T_i (dC.c_i + dD.z_i) - B / (1 - alpha_i);   B += w_i (dC.c_i + dD.z_i).
// Each (tile, Gaussian) pair's 10 cotangent sums are reduced per warp (staged rows summed over
// the lanes), across the CTA's warps in shared memory, and written once to the pair's emission
// slot: deterministic,
// no global atomics; K8 sums a Gaussian's slots in fp64. Partials 5-6 (mean) and 7-9
// (covariance) carry the staged conic's exp2 scale k and k^2 and omit the opacity factor (op,
// op / 2); K8 applies both in fp64.
#include "blend_common.cuh"
#include "kernels.cuh"

#ifndef GSB_BWD_MIN_BLOCKS
#define GSB_BWD_MIN_BLOCKS 1
#endif

namespace gsb {

namespace {

constexpr int kBwdBatch = 32;
// Per-warp reduction buffer: a processed entry's 10 per-lane sums are staged as rows of 32 lanes
// (stride 36 floats: 16-byte aligned, conflict-free float4 reads), and every kFlush entries the
// warp sums each row over its lanes (lane i takes rows i, i + 32, ...). No shuffles or selects.
// 6 entries per flush: 60 rows over 32 lanes is 2 full passes (4 entries left the second pass
// a quarter full); measured -4% on the kernel against 4, equal to 8 (whose PPT2 build overflows
// the 48 KB static shared memory)
constexpr int kFlush = 6;
constexpr int kRowStride = 36;

}  // namespace

template <int PPT>
__global__ void __launch_bounds__(kTileThreads / PPT, GSB_BWD_MIN_BLOCKS) blend_bwd_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals, const Splat* __restrict__ rec,
    const uint32_t* __restrict__ emit_off, ViewParams v, const float* __restrict__ t_final,
    const int32_t* __restrict__ n_proc, const float* __restrict__ dl_dcolor,
    const float* __restrict__ dl_ddepth, const float* __restrict__ depth_scale, float* __restrict__ partials,
    const unsigned long long* __restrict__ cnt, const float* __restrict__ ck, int nseg,
    const float* __restrict__ color_final, const float* __restrict__ depth_final, const uint32_t* __restrict__ order) {
    pdl_enter();
    if (overflowed(cnt)) return;  // pair capacity exceeded: the host re-runs the step
    using S = Strip<PPT>;
    constexpr int NT = S::kThreads, NW = NT / 32, NP = (PPT + 1) / 2;  // PPT = 1: high half never live
    __shared__ StageBuf<kBwdBatch> sb;
    __shared__ uint32_t s_slot[kBwdBatch];
    __shared__ uint32_t s_mask[NW];
    __shared__ float s_red[NW > 1 ? NW : 1][kBwdBatch][kNumPartials];
    __shared__ int s_max[NW];
    __shared__ __align__(16) float s_pv[NW][kFlush][kNumPartials][kRowStride];
    __shared__ int s_pk[NW][kFlush];
    const int tile = order ? static_cast<int>(order[blockIdx.x]) : static_cast<int>(blockIdx.x);
    const S sc(v.tiles_x, tile, threadIdx.x >> 5);
    // sums the warp's staged rows over its lanes and stores them per (entry, partial)
    auto flush = [&](int nb) {
        __syncwarp();
        for (int idx = sc.lane; idx < nb * kNumPartials; idx += 32) {
            const int e = idx / kNumPartials, c = idx - e * kNumPartials;
            const float4* row = reinterpret_cast<const float4*>(&s_pv[sc.warp][e][c][0]);
            float4 a = row[0];
#pragma unroll
            for (int i = 1; i < 8; ++i) {
                const float4 b = row[i];
                const float2 lo = __fadd2_rn(make_float2(a.x, a.y), make_float2(b.x, b.y));
                const float2 hi = __fadd2_rn(make_float2(a.z, a.w), make_float2(b.z, b.w));
                a = make_float4(lo.x, lo.y, hi.x, hi.y);
            }
            const float tot = (a.x + a.y) + (a.z + a.w);
            const int k = s_pk[sc.warp][e];
            if (NW == 1) partials[static_cast<size_t>(s_slot[k]) * kNumPartials + c] = tot;
            else s_red[sc.warp][k][c] = tot;
        }
        __syncwarp();
    };
    const uint2 range = ranges[tile];
    [[maybe_unused]] const unsigned long long* const counters = cnt;  // (the batch loop's `cnt` is its entry count)
    GSB_CHECK(range.x <= range.y && range.y <= counters[kCntPairs]);
    // this CTA's list segment [lo_s, hi_s) (blockIdx.y); the whole list when nseg = 1
    const int n_list = static_cast<int>(range.y - range.x);
    const int L = seg_len(n_list, nseg);
    const int lo_s = static_cast<int>(blockIdx.y) * L;
    if (lo_s >= n_list) return;  // whole CTA (before any barrier)
    const int hi_s = min(lo_s + L, n_list);
    const double ox = sc.tx * kTile, oy = sc.ty * kTile;
    const float fx = static_cast<float>(sc.lx);
    const float dscale = dl_ddepth ? (depth_scale ? *depth_scale : 1.f) : 0.f;
    const size_t P = static_cast<size_t>(v.width) * v.height;

    float2 T[NP], B[NP], g0[NP], g1[NP], g2[NP], gz[NP];
    int last[2 * NP];
    int my_last = lo_s;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        float t[2] = {0.f, 0.f}, a[2] = {0.f, 0.f}, b[2] = {0.f, 0.f}, c[2] = {0.f, 0.f}, z[2] = {0.f, 0.f};
        float bb[2] = {0.f, 0.f};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int p = 2 * q + h, y = sc.py0 + p;
            last[p] = 0;
            if (p < PPT && sc.px < v.width && y < v.height) {
                const size_t o = static_cast<size_t>(y) * v.width + sc.px;
                last[p] = n_proc[o];
                a[h] = dl_dcolor[o];
                b[h] = dl_dcolor[P + o];
                c[h] = dl_dcolor[2 * P + o];
                z[h] = dl_ddepth ? dl_ddepth[o] * dscale : 0.f;
                // rasterizer.cpp:264: a pixel with an all-zero cotangent contributes nothing
                if (a[h] == 0.f && b[h] == 0.f && c[h] == 0.f && z[h] == 0.f) last[p] = 0;
                if (last[p] > hi_s) {
                    // contributions continue past this segment: start from the forward's state
                    // before entry hi_s, with B = the cotangent-weighted colour / depth still to come
                    const float* cp = ck + static_cast<size_t>(hi_s / L - 1) * kCkFields * P;
                    t[h] = cp[o];
                    bb[h] = a[h] * (color_final[o] - cp[P + o]) + b[h] * (color_final[P + o] - cp[2 * P + o]) +
                            c[h] * (color_final[2 * P + o] - cp[3 * P + o]) + z[h] * (depth_final[o] - cp[4 * P + o]);
                } else {
                    t[h] = t_final[o];
                }
            }
            my_last = max(my_last, min(last[p], hi_s));
        }
        T[q] = make_float2(t[0], t[1]);
        B[q] = make_float2(bb[0], bb[1]);
        g0[q] = make_float2(a[0], a[1]);
        g1[q] = make_float2(b[0], b[1]);
        g2[q] = make_float2(c[0], c[1]);
        gz[q] = make_float2(z[0], z[1]);
    }
    int max_last = __reduce_max_sync(0xffffffffu, my_last);
    if (NW > 1) {
        if (sc.lane == 0) s_max[sc.warp] = max_last;
        __syncthreads();
        max_last = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) max_last = max(max_last, s_max[w]);
    }
    // entries of the segment no pixel reached still own a partial slot: zero it
    for (int j = max_last + threadIdx.x; j < hi_s; j += NT) {
        const uint32_t r = vals[range.x + j];
        GSB_CHECK(r < counters[kCntVisible]);
        const uint32_t slot = emission_index(rec[r], emit_off[r], sc.tx, sc.ty);
        GSB_CHECK(slot >= emit_off[r] && slot < emit_off[r + 1] && slot < counters[kCntPairs]);
        float2* dst = reinterpret_cast<float2*>(partials + static_cast<size_t>(slot) * kNumPartials);
#pragma unroll
        for (int k = 0; k < kNumPartials / 2; ++k) dst[k] = make_float2(0.f, 0.f);
    }

    // the next batch's records are loaded one batch ahead (their dependent global loads overlap
    // the current batch's walk)
    Splat nsp;
    uint32_t noff = 0;
    if (max_last > lo_s && threadIdx.x < max_last - max(lo_s, max_last - kBwdBatch)) {
        const uint32_t r = vals[range.x + max(lo_s, max_last - kBwdBatch) + threadIdx.x];
        nsp = rec[r];
        noff = emit_off[r];
    }
    for (int hi = max_last; hi > lo_s; hi -= kBwdBatch) {
        const int lo = max(lo_s, hi - kBwdBatch);
        const int cnt = hi - lo;
        if (NW > 1) __syncthreads();
        if (threadIdx.x < cnt) {
            sb.put(threadIdx.x, stage_of(nsp, ox, oy));
            s_slot[threadIdx.x] = emission_index(nsp, noff, sc.tx, sc.ty);
            GSB_CHECK(s_slot[threadIdx.x] < counters[kCntPairs]);
        }
        {
            const int nlo = max(lo_s, lo - kBwdBatch);
            if (threadIdx.x < lo - nlo) {
                const uint32_t r = vals[range.x + nlo + threadIdx.x];
                GSB_CHECK(r < counters[kCntVisible]);
                nsp = rec[r];
                noff = emit_off[r];
            }
        }
        if (sc.lane == 0) s_mask[sc.warp] = 0u;
        // bounding box of this warp's pixels whose contributor range reaches into the batch
        unsigned act = 0u;
#pragma unroll
        for (int p = 0; p < 2 * NP; ++p)
            if (last[p] > lo) act |= 1u << p;
        const int4 ab = warp_bbox<PPT>(act, sc);
        if (NW > 1) __syncthreads(); else __syncwarp();
        // ballot the staged entries that meet the box, walk them back to front
        unsigned todo = __ballot_sync(0xffffffffu, sc.lane < cnt && rect_meets(sb.rect[sc.lane], ab));
        int nb = 0;  // entries staged in s_pv (warp-uniform)
        while (todo) {
            const int k = 31 - __clz(todo);
            todo &= ~(1u << k);
            const int4 rc = sb.rect[k];
            const int j = lo + k;
            const bool colin = sc.px >= rc.x && sc.px <= rc.z;
            const float2 m = sb.mean[k];
            const float4 cn = sb.con[k];
            const float4 col = sb.col[k];
            float2 acc[kNumPartials];  // the first pixel pair initialises (no additions of 0)
            bool any = false;
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                const int p0 = 2 * q, y0 = sc.py0 + p0;
                const bool a0 = colin && j < last[p0] && y0 >= rc.y && y0 <= rc.w;
                const bool a1 = colin && j < last[p0 + 1] && y0 + 1 >= rc.y && y0 + 1 <= rc.w;
                // no branch on (a0 || a1): inactive halves contribute exact zeros (al = 0 ->
                // w = 0, gd = 0, T kept), and the pairs of a thread stay independent for ILP
                any |= a0 || a1;
                const float fy = static_cast<float>(sc.ly0 + p0);
                const AlphaP e = alpha_pair(m, cn, fx, make_float2(fy, fy + 1.f));
                const float2 al = make_float2(a0 ? e.alpha.x : 0.f, a1 ? e.alpha.y : 0.f);
                const float2 om = __fadd2_rn(f2(1.f), neg2(al));
                const float2 inv = make_float2(rcp_approx(om.x), rcp_approx(om.y));
                const float2 ti = __fmul2_rn(T[q], inv);
                const float2 w = __fmul2_rn(al, ti);
                const float2 A = __ffma2_rn(g0[q], f2(col.x),
                                            __ffma2_rn(g1[q], f2(col.y),
                                                       __ffma2_rn(g2[q], f2(col.z), __fmul2_rn(gz[q], f2(col.w)))));
                const float2 dalpha = __ffma2_rn(ti, A, __fmul2_rn(neg2(inv), B[q]));
                B[q] = __ffma2_rn(w, A, B[q]);
                // an inactive half has al = 0 -> om = 1 -> rcp.approx(1) = 1 exactly -> ti = T
                T[q] = ti;
                // rasterizer.cpp:297: the clamp is flat -> no opacity / mean / covariance terms
                const float2 gdr = __fmul2_rn(e.g, dalpha);
                const float2 gd = make_float2(a0 && e.a_raw.x < kAlphaMaxF ? gdr.x : 0.f,
                                              a1 && e.a_raw.y < kAlphaMaxF ? gdr.y : 0.f);
                // mean / covariance terms without the opacity (K8 applies op and op / 2)
                const float2 h0 = __fmul2_rn(gd, e.u0);
                const float2 h1 = __fmul2_rn(gd, e.u1);
                if (q == 0) {
                    acc[0] = __fmul2_rn(w, g0[q]);
                    acc[1] = __fmul2_rn(w, g1[q]);
                    acc[2] = __fmul2_rn(w, g2[q]);
                    acc[3] = __fmul2_rn(w, gz[q]);
                    acc[4] = gd;
                    acc[5] = h0;
                    acc[6] = h1;
                    acc[7] = __fmul2_rn(h0, e.u0);
                    acc[8] = __fmul2_rn(h0, e.u1);
                    acc[9] = __fmul2_rn(h1, e.u1);
                } else {
                    acc[0] = __ffma2_rn(w, g0[q], acc[0]);
                    acc[1] = __ffma2_rn(w, g1[q], acc[1]);
                    acc[2] = __ffma2_rn(w, g2[q], acc[2]);
                    acc[3] = __ffma2_rn(w, gz[q], acc[3]);
                    acc[4] = __fadd2_rn(acc[4], gd);
                    acc[5] = __fadd2_rn(acc[5], h0);
                    acc[6] = __fadd2_rn(acc[6], h1);
                    acc[7] = __ffma2_rn(h0, e.u0, acc[7]);
                    acc[8] = __ffma2_rn(h0, e.u1, acc[8]);
                    acc[9] = __ffma2_rn(h1, e.u1, acc[9]);
                }
            }
            if (!__any_sync(0xffffffffu, any)) continue;
#pragma unroll
            for (int c = 0; c < kNumPartials; ++c) s_pv[sc.warp][nb][c][sc.lane] = acc[c].x + acc[c].y;
            if (sc.lane == 0) {
                s_pk[sc.warp][nb] = k;
                s_mask[sc.warp] |= 1u << k;
            }
            if (++nb == kFlush) {
                flush(nb);
                nb = 0;
            }
        }
        if (nb) flush(nb);
        nb = 0;
        if (NW == 1) {
            __syncwarp();
            // entries of this batch the warp never reduced (no pixel of the tile hit them)
            for (int k = sc.lane; k < cnt; k += 32)
                if (!((s_mask[0] >> k) & 1u)) {
                    float2* dst = reinterpret_cast<float2*>(partials + static_cast<size_t>(s_slot[k]) * kNumPartials);
#pragma unroll
                    for (int c = 0; c < kNumPartials / 2; ++c) dst[c] = make_float2(0.f, 0.f);
                }
            __syncwarp();
        } else {
            __syncthreads();
            for (int t = threadIdx.x; t < cnt * kNumPartials; t += NT) {
                const int k = t / kNumPartials, c = t - k * kNumPartials;
                float a = 0.f;
#pragma unroll
                for (int w = 0; w < NW; ++w)
                    if ((s_mask[w] >> k) & 1u) a += s_red[w][k][c];
                partials[static_cast<size_t>(s_slot[k]) * kNumPartials + c] = a;
            }
        }
    }
}

void launch_blend_bwd(const uint2* ranges, const uint32_t* vals, const Splat* rec, const uint32_t* emit_off,
                      const ViewParams& v, const float* t_final, const int32_t* n_proc,
                      const float* dl_dcolor, const float* dl_ddepth, const float* depth_scale,
                      float* partials, const unsigned long long* cnt, const float* ck, int nseg,
                      const float* color, const float* depth, cudaStream_t st) {
    const dim3 n_tiles(v.tiles_x * v.tiles_y, nseg);
    const uint32_t* order = tile_order(ranges, v.tiles_x * v.tiles_y);
    // 4 pixels per thread (2 warps per tile) unless overridden to 2 (4 warps per tile)
    if (blend_ppt(v, true) == 2)
        launch_pdl(blend_bwd_kernel<2>, n_tiles, 128, st, ranges, vals, rec, emit_off, v, t_final, n_proc, dl_dcolor,
                                                     dl_ddepth, depth_scale, partials, cnt, ck, nseg, color, depth, order);
    else
        launch_pdl(blend_bwd_kernel<4>, n_tiles, 64, st, ranges, vals, rec, emit_off, v, t_final, n_proc, dl_dcolor,
                                                    dl_ddepth, depth_scale, partials, cnt, ck, nseg, color, depth, order);
}

}  // namespace gsb
