// K2-K4 sorts, hand-written for sm_100a (replaces the library radix sorts): the (depth, index)
// order of the visible Gaussians (rasterizer.cpp:69-72) and the stable (tile, depth rank) order
// of the duplicated keys with the tile ranges (bin_tiles, rasterizer.cpp:76-91).
//
// Every kernel takes its element count from the frame's device counters, so nothing waits for
// the host and the buffers can be sized generously at no cost: a sort of 300k visible
// Gaussians costs the same whether its buffers hold 1M or 4M entries.
//
// LSD radix sort, one pass per digit ("onesweep"): a persistent grid takes tiles of 2048 keys
// in order from an atomic ticket; each tile ranks its keys stably (warp match + per-warp digit
// counters), publishes its per-digit counts and resolves the counts of all earlier tiles by
// decoupled look-back on 64-bit status words (value | flag | epoch: the epoch is unique per pass,
// so the status array is never cleared), reorders the tile in shared memory by digit and writes
// each digit run contiguously. The digit histograms of every pass come from one upfront read of
// the keys (depth) or from the pair emission itself (tiles).
#include "kernels.cuh"
#include "sort.cuh"

namespace gsb {

namespace {

constexpr int NT = kSortThreads, NW = NT / 32, IT = kSortItems, TILE = kSortTile;
static_assert(NT == kRadix, "one thread per digit in the look-back");

constexpr uint32_t kFlagAgg = 1u, kFlagPrefix = 2u;

// (the kernels below are chained with programmatic dependent launch: pdl_enter, common.cuh)

__device__ __forceinline__ unsigned long long pack_status(uint32_t epoch, uint32_t flag, uint32_t value) {
    return (static_cast<unsigned long long>(epoch) << 34) | (static_cast<unsigned long long>(flag) << 32) | value;
}

__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Sum of the values of tiles [0, tile) for one lane of the status array (`stride` words per
// tile), after publishing this tile's own `value` as an aggregate; then publishes the inclusive
// prefix. Waits only on lower tiles, which were ticketed earlier by running CTAs. The walk reads
// a window of kLookWin predecessors per round trip (independent loads in flight together), so
// the chain of dependent L2 round trips is ~tile / kLookWin long instead of ~tile.
#ifndef GSB_LOOKBACK_WIN
#define GSB_LOOKBACK_WIN 8
#endif
constexpr int kLookWin = GSB_LOOKBACK_WIN;

__device__ __forceinline__ uint32_t look_back(unsigned long long* status, uint32_t tile, int stride, uint32_t epoch,
                                              uint32_t value) {
    unsigned long long* my = status + static_cast<size_t>(tile) * stride;
    if (tile == 0) {
        st_relaxed(my, pack_status(epoch, kFlagPrefix, value));
        return 0u;
    }
    st_relaxed(my, pack_status(epoch, kFlagAgg, value));
    uint32_t excl = 0;
    int j = static_cast<int>(tile) - 1;
    for (;;) {
        unsigned long long s[kLookWin];
#pragma unroll
        for (int w = 0; w < kLookWin; ++w)
            s[w] = j - w >= 0 ? ld_relaxed(status + static_cast<size_t>(j - w) * stride) : 0ull;
        // take the published predecessors nearest first, up to the first inclusive prefix; stop
        // at the first one not yet published in this pass and poll again from there
        int adv = 0;
        bool done = false, stall = false;
#pragma unroll
        for (int w = 0; w < kLookWin; ++w) {
            if (done || stall) continue;
            const unsigned long long x = s[w];
            if (j - w < 0 || static_cast<uint32_t>(x >> 34) != epoch) {
                stall = true;
            } else {
                excl += static_cast<uint32_t>(x);
                ++adv;
                done = ((x >> 32) & 3u) == kFlagPrefix;
            }
        }
        if (done) break;
        j -= adv;
    }
    st_relaxed(my, pack_status(epoch, kFlagPrefix, excl + value));
    return excl;
}

// The same for one status word per tile, walked by a whole warp: lane l reads predecessor
// j - l, so one round trip covers 32 tiles. Every lane returns the exclusive prefix.
__device__ __forceinline__ uint32_t look_back_warp(unsigned long long* status, uint32_t tile, uint32_t epoch,
                                                   uint32_t value) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) st_relaxed(status, pack_status(epoch, kFlagPrefix, value));
        return 0u;
    }
    if (lane == 0) st_relaxed(status + tile, pack_status(epoch, kFlagAgg, value));
    uint32_t excl = 0;
    int j = static_cast<int>(tile) - 1;
    for (;;) {
        const int idx = j - lane;
        const unsigned long long x = idx >= 0 ? ld_relaxed(status + idx) : pack_status(epoch, kFlagPrefix, 0u);
        const bool ready = static_cast<uint32_t>(x >> 34) == epoch;
        const unsigned nr = __ballot_sync(0xffffffffu, !ready);
        const unsigned pre = __ballot_sync(0xffffffffu, ready && ((x >> 32) & 3u) == kFlagPrefix);
        const int first_nr = nr ? __ffs(nr) - 1 : 32;
        const int first_pre = pre ? __ffs(pre) - 1 : 32;
        if (first_pre < first_nr) {
            excl += __reduce_add_sync(0xffffffffu, lane <= first_pre ? static_cast<uint32_t>(x) : 0u);
            break;
        }
        excl += __reduce_add_sync(0xffffffffu, lane < first_nr ? static_cast<uint32_t>(x) : 0u);
        j -= first_nr;
    }
    if (lane == 0) st_relaxed(status + tile, pack_status(epoch, kFlagPrefix, excl + value));
    return excl;
}

// exclusive scan of one value per thread over the CTA (NT threads); *total = sum of all
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* s_warp, uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    uint32_t wo = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        const uint32_t t = s_warp[w];
        wo += w < warp ? t : 0u;
        tot += t;
    }
    __syncthreads();
    *total = tot;
    return wo + inc - x;
}

__device__ __forceinline__ uint32_t clamp_count(const unsigned long long* count, uint32_t cap) {
    const unsigned long long c = *count;
    return c > cap ? 0u : static_cast<uint32_t>(c);  // an overflowed count sorts nothing
}

}  // namespace

// ------------------------------------------------------------------------------------------
// one LSD pass over digit (key >> shift) & (2^bits - 1); hist = this pass's digit histogram
template <typename KeyT, bool KEYS_OUT>
// the 32-bit (depth) passes with an explicit 1-CTA bound (ptxas then allocates for it: -5% on the
// depth sort), the 16-bit (tile) passes unconstrained (the same bound costs them +10%); a 0
// bound emits no .minnctapersm (diag/variant_levels.sh)
__global__ void __launch_bounds__(NT, sizeof(KeyT) == 4 ? 1 : 0) onesweep_kernel(const KeyT* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                      KeyT* __restrict__ kout, uint32_t* __restrict__ vout,
                                                      const unsigned long long* __restrict__ count, uint32_t cap,
                                                      int shift, int bits, const uint32_t* __restrict__ hist,
                                                      uint32_t* __restrict__ ticket,
                                                      unsigned long long* __restrict__ status, uint32_t epoch) {
    pdl_enter();
    __shared__ uint32_t s_base[kRadix], s_tstart[kRadix], s_run[kRadix];
    __shared__ uint32_t s_whist[NW][kRadix];
    __shared__ uint32_t s_warp[NW];
    __shared__ KeyT s_keys[TILE];
    __shared__ uint32_t s_vals[TILE];
    __shared__ uint32_t s_tile;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t n = clamp_count(count, cap);
    const uint32_t ntiles = (n + TILE - 1) / TILE;
    const uint32_t ndig = 1u << bits, mask = ndig - 1u;
    {
        uint32_t tot;
        s_base[tid] = block_excl_scan(static_cast<uint32_t>(tid) < ndig ? hist[tid] : 0u, s_warp, &tot);
    }
    const uint32_t lt = (1u << lane) - 1u;
    for (;;) {
        if (tid == 0) s_tile = atomicAdd(ticket, 1u);
        for (int i = tid; i < NW * kRadix; i += NT) (&s_whist[0][0])[i] = 0u;
        __syncthreads();
        const uint32_t tile = s_tile;
        if (tile >= ntiles) break;
        const uint32_t t0 = tile * TILE;
        KeyT key[IT];
        uint32_t val[IT], dig[IT], rnk[IT];
        // warp-striped: item i of lane l is element t0 + warp*32*IT + 32 i + l (index order =
        // (i, lane) order, which the ranking below preserves)
#pragma unroll
        for (int i = 0; i < IT; ++i) {
            const uint32_t idx = t0 + warp * (32 * IT) + i * 32 + lane;
            if (idx < n) {
                key[i] = kin[idx];
                val[i] = vin[idx];
                dig[i] = (static_cast<uint32_t>(key[i]) >> shift) & mask;
            } else {
                key[i] = 0;
                val[i] = 0u;
                dig[i] = kRadix;  // past the count: neither ranked nor written
            }
        }
#pragma unroll
        for (int i = 0; i < IT; ++i) {
            const uint32_t peers = __match_any_sync(0xffffffffu, dig[i]);
            const int leader = 31 - __clz(peers);
            uint32_t b = 0u;
            if (lane == leader && dig[i] < kRadix) {
                b = s_whist[warp][dig[i]];
                s_whist[warp][dig[i]] = b + __popc(peers);
            }
            b = __shfl_sync(0xffffffffu, b, leader);
            rnk[i] = b + __popc(peers & lt);
            __syncwarp();
        }
        __syncthreads();
        // per digit (thread = digit): offsets of the warps, tile count, earlier tiles' count
        uint32_t tot = 0u;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const uint32_t c = s_whist[w][tid];
            s_whist[w][tid] = tot;
            tot += c;
        }
        uint32_t before = 0u;
        if (static_cast<uint32_t>(tid) < ndig) before = look_back(status + tid, tile, kRadix, epoch, tot);
        uint32_t ttot;
        const uint32_t ts = block_excl_scan(tot, s_warp, &ttot);
        s_tstart[tid] = ts;
        s_run[tid] = s_base[tid] + before - ts;  // global position of local slot j of digit tid = s_run + j
        __syncthreads();
#pragma unroll
        for (int i = 0; i < IT; ++i) {
            if (dig[i] < kRadix) {
                const uint32_t lp = s_tstart[dig[i]] + s_whist[warp][dig[i]] + rnk[i];
                GSB_CHECK(lp < static_cast<uint32_t>(TILE));
                s_keys[lp] = key[i];
                s_vals[lp] = val[i];
            }
        }
        __syncthreads();
        const uint32_t tn = min(static_cast<uint32_t>(TILE), n - t0);
        for (uint32_t j = tid; j < tn; j += NT) {
            const KeyT k = s_keys[j];
            const uint32_t g = s_run[(static_cast<uint32_t>(k) >> shift) & mask] + j;
            GSB_CHECK(g < n);
            if (KEYS_OUT) kout[g] = k;
            vout[g] = s_vals[j];
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------------
// digit histograms of `passes` 8-bit passes over 32-bit keys (the depth sort), one read
__global__ void __launch_bounds__(NT) radix_hist_kernel(const uint32_t* __restrict__ keys,
                                                        const unsigned long long* __restrict__ count, uint32_t cap,
                                                        int passes, uint32_t* __restrict__ hist) {
    pdl_enter();
    __shared__ uint32_t s[4][kRadix];
    for (int i = threadIdx.x; i < 4 * kRadix; i += NT) (&s[0][0])[i] = 0u;
    __syncthreads();
    const uint32_t n = clamp_count(count, cap);
    for (uint32_t i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
        const uint32_t k = keys[i];
        for (int p = 0; p < passes; ++p) atomicAdd(&s[p][(k >> (8 * p)) & 0xffu], 1u);
    }
    __syncthreads();
    for (int p = 0; p < passes; ++p) {
        const uint32_t c = s[p][threadIdx.x];
        if (c) atomicAdd(&hist[p * kRadix + threadIdx.x], c);
    }
}

// ------------------------------------------------------------------------------------------
// Exact (fp64 depth, map index) order inside runs of equal 24-bit keys (the key is a monotone
// function of the fp64 depth, so only equal-key runs can be out of order). Runs are common
// (fp32 positions under an axis-aligned pose give exactly equal depths; C3 has runs of up to
// ~40), so every element of a run computes its own rank in the run by comparing against all
// members (independent loads, the same addresses across the run's lanes) and scatters itself to
// run start + rank; elements outside runs are copied. Out of place: gid_in -> gid_out.
__global__ void __launch_bounds__(NT) fix_ties_kernel(const uint32_t* __restrict__ key,
                                                      const int32_t* __restrict__ gid_in,
                                                      const unsigned long long* __restrict__ depth,
                                                      const unsigned long long* __restrict__ cnt,
                                                      int32_t* __restrict__ gid_out) {
    pdl_enter();
    const int n = static_cast<int>(cnt[kCntVisible]);
    for (int p = blockIdx.x * NT + threadIdx.x; p < n; p += gridDim.x * NT) {
        const uint32_t k = key[p];
        const int g = gid_in[p];
        if (!((p > 0 && key[p - 1] == k) || (p + 1 < n && key[p + 1] == k))) {
            gid_out[p] = g;
            continue;
        }
        int s = p, e = p + 1;
        while (s > 0 && key[s - 1] == k) --s;
        while (e < n && key[e] == k) ++e;
        const unsigned long long d = depth[g];
        int r = 0;
#pragma unroll 4
        for (int q = s; q < e; ++q) {
            const int gq = gid_in[q];
            const unsigned long long dq = depth[gq];
            r += (dq < d || (dq == d && gq < g)) ? 1 : 0;
        }
        GSB_CHECK(s + r < e);  // the run members' ranks are a permutation of [0, e - s)
        gid_out[s + r] = g;
    }
}

// ------------------------------------------------------------------------------------------
// Rank-ordered copy of the projected records (the reference's sorted `projected` vector) fused
// with the exclusive scan of their tile counts: emit_off[r] = first (tile, Gaussian) pair of
// rank r, emit_off[n_vis] = total pairs; also rank_of[map index] = rank for K8. Tiles of
// 4 x NT ranks (4 consecutive per thread), one look-back word per tile (walked by a warp).
constexpr int kPackItems = 4;

#ifndef GSB_PACK_MIN_BLOCKS
#define GSB_PACK_MIN_BLOCKS 2  // 2 resident CTAs per SM (from 118 to 96 registers): -6% on K2 + pack
#endif
__global__ void __launch_bounds__(NT, GSB_PACK_MIN_BLOCKS) pack_scan_kernel(const int32_t* __restrict__ gid_sorted,
                                                       const Splat* __restrict__ rec_by_gid,
                                                       const unsigned long long* __restrict__ depth_by_gid,
                                                       const unsigned long long* __restrict__ cnt,
                                                       Splat* __restrict__ rec_sorted,
                                                       unsigned long long* __restrict__ depth_sorted,
                                                       int32_t* __restrict__ rank_of,
                                                       uint32_t* __restrict__ emit_off, uint32_t* __restrict__ ticket,
                                                       unsigned long long* __restrict__ status, uint32_t epoch) {
    pdl_enter();
    constexpr int PT = kPackItems * NT;
    static_assert(kPackItems == 4, "one 16-byte load / store of ranks per thread");
    __shared__ uint32_t s_warp[NW];
    __shared__ uint32_t s_tile, s_before;
    __shared__ uint32_t s_nt[NW][32 * kPackItems];  // tile counts of each warp's records
    const int tid = threadIdx.x;
    const uint32_t nv = static_cast<uint32_t>(cnt[kCntVisible]);
    const uint32_t ntiles = (nv + PT - 1) / PT;
    if (nv == 0 && blockIdx.x == 0 && tid == 0) emit_off[0] = 0u;
    for (;;) {
        if (tid == 0) s_tile = atomicAdd(ticket, 1u);
        __syncthreads();
        const uint32_t tile = s_tile;
        if (tile >= ntiles) break;
        // blocked: thread t owns ranks r0 .. r0 + 3 (one 16-byte load of the sorted map indices)
        const uint32_t r0 = tile * PT + kPackItems * tid;
        int g[kPackItems];
        if (r0 + kPackItems <= nv) {
            const int4 q = *reinterpret_cast<const int4*>(gid_sorted + r0);
            g[0] = q.x; g[1] = q.y; g[2] = q.z; g[3] = q.w;
        } else {
#pragma unroll
            for (int i = 0; i < kPackItems; ++i) g[i] = r0 + i < nv ? gid_sorted[r0 + i] : -1;
        }
        // the warp's 128 records are copied cooperatively: per instruction 8 records, 4 lanes per
        // record (16 bytes each) -> each 64-byte record read whole and 512 contiguous bytes written
        // (a per-thread copy of its own 4 records scatters every store instruction over 32 rows)
        {
            const int lane = tid & 31;
            const uint32_t wr0 = tile * PT + kPackItems * (tid & ~31);  // the warp's first rank
            const int item = (lane >> 2) & 3, chunk = lane & 3;
            uint4 buf[16];
            int dst[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int owner = 2 * j + (lane >> 4);  // record k = 8 j + lane / 4 = 4 owner + item
                int gi = __shfl_sync(0xffffffffu, g[0], owner);
                const int g1 = __shfl_sync(0xffffffffu, g[1], owner);
                const int g2 = __shfl_sync(0xffffffffu, g[2], owner);
                const int g3 = __shfl_sync(0xffffffffu, g[3], owner);
                gi = item == 1 ? g1 : item == 2 ? g2 : item == 3 ? g3 : gi;
                dst[j] = gi;
                if (gi >= 0) buf[j] = reinterpret_cast<const uint4*>(rec_by_gid + gi)[chunk];
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const uint32_t k = 8 * j + (lane >> 2);
                if (dst[j] >= 0) {
                    reinterpret_cast<uint4*>(rec_sorted + wr0 + k)[chunk] = buf[j];
                    if (chunk == 3) s_nt[tid >> 5][k] = buf[j].w;  // Splat::ntiles
                }
            }
            __syncwarp();
        }
        uint32_t nt[kPackItems];
        uint32_t mine = 0u;
#pragma unroll
        for (int i = 0; i < kPackItems; ++i) {
            nt[i] = 0u;
            if (g[i] >= 0) {
                depth_sorted[r0 + i] = depth_by_gid[g[i]];
                rank_of[g[i]] = static_cast<int32_t>(r0 + i);
                nt[i] = s_nt[tid >> 5][kPackItems * (tid & 31) + i];
            }
            mine += nt[i];
        }
        uint32_t carry;
        const uint32_t loc = block_excl_scan(mine, s_warp, &carry);
        if (tid < 32) {
            const uint32_t b = look_back_warp(status, tile, epoch, carry);  // (carry is CTA-uniform)
            if (tid == 0) s_before = b;
        }
        __syncthreads();
        uint32_t o[kPackItems + 1];
        o[0] = s_before + loc;
#pragma unroll
        for (int i = 0; i < kPackItems; ++i) o[i + 1] = o[i] + nt[i];
        if (r0 + kPackItems <= nv) {
            *reinterpret_cast<uint4*>(emit_off + r0) = make_uint4(o[0], o[1], o[2], o[3]);
        } else {
#pragma unroll
            for (int i = 0; i < kPackItems; ++i)
                if (r0 + i < nv) emit_off[r0 + i] = o[i];
        }
#pragma unroll
        for (int i = 0; i < kPackItems; ++i)
            if (r0 + i == nv - 1) emit_off[nv] = o[i + 1];
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------------
// Duplicate-key emission (bin_tiles, rasterizer.cpp:76-91): a warp owns 32 consecutive depth
// ranks, whose pairs are contiguous in the scan, and writes them 32 pairs at a time, one per
// lane (each lane finds its pair's rank by a shuffle search; row/column of the tile rect by a
// magic-number multiply). Keys are tile ids, values depth
// ranks, so the stable sort by tile yields each tile's list in (depth, index) order — the
// reference's push_back order. Persistent grid; also builds the digit histograms of the tile
// sort's passes (low `b0` bits, then the rest). Pairs beyond the capacity raise the overflow
// flag instead (nothing is written).
template <typename KeyT>
__global__ void __launch_bounds__(NT) emit_pairs_kernel(const uint32_t* __restrict__ emit_off,
                                                        const Splat* __restrict__ rec,
                                                        unsigned long long* __restrict__ cnt, uint32_t cap,
                                                        int tiles_x, int b0, int passes, KeyT* __restrict__ keys,
                                                        uint32_t* __restrict__ vals, uint32_t* __restrict__ hist) {
    pdl_enter();
    __shared__ uint32_t s_hist[2][kRadix];
    for (int i = threadIdx.x; i < 2 * kRadix; i += NT) (&s_hist[0][0])[i] = 0u;
    __syncthreads();
    const int n_vis = static_cast<int>(cnt[kCntVisible]);
    if (cnt[kCntPairs] > cap) {
        if (blockIdx.x == 0 && threadIdx.x == 0) cnt[kCntOverflow] = 1ull;
        return;
    }
    const uint32_t m0 = (1u << b0) - 1u;
    const int lane = threadIdx.x & 31;
    const int warps = gridDim.x * NW;
    for (int grp = blockIdx.x * NW + (threadIdx.x >> 5); grp * 32 < n_vis; grp += warps) {
        const int r = grp * 32 + lane;
        // lane l: rank grp*32 + l's first pair (ranks past the count: past every pair), its
        // tile-rect origin key, rect width and the reciprocal for row / column
        uint32_t off = 0xffffffffu, magic = 0u;
        int base_key = 0, ntx = 1;
        if (r < n_vis) {
            off = emit_off[r];
            const Splat& s = rec[r];
            const int tx0 = s.x0 >> 4, ty0 = s.y0 >> 4;
            base_key = ty0 * tiles_x + tx0;
            ntx = (s.x1 >> 4) - tx0 + 1;
            magic = 0xffffffffu / static_cast<uint32_t>(ntx) + 1u;  // (wraps to 0 for ntx = 1: not used)
        }
        const uint32_t beg = __shfl_sync(0xffffffffu, off, 0);
        const uint32_t end = emit_off[min(grp * 32 + 32, n_vis)];
        const uint32_t rbase = static_cast<uint32_t>(grp * 32);
        // the group's pairs are contiguous: lane l writes pair base + l (coalesced) and finds its
        // rank as the largest l' with off_l' <= pair (offsets non-decreasing: 5 shuffle steps)
        for (uint32_t base = beg; base < end; base += 32) {
            const uint32_t e = base + lane;
            int rl = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const uint32_t oc = __shfl_sync(0xffffffffu, off, rl + step);
                if (oc <= e) rl += step;
            }
            const uint32_t o = __shfl_sync(0xffffffffu, off, rl);
            const int bk = __shfl_sync(0xffffffffu, base_key, rl);
            const int nx = __shfl_sync(0xffffffffu, ntx, rl);
            const uint32_t mg = __shfl_sync(0xffffffffu, magic, rl);
            if (e < end) {
                const uint32_t l = e - o;
                const uint32_t row = nx == 1 ? l : __umulhi(l, mg);
                const uint32_t k = static_cast<uint32_t>(bk) + row * static_cast<uint32_t>(tiles_x) + (l - row * nx);
                GSB_CHECK(e < cap && l - row * nx < static_cast<uint32_t>(nx) && rbase + rl < static_cast<uint32_t>(n_vis));
                keys[e] = static_cast<KeyT>(k);
                vals[e] = rbase + rl;
                atomicAdd(&s_hist[0][k & m0], 1u);
                if (passes > 1) atomicAdd(&s_hist[1][k >> b0], 1u);
            }
        }
    }
    __syncthreads();
    for (int p = 0; p < passes; ++p) {
        const uint32_t c = s_hist[p][threadIdx.x];
        if (c) atomicAdd(&hist[p * kRadix + threadIdx.x], c);
    }
}

// tile ranges from the sorted keys: a thread covers one 16-byte load of keys plus its neighbours
template <typename KeyT>
__global__ void tile_ranges_kernel(const KeyT* __restrict__ keys, const unsigned long long* __restrict__ cnt,
                                   uint32_t cap, uint2* __restrict__ ranges) {
    pdl_enter();
    constexpr int KV = 16 / sizeof(KeyT);
    const uint32_t n = clamp_count(cnt + kCntPairs, cap);
    for (uint32_t i0 = KV * (blockIdx.x * blockDim.x + threadIdx.x); i0 < n; i0 += KV * gridDim.x * blockDim.x) {
        KeyT k[KV];
        *reinterpret_cast<uint4*>(k) = *reinterpret_cast<const uint4*>(keys + i0);  // buffers: multiples of 64
        const uint32_t prev = i0 > 0 ? static_cast<uint32_t>(keys[i0 - 1]) : 0xffffffffu;
        const uint32_t next = i0 + KV < n ? static_cast<uint32_t>(keys[i0 + KV]) : 0xffffffffu;
        uint32_t p = prev;
#pragma unroll
        for (int j = 0; j < KV; ++j) {
            const uint32_t i = i0 + j;
            if (i >= n) break;
            const uint32_t kj = k[j];
            const uint32_t nk = j < KV - 1 ? (i + 1 < n ? static_cast<uint32_t>(k[j + 1]) : 0xffffffffu) : next;
            if (p != kj) ranges[kj].x = i;
            if (nk != kj) ranges[kj].y = i + 1;
            p = kj;
        }
    }
}

// ------------------------------------------------------------------------------------------
// Start of a render: zero the tile ranges (tiles without pairs keep (0, 0)), the device counters
// and the sort block in one PDL launch (three memsets used to break the kernel chain)
__global__ void __launch_bounds__(1024) frame_init_kernel(uint2* __restrict__ ranges, int tiles,
                                                          unsigned long long* __restrict__ counters,
                                                          uint32_t* __restrict__ sb, int sb_words) {
    pdl_enter();
    for (int i = threadIdx.x; i < tiles; i += blockDim.x) ranges[i] = make_uint2(0u, 0u);
    if (threadIdx.x < kNumCounters) counters[threadIdx.x] = 0ull;
    if (sb)
        for (int i = threadIdx.x; i < sb_words; i += blockDim.x) sb[i] = 0u;
}

// ============================================================================ host launchers
namespace {
int g_sm_count = 0;
int sm_count() {
    if (!g_sm_count) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
        if (g_sm_count <= 0) g_sm_count = 148;
    }
    return g_sm_count;
}
int persistent_grid(int64_t max_tiles, int per_sm) {
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(max_tiles, static_cast<int64_t>(sm_count()) * per_sm)));
}
}  // namespace


size_t sort_status_words(int64_t max_elems) {
    return static_cast<size_t>((max_elems + kSortTile - 1) / kSortTile + 1) * kRadix;
}

void launch_depth_sort(uint32_t* keys_a, uint32_t* keys_b, int32_t* vis_gid, int32_t* gid_tmp, int32_t* gid_sorted,
                       const unsigned long long* depth_by_gid, unsigned long long* cnt, int max_n, SortBlock* sb,
                       unsigned long long* status, uint32_t epoch, cudaStream_t st) {
    if (max_n <= 0) return;
    const uint32_t cap = static_cast<uint32_t>(max_n);
    const unsigned long long* nvis = cnt + kCntVisible;
    launch_pdl(radix_hist_kernel, persistent_grid(div_up(max_n, NT * 8), 2), NT, st, static_cast<const uint32_t*>(keys_a),
               nvis, cap, 3, sb->hist[0]);
    const int grid = persistent_grid(div_up(max_n, TILE), 4);
    // (keys_a, vis_gid) -> (keys_b, gid_tmp) -> (keys_a, gid_sorted) -> (keys_b, gid_tmp) -> exact tie
    // order into gid_sorted; vis_gid (K1's append order) is kept for K8
    launch_pdl(onesweep_kernel<uint32_t, true>, grid, NT, st, keys_a, reinterpret_cast<const uint32_t*>(vis_gid), keys_b,
                                                         reinterpret_cast<uint32_t*>(gid_tmp), nvis, cap, 0, 8,
                                                         sb->hist[0], &sb->ticket[0], status, epoch);
    launch_pdl(onesweep_kernel<uint32_t, true>, grid, NT, st, keys_b, reinterpret_cast<const uint32_t*>(gid_tmp), keys_a,
                                                         reinterpret_cast<uint32_t*>(gid_sorted), nvis, cap, 8, 8,
                                                         sb->hist[1], &sb->ticket[1], status, epoch + 1);
    launch_pdl(onesweep_kernel<uint32_t, true>, grid, NT, st, keys_a, reinterpret_cast<const uint32_t*>(gid_sorted), keys_b,
                                                         reinterpret_cast<uint32_t*>(gid_tmp), nvis, cap, 16, 8,
                                                         sb->hist[2], &sb->ticket[2], status, epoch + 2);
    launch_pdl(fix_ties_kernel, persistent_grid(div_up(max_n, NT), 4), NT, st, keys_b, gid_tmp, depth_by_gid, cnt,
                                                                          gid_sorted);
}

void launch_pack_scan(const int32_t* gid_sorted, const Splat* rec_by_gid, const unsigned long long* depth_by_gid,
                      const unsigned long long* cnt, int max_n, Splat* rec_sorted, unsigned long long* depth_sorted,
                      int32_t* rank_of,
                      uint32_t* emit_off, SortBlock* sb, unsigned long long* status, uint32_t epoch, cudaStream_t st) {
    if (max_n <= 0) return;
    launch_pdl(pack_scan_kernel, persistent_grid(div_up(max_n, kPackItems * NT), 4), NT, st, 
        gid_sorted, rec_by_gid, depth_by_gid, cnt, rec_sorted, depth_sorted, rank_of, emit_off, &sb->ticket[3], status, epoch);
}

template <typename KeyT>
static void tile_sort_impl(const uint32_t* emit_off, const Splat* rec, unsigned long long* cnt, int max_n,
                           uint32_t cap, int tiles_x, int tiles, KeyT* ka, KeyT* kb, uint32_t* va, uint32_t* vb,
                           uint2* ranges, SortBlock* sb, unsigned long long* status, uint32_t epoch, cudaStream_t st) {
    int bits = 1;
    while ((1 << bits) < tiles) ++bits;
    const int passes = bits <= 8 ? 1 : 2;
    const int b0 = passes == 1 ? bits : (bits + 1) / 2;
    // the last pass always lands in (kb, vb): one pass reads the emission from (ka, va), two
    // passes emit into (kb, vb) and go through (ka, va)
    KeyT* ke = passes == 1 ? ka : kb;
    uint32_t* ve = passes == 1 ? va : vb;
    launch_pdl(emit_pairs_kernel<KeyT>, persistent_grid(div_up(max_n, NT), 2), NT, st, emit_off, rec, cnt, cap, tiles_x, b0,
                                                                                 passes, ke, ve, sb->hist[3]);
    const int grid = persistent_grid(div_up(static_cast<int64_t>(cap), TILE), 4);
    const unsigned long long* npairs = cnt + kCntPairs;
    if (passes == 1) {
        launch_pdl(onesweep_kernel<KeyT, true>, grid, NT, st, ka, va, kb, vb, npairs, cap, 0, b0, sb->hist[3],
                                                         &sb->ticket[4], status, epoch);
    } else {
        launch_pdl(onesweep_kernel<KeyT, true>, grid, NT, st, kb, vb, ka, va, npairs, cap, 0, b0, sb->hist[3],
                                                         &sb->ticket[4], status, epoch);
        launch_pdl(onesweep_kernel<KeyT, true>, grid, NT, st, ka, va, kb, vb, npairs, cap, b0, bits - b0, sb->hist[4],
                                                         &sb->ticket[5], status, epoch + 1);
    }
    constexpr int KV = 16 / sizeof(KeyT);
    launch_pdl(tile_ranges_kernel<KeyT>, persistent_grid(div_up(static_cast<int64_t>(cap), KV * 256), 8), 256, st, 
        kb, cnt, cap, ranges);
}

void launch_frame_init(uint2* ranges, int tiles, unsigned long long* counters, SortBlock* sb, cudaStream_t st) {
    launch_pdl(frame_init_kernel, 1, 1024, st, ranges, tiles, counters, reinterpret_cast<uint32_t*>(sb),
               sb ? static_cast<int>(sizeof(SortBlock) / sizeof(uint32_t)) : 0);
}

int launch_tile_sort(const uint32_t* emit_off, const Splat* rec, unsigned long long* cnt, int max_n, uint32_t cap,
                     int tiles_x, int tiles, void* keys_a, void* keys_b, uint32_t* vals_a, uint32_t* vals_b,
                     uint2* ranges, SortBlock* sb, unsigned long long* status, uint32_t epoch, cudaStream_t st) {
    if (max_n <= 0 || cap == 0) return 0;
    if (tiles <= 0xffff)
        tile_sort_impl<uint16_t>(emit_off, rec, cnt, max_n, cap, tiles_x, tiles, static_cast<uint16_t*>(keys_a),
                                 static_cast<uint16_t*>(keys_b), vals_a, vals_b, ranges, sb, status, epoch, st);
    else
        tile_sort_impl<uint32_t>(emit_off, rec, cnt, max_n, cap, tiles_x, tiles, static_cast<uint32_t*>(keys_a),
                                 static_cast<uint32_t*>(keys_b), vals_a, vals_b, ranges, sb, status, epoch, st);
    return tiles > 256 ? 4 : 3;  // launches
}

}  // namespace gsb
