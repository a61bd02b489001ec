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
// prefix. Waits only on lower tiles, which were ticketed earlier by running CTAs.
__device__ __forceinline__ uint32_t look_back(unsigned long long* status, uint32_t tile, int stride, uint32_t epoch,
                                              uint32_t value) {
    unsigned long long* my = status + static_cast<size_t>(tile) * stride;
    if (tile == 0) {
        st_relaxed(my, pack_status(epoch, kFlagPrefix, value));
        return 0u;
    }
    st_relaxed(my, pack_status(epoch, kFlagAgg, value));
    uint32_t excl = 0;
    for (int j = static_cast<int>(tile) - 1;;) {
        const unsigned long long s = ld_relaxed(status + static_cast<size_t>(j) * stride);
        if (static_cast<uint32_t>(s >> 34) != epoch) continue;  // not yet published in this pass
        excl += static_cast<uint32_t>(s);
        if (((s >> 32) & 3u) == kFlagPrefix) break;
        --j;
    }
    st_relaxed(my, pack_status(epoch, kFlagPrefix, excl + value));
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
__global__ void __launch_bounds__(NT) onesweep_kernel(const KeyT* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                      KeyT* __restrict__ kout, uint32_t* __restrict__ vout,
                                                      const unsigned long long* __restrict__ count, uint32_t cap,
                                                      int shift, int bits, const uint32_t* __restrict__ hist,
                                                      uint32_t* __restrict__ ticket,
                                                      unsigned long long* __restrict__ status, uint32_t epoch) {
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
                s_keys[lp] = key[i];
                s_vals[lp] = val[i];
            }
        }
        __syncthreads();
        const uint32_t tn = min(static_cast<uint32_t>(TILE), n - t0);
        for (uint32_t j = tid; j < tn; j += NT) {
            const KeyT k = s_keys[j];
            const uint32_t g = s_run[(static_cast<uint32_t>(k) >> shift) & mask] + j;
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
// function of the fp64 depth, so only equal-key runs can be out of order). Grid-stride over
// the device count.
__global__ void __launch_bounds__(NT) fix_ties_kernel(const uint32_t* __restrict__ key, int32_t* __restrict__ gid,
                                                      const unsigned long long* __restrict__ depth,
                                                      const unsigned long long* __restrict__ cnt) {
    const int n = static_cast<int>(cnt[kCntVisible]);
    for (int i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT) {
        const uint32_t k = key[i];
        if ((i > 0 && key[i - 1] == k) || i + 1 >= n || key[i + 1] != k) continue;  // not a run start
        int end = i + 1;
        while (end < n && key[end] == k) ++end;
        for (int a = i + 1; a < end; ++a) {
            const int g = gid[a];
            const unsigned long long d = depth[g];
            int b = a - 1;
            while (b >= i) {
                const int gb = gid[b];
                const unsigned long long db = depth[gb];
                if (db < d || (db == d && gb < g)) break;
                gid[b + 1] = gb;
                --b;
            }
            gid[b + 1] = g;
        }
    }
}

// ------------------------------------------------------------------------------------------
// Rank-ordered copy of the projected records (the reference's sorted `projected` vector) fused
// with the exclusive scan of their tile counts: emit_off[r] = first (tile, Gaussian) pair of
// rank r, emit_off[n_vis] = total pairs. Tiles of IT*NT ranks (striped: coalesced writes), one
// look-back word per tile.
constexpr int kPackItems = 4;

__global__ void __launch_bounds__(NT) pack_scan_kernel(const int32_t* __restrict__ gid_sorted,
                                                       const Splat* __restrict__ rec_by_gid,
                                                       const unsigned long long* __restrict__ depth_by_gid,
                                                       const unsigned long long* __restrict__ cnt,
                                                       Splat* __restrict__ rec_sorted,
                                                       unsigned long long* __restrict__ depth_sorted,
                                                       uint32_t* __restrict__ emit_off, uint32_t* __restrict__ ticket,
                                                       unsigned long long* __restrict__ status, uint32_t epoch) {
    constexpr int PT = kPackItems * NT;
    __shared__ uint32_t s_warp[NW];
    __shared__ uint32_t s_tile, s_before;
    const int tid = threadIdx.x;
    const uint32_t nv = static_cast<uint32_t>(cnt[kCntVisible]);
    const uint32_t ntiles = (nv + PT - 1) / PT;
    if (nv == 0 && blockIdx.x == 0 && tid == 0) emit_off[0] = 0u;
    for (;;) {
        if (tid == 0) s_tile = atomicAdd(ticket, 1u);
        __syncthreads();
        const uint32_t tile = s_tile;
        if (tile >= ntiles) break;
        uint32_t loc[kPackItems], nt[kPackItems];
        uint32_t carry = 0u;
#pragma unroll
        for (int i = 0; i < kPackItems; ++i) {
            const uint32_t r = tile * PT + i * NT + tid;
            nt[i] = 0u;
            if (r < nv) {
                const int g = gid_sorted[r];
                const Splat s = rec_by_gid[g];
                rec_sorted[r] = s;
                depth_sorted[r] = depth_by_gid[g];
                nt[i] = s.ntiles;
            }
            uint32_t tot;
            loc[i] = carry + block_excl_scan(nt[i], s_warp, &tot);
            carry += tot;
        }
        if (tid == 0) s_before = look_back(status, tile, 1, epoch, carry);
        __syncthreads();
        const uint32_t before = s_before;
#pragma unroll
        for (int i = 0; i < kPackItems; ++i) {
            const uint32_t r = tile * PT + i * NT + tid;
            if (r < nv) {
                emit_off[r] = before + loc[i];
                if (r == nv - 1) emit_off[nv] = before + loc[i] + nt[i];
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------------
// Duplicate-key emission (bin_tiles, rasterizer.cpp:76-91): a warp owns 32 consecutive depth
// ranks, whose pairs are contiguous in the scan, and writes them rank by rank with all lanes
// (row/column of the tile rect by a magic-number multiply). Keys are tile ids, values depth
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
        int off = 0, len = 0, tx0 = 0, ty0 = 0, ntx = 1;
        uint32_t magic = 0;
        if (r < n_vis) {
            off = static_cast<int>(emit_off[r]);
            len = static_cast<int>(emit_off[r + 1]) - off;
            const Splat& s = rec[r];
            tx0 = s.x0 >> 4;
            ty0 = s.y0 >> 4;
            ntx = (s.x1 >> 4) - tx0 + 1;
            magic = 0xffffffffu / static_cast<uint32_t>(ntx) + 1u;  // (wraps to 0 for ntx = 1: not used)
        }
        const uint32_t rbase = static_cast<uint32_t>(grp * 32);
        for (int i = 0; i < 32; ++i) {
            const int c = __shfl_sync(0xffffffffu, len, i);
            if (c == 0) continue;
            const int o = __shfl_sync(0xffffffffu, off, i);
            const int base_key = __shfl_sync(0xffffffffu, ty0 * tiles_x + tx0, i);
            const int nx = __shfl_sync(0xffffffffu, ntx, i);
            const uint32_t mg = __shfl_sync(0xffffffffu, magic, i);
            for (int l = lane; l < c; l += 32) {
                const int row = nx == 1 ? l : static_cast<int>(__umulhi(static_cast<uint32_t>(l), mg));
                const uint32_t k = static_cast<uint32_t>(base_key + row * tiles_x + (l - row * nx));
                keys[o + l] = static_cast<KeyT>(k);
                vals[o + l] = rbase + i;
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
    radix_hist_kernel<<<persistent_grid(div_up(max_n, NT * 8), 2), NT, 0, st>>>(keys_a, nvis, cap, 3, sb->hist[0]);
    const int grid = persistent_grid(div_up(max_n, TILE), 4);
    // (keys_a, vis_gid) -> (keys_b, gid_sorted) -> (keys_a, gid_tmp) -> (keys_b, gid_sorted); vis_gid
    // (K1's append order) is kept for K8b
    onesweep_kernel<uint32_t, true><<<grid, NT, 0, st>>>(keys_a, reinterpret_cast<const uint32_t*>(vis_gid), keys_b,
                                                         reinterpret_cast<uint32_t*>(gid_sorted), nvis, cap, 0, 8,
                                                         sb->hist[0], &sb->ticket[0], status, epoch);
    onesweep_kernel<uint32_t, true><<<grid, NT, 0, st>>>(keys_b, reinterpret_cast<const uint32_t*>(gid_sorted), keys_a,
                                                         reinterpret_cast<uint32_t*>(gid_tmp), nvis, cap, 8, 8,
                                                         sb->hist[1], &sb->ticket[1], status, epoch + 1);
    onesweep_kernel<uint32_t, true><<<grid, NT, 0, st>>>(keys_a, reinterpret_cast<const uint32_t*>(gid_tmp), keys_b,
                                                         reinterpret_cast<uint32_t*>(gid_sorted), nvis, cap, 16, 8,
                                                         sb->hist[2], &sb->ticket[2], status, epoch + 2);
    fix_ties_kernel<<<persistent_grid(div_up(max_n, NT), 4), NT, 0, st>>>(keys_b, gid_sorted, depth_by_gid, cnt);
}

void launch_pack_scan(const int32_t* gid_sorted, const Splat* rec_by_gid, const unsigned long long* depth_by_gid,
                      const unsigned long long* cnt, int max_n, Splat* rec_sorted, unsigned long long* depth_sorted,
                      uint32_t* emit_off, SortBlock* sb, unsigned long long* status, uint32_t epoch, cudaStream_t st) {
    if (max_n <= 0) return;
    pack_scan_kernel<<<persistent_grid(div_up(max_n, kPackItems * NT), 4), NT, 0, st>>>(
        gid_sorted, rec_by_gid, depth_by_gid, cnt, rec_sorted, depth_sorted, emit_off, &sb->ticket[3], status, epoch);
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
    emit_pairs_kernel<KeyT><<<persistent_grid(div_up(max_n, NT), 2), NT, 0, st>>>(emit_off, rec, cnt, cap, tiles_x, b0,
                                                                                 passes, ke, ve, sb->hist[3]);
    const int grid = persistent_grid(div_up(static_cast<int64_t>(cap), TILE), 4);
    const unsigned long long* npairs = cnt + kCntPairs;
    if (passes == 1) {
        onesweep_kernel<KeyT, true><<<grid, NT, 0, st>>>(ka, va, kb, vb, npairs, cap, 0, b0, sb->hist[3],
                                                         &sb->ticket[4], status, epoch);
    } else {
        onesweep_kernel<KeyT, true><<<grid, NT, 0, st>>>(kb, vb, ka, va, npairs, cap, 0, b0, sb->hist[3],
                                                         &sb->ticket[4], status, epoch);
        onesweep_kernel<KeyT, true><<<grid, NT, 0, st>>>(ka, va, kb, vb, npairs, cap, b0, bits - b0, sb->hist[4],
                                                         &sb->ticket[5], status, epoch + 1);
    }
    constexpr int KV = 16 / sizeof(KeyT);
    tile_ranges_kernel<KeyT><<<persistent_grid(div_up(static_cast<int64_t>(cap), KV * 256), 8), 256, 0, st>>>(
        kb, cnt, cap, ranges);
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
