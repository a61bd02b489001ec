// Tile binning glue (K2-K4: key gather, rank-ordered pack, duplicate-key emission, tile
// ranges) and the on-request CSR materialisation of the contributor lists.
#include "blend_common.cuh"
#include "kernels.cuh"

namespace gsb {

// Depth order = the reference's comparator (depth asc, map index asc), rasterizer.cpp:69-72.
// The radix sort runs on a 24-bit key derived from the fp32-rounded depth (a monotone
// non-decreasing function of the fp64 depth: 3 passes instead of 8 for the fp64 bits), so only
// runs of equal keys can be out of order; each such run (almost always 2 elements) is
// insertion-sorted here by (fp64 depth, map index).
// The result is exactly the fp64 (depth, index) order, independent of the append order.
__global__ void fix_ties_kernel(const uint32_t* __restrict__ key, int32_t* __restrict__ gid,
                                const unsigned long long* __restrict__ depth, unsigned long long* __restrict__ cnt,
                                int max_n) {
    // the sort covered max_n ranks: a larger visible count is clamped and flagged (the step is
    // re-run at exact size), so every later kernel sees a consistent truncated set
    const unsigned long long nv = cnt[kCntVisible];
    const int n = static_cast<int>(min(nv, static_cast<unsigned long long>(max_n)));
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 && nv > static_cast<unsigned long long>(max_n)) {
        cnt[kCntVisible] = static_cast<unsigned long long>(max_n);
        cnt[kCntOverflow] = 1ull;
    }
    if (i >= n) return;
    const uint32_t k = key[i];
    if ((i > 0 && key[i - 1] == k) || i + 1 >= n || key[i + 1] != k) return;  // not a run start
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

void launch_fix_ties(const uint32_t* key32_sorted, int32_t* gid_sorted, const unsigned long long* depth_by_gid,
                     unsigned long long* cnt, int max_n, cudaStream_t st) {
    if (max_n > 0)
        fix_ties_kernel<<<div_up(max_n, 256), 256, 0, st>>>(key32_sorted, gid_sorted, depth_by_gid, cnt, max_n);
}

// rank-ordered copy of the projected records (the reference's sorted `projected` vector);
// the tile counts past the last visible rank are zeroed so the scan can run at capacity
__global__ void pack_kernel(const int32_t* __restrict__ gid_sorted, const Splat* __restrict__ rec_by_gid,
                            const unsigned long long* __restrict__ depth_by_gid,
                            const unsigned long long* __restrict__ cnt, int max_n, Splat* __restrict__ rec_sorted,
                            uint32_t* __restrict__ ntiles, unsigned long long* __restrict__ depth_sorted) {
    const int n = static_cast<int>(cnt[kCntVisible]);
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) {
        if (r <= max_n) ntiles[r] = 0u;
        return;
    }
    const int g = gid_sorted[r];
    const Splat s = rec_by_gid[g];
    rec_sorted[r] = s;
    ntiles[r] = s.ntiles;
    depth_sorted[r] = depth_by_gid[g];
}

void launch_pack(const int32_t* gid_sorted, const Splat* rec_by_gid, const unsigned long long* depth_by_gid,
                 const unsigned long long* cnt, int max_n, Splat* rec_sorted, uint32_t* ntiles,
                 unsigned long long* depth_sorted, cudaStream_t st) {
    pack_kernel<<<div_up(max_n + 1, 256), 256, 0, st>>>(gid_sorted, rec_by_gid, depth_by_gid, cnt, max_n, rec_sorted,
                                                        ntiles, depth_sorted);
}

// Duplicate-key emission (bin_tiles, rasterizer.cpp:76-91). A warp owns 32 consecutive depth
// ranks; their pairs are contiguous in the exclusive scan, so the warp writes them rank by
// rank with all lanes (coalesced, load-balanced across large and small footprints). Keys are
// tile ids; values are depth ranks, so a stable sort by tile yields each tile's list in
// (depth, index) order, exactly the reference's push_back order (ty outer, tx inner).
// Pairs beyond the capacity raise the overflow flag instead (nothing is written).
// KeyT: uint16_t while the tile count fits (every (tile, rank) pair then moves 6 bytes per sort
// pass instead of 8), uint32_t otherwise.
template <typename KeyT>
__global__ void __launch_bounds__(256) emit_pairs_kernel(const uint32_t* __restrict__ emit_off,
                                                         const Splat* __restrict__ rec,
                                                         unsigned long long* __restrict__ cnt, uint32_t cap,
                                                         int tiles_x, KeyT* __restrict__ keys,
                                                         uint32_t* __restrict__ vals) {
    const int n_vis = static_cast<int>(cnt[kCntVisible]);
    if (cnt[kCntPairs] > cap) {
        if (blockIdx.x == 0 && threadIdx.x == 0) cnt[kCntOverflow] = 1ull;
        return;
    }
    const int lane = threadIdx.x & 31;
    const int r = (blockIdx.x * blockDim.x + threadIdx.x);
    if (r - lane >= n_vis) return;  // whole warp past the visible ranks
    // per rank: offset, count, rect origin and width, and the magic multiplier of the width
    // (l / nx = umulhi(l, ceil(2^32 / nx)), exact for l, nx < 2^16) so no pair divides
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
    const uint32_t rbase = static_cast<uint32_t>(r - lane);
    for (int i = 0; i < 32; ++i) {
        const int c = __shfl_sync(0xffffffffu, len, i);
        if (c == 0) continue;
        const int o = __shfl_sync(0xffffffffu, off, i);
        const int base_key = __shfl_sync(0xffffffffu, ty0 * tiles_x + tx0, i);
        const int nx = __shfl_sync(0xffffffffu, ntx, i);
        const uint32_t mg = __shfl_sync(0xffffffffu, magic, i);
        for (int l = lane; l < c; l += 32) {
            const int row = nx == 1 ? l : static_cast<int>(__umulhi(static_cast<uint32_t>(l), mg));
            keys[o + l] = static_cast<KeyT>(base_key + row * tiles_x + (l - row * nx));
            vals[o + l] = rbase + i;
        }
    }
}

void launch_emit_pairs(const uint32_t* emit_off, const Splat* rec, unsigned long long* cnt, int max_n, uint32_t cap,
                       int tiles_x, uint32_t* keys, uint32_t* vals, cudaStream_t st) {
    if (max_n > 0)
        emit_pairs_kernel<uint32_t><<<div_up(max_n, 256), 256, 0, st>>>(emit_off, rec, cnt, cap, tiles_x, keys, vals);
}

void launch_emit_pairs(const uint32_t* emit_off, const Splat* rec, unsigned long long* cnt, int max_n, uint32_t cap,
                       int tiles_x, uint16_t* keys, uint32_t* vals, cudaStream_t st) {
    if (max_n > 0)
        emit_pairs_kernel<uint16_t><<<div_up(max_n, 256), 256, 0, st>>>(emit_off, rec, cnt, cap, tiles_x, keys, vals);
}

// keys are sorted at capacity: the pairs past the device count carry the sentinel key. A
// thread covers the keys of one 16-byte load (4 uint32 or 8 uint16) plus the two neighbours.
template <typename KeyT>
__global__ void tile_ranges_kernel(const KeyT* __restrict__ keys, const unsigned long long* __restrict__ cnt,
                                   uint32_t cap, uint32_t tiles, uint2* __restrict__ ranges) {
    constexpr int KV = 16 / sizeof(KeyT);
    const unsigned long long n64 = cnt[kCntPairs];
    if (n64 > cap) return;
    const uint32_t n = static_cast<uint32_t>(n64);
    const uint32_t i0 = KV * (blockIdx.x * blockDim.x + threadIdx.x);
    if (i0 >= n) return;
    KeyT k[KV];
    *reinterpret_cast<uint4*>(k) = *reinterpret_cast<const uint4*>(keys + i0);  // cap is a multiple of 64
    uint32_t prev = i0 > 0 ? keys[i0 - 1] : 0xffffffffu;
    const uint32_t next = i0 + KV < n ? keys[i0 + KV] : 0xffffffffu;
#pragma unroll
    for (int j = 0; j < KV; ++j) {
        const uint32_t i = i0 + j;
        const uint32_t kj = k[j];
        if (i >= n || kj >= tiles) break;  // sentinels (a truncated, flagged render) end the list
        const uint32_t nk = (j < KV - 1 && i + 1 < n) ? static_cast<uint32_t>(k[j + 1]) : (j == KV - 1 ? next : 0xffffffffu);
        if (i == 0 || prev != kj) ranges[kj].x = i;
        if (i == n - 1 || nk != kj) ranges[kj].y = i + 1;
        prev = kj;
    }
}

void launch_tile_ranges(const uint32_t* keys, const unsigned long long* cnt, uint32_t cap, int tiles,
                        uint2* ranges, cudaStream_t st) {
    if (cap > 0)
        tile_ranges_kernel<uint32_t><<<div_up(div_up(static_cast<int>(cap), 4), 256), 256, 0, st>>>(
            keys, cnt, cap, static_cast<uint32_t>(tiles), ranges);
}

void launch_tile_ranges(const uint16_t* keys, const unsigned long long* cnt, uint32_t cap, int tiles,
                        uint2* ranges, cudaStream_t st) {
    if (cap > 0)
        tile_ranges_kernel<uint16_t><<<div_up(div_up(static_cast<int>(cap), 8), 256), 256, 0, st>>>(
            keys, cnt, cap, static_cast<uint32_t>(tiles), ranges);
}

// RenderOutput::contribs materialised on request (tests, gradcheck): one thread per pixel
// replays the forward with the same staged alpha and the fp64 transmittance of the reference,
// writing (map index, alpha as the double the transmittance update used).
__global__ void materialize_kernel(const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals,
                                   const Splat* __restrict__ rec, ViewParams v, const uint32_t* __restrict__ offsets,
                                   int32_t* __restrict__ out_gid, double* __restrict__ out_alpha) {
    const int tx = blockIdx.x % v.tiles_x, ty = blockIdx.x / v.tiles_x;
    const int lx = threadIdx.x & 15, ly = threadIdx.x >> 4;
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
        const Staged s = stage_of(sp, ox, oy);
        const AlphaS e = alpha_scalar(s.mean, s.con, static_cast<float>(lx), static_cast<float>(ly));
        const double f = one_minus_alpha_d(e.a_raw, e.alpha);
        out_gid[w] = sp.gid;
        out_alpha[w] = __dadd_rn(1.0, -f);
        ++w;
        T = __dmul_rn(T, f);
        if (T < kTMin) break;
    }
}

void launch_materialize(const uint2* ranges, const uint32_t* vals, const Splat* rec, const ViewParams& v,
                        const uint32_t* offsets, int32_t* out_gid, double* out_alpha, cudaStream_t st) {
    const int n_tiles = v.tiles_x * v.tiles_y;
    materialize_kernel<<<n_tiles, kTileThreads, 0, st>>>(ranges, vals, rec, v, offsets, out_gid, out_alpha);
}

}  // namespace gsb
