// Tile binning glue (K2-K4: key gather, rank-ordered pack, duplicate-key emission, tile
// ranges) and the on-request CSR materialisation of the contributor lists.
#include "blend_common.cuh"
#include "kernels.cuh"

namespace gsb {

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
