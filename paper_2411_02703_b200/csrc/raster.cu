// On-request CSR materialisation of the contributor lists (tests, gradcheck). The binning
// itself (sorts, pack, emission, ranges) is in sort.cu.
#include "blend_common.cuh"
#include "kernels.cuh"

namespace gsb {

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
