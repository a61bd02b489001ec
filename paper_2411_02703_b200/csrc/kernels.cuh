// Host-side launchers for the gsmap_b200 kernels (one declaration per kernel family).
#pragma once

#include "common.cuh"

namespace gsb {

// loss buffer layout (loss.cu): which per-block partial slots a loss launch filled
enum LossField : int { kLossL1 = 0, kLossSq = 1, kLossSsim = 2, kLossDabs = 3, kLossNv = 4, kLossFields = 5 };
struct LossLayout {
    int n[kLossFields];  // blocks that wrote each field's slots
    int stride;          // slots per field
};

// geometry.cu (FP64, --fmad=false)
// counters (Counter in common.cuh): [0] visible, [1] (tile, gaussian) pairs, [2] K1a
// candidates, [3] overflow. Kernels after K1 read their counts from there; max_* arguments
// are host-side capacities that size the grids.
void launch_cull(const float* params, int64_t cap, int n, const ViewParams& v, int32_t* cand,
                 unsigned long long* counters, cudaStream_t st);
void launch_preprocess_fwd(const float* params, int64_t cap, const int8_t* degree, const int32_t* cand,
                           int max_cand, const ViewParams& v, Splat* rec_by_gid, unsigned long long* depth_key,
                           int32_t* vis_gid, uint32_t* key32, unsigned long long* counters, cudaStream_t st);
// K8 (partial reduction -> per-Gaussian VJP); sums = [max_ranks][10] fp32 scratch; rank_of =
// depth rank per visible map index (written by pack), vis_gid = K1's visible list
void launch_preprocess_bwd(const float* params, int64_t cap, const int8_t* degree, const ViewParams& v,
                           const uint32_t* emit_off, const float* partials, float* sums,
                           const unsigned long long* counters,
                           int max_ranks, float* grads, int64_t gcap, bool accumulate, const int32_t* rank_of,
                           const int32_t* vis_gid, cudaStream_t st);

// project_sparse_depth: points [n][stride] (x, y, z first, fp64, device) -> depth [h][w] fp64
void launch_sparse_depth(const double* pts, int stride, int64_t n, const ViewParams& v, double* depth,
                         cudaStream_t st);

// init_gaussians_from_points: uniform grid (lo, cell), occupied cells in a hash table
struct KnnGrid {
    double lo[3];
    double cell;
    int64_t max_ring;
};
void launch_knn_bbox(const double* pts6, int64_t n, unsigned long long* out6 /* ordered min xyz, max xyz */,
                     cudaStream_t st);
LossLayout launch_eval(const float* color, const float* depth, const float* gt_color, const float* gt_depth, int h,
                       int w, float* quant, float* wbuf, LossScalars* acc, cudaStream_t st);
void launch_vis_filter(const double* pts6, int64_t n, const ViewParams& v, const float* vis, double tau,
                       int32_t* keep, cudaStream_t st);
void launch_compact_points(const double* src6, int64_t n, const int32_t* keep, const int32_t* pos, double* dst6,
                           cudaStream_t st);
void launch_knn_count_runs(const uint64_t* sorted_keys, int64_t n, unsigned long long* runs, cudaStream_t st);
void launch_knn_keys(const double* pts6, int64_t n, const KnnGrid& g, uint64_t* keys, int32_t* idx, cudaStream_t st);
void launch_knn_table(const uint64_t* sorted_keys, int64_t n, uint64_t* hkeys, int2* hvals, uint32_t hmask,
                      cudaStream_t st);
void launch_knn_init(const double* pts6, int64_t n, int k, const KnnGrid& g, const uint64_t* hkeys, const int2* hvals,
                     uint32_t hmask, const int32_t* sorted_idx, float* params, int64_t cap, int64_t first,
                     cudaStream_t st);

// raster.cu
int launch_blend_fwd(const uint2* ranges, const uint32_t* vals, const Splat* rec, const ViewParams& v,
                      float* color, float* depth, float* vis, float* t_final, int32_t* n_proc,
                      int32_t* n_contrib /* written only when stats */, bool stats,
                      float* checkpoints /* [nseg - 1][5][pixels] */, int nseg,
                      float* seg_scratch /* [(9 nseg + 2) pixels]: segmented forward, nullable */,
                      const unsigned long long* counters /* bounds of the checked build */, cudaStream_t st);
void launch_blend_bwd(const uint2* ranges, const uint32_t* vals, const Splat* rec, const uint32_t* emit_off,
                      const ViewParams& v, const float* t_final, const int32_t* n_proc,
                      const float* dl_dcolor, const float* dl_ddepth, const float* depth_scale,
                      float* partials, const unsigned long long* counters, const float* checkpoints, int nseg,
                      const float* color, const float* depth, cudaStream_t st);
void read_blend_stats(unsigned long long out[2], bool reset);
void set_blend_ppt(int fwd, int bwd);
void set_blend_df_list(int entries);
void set_blend_segments(int nseg);
void set_blend_seg_forward(int on);
void launch_materialize(const uint2* ranges, const uint32_t* vals, const Splat* rec, const ViewParams& v,
                        const uint32_t* offsets, int32_t* out_gid, double* out_alpha, cudaStream_t st);

// loss.cu. The loss buffer is a LossScalars header followed by per-block partial slots
// (loss_buffer_bytes); the launchers return which slots they filled and loss_finalize sums them
// in a fixed order into the header (deterministic, no atomics).
int loss_slot_stride(int h, int w);
size_t loss_buffer_bytes(int h, int w);
LossLayout launch_loss_pixel(const float* color, const float* depth, const float* vis, const float* gt_color,
                             const float* gt_depth, int h, int w, double lambda, float* dl_dcolor,
                             float* depth_cot, LossScalars* acc, cudaStream_t st);
// depth != nullptr: also computes loss_pixel's terms (L1 / psnr / masked depth) in the adjoint pass
LossLayout launch_ssim(const float* color, const float* gt_color, int h, int w, double lambda, float* wbuf,
                       float* dl_dcolor, LossScalars* acc, const float* depth, const float* vis,
                       const float* gt_depth, float* depth_cot, cudaStream_t st);
void launch_loss_finalize(LossScalars* acc, const LossLayout& layout, double lambda_d, cudaStream_t st);
void launch_downsample(const float* in, int h, int w, int channels, bool depth, float* out, cudaStream_t st);

// adam.cu
void launch_adam(float* params, float* m, float* v, const int32_t* birth, const int8_t* degree, const float* grads,
                 int64_t gcap, int64_t cap, int n, const double lr[5], double scene_extent, int64_t t_common,
                 const unsigned long long* counters /* nullable: skip on overflow */, int max_degree,
                 cudaStream_t st);
void launch_position_minmax(const float* params, int64_t cap, int n, float* out6, cudaStream_t st);
void launch_prune_flags(const float* params, int64_t cap, int n, double thr, int32_t* keep, cudaStream_t st);
void launch_compact(const float* src, float* dst, int64_t scap, int64_t dcap, int planes, int n, const int32_t* keep,
                    const int32_t* pos, cudaStream_t st);
void launch_compact(const int32_t* src, int32_t* dst, int n, const int32_t* keep, const int32_t* pos, cudaStream_t st);
void launch_compact(const int8_t* src, int8_t* dst, int n, const int32_t* keep, const int32_t* pos, cudaStream_t st);
void launch_to_hwc_double(const float* planes, int h, int w, int channels, double* out, cudaStream_t st);
void launch_from_hwc_double(const double* hwc, int h, int w, int channels, float* planes, cudaStream_t st);

}  // namespace gsb
