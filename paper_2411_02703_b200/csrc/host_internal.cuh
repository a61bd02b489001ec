// Internal interface of the C-ABI's host side (include/gsmap_b200.h), shared by host.cu (handles,
// render / backward / loss / Adam, train_keyframe_step), host_mapping.cu (the mapping-loop
// helpers: init, filter, integrate, prune, sparse depth, SH schedule) and host_io.cu
// (checkpoint v1, optimizer state, evaluation): the handle structs, buffer types, error
// plumbing and the internal functions. Exceptions never cross the boundary: every entry point
// returns a status and keeps a thread-local message (gs_last_error).
#pragma once
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <functional>
#include <optional>
#include <fstream>
#include <iomanip>
#include <limits>
#include <sstream>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/gsmap_b200.h"
#include "common.cuh"
#include "kernels.cuh"
#include "blend_common.cuh"
#include "sort.cuh"

using namespace gsb;

namespace gsb_host {

extern thread_local std::string g_err;

struct GsError : std::runtime_error {
    int code;
    GsError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw GsError(code, msg); }

inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        fail(e == cudaErrorMemoryAllocation ? GS_ENOMEM : GS_ECUDA,
             std::string(what) + ": " + cudaGetErrorString(e));
    }
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return GS_OK;
    } catch (const GsError& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return GS_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return GS_ELOGIC;
    }
}

// Grow-only device buffer (no per-iteration cudaMalloc on the hot path). Buffers of objects
// created and destroyed in the mapping loop (keyframes) come from the device's stream-ordered
// memory pool instead (`pool` = the context's stream member, so a gs_context_set_stream moves
// their allocations and frees along): their frees return memory to the pool without the
// device-wide synchronisation and unmapping of cudaFree (~50 ms per keyframe).
// Look-back epochs of the hand-written sorts (sort.cu): every sort pass in the process gets a
// fresh value in [1, 2^30), so a status array never needs clearing between passes. The counter
// is process-wide, not per context: status arrays come from the device's shared memory pool,
// and a recycled block may hold words another context published under a per-context epoch that
// this context would reach later (a false "published" match in the look-back). A status array
// is zeroed when it is (re)allocated and again whenever the counter wraps (sort_epoch_era).
uint32_t sort_epochs(uint32_t k);
uint32_t sort_epoch_era();

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    const cudaStream_t* pool = nullptr;
    bool pooled = false;
    template <class T>
    T* as() const { return static_cast<T*>(p); }
    void ensure(size_t need) {
        if (need <= bytes) return;
        release();
        const size_t alloc = std::max<size_t>(need + need / 4, 256);
        if (pool) {
            ck(cudaMallocAsync(&p, alloc, *pool), "cudaMallocAsync");
            // usable by every stream from here on (keyframe uploads run on the copy stream)
            ck(cudaStreamSynchronize(*pool), "sync");
            pooled = true;
        } else {
            ck(cudaMalloc(&p, alloc), "cudaMalloc");
            pooled = false;
        }
        bytes = alloc;
    }
    void release() {
        if (p) {
            if (pooled) cudaFreeAsync(p, *pool);
            else cudaFree(p);
        }
        p = nullptr;
        bytes = 0;
    }
};

struct PinnedBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void ensure(size_t need) {
        if (need <= bytes) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        ck(cudaMallocHost(&p, need), "cudaMallocHost");
        bytes = need;
    }
    ~PinnedBuf() {
        if (p) cudaFreeHost(p);
    }
};

inline void validate_camera(const gs_camera& c) {  // core/types.hpp:22-29
    if (c.fx <= 0.0 || c.fy <= 0.0) fail(GS_EINVAL, "CameraModel: focal lengths must be positive");
    if (c.width <= 0 || c.height <= 0) fail(GS_EINVAL, "CameraModel: image size must be positive");
    if (c.cx < 0.0 || c.cx >= c.width || c.cy < 0.0 || c.cy >= c.height)
        fail(GS_EINVAL, "CameraModel: principal point outside image");
}

inline gs_camera scaled(const gs_camera& c, int level) {  // core/types.hpp:34-44
    gs_camera s = c;
    const double f = static_cast<double>(1 << level);
    s.fx = c.fx / f;
    s.fy = c.fy / f;
    s.cx = (c.cx + 0.5) / f - 0.5;
    s.cy = (c.cy + 0.5) / f - 0.5;
    s.width = (c.width + (1 << level) - 1) >> level;
    s.height = (c.height + (1 << level) - 1) >> level;
    return s;
}

inline ViewParams make_view(const gs_pose& p, const gs_camera& c) {
    ViewParams v;
    v.qw = p.qw; v.qx = p.qx; v.qy = p.qy; v.qz = p.qz;
    v.tx = p.tx; v.ty = p.ty; v.tz = p.tz;
    v.fx = c.fx; v.fy = c.fy; v.cx = c.cx; v.cy = c.cy;
    v.width = c.width; v.height = c.height;
    v.tiles_x = div_up(c.width, kTile);
    v.tiles_y = div_up(c.height, kTile);
    return v;
}

inline int n_active_planes(int max_degree) { return kGeomParams + 3 * (max_degree + 1) * (max_degree + 1); }

}  // namespace gsb_host
using namespace gsb_host;

// ============================================================================ handles
// grow-only scratch of the per-keyframe mapping calls (filter / init / sparse depth / prune):
// one slot per role, so nested calls never share a slot and no call pays cudaMalloc twice
enum ScratchSlot {
    kScPoints, kScKept, kScKeep, kScPos, kScKeys, kScKeys2, kScIdx, kScIdx2, kScBBox, kScHashK, kScHashV,
    kScDepth, kScColor, kScPruneKeep, kScPrunePos, kScPruneTmp, kNumScratch
};

struct gs_context {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    DevBuf cub_tmp;
    DevBuf scratch[kNumScratch];
    DevBuf& sc(ScratchSlot s) { return scratch[s]; }
    PinnedBuf pinned;
    cudaStream_t copy_stream = nullptr;  // host uploads (overlap the compute stream)
    // the training step's gradient zeroing runs here, beside the render (which does not touch the
    // gradient planes); the backward waits for it
    cudaStream_t aux_stream = nullptr;
    cudaEvent_t aux_in = nullptr, aux_out = nullptr;
    cudaStream_t aux() {
        if (!aux_stream) {
            ck(cudaStreamCreateWithFlags(&aux_stream, cudaStreamNonBlocking), "cudaStreamCreate");
            ck(cudaEventCreateWithFlags(&aux_in, cudaEventDisableTiming), "cudaEventCreate");
            ck(cudaEventCreateWithFlags(&aux_out, cudaEventDisableTiming), "cudaEventCreate");
        }
        return aux_stream;
    }
    bool defer_sync = false;             // diagnostics: train steps skip the loss read-back
    cudaStream_t copies() {
        if (!copy_stream) ck(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking), "cudaStreamCreate");
        return copy_stream;
    }
    int64_t launches = 0;
    gs_frame* scratch_frame = nullptr;
    // train steps alternate between two frames: while step s's report is read back, the next
    // step's render (known from gs_train_step_prefetch) is already enqueued into the other frame
    gs_frame* train_frames[2] = {nullptr, nullptr};
    int train_parity = 0;
    cudaEvent_t loss_ready = nullptr;  // the step's read-back copies (waited on instead of the stream)
    int64_t spec_enqueued = 0, spec_used = 0;  // diagnostics
    // diagnostics of the capacity policy: pair-capacity growths after a read-back, and train
    // steps re-run because a render overflowed its capacity
    int64_t cap_growths = 0, overflow_reruns = 0, count_syncs = 0;
    // look-back epochs of the hand-written sorts (sort.cu): see sort_epochs()
    uint32_t epochs(uint32_t k) { return sort_epochs(k); }
    struct Speculation {
        bool valid = false;
        const gs_map* map = nullptr;
        const gs_keyframe* kf = nullptr;
        int level = -1;
        uint64_t version = 0;
        gs_camera cam{};
        gs_pose pose{};
        int frame = 0;
    } spec;
    gs_grads* scratch_grads = nullptr;
    DevBuf batch_stats, shard_grads;  // gs_train_batch: per-view loss records, reduce-scattered gradients
    // optional per-kernel event timing (bench roofline); events are pooled
    bool profile = false;
    int prof_level = -1;  // pyramid level of the train step being enqueued (-1: none), tags scopes
    struct ProfRec {
        const char* name;
        int level;
        cudaEvent_t a, b;
        double host_us;  // host time spent enqueueing the scope
    };
    std::vector<ProfRec> prof;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_next = 0;

    cudaEvent_t ev() {
        if (ev_next == ev_pool.size()) {
            cudaEvent_t e;
            ck(cudaEventCreate(&e), "cudaEventCreate");
            ev_pool.push_back(e);
        }
        return ev_pool[ev_next++];
    }
    void use() { ck(cudaSetDevice(device), "cudaSetDevice"); }
    void launched(int k = 1) {
        launches += k;
        ck(cudaGetLastError(), "kernel launch");
    }
    void* cub(size_t bytes) {
        cub_tmp.ensure(bytes);
        return cub_tmp.p;
    }
};

namespace gsb_host {
// Brackets one kernel family with CUDA events on the context stream when profiling is on.
struct Scope {
    gs_context* C;
    const char* name;
    cudaEvent_t a = nullptr;
    std::chrono::steady_clock::time_point h0;
    Scope(gs_context* c, const char* n) : C(c), name(n) {
        if (C->profile) {
            h0 = std::chrono::steady_clock::now();
            a = C->ev();
            cudaEventRecord(a, C->stream);
        }
    }
    ~Scope() {
        if (C->profile && a) {
            cudaEvent_t b = C->ev();
            cudaEventRecord(b, C->stream);
            const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count();
            C->prof.push_back({name, C->prof_level, a, b, us});
        }
    }
};
}  // namespace gsb_host

// Map-sized arrays (planes, Adam state, gradients) and the mapping calls' scratch come from the device's
// stream-ordered pool on the context stream: the map grows in the mapping loop, and pooled
// frees / reallocations skip cudaFree's device-wide synchronisation and unmapping (measured:
// 16 ms to 1 s per growth with cudaMalloc / cudaFree, run to run).
template <class T>
T* pool_alloc(size_t count, cudaStream_t st, const char* what) {
    void* p = nullptr;
    ck(cudaMallocAsync(&p, sizeof(T) * count, st), what);
    return static_cast<T*>(p);
}
inline void pool_free(void* p, cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
}

struct gs_map {
    gs_context* ctx = nullptr;
    int64_t n = 0, cap = 0;
    float* params = nullptr;
    float* m = nullptr;
    float* v = nullptr;
    int32_t* birth = nullptr;  // per Gaussian: adam_count when its optimizer state was reset
    int8_t* degree = nullptr;
    std::vector<int8_t> deg_host;
    int max_degree = 0;
    double scene_extent = 1.0;
    int64_t global_step = 0;
    int64_t adam_count = 0;  // updates applied to this map; Gaussian i's Adam step = adam_count - birth[i]
    uint64_t version = 0;    // bumped by every change a render would see (speculative renders check it)
    DevBuf minmax;

    int min_degree = 0;
    // sharded optimizer state (gs_train_batch mode 1): each rank's m / v are current only on its
    // own Gaussian range [rank * chunk, (rank + 1) * chunk); 0 = replicated
    int64_t opt_shard_chunk = 0;
    int opt_shard_ranks = 0;
    void free_all() {
        cudaStream_t st = ctx->stream;
        for (void* p : {static_cast<void*>(params), static_cast<void*>(m), static_cast<void*>(v),
                        static_cast<void*>(birth), static_cast<void*>(degree)})
            pool_free(p, st);
        params = m = v = nullptr;
        birth = nullptr;
        degree = nullptr;
    }
    void recompute_max_degree() {  // called after every host-visible change of the Gaussians
        ++version;
        int d = 0, lo = 3;
        for (int8_t x : deg_host) {
            d = std::max<int>(d, x);
            lo = std::min<int>(lo, x);
        }
        max_degree = d;
        min_degree = deg_host.empty() ? 0 : lo;
    }
};

struct gs_frame {
    gs_context* ctx = nullptr;
    bool rendered = false;
    ViewParams view{};
    int64_t map_n = 0, n_vis = 0, n_pairs = 0;
    // Device counts (Counter) are read back lazily: n_vis / n_pairs / overflow are valid only
    // when counts_known. Pair buffers are sized by a capacity remembered per resolution.
    DevBuf counters;
    bool counts_known = false, overflow = false;
    uint32_t status_era = ~0u;  // sort_epoch_era() when sort_status was last cleared
    uint32_t pair_cap = 0;
    int vis_cap = 0;  // ranks the depth sort and the rank-indexed kernels cover
    struct Caps {
        uint32_t pairs = 0;  // (tile, gaussian) pairs
        int vis = 0;         // visible Gaussians
    };
    std::vector<std::pair<int64_t, Caps>> caps;  // (width << 32 | height) -> capacities
    // the two train frames share one table, so a capacity one learns (an overflow re-run)
    // also sizes the other's next render of that level
    std::vector<std::pair<int64_t, Caps>>* shared_caps = nullptr;
    gs_frame* sibling = nullptr;  // the other train frame (buffers reserved together)
    Caps& cap_slot(int w, int h) {
        auto& table = shared_caps ? *shared_caps : caps;
        const int64_t key = (static_cast<int64_t>(w) << 32) | static_cast<uint32_t>(h);
        for (auto& c : table)
            if (c.first == key) return c.second;
        table.emplace_back(key, Caps{});
        return table.back().second;
    }
    // per-Gaussian / per-rank / per-pair scratch
    DevBuf rec_by_gid, vis_flag, key_by_gid, vis_gid, keys_a, keys_b, gid_sorted, rec_sorted, ntiles, emit_off,
        num_sel, pair_keys, pair_keys2, pair_vals, pair_vals2, ranges, partials, rank_sums, depth_sorted, gid_tmp,
        sort_block, sort_status;
    // per-pixel
    DevBuf color, depth, vis, t_final, n_proc, n_contrib, dl_dcolor, depth_cot, wbuf, host_stage;
    DevBuf checkpoints;  // backward list-segment checkpoints [nseg - 1][5][pixels]
    DevBuf seg_scratch;  // segmented forward: per-segment local states, Tl and stop segment
    int nseg = 1;
    DevBuf loss;  // LossScalars
    DevBuf rank_of;  // K8: depth rank per visible map index (written by pack)
    DevBuf eval_quant, eval_gt, eval_stage;  // evaluate_view scratch
    bool has_cotangent = false;
    bool has_contrib = false;  // n_contrib written (the training path's scratch frame skips it)
    // every device buffer of the frame (gs_frame_destroy and the context's internal frames)
    void release_all() {
        for (DevBuf* b : {&counters, &rec_by_gid, &vis_flag, &key_by_gid, &vis_gid, &keys_a, &keys_b, &gid_sorted,
                          &rec_sorted, &ntiles, &emit_off, &num_sel, &pair_keys, &pair_keys2, &pair_vals, &pair_vals2,
                          &ranges, &partials, &rank_sums, &depth_sorted, &gid_tmp, &sort_block, &sort_status, &color,
                          &depth, &vis, &t_final, &n_proc, &n_contrib, &dl_dcolor, &depth_cot, &wbuf, &host_stage,
                          &checkpoints, &seg_scratch, &loss, &rank_of, &eval_quant, &eval_gt, &eval_stage})
            b->release();
    }
    int loss_level = -1;
    double loss_lambda = 0.0, loss_lambda_d = 0.0;
};

struct gs_grads {
    gs_context* ctx = nullptr;
    float* planes = nullptr;
    int64_t cap = 0;
    int64_t n = -1;      // Gaussians the gradient set describes (-1 = unset)
    bool clean = false;  // all planes zero since the last gs_grads_zero (no backward yet)
    bool external = false;
    void ensure(int64_t need) {
        if (need <= cap) return;
        if (external) fail(GS_EINVAL, "gs_grads: external buffer too small for the map");
        pool_free(planes, ctx->stream);
        planes = nullptr;
        const int64_t c = (std::max<int64_t>(need + need / 4, 1024) + 63) / 64 * 64;
        planes = pool_alloc<float>(kNumParams * c, ctx->stream, "alloc grads");
        ck(cudaMemsetAsync(planes, 0, sizeof(float) * kNumParams * c, ctx->stream), "memset grads");
        cap = c;
    }
};

struct gs_keyframe {
    gs_context* ctx = nullptr;
    gs_pose pose{};
    int32_t initial_iters = 0, consumed = 0;
    std::vector<int> hs, ws;
    std::vector<DevBuf> color, depth;  // per level: planes [3][h][w] and [h][w]
    DevBuf stage;                      // fp64 HWC staging for host uploads
    // host uploads run on the context's copy stream: `ready[l]` marks level l's conversion,
    // `used` the compute stream's last read of any level (an upload waits for it first)
    std::vector<cudaEvent_t> ready;
    std::vector<char> pending;
    cudaEvent_t used = nullptr;
    bool used_valid = false;
    ~gs_keyframe() {
        for (auto& b : color) b.release();
        for (auto& b : depth) b.release();
        stage.release();
        for (cudaEvent_t e : ready)
            if (e) cudaEventDestroy(e);
        if (used) cudaEventDestroy(used);
    }
    // the compute stream must see level l's latest upload before reading it
    void acquire(int l, cudaStream_t st) {
        if (l < static_cast<int>(pending.size()) && pending[l]) {
            ck(cudaStreamWaitEvent(st, ready[l], 0), "wait upload");
            pending[l] = 0;
        }
    }
    // after enqueueing reads of the level buffers on the compute stream
    void release_reads(cudaStream_t st) {
        if (!used) ck(cudaEventCreateWithFlags(&used, cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaEventRecord(used, st), "record use");
        used_valid = true;
    }
};

// ============================================================================ internals (host.cu)
namespace gsb_host {
void map_reserve(gs_map* M, int64_t need);
void upload_gaussians(gs_map* M, const gs_gaussian* g, int64_t first, int64_t cnt);
void refresh_extent(gs_map* M);
void frame_pixels(gs_frame* F, const ViewParams& v);
void take_counts(gs_frame* F, const unsigned long long* cnt);
void ensure_counts(gs_frame* F);
uint32_t grown_cap(int64_t pairs);
void render_impl(gs_map* M, const gs_pose& pose, const gs_camera& cam, gs_frame* F, bool exact_counts,
                 bool stats = true);
void need_rendered(gs_frame* F);
void render_checked(gs_map* M, const gs_pose& pose, const gs_camera& cam, gs_frame* F);
void need_counts(gs_frame* F);
void grads_zero(gs_grads* G, gs_map* M);
void backward_impl(gs_map* M, gs_frame* F, const float* dl_dcolor, const float* dl_ddepth,
                   const float* depth_scale, gs_grads* G);
void adam_impl(gs_map* M, gs_grads* G, const gs_learning_rates& lr, const unsigned long long* counters = nullptr);
void loss_impl(gs_frame* F, gs_keyframe* K, int level, const gs_train_config& cfg);
gs_loss_result read_loss(gs_frame* F, const std::function<void()>& between = {});
int schedule_level(const gs_keyframe* K, const gs_train_config& cfg);
void keyframe_build(gs_keyframe* K, const float* color0, const float* depth0, int h, int w, int levels,
                    bool device_src);
gs_frame* scratch_frame(gs_context* C);
gs_frame* train_frame(gs_context* C, int i);
gs_grads* scratch_grads(gs_context* C);
void train_view(gs_map* M, gs_keyframe* K, const gs_train_config& cfg, const gs_camera& cam, gs_frame* F,
                gs_grads* G, int* level_out, bool exact_counts);
// comm.cu
void need_replicated_optimizer(const gs_map* M, const char* what);
// host_mapping.cu
void init_points_device(gs_map* M, const double* dpts, int64_t n);
int64_t filter_points_device(gs_map* M, const double* dpts, int64_t n, const gs_pose& pose, const gs_camera& cam,
                             double tau_alpha, DevBuf& out);
}  // namespace gsb_host
