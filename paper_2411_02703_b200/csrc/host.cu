// Host side of the C-ABI (include/gsmap_b200.h): device state, buffer management and the
// orchestration of the hot step train_keyframe_step (mapper.cpp:214-238) over the kernels.
// Exceptions never cross the boundary: every entry point returns a status and keeps a
// thread-local message (gs_last_error).
#include <cub/cub.cuh>

#include <algorithm>
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

using namespace gsb;

namespace {

thread_local std::string g_err;

struct GsError : std::runtime_error {
    int code;
    GsError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void fail(int code, const std::string& msg) { throw GsError(code, msg); }

void ck(cudaError_t e, const char* what) {
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
// memory pool instead (`pool` = the stream they are used on): their frees return memory to the
// pool without the device-wide synchronisation and unmapping of cudaFree (~50 ms per keyframe).
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaStream_t pool = nullptr;
    bool pooled = false;
    template <class T>
    T* as() const { return static_cast<T*>(p); }
    void ensure(size_t need) {
        if (need <= bytes) return;
        release();
        const size_t alloc = std::max<size_t>(need + need / 4, 256);
        if (pool) {
            ck(cudaMallocAsync(&p, alloc, pool), "cudaMallocAsync");
            // usable by every stream from here on (keyframe uploads run on the copy stream)
            ck(cudaStreamSynchronize(pool), "sync");
            pooled = true;
        } else {
            ck(cudaMalloc(&p, alloc), "cudaMalloc");
            pooled = false;
        }
        bytes = alloc;
    }
    void release() {
        if (p) {
            if (pooled) cudaFreeAsync(p, pool);
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

void validate_camera(const gs_camera& c) {  // core/types.hpp:22-29
    if (c.fx <= 0.0 || c.fy <= 0.0) fail(GS_EINVAL, "CameraModel: focal lengths must be positive");
    if (c.width <= 0 || c.height <= 0) fail(GS_EINVAL, "CameraModel: image size must be positive");
    if (c.cx < 0.0 || c.cx >= c.width || c.cy < 0.0 || c.cy >= c.height)
        fail(GS_EINVAL, "CameraModel: principal point outside image");
}

gs_camera scaled(const gs_camera& c, int level) {  // core/types.hpp:34-44
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

ViewParams make_view(const gs_pose& p, const gs_camera& c) {
    ViewParams v;
    v.qw = p.qw; v.qx = p.qx; v.qy = p.qy; v.qz = p.qz;
    v.tx = p.tx; v.ty = p.ty; v.tz = p.tz;
    v.fx = c.fx; v.fy = c.fy; v.cx = c.cx; v.cy = c.cy;
    v.width = c.width; v.height = c.height;
    v.tiles_x = div_up(c.width, kTile);
    v.tiles_y = div_up(c.height, kTile);
    return v;
}

int n_active_planes(int max_degree) { return kGeomParams + 3 * (max_degree + 1) * (max_degree + 1); }

}  // namespace

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
    // optional per-kernel event timing (bench roofline); events are pooled
    bool profile = false;
    struct ProfRec {
        const char* name;
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

namespace {
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
            C->prof.push_back({name, a, b, us});
        }
    }
};
}  // namespace

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
    uint32_t pair_cap = 0;
    int vis_cap = 0;  // ranks the depth sort and the rank-indexed kernels cover
    struct Caps {
        uint32_t pairs = 0;  // (tile, gaussian) pairs
        int vis = 0;         // visible Gaussians
    };
    std::vector<std::pair<int64_t, Caps>> caps;  // (width << 32 | height) -> capacities
    Caps& cap_slot(int w, int h) {
        const int64_t key = (static_cast<int64_t>(w) << 32) | static_cast<uint32_t>(h);
        for (auto& c : caps)
            if (c.first == key) return c.second;
        caps.emplace_back(key, Caps{});
        return caps.back().second;
    }
    // per-Gaussian / per-rank / per-pair scratch
    DevBuf rec_by_gid, vis_flag, key_by_gid, vis_gid, keys_a, keys_b, gid_sorted, rec_sorted, ntiles, emit_off,
        num_sel, pair_keys, pair_keys2, pair_vals, pair_vals2, ranges, partials, rank_sums, depth_sorted;
    // per-pixel
    DevBuf color, depth, vis, t_final, n_proc, n_contrib, dl_dcolor, depth_cot, wbuf, host_stage;
    DevBuf checkpoints;  // backward list-segment checkpoints [nseg - 1][5][pixels]
    DevBuf seg_scratch;  // segmented forward: per-segment local states, Tl and stop segment
    int nseg = 1;
    DevBuf loss;  // LossScalars
    DevBuf rank_of;  // K8b: depth rank per map index (-1 = culled)
    DevBuf eval_quant, eval_gt, eval_stage;  // evaluate_view scratch
    bool has_cotangent = false;
    bool has_contrib = false;  // n_contrib written (the training path's scratch frame skips it)
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

// ============================================================================ internals
namespace {

void map_reserve(gs_map* M, int64_t need) {
    if (need <= M->cap) return;
    Scope sc(M->ctx, "map_reserve");
    // multiples of 64: every plane base stays 16-byte aligned (vectorised Adam)
    const int64_t nc = (std::max<int64_t>(need, M->cap + M->cap / 2) + 63) / 64 * 64;
    cudaStream_t st = M->ctx->stream;
    float *p = nullptr, *m = nullptr, *v = nullptr;
    int32_t* s = nullptr;
    int8_t* d = nullptr;
    p = pool_alloc<float>(kNumParams * nc, st, "alloc params");
    m = pool_alloc<float>(kNumParams * nc, st, "alloc adam m");
    v = pool_alloc<float>(kNumParams * nc, st, "alloc adam v");
    s = pool_alloc<int32_t>(nc, st, "alloc birth");
    d = pool_alloc<int8_t>(nc, st, "alloc degree");
    ck(cudaMemsetAsync(m, 0, sizeof(float) * kNumParams * nc, st), "memset");
    ck(cudaMemsetAsync(v, 0, sizeof(float) * kNumParams * nc, st), "memset");
    ck(cudaMemsetAsync(p, 0, sizeof(float) * kNumParams * nc, st), "memset");
    if (M->n > 0) {
        ck(cudaMemcpy2DAsync(p, sizeof(float) * nc, M->params, sizeof(float) * M->cap, sizeof(float) * M->n,
                             kNumParams, cudaMemcpyDeviceToDevice, st), "copy params");
        ck(cudaMemcpy2DAsync(m, sizeof(float) * nc, M->m, sizeof(float) * M->cap, sizeof(float) * M->n,
                             kNumParams, cudaMemcpyDeviceToDevice, st), "copy m");
        ck(cudaMemcpy2DAsync(v, sizeof(float) * nc, M->v, sizeof(float) * M->cap, sizeof(float) * M->n,
                             kNumParams, cudaMemcpyDeviceToDevice, st), "copy v");
        ck(cudaMemcpyAsync(s, M->birth, sizeof(int32_t) * M->n, cudaMemcpyDeviceToDevice, st), "copy birth");
        ck(cudaMemcpyAsync(d, M->degree, sizeof(int8_t) * M->n, cudaMemcpyDeviceToDevice, st), "copy degree");
    }
    ck(cudaStreamSynchronize(st), "sync");
    M->free_all();
    M->params = p; M->m = m; M->v = v; M->birth = s; M->degree = d;
    M->cap = nc;
}

// upload AoS fp64 Gaussians [first, first+cnt) into the fp32 planes
void upload_gaussians(gs_map* M, const gs_gaussian* g, int64_t first, int64_t cnt) {
    if (cnt <= 0) return;
    std::vector<float> soa(static_cast<size_t>(kNumParams) * cnt);
    for (int64_t i = 0; i < cnt; ++i)
        for (int k = 0; k < kNumParams; ++k) soa[static_cast<size_t>(k) * cnt + i] = static_cast<float>(g[i].p[k]);
    std::vector<int8_t> deg(cnt);
    for (int64_t i = 0; i < cnt; ++i) {
        if (g[i].active_degree < 0 || g[i].active_degree > 3) fail(GS_EINVAL, "eval_sh: active_degree out of range");
        deg[i] = static_cast<int8_t>(g[i].active_degree);
    }
    ck(cudaMemcpy2DAsync(M->params + first, sizeof(float) * M->cap, soa.data(), sizeof(float) * cnt,
                         sizeof(float) * cnt, kNumParams, cudaMemcpyHostToDevice, M->ctx->stream), "upload params");
    ck(cudaMemcpyAsync(M->degree + first, deg.data(), cnt, cudaMemcpyHostToDevice, M->ctx->stream), "upload degree");
    ck(cudaStreamSynchronize(M->ctx->stream), "sync");
    if (static_cast<int64_t>(M->deg_host.size()) < first + cnt) M->deg_host.resize(first + cnt);
    std::copy(deg.begin(), deg.end(), M->deg_host.begin() + first);
    M->recompute_max_degree();
}

void refresh_extent(gs_map* M) {  // gaussian_map.cpp:87-99
    if (M->n == 0) {
        M->scene_extent = 1.0;
        return;
    }
    M->minmax.ensure(6 * sizeof(unsigned int));
    launch_position_minmax(M->params, M->cap, static_cast<int>(M->n), M->minmax.as<float>(), M->ctx->stream);
    M->ctx->launched();
    unsigned int enc[6];
    ck(cudaMemcpyAsync(enc, M->minmax.p, sizeof(enc), cudaMemcpyDeviceToHost, M->ctx->stream), "d2h");
    ck(cudaStreamSynchronize(M->ctx->stream), "sync");
    double lo[3], hi[3];
    auto dec = [](unsigned int u) {
        const unsigned int b = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
        float f;
        std::memcpy(&f, &b, 4);
        return static_cast<double>(f);
    };
    for (int c = 0; c < 3; ++c) {
        lo[c] = dec(enc[c]);
        hi[c] = dec(enc[3 + c]);
    }
    const double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
    M->scene_extent = std::max(0.5 * std::sqrt((dx * dx + dy * dy) + dz * dz), 1e-6);
}

void frame_pixels(gs_frame* F, const ViewParams& v) {
    const size_t P = static_cast<size_t>(v.width) * v.height;
    F->color.ensure(3 * P * sizeof(float));
    F->depth.ensure(P * sizeof(float));
    F->vis.ensure(P * sizeof(float));
    F->t_final.ensure(P * sizeof(float));
    F->n_proc.ensure(P * sizeof(int32_t));
    F->n_contrib.ensure(P * sizeof(int32_t));
    F->dl_dcolor.ensure(3 * P * sizeof(float));
    F->depth_cot.ensure(P * sizeof(float));
    F->loss.ensure(sizeof(LossScalars));
    F->ranges.ensure(static_cast<size_t>(v.tiles_x) * v.tiles_y * sizeof(uint2));
}

unsigned long long* dev_counters(gs_frame* F) { return F->counters.as<unsigned long long>(); }

void take_counts(gs_frame* F, const unsigned long long* cnt) {
    F->n_vis = static_cast<int64_t>(cnt[kCntVisible]);
    F->n_pairs = static_cast<int64_t>(cnt[kCntPairs]);
    F->overflow = cnt[kCntOverflow] != 0;
    F->counts_known = true;
    if (F->n_pairs > 0xffffffffLL) fail(GS_ELOGIC, "render: more than 2^32 (tile, gaussian) pairs");
}

// one host round trip for the frame's device counts (no-op when already read)
void ensure_counts(gs_frame* F) {
    if (F->counts_known) return;
    gs_context* C = F->ctx;
    C->pinned.ensure(sizeof(LossScalars) + 64);
    ck(cudaMemcpyAsync(C->pinned.p, F->counters.p, kNumCounters * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                       C->stream), "d2h counters");
    ck(cudaStreamSynchronize(C->stream), "sync counters");
    take_counts(F, static_cast<const unsigned long long*>(C->pinned.p));
}

uint32_t grown_cap(int64_t pairs) {
    const int64_t c = (pairs + pairs / 8 + 65536 + 63) / 64 * 64;  // multiple of 64 (vector loads)
    return static_cast<uint32_t>(std::min<int64_t>(c, 0xffffffc0LL));
}

// render (rasterizer.cpp:100-199) without the CSR: project -> compact -> depth sort -> pack ->
// scan -> emit (tile, rank) pairs -> stable tile sort -> ranges -> blend. Nothing here waits
// for the device: the sorts and scans run at capacity (the map size for ranks, the
// resolution's pair capacity for pairs) with sentinel keys past the device counts. With
// exact_counts (or an unknown capacity) the pair count is read back first and the capacity
// grown to fit, so the render cannot overflow.
void render_impl(gs_map* M, const gs_pose& pose, const gs_camera& cam, gs_frame* F, bool exact_counts,
                 bool stats = true) {
    validate_camera(cam);
    gs_context* C = M->ctx;
    C->use();
    cudaStream_t st = C->stream;
    const ViewParams v = make_view(pose, cam);
    F->view = v;
    F->map_n = M->n;
    F->rendered = false;
    F->has_cotangent = false;
    frame_pixels(F, v);
    const int n = static_cast<int>(M->n);
    const int T = v.tiles_x * v.tiles_y;
    ck(cudaMemsetAsync(F->ranges.p, 0, sizeof(uint2) * T, st), "memset ranges");
    F->counters.ensure(kNumCounters * sizeof(unsigned long long));
    ck(cudaMemsetAsync(F->counters.p, 0, kNumCounters * sizeof(unsigned long long), st), "memset counters");
    F->n_vis = 0;
    F->n_pairs = 0;
    F->overflow = false;
    F->counts_known = n == 0;
    F->pair_cap = 0;
    F->vis_cap = 0;
    unsigned long long* cnt = dev_counters(F);
    if (n > 0) {
        F->rec_by_gid.ensure(sizeof(Splat) * n);
        F->vis_flag.ensure(sizeof(int32_t) * n);  // K1a candidate list
        F->key_by_gid.ensure(sizeof(unsigned long long) * n);
        F->vis_gid.ensure(sizeof(int32_t) * n);
        F->keys_a.ensure(sizeof(uint32_t) * n);
        F->keys_b.ensure(sizeof(uint32_t) * n);
        F->gid_sorted.ensure(sizeof(int32_t) * n);
        F->rec_sorted.ensure(sizeof(Splat) * n);
        F->depth_sorted.ensure(sizeof(unsigned long long) * n);
        F->ntiles.ensure(sizeof(uint32_t) * (n + 1));
        F->emit_off.ensure(sizeof(uint32_t) * (n + 1));
        // sentinel depth keys past the visible count (real keys are positive fp32 bits)
        ck(cudaMemsetAsync(F->keys_a.p, 0xff, sizeof(uint32_t) * n, st), "memset keys");
        {
            Scope sc(C, "preprocess_fwd");
            launch_cull(M->params, M->cap, n, v, F->vis_flag.as<int32_t>(), cnt, st);
            launch_preprocess_fwd(M->params, M->cap, M->degree, F->vis_flag.as<int32_t>(), n, v,
                                  F->rec_by_gid.as<Splat>(), F->key_by_gid.as<unsigned long long>(),
                                  F->vis_gid.as<int32_t>(), F->keys_a.as<uint32_t>(), cnt, st);
            C->launched(2);
        }
        gs_frame::Caps& cs = F->cap_slot(v.width, v.height);
        if (cs.pairs == 0 || exact_counts) {
            ensure_counts(F);
            cs.pairs = std::max(cs.pairs, grown_cap(F->n_pairs));
            cs.vis = std::max(cs.vis, static_cast<int>((F->n_vis + F->n_vis / 8 + 4096 + 63) / 64 * 64));
        }
        const uint32_t cap = cs.pairs;
        const int nv = std::min(n, cs.vis);  // a larger visible count raises the overflow flag
        F->pair_cap = cap;
        F->vis_cap = nv;
        {
            // (depth, index) order (rasterizer.cpp:69-72): stable radix sort on the fp32-rounded
            // depth, then exact (fp64 depth, index) order inside runs of equal fp32 keys
            Scope sc_sort(C, "depth_sort_pack_scan");
            size_t tb = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, tb, F->keys_a.as<uint32_t>(), F->keys_b.as<uint32_t>(),
                                            F->vis_gid.as<int32_t>(), F->gid_sorted.as<int32_t>(), nv, 0, kDepthKeyBits, st);
            ck(cub::DeviceRadixSort::SortPairs(C->cub(tb), tb, F->keys_a.as<uint32_t>(), F->keys_b.as<uint32_t>(),
                                               F->vis_gid.as<int32_t>(), F->gid_sorted.as<int32_t>(), nv, 0, kDepthKeyBits, st),
               "depth sort");
            launch_fix_ties(F->keys_b.as<uint32_t>(), F->gid_sorted.as<int32_t>(),
                            F->key_by_gid.as<unsigned long long>(), cnt, nv, st);
            launch_pack(F->gid_sorted.as<int32_t>(), F->rec_by_gid.as<Splat>(), F->key_by_gid.as<unsigned long long>(),
                        cnt, nv, F->rec_sorted.as<Splat>(), F->ntiles.as<uint32_t>(),
                        F->depth_sorted.as<unsigned long long>(), st);
            C->launched(2);
            tb = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, tb, F->ntiles.as<uint32_t>(), F->emit_off.as<uint32_t>(), nv + 1, st);
            ck(cub::DeviceScan::ExclusiveSum(C->cub(tb), tb, F->ntiles.as<uint32_t>(), F->emit_off.as<uint32_t>(),
                                             nv + 1, st), "scan");
        }
        {
            Scope sc_keys(C, "tile_keys_sort_ranges");
            F->pair_keys.ensure(sizeof(uint32_t) * cap);
            F->pair_keys2.ensure(sizeof(uint32_t) * cap);
            F->pair_vals.ensure(sizeof(uint32_t) * cap);
            F->pair_vals2.ensure(sizeof(uint32_t) * cap);
            ck(cudaMemsetAsync(F->pair_keys.p, 0xff, sizeof(uint32_t) * cap, st), "memset pair keys");
            launch_emit_pairs(F->emit_off.as<uint32_t>(), F->rec_sorted.as<Splat>(), cnt, nv, cap, v.tiles_x,
                              F->pair_keys.as<uint32_t>(), F->pair_vals.as<uint32_t>(), st);
            C->launched();
            int bits = 1;  // the sentinel's low bits (2^bits - 1) must sort after every tile id
            while ((1u << bits) <= static_cast<uint32_t>(T)) ++bits;
            size_t tb = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, tb, F->pair_keys.as<uint32_t>(), F->pair_keys2.as<uint32_t>(),
                                            F->pair_vals.as<uint32_t>(), F->pair_vals2.as<uint32_t>(),
                                            static_cast<int>(cap), 0, bits, st);
            ck(cub::DeviceRadixSort::SortPairs(C->cub(tb), tb, F->pair_keys.as<uint32_t>(),
                                               F->pair_keys2.as<uint32_t>(), F->pair_vals.as<uint32_t>(),
                                               F->pair_vals2.as<uint32_t>(), static_cast<int>(cap), 0, bits, st),
               "tile sort");
            launch_tile_ranges(F->pair_keys2.as<uint32_t>(), cnt, cap, T, F->ranges.as<uint2>(), st);
            C->launched();
        }
    }
    {
        Scope sc(C, "blend_fwd");
        F->nseg = blend_segments(v);
        const size_t P = static_cast<size_t>(v.width) * v.height;
        if (F->nseg > 1) {
            F->checkpoints.ensure(sizeof(float) * (F->nseg - 1) * kCkFields * P);
            F->seg_scratch.ensure(sizeof(float) * (9 * F->nseg + 2) * P);
        }
        launch_blend_fwd(F->ranges.as<uint2>(), n > 0 ? F->pair_vals2.as<uint32_t>() : nullptr,
                         n > 0 ? F->rec_sorted.as<Splat>() : nullptr, v, F->color.as<float>(),
                         F->depth.as<float>(), F->vis.as<float>(), F->t_final.as<float>(),
                         F->n_proc.as<int32_t>(), F->n_contrib.as<int32_t>(), stats, F->checkpoints.as<float>(),
                         F->nseg, n > 0 && F->nseg > 1 ? F->seg_scratch.as<float>() : nullptr, st);
        C->launched();
    }
    F->rendered = true;
    F->has_contrib = stats;
}

void need_rendered(gs_frame* F) {
    if (!F->rendered) fail(GS_ELOGIC, "render_backward: contributor lists missing or inconsistent");
}

// the public render: synchronous like the reference's, re-rendered at exact capacity if the
// remembered pair capacity was too small
void render_checked(gs_map* M, const gs_pose& pose, const gs_camera& cam, gs_frame* F) {
    render_impl(M, pose, cam, F, false);
    ensure_counts(F);
    if (F->overflow) {
        render_impl(M, pose, cam, F, true);
        ensure_counts(F);
        if (F->overflow) fail(GS_ELOGIC, "render: pair capacity overflow after exact sizing");
    }
}

// counts for the read-back entry points (the frame is never left overflowed by the API)
void need_counts(gs_frame* F) {
    need_rendered(F);
    ensure_counts(F);
    if (F->overflow) fail(GS_ELOGIC, "frame: pair capacity overflow (render again)");
    if (!F->has_contrib) fail(GS_ELOGIC, "frame: contributor counts not recorded for this render");
}

void grads_zero(gs_grads* G, gs_map* M) {
    G->ensure(std::max<int64_t>(M->n, 1));
    if (M->n > 0) {
        const int planes = n_active_planes(M->max_degree);
        ck(cudaMemset2DAsync(G->planes, sizeof(float) * G->cap, 0, sizeof(float) * M->n, planes, M->ctx->stream),
           "memset grads");
    }
    G->n = M->n;
    G->clean = true;
}

void backward_impl(gs_map* M, gs_frame* F, const float* dl_dcolor, const float* dl_ddepth,
                   const float* depth_scale, gs_grads* G) {
    gs_context* C = M->ctx;
    cudaStream_t st = C->stream;
    need_rendered(F);
    if (F->map_n != M->n) fail(GS_ELOGIC, "render_backward: contributor lists missing or inconsistent");
    if (M->n == 0 || F->pair_cap == 0) return;
    if (F->counts_known && (F->n_vis == 0 || F->n_pairs == 0)) return;
    F->partials.ensure(sizeof(float) * kNumPartials * F->pair_cap);
    F->rank_sums.ensure(sizeof(double) * kNumPartials * F->vis_cap);
    {
        Scope sc(C, "blend_bwd");
        launch_blend_bwd(F->ranges.as<uint2>(), F->pair_vals2.as<uint32_t>(), F->rec_sorted.as<Splat>(),
                         F->emit_off.as<uint32_t>(), F->view, F->t_final.as<float>(), F->n_proc.as<int32_t>(),
                         dl_dcolor, dl_ddepth, depth_scale, F->partials.as<float>(), dev_counters(F),
                         F->checkpoints.as<float>(), F->nseg, F->color.as<float>(), F->depth.as<float>(), st);
        C->launched();
    }
    {
        Scope sc(C, "preprocess_bwd");
        const bool by_gid = true;  // K8b in visible-list order (coalesced plane traffic), see geometry.cu
        F->rank_of.ensure(sizeof(int32_t) * std::max<int64_t>(M->n, 1));
        launch_preprocess_bwd(M->params, M->cap, M->degree, F->view, F->rec_sorted.as<Splat>(),
                              F->emit_off.as<uint32_t>(), F->partials.as<float>(), F->rank_sums.as<double>(),
                              dev_counters(F), F->vis_cap, G->planes, G->cap, !G->clean, by_gid,
                              F->rank_of.as<int32_t>(), static_cast<int>(M->n), F->vis_gid.as<int32_t>(), st);
        G->clean = false;
        C->launched(3);  // K8a reduce, rank scatter, K8b
    }
}

// counters: the frame whose gradients these are (the update is skipped if it overflowed)
void adam_impl(gs_map* M, gs_grads* G, const gs_learning_rates& lr, const unsigned long long* counters = nullptr) {
    if (G->n != M->n) fail(GS_EINVAL, "apply_gradients: gradient count does not match map size");
    const double l[5] = {lr.position, lr.rotation, lr.log_scale, lr.opacity, lr.sh};
    Scope sc(M->ctx, "adam");
    launch_adam(M->params, M->m, M->v, M->birth, M->degree, G->planes, G->cap, M->cap, static_cast<int>(M->n), l,
                M->scene_extent, M->adam_count + 1, counters, M->max_degree, M->ctx->stream);
    ++M->adam_count;
    ++M->version;
    M->ctx->launched();
    ++M->global_step;
}

void loss_impl(gs_frame* F, gs_keyframe* K, int level, const gs_train_config& cfg) {
    if (level < 0 || level >= static_cast<int>(K->hs.size()))
        fail(GS_EINVAL, "compute_loss: pyramid level out of range");
    need_rendered(F);
    const int h = K->hs[level], w = K->ws[level];
    if (F->view.height != h || F->view.width != w)
        fail(GS_EINVAL, "compute_loss: rendered resolution does not match level");
    gs_context* C = F->ctx;
    cudaStream_t st = C->stream;
    K->acquire(level, st);
    ck(cudaMemsetAsync(F->loss.p, 0, sizeof(LossScalars), st), "memset loss");
    Scope sc(C, "loss_l1_ssim_depth");
    if (cfg.lambda != 0.0) {
        if (h < 11 || w < 11) fail(GS_EINVAL, "ssim: image smaller than the 11x11 window");
        F->wbuf.ensure(sizeof(float) * 9 * static_cast<size_t>(h - 10) * (w - 10));
        // SSIM forward, then its adjoint fused with the per-pixel L1 / psnr / depth terms
        launch_ssim(F->color.as<float>(), K->color[level].as<float>(), h, w, cfg.lambda, F->wbuf.as<float>(),
                    F->dl_dcolor.as<float>(), F->loss.as<LossScalars>(), F->depth.as<float>(), F->vis.as<float>(),
                    K->depth[level].as<float>(), F->depth_cot.as<float>(), st);
        C->launched(2);
    } else {
        launch_loss_pixel(F->color.as<float>(), F->depth.as<float>(), F->vis.as<float>(), K->color[level].as<float>(),
                          K->depth[level].as<float>(), h, w, cfg.lambda, F->dl_dcolor.as<float>(),
                          F->depth_cot.as<float>(), F->loss.as<LossScalars>(), st);
        C->launched();
    }
    launch_loss_finalize(F->loss.as<LossScalars>(), cfg.lambda_d, st);
    C->launched();
    K->release_reads(st);
    F->has_cotangent = true;
    F->loss_level = level;
    F->loss_lambda = cfg.lambda;
    F->loss_lambda_d = cfg.lambda_d;
}

// loss scalars and the frame's counts in one round trip
// `between` (optional) enqueues more work after the read-back copies and before the host waits
// for them (the next step's speculative render): the host then waits on the copies alone
gs_loss_result read_loss(gs_frame* F, const std::function<void()>& between = {}) {
    gs_context* C = F->ctx;
    C->pinned.ensure(sizeof(LossScalars) + 64);
    char* pin = static_cast<char*>(C->pinned.p);
    ck(cudaMemcpyAsync(pin, F->loss.p, sizeof(LossScalars), cudaMemcpyDeviceToHost, C->stream), "d2h loss");
    if (!F->counts_known)
        ck(cudaMemcpyAsync(pin + sizeof(LossScalars), F->counters.p, kNumCounters * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, C->stream), "d2h counters");
    if (between) {
        if (!C->loss_ready) ck(cudaEventCreateWithFlags(&C->loss_ready, cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaEventRecord(C->loss_ready, C->stream), "record read-back");
        between();
        ck(cudaEventSynchronize(C->loss_ready), "sync loss");
    } else {
        ck(cudaStreamSynchronize(C->stream), "sync loss");
    }
    if (!F->counts_known) take_counts(F, reinterpret_cast<const unsigned long long*>(pin + sizeof(LossScalars)));
    LossScalars s;
    std::memcpy(&s, pin, sizeof(s));
    const int h = F->view.height, w = F->view.width;
    const double inv_n = 1.0 / (static_cast<double>(h) * w * 3);
    gs_loss_result r{};
    r.l1 = s.l1_sum * inv_n;
    r.ssim = F->loss_lambda != 0.0 ? s.ssim_sum / (static_cast<double>(h - 10) * (w - 10) * 3) : 0.0;
    r.color_loss = (1.0 - F->loss_lambda) * r.l1 + (F->loss_lambda != 0.0 ? F->loss_lambda * (1.0 - r.ssim) : 0.0);
    r.depth_loss = s.n_valid > 0 ? s.depth_abs_sum / static_cast<double>(s.n_valid) : 0.0;
    r.total = r.color_loss + F->loss_lambda_d * r.depth_loss;
    const double mse = s.sq_sum * inv_n;
    r.psnr = mse == 0.0 ? 100.0 : 10.0 * std::log10(1.0 / mse);
    return r;
}

int schedule_level(const gs_keyframe* K, const gs_train_config& cfg) {  // mapper.cpp:221-224
    const int n = static_cast<int>(K->hs.size()) - 1;
    const int ipl = cfg.iters_per_level > 0 ? cfg.iters_per_level
                                            : std::max(1, K->initial_iters / (cfg.pyramid_levels + 1));
    return n - std::min(n, K->consumed / ipl);
}

void keyframe_build(gs_keyframe* K, const float* color0, const float* depth0, int h, int w, int levels,
                    bool device_src) {
    if (levels < 0) fail(GS_EINVAL, "build_pyramid: levels must be >= 0");
    if (h < (1 << levels) || w < (1 << levels)) fail(GS_EINVAL, "build_pyramid: image too small for requested levels");
    cudaStream_t st = K->ctx->stream;
    K->hs.assign(levels + 1, 0);
    K->ws.assign(levels + 1, 0);
    K->color.resize(levels + 1);
    K->depth.resize(levels + 1);
    for (auto* v : {&K->color, &K->depth})
        for (DevBuf& b : *v) b.pool = st;
    K->stage.pool = st;
    if (!device_src) K->stage.ensure(sizeof(double) * 4 * static_cast<size_t>(h) * w);  // host-upload staging
    int ch = h, cw = w;
    for (int l = 0; l <= levels; ++l) {
        K->hs[l] = ch;
        K->ws[l] = cw;
        K->color[l].ensure(sizeof(float) * 3 * ch * cw);
        K->depth[l].ensure(sizeof(float) * ch * cw);
        ch = (ch + 1) / 2;
        cw = (cw + 1) / 2;
    }
    const cudaMemcpyKind kind = device_src ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    ck(cudaMemcpyAsync(K->color[0].p, color0, sizeof(float) * 3 * h * w, kind, st), "upload color");
    ck(cudaMemcpyAsync(K->depth[0].p, depth0, sizeof(float) * h * w, kind, st), "upload depth");
    for (int l = 1; l <= levels; ++l) {
        launch_downsample(K->color[l - 1].as<float>(), K->hs[l - 1], K->ws[l - 1], 3, false, K->color[l].as<float>(), st);
        launch_downsample(K->depth[l - 1].as<float>(), K->hs[l - 1], K->ws[l - 1], 1, true, K->depth[l].as<float>(), st);
        K->ctx->launched(2);
    }
    ck(cudaStreamSynchronize(st), "sync keyframe");
}

gs_frame* scratch_frame(gs_context* C) {
    if (!C->scratch_frame) {
        C->scratch_frame = new gs_frame();
        C->scratch_frame->ctx = C;
    }
    return C->scratch_frame;
}

gs_frame* train_frame(gs_context* C, int i) {
    if (!C->train_frames[i]) {
        C->train_frames[i] = new gs_frame();
        C->train_frames[i]->ctx = C;
    }
    return C->train_frames[i];
}

gs_grads* scratch_grads(gs_context* C) {
    if (!C->scratch_grads) {
        C->scratch_grads = new gs_grads();
        C->scratch_grads->ctx = C;
    }
    return C->scratch_grads;
}

void train_view(gs_map* M, gs_keyframe* K, const gs_train_config& cfg, const gs_camera& cam, gs_frame* F,
                gs_grads* G, int* level_out, bool exact_counts) {
    const int level = schedule_level(K, cfg);
    const gs_camera lc = scaled(cam, level);
    render_impl(M, K->pose, lc, F, exact_counts, F != M->ctx->scratch_frame);
    loss_impl(F, K, level, cfg);
    backward_impl(M, F, F->dl_dcolor.as<float>(), F->depth_cot.as<float>(), &F->loss.as<LossScalars>()->depth_scale, G);
    *level_out = level;
}

}  // namespace

// ============================================================================ C-ABI
extern "C" {

const char* gs_last_error(void) { return g_err.c_str(); }
const char* gs_version(void) { return "gsmap_b200 0.1 (sm_100a)"; }

int gs_context_create(int device, void* stream, gs_context** out) {
    return guard([&] {
        auto* C = new gs_context();
        C->device = device;
        try {
            C->use();
            // freed pool memory stays reserved for reuse (keyframes come and go in the mapping loop)
            cudaMemPool_t mp = nullptr;
            if (cudaDeviceGetDefaultMemPool(&mp, device) == cudaSuccess) {
                uint64_t keep = UINT64_MAX;
                cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &keep);
            }
            if (stream) {
                C->stream = static_cast<cudaStream_t>(stream);
            } else {
                ck(cudaStreamCreateWithFlags(&C->stream, cudaStreamNonBlocking), "cudaStreamCreate");
                C->own_stream = true;
            }
            for (DevBuf& b : C->scratch) b.pool = C->stream;
        } catch (...) {
            delete C;
            throw;
        }
        *out = C;
    });
}

int gs_context_destroy(gs_context* C) {
    return guard([&] {
        if (!C) return;
        C->use();
        cudaStreamSynchronize(C->stream);
        delete C->scratch_frame;
        delete C->train_frames[0];
        delete C->train_frames[1];
        if (C->loss_ready) cudaEventDestroy(C->loss_ready);
        if (C->scratch_grads && C->scratch_grads->planes && !C->scratch_grads->external)
            pool_free(C->scratch_grads->planes, C->stream);
        delete C->scratch_grads;
        if (C->copy_stream) {
            cudaStreamSynchronize(C->copy_stream);
            cudaStreamDestroy(C->copy_stream);
        }
        C->cub_tmp.release();
        for (DevBuf& b : C->scratch) b.release();
        if (C->own_stream) cudaStreamDestroy(C->stream);
        delete C;
    });
}

int gs_context_synchronize(gs_context* C) {
    return guard([&] {
        if (C->copy_stream) ck(cudaStreamSynchronize(C->copy_stream), "cudaStreamSynchronize");
        ck(cudaStreamSynchronize(C->stream), "cudaStreamSynchronize");
    });
}

int gs_context_set_stream(gs_context* C, void* stream) {
    return guard([&] {
        ck(cudaStreamSynchronize(C->stream), "sync");
        if (C->own_stream) cudaStreamDestroy(C->stream);
        C->own_stream = false;
        C->stream = static_cast<cudaStream_t>(stream);
    });
}

int gs_context_launch_count(gs_context* C, int64_t* count) {
    return guard([&] { *count = C->launches; });
}

int gs_debug_set_blend_ppt(int fwd, int bwd) {
    return guard([&] { set_blend_ppt(fwd, bwd); });
}

int gs_debug_set_blend_df_list(int entries) {
    return guard([&] { set_blend_df_list(entries); });
}

int gs_debug_profile_host(gs_context* C, char* names, int32_t names_len, double* host_ms, int32_t max_entries,
                          int32_t* n_entries) {
    return guard([&] {
        std::vector<std::string> keys;
        std::vector<double> ms;
        for (const auto& r : C->prof) {
            size_t k = 0;
            while (k < keys.size() && keys[k] != r.name) ++k;
            if (k == keys.size()) {
                keys.emplace_back(r.name);
                ms.push_back(0.0);
            }
            ms[k] += r.host_us * 1e-3;
        }
        std::string joined;
        const int n = std::min<int>(static_cast<int>(keys.size()), max_entries);
        for (int i = 0; i < n; ++i) {
            joined += keys[i];
            joined += '\n';
            host_ms[i] = ms[i];
        }
        if (static_cast<int>(joined.size()) + 1 > names_len) fail(GS_EINVAL, "profile_host: names buffer too small");
        std::memcpy(names, joined.c_str(), joined.size() + 1);
        *n_entries = n;
    });
}

int gs_debug_defer_step_sync(gs_context* C, int defer) {
    return guard([&] { C->defer_sync = defer != 0; });
}

int gs_debug_set_blend_segments(int nseg) {
    return guard([&] { set_blend_segments(nseg); });
}

int gs_debug_set_seg_forward(int max_tiles) {
    return guard([&] { set_blend_seg_forward(max_tiles); });
}

int gs_debug_counters(gs_context* C, int64_t* out2, int reset) {
    return guard([&] {
        C->use();
        ck(cudaStreamSynchronize(C->stream), "sync");
        unsigned long long v[2];
        read_blend_stats(v, reset != 0);
        out2[0] = static_cast<int64_t>(v[0]);
        out2[1] = static_cast<int64_t>(v[1]);
    });
}

int gs_context_profile(gs_context* C, int enable) {
    return guard([&] {
        ck(cudaStreamSynchronize(C->stream), "sync");
        C->profile = enable != 0;
        C->prof.clear();
        C->ev_next = 0;
    });
}

int gs_context_profile_read(gs_context* C, char* names, int32_t names_len, double* total_ms, int64_t* launches,
                            int32_t max_entries, int32_t* n_entries) {
    return guard([&] {
        ck(cudaStreamSynchronize(C->stream), "sync");
        std::vector<std::string> keys;
        std::vector<double> ms;
        std::vector<int64_t> cnt;
        for (const auto& r : C->prof) {
            float t = 0.f;
            ck(cudaEventElapsedTime(&t, r.a, r.b), "cudaEventElapsedTime");
            size_t k = 0;
            while (k < keys.size() && keys[k] != r.name) ++k;
            if (k == keys.size()) {
                keys.emplace_back(r.name);
                ms.push_back(0.0);
                cnt.push_back(0);
            }
            ms[k] += t;
            cnt[k] += 1;
        }
        std::string joined;
        const int n = std::min<int>(static_cast<int>(keys.size()), max_entries);
        for (int i = 0; i < n; ++i) {
            joined += keys[i];
            joined += '\n';
            total_ms[i] = ms[i];
            launches[i] = cnt[i];
        }
        if (static_cast<int>(joined.size()) + 1 > names_len) fail(GS_EINVAL, "profile_read: names buffer too small");
        std::memcpy(names, joined.c_str(), joined.size() + 1);
        *n_entries = n;
    });
}

int gs_camera_validate(const gs_camera* cam) { return guard([&] { validate_camera(*cam); }); }
int gs_camera_scaled(const gs_camera* cam, int level, gs_camera* out) { return guard([&] { *out = scaled(*cam, level); }); }

// ---------------------------------------------------------------- map
int gs_map_create(gs_context* C, gs_map** out) {
    return guard([&] {
        auto* M = new gs_map();
        M->ctx = C;
        *out = M;
    });
}

int gs_map_destroy(gs_map* M) {
    return guard([&] {
        if (!M) return;
        if (M->ctx->spec.map == M) M->ctx->spec.valid = false;
        M->ctx->use();
        cudaStreamSynchronize(M->ctx->stream);
        M->free_all();
        M->minmax.release();
        delete M;
    });
}

int gs_map_size(const gs_map* M, int64_t* n) { return guard([&] { *n = M->n; }); }

int gs_map_append(gs_map* M, const gs_gaussian* g, int64_t n) {
    return guard([&] {
        M->ctx->use();
        if (n < 0) fail(GS_EINVAL, "append: negative count");
        map_reserve(M, M->n + n);
        // fresh optimizer state for the new range (gaussian_map.cpp:33)
        cudaStream_t st = M->ctx->stream;
        if (n > 0) {
            ck(cudaMemset2DAsync(M->m + M->n, sizeof(float) * M->cap, 0, sizeof(float) * n, kNumParams, st), "memset");
            ck(cudaMemset2DAsync(M->v + M->n, sizeof(float) * M->cap, 0, sizeof(float) * n, kNumParams, st), "memset");
            const std::vector<int32_t> b(n, static_cast<int32_t>(M->adam_count));  // fresh state: step 0
            ck(cudaMemcpyAsync(M->birth + M->n, b.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st), "h2d birth");
            ck(cudaStreamSynchronize(st), "sync");
        }
        upload_gaussians(M, g, M->n, n);
        M->n += n;
        refresh_extent(M);
    });
}

int gs_map_set_gaussians(gs_map* M, const gs_gaussian* g, int64_t n) {
    return guard([&] {
        M->ctx->use();
        if (n != M->n) fail(GS_EINVAL, "set_gaussians: count does not match map size");
        upload_gaussians(M, g, 0, n);
    });
}

int gs_map_get_gaussians(gs_map* M, gs_gaussian* out, int64_t n) {
    return guard([&] {
        M->ctx->use();
        if (n != M->n) fail(GS_EINVAL, "get_gaussians: count does not match map size");
        if (n == 0) return;
        std::vector<float> soa(static_cast<size_t>(kNumParams) * n);
        ck(cudaMemcpy2DAsync(soa.data(), sizeof(float) * n, M->params, sizeof(float) * M->cap, sizeof(float) * n,
                             kNumParams, cudaMemcpyDeviceToHost, M->ctx->stream), "download params");
        ck(cudaStreamSynchronize(M->ctx->stream), "sync");
        for (int64_t i = 0; i < n; ++i) {
            for (int k = 0; k < kNumParams; ++k) out[i].p[k] = soa[static_cast<size_t>(k) * n + i];
            out[i].active_degree = M->deg_host[i];
            out[i].pad = 0;
        }
    });
}

int gs_map_get_adam(gs_map* M, double* m59, double* v59, int64_t* step, int64_t n) {
    return guard([&] {
        M->ctx->use();
        if (n != M->n) fail(GS_EINVAL, "get_adam: count does not match map size");
        if (n == 0) return;
        std::vector<float> a(static_cast<size_t>(kNumParams) * n), b(a.size());
        std::vector<int32_t> s(n);
        cudaStream_t st = M->ctx->stream;
        ck(cudaMemcpy2DAsync(a.data(), sizeof(float) * n, M->m, sizeof(float) * M->cap, sizeof(float) * n, kNumParams,
                             cudaMemcpyDeviceToHost, st), "d2h");
        ck(cudaMemcpy2DAsync(b.data(), sizeof(float) * n, M->v, sizeof(float) * M->cap, sizeof(float) * n, kNumParams,
                             cudaMemcpyDeviceToHost, st), "d2h");
        ck(cudaMemcpyAsync(s.data(), M->birth, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st), "d2h");
        ck(cudaStreamSynchronize(st), "sync");
        for (int64_t i = 0; i < n; ++i) {
            for (int k = 0; k < kNumParams; ++k) {
                if (m59) m59[i * kNumParams + k] = a[static_cast<size_t>(k) * n + i];
                if (v59) v59[i * kNumParams + k] = b[static_cast<size_t>(k) * n + i];
            }
            if (step) step[i] = M->adam_count - s[i];
        }
    });
}

int gs_map_set_adam(gs_map* M, const double* m59, const double* v59, const int64_t* step, int64_t n) {
    return guard([&] {
        M->ctx->use();
        if (n != M->n) fail(GS_EINVAL, "set_adam: count does not match map size");
        if (n == 0) return;
        std::vector<float> a(static_cast<size_t>(kNumParams) * n), b(a.size());
        std::vector<int32_t> s(n);
        for (int64_t i = 0; i < n; ++i) {
            for (int k = 0; k < kNumParams; ++k) {
                a[static_cast<size_t>(k) * n + i] = static_cast<float>(m59[i * kNumParams + k]);
                b[static_cast<size_t>(k) * n + i] = static_cast<float>(v59[i * kNumParams + k]);
            }
            s[i] = static_cast<int32_t>(M->adam_count - step[i]);
        }
        cudaStream_t st = M->ctx->stream;
        ck(cudaMemcpy2DAsync(M->m, sizeof(float) * M->cap, a.data(), sizeof(float) * n, sizeof(float) * n, kNumParams,
                             cudaMemcpyHostToDevice, st), "h2d");
        ck(cudaMemcpy2DAsync(M->v, sizeof(float) * M->cap, b.data(), sizeof(float) * n, sizeof(float) * n, kNumParams,
                             cudaMemcpyHostToDevice, st), "h2d");
        ck(cudaMemcpyAsync(M->birth, s.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st), "h2d");
        ck(cudaStreamSynchronize(st), "sync");
    });
}

int gs_map_scene_extent(const gs_map* M, double* e) { return guard([&] { *e = M->scene_extent; }); }
int gs_map_set_scene_extent(gs_map* M, double e) { return guard([&] { M->scene_extent = e; }); }
int gs_map_global_step(const gs_map* M, int64_t* s) { return guard([&] { *s = M->global_step; }); }
int gs_map_set_global_step(gs_map* M, int64_t s) { return guard([&] { M->global_step = s; }); }

int gs_map_raise_sh_degree(gs_map* M, int degree) {  // gaussian_map.cpp:75-79
    return guard([&] {
        M->ctx->use();
        const int d = std::clamp(degree, 0, 3);
        for (auto& x : M->deg_host) x = static_cast<int8_t>(std::max<int>(x, d));
        if (M->n > 0)
            ck(cudaMemcpyAsync(M->degree, M->deg_host.data(), M->n, cudaMemcpyHostToDevice, M->ctx->stream), "h2d");
        ck(cudaStreamSynchronize(M->ctx->stream), "sync");
        M->recompute_max_degree();
    });
}

int gs_map_max_active_degree(gs_map* M, int* degree) { return guard([&] { *degree = M->max_degree; }); }

int gs_project_sparse_depth(gs_context* C, const double* points, int64_t n, int32_t stride, const gs_pose* pose,
                            const gs_camera* cam, double* depth) {  // sequence.cpp:246-259
    return guard([&] {
        validate_camera(*cam);
        if (n < 0 || stride < 3) fail(GS_EINVAL, "project_sparse_depth: bad point array");
        C->use();
        cudaStream_t st = C->stream;
        const ViewParams v = make_view(*pose, *cam);
        const size_t P = static_cast<size_t>(cam->width) * cam->height;
        DevBuf &pts = C->sc(kScPoints), &out = C->sc(kScDepth);
        pts.ensure(sizeof(double) * static_cast<size_t>(std::max<int64_t>(n, 1)) * stride);
        out.ensure(sizeof(double) * P);
        if (n > 0)
            ck(cudaMemcpyAsync(pts.p, points, sizeof(double) * static_cast<size_t>(n) * stride, cudaMemcpyHostToDevice,
                               st), "h2d points");
        launch_sparse_depth(pts.as<double>(), stride, n, v, out.as<double>(), st);
        C->launched(3);
        ck(cudaMemcpyAsync(depth, out.p, sizeof(double) * P, cudaMemcpyDeviceToHost, st), "d2h depth");
        ck(cudaStreamSynchronize(st), "sync");
    });
}

int gs_maybe_upgrade_sh(gs_map* M, int32_t sh_interval, int32_t* degree) {  // mapper.cpp:240-246
    return guard([&] {
        if (sh_interval <= 0) {
            *degree = M->max_degree;
            return;
        }
        const int target = static_cast<int>(std::min<int64_t>(3, M->global_step / sh_interval));
        const int d = std::clamp(target, 0, 3);
        if (d <= M->min_degree) {  // every Gaussian is already there (the common case): O(1)
            *degree = target;
            return;
        }
        bool change = false;
        for (auto& x : M->deg_host)
            if (x < d) {
                x = static_cast<int8_t>(d);
                change = true;
            }
        if (change && M->n > 0) {
            M->ctx->use();
            ck(cudaMemcpyAsync(M->degree, M->deg_host.data(), M->n, cudaMemcpyHostToDevice, M->ctx->stream), "h2d");
            ck(cudaStreamSynchronize(M->ctx->stream), "sync");
        }
        M->recompute_max_degree();
        *degree = target;
    });
}

// init_gaussians_from_points on device-resident points [n][6] (n > 0); appends to the map
void init_points_device(gs_map* M, const double* dpts, int64_t n) {
        gs_context* C = M->ctx;
        cudaStream_t st = C->stream;
        DevBuf &keys = C->sc(kScKeys), &keys2 = C->sc(kScKeys2), &idx = C->sc(kScIdx), &idx2 = C->sc(kScIdx2),
               &bb = C->sc(kScBBox), &hk = C->sc(kScHashK), &hv = C->sc(kScHashV);
        keys.ensure(sizeof(uint64_t) * n);
        keys2.ensure(sizeof(uint64_t) * n);
        idx.ensure(sizeof(int32_t) * n);
        idx2.ensure(sizeof(int32_t) * n);
        bb.ensure(sizeof(unsigned long long) * 8);
        launch_knn_bbox(dpts, n, bb.as<unsigned long long>(), st);
        unsigned long long enc[6];
        ck(cudaMemcpyAsync(enc, bb.p, sizeof(enc), cudaMemcpyDeviceToHost, st), "d2h");
        ck(cudaStreamSynchronize(st), "sync");
        double lo[3], hi[3];
        auto dec = [](unsigned long long u) {
            const unsigned long long b = (u & 0x8000000000000000ull) ? (u & 0x7fffffffffffffffull) : ~u;
            double d;
            std::memcpy(&d, &b, sizeof d);
            return d;
        };
        for (int a = 0; a < 3; ++a) {
            lo[a] = dec(enc[a]);
            hi[a] = dec(enc[3 + a]);
        }
        const double ext[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
        const double vol = std::max(ext[0], 1e-9) * std::max(ext[1], 1e-9) * std::max(ext[2], 1e-9);
        KnnGrid g{};
        for (int a = 0; a < 3; ++a) g.lo[a] = lo[a];
        g.cell = std::cbrt(vol / static_cast<double>(n)) * 1.5;
        size_t tb = 0;
        auto sort_keys = [&]() {
            launch_knn_keys(dpts, n, g, keys.as<uint64_t>(), idx.as<int32_t>(), st);
            tb = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.as<uint64_t>(), keys2.as<uint64_t>(), idx.as<int32_t>(),
                                            idx2.as<int32_t>(), static_cast<int>(n), 0, 64, st);
            ck(cub::DeviceRadixSort::SortPairs(C->cub(tb), tb, keys.as<uint64_t>(), keys2.as<uint64_t>(),
                                               idx.as<int32_t>(), idx2.as<int32_t>(), static_cast<int>(n), 0, 64, st),
               "knn sort");
        };
        // adapt the cell so occupied cells hold ~4 points (fixtures/synthetic.cpp init_from_points)
        for (int it = 0; it < 2; ++it) {
            sort_keys();
            launch_knn_count_runs(keys2.as<uint64_t>(), n, bb.as<unsigned long long>() + 6, st);
            unsigned long long runs = 1;
            ck(cudaMemcpyAsync(&runs, bb.as<unsigned long long>() + 6, sizeof(runs), cudaMemcpyDeviceToHost, st), "d2h");
            ck(cudaStreamSynchronize(st), "sync");
            g.cell *= std::cbrt(4.0 / (static_cast<double>(n) / static_cast<double>(std::max(runs, 1ull))));
        }
        sort_keys();
        g.max_ring = std::max({static_cast<int64_t>(ext[0] / g.cell) + 1, static_cast<int64_t>(ext[1] / g.cell) + 1,
                               static_cast<int64_t>(ext[2] / g.cell) + 1});
        uint32_t hsize = 1024;
        while (hsize < 2 * static_cast<uint64_t>(n)) hsize <<= 1;
        hk.ensure(sizeof(uint64_t) * hsize);
        hv.ensure(sizeof(int2) * hsize);
        launch_knn_table(keys2.as<uint64_t>(), n, hk.as<uint64_t>(), hv.as<int2>(), hsize - 1, st);
        // new Gaussians at [first, first + n): fresh optimizer state, degree 0 (gaussian_map.cpp:33)
        const int64_t first = M->n;
        map_reserve(M, first + n);
        ck(cudaMemset2DAsync(M->m + first, sizeof(float) * M->cap, 0, sizeof(float) * n, kNumParams, st), "memset");
        ck(cudaMemset2DAsync(M->v + first, sizeof(float) * M->cap, 0, sizeof(float) * n, kNumParams, st), "memset");
        ck(cudaMemsetAsync(M->degree + first, 0, n, st), "memset");
        const std::vector<int32_t> birth(n, static_cast<int32_t>(M->adam_count));
        ck(cudaMemcpyAsync(M->birth + first, birth.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st), "h2d");
        const int k = static_cast<int>(std::min<int64_t>(3, n - 1));
        launch_knn_init(dpts, n, k, g, hk.as<uint64_t>(), hv.as<int2>(), hsize - 1, idx2.as<int32_t>(),
                        M->params, M->cap, first, st);
        C->launched(8);
        ck(cudaStreamSynchronize(st), "sync");
        M->deg_host.resize(first + n, 0);
        M->n = first + n;
        M->recompute_max_degree();
        refresh_extent(M);
}

int gs_map_init_from_points(gs_map* M, const double* pts6, int64_t n, int64_t* added) {  // mapper.cpp:43-61
    return guard([&] {
        *added = 0;
        if (n <= 0) return;  // points.empty() -> 0
        if (n > 0x7fffffff) fail(GS_EINVAL, "init_from_points: too many points");
        M->ctx->use();
        DevBuf& pts = M->ctx->sc(kScPoints);
        pts.ensure(sizeof(double) * 6 * n);
        ck(cudaMemcpyAsync(pts.p, pts6, sizeof(double) * 6 * n, cudaMemcpyHostToDevice, M->ctx->stream), "h2d points");
        init_points_device(M, pts.as<double>(), n);
        *added = n;
    });
}

// filter_points_by_visibility on the device: render the map at the pose, flag, compact (stable);
// returns the kept count, kept points in `out` (device, [kept][6])
int64_t filter_points_device(gs_map* M, const double* dpts, int64_t n, const gs_pose& pose, const gs_camera& cam,
                             double tau_alpha, DevBuf& out) {
    if (tau_alpha < 0.0 || tau_alpha > 1.0)
        fail(GS_EINVAL, "filter_points_by_visibility: tau_alpha must be in [0,1]");
    gs_context* C = M->ctx;
    cudaStream_t st = C->stream;
    gs_frame* F = scratch_frame(C);
    render_impl(M, pose, cam, F, true, false);
    DevBuf &keep = C->sc(kScKeep), &pos = C->sc(kScPos);
    keep.ensure(sizeof(int32_t) * (n + 1));
    pos.ensure(sizeof(int32_t) * (n + 1));
    ck(cudaMemsetAsync(keep.as<int32_t>() + n, 0, sizeof(int32_t), st), "memset");
    launch_vis_filter(dpts, n, F->view, F->vis.as<float>(), tau_alpha, keep.as<int32_t>(), st);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, keep.as<int32_t>(), pos.as<int32_t>(), n + 1, st);
    ck(cub::DeviceScan::ExclusiveSum(C->cub(tb), tb, keep.as<int32_t>(), pos.as<int32_t>(), n + 1, st), "scan");
    int32_t kept = 0;
    ck(cudaMemcpyAsync(&kept, pos.as<int32_t>() + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "d2h");
    ck(cudaStreamSynchronize(st), "sync");
    out.ensure(sizeof(double) * 6 * std::max<int64_t>(kept, 1));
    launch_compact_points(dpts, n, keep.as<int32_t>(), pos.as<int32_t>(), out.as<double>(), st);
    C->launched(3);
    return kept;
}

// ------------------------------------------------------------------ checkpoint v1 (io/checkpoint.cpp)
// Text header then one 476-byte record per Gaussian: the 59 parameters as fp64 in reference
// order (position, rotation w x y z, log_scale, opacity_logit, sh[16][3]) and int32
// active_degree. The device map holds fp32 parameters, so a save writes their exact fp64
// widening and a load rounds to fp32 (a map saved here reloads bit-identically).
int gs_save_checkpoint(gs_map* M, const char* path) {
    return guard([&] {  // save_checkpoint, io/checkpoint.cpp:17-35
        M->ctx->use();
        std::ofstream out(path, std::ios::binary);
        if (!out) fail(GS_ERUNTIME, std::string("save_checkpoint: cannot open ") + path);
        const int64_t n = M->n;
        int maxd = 0;
        for (int64_t i = 0; i < n; ++i) maxd = std::max<int>(maxd, M->deg_host[i]);
        out << "gsmap-checkpoint" << ' ' << 1 << '\n' << "count " << static_cast<size_t>(n) << '\n'
            << "sh_degree " << maxd << '\n' << "end_header\n";
        constexpr int64_t kChunk = 1 << 16;
        constexpr size_t kRec = sizeof(double) * kNumParams + sizeof(int32_t);
        std::vector<float> soa(static_cast<size_t>(kNumParams) * std::min(n, kChunk));
        std::vector<char> rec(kRec * std::min(n, kChunk));
        for (int64_t b = 0; b < n; b += kChunk) {
            const int64_t m = std::min(kChunk, n - b);
            ck(cudaMemcpy2DAsync(soa.data(), sizeof(float) * m, M->params + b, sizeof(float) * M->cap,
                                 sizeof(float) * m, kNumParams, cudaMemcpyDeviceToHost, M->ctx->stream), "d2h params");
            ck(cudaStreamSynchronize(M->ctx->stream), "sync");
            for (int64_t i = 0; i < m; ++i) {
                char* r = rec.data() + kRec * i;
                for (int k = 0; k < kNumParams; ++k) {
                    const double v = soa[static_cast<size_t>(k) * m + i];
                    std::memcpy(r + sizeof(double) * k, &v, sizeof(double));
                }
                const int32_t deg = M->deg_host[b + i];
                std::memcpy(r + sizeof(double) * kNumParams, &deg, sizeof(deg));
            }
            out.write(rec.data(), static_cast<std::streamsize>(kRec * m));
        }
        if (!out) fail(GS_ERUNTIME, std::string("save_checkpoint: write failed for ") + path);
    });
}

int gs_load_checkpoint(gs_context* C, const char* path, gs_map** out) {
    return guard([&] {  // load_checkpoint, io/checkpoint.cpp:37-71
        *out = nullptr;
        std::ifstream in(path, std::ios::binary);
        if (!in) fail(GS_ERUNTIME, std::string("load_checkpoint: cannot open ") + path);
        std::string line, magic;
        std::getline(in, line);
        std::istringstream head(line);
        int version = 0;
        head >> magic >> version;
        if (magic != "gsmap-checkpoint") fail(GS_ERUNTIME, std::string("load_checkpoint: not a checkpoint file: ") + path);
        if (version != 1) fail(GS_ERUNTIME, std::string("load_checkpoint: unsupported version in ") + path);
        size_t count = 0;
        while (std::getline(in, line) && line != "end_header") {
            std::istringstream is(line);
            std::string key;
            is >> key;
            if (key == "count") is >> count;
        }
        std::vector<gs_gaussian> gs(count);
        for (gs_gaussian& g : gs) {
            in.read(reinterpret_cast<char*>(g.p), sizeof(g.p));
            int32_t deg = 0;
            in.read(reinterpret_cast<char*>(&deg), sizeof(deg));
            g.active_degree = deg;
            g.pad = 0;
        }
        if (!in) fail(GS_ERUNTIME, std::string("load_checkpoint: truncated file ") + path);
        gs_map* M = nullptr;
        int st = gs_map_create(C, &M);
        if (st != GS_OK) fail(st, g_err);
        st = gs_map_append(M, gs.data(), static_cast<int64_t>(gs.size()));
        if (st != GS_OK) {
            const std::string msg = g_err;
            gs_map_destroy(M);
            fail(st, msg);
        }
        *out = M;
    });
}

// Optimizer state beside a v1 checkpoint ("add Adam state for true resume"; the
// reference's format has none, load_checkpoint starts Adam afresh): text header, then per
// Gaussian m[59], v[59] (fp64 widening of the device's fp32 moments) and the int64 Adam step.
int gs_save_training_state(gs_map* M, const char* path) {
    return guard([&] {
        M->ctx->use();
        const int64_t n = M->n;
        std::vector<double> m(static_cast<size_t>(kNumParams) * n), v(m.size());
        std::vector<int64_t> step(n);
        if (n > 0) {
            const int st = gs_map_get_adam(M, m.data(), v.data(), step.data(), n);
            if (st != GS_OK) fail(st, g_err);
        }
        std::ofstream out(path, std::ios::binary);
        if (!out) fail(GS_ERUNTIME, std::string("save_training_state: cannot open ") + path);
        // scene_extent too: the reference refreshes it only on append (gaussian_map.cpp:87-99), so a
        // reloaded map would otherwise rescale the position learning rate by its trained extent
        out << "gsmap-adam-state 1\ncount " << n << "\nglobal_step " << M->global_step << "\nscene_extent "
            << std::setprecision(17) << M->scene_extent << "\nend_header\n";
        for (int64_t i = 0; i < n; ++i) {
            out.write(reinterpret_cast<const char*>(&m[kNumParams * i]), sizeof(double) * kNumParams);
            out.write(reinterpret_cast<const char*>(&v[kNumParams * i]), sizeof(double) * kNumParams);
            out.write(reinterpret_cast<const char*>(&step[i]), sizeof(int64_t));
        }
        if (!out) fail(GS_ERUNTIME, std::string("save_training_state: write failed for ") + path);
    });
}

int gs_load_training_state(gs_map* M, const char* path) {
    return guard([&] {
        M->ctx->use();
        std::ifstream in(path, std::ios::binary);
        if (!in) fail(GS_ERUNTIME, std::string("load_training_state: cannot open ") + path);
        std::string line, magic;
        std::getline(in, line);
        std::istringstream head(line);
        int version = 0;
        head >> magic >> version;
        if (magic != "gsmap-adam-state" || version != 1)
            fail(GS_ERUNTIME, std::string("load_training_state: not an optimizer state file: ") + path);
        int64_t count = -1, gstep = 0;
        double extent = M->scene_extent;
        while (std::getline(in, line) && line != "end_header") {
            std::istringstream is(line);
            std::string key;
            is >> key;
            if (key == "count") is >> count;
            if (key == "global_step") is >> gstep;
            if (key == "scene_extent") is >> extent;
        }
        if (count != M->n) fail(GS_EINVAL, "load_training_state: Gaussian count does not match the map");
        std::vector<double> m(static_cast<size_t>(kNumParams) * count), v(m.size());
        std::vector<int64_t> step(count);
        for (int64_t i = 0; i < count; ++i) {
            in.read(reinterpret_cast<char*>(&m[kNumParams * i]), sizeof(double) * kNumParams);
            in.read(reinterpret_cast<char*>(&v[kNumParams * i]), sizeof(double) * kNumParams);
            in.read(reinterpret_cast<char*>(&step[i]), sizeof(int64_t));
        }
        if (!in) fail(GS_ERUNTIME, std::string("load_training_state: truncated file ") + path);
        if (count > 0) {
            const int st = gs_map_set_adam(M, m.data(), v.data(), step.data(), count);
            if (st != GS_OK) fail(st, g_err);
        }
        M->global_step = gstep;
        M->scene_extent = extent;
    });
}

int gs_integrate_keyframe(gs_map* M, const gs_pose* pose, const gs_camera* cam, const double* color,
                          const double* points6, int64_t n, double tau_alpha, int32_t initial_iters, int32_t levels,
                          gs_keyframe** out_kf, int64_t* added) {
    return guard([&] {  // pipeline.cpp:148-155 (+ the keyframe's sparse depth, pipeline.cpp:108)
        validate_camera(*cam);
        gs_context* C = M->ctx;
        C->use();
        *out_kf = nullptr;
        *added = 0;
        if (tau_alpha < 0.0 || tau_alpha > 1.0)
            fail(GS_EINVAL, "filter_points_by_visibility: tau_alpha must be in [0,1]");
        if (n < 0 || n > 0x7fffffff) fail(GS_EINVAL, "integrate_keyframe: bad point count");
        if (!color) fail(GS_EINVAL, "integrate_keyframe: missing colour image");
        cudaStream_t st = C->stream;
        const int h = cam->height, w = cam->width;
        const size_t P = static_cast<size_t>(h) * w;
        // the cloud crosses once: filter -> init, and the sparse depth, read the same device copy
        DevBuf &pts = C->sc(kScPoints), &kept = C->sc(kScKept), &dd = C->sc(kScDepth), &cs = C->sc(kScColor);
        std::optional<Scope> sc_up(std::in_place, C, "kf_upload_sparse_depth");
        pts.ensure(sizeof(double) * 6 * std::max<int64_t>(n, 1));
        if (n > 0)
            ck(cudaMemcpyAsync(pts.p, points6, sizeof(double) * 6 * n, cudaMemcpyHostToDevice, st), "h2d points");
        // sparse depth first: project_sparse_depth reads the frame's full cloud (sequence.cpp:246-259)
        dd.ensure(sizeof(double) * P + sizeof(float) * P);
        launch_sparse_depth(pts.as<double>(), 6, n, make_view(*pose, *cam), dd.as<double>(), st);
        float* depth_f = reinterpret_cast<float*>(dd.as<double>() + P);
        launch_from_hwc_double(dd.as<double>(), h, w, 1, depth_f, st);
        cs.ensure(sizeof(double) * 3 * P + sizeof(float) * 3 * P);
        ck(cudaMemcpyAsync(cs.p, color, sizeof(double) * 3 * P, cudaMemcpyHostToDevice, st), "h2d colour");
        float* color_f = reinterpret_cast<float*>(cs.as<double>() + 3 * P);
        launch_from_hwc_double(cs.as<double>(), h, w, 3, color_f, st);
        C->launched(5);
        sc_up.reset();
        auto* K = new gs_keyframe();
        K->ctx = C;
        K->pose = *pose;
        K->initial_iters = initial_iters;
        try {
            {
                Scope sc(C, "kf_pyramid");
                keyframe_build(K, color_f, depth_f, h, w, levels, true);
            }
            if (n > 0) {
                int64_t k = 0;
                {
                    Scope sc(C, "kf_filter_points");
                    k = filter_points_device(M, pts.as<double>(), n, *pose, *cam, tau_alpha, kept);
                }
                if (k > 0) {
                    Scope sc(C, "kf_init_gaussians");
                    init_points_device(M, kept.as<double>(), k);
                }
                *added = k;
            }
        } catch (...) {
            delete K;
            throw;
        }
        *out_kf = K;
    });
}

// diagnostics: K8b thread order (0 rank, 1 map, 2 visible list; -1 = automatic)
// diagnostics: speculative next-step renders enqueued / used so far on this context
int gs_debug_speculation(gs_context* C, int64_t* out2) {
    return guard([&] {
        out2[0] = C->spec_enqueued;
        out2[1] = C->spec_used;
    });
}

int gs_debug_set_k8_order(int order) {
    return guard([&] { set_k8_order(order); });
}

int gs_evaluate_view(gs_map* M, const gs_pose* pose, const gs_camera* cam, const double* gt_color,
                     const double* gt_depth, gs_eval_metrics* out) {
    return guard([&] {  // evaluate_sequence (pipeline.cpp:41-64), one frame
        gs_context* C = M->ctx;
        C->use();
        validate_camera(*cam);
        if (!gt_color) fail(GS_EINVAL, "evaluate_view: missing ground-truth colour");
        if (cam->width < 11 || cam->height < 11) fail(GS_EINVAL, "ssim: image smaller than the 11x11 window");
        gs_frame* F = scratch_frame(C);
        render_checked(M, *pose, *cam, F);
        cudaStream_t st = C->stream;
        const int h = cam->height, w = cam->width;
        const size_t P = static_cast<size_t>(h) * w;
        F->eval_quant.ensure(sizeof(float) * 3 * P);
        F->eval_gt.ensure(sizeof(float) * 4 * P);
        F->eval_stage.ensure(sizeof(double) * 4 * P);
        F->wbuf.ensure(sizeof(float) * 9 * static_cast<size_t>(h - 10) * (w - 10));
        double* stage = F->eval_stage.as<double>();
        float* gt = F->eval_gt.as<float>();
        ck(cudaMemcpyAsync(stage, gt_color, sizeof(double) * 3 * P, cudaMemcpyHostToDevice, st), "h2d gt colour");
        launch_from_hwc_double(stage, h, w, 3, gt, st);
        if (gt_depth) {
            ck(cudaMemcpyAsync(stage + 3 * P, gt_depth, sizeof(double) * P, cudaMemcpyHostToDevice, st), "h2d gt depth");
            launch_from_hwc_double(stage + 3 * P, h, w, 1, gt + 3 * P, st);
        }
        ck(cudaMemsetAsync(F->loss.p, 0, sizeof(LossScalars), st), "memset");
        launch_eval(F->color.as<float>(), F->depth.as<float>(), gt, gt_depth ? gt + 3 * P : nullptr, h, w,
                    F->eval_quant.as<float>(), F->wbuf.as<float>(), F->loss.as<LossScalars>(), st);
        C->launched(gt_depth ? 4 : 3);
        LossScalars r;
        ck(cudaMemcpyAsync(&r, F->loss.p, sizeof(r), cudaMemcpyDeviceToHost, st), "d2h");
        ck(cudaStreamSynchronize(st), "sync");
        F->has_cotangent = false;
        const double mse = r.sq_sum / (3.0 * static_cast<double>(P));
        out->psnr = mse == 0.0 ? 100.0 : 10.0 * std::log10(1.0 / mse);  // metrics.cpp:165-175
        out->ssim = r.ssim_sum / (3.0 * static_cast<double>(h - 10) * (w - 10));
        out->depth_rmse = r.n_valid ? std::sqrt(r.depth_abs_sum / static_cast<double>(r.n_valid))
                                    : std::numeric_limits<double>::quiet_NaN();
    });
}

int gs_filter_points_by_visibility(gs_map* M, const double* pts6, int64_t n, const gs_pose* pose,
                                   const gs_camera* cam, double tau_alpha, double* kept6, int64_t* n_kept) {
    return guard([&] {  // keyframe.cpp:49-74
        validate_camera(*cam);
        M->ctx->use();
        *n_kept = 0;
        if (tau_alpha < 0.0 || tau_alpha > 1.0)
            fail(GS_EINVAL, "filter_points_by_visibility: tau_alpha must be in [0,1]");
        if (n <= 0) return;
        DevBuf &pts = M->ctx->sc(kScPoints), &out = M->ctx->sc(kScKept);
        pts.ensure(sizeof(double) * 6 * n);
        ck(cudaMemcpyAsync(pts.p, pts6, sizeof(double) * 6 * n, cudaMemcpyHostToDevice, M->ctx->stream), "h2d");
        const int64_t kept = filter_points_device(M, pts.as<double>(), n, *pose, *cam, tau_alpha, out);
        if (kept > 0)
            ck(cudaMemcpyAsync(kept6, out.p, sizeof(double) * 6 * kept, cudaMemcpyDeviceToHost, M->ctx->stream), "d2h");
        ck(cudaStreamSynchronize(M->ctx->stream), "sync");
        *n_kept = kept;
    });
}

int gs_map_integrate_points(gs_map* M, const double* pts6, int64_t n, const gs_pose* pose, const gs_camera* cam,
                            double tau_alpha, int64_t* added) {
    return guard([&] {  // pipeline.cpp:151-155: filter_points_by_visibility -> init_gaussians_from_points
        validate_camera(*cam);
        M->ctx->use();
        *added = 0;
        if (tau_alpha < 0.0 || tau_alpha > 1.0)
            fail(GS_EINVAL, "filter_points_by_visibility: tau_alpha must be in [0,1]");
        if (n <= 0) return;
        if (n > 0x7fffffff) fail(GS_EINVAL, "integrate_points: too many points");
        DevBuf &pts = M->ctx->sc(kScPoints), &out = M->ctx->sc(kScKept);
        pts.ensure(sizeof(double) * 6 * n);
        ck(cudaMemcpyAsync(pts.p, pts6, sizeof(double) * 6 * n, cudaMemcpyHostToDevice, M->ctx->stream), "h2d");
        const int64_t kept = filter_points_device(M, pts.as<double>(), n, *pose, *cam, tau_alpha, out);
        if (kept > 0) init_points_device(M, out.as<double>(), kept);
        *added = kept;
    });
}

int gs_map_prune(gs_map* M, double opacity_threshold, int64_t* removed) {  // gaussian_map.cpp:56-73
    return guard([&] {
        if (opacity_threshold <= 0.0 || opacity_threshold >= 1.0)
            fail(GS_EINVAL, "prune: threshold must be in (0, 1)");
        M->ctx->use();
        *removed = 0;
        const int n = static_cast<int>(M->n);
        if (n == 0) return;
        gs_context* C = M->ctx;
        cudaStream_t st = C->stream;
        DevBuf &keep = C->sc(kScPruneKeep), &pos = C->sc(kScPrunePos);
        keep.ensure(sizeof(int32_t) * (n + 1));
        pos.ensure(sizeof(int32_t) * (n + 1));
        ck(cudaMemsetAsync(keep.as<int32_t>() + n, 0, sizeof(int32_t), st), "memset");
        launch_prune_flags(M->params, M->cap, n, opacity_threshold, keep.as<int32_t>(), st);
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, keep.as<int32_t>(), pos.as<int32_t>(), n + 1, st);
        ck(cub::DeviceScan::ExclusiveSum(C->cub(tb), tb, keep.as<int32_t>(), pos.as<int32_t>(), n + 1, st), "scan");
        int32_t kept = 0;
        ck(cudaMemcpyAsync(&kept, pos.as<int32_t>() + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "d2h");
        ck(cudaStreamSynchronize(st), "sync");
        C->launched(2);
        if (kept == n) return;
        // stable compaction through a staging block of kChunk planes (context scratch, reused):
        // compact a block of planes into it, copy the kept prefix back; no map-sized allocation.
        // Entries past `kept` are don't-care (append / init reset every range they fill).
        constexpr int kChunk = 16;
        const int64_t cap = M->cap;
        DevBuf& tmp = C->sc(kScPruneTmp);
        tmp.ensure(sizeof(float) * kChunk * cap);
        const int32_t* kp = keep.as<int32_t>();
        const int32_t* ps = pos.as<int32_t>();
        for (float* arr : {M->params, M->m, M->v}) {
            for (int c0 = 0; c0 < kNumParams; c0 += kChunk) {
                const int np = std::min(kChunk, kNumParams - c0);
                launch_compact(arr + c0 * cap, tmp.as<float>(), cap, cap, np, n, kp, ps, st);
                ck(cudaMemcpy2DAsync(arr + c0 * cap, sizeof(float) * cap, tmp.p, sizeof(float) * cap,
                                     sizeof(float) * kept, np, cudaMemcpyDeviceToDevice, st), "copy back");
                C->launched();
            }
        }
        launch_compact(M->birth, tmp.as<int32_t>(), n, kp, ps, st);
        ck(cudaMemcpyAsync(M->birth, tmp.p, sizeof(int32_t) * kept, cudaMemcpyDeviceToDevice, st), "copy back");
        launch_compact(M->degree, reinterpret_cast<int8_t*>(tmp.p), n, kp, ps, st);
        ck(cudaMemcpyAsync(M->degree, tmp.p, kept, cudaMemcpyDeviceToDevice, st), "copy back");
        C->launched(2);
        M->deg_host.resize(kept);
        ck(cudaMemcpyAsync(M->deg_host.data(), M->degree, kept, cudaMemcpyDeviceToHost, st), "d2h degree");
        ck(cudaStreamSynchronize(st), "sync");
        M->recompute_max_degree();
        M->n = kept;
        *removed = n - kept;
    });
}

int gs_map_device_planes(gs_map* M, float** params, float** m, float** v, int64_t* cap) {
    return guard([&] {
        if (params) *params = M->params;
        if (m) *m = M->m;
        if (v) *v = M->v;
        if (cap) *cap = M->cap;
    });
}

// ---------------------------------------------------------------- frames
int gs_frame_create(gs_context* C, gs_frame** out) {
    return guard([&] {
        auto* F = new gs_frame();
        F->ctx = C;
        *out = F;
    });
}

int gs_frame_destroy(gs_frame* F) {
    return guard([&] {
        if (!F) return;
        F->ctx->use();
        cudaStreamSynchronize(F->ctx->stream);
        for (DevBuf* b : {&F->rec_by_gid, &F->vis_flag, &F->key_by_gid, &F->vis_gid, &F->keys_a, &F->keys_b,
                          &F->gid_sorted, &F->rec_sorted, &F->ntiles, &F->emit_off, &F->num_sel, &F->depth_sorted,
                          &F->pair_keys,
                          &F->pair_keys2, &F->pair_vals, &F->pair_vals2, &F->ranges, &F->partials, &F->rank_sums, &F->color,
                          &F->depth, &F->vis, &F->t_final, &F->n_proc, &F->n_contrib, &F->dl_dcolor, &F->depth_cot,
                          &F->wbuf, &F->host_stage, &F->loss, &F->checkpoints, &F->seg_scratch})
            b->release();
        delete F;
    });
}

int gs_render(gs_map* M, const gs_pose* pose, const gs_camera* cam, gs_frame* F) {
    return guard([&] { render_checked(M, *pose, *cam, F); });
}

int gs_frame_stats_get(gs_frame* F, gs_frame_stats* out) {
    return guard([&] {
        need_counts(F);
        out->n_visible = F->n_vis;
        out->n_pairs = F->n_pairs;
        out->tiles_x = F->view.tiles_x;
        out->tiles_y = F->view.tiles_y;
        out->width = F->view.width;
        out->height = F->view.height;
        const size_t P = static_cast<size_t>(F->view.width) * F->view.height;
        std::vector<int32_t> nc(P);
        ck(cudaMemcpyAsync(nc.data(), F->n_contrib.p, sizeof(int32_t) * P, cudaMemcpyDeviceToHost, F->ctx->stream), "d2h");
        ck(cudaStreamSynchronize(F->ctx->stream), "sync");
        int64_t s = 0;
        for (int32_t x : nc) s += x;
        out->n_contrib = s;
    });
}

int gs_frame_read(gs_frame* F, double* color, double* depth, double* vis) {
    return guard([&] {
        need_rendered(F);
        F->ctx->use();
        const int h = F->view.height, w = F->view.width;
        const size_t P = static_cast<size_t>(h) * w;
        F->host_stage.ensure(sizeof(double) * 5 * P);
        double* stage = F->host_stage.as<double>();
        cudaStream_t st = F->ctx->stream;
        launch_to_hwc_double(F->color.as<float>(), h, w, 3, stage, st);
        launch_to_hwc_double(F->depth.as<float>(), h, w, 1, stage + 3 * P, st);
        launch_to_hwc_double(F->vis.as<float>(), h, w, 1, stage + 4 * P, st);
        F->ctx->launched(3);
        if (color) ck(cudaMemcpyAsync(color, stage, sizeof(double) * 3 * P, cudaMemcpyDeviceToHost, st), "d2h");
        if (depth) ck(cudaMemcpyAsync(depth, stage + 3 * P, sizeof(double) * P, cudaMemcpyDeviceToHost, st), "d2h");
        if (vis) ck(cudaMemcpyAsync(vis, stage + 4 * P, sizeof(double) * P, cudaMemcpyDeviceToHost, st), "d2h");
        ck(cudaStreamSynchronize(st), "sync");
    });
}

int gs_frame_device_images(gs_frame* F, float** color, float** depth, float** vis) {
    return guard([&] {
        need_rendered(F);
        if (color) *color = F->color.as<float>();
        if (depth) *depth = F->depth.as<float>();
        if (vis) *vis = F->vis.as<float>();
    });
}

int gs_frame_read_pixel_state(gs_frame* F, int32_t* n_contrib, float* t_final) {
    return guard([&] {
        need_rendered(F);
        const size_t P = static_cast<size_t>(F->view.width) * F->view.height;
        cudaStream_t st = F->ctx->stream;
        if (n_contrib) ck(cudaMemcpyAsync(n_contrib, F->n_contrib.p, sizeof(int32_t) * P, cudaMemcpyDeviceToHost, st), "d2h");
        if (t_final) ck(cudaMemcpyAsync(t_final, F->t_final.p, sizeof(float) * P, cudaMemcpyDeviceToHost, st), "d2h");
        ck(cudaStreamSynchronize(st), "sync");
    });
}

int gs_frame_read_projected(gs_frame* F, int32_t* index, double* mean2, int32_t* rect4, float* conic3,
                            float* opacity, float* color3, double* depth) {
    return guard([&] {
        need_counts(F);
        const int64_t nv = F->n_vis;
        if (nv == 0) return;
        std::vector<Splat> rec(nv);
        std::vector<unsigned long long> keys(nv);
        cudaStream_t st = F->ctx->stream;
        ck(cudaMemcpyAsync(rec.data(), F->rec_sorted.p, sizeof(Splat) * nv, cudaMemcpyDeviceToHost, st), "d2h");
        ck(cudaMemcpyAsync(keys.data(), F->depth_sorted.p, sizeof(unsigned long long) * nv, cudaMemcpyDeviceToHost, st),
           "d2h");
        ck(cudaStreamSynchronize(st), "sync");
        for (int64_t r = 0; r < nv; ++r) {
            const Splat& s = rec[r];
            if (index) index[r] = s.gid;
            if (mean2) { mean2[2 * r] = s.mx; mean2[2 * r + 1] = s.my; }
            if (rect4) {
                rect4[4 * r] = s.x0; rect4[4 * r + 1] = s.y0; rect4[4 * r + 2] = s.x1; rect4[4 * r + 3] = s.y1;
            }
            if (conic3) { conic3[3 * r] = s.ca; conic3[3 * r + 1] = s.cb; conic3[3 * r + 2] = s.cc; }
            if (opacity) opacity[r] = s.opacity;
            if (color3) { color3[3 * r] = s.r; color3[3 * r + 1] = s.g; color3[3 * r + 2] = s.b; }
            if (depth) {
                double d;
                std::memcpy(&d, &keys[r], sizeof(double));
                depth[r] = d;
            }
        }
    });
}

int gs_frame_read_tiles(gs_frame* F, int64_t* tile_offsets, int32_t* entries) {
    return guard([&] {
        need_counts(F);
        const int T = F->view.tiles_x * F->view.tiles_y;
        const int64_t K = F->n_pairs;
        std::vector<uint2> ranges(T);
        std::vector<uint32_t> vals(K);
        std::vector<Splat> rec(F->n_vis);
        cudaStream_t st = F->ctx->stream;
        ck(cudaMemcpyAsync(ranges.data(), F->ranges.p, sizeof(uint2) * T, cudaMemcpyDeviceToHost, st), "d2h");
        if (K) ck(cudaMemcpyAsync(vals.data(), F->pair_vals2.p, sizeof(uint32_t) * K, cudaMemcpyDeviceToHost, st), "d2h");
        if (F->n_vis)
            ck(cudaMemcpyAsync(rec.data(), F->rec_sorted.p, sizeof(Splat) * F->n_vis, cudaMemcpyDeviceToHost, st), "d2h");
        ck(cudaStreamSynchronize(st), "sync");
        int64_t k = 0;
        tile_offsets[0] = 0;
        for (int t = 0; t < T; ++t) {
            for (uint32_t i = ranges[t].x; i < ranges[t].y; ++i) entries[k++] = rec[vals[i]].gid;
            tile_offsets[t + 1] = k;
        }
        if (k != K) fail(GS_ELOGIC, "read_tiles: tile ranges do not cover every pair");
    });
}

int gs_frame_materialize(gs_frame* F, uint32_t* offsets, int32_t* gaussian, double* alpha) {
    return guard([&] {
        need_counts(F);
        const int h = F->view.height, w = F->view.width;
        const size_t P = static_cast<size_t>(h) * w;
        std::vector<int32_t> nc(P);
        cudaStream_t st = F->ctx->stream;
        ck(cudaMemcpyAsync(nc.data(), F->n_contrib.p, sizeof(int32_t) * P, cudaMemcpyDeviceToHost, st), "d2h");
        ck(cudaStreamSynchronize(st), "sync");
        std::vector<uint32_t> off(P + 1, 0);
        for (size_t p = 0; p < P; ++p) off[p + 1] = off[p] + static_cast<uint32_t>(nc[p]);
        if (offsets) std::memcpy(offsets, off.data(), sizeof(uint32_t) * (P + 1));
        const uint32_t total = off[P];
        if (total == 0 || (!gaussian && !alpha)) return;
        DevBuf doff, dg, da;
        doff.ensure(sizeof(uint32_t) * (P + 1));
        dg.ensure(sizeof(int32_t) * total);
        da.ensure(sizeof(double) * total);
        ck(cudaMemcpyAsync(doff.p, off.data(), sizeof(uint32_t) * (P + 1), cudaMemcpyHostToDevice, st), "h2d");
        launch_materialize(F->ranges.as<uint2>(), F->pair_vals2.as<uint32_t>(), F->rec_sorted.as<Splat>(), F->view,
                           doff.as<uint32_t>(), dg.as<int32_t>(), da.as<double>(), st);
        F->ctx->launched();
        if (gaussian) ck(cudaMemcpyAsync(gaussian, dg.p, sizeof(int32_t) * total, cudaMemcpyDeviceToHost, st), "d2h");
        if (alpha) ck(cudaMemcpyAsync(alpha, da.p, sizeof(double) * total, cudaMemcpyDeviceToHost, st), "d2h");
        ck(cudaStreamSynchronize(st), "sync");
        doff.release();
        dg.release();
        da.release();
    });
}

// ---------------------------------------------------------------- gradients
int gs_grads_create(gs_context* C, gs_grads** out) {
    return guard([&] {
        auto* G = new gs_grads();
        G->ctx = C;
        *out = G;
    });
}

int gs_grads_create_external(gs_context* C, float* ptr, int64_t capacity, gs_grads** out) {
    return guard([&] {
        auto* G = new gs_grads();
        G->ctx = C;
        G->planes = ptr;
        G->cap = capacity;
        G->external = true;
        *out = G;
    });
}

int gs_grads_destroy(gs_grads* G) {
    return guard([&] {
        if (!G) return;
        if (G->planes && !G->external) pool_free(G->planes, G->ctx->stream);
        delete G;
    });
}

int gs_grads_zero(gs_grads* G, gs_map* M) { return guard([&] { grads_zero(G, M); }); }

int gs_grads_read(gs_grads* G, double* out59, int64_t n) {
    return guard([&] {
        if (n != G->n) fail(GS_EINVAL, "grads_read: count does not match");
        if (n == 0) return;
        std::vector<float> soa(static_cast<size_t>(kNumParams) * n);
        ck(cudaMemcpy2DAsync(soa.data(), sizeof(float) * n, G->planes, sizeof(float) * G->cap, sizeof(float) * n,
                             kNumParams, cudaMemcpyDeviceToHost, G->ctx->stream), "d2h grads");
        ck(cudaStreamSynchronize(G->ctx->stream), "sync");
        for (int64_t i = 0; i < n; ++i)
            for (int k = 0; k < kNumParams; ++k) out59[i * kNumParams + k] = soa[static_cast<size_t>(k) * n + i];
    });
}

int gs_grads_write(gs_grads* G, const double* in59, int64_t n) {
    return guard([&] {
        G->ensure(std::max<int64_t>(n, 1));
        std::vector<float> soa(static_cast<size_t>(kNumParams) * n);
        for (int64_t i = 0; i < n; ++i)
            for (int k = 0; k < kNumParams; ++k) soa[static_cast<size_t>(k) * n + i] = static_cast<float>(in59[i * kNumParams + k]);
        if (n > 0)
            ck(cudaMemcpy2DAsync(G->planes, sizeof(float) * G->cap, soa.data(), sizeof(float) * n, sizeof(float) * n,
                                 kNumParams, cudaMemcpyHostToDevice, G->ctx->stream), "h2d grads");
        ck(cudaStreamSynchronize(G->ctx->stream), "sync");
        G->n = n;
        G->clean = false;
    });
}

int gs_grads_device_planes(gs_grads* G, float** planes, int64_t* cap) {
    return guard([&] {
        *planes = G->planes;
        *cap = G->cap;
    });
}

int gs_render_backward(gs_map* M, const gs_pose* pose, const gs_camera* cam, gs_frame* F, const double* dl_dcolor,
                       const double* dl_ddepth, int32_t h, int32_t w, gs_grads* G) {
    return guard([&] {
        validate_camera(*cam);
        M->ctx->use();
        (void)pose;
        if (h != cam->height || w != cam->width) fail(GS_EINVAL, "render_backward: dl_dcolor dimensions mismatch");
        need_rendered(F);
        if (F->view.width != cam->width || F->view.height != cam->height)
            fail(GS_ELOGIC, "render_backward: contributor lists missing or inconsistent");
        const size_t P = static_cast<size_t>(h) * w;
        cudaStream_t st = M->ctx->stream;
        DevBuf tmp;
        tmp.ensure(sizeof(double) * 4 * P);
        ck(cudaMemcpyAsync(tmp.p, dl_dcolor, sizeof(double) * 3 * P, cudaMemcpyHostToDevice, st), "h2d");
        ck(cudaMemcpyAsync(tmp.as<double>() + 3 * P, dl_ddepth, sizeof(double) * P, cudaMemcpyHostToDevice, st), "h2d");
        launch_from_hwc_double(tmp.as<double>(), h, w, 3, F->dl_dcolor.as<float>(), st);
        launch_from_hwc_double(tmp.as<double>() + 3 * P, h, w, 1, F->depth_cot.as<float>(), st);
        M->ctx->launched(2);
        grads_zero(G, M);
        backward_impl(M, F, F->dl_dcolor.as<float>(), F->depth_cot.as<float>(), nullptr, G);
        ck(cudaStreamSynchronize(st), "sync");
        tmp.release();
    });
}

int gs_apply_gradients(gs_map* M, gs_grads* G, const gs_learning_rates* lr) {
    return guard([&] {
        M->ctx->use();
        adam_impl(M, G, *lr);
    });
}

// ---------------------------------------------------------------- keyframes / loss / step
int gs_keyframe_create(gs_context* C, const gs_pose* pose, const double* color, const double* sparse_depth, int32_t h,
                       int32_t w, int32_t initial_iters, int32_t levels, gs_keyframe** out) {
    return guard([&] {
        C->use();
        auto* K = new gs_keyframe();
        K->ctx = C;
        K->pose = *pose;
        K->initial_iters = initial_iters;
        try {
            const size_t P = static_cast<size_t>(h) * w;
            std::vector<float> cp(3 * P), dp(P);
            for (size_t p = 0; p < P; ++p) {
                for (int c = 0; c < 3; ++c) cp[c * P + p] = static_cast<float>(color[p * 3 + c]);
                dp[p] = static_cast<float>(sparse_depth[p]);
            }
            keyframe_build(K, cp.data(), dp.data(), h, w, levels, false);
        } catch (...) {
            delete K;
            throw;
        }
        *out = K;
    });
}

int gs_keyframe_create_device(gs_context* C, const gs_pose* pose, const float* color_planes, const float* depth,
                              int32_t h, int32_t w, int32_t initial_iters, int32_t levels, gs_keyframe** out) {
    return guard([&] {
        C->use();
        auto* K = new gs_keyframe();
        K->ctx = C;
        K->pose = *pose;
        K->initial_iters = initial_iters;
        try {
            keyframe_build(K, color_planes, depth, h, w, levels, true);
        } catch (...) {
            delete K;
            throw;
        }
        *out = K;
    });
}

int gs_keyframe_destroy(gs_keyframe* K) {
    return guard([&] {
        if (!K) return;
        if (K->ctx->spec.kf == K) K->ctx->spec.valid = false;  // no stale match on a reused address
        cudaStreamSynchronize(K->ctx->stream);
        if (K->ctx->copy_stream) cudaStreamSynchronize(K->ctx->copy_stream);
        delete K;
    });
}

int gs_keyframe_consumed(gs_keyframe* K, int32_t* c) { return guard([&] { *c = K->consumed; }); }
int gs_keyframe_set_consumed(gs_keyframe* K, int32_t c) { return guard([&] { K->consumed = c; }); }
int gs_keyframe_levels(gs_keyframe* K, int32_t* n) { return guard([&] { *n = static_cast<int32_t>(K->hs.size()); }); }

void upload_level_impl(gs_keyframe* K, int32_t level, const double* color, const double* depth);

int gs_keyframe_upload_level(gs_keyframe* K, int32_t level, const double* color, const double* depth) {
    return guard([&] { upload_level_impl(K, level, color, depth); });
}

void upload_level_impl(gs_keyframe* K, int32_t level, const double* color, const double* depth) {
    {
        if (level < 0 || level >= static_cast<int>(K->hs.size())) fail(GS_EINVAL, "level out of range");
        const int h = K->hs[level], w = K->ws[level];
        const size_t P = static_cast<size_t>(h) * w;
        // asynchronous on the copy stream (host buffers must stay valid until the next
        // synchronising call on this keyframe's context): overlaps the compute stream's work
        cudaStream_t st = K->ctx->copies();
        if (K->used_valid) ck(cudaStreamWaitEvent(st, K->used, 0), "wait last use");
        K->stage.ensure(sizeof(double) * 4 * P);
        ck(cudaMemcpyAsync(K->stage.p, color, sizeof(double) * 3 * P, cudaMemcpyHostToDevice, st), "h2d color");
        ck(cudaMemcpyAsync(K->stage.as<double>() + 3 * P, depth, sizeof(double) * P, cudaMemcpyHostToDevice, st),
           "h2d depth");
        launch_from_hwc_double(K->stage.as<double>(), h, w, 3, K->color[level].as<float>(), st);
        launch_from_hwc_double(K->stage.as<double>() + 3 * P, h, w, 1, K->depth[level].as<float>(), st);
        K->ctx->launched(2);
        if (K->ready.size() < K->hs.size()) {
            K->ready.resize(K->hs.size(), nullptr);
            K->pending.resize(K->hs.size(), 0);
        }
        if (!K->ready[level]) ck(cudaEventCreateWithFlags(&K->ready[level], cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaEventRecord(K->ready[level], st), "record upload");
        K->pending[level] = 1;
    }
}

int gs_keyframe_read_level(gs_keyframe* K, int32_t level, double* color, double* depth) {
    return guard([&] {
        if (level < 0 || level >= static_cast<int>(K->hs.size())) fail(GS_EINVAL, "level out of range");
        const int h = K->hs[level], w = K->ws[level];
        const size_t P = static_cast<size_t>(h) * w;
        std::vector<float> cp(3 * P), dp(P);
        cudaStream_t st = K->ctx->stream;
        K->acquire(level, st);
        ck(cudaMemcpyAsync(cp.data(), K->color[level].p, sizeof(float) * 3 * P, cudaMemcpyDeviceToHost, st), "d2h");
        ck(cudaMemcpyAsync(dp.data(), K->depth[level].p, sizeof(float) * P, cudaMemcpyDeviceToHost, st), "d2h");
        ck(cudaStreamSynchronize(st), "sync");
        for (size_t p = 0; p < P; ++p) {
            if (color)
                for (int c = 0; c < 3; ++c) color[p * 3 + c] = cp[c * P + p];
            if (depth) depth[p] = dp[p];
        }
    });
}

int gs_compute_loss(gs_frame* F, gs_keyframe* K, int32_t level, const gs_train_config* cfg, gs_loss_result* out,
                    double* dl_dcolor, double* dl_ddepth) {
    return guard([&] {
        F->ctx->use();
        loss_impl(F, K, level, *cfg);
        if (out) *out = read_loss(F);
        const int h = F->view.height, w = F->view.width;
        const size_t P = static_cast<size_t>(h) * w;
        if (dl_dcolor || dl_ddepth) {
            cudaStream_t st = F->ctx->stream;
            std::vector<float> dc(3 * P), dd(P);
            LossScalars s;
            ck(cudaMemcpyAsync(dc.data(), F->dl_dcolor.p, sizeof(float) * 3 * P, cudaMemcpyDeviceToHost, st), "d2h");
            ck(cudaMemcpyAsync(dd.data(), F->depth_cot.p, sizeof(float) * P, cudaMemcpyDeviceToHost, st), "d2h");
            ck(cudaMemcpyAsync(&s, F->loss.p, sizeof(s), cudaMemcpyDeviceToHost, st), "d2h");
            ck(cudaStreamSynchronize(st), "sync");
            for (size_t p = 0; p < P; ++p) {
                if (dl_dcolor)
                    for (int c = 0; c < 3; ++c) dl_dcolor[p * 3 + c] = dc[c * P + p];
                if (dl_ddepth) dl_ddepth[p] = static_cast<double>(dd[p]) * s.depth_scale;
            }
        }
    });
}

int gs_render_backward_frame(gs_map* M, const gs_pose* pose, const gs_camera* cam, gs_frame* F, gs_grads* G) {
    return guard([&] {
        (void)pose;
        (void)cam;
        M->ctx->use();
        if (!F->has_cotangent) fail(GS_ELOGIC, "render_backward_frame: no cotangent (call gs_compute_loss first)");
        G->ensure(std::max<int64_t>(M->n, 1));
        if (G->n != M->n) grads_zero(G, M);
        backward_impl(M, F, F->dl_dcolor.as<float>(), F->depth_cot.as<float>(),
                      &F->loss.as<LossScalars>()->depth_scale, G);
    });
}

struct Prefetch {
    gs_keyframe* K = nullptr;
    int32_t level = 0;
    const double *color = nullptr, *depth = nullptr;
};
void train_step_impl(gs_map* M, gs_keyframe* K, const gs_train_config* cfg, const gs_camera* cam,
                     gs_step_report* report, const Prefetch* pf);

int gs_train_step(gs_map* M, gs_keyframe* K, const gs_train_config* cfg, const gs_camera* cam, gs_step_report* report) {
    return guard([&] { train_step_impl(M, K, cfg, cam, report, nullptr); });
}

int gs_train_step_prefetch(gs_map* M, gs_keyframe* K, const gs_train_config* cfg, const gs_camera* cam,
                           gs_keyframe* next_kf, int32_t next_level, const double* next_color,
                           const double* next_depth, gs_step_report* report) {
    return guard([&] {
        if (next_kf && (next_color == nullptr) != (next_depth == nullptr))
            fail(GS_EINVAL, "train_step_prefetch: pass both next images or neither");
        Prefetch pf{next_kf, next_level, next_color, next_depth};
        train_step_impl(M, K, cfg, cam, report, next_kf ? &pf : nullptr);
    });
}

bool same_camera(const gs_camera& a, const gs_camera& b) {
    return a.fx == b.fx && a.fy == b.fy && a.cx == b.cx && a.cy == b.cy && a.width == b.width && a.height == b.height;
}

void train_step_impl(gs_map* M, gs_keyframe* K, const gs_train_config* cfg, const gs_camera* cam,
                     gs_step_report* report, const Prefetch* pf) {
    {
        gs_context* C = M->ctx;
        C->use();
        *report = gs_step_report{};
        if (K->hs.empty()) fail(GS_EINVAL, "train_keyframe_step: keyframe pyramid not built");
        auto upload = [&] {
            if (pf && pf->color) upload_level_impl(pf->K, pf->level, pf->color, pf->depth);
        };
        if (K->consumed >= K->initial_iters) {  // std::nullopt (mapper.cpp:219)
            upload();
            return;
        }
        gs_grads* G = scratch_grads(C);
        const int level = schedule_level(K, *cfg);
        const gs_camera lc = scaled(*cam, level);
        // this step's render was enqueued speculatively by the previous call when it predicted
        // this (keyframe, level, camera) and the map has not changed since
        auto& sp = C->spec;
        const bool have = sp.valid && sp.map == M && sp.kf == K && sp.level == level && sp.version == M->version &&
                          same_camera(sp.cam, *cam) && std::memcmp(&sp.pose, &K->pose, sizeof(gs_pose)) == 0;
        const int fi = have ? sp.frame : C->train_parity;
        sp.valid = false;
        C->spec_used += have;
        gs_frame* F = train_frame(C, fi);
        // with a named next step, its render goes to the other frame; without one, steps stay on
        // one frame (its remembered capacities then track a growing map step by step)
        C->train_parity = pf ? fi ^ 1 : fi;
        gs_loss_result lr{};
        bool prefetched = false;
        // a level this very step reads is uploaded only after the step is final (an overflow
        // re-run must not see the next input)
        const bool late_upload = pf && pf->K == K && pf->level == level;
        // the next step's render, enqueued while this step's read-back is in flight: the host's
        // return, report and next call then overlap device work instead of idling it
        auto speculate = [&] {
            if (!pf || !pf->K || pf->K->hs.empty() || pf->level < 0 ||
                pf->level >= static_cast<int>(pf->K->hs.size()) || M->n == 0)
                return;
            const gs_camera nc = scaled(*cam, pf->level);
            gs_frame* B = train_frame(C, fi ^ 1);
            const gs_frame::Caps& cs = B->cap_slot(nc.width, nc.height);
            if (cs.pairs == 0) return;  // first render at this size needs exact counts (a sync)
            render_impl(M, pf->K->pose, nc, B, false, false);
            sp = gs_context::Speculation{true, M, pf->K, pf->level, M->version, *cam, pf->K->pose, fi ^ 1};
            ++C->spec_enqueued;
        };
        // one host round trip per step (the loss read); a step whose render overflowed the
        // remembered pair capacity changed nothing on the device and is re-run at exact size
        for (int attempt = 0;; ++attempt) {
            grads_zero(G, M);
            if (!(have && attempt == 0)) render_impl(M, K->pose, lc, F, attempt > 0, false);
            loss_impl(F, K, level, *cfg);
            backward_impl(M, F, F->dl_dcolor.as<float>(), F->depth_cot.as<float>(),
                          &F->loss.as<LossScalars>()->depth_scale, G);
            adam_impl(M, G, cfg->lr, dev_counters(F));
            // the next step's input upload is issued behind this step's enqueued work, on the
            // copy stream (it waits for this step's last read of that level buffer)
            if (!prefetched && !late_upload) {
                upload();
                prefetched = true;
            }
            if (C->defer_sync) {  // no read-back: no loss, no overflow re-run (diagnostics)
                lr.total = lr.psnr = std::nan("");
                break;
            }
            if (attempt == 0 && pf) lr = read_loss(F, speculate);
            else lr = read_loss(F);
            if (!F->overflow) break;
            sp.valid = false;  // rendered from the map before this step's (re-run) update
            --M->adam_count;
            --M->global_step;
            if (attempt > 0) fail(GS_ELOGIC, "render: pair capacity overflow after exact sizing");
        }
        if (!prefetched) upload();
        ++K->consumed;
        report->ran = 1;
        report->level = level;
        report->loss = lr.total;
        report->psnr = lr.psnr;
    }
}

int gs_train_accumulate(gs_map* M, gs_keyframe* K, const gs_train_config* cfg, const gs_camera* cam, gs_frame* F,
                        gs_grads* G, int32_t sync, gs_step_report* report) {
    return guard([&] {
        M->ctx->use();
        *report = gs_step_report{};
        if (K->hs.empty()) fail(GS_EINVAL, "train_keyframe_step: keyframe pyramid not built");
        if (K->consumed >= K->initial_iters) return;
        if (!F) F = scratch_frame(M->ctx);
        G->ensure(std::max<int64_t>(M->n, 1));
        if (G->n != M->n) grads_zero(G, M);
        int level = 0;
        // without a loss read-back (sync = 0) the pair count is read before binning instead, so
        // the accumulation can never be dropped by an overflow
        for (int attempt = 0;; ++attempt) {
            train_view(M, K, *cfg, *cam, F, G, &level, attempt > 0 || !sync);
            if (!sync) break;
            const gs_loss_result lr = read_loss(F);
            report->loss = lr.total;
            report->psnr = lr.psnr;
            if (!F->overflow) break;
            if (attempt > 0) fail(GS_ELOGIC, "render: pair capacity overflow after exact sizing");
        }
        ++K->consumed;
        report->ran = 1;
        report->level = level;
    });
}

}  // extern "C"
