// Host side of the C-ABI (include/gsmap_b200.h): the handles (context, map, frame, gradients,
// keyframe), buffer management and the orchestration of the hot step train_keyframe_step
// (mapper.cpp:214-238) over the kernels. Mapping-loop helpers: host_mapping.cu; checkpoint,
// optimizer state and evaluation: host_io.cu; shared declarations: host_internal.cuh.
#include "host_internal.cuh"

// ============================================================================ internals
namespace gsb_host {

thread_local std::string g_err;

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
    F->loss.ensure(loss_buffer_bytes(v.height, v.width));
    // tile ranges, then the blends' tile launch order (blend_common.cuh tile_order)
    F->ranges.ensure(static_cast<size_t>(v.tiles_x) * v.tiles_y * (sizeof(uint2) + sizeof(uint32_t)));
}

// every device buffer a render + loss + backward of view v needs (map size n, pair capacity
// cap): sized up front, so no allocation (cudaMalloc / cudaFree synchronise the device) happens
// inside a step once a frame has seen the resolution. The train frames reserve each other too.
namespace {
std::atomic<uint32_t> g_sort_epoch{0};
std::atomic<uint32_t> g_sort_era{0};
}  // namespace

uint32_t sort_epochs(uint32_t k) {
    for (;;) {
        uint32_t cur = g_sort_epoch.load();
        uint32_t base = cur;
        if (base + k + 1 >= (1u << 30)) base = 0;  // wrap: every status array is cleared before reuse
        if (g_sort_epoch.compare_exchange_weak(cur, base + k)) {
            if (base != cur) g_sort_era.fetch_add(1);
            return base + 1;
        }
    }
}

uint32_t sort_epoch_era() { return g_sort_era.load(); }

void reserve_frame(gs_frame* F, const ViewParams& v, int64_t n, uint32_t cap) {
    frame_pixels(F, v);
    const size_t P = static_cast<size_t>(v.width) * v.height;
    F->counters.ensure(kNumCounters * sizeof(unsigned long long));
    if (v.width >= 11 && v.height >= 11) F->wbuf.ensure(sizeof(float) * 9 * static_cast<size_t>(v.height - 10) * (v.width - 10));
    const int nseg = blend_segments(v);
    if (nseg > 1) {
        F->checkpoints.ensure(sizeof(float) * (nseg - 1) * kCkFields * P);
        F->seg_scratch.ensure(sizeof(float) * (9 * nseg + 2) * P);
    }
    if (n <= 0) return;
    F->rec_by_gid.ensure(sizeof(Splat) * n);
    F->vis_flag.ensure(sizeof(int32_t) * n);  // K1a candidate list
    F->key_by_gid.ensure(sizeof(unsigned long long) * n);
    F->vis_gid.ensure(sizeof(int32_t) * n);
    F->keys_a.ensure(sizeof(uint32_t) * n);
    F->keys_b.ensure(sizeof(uint32_t) * n);
    F->gid_sorted.ensure(sizeof(int32_t) * n);
    F->gid_tmp.ensure(sizeof(int32_t) * n);
    F->rec_sorted.ensure(sizeof(Splat) * n);
    F->depth_sorted.ensure(sizeof(unsigned long long) * n);
    F->ntiles.ensure(sizeof(uint32_t) * (n + 1));
    F->emit_off.ensure(sizeof(uint32_t) * (n + 1));
    F->sort_block.ensure(sizeof(SortBlock));
    F->rank_of.ensure(sizeof(int32_t) * n);
    F->rank_sums.ensure(sizeof(float) * kNumPartials * n);
    if (cap == 0) return;
    {
        const void* before = F->sort_status.p;
        const size_t words = sort_status_words(std::max<int64_t>(n, cap));
        F->sort_status.ensure(sizeof(unsigned long long) * words);
        if (F->sort_status.p != before || F->status_era != sort_epoch_era()) {
            // fresh (possibly recycled) memory, or the epoch counter wrapped: no stale epochs
            ck(cudaMemsetAsync(F->sort_status.p, 0, F->sort_status.bytes, F->ctx->stream), "memset sort status");
            F->status_era = sort_epoch_era();
        }
    }
    const size_t kb = v.tiles_x * v.tiles_y <= 0xffff ? sizeof(uint16_t) : sizeof(uint32_t);
    F->pair_keys.ensure(kb * cap);
    F->pair_keys2.ensure(kb * cap);
    F->pair_vals.ensure(sizeof(uint32_t) * cap);
    F->pair_vals2.ensure(sizeof(uint32_t) * cap);
    F->partials.ensure(sizeof(float) * kNumPartials * cap);
}

unsigned long long* dev_counters(gs_frame* F) { return F->counters.as<unsigned long long>(); }

void take_counts(gs_frame* F, const unsigned long long* cnt) {
    F->n_vis = static_cast<int64_t>(cnt[kCntVisible]);
    F->n_pairs = static_cast<int64_t>(cnt[kCntPairs]);
    F->overflow = cnt[kCntOverflow] != 0;
    F->counts_known = true;
    if (F->n_pairs > 0xffffffffLL) fail(GS_ELOGIC, "render: more than 2^32 (tile, gaussian) pairs");
    // keep the resolution's pair capacity >= 4/3 of the latest count (a growing map then never
    // overflows a render: the buffers grow before they are needed)
    if (F->rendered) {
        gs_frame::Caps& cs = F->cap_slot(F->view.width, F->view.height);
        if (cs.pairs > 0 && 4 * F->n_pairs > 3 * static_cast<int64_t>(cs.pairs)) {
            cs.pairs = std::max(cs.pairs, grown_cap(F->n_pairs));
            ++F->ctx->cap_growths;
        }
    }
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
    const int64_t c = (2 * pairs + 65536 + 63) / 64 * 64;  // multiple of 64 (vector loads)
    return static_cast<uint32_t>(std::min<int64_t>(c, 0xffffffc0LL));
}

// render (rasterizer.cpp:100-199) without the CSR: project -> compact -> depth sort -> pack ->
// scan -> emit (tile, rank) pairs -> stable tile sort -> ranges -> blend. Nothing here waits
// for the device: the sorts and scans run at capacity (the map size for ranks, the
// resolution's pair capacity for pairs) with sentinel keys past the device counts. With
// exact_counts (or an unknown capacity) the pair count is read back first and the capacity
// grown to fit, so the render cannot overflow.
void render_impl(gs_map* M, const gs_pose& pose, const gs_camera& cam, gs_frame* F, bool exact_counts,
                 bool stats) {
    validate_camera(cam);
    gs_context* C = M->ctx;
    C->use();
    cudaStream_t st = C->stream;
    const ViewParams v = make_view(pose, cam);
    F->view = v;
    F->map_n = M->n;
    F->rendered = false;
    F->has_cotangent = false;
    const int n = static_cast<int>(M->n);
    const int T = v.tiles_x * v.tiles_y;
    reserve_frame(F, v, 0, 0);
    F->counters.ensure(kNumCounters * sizeof(unsigned long long));
    F->n_vis = 0;
    F->n_pairs = 0;
    F->overflow = false;
    F->counts_known = n == 0;
    F->pair_cap = 0;
    F->vis_cap = 0;
    unsigned long long* cnt = dev_counters(F);
    if (n > 0) reserve_frame(F, v, n, 0);
    launch_frame_init(F->ranges.as<uint2>(), T, cnt, n > 0 ? F->sort_block.as<SortBlock>() : nullptr, st);
    C->launched();
    if (n > 0) {
        {
            Scope sc(C, "preprocess_fwd");
            launch_cull(M->params, M->cap, n, v, F->vis_flag.as<int32_t>(), cnt, st);
            launch_preprocess_fwd(M->params, M->cap, M->degree, F->vis_flag.as<int32_t>(), n, v,
                                  F->rec_by_gid.as<Splat>(), F->key_by_gid.as<unsigned long long>(),
                                  F->vis_gid.as<int32_t>(), F->keys_a.as<uint32_t>(), cnt, st);
            C->launched(2);
        }
        // the pair capacity of this resolution: learned from the first render's exact count,
        // kept at >= 4/3 of the last count seen (take_counts); the sorts cost what the device
        // count says, not what the buffers hold
        gs_frame::Caps& cs = F->cap_slot(v.width, v.height);
        if (cs.pairs == 0 || exact_counts) {
            ++C->count_syncs;
            ensure_counts(F);
            cs.pairs = std::max(cs.pairs, grown_cap(F->n_pairs));
        }
        const uint32_t cap = cs.pairs;
        F->pair_cap = cap;
        F->vis_cap = n;
        reserve_frame(F, v, n, cap);
        if (F->sibling) reserve_frame(F->sibling, v, n, cap);
        SortBlock* sb = F->sort_block.as<SortBlock>();
        unsigned long long* status = F->sort_status.as<unsigned long long>();
        {
            // (depth, index) order (rasterizer.cpp:69-72): radix sort on the 24-bit depth key,
            // then exact (fp64 depth, index) order inside runs of equal keys; rank-ordered
            // records and the scan of their tile counts
            Scope sc_sort(C, "depth_sort_pack_scan");
            launch_depth_sort(F->keys_a.as<uint32_t>(), F->keys_b.as<uint32_t>(), F->vis_gid.as<int32_t>(),
                              F->gid_tmp.as<int32_t>(), F->gid_sorted.as<int32_t>(),
                              F->key_by_gid.as<unsigned long long>(), cnt, n, sb, status, C->epochs(3), st);
            launch_pack_scan(F->gid_sorted.as<int32_t>(), F->rec_by_gid.as<Splat>(),
                             F->key_by_gid.as<unsigned long long>(), cnt, n, F->rec_sorted.as<Splat>(),
                             F->depth_sorted.as<unsigned long long>(), F->rank_of.as<int32_t>(), F->emit_off.as<uint32_t>(), sb, status,
                             C->epochs(1), st);
            C->launched(6);
        }
        {
            Scope sc_keys(C, "tile_keys_sort_ranges");
            C->launched(launch_tile_sort(F->emit_off.as<uint32_t>(), F->rec_sorted.as<Splat>(), cnt, n, cap, v.tiles_x,
                                         T, F->pair_keys.p, F->pair_keys2.p, F->pair_vals.as<uint32_t>(),
                                         F->pair_vals2.as<uint32_t>(), F->ranges.as<uint2>(), sb, status,
                                         C->epochs(2), st));
        }
    }
    {
        Scope sc(C, "blend_fwd");
        F->nseg = blend_segments(v);
        const size_t P = static_cast<size_t>(v.width) * v.height;
        if (F->nseg > 1) {  // (reserve_frame sized them)
            F->checkpoints.ensure(sizeof(float) * (F->nseg - 1) * kCkFields * P);
            F->seg_scratch.ensure(sizeof(float) * (9 * F->nseg + 2) * P);
        }
        const int k = launch_blend_fwd(F->ranges.as<uint2>(), n > 0 ? F->pair_vals2.as<uint32_t>() : nullptr,
                         n > 0 ? F->rec_sorted.as<Splat>() : nullptr, v, F->color.as<float>(),
                         F->depth.as<float>(), F->vis.as<float>(), F->t_final.as<float>(),
                         F->n_proc.as<int32_t>(), F->n_contrib.as<int32_t>(), stats, F->checkpoints.as<float>(),
                         F->nseg, n > 0 && F->nseg > 1 ? F->seg_scratch.as<float>() : nullptr, dev_counters(F), st);
        C->launched(k);
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

// grads_zero for a training step: the memset runs on the context's aux stream from the point the
// compute stream has reached (every earlier read of the planes is done), overlapping the render;
// the compute stream waits for it right before the backward (join_grads_zero)
void grads_zero_async(gs_grads* G, gs_map* M) {
#if defined(GSB_SYNC_GRADS_ZERO)
    grads_zero(G, M);
    return;
#endif
    G->ensure(std::max<int64_t>(M->n, 1));
    gs_context* C = M->ctx;
    if (M->n > 0) {
        cudaStream_t ax = C->aux();
        ck(cudaEventRecord(C->aux_in, C->stream), "event record");
        ck(cudaStreamWaitEvent(ax, C->aux_in, 0), "stream wait");
        const int planes = n_active_planes(M->max_degree);
        ck(cudaMemset2DAsync(G->planes, sizeof(float) * G->cap, 0, sizeof(float) * M->n, planes, ax), "memset grads");
        ck(cudaEventRecord(C->aux_out, ax), "event record");
    }
    G->n = M->n;
    G->clean = true;
}

void join_grads_zero(gs_context* C) {
    if (C->aux_stream) ck(cudaStreamWaitEvent(C->stream, C->aux_out, 0), "stream wait");
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
        launch_preprocess_bwd(M->params, M->cap, M->degree, F->view, F->emit_off.as<uint32_t>(),
                              F->partials.as<float>(), F->rank_sums.as<float>(), dev_counters(F), F->vis_cap,
                              G->planes, G->cap, !G->clean, F->rank_of.as<int32_t>(), F->vis_gid.as<int32_t>(), st);
        G->clean = false;
        C->launched(2);  // K8a reduce, K8b VJP
    }
}

// counters: the frame whose gradients these are (the update is skipped if it overflowed)
void adam_impl(gs_map* M, gs_grads* G, const gs_learning_rates& lr, const unsigned long long* counters) {
    if (G->n != M->n) fail(GS_EINVAL, "apply_gradients: gradient count does not match map size");
    need_replicated_optimizer(M, "apply_gradients");
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
    // (no zeroing of the loss buffer: every slot the finalize reads is written by this call's
    // kernels, and the finalize writes every header field)
    Scope sc(C, "loss_l1_ssim_depth");
    LossLayout layout{};
    if (cfg.lambda != 0.0) {
        if (h < 11 || w < 11) fail(GS_EINVAL, "ssim: image smaller than the 11x11 window");
        F->wbuf.ensure(sizeof(float) * 9 * static_cast<size_t>(h - 10) * (w - 10));
        // SSIM forward, then its adjoint fused with the per-pixel L1 / psnr / depth terms
        layout = launch_ssim(F->color.as<float>(), K->color[level].as<float>(), h, w, cfg.lambda, F->wbuf.as<float>(),
                    F->dl_dcolor.as<float>(), F->loss.as<LossScalars>(), F->depth.as<float>(), F->vis.as<float>(),
                    K->depth[level].as<float>(), F->depth_cot.as<float>(), st);
        C->launched(2);
    } else {
        layout = launch_loss_pixel(F->color.as<float>(), F->depth.as<float>(), F->vis.as<float>(), K->color[level].as<float>(),
                          K->depth[level].as<float>(), h, w, cfg.lambda, F->dl_dcolor.as<float>(),
                          F->depth_cot.as<float>(), F->loss.as<LossScalars>(), st);
        C->launched();
    }
    launch_loss_finalize(F->loss.as<LossScalars>(), layout, cfg.lambda_d, st);
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
gs_loss_result read_loss(gs_frame* F, const std::function<void()>& between) {
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
        for (DevBuf& b : *v) b.pool = &K->ctx->stream;
    K->stage.pool = &K->ctx->stream;
    // host-upload staging at the level-0 size once: an upload of any level then never grows it
    // (a growth would free a buffer an in-flight copy-stream upload may still be writing)
    if (!device_src) K->stage.ensure(sizeof(double) * 4 * static_cast<size_t>(h) * w);
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
    if (!C->train_frames[0]) {
        for (gs_frame*& f : C->train_frames) {
            f = new gs_frame();
            f->ctx = C;
        }
        C->train_frames[1]->shared_caps = &C->train_frames[0]->caps;
        C->train_frames[0]->sibling = C->train_frames[1];
        C->train_frames[1]->sibling = C->train_frames[0];
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

// host upload of one pyramid level on the copy stream (gs_keyframe_upload_level, and the
// prefetch of gs_train_step_prefetch)
void upload_level_impl(gs_keyframe* K, int32_t level, const double* color, const double* depth) {
    {
        if (level < 0 || level >= static_cast<int>(K->hs.size())) fail(GS_EINVAL, "level out of range");
        const int h = K->hs[level], w = K->ws[level];
        const size_t P = static_cast<size_t>(h) * w;
        // asynchronous on the copy stream (host buffers must stay valid until the next
        // synchronising call on this keyframe's context): overlaps the compute stream's work
        cudaStream_t st = K->ctx->copies();
        if (K->used_valid) ck(cudaStreamWaitEvent(st, K->used, 0), "wait last use");
        if (K->stage.bytes < sizeof(double) * 4 * P) {
            // first host upload of a device-built keyframe: size the stage for level 0 with no
            // copy-stream work in flight on the old buffer
            ck(cudaStreamSynchronize(st), "sync copy stream");
            K->stage.ensure(sizeof(double) * 4 * static_cast<size_t>(K->hs[0]) * K->ws[0]);
        }
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

// the step after this one, named by gs_train_step_prefetch
struct Prefetch {
    gs_keyframe* K = nullptr;
    int32_t level = 0;
    const double *color = nullptr, *depth = nullptr;
};

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
            C->prof_level = pf->level;
            render_impl(M, pf->K->pose, nc, B, false, false);
            C->prof_level = level;
            sp = gs_context::Speculation{true, M, pf->K, pf->level, M->version, *cam, pf->K->pose, fi ^ 1};
            ++C->spec_enqueued;
        };
        // one host round trip per step (the loss read); a step whose render overflowed the
        // remembered pair capacity changed nothing on the device and is re-run at exact size
        for (int attempt = 0;; ++attempt) {
            grads_zero_async(G, M);
            C->prof_level = level;
            if (!(have && attempt == 0)) render_impl(M, K->pose, lc, F, attempt > 0, false);
            loss_impl(F, K, level, *cfg);
            join_grads_zero(C);
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
            ++C->overflow_reruns;
            --M->adam_count;
            --M->global_step;
            if (attempt > 0) fail(GS_ELOGIC, "render: pair capacity overflow after exact sizing");
        }
        C->prof_level = -1;
        if (!prefetched) upload();
        ++K->consumed;
        report->ran = 1;
        report->level = level;
        report->loss = lr.total;
        report->psnr = lr.psnr;
    }
}

}  // namespace gsb_host

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
            for (DevBuf& b : C->scratch) b.pool = &C->stream;
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
        for (gs_frame* F : {C->scratch_frame, C->train_frames[0], C->train_frames[1]}) {
            if (F) F->release_all();
            delete F;
        }
        if (C->loss_ready) cudaEventDestroy(C->loss_ready);
        if (C->aux_stream) {
            cudaStreamSynchronize(C->aux_stream);
            cudaStreamDestroy(C->aux_stream);
            cudaEventDestroy(C->aux_in);
            cudaEventDestroy(C->aux_out);
        }
        for (cudaEvent_t e : C->ev_pool) cudaEventDestroy(e);
        if (C->scratch_grads && C->scratch_grads->planes && !C->scratch_grads->external)
            pool_free(C->scratch_grads->planes, C->stream);
        delete C->scratch_grads;
        if (C->copy_stream) {
            cudaStreamSynchronize(C->copy_stream);
            cudaStreamDestroy(C->copy_stream);
        }
        C->cub_tmp.release();
        C->batch_stats.release();
        C->shard_grads.release();
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
        C->use();
        // nothing may still run on the old stream: its pooled buffers are re-pointed (they hold
        // &C->stream) and the stream itself may be destroyed
        if (C->copy_stream) ck(cudaStreamSynchronize(C->copy_stream), "sync copy stream");
        ck(cudaStreamSynchronize(C->stream), "sync");
        C->spec.valid = false;
        if (C->own_stream) cudaStreamDestroy(C->stream);
        if (stream) {
            C->stream = static_cast<cudaStream_t>(stream);
            C->own_stream = false;
        } else {
            ck(cudaStreamCreateWithFlags(&C->stream, cudaStreamNonBlocking), "cudaStreamCreate");
            C->own_stream = true;
        }
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
            // scopes enqueued by a train step carry its pyramid level: "name@L<level>"
            const std::string key = r.level >= 0 ? std::string(r.name) + "@L" + std::to_string(r.level) : r.name;
            size_t k = 0;
            while (k < keys.size() && keys[k] != key) ++k;
            if (k == keys.size()) {
                keys.emplace_back(key);
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
        need_replicated_optimizer(M, "append");
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
        need_replicated_optimizer(M, "get_adam");
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
        need_replicated_optimizer(M, "set_adam");
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

// diagnostics: K8b thread order (0 rank, 1 map, 2 visible list; -1 = automatic)
// diagnostics: speculative next-step renders enqueued / used so far on this context
int gs_debug_speculation(gs_context* C, int64_t* out2) {
    return guard([&] {
        out2[0] = C->spec_enqueued;
        out2[1] = C->spec_used;
    });
}

int gs_debug_capacity(gs_context* C, int64_t* out3) {
    return guard([&] {
        out3[0] = C->cap_growths;
        out3[1] = C->overflow_reruns;
        out3[2] = C->count_syncs;
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
        F->release_all();
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

// A RenderOutput that did not come from a device render (compute_loss takes any images,
// mapper.hpp:61-62): host fp64 HWC images into the frame's planes. The frame then has images
// but no contributor lists, so render_backward on it fails like the reference's CSR check.
int gs_frame_set_images(gs_frame* F, const double* color, const double* depth, const double* vis, int32_t h,
                        int32_t w) {
    return guard([&] {
        if (h <= 0 || w <= 0) fail(GS_EINVAL, "frame_set_images: image size must be positive");
        if (!color || !depth || !vis) fail(GS_EINVAL, "frame_set_images: null image");
        F->ctx->use();
        ViewParams v{};
        v.width = w;
        v.height = h;
        v.tiles_x = div_up(w, kTile);
        v.tiles_y = div_up(h, kTile);
        frame_pixels(F, v);
        const size_t P = static_cast<size_t>(h) * w;
        cudaStream_t st = F->ctx->stream;
        DevBuf tmp;
        tmp.ensure(sizeof(double) * 5 * P);
        ck(cudaMemcpyAsync(tmp.p, color, sizeof(double) * 3 * P, cudaMemcpyHostToDevice, st), "h2d");
        ck(cudaMemcpyAsync(tmp.as<double>() + 3 * P, depth, sizeof(double) * P, cudaMemcpyHostToDevice, st), "h2d");
        ck(cudaMemcpyAsync(tmp.as<double>() + 4 * P, vis, sizeof(double) * P, cudaMemcpyHostToDevice, st), "h2d");
        launch_from_hwc_double(tmp.as<double>(), h, w, 3, F->color.as<float>(), st);
        launch_from_hwc_double(tmp.as<double>() + 3 * P, h, w, 1, F->depth.as<float>(), st);
        launch_from_hwc_double(tmp.as<double>() + 4 * P, h, w, 1, F->vis.as<float>(), st);
        F->ctx->launched(3);
        ck(cudaStreamSynchronize(st), "sync");
        tmp.release();
        F->view = v;
        F->rendered = true;
        F->has_cotangent = false;
        F->has_contrib = false;
        F->map_n = -1;  // no lists: render_backward refuses this frame
        F->n_vis = F->n_pairs = 0;
        F->counts_known = true;
        F->overflow = false;
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

int gs_keyframe_upload_level(gs_keyframe* K, int32_t level, const double* color, const double* depth) {
    return guard([&] { upload_level_impl(K, level, color, depth); });
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
