// Mapping-loop helpers around the hot step, on the device map:
// init_gaussians_from_points (grid 3-NN), filter_points_by_visibility, the fused keyframe
// integration, prune, project_sparse_depth and the SH schedule (pipeline.cpp:130-160).
#include "host_internal.cuh"

namespace gsb_host {

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

}  // namespace gsb_host

extern "C" {

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

int gs_map_init_from_points(gs_map* M, const double* pts6, int64_t n, int64_t* added) {  // mapper.cpp:43-61
    return guard([&] {
        *added = 0;
        need_replicated_optimizer(M, "init_gaussians_from_points");
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

int gs_integrate_keyframe(gs_map* M, const gs_pose* pose, const gs_camera* cam, const double* color,
                          const double* points6, int64_t n, double tau_alpha, int32_t initial_iters, int32_t levels,
                          gs_keyframe** out_kf, int64_t* added) {
    return guard([&] {  // pipeline.cpp:148-155 (+ the keyframe's sparse depth, pipeline.cpp:108)
        need_replicated_optimizer(M, "integrate_keyframe");
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

int gs_map_prune(gs_map* M, double opacity_threshold, int64_t* removed) {  // gaussian_map.cpp:56-73
    return guard([&] {
        if (opacity_threshold <= 0.0 || opacity_threshold >= 1.0)
            fail(GS_EINVAL, "prune: threshold must be in (0, 1)");
        need_replicated_optimizer(M, "prune");
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

}  // extern "C"
