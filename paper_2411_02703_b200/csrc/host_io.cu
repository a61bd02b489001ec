// On-disk formats and evaluation over the device map: checkpoint v1
// (io/checkpoint.cpp), the optimizer-state sidecar for a true resume, and one frame of
// evaluate_sequence (pipeline.cpp:34-64).
#include "host_internal.cuh"

extern "C" {

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
        need_replicated_optimizer(M, "save_training_state");
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
        need_replicated_optimizer(M, "load_training_state");
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
        F->loss.ensure(loss_buffer_bytes(h, w));
        ck(cudaMemsetAsync(F->loss.p, 0, loss_buffer_bytes(h, w), st), "memset");
        const LossLayout layout = launch_eval(F->color.as<float>(), F->depth.as<float>(), gt,
                                              gt_depth ? gt + 3 * P : nullptr, h, w, F->eval_quant.as<float>(),
                                              F->wbuf.as<float>(), F->loss.as<LossScalars>(), st);
        launch_loss_finalize(F->loss.as<LossScalars>(), layout, 0.0, st);
        C->launched(gt_depth ? 5 : 4);
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

}  // extern "C"
