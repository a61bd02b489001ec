// Keyframe-batch training over NCCL, callable from the C++ mapping
// thread through the C-ABI: gs_train_batch renders this rank's views, sums their gradients on
// the device (GaussianGrad::add, gaussian.hpp:51-57), reduces them over the ranks and applies ONE
// Adam step (GaussianMap::apply_gradients, gaussian_map.cpp:37-54).
//
//   mode 0 (replicated): ncclAllReduce of the S_p = 11 + 3(d+1)^2 active gradient planes (a
//          contiguous prefix of the [59][cap] plane layout), then the same Adam step on every
//          rank's replica: the replicas stay bit-identical.
//   mode 1 (sharded, the choice at SH degree >= 1): ncclReduceScatter of every active plane by
//          Gaussian range, Adam on the rank's own range only (1/R of the optimizer's HBM
//          traffic), ncclAllGather of the updated parameter planes. Adam m / v stay sharded (each
//          rank holds its range's state); gs_comm_gather_optimizer_state re-replicates them, and
//          every call that reads or re-lays out the optimizer state refuses a sharded map.
//
// NCCL is bound at run time (dlopen of libnccl.so.2): a process that already loaded torch's NCCL
// shares it, and the library itself has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "host_internal.cuh"

namespace {

struct NcclApi {
    void* handle = nullptr;
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclCommCount) comm_count = nullptr;
    decltype(&ncclCommUserRank) comm_user_rank = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclReduceScatter) reduce_scatter = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string why;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            api.handle = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (api.handle) break;
        }
        if (!api.handle) {
            why = std::string("NCCL unavailable: ") + dlerror();
            return;
        }
        auto sym = [&](auto& fn, const char* s) { fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(api.handle, s)); };
        sym(api.get_unique_id, "ncclGetUniqueId");
        sym(api.comm_init_rank, "ncclCommInitRank");
        sym(api.comm_destroy, "ncclCommDestroy");
        sym(api.comm_count, "ncclCommCount");
        sym(api.comm_user_rank, "ncclCommUserRank");
        sym(api.all_reduce, "ncclAllReduce");
        sym(api.reduce_scatter, "ncclReduceScatter");
        sym(api.all_gather, "ncclAllGather");
        sym(api.group_start, "ncclGroupStart");
        sym(api.group_end, "ncclGroupEnd");
        sym(api.error_string, "ncclGetErrorString");
        if (!api.get_unique_id || !api.comm_init_rank || !api.all_reduce || !api.reduce_scatter || !api.all_gather ||
            !api.group_start || !api.group_end) {
            why = "NCCL: missing entry points in libnccl.so.2";
            api.handle = nullptr;
        }
    });
    if (!api.handle) fail(GS_ENCCL, why);
    return api;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        fail(GS_ENCCL, std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "NCCL error"));
}

}  // namespace

struct gs_comm {
    gs_context* ctx = nullptr;
    ncclComm_t comm = nullptr;
    bool owned = false;
    int nranks = 1, rank = 0;
};

namespace gsb_host {

void need_replicated_optimizer(const gs_map* M, const char* what) {
    if (M->opt_shard_chunk > 0)
        fail(GS_ELOGIC, std::string(what) + ": the optimizer state is sharded over ranks "
                                            "(call gs_comm_gather_optimizer_state first)");
}

}  // namespace gsb_host

namespace {

int64_t shard_chunk(int64_t n, int nranks) {
    const int64_t per = (n + nranks - 1) / nranks;
    return std::max<int64_t>(64, (per + 63) / 64 * 64);  // 16-byte aligned plane slices
}

// all-gather every plane of an optimizer array from its owners (in place)
void gather_planes(gs_comm* K, float* base, int64_t cap, int planes, int64_t chunk) {
    const NcclApi& A = nccl();
    cudaStream_t st = K->ctx->stream;
    nck(A.group_start(), "ncclGroupStart");
    for (int p = 0; p < planes; ++p) {
        float* plane = base + static_cast<int64_t>(p) * cap;
        nck(A.all_gather(plane + K->rank * chunk, plane, static_cast<size_t>(chunk), ncclFloat, K->comm, st),
            "ncclAllGather");
    }
    nck(A.group_end(), "ncclGroupEnd");
}

void gather_optimizer(gs_map* M, gs_comm* K) {
    if (M->opt_shard_chunk <= 0) return;
    if (!K || K->nranks != M->opt_shard_ranks)
        fail(GS_EINVAL, "gather_optimizer_state: communicator does not match the sharded state");
    gather_planes(K, M->m, M->cap, kNumParams, M->opt_shard_chunk);
    gather_planes(K, M->v, M->cap, kNumParams, M->opt_shard_chunk);
    M->opt_shard_chunk = 0;
    M->opt_shard_ranks = 0;
}

}  // namespace

extern "C" {

int gs_comm_unique_id(uint8_t* id128) {
    return guard([&] {
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
        ncclUniqueId id;
        nck(nccl().get_unique_id(&id), "ncclGetUniqueId");
        std::memcpy(id128, &id, sizeof(id));
    });
}

int gs_comm_create(gs_context* C, const uint8_t* id128, int32_t nranks, int32_t rank, gs_comm** out) {
    return guard([&] {
        if (nranks < 1 || rank < 0 || rank >= nranks) fail(GS_EINVAL, "gs_comm_create: bad rank / rank count");
        C->use();
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof(id));
        auto* K = new gs_comm();
        K->ctx = C;
        try {
            nck(nccl().comm_init_rank(&K->comm, nranks, id, rank), "ncclCommInitRank");
        } catch (...) {
            delete K;
            throw;
        }
        K->owned = true;
        K->nranks = nranks;
        K->rank = rank;
        *out = K;
    });
}

int gs_comm_wrap(gs_context* C, void* nccl_comm, gs_comm** out) {
    return guard([&] {
        if (!nccl_comm) fail(GS_EINVAL, "gs_comm_wrap: null communicator");
        const NcclApi& A = nccl();
        auto* K = new gs_comm();
        K->ctx = C;
        K->comm = static_cast<ncclComm_t>(nccl_comm);
        int n = 1, r = 0;
        if (A.comm_count) nck(A.comm_count(K->comm, &n), "ncclCommCount");
        if (A.comm_user_rank) nck(A.comm_user_rank(K->comm, &r), "ncclCommUserRank");
        K->nranks = n;
        K->rank = r;
        *out = K;
    });
}

int gs_comm_destroy(gs_comm* K) {
    return guard([&] {
        if (!K) return;
        if (K->owned && K->comm) {
            K->ctx->use();
            cudaStreamSynchronize(K->ctx->stream);
            nccl().comm_destroy(K->comm);
        }
        delete K;
    });
}

int gs_comm_size(gs_comm* K, int32_t* nranks, int32_t* rank) {
    return guard([&] {
        *nranks = K->nranks;
        *rank = K->rank;
    });
}

int gs_comm_gather_optimizer_state(gs_map* M, gs_comm* K) {
    return guard([&] {
        M->ctx->use();
        gather_optimizer(M, K);
        ck(cudaStreamSynchronize(M->ctx->stream), "sync");
    });
}

int gs_map_optimizer_sharded(const gs_map* M, int32_t* sharded) {
    return guard([&] { *sharded = M->opt_shard_chunk > 0; });
}

int gs_train_batch(gs_map* M, gs_keyframe** kfs, int32_t n_views, const gs_train_config* cfg, const gs_camera* cam,
                   gs_comm* K, int32_t mode, gs_step_report* reports) {
    return guard([&] {
        gs_context* C = M->ctx;
        C->use();
        if (n_views < 0 || (n_views > 0 && (!kfs || !reports))) fail(GS_EINVAL, "train_batch: bad view list");
        if (mode != 0 && mode != 1) fail(GS_EINVAL, "train_batch: mode must be 0 (all-reduce) or 1 (sharded Adam)");
        if (K && K->ctx->device != C->device) fail(GS_EINVAL, "train_batch: communicator on another device");
        const int R = K ? K->nranks : 1;
        const bool sharded = mode == 1 && K;
        if (!sharded) need_replicated_optimizer(M, "train_batch");
        cudaStream_t st = C->stream;
        for (int k = 0; k < n_views; ++k) {
            reports[k] = gs_step_report{};
            if (kfs[k]->hs.empty()) fail(GS_EINVAL, "train_keyframe_step: keyframe pyramid not built");
        }
        const int64_t n = M->n;
        const int64_t chunk = sharded ? shard_chunk(n, R) : 0;
        if (sharded) {
            map_reserve(M, chunk * R);  // whole chunks per rank inside every plane
            if (M->opt_shard_chunk > 0 && (M->opt_shard_chunk != chunk || M->opt_shard_ranks != R))
                gather_optimizer(M, K);  // the ranges moved (map size changed): re-replicate first
        }
        gs_grads* G = scratch_grads(C);
        G->ensure(std::max<int64_t>({n, chunk * R, 1}));
        gs_frame* F = scratch_frame(C);
        // per-view loss scalars + counters, read back once for the whole batch
        const size_t rec = sizeof(LossScalars) + kNumCounters * sizeof(unsigned long long);
        C->batch_stats.ensure(rec * std::max(n_views, 1));
        std::vector<int> level(n_views, -1);
        std::vector<char> host(rec * std::max(n_views, 1));
        for (int attempt = 0;; ++attempt) {
            grads_zero(G, M);
            for (int k = 0; k < n_views; ++k) {
                gs_keyframe* KF = kfs[k];
                if (KF->consumed >= KF->initial_iters) continue;  // std::nullopt (mapper.cpp:219)
                train_view(M, KF, *cfg, *cam, F, G, &level[k], attempt > 0);
                char* dst = C->batch_stats.as<char>() + rec * k;
                ck(cudaMemcpyAsync(dst, F->loss.p, sizeof(LossScalars), cudaMemcpyDeviceToDevice, st), "d2d loss");
                ck(cudaMemcpyAsync(dst + sizeof(LossScalars), F->counters.p, kNumCounters * sizeof(unsigned long long),
                                   cudaMemcpyDeviceToDevice, st), "d2d counters");
            }
            if (n_views > 0)
                ck(cudaMemcpyAsync(host.data(), C->batch_stats.p, rec * n_views, cudaMemcpyDeviceToHost, st), "d2h");
            ck(cudaStreamSynchronize(st), "sync batch");
            bool overflow = false;
            for (int k = 0; k < n_views; ++k) {
                if (level[k] < 0) continue;
                const auto* cnt = reinterpret_cast<const unsigned long long*>(host.data() + rec * k + sizeof(LossScalars));
                overflow |= cnt[kCntOverflow] != 0;
            }
            if (!overflow) break;
            ++C->overflow_reruns;  // a view outgrew its pair capacity: this rank re-runs its views exactly
            if (attempt > 0) fail(GS_ELOGIC, "render: pair capacity overflow after exact sizing");
        }
        const int planes = n_active_planes(M->max_degree);
        const double l[5] = {cfg->lr.position, cfg->lr.rotation, cfg->lr.log_scale, cfg->lr.opacity, cfg->lr.sh};
        {
            Scope sc(C, "batch_reduce_adam");
            if (!sharded) {
                if (K && R > 1)
                    nck(nccl().all_reduce(G->planes, G->planes, static_cast<size_t>(planes) * G->cap, ncclFloat, ncclSum,
                                          K->comm, st), "ncclAllReduce");
                adam_impl(M, G, cfg->lr, nullptr);
            } else {
                // reduce-scatter by Gaussian range -> Adam on the own range -> all-gather the planes
                C->shard_grads.ensure(sizeof(float) * planes * chunk);
                float* sg = C->shard_grads.as<float>();
                const NcclApi& A = nccl();
                nck(A.group_start(), "ncclGroupStart");
                for (int p = 0; p < planes; ++p)
                    nck(A.reduce_scatter(G->planes + p * G->cap, sg + p * chunk, static_cast<size_t>(chunk), ncclFloat,
                                         ncclSum, K->comm, st), "ncclReduceScatter");
                nck(A.group_end(), "ncclGroupEnd");
                const int64_t first = K->rank * chunk;
                const int cnt = static_cast<int>(std::max<int64_t>(0, std::min(chunk, n - first)));
                if (cnt > 0)
                    launch_adam(M->params + first, M->m + first, M->v + first, M->birth + first, M->degree + first, sg,
                                chunk, M->cap, cnt, l, M->scene_extent, M->adam_count + 1, nullptr, M->max_degree, st);
                C->launched();
                gather_planes(K, M->params, M->cap, planes, chunk);
                ++M->adam_count;
                ++M->version;
                ++M->global_step;
                M->opt_shard_chunk = chunk;
                M->opt_shard_ranks = R;
            }
        }
        ck(cudaStreamSynchronize(st), "sync batch step");
        for (int k = 0; k < n_views; ++k) {
            if (level[k] < 0) continue;
            LossScalars s;
            std::memcpy(&s, host.data() + rec * k, sizeof(s));
            const gs_camera lc = scaled(*cam, level[k]);
            const double inv_n = 1.0 / (static_cast<double>(lc.height) * lc.width * 3);
            const double l1 = s.l1_sum * inv_n;
            const double ssim = cfg->lambda != 0.0 ? s.ssim_sum / (static_cast<double>(lc.height - 10) * (lc.width - 10) * 3) : 0.0;
            const double color = (1.0 - cfg->lambda) * l1 + (cfg->lambda != 0.0 ? cfg->lambda * (1.0 - ssim) : 0.0);
            const double depth = s.n_valid > 0 ? s.depth_abs_sum / static_cast<double>(s.n_valid) : 0.0;
            const double mse = s.sq_sum * inv_n;
            reports[k].ran = 1;
            reports[k].level = level[k];
            reports[k].loss = color + cfg->lambda_d * depth;
            reports[k].psnr = mse == 0.0 ? 100.0 : 10.0 * std::log10(1.0 / mse);
            ++kfs[k]->consumed;
        }
    });
}

}  // extern "C"
