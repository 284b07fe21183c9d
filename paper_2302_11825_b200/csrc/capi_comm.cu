// capi_comm.cu — multi-GPU rounds inside the library: a communicator and
// the sharded updateSolution round (cache.cpp:622-684) behind the C ABI, so a C++
// caller of include/bvc_b200.h runs the multi-GPU path without Python.
//
// The reference has no multi-process path (its parallelism is parallelFor,
// parallel.h:25-50); this is the B200 decomposition of the same round:
//   * rank r of W generates the boundary samples [rN/W, (r+1)N/W) of the round; the
//     walks' Philox streams are keyed by the GLOBAL sample index, so the union of the
//     shards is bitwise the single-GPU cache; its fallback-band walks run on the side
//     stream meanwhile (keyed by the points' global index, bvc_points_set_index_base);
//   * one all-gather of the 48-byte samples (NCCL over NVLink/NVSwitch, or a
//     caller-supplied host-staged exchange) assembles the whole cache on every rank;
//     shards are padded to ceil(N/W) samples so the exchange is one equal-count call;
//   * every rank builds the (cheap, deterministic) source cache itself and gathers its
//     own points: no reduction, each point has one owner, sums are bitwise those of
//     the single-GPU round.
// NCCL is resolved at run time (dlopen of libnccl.so.2, an already-loaded copy first)
// so the library still loads on a host without NCCL; only bvc_comm_init_nccl needs it.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "capi_common.cuh"

struct bvc_comm_s {
    int nranks = 1, rank = 0, device = 0;
    ncclComm_t nccl = nullptr;
    bvc_allgather_fn fn = nullptr;  // host-staged exchange (bvc_comm_init_callback)
    void* user = nullptr;
};

namespace bvc_capi {
namespace {

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        // a copy already in the process (e.g. torch's) first, then the loader's search path
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        n.getUniqueId = reinterpret_cast<decltype(n.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        n.commInitRank = reinterpret_cast<decltype(n.commInitRank)>(dlsym(h, "ncclCommInitRank"));
        n.allGather = reinterpret_cast<decltype(n.allGather)>(dlsym(h, "ncclAllGather"));
        n.commDestroy = reinterpret_cast<decltype(n.commDestroy)>(dlsym(h, "ncclCommDestroy"));
        n.errorString = reinterpret_cast<decltype(n.errorString)>(dlsym(h, "ncclGetErrorString"));
        if (n.getUniqueId && n.commInitRank && n.allGather && n.commDestroy && n.errorString) n.h = h;
    });
    if (!n.h) throw Error(BVC_ERR_CUDA, "NCCL is not available (libnccl.so.2 could not be loaded)");
    return n;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw Error(BVC_ERR_CUDA, std::string(what) + ": " + nccl().errorString(r));
}

// the all-gather of equal-size byte shards: recv[q * bytes ...] = rank q's send
void allgather(bvc_comm_s* C, const void* send, void* recv, size_t bytes) {
    if (C->nccl) {
        nccl_check(nccl().allGather(send, recv, bytes, ncclChar, C->nccl, g_stream), "ncclAllGather");
        return;
    }
    if (C->nranks == 1) {
        if (bytes) CK(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, g_stream));
        return;
    }
    // host-staged: the callback runs with the stream drained and completes the exchange
    CK(cudaStreamSynchronize(g_stream));
    int rc = C->fn(send, recv, bytes, C->user, static_cast<void*>(g_stream));
    if (rc != 0) throw Error(BVC_ERR_CUDA, "communicator all-gather callback failed (" + std::to_string(rc) + ")");
}

}  // namespace

// rank's share [begin, end) of n units and the padded per-rank capacity ceil(n / W)
void shard_layout(long long n, int nranks, int rank, long long& begin, long long& end, long long& cap) {
    need(nranks >= 1 && rank >= 0 && rank < nranks, "rank outside the communicator");
    begin = n * rank / nranks;
    end = n * (rank + 1) / nranks;
    cap = (n + nranks - 1) / nranks;
}

// one updateSolution round sharded over the communicator's ranks (see the file comment)
bvc_eval_points_s* update_round_sharded(bvc_comm_s* C, bvc_scene_s* s, const bvc_problem& pb, bvc_region_s* r,
                                        const bvc_cache_config& cfg,
                                        const std::function<bvc_eval_points_s*()>& points, uint64_t seed,
                                        uint64_t round, int gradients, bvc_round_stats* stats) {
    require_device();
    need(s && r, "null argument");
    validate_kernel(pb.kernel);
    if (cfg.sourceBall && gradients) throw Error(BVC_ERR_SOLVER, "ball-kernel source mode does not support gradient splats");
    make_splat_config(s, pb, cfg);
    const int N = std::max(1, cfg.nBoundary);
    long long b, e, cap;
    shard_layout(N, C->nranks, C->rank, b, e, cap);
    cudaEvent_t e0 = round_event(2), e1 = round_event(3), e2 = round_event(4);
    KernelTimer::arm();
    CK(cudaEventRecord(e0, g_stream));
    // 1. the rank's shard, its band walks on the side stream
    bvc_boundary_cache_s shard;
    GenStats st;
    bvc_eval_points_s* p = generate_shard_with_band(s, pb, r, cfg, seed, round, static_cast<int>(b),
                                                    static_cast<int>(e), points, gradients != 0, &shard, st);
    // 2. one equal-count all-gather of the padded shards, then the shards' samples in
    //    global order (one device copy per rank)
    const size_t bytes = static_cast<size_t>(cap) * sizeof(CacheSample);
    auto* send = ws().get<CacheSample>(kWsCommSend, static_cast<size_t>(cap));
    auto* recv = ws().get<CacheSample>(kWsCommRecv, static_cast<size_t>(cap) * C->nranks);
    if (e > b) CK(cudaMemcpyAsync(send, shard.samples.p, (e - b) * sizeof(CacheSample), cudaMemcpyDeviceToDevice, g_stream));
    if (e - b < cap) CK(cudaMemsetAsync(send + (e - b), 0, (cap - (e - b)) * sizeof(CacheSample), g_stream));
    allgather(C, send, recv, bytes);
    bvc_boundary_cache_s full;
    full.n = N;
    full.dim = shard.dim;
    full.voronoi = 0;
    full.length = shard.length;
    full.samples.resize(N);
    for (int q = 0; q < C->nranks; ++q) {
        long long qb, qe, qc;
        shard_layout(N, C->nranks, q, qb, qe, qc);
        if (qe > qb)
            CK(cudaMemcpyAsync(full.samples.p + qb, recv + static_cast<size_t>(q) * cap, (qe - qb) * sizeof(CacheSample),
                               cudaMemcpyDeviceToDevice, g_stream));
    }
    if (cfg.voronoi) assign_voronoi(r, &full);  // needs the whole round's samples (cache.cpp:388)
    // 3. the source cache, identical on every rank (deterministic in (seed, round))
    bvc_source_cache_s sc;
    generate_source(pb, r, cfg, seed, round, &sc);
    CK(cudaEventRecord(e1, g_stream));
    // 4. this rank's points
    splat_round(s, pb, r, cfg, &full, sc.m ? &sc : nullptr, p, seed, round, gradients, nullptr);
    CK(cudaEventRecord(e2, g_stream));
    CK(cudaEventSynchronize(e2));
    KernelTimer::resolve();
    st.resolve();
    if (stats) {
        stats->resampled = st.resampled;
        stats->cacheWalks = st.walks;
        stats->cacheTruncated = st.truncated;
        stats->cacheSteps = st.steps;
        stats->generateSeconds = device_seconds(e0, e1);
        stats->splatSeconds = device_seconds(e1, e2);
    }
    return p;
}

}  // namespace bvc_capi

extern "C" {

int bvc_comm_unique_id(void* id) {
    API({
        need(id != nullptr, "null argument");
        ncclUniqueId u;
        nccl_check(nccl().getUniqueId(&u), "ncclGetUniqueId");
        std::memcpy(id, &u, sizeof(u));
    })
}

int bvc_comm_init_nccl(const void* id, int nranks, int rank, bvc_comm* out) {
    API({
        require_device();
        need(id && out, "null argument");
        need(nranks >= 1 && rank >= 0 && rank < nranks, "rank outside the communicator");
        auto c = std::make_unique<bvc_comm_s>();
        c->nranks = nranks;
        c->rank = rank;
        CK(cudaGetDevice(&c->device));
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        nccl_check(nccl().commInitRank(&c->nccl, nranks, u, rank), "ncclCommInitRank");
        *out = c.release();
    })
}

int bvc_comm_init_callback(int nranks, int rank, bvc_allgather_fn fn, void* user, bvc_comm* out) {
    API({
        need(out && (fn || nranks == 1), "null argument");
        need(nranks >= 1 && rank >= 0 && rank < nranks, "rank outside the communicator");
        auto c = std::make_unique<bvc_comm_s>();
        c->nranks = nranks;
        c->rank = rank;
        c->fn = fn;
        c->user = user;
        *out = c.release();
    })
}

int bvc_comm_info(bvc_comm c, int* nranks, int* rank) {
    API({
        need(c != nullptr, "null communicator");
        if (nranks) *nranks = c->nranks;
        if (rank) *rank = c->rank;
    })
}

int bvc_comm_destroy(bvc_comm c) {
    API({
        if (c && c->nccl) nccl_check(nccl().commDestroy(c->nccl), "ncclCommDestroy");
        delete c;
    })
}

int bvc_shard_layout(long long n, int nranks, int rank, long long* begin, long long* end, long long* capacity) {
    API({
        long long b, e, cap;
        shard_layout(n, nranks, rank, b, e, cap);
        if (begin) *begin = b;
        if (end) *end = e;
        if (capacity) *capacity = cap;
    })
}

int bvc_update_solution_sharded(bvc_comm comm, bvc_scene s, const bvc_problem* pb, bvc_region r,
                                const bvc_cache_config* cfg, bvc_eval_points pts, uint64_t seed, uint64_t round,
                                int gradients, bvc_round_stats* stats) {
    API({
        need(comm && s && pb && r && cfg && pts, "null argument");
        update_round_sharded(comm, s, *pb, r, *cfg, [pts]() { return pts; }, seed, round, gradients, stats);
    })
}

int bvc_update_solution_sharded_host(bvc_comm comm, bvc_scene s, const bvc_problem* pb, bvc_region r,
                                     const bvc_cache_config* cfg, const double* x, size_t n, long long indexBase,
                                     uint64_t seed, uint64_t round, int gradients, double* u, double* grad,
                                     bvc_round_stats* stats) {
    API({
        need(comm && s && pb && r && cfg && (x || n == 0) && (u || n == 0), "null argument");
        need(!grad || gradients, "gradient output requested without gradients");
        need(indexBase >= 0, "negative point index base");
        std::unique_ptr<bvc_eval_points_s> P;
        update_round_sharded(comm, s, *pb, r, *cfg,
                             [&]() -> bvc_eval_points_s* {  // on the side stream, under the shard's walks
                                 P = make_points(x, n, s->host.dim);
                                 P->base = indexBase;
                                 mark_points(s, r, *cfg, P.get());
                                 ensure_order(P.get());
                                 return P.get();
                             },
                             seed, round, gradients, stats);
        if (n == 0) return BVC_OK;
        const int d = P->dim;
        double* o = ws().get<double>(kWsEvalOut, (1 + d) * n);
        launch_solution(P.get(), o, o + n);
        CK(cudaMemcpyAsync(u, o, n * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
        if (grad) CK(cudaMemcpyAsync(grad, o + n, d * n * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
    })
}

}  // extern "C"
