// capi_common.cuh — what the C-ABI translation units share: the stream and error
// state, device buffers and the scratch workspace, the opaque handle types of
// include/bvc_b200.h, and the orchestration entry points each capi_*.cu defines.
//
//   capi.cu          runtime state, scene / region handles and queries
//   capi_cache.cu    generateBoundaryCache / generateSourceCache (cache.cpp:301-406)
//   capi_points.cu   EvaluationPoint handles, markEvaluationPoints (cache.cpp:263-276)
//   capi_splat.cu    splats, corrected splats, updateSolution (cache.cpp:426-684)
//   capi_walks.cu    pointwise estimators (pointwise.cpp:225-288) and fallback walks
//   capi_stream.cu   runStreamlines (runner.cpp:285-373)
#pragma once
#include <functional>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/bvc_b200.h"
#include "gather.h"
#include "host_scene.h"
#include "internal.h"

namespace bvc_capi {

using bvc_host::Error;
using namespace bvc_impl;
using bvc_dev::Node2;
using bvc_dev::Prim2;

extern thread_local std::string g_error;
extern __thread cudaStream_t g_stream;  // __thread: POD, no TLS-init wrapper
// One-shot host callback run right after a cache-walk job is enqueued: the host-buffer
// round (bvc_update_solution_host) uploads and classifies its points on a second
// stream while the walks run.
extern thread_local std::function<void()> g_afterWalkLaunch;
inline void after_walk_launch() {
    if (g_afterWalkLaunch) {
        std::function<void()> f = std::move(g_afterWalkLaunch);
        g_afterWalkLaunch = nullptr;
        f();
    }
}
// the library's work stream for the lifetime of a scope
struct StreamScope {
    cudaStream_t saved;
    explicit StreamScope(cudaStream_t s) : saved(g_stream) { g_stream = s; }
    ~StreamScope() { g_stream = saved; }
    StreamScope(const StreamScope&) = delete;
    StreamScope& operator=(const StreamScope&) = delete;
};
// diagnostic traversal counting (bvc_walk_traffic_profile); off in production
extern __thread bool g_profile;
extern __thread unsigned long long g_profileTotals[2];

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(bvc_host::kCuda, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

inline float int_as_float_host(int v) {
    float f;
    std::memcpy(&f, &v, sizeof f);
    return f;
}

void require_device();

void ensure_pool();
// bvc_set_device / bvc_set_stream: the calling thread's device and its stream there
void bind_device(int device);
void bind_stream(cudaStream_t s);

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0, cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { if (p) cudaFreeAsync(p, g_stream); }
    // stream-ordered allocations from a pool that retains freed memory, so that
    // per-call handles (evaluation points, caches) do not pay cudaMalloc/cudaFree
    void resize(size_t count) {
        if (count > cap) {
            ensure_pool();
            if (p) CK(cudaFreeAsync(p, g_stream));
            p = nullptr;
            CK(cudaMallocAsync(reinterpret_cast<void**>(&p), std::max<size_t>(count, 1) * sizeof(T), g_stream));
            cap = count;
        }
        n = count;
    }
    void upload(const T* h, size_t count) {
        resize(count);
        if (count) CK(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, g_stream));
    }
    void download(T* h, size_t count) const {
        if (count) CK(cudaMemcpyAsync(h, p, count * sizeof(T), cudaMemcpyDeviceToHost, g_stream));
    }
    void zero() { if (n) CK(cudaMemsetAsync(p, 0, n * sizeof(T), g_stream)); }
};

// grow-only scratch buffers keyed by slot
struct Workspace {
    std::vector<std::unique_ptr<DevBuf<char>>> slots;
    template <class T>
    T* get(int slot, size_t count) {
        if (static_cast<int>(slots.size()) <= slot) slots.resize(slot + 1);
        if (!slots[slot]) slots[slot] = std::make_unique<DevBuf<char>>();
        slots[slot]->resize(count * sizeof(T));
        return reinterpret_cast<T*>(slots[slot]->p);
    }
};
// ws() hands out the active workspace: the main one, or (inside a SideScope) the side
// stream's own, so work on the two streams never shares scratch buffers
extern __thread Workspace* g_wsActive;
Workspace& ws();
// a second stream with its own workspace (one per device), for work that overlaps the
// main stream's cache walks
struct SideScope {
    StreamScope stream;
    Workspace* saved;
    SideScope();
    ~SideScope() { g_wsActive = saved; }
    SideScope(const SideScope&) = delete;
    SideScope& operator=(const SideScope&) = delete;
};
enum Slot {
    kWsSamplesTmp, kWsStartU, kWsIsD, kWsGradR, kWsOutside, kWsDIdx, kWsCount, kWsXD, kWsND, kWsRD, kWsGidD, kWsOutU,
    kWsOutD, kWsCounter, kWsSteps, kWsTrunc, kWsFailed, kWsPack, kWsPart, kWsSkipB, kWsSkipS, kWsPts, kWsCtr,
    kWsSortKeysIn, kWsSortKeysOut, kWsSortValsIn, kWsSortTemp, kWsMean, kWsSe, kWsTruncPt, kWsHost1, kWsRegion,
    kWsMean2, kWsSe2, kWsGidU, kWsSrcTmp, kWsSrcFlag, kWsEvalIn, kWsEvalOut, kWsTileBox, kWsUnitCtr,
    kWsCorrCounts, kWsCorrOffsets, kWsCorrStarts, kWsCorrGid, kWsCorrW, kWsCorrOut, kWsCorrMean, kWsCorrScan,
    kWsCorrFlag, kWsBallRs, kWsHull, kWsXs64, kWsBounds, kWsFlag2, kWsHintU, kWsHintD, kWsCommSend, kWsCommRecv, kWsRoundCtr, kWsBadIdx, kWsBadCnt
};

int fail(const std::exception& e);

#define API(...)                          \
    try {                                 \
        __VA_ARGS__;                      \
        return BVC_OK;                    \
    } catch (const std::exception& e) {   \
        return fail(e);                   \
    }

inline void need(bool ok, const char* msg, int code = BVC_ERR_INVALID_ARGUMENT) {
    if (!ok) throw Error(code, msg);
}

inline bvc_dev::DevField to_dev(const bvc_field& f) {
    bvc_dev::DevField d{};
    d.kind = f.kind;
    d.n = f.n;
    for (int i = 0; i < bvc_dev::kFieldMaxParams; ++i) d.p[i] = static_cast<float>(f.p[i]);
    return d;
}

inline void validate_kernel(const bvc_kernel_spec& k) {  // KernelSpec::validate (kernels.h:32-37)
    if ((k.sigma == 0.0) != (k.kind == BVC_KERNEL_POISSON))
        throw Error(BVC_ERR_INVALID_ARGUMENT, "kernel: sigma = 0 iff kind = Poisson");
    if (k.sigma < 0.0) throw Error(BVC_ERR_INVALID_ARGUMENT, "kernel: sigma must be >= 0");
    if (k.dim != 2 && k.dim != 3) throw Error(BVC_ERR_INVALID_ARGUMENT, "kernel: dimension must be 2 or 3");
}

inline void key_of(uint64_t seed, uint64_t salt, uint64_t round, uint32_t& k0, uint32_t& k1) {
    uint64_t k = bvc_dev::mixKey(bvc_dev::mixKey(bvc_dev::mix64(seed), salt), round);
    k0 = static_cast<uint32_t>(k);
    k1 = static_cast<uint32_t>(k >> 32);
}

// salts of the reference (cache.cpp:15-22)
constexpr uint64_t kBoundaryPosSalt = 0x1001, kBoundaryWalkSalt = 0x1002, kBoundaryRedrawSalt = 0x1003,
                   kSourceSalt = 0x1004, kFallbackSalt = 0x1005, kFallbackGradSalt = 0x1006, kPointwiseSalt = 0x2001,
                   kBoundaryCorrSalt = 0x1007, kSourceCorrSalt = 0x1008;

inline double device_seconds(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e-3;
}

// BVH leaf size (<= 8: the leaf code keeps count - 1 in 3 bits). Measured walk
// time by leaf size 1/2/3/4/8: 3D C4 642/613/620/643/743 ms, C5 leaf 2 -9% vs 4;
// 2D C2 7.84/7.34/7.34/7.55/8.21 ms, C3 185/186/189/195/218 ms, but the 1024-segment
// C1 1.65 (leaf 2) vs 1.46 ms (leaf 4). BVC_LEAF2 / BVC_LEAF3 override (tuning).
int leaf_size(int dim, int ns);

struct GenStats {
    long long walks = 0, truncated = 0, steps = 0, resampled = 0;
    // The walk jobs of one generation count on the device ([steps, truncated, walks]):
    // snapshot() enqueues one copy into pinned memory at the end of the generation and
    // resolve() adds it once the caller has synchronised its stream anyway (no host round
    // trip per walk job).
    unsigned long long* dev = nullptr;
    const volatile unsigned long long* pinned = nullptr;
    unsigned long long* device_counters();
    void snapshot();
    void resolve();
};

}  // namespace bvc_capi

using namespace bvc_capi;

// ---------------------------------------------------------------------------
// opaque handles of include/bvc_b200.h
// ---------------------------------------------------------------------------
struct bvc_scene_s {
    bvc_host::HostScene host;
    bvc_host::HostBvh bvh;
    // lazy device state (upload, hint grid, far field) is built once, under lazyMu, and
    // published only after its stream has finished: any host thread and stream may then
    // read it (the flags are atomics, set after the data)
    std::recursive_mutex lazyMu;
    std::atomic<bool> uploaded{false};
    DevBuf<Node2> nodes;
    DevBuf<Prim2> prims;
    DevBuf<float2> segNormal, silP;
    DevBuf<float4> segAB, silN;
    DevBuf<double4> segAB64;  // FP64 endpoints by segment id: exact classification decisions
    DevBuf<int> silAlways;
    // boundary sampler over all segments (BoundarySampler sampling.cpp:8-18)
    DevBuf<double> cdf;
    DevBuf<int> cdfIds;
    DevBuf<float> segArc, segLen;
    double total = 0.0;
    // 3D (triangle meshes)
    DevBuf<bvc_dev::Node3> nodes3;
    DevBuf<bvc_dev::Prim3> prims3;
    DevBuf<float4> triNormal, triA, triB, triC, sil3A, sil3B, sil3N1, sil3N2;
    DevBuf<int4> triSil;
    DevBuf<float4> silRec;  // silhouette-edge records in leaf order (WalkEnv3::silRec)
    // far-field distance grid (FarField, internal.h), built on first walk use. Opt-in
    // (BVC_FARFIELD=1): smaller balls in the far field keep the estimator unbiased but
    // change where walks enter the eps-shell, i.e. the O(eps) shell bias, so results
    // stop matching the reference's exact-radius walks at the parity bar (measured:
    // disk-poisson at the centre -0.24949 vs the reference's -0.24999, se 1e-5). Walk
    // time: C1 -35%, C3 -8%, C4 -6%; with Neumann walls it loses the star radius
    // (C2 +17%) and is not applied to Neumann scenes.
    DevBuf<float> ffGrid;
    FarField ff{};
    std::atomic<bool> ffBuilt{false};
    FarField farfield();
    // warm-start grid (HintGrid, internal.h), built on first walk use
    DevBuf<HintCell> hgCells;
    HintGrid hg{};
    std::atomic<bool> hgBuilt{false};
    HintGrid hintgrid();

    // per primitive id: class (host_scene.h primClass; also the GPU build input) and,
    // in 3D, its leaf index (walk warm starts name leaf slots)
    DevBuf<int> cls, leafOf;
    DevBuf<int2> segSilD;
    int bvhHeight = 0;

    // BVH builder: "sah" = binned SAH on the device (sahbvh.cu; the default for 3D and
    // 2D scenes of >= 4096 segments), "lbvh" = linear BVH on the device (lbvh.cu),
    // "host" = the host builder (host_scene.cpp; the default for small 2D scenes,
    // median splits). BVC_BVH overrides the choice.
    std::string builder() const;
    bool build_on_gpu() const { return builder() != "host"; }
    void gpu_build(int dim, const float4* a, const float4* b, const float4* c, const int2* sil);

    // straight Neumann runs for the walks' rays (2D; WalkEnv::runSeg)
    DevBuf<float4> runSeg, drunSeg;  // Neumann runs (rays), Dirichlet runs (star queries)
    DevBuf<int> runId, drunId;
    int runN = 0, drunN = 0;
    void build_runs();
    void upload2();
    void upload3();
    void build_sil_records();
    bvc_dev::SceneView3 view3();

    void upload();
    bvc_dev::SceneView2 view();
};

struct bvc_region_s {
    bvc_host::HostRegion host;
    bvc_scene_s boundary;
    DevBuf<int> kinds, source;
    std::mutex mu;
    std::atomic<bool> up{false};
    void upload() {
        boundary.upload();
        if (up) return;
        std::lock_guard<std::mutex> lk(mu);
        if (up) return;
        kinds.upload(host.kinds.data(), host.kinds.size());
        source.upload(host.source.data(), host.source.size());
        CK(cudaStreamSynchronize(g_stream));  // published to every thread and stream
        up = true;
    }
};

struct bvc_boundary_cache_s {
    int n = 0, dim = 2, voronoi = 0;
    double length = 0.0;
    DevBuf<CacheSample> samples;
};

struct bvc_source_cache_s {
    int m = 0, dim = 2;
    double area = 0.0;
    DevBuf<SourceSampleDev> samples;
};

struct bvc_eval_points_s {
    size_t n = 0;
    int dim = 2;
    // global index of point 0 when the caller's point set is one shard of a larger one
    // (bvc_points_set_index_base): per-point RNG streams (band walks, clamp
    // corrections) are keyed by base + index, so a sharded run draws what one GPU would
    long long base = 0;
    DevBuf<double> x;
    DevBuf<uint8_t> fallback, unreliable;
    DevBuf<double> bsum, ssum, bgsum, sgsum, walkSum, gwalkSum;
    DevBuf<long long> nb, ms, nbg, msg, walkCount, walkTrunc, gwalkCount, skipped;
    // spatially sorted non-fallback points first, fallback points last
    bool orderValid = false;
    int active = 0;
    DevBuf<int> order;
    DevBuf<float> xs;
    // ball-kernel mode (cache.h:77): radius per point, valid once marked / uploaded
    DevBuf<double> ballR;
    bool ballValid = false;

    PointsDev dev() {
        return PointsDev{bsum.p, ssum.p, nb.p, ms.p, bgsum.p, sgsum.p, nbg.p, msg.p, skipped.p};
    }
};

namespace bvc_capi {

// orchestration shared across the capi_*.cu files
void ensure_order(bvc_eval_points_s* P);                                      // capi_points.cu
void alloc_points(bvc_eval_points_s* P);
void zero_points(bvc_eval_points_s* P);
std::unique_ptr<bvc_eval_points_s> make_points(const double* x, size_t n, int dim);
void mark_points(bvc_scene_s* s, bvc_region_s* r, const bvc_cache_config& cfg, bvc_eval_points_s* p);
void launch_solution(bvc_eval_points_s* P, double* u, double* g);              // EvaluationPoint::solution
WalkEnv make_env(bvc_scene_s* S, const bvc_problem& pb, const bvc_walk_config& wc, uint64_t seed, uint64_t salt,
                 uint64_t round);                                               // capi_cache.cu
WalkEnv3 make_env3(bvc_scene_s* S, const bvc_problem& pb, const bvc_walk_config& wc, uint64_t seed, uint64_t salt,
                   uint64_t round);
void generate_cache(bvc_scene_s* S, const bvc_problem& pb, bvc_region_s* R, const bvc_cache_config& cfg, uint64_t seed,
                    uint64_t round, int begin, int end, bvc_boundary_cache_s* out, GenStats& st);
void generate_source(const bvc_problem& pb, bvc_region_s* R, const bvc_cache_config& cfg, uint64_t seed, uint64_t round,
                     bvc_source_cache_s* out);
void assign_voronoi(bvc_region_s* R, bvc_boundary_cache_s* c);
int gather_kind(const bvc_kernel_spec& k);                                      // capi_splat.cu
bvc_splat_config make_splat_config(bvc_scene_s* S, const bvc_problem& pb, const bvc_cache_config& cfg);
void splat(bvc_boundary_cache_s* b, bvc_source_cache_s* s, bvc_eval_points_s* P, const bvc_splat_config& cfg,
           size_t begin, size_t end, bool val, bool grad, int mode = 0, double clamp = 0.0);
void fallback_walks(bvc_scene_s* S, const bvc_problem& pb, const bvc_cache_config& cfg, bvc_eval_points_s* P,
                    uint64_t seed, uint64_t round, bool gradients);             // capi_walks.cu
bvc_eval_points_s* generate_shard_with_band(bvc_scene_s* s, const bvc_problem& pb, bvc_region_s* r,
                                           const bvc_cache_config& cfg, uint64_t seed, uint64_t round, int begin,
                                           int end, const std::function<bvc_eval_points_s*()>& points,
                                           bool gradients, bvc_boundary_cache_s* out, GenStats& st);  // capi_cache.cu
// updateSolution's splat dispatch (cache.cpp:639-663) over a round's caches
void splat_round(bvc_scene_s* s, const bvc_problem& pb, bvc_region_s* r, const bvc_cache_config& cfg,
                 bvc_boundary_cache_s* bc, bvc_source_cache_s* sc, bvc_eval_points_s* p, uint64_t seed,
                 uint64_t round, int gradients, const bvc_boundary_evaluator* correctionEval);  // capi_splat.cu
// per-thread, per-device events reused by every round (no create/destroy per call):
// 0-1 stream dependencies, 2-4 round phases, 5-8 the round's main kernels (KernelTimer)
int read_device_int(const int* dev);  // via pinned memory (capi.cu)
cudaEvent_t round_event(int which);                                             // capi.cu

// Device time of a round's two hot launches (the main cache-walk job and the main gather),
// bracketed by events on the launching stream: the rooflines' per-launch durations
// (bvc_last_round_kernel_seconds). Armed by a round; only the first launch of each kind
// inside it is timed, and the values are read once the round has synchronized.
struct KernelTimer {
    enum { kWalk = 0, kGather = 1 };
    static void arm();                  // a round starts: forget the previous round's launches
    static void begin(int which);       // before the launch (no-op unless armed and not yet timed)
    static void end(int which);         // after it
    static void resolve();              // after the round's sync: elapsed times -> last()
    static const double* last();        // [walk, gather] seconds of the last resolved round (0 = none)
};

}  // namespace bvc_capi
