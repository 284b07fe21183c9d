// capi.cu — the C ABI (include/bvc_b200.h) over the sm_100a BVC kernels.
//
// Orchestrates the reference's operator API on the device:
//   generateBoundaryCache (cache.cpp:301-390), generateSourceCache (392-406),
//   markEvaluationPoints (263-276), splatSolution / splatGradient (426-497),
//   updateSolution (622-684) and the pointwise estimators (pointwise.cpp:225-288).
// Host preprocessing (scene build, solve region, BVH) is host_scene.cpp.
// There is no CPU fallback: every compute entry point fails with
// BVC_ERR_NO_DEVICE when no CUDA device is present.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <memory>
#include <string>
#include <vector>

#include "../../include/bvc_b200.h"
#include "gather.h"
#include "host_scene.h"
#include "internal.h"

using bvc_host::Error;
using namespace bvc_impl;
using bvc_dev::Node2;
using bvc_dev::Prim2;

namespace {

thread_local std::string g_error;
cudaStream_t g_stream = nullptr;
// diagnostic traversal counting (bvc_walk_traffic_profile); off in production
bool g_profile = false;
unsigned long long g_profileTotals[2] = {0, 0};
std::atomic<long long> g_launches{0};

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(bvc_host::kCuda, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

inline float __int_as_float_host(int v) {
    float f;
    std::memcpy(&f, &v, sizeof f);
    return f;
}

void require_device() {
    static int state = -1;  // -1 unknown, 0 none, 1 ok
    if (state < 0) {
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        state = (e == cudaSuccess && n > 0) ? 1 : 0;
        if (e != cudaSuccess) cudaGetLastError();
    }
    if (!state) throw Error(bvc_host::kNoDevice, "no CUDA device: the BVC path has no CPU fallback");
}

void ensure_pool() {
    static int device = -1;
    int d = 0;
    cudaGetDevice(&d);
    if (d == device) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    device = d;
}

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
Workspace& ws() {
    static Workspace w;
    return w;
}
enum Slot {
    kWsSamplesTmp, kWsStartU, kWsIsD, kWsGradR, kWsOutside, kWsDIdx, kWsCount, kWsXD, kWsND, kWsRD, kWsGidD, kWsOutU,
    kWsOutD, kWsCounter, kWsSteps, kWsTrunc, kWsFailed, kWsPack, kWsPart, kWsSkipB, kWsSkipS, kWsPts, kWsCtr,
    kWsSortKeysIn, kWsSortKeysOut, kWsSortValsIn, kWsSortTemp, kWsMean, kWsSe, kWsTruncPt, kWsHost1, kWsRegion,
    kWsMean2, kWsSe2, kWsGidU, kWsSrcTmp, kWsSrcFlag, kWsEvalIn, kWsEvalOut, kWsTileBox, kWsUnitCtr,
    kWsCorrCounts, kWsCorrOffsets, kWsCorrStarts, kWsCorrGid, kWsCorrW, kWsCorrOut, kWsCorrMean, kWsCorrScan,
    kWsCorrFlag, kWsBallRs, kWsHull, kWsXs64, kWsBounds, kWsFlag2, kWsHintU, kWsHintD
};

int fail(const std::exception& e) {
    g_error = e.what();
    if (auto* be = dynamic_cast<const Error*>(&e)) return be->code;
    if (dynamic_cast<const std::bad_alloc*>(&e)) return BVC_ERR_CUDA;
    return BVC_ERR_SOLVER;
}

#define API(...)                          \
    try {                                 \
        __VA_ARGS__;                      \
        return BVC_OK;                    \
    } catch (const std::exception& e) {   \
        return fail(e);                   \
    }

void need(bool ok, const char* msg, int code = BVC_ERR_INVALID_ARGUMENT) {
    if (!ok) throw Error(code, msg);
}

bvc_dev::DevField to_dev(const bvc_field& f) {
    bvc_dev::DevField d{};
    d.kind = f.kind;
    d.n = f.n;
    for (int i = 0; i < bvc_dev::kFieldMaxParams; ++i) d.p[i] = static_cast<float>(f.p[i]);
    return d;
}

void validate_kernel(const bvc_kernel_spec& k) {  // KernelSpec::validate (kernels.h:32-37)
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

double device_seconds(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e-3;
}

}  // namespace

namespace bvc_impl {
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
int api_fail(const std::exception& e) { return fail(e); }
}  // namespace bvc_impl

// ---------------------------------------------------------------------------
// handles
// ---------------------------------------------------------------------------
// BVH leaf size (<= 8: the leaf code keeps count - 1 in 3 bits). Measured walk
// time by leaf size 1/2/3/4/8: 3D C4 642/613/620/643/743 ms, C5 leaf 2 -9% vs 4;
// 2D C2 7.84/7.34/7.34/7.55/8.21 ms, C3 185/186/189/195/218 ms, but the 1024-segment
// C1 1.65 (leaf 2) vs 1.46 ms (leaf 4). BVC_LEAF2 / BVC_LEAF3 override (tuning).
int leaf_size(int dim, int ns) {
    const char* e = std::getenv(dim == 2 ? "BVC_LEAF2" : "BVC_LEAF3");
    int def = (dim == 3 || ns > 1024) ? 2 : 4;
    int v = e ? std::atoi(e) : def;
    return v >= 1 && v <= 8 ? v : def;
}

struct bvc_scene_s {
    bvc_host::HostScene host;
    bvc_host::HostBvh bvh;
    bool uploaded = false;
    DevBuf<Node2> nodes;
    DevBuf<Prim2> prims;
    DevBuf<float2> segNormal, silP;
    DevBuf<float4> segAB, silN;
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
    // far-field distance grid (FarField, internal.h), built on first walk use. Opt-in
    // (BVC_FARFIELD=1): smaller balls in the far field keep the estimator unbiased but
    // change where walks enter the eps-shell, i.e. the O(eps) shell bias, so results
    // stop matching the reference's exact-radius walks at the parity bar (measured:
    // disk-poisson at the centre -0.24949 vs the reference's -0.24999, se 1e-5). Walk
    // time: C1 -35%, C3 -8%, C4 -6%; with Neumann walls it loses the star radius
    // (C2 +17%) and is not applied to Neumann scenes.
    DevBuf<float> ffGrid;
    FarField ff{};
    bool ffBuilt = false;
    FarField farfield() {
        const char* e = std::getenv("BVC_FARFIELD");
        if (!(e && std::string(e) == "1") || host.hasNeumann()) return FarField{};
        if (ffBuilt) return ff;
        upload();
        int dim = host.dim;
        const int nLong = dim == 2 ? 1024 : 128;  // 1M / 2M vertices
        double ext = 0.0, lo[3], hi[3];
        for (int k = 0; k < dim; ++k) {
            double pad = 0.01 * host.diagonal;
            lo[k] = host.lo[k] - pad;
            hi[k] = host.hi[k] + pad;
            ext = std::max(ext, hi[k] - lo[k]);
        }
        double h = ext / (nLong - 1);
        int n[3] = {1, 1, 1};
        for (int k = 0; k < dim; ++k) n[k] = static_cast<int>(std::ceil((hi[k] - lo[k]) / h)) + 1;
        ff = FarField{};
        ff.lox = static_cast<float>(lo[0]);
        ff.loy = static_cast<float>(lo[1]);
        ff.loz = dim == 3 ? static_cast<float>(lo[2]) : 0.f;
        ff.h = static_cast<float>(h);
        ff.invH = static_cast<float>(1.0 / h);
        ff.tau = static_cast<float>(8.0 * h);
        ff.margin = static_cast<float>(1e-6 * host.diagonal + 1e-3 * h);  // FP32 rounding of d(v) and |x - v|
        ff.nx = n[0];
        ff.ny = n[1];
        ff.nz = n[2];
        ffGrid.resize(static_cast<size_t>(n[0]) * n[1] * n[2]);
        ff.d = ffGrid.p;
        if (dim == 2) launch_farfield2(view(), ff, ffGrid.p, g_stream);
        else launch_farfield3(view3(), ff, ffGrid.p, g_stream);
        CK(cudaGetLastError());
        ffBuilt = true;
        return ff;
    }

    // per primitive id: class (host_scene.h primClass; also the GPU build input) and,
    // in 3D, its leaf index (walk warm starts name leaf slots)
    DevBuf<int> cls, leafOf;
    DevBuf<int2> segSilD;
    int bvhHeight = 0;

    // BVH builder: "sah" = binned SAH on the device (sahbvh.cu; the default for 3D and
    // 2D scenes of >= 4096 segments), "lbvh" = linear BVH on the device (lbvh.cu),
    // "host" = the host builder (host_scene.cpp; the default for small 2D scenes,
    // median splits). BVC_BVH overrides the choice.
    std::string builder() const {
        const char* e = std::getenv("BVC_BVH");
        std::string v = e ? e : "";
        if (v == "gpu") v = "lbvh";
        if (v != "sah" && v != "lbvh" && v != "host") v = (host.dim == 3 || host.ns >= 4096) ? "sah" : "host";
        return host.ns > 64 ? v : "host";  // tiny scenes: one host pass
    }
    bool build_on_gpu() const { return builder() != "host"; }
    void gpu_build(int dim, const float4* a, const float4* b, const float4* c, const int2* sil) {
        int n = host.ns, leaf = leaf_size(dim, n);
        double pad = 9.5367431640625e-7 * std::max(host.diagonal, 1e-30);
        size_t nn = static_cast<size_t>(std::max(n - 1, 1));
        if (dim == 2) { nodes.resize(nn); prims.resize(std::max(n, 1)); }
        else { nodes3.resize(nn); prims3.resize(std::max(n, 1)); }
        void* nodesOut = dim == 2 ? static_cast<void*>(nodes.p) : static_cast<void*>(nodes3.p);
        void* primsOut = dim == 2 ? static_cast<void*>(prims.p) : static_cast<void*>(prims3.p);
        int h;
        if (builder() == "lbvh") {
            h = build_lbvh(dim, a, b, c, cls.p, sil, n, leaf, host.lo, host.hi, pad, dim == 2 ? 1 : 0, nodesOut,
                           primsOut, g_stream);
        } else {
            DevBuf<int> ids;
            ids.resize(n);
            h = build_sah_gpu(dim, a, b, c, cls.p, n, leaf, pad, dim == 2 ? 1 : 0, nodesOut, ids.p, g_stream);
            launch_leaf_prims(dim, a, b, c, cls.p, sil, ids.p, n, primsOut, g_stream);
            CK(cudaStreamSynchronize(g_stream));
        }
        CK(cudaGetLastError());
        if (h < 0 || h >= 47)  // deeper than the device traversal stack
            throw Error(BVC_ERR_SOLVER, "GPU BVH build: tree deeper than the traversal stack; use BVC_BVH=host");
        bvhHeight = h;
    }

    void upload3() {
        auto f4 = [](const double* p, float w) { return make_float4(p[0], p[1], p[2], w); };
        if (!build_on_gpu()) {
            bvh = bvc_host::buildBvh(host, leaf_size(3, host.ns));
            size_t nn = bvh.children.size() / 2;
            std::vector<bvc_dev::Node3> hn(nn);
            for (size_t i = 0; i < nn; ++i) {
                const float* b = &bvh.boxes[12 * i];
                hn[i].llo = make_float4(b[0], b[1], b[2], 0.f);
                hn[i].lhi = make_float4(b[3], b[4], b[5], 0.f);
                hn[i].rlo = make_float4(b[6], b[7], b[8], 0.f);
                hn[i].rhi = make_float4(b[9], b[10], b[11], 0.f);
                hn[i].left = bvh.children[2 * i];
                hn[i].right = bvh.children[2 * i + 1];
                hn[i].mask = bvh.masks[i];
                hn[i].pad = 0;
            }
            nodes3.upload(hn.data(), nn);
            std::vector<bvc_dev::Prim3> hp(host.ns);
            for (int j = 0; j < host.ns; ++j) {
                int id = bvh.order[j];
                hp[j].a = f4(host.vert(host.idx[3 * id]), __int_as_float_host(id));
                hp[j].b = f4(host.vert(host.idx[3 * id + 1]), __int_as_float_host(bvc_host::primClass(host, id)));
                hp[j].c = f4(host.vert(host.idx[3 * id + 2]), 0.f);
            }
            prims3.upload(hp.data(), hp.size());
        }
        std::vector<float4> hn4(host.ns), ha(host.ns), hb(host.ns), hc(host.ns);
        std::vector<int4> hs(host.ns);
        std::vector<double> cd(host.ns);
        double run = 0.0;
        for (int i = 0; i < host.ns; ++i) {
            hn4[i] = f4(&host.normal[3 * static_cast<size_t>(i)], 0.f);
            ha[i] = f4(host.vert(host.idx[3 * i]), 0.f);
            hb[i] = f4(host.vert(host.idx[3 * i + 1]), 0.f);
            hc[i] = f4(host.vert(host.idx[3 * i + 2]), 0.f);
            hs[i] = make_int4(host.triSil[3 * i], host.triSil[3 * i + 1], host.triSil[3 * i + 2], -1);
            run += host.measure[i];
            cd[i] = run;
        }
        total = run;
        triNormal.upload(hn4.data(), hn4.size());
        triA.upload(ha.data(), ha.size());
        triB.upload(hb.data(), hb.size());
        triC.upload(hc.data(), hc.size());
        triSil.upload(hs.data(), hs.size());
        cdf.upload(cd.data(), cd.size());
        size_t ne = std::max<size_t>(host.sil3Always.size(), 1);
        std::vector<float4> ea(ne), eb(ne), e1(ne), e2(ne);
        for (size_t k = 0; k < host.sil3Always.size(); ++k) {
            ea[k] = f4(&host.sil3A[3 * k], 0.f);
            eb[k] = f4(&host.sil3B[3 * k], 0.f);
            e1[k] = f4(&host.sil3N1[3 * k], host.sil3Always[k] ? 1.f : 0.f);
            e2[k] = f4(&host.sil3N2[3 * k], 0.f);
        }
        sil3A.upload(ea.data(), ne);
        sil3B.upload(eb.data(), ne);
        sil3N1.upload(e1.data(), ne);
        sil3N2.upload(e2.data(), ne);
        std::vector<int> hcls(host.ns);
        for (int i = 0; i < host.ns; ++i) hcls[i] = bvc_host::primClass(host, i);
        cls.upload(hcls.data(), hcls.size());
        if (build_on_gpu()) gpu_build(3, triA.p, triB.p, triC.p, nullptr);
        leafOf.resize(std::max(host.ns, 1));  // triangle id -> leaf index (walk warm starts)
        launch_leaf_index(3, prims3.p, host.ns, leafOf.p, g_stream);
        uploaded = true;
    }
    bvc_dev::SceneView3 view3() {
        upload();
        bvc_dev::SceneView3 v;
        v.nodes = nodes3.p;
        v.prims = prims3.p;
        v.triNormal = triNormal.p;
        v.nt = host.ns;
        v.diagonal = static_cast<float>(host.diagonal);
        v.counts = nullptr;
        return v;
    }

    void upload() {
        if (uploaded) return;
        require_device();
        if (host.dim == 3) {
            upload3();
            return;
        }
        if (!build_on_gpu()) {
            bvh = bvc_host::buildBvh(host, leaf_size(2, host.ns));
            size_t nn = bvh.children.size() / 2;
            std::vector<Node2> hn(nn);
            for (size_t i = 0; i < nn; ++i) {
                const float* b = &bvh.boxes[8 * i];
                hn[i].lbox = make_float4(b[0], b[1], b[2], b[3]);
                hn[i].rbox = make_float4(b[4], b[5], b[6], b[7]);
                hn[i].left = bvh.children[2 * i];
                hn[i].right = bvh.children[2 * i + 1];
                hn[i].mask = bvh.masks[i];
                hn[i].pad = 0;
            }
            nodes.upload(hn.data(), nn);
            std::vector<Prim2> hp(host.ns);
            for (int j = 0; j < host.ns; ++j) {
                int id = bvh.order[j];
                const double *a = host.vert(host.idx[2 * id]), *b = host.vert(host.idx[2 * id + 1]);
                hp[j].seg = make_float4(a[0], a[1], b[0], b[1]);
                hp[j].id = id;
                hp[j].label = bvc_host::primClass(host, id);
                hp[j].sil0 = host.segSil[2 * id];
                hp[j].sil1 = host.segSil[2 * id + 1];
            }
            prims.upload(hp.data(), hp.size());
        }
        std::vector<float2> hnrm(host.ns);
        std::vector<float4> hab(host.ns);
        std::vector<float> harc(host.ns), hlen(host.ns);
        for (int i = 0; i < host.ns; ++i) {
            hnrm[i] = make_float2(host.normal[2 * i], host.normal[2 * i + 1]);
            const double *a = host.vert(host.idx[2 * i]), *b = host.vert(host.idx[2 * i + 1]);
            hab[i] = make_float4(a[0], a[1], b[0], b[1]);
            harc[i] = static_cast<float>(host.arc[i]);
            hlen[i] = static_cast<float>(host.measure[i]);
        }
        segNormal.upload(hnrm.data(), hnrm.size());
        segAB.upload(hab.data(), hab.size());
        segArc.upload(harc.data(), harc.size());
        segLen.upload(hlen.data(), hlen.size());
        size_t nsil = host.silAlways.size();
        std::vector<float2> hsp(std::max<size_t>(nsil, 1));
        std::vector<float4> hsn(std::max<size_t>(nsil, 1));
        std::vector<int> hsa(std::max<size_t>(nsil, 1), 0);
        for (size_t k = 0; k < nsil; ++k) {
            hsp[k] = make_float2(host.silP[2 * k], host.silP[2 * k + 1]);
            hsn[k] = make_float4(host.silN1[2 * k], host.silN1[2 * k + 1], host.silN2[2 * k], host.silN2[2 * k + 1]);
            hsa[k] = host.silAlways[k];
        }
        silP.upload(hsp.data(), hsp.size());
        silN.upload(hsn.data(), hsn.size());
        silAlways.upload(hsa.data(), hsa.size());
        std::vector<int> hcls(host.ns);
        for (int i = 0; i < host.ns; ++i) hcls[i] = bvc_host::primClass(host, i);
        cls.upload(hcls.data(), hcls.size());
        if (build_on_gpu()) {
            std::vector<int2> hsl(host.ns);
            for (int i = 0; i < host.ns; ++i) hsl[i] = make_int2(host.segSil[2 * i], host.segSil[2 * i + 1]);
            segSilD.upload(hsl.data(), hsl.size());
            gpu_build(2, segAB.p, nullptr, nullptr, segSilD.p);
        }
        std::vector<double> hc(host.ns);
        std::vector<int> hid(host.ns);
        double run = 0.0;
        for (int i = 0; i < host.ns; ++i) {
            run += host.measure[i];
            hc[i] = run;
            hid[i] = i;
        }
        total = run;
        cdf.upload(hc.data(), hc.size());
        cdfIds.upload(hid.data(), hid.size());
        uploaded = true;
    }
    bvc_dev::SceneView2 view() {
        upload();
        bvc_dev::SceneView2 v;
        v.nodes = nodes.p;
        v.prims = prims.p;
        v.segNormal = segNormal.p;
        v.segAB = segAB.p;
        v.silP = silP.p;
        v.silN = silN.p;
        v.silAlways = silAlways.p;
        v.ns = host.ns;
        v.diagonal = static_cast<float>(host.diagonal);
        v.counts = nullptr;
        return v;
    }
};

struct bvc_region_s {
    bvc_host::HostRegion host;
    bvc_scene_s boundary;
    DevBuf<int> kinds, source;
    void upload() {
        boundary.upload();
        if (!kinds.n) {
            kinds.upload(host.kinds.data(), host.kinds.size());
            source.upload(host.source.data(), host.source.size());
        }
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

namespace {

// order-preserving map of a double to an unsigned 64-bit key (for atomicMin/Max)
__device__ __forceinline__ unsigned long long dkey(double v) {
    unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double dval(unsigned long long k) {
    return __longlong_as_double(static_cast<long long>((k >> 63) ? (k & 0x7fffffffffffffffULL) : ~k));
}
// bounding box of the points: keys[0..2] = min, [3..5] = max (initialised by the host)
__global__ void bounds_kernel(const double* x, int n, int dim, unsigned long long* keys) {
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        for (int d = 0; d < dim; ++d) {
            double v = x[static_cast<size_t>(dim) * i + d];
            lo[d] = fmin(lo[d], v);
            hi[d] = fmax(hi[d], v);
        }
    for (int d = 0; d < dim; ++d)
        for (int o = 16; o > 0; o >>= 1) {
            lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
            hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
        }
    if ((threadIdx.x & 31) == 0)
        for (int d = 0; d < dim; ++d) {
            atomicMin(keys + d, dkey(lo[d]));
            atomicMax(keys + 3 + d, dkey(hi[d]));
        }
}

__global__ void morton_keys_kernel(const double* x, const uint8_t* fb, int n, int dim,
                                   const unsigned long long* bounds, unsigned* keys, int* vals) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double lo0 = dval(bounds[0]), lo1 = dval(bounds[1]), lo2 = dim == 3 ? dval(bounds[2]) : 0.0;
    double ext = 0.0;
    for (int d = 0; d < dim; ++d) ext = fmax(ext, dval(bounds[3 + d]) - dval(bounds[d]));
    double inv = ext > 0 ? 1.0 / ext : 1.0;
    auto spread2 = [](unsigned v) {  // 15 bits -> every other bit
        v &= 0x7fff;
        v = (v | (v << 8)) & 0x00ff00ff;
        v = (v | (v << 4)) & 0x0f0f0f0f;
        v = (v | (v << 2)) & 0x33333333;
        v = (v | (v << 1)) & 0x55555555;
        return v;
    };
    auto spread3 = [](unsigned v) {  // 10 bits -> every third bit
        v &= 0x3ff;
        v = (v | (v << 16)) & 0x030000ff;
        v = (v | (v << 8)) & 0x0300f00f;
        v = (v | (v << 4)) & 0x030c30c3;
        v = (v | (v << 2)) & 0x09249249;
        return v;
    };
    unsigned key;
    if (dim == 2) {
        unsigned a = static_cast<unsigned>(fmin(fmax((x[2 * i] - lo0) * inv, 0.0), 1.0) * 32767.0);
        unsigned b = static_cast<unsigned>(fmin(fmax((x[2 * i + 1] - lo1) * inv, 0.0), 1.0) * 32767.0);
        key = spread2(a) | (spread2(b) << 1);
    } else {
        unsigned a = static_cast<unsigned>(fmin(fmax((x[3 * i] - lo0) * inv, 0.0), 1.0) * 1023.0);
        unsigned b = static_cast<unsigned>(fmin(fmax((x[3 * i + 1] - lo1) * inv, 0.0), 1.0) * 1023.0);
        unsigned c = static_cast<unsigned>(fmin(fmax((x[3 * i + 2] - lo2) * inv, 0.0), 1.0) * 1023.0);
        key = spread3(a) | (spread3(b) << 1) | (spread3(c) << 2);
    }
    if (fb && fb[i]) key |= 0x80000000u;
    keys[i] = key;
    vals[i] = i;
}

__global__ void count_active_kernel(const uint8_t* fb, int n, int* count) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    int v = (i < n && !fb[i]) ? 1 : 0;
    v = __reduce_add_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(count, v);
}

void ensure_order(bvc_eval_points_s* P) {
    if (P->orderValid) return;
    int n = static_cast<int>(P->n);
    P->order.resize(n);
    if (n == 0) {
        P->active = 0;
        P->orderValid = true;
        return;
    }
    // bounding box on the device (no host copy of the points is kept)
    unsigned long long* bk = ws().get<unsigned long long>(kWsBounds, 6);
    const unsigned long long init[6] = {~0ULL, ~0ULL, ~0ULL, 0ULL, 0ULL, 0ULL};
    CK(cudaMemcpyAsync(bk, init, sizeof(init), cudaMemcpyHostToDevice, g_stream));
    bounds_kernel<<<std::min((n + 255) / 256, 1184), 256, 0, g_stream>>>(P->x.p, n, P->dim, bk);
    unsigned* kin = ws().get<unsigned>(kWsSortKeysIn, n);
    unsigned* kout = ws().get<unsigned>(kWsSortKeysOut, n);
    int* vin = ws().get<int>(kWsSortValsIn, n);
    morton_keys_kernel<<<(n + 255) / 256, 256, 0, g_stream>>>(P->x.p, P->fallback.p, n, P->dim, bk, kin, vin);
    count_launch(2);
    size_t tmp = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, P->order.p, n, 0, 32, g_stream));
    void* t = ws().get<char>(kWsSortTemp, tmp);
    CK(cub::DeviceRadixSort::SortPairs(t, tmp, kin, kout, vin, P->order.p, n, 0, 32, g_stream));
    count_launch();
    int* cnt = ws().get<int>(kWsCount, 1);
    CK(cudaMemsetAsync(cnt, 0, sizeof(int), g_stream));
    count_active_kernel<<<(n + 255) / 256, 256, 0, g_stream>>>(P->fallback.p, n, cnt);
    count_launch();
    CK(cudaMemcpyAsync(&P->active, cnt, sizeof(int), cudaMemcpyDeviceToHost, g_stream));
    CK(cudaStreamSynchronize(g_stream));
    P->xs.resize(static_cast<size_t>(P->dim) * std::max(P->active, 1));
    gather_points(P->x.p, P->order.p, P->active, P->dim, P->xs.p, g_stream);
    P->orderValid = true;
}

WalkEnv make_env(bvc_scene_s* S, const bvc_problem& pb, const bvc_walk_config& wc, uint64_t seed, uint64_t salt,
                 uint64_t round) {
    validate_kernel(pb.kernel);
    if (pb.kernel.dim != 2) throw Error(BVC_ERR_SOLVER, "walk estimators support dim == 2 only");
    WalkEnv E{};
    E.S = S->view();
    E.P.screened = pb.kernel.kind == BVC_KERNEL_SCREENED;
    E.P.sigma = static_cast<float>(pb.kernel.sigma);
    E.P.sqrtSigma = static_cast<float>(std::sqrt(pb.kernel.sigma));
    E.P.dim = 2;
    E.P.f = to_dev(pb.f);
    E.P.g = to_dev(pb.g);
    E.P.h = to_dev(pb.h);
    double diag = S->host.diagonal;
    double eps = wc.epsilon > 0.0 ? wc.epsilon : 1e-3 * diag;         // pointwise.h:36-38
    double rmin = wc.rMin > 0.0 ? wc.rMin : eps;                        // pointwise.h:39-44
    if (rmin > eps) throw Error(BVC_ERR_INVALID_ARGUMENT, "walk config: r_min must lie in (0, epsilon]");
    E.eps = static_cast<float>(eps);
    E.rmin = static_cast<float>(rmin);
    // the reference's tGuard is 1e-9 diag (pointwise.cpp:115); FP32 positions need a
    // guard above their rounding, and the current segment is skipped explicitly
    E.tguard = static_cast<float>(1e-9 * diag);  // pointwise.cpp:115; the standing segment is skipped
    E.insideTol = S->host.closed() ? static_cast<float>(std::max(1e-9, 1e-7) * diag) : -1.0f;
    E.scale = static_cast<float>(diag);
    E.nudge = static_cast<float>(9.5367431640625e-7 * diag);  // 2^-20 diag, << eps
    E.cx = static_cast<float>(0.5 * (S->host.lo[0] + S->host.hi[0]));
    E.cy = static_cast<float>(0.5 * (S->host.lo[1] + S->host.hi[1]));
    E.escape = static_cast<float>(diag);
    E.maxSteps = std::max(1, wc.maxSteps);
    E.hasNeumann = S->host.hasNeumann() ? 1 : 0;
    E.hasSource = pb.f.kind != BVC_FIELD_NONE ? 1 : 0;
    E.hasH = pb.h.kind != BVC_FIELD_NONE ? 1 : 0;
    E.closed = S->host.closed() ? 1 : 0;
    if (!(S->host.dirichletMeasure > 0.0))
        throw Error(BVC_ERR_SOLVER, "walk cannot terminate: scene has no Dirichlet boundary");
    key_of(seed, salt, round, E.k0, E.k1);
    E.ff = S->farfield();
    return E;
}

struct GenStats {
    long long walks = 0, truncated = 0, steps = 0, resampled = 0;
};

// walks for the samples [0, n) of `samples` (already positioned); writes uHat/dHat
// and returns per-sample failure flags in `failed` (device)
void run_cache_walks(bvc_scene_s* S, bvc_region_s* R, const WalkEnv& E, const bvc_cache_config& cfg,
                     CacheSample* samples, int n, long long gidBase, const long long* gid, uint8_t* failed,
                     GenStats& st) {
    float2* startU = ws().get<float2>(kWsStartU, n);
    int* isD = ws().get<int>(kWsIsD, n);
    float* gradR = ws().get<float>(kWsGradR, n);
    launch_prepare_samples(E, samples, n, R->kinds.p, R->source.p, startU, isD, gradR, failed, g_stream);
    int* dIdx = ws().get<int>(kWsDIdx, n);
    int* cnt = ws().get<int>(kWsCount, 1);
    launch_compact(isD, n, dIdx, cnt, g_stream);
    int nD = 0;
    CK(cudaMemcpyAsync(&nD, cnt, sizeof(int), cudaMemcpyDeviceToHost, g_stream));
    CK(cudaStreamSynchronize(g_stream));
    float2* xD = ws().get<float2>(kWsXD, std::max(nD, 1));
    float2* nrmD = ws().get<float2>(kWsND, std::max(nD, 1));
    float* rD = ws().get<float>(kWsRD, std::max(nD, 1));
    long long* gidD = ws().get<long long>(kWsGidD, std::max(nD, 1));
    launch_gather_dpoints(samples, dIdx, nD, gradR, gidBase, gid, xD, nrmD, rD, gidD, g_stream);
    int nU = std::max(1, cfg.nWalksNeumann), nDw = std::max(1, cfg.nWalksDirichlet);
    int* hintU = ws().get<int>(kWsHintU, std::max(n, 1));
    int* hintD = ws().get<int>(kWsHintD, std::max(nD, 1));
    launch_start_hints(samples, n, R->source.p, S->cls.p, nullptr, dIdx, nD, hintU, hintD, g_stream);
    WalkJob J{};
    J.hintU = hintU;
    J.hintD = hintD;
    J.nU = nU;
    J.nPtsU = n;
    J.startU = startU;
    J.gidU = gid;
    J.gidBaseU = gidBase;
    J.outU = ws().get<float>(kWsOutU, static_cast<size_t>(n) * nU);
    J.nD = nDw;
    J.nPtsD = nD;
    J.xD = xD;
    J.normalD = nrmD;
    J.radiusD = rD;
    J.gidD = gidD;
    J.outD = ws().get<float>(kWsOutD, std::max<size_t>(static_cast<size_t>(nD) * nDw, 1));
    auto* ctr = ws().get<unsigned long long>(kWsCounter, 3);
    CK(cudaMemsetAsync(ctr, 0, 3 * sizeof(unsigned long long), g_stream));
    J.counter = ctr;
    J.steps = ctr + 1;
    J.truncTotal = ctr + 2;
    if (g_profile) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        size_t slots = static_cast<size_t>(sms) * 32 * 256 * 2;
        auto* cnt = ws().get<unsigned long long>(kWsEvalOut, slots);
        CK(cudaMemsetAsync(cnt, 0, slots * sizeof(unsigned long long), g_stream));
        WalkEnv Ec = E;
        Ec.S.counts = cnt;
        launch_walk_job(Ec, J, g_stream);
        std::vector<unsigned long long> h(slots);
        CK(cudaMemcpyAsync(h.data(), cnt, slots * sizeof(unsigned long long), cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
        for (size_t i = 0; i < slots; ++i) g_profileTotals[i & 1] += h[i];
    } else {
        launch_walk_job(E, J, g_stream);
    }
    launch_finish_samples(samples, n, J.outU, nU, dIdx, nD, J.outD, nDw, failed, g_stream);
    unsigned long long h[3];
    CK(cudaMemcpyAsync(h, ctr, sizeof(h), cudaMemcpyDeviceToHost, g_stream));
    CK(cudaStreamSynchronize(g_stream));
    st.walks += static_cast<long long>(n) * nU + static_cast<long long>(nD) * nDw;
    st.steps += static_cast<long long>(h[1]);
    st.truncated += static_cast<long long>(h[2]);
}

__global__ void redraw_copy_kernel(const CacheSample* src, const int* idx, int n, CacheSample* dst);

WalkEnv3 make_env3(bvc_scene_s* S, const bvc_problem& pb, const bvc_walk_config& wc, uint64_t seed, uint64_t salt,
                   uint64_t round) {
    validate_kernel(pb.kernel);
    if (pb.kernel.dim != 3) throw Error(BVC_ERR_INVALID_ARGUMENT, "3D scene needs a dim-3 kernel");
    if (pb.f.kind != BVC_FIELD_NONE)
        throw Error(BVC_ERR_SOLVER, "source terms are not supported by the 3D walks (kernels.cpp:98-99 is 2D-only)");
    if (!(S->host.dirichletMeasure > 0.0))
        throw Error(BVC_ERR_SOLVER, "walk cannot terminate: scene has no Dirichlet boundary");
    WalkEnv3 E{};
    E.S = S->view3();
    E.triSil = S->triSil.p;
    E.silA = S->sil3A.p;
    E.silB = S->sil3B.p;
    E.silN1 = S->sil3N1.p;
    E.silN2 = S->sil3N2.p;
    E.P.screened = pb.kernel.kind == BVC_KERNEL_SCREENED;
    E.P.sigma = static_cast<float>(pb.kernel.sigma);
    E.P.sqrtSigma = static_cast<float>(std::sqrt(pb.kernel.sigma));
    E.P.dim = 3;
    E.P.f = to_dev(pb.f);
    E.P.g = to_dev(pb.g);
    E.P.h = to_dev(pb.h);
    double diag = S->host.diagonal;
    double eps = wc.epsilon > 0.0 ? wc.epsilon : 1e-3 * diag;
    double rmin = wc.rMin > 0.0 ? wc.rMin : eps;
    if (rmin > eps) throw Error(BVC_ERR_INVALID_ARGUMENT, "walk config: r_min must lie in (0, epsilon]");
    E.eps = static_cast<float>(eps);
    E.rmin = static_cast<float>(rmin);
    E.tguard = static_cast<float>(1e-9 * diag);
    E.insideTol = S->host.component.empty() || *std::max_element(S->host.component.begin(), S->host.component.end()) == 0
                      ? static_cast<float>(1e-7 * diag) : -1.0f;  // parity is meaningless for soups
    E.scale = static_cast<float>(diag);
    E.nudge = static_cast<float>(9.5367431640625e-7 * diag);
    E.cx = static_cast<float>(0.5 * (S->host.lo[0] + S->host.hi[0]));
    E.cy = static_cast<float>(0.5 * (S->host.lo[1] + S->host.hi[1]));
    E.cz = static_cast<float>(0.5 * (S->host.lo[2] + S->host.hi[2]));
    E.escape = static_cast<float>(diag);
    E.maxSteps = std::max(1, wc.maxSteps);
    E.hasNeumann = S->host.hasNeumann() ? 1 : 0;
    E.hasH = pb.h.kind != BVC_FIELD_NONE ? 1 : 0;
    E.closed = E.insideTol > 0.f ? 1 : 0;
    key_of(seed, salt, round, E.k0, E.k1);
    E.ff = S->farfield();
    return E;
}

void run_cache_walks3(bvc_scene_s* S, bvc_region_s* R, const WalkEnv3& E, const bvc_cache_config& cfg,
                      CacheSample* samples, int n, long long gidBase, const long long* gid, uint8_t* failed,
                      GenStats& st) {
    float4* startU = ws().get<float4>(kWsStartU, n);
    int* isD = ws().get<int>(kWsIsD, n);
    float* gradR = ws().get<float>(kWsGradR, n);
    launch_prepare3(E, samples, n, R->kinds.p, startU, isD, gradR, failed, g_stream);
    int* dIdx = ws().get<int>(kWsDIdx, n);
    int* cnt = ws().get<int>(kWsCount, 1);
    launch_compact(isD, n, dIdx, cnt, g_stream);
    int nD = 0;
    CK(cudaMemcpyAsync(&nD, cnt, sizeof(int), cudaMemcpyDeviceToHost, g_stream));
    CK(cudaStreamSynchronize(g_stream));
    float4* xD = ws().get<float4>(kWsXD, std::max(nD, 1));
    float4* nrmD = ws().get<float4>(kWsND, std::max(nD, 1));
    float* rD = ws().get<float>(kWsRD, std::max(nD, 1));
    long long* gidD = ws().get<long long>(kWsGidD, std::max(nD, 1));
    launch_gather_dpoints3(samples, dIdx, nD, gradR, gidBase, gid, xD, nrmD, rD, gidD, g_stream);
    int nU = std::max(1, cfg.nWalksNeumann), nDw = std::max(1, cfg.nWalksDirichlet);
    int* hintU = ws().get<int>(kWsHintU, std::max(n, 1));
    int* hintD = ws().get<int>(kWsHintD, std::max(nD, 1));
    launch_start_hints(samples, n, R->source.p, S->cls.p, S->leafOf.p, dIdx, nD, hintU, hintD, g_stream);
    WalkJob3 J{};
    J.hintU = hintU;
    J.hintD = hintD;
    J.nU = nU;
    J.nPtsU = n;
    J.startU = startU;
    J.gidU = gid;
    J.gidBaseU = gidBase;
    J.outU = ws().get<float>(kWsOutU, static_cast<size_t>(n) * nU);
    J.nD = nDw;
    J.nPtsD = nD;
    J.xD = xD;
    J.normalD = nrmD;
    J.radiusD = rD;
    J.gidD = gidD;
    J.outD = ws().get<float>(kWsOutD, std::max<size_t>(static_cast<size_t>(nD) * nDw, 1));
    auto* ctr = ws().get<unsigned long long>(kWsCounter, 3);
    CK(cudaMemsetAsync(ctr, 0, 3 * sizeof(unsigned long long), g_stream));
    J.counter = ctr;
    J.steps = ctr + 1;
    J.truncTotal = ctr + 2;
    if (g_profile) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        size_t slots = static_cast<size_t>(sms) * 32 * 256 * 2;
        auto* cc = ws().get<unsigned long long>(kWsEvalOut, slots);
        CK(cudaMemsetAsync(cc, 0, slots * sizeof(unsigned long long), g_stream));
        WalkEnv3 Ec = E;
        Ec.S.counts = cc;
        launch_walk_job3(Ec, J, g_stream);
        std::vector<unsigned long long> h(slots);
        CK(cudaMemcpyAsync(h.data(), cc, slots * sizeof(unsigned long long), cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
        for (size_t i = 0; i < slots; ++i) g_profileTotals[i & 1] += h[i];
    } else {
        launch_walk_job3(E, J, g_stream);
    }
    launch_finish_samples(samples, n, J.outU, nU, dIdx, nD, J.outD, nDw, failed, g_stream);
    unsigned long long h[3];
    CK(cudaMemcpyAsync(h, ctr, sizeof(h), cudaMemcpyDeviceToHost, g_stream));
    CK(cudaStreamSynchronize(g_stream));
    st.walks += static_cast<long long>(n) * nU + static_cast<long long>(nD) * nDw;
    st.steps += static_cast<long long>(h[1]);
    st.truncated += static_cast<long long>(h[2]);
}

void generate_cache3(bvc_scene_s* S, const bvc_problem& pb, bvc_region_s* R, const bvc_cache_config& cfg, uint64_t seed,
                     uint64_t round, int begin, int end, bvc_boundary_cache_s* out, GenStats& st) {
    const int N = std::max(1, cfg.nBoundary);
    const int n = end - begin;
    out->n = n;
    out->dim = 3;
    out->voronoi = 0;
    out->length = R->boundary.total;
    out->samples.resize(std::max(n, 1));
    if (n == 0) return;
    if (cfg.voronoi) throw Error(BVC_ERR_INVALID_ARGUMENT, "Voronoi weights are defined for 2D loops only");
    bvc_scene_s& B = R->boundary;
    uint32_t k0, k1;
    key_of(seed, kBoundaryPosSalt, round, k0, k1);
    launch_sample_mesh(B.cdf.p, B.host.ns, B.total, B.triA.p, B.triB.p, B.triC.p, B.triNormal.p, N, begin, n, nullptr,
                       cfg.stratified, k0, k1, out->samples.p, g_stream);
    WalkEnv3 E = make_env3(S, pb, cfg.walk, seed, kBoundaryWalkSalt, round);
    uint8_t* failed = ws().get<uint8_t>(kWsFailed, n);
    run_cache_walks3(S, R, E, cfg, out->samples.p, n, begin, nullptr, failed, st);
    std::vector<uint8_t> hf(n);
    CK(cudaMemcpyAsync(hf.data(), failed, n, cudaMemcpyDeviceToHost, g_stream));
    CK(cudaStreamSynchronize(g_stream));
    std::vector<int> bad;
    for (int i = 0; i < n; ++i) if (hf[i]) bad.push_back(i);
    WalkEnv3 Er = make_env3(S, pb, cfg.walk, seed, kBoundaryRedrawSalt, round);
    for (int guard = 1; !bad.empty(); ++guard) {
        if (guard > 64) throw Error(BVC_ERR_SOLVER, "boundary cache: sample kept failing after 64 redraws");
        int nb = static_cast<int>(bad.size());
        st.resampled += nb;
        std::vector<long long> hc(nb);
        for (int j = 0; j < nb; ++j) hc[j] = (static_cast<long long>(begin) + bad[j]) * 131 + guard;
        long long* dctr = ws().get<long long>(kWsCtr, nb);
        CK(cudaMemcpyAsync(dctr, hc.data(), nb * sizeof(long long), cudaMemcpyHostToDevice, g_stream));
        CacheSample* tmp = ws().get<CacheSample>(kWsSamplesTmp, nb);
        uint32_t r0, r1;
        key_of(seed, kBoundaryRedrawSalt, round, r0, r1);
        launch_sample_mesh(B.cdf.p, B.host.ns, B.total, B.triA.p, B.triB.p, B.triC.p, B.triNormal.p, N, 0, nb, dctr, 0, r0,
                           r1, tmp, g_stream);
        uint8_t* f2 = ws().get<uint8_t>(kWsSrcFlag, nb);
        run_cache_walks3(S, R, Er, cfg, tmp, nb, 0, dctr, f2, st);
        int* didx = ws().get<int>(kWsDIdx, nb);
        CK(cudaMemcpyAsync(didx, bad.data(), nb * sizeof(int), cudaMemcpyHostToDevice, g_stream));
        redraw_copy_kernel<<<(nb + 127) / 128, 128, 0, g_stream>>>(tmp, didx, nb, out->samples.p);
        count_launch();
        std::vector<uint8_t> hf2(nb);
        CK(cudaMemcpyAsync(hf2.data(), f2, nb, cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
        std::vector<int> still;
        for (int j = 0; j < nb; ++j) if (hf2[j]) still.push_back(bad[j]);
        bad.swap(still);
    }
}

__global__ void redraw_copy_kernel(const CacheSample* src, const int* idx, int n, CacheSample* dst) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) dst[idx[j]] = src[j];
}

// assignVoronoiWeights (cache.cpp:280-297), on the host (rare mode): per region
// loop, each sample's weight is half the arc distance to its two neighbours
void assign_voronoi(bvc_region_s* R, bvc_boundary_cache_s* c) {
    need(c->dim == 2, "Voronoi weights are defined for 2D loops only");
    int n = c->n;
    if (n == 0) return;
    std::vector<CacheSample> hs(n);
    c->samples.download(hs.data(), n);
    CK(cudaStreamSynchronize(g_stream));
    const auto& bh = R->boundary.host;
    std::vector<std::vector<std::pair<double, int>>> per(bh.loopLength.size());
    for (int i = 0; i < n; ++i) per[bh.loop[hs[i].segment]].push_back({hs[i].arc, i});
    for (size_t li = 0; li < per.size(); ++li) {
        auto& e = per[li];
        if (e.empty()) continue;
        std::sort(e.begin(), e.end());
        size_t m = e.size();
        double L = bh.loopLength[li];
        for (size_t k = 0; k < m; ++k) {
            double w;
            if (m == 1) w = L;
            else {
                double prev = k > 0 ? e[k].first - e[k - 1].first : e[0].first + L - e[m - 1].first;
                double next = k + 1 < m ? e[k + 1].first - e[k].first : e[0].first + L - e[m - 1].first;
                w = 0.5 * (prev + next);
            }
            hs[e[k].second].weight = static_cast<float>(w);
        }
    }
    c->samples.upload(hs.data(), n);
    c->voronoi = 1;
}

void generate_cache(bvc_scene_s* S, const bvc_problem& pb, bvc_region_s* R, const bvc_cache_config& cfg, uint64_t seed,
                    uint64_t round, int begin, int end, bvc_boundary_cache_s* out, GenStats& st) {
    require_device();
    need(S && R, "null scene or region");
    R->upload();
    const int N = std::max(1, cfg.nBoundary);
    need(begin >= 0 && begin <= end && end <= N, "shard range outside [0, nBoundary]");
    if (S->host.dim == 3) {
        S->upload();
        generate_cache3(S, pb, R, cfg, seed, round, begin, end, out, st);
        return;
    }
    const int n = end - begin;
    out->n = n;
    out->dim = 2;
    out->voronoi = 0;  // set by assign_voronoi once the whole round is present
    out->length = R->boundary.total;
    out->samples.resize(std::max(n, 1));
    if (n == 0) return;
    bvc_scene_s& B = R->boundary;
    uint32_t k0, k1;
    key_of(seed, kBoundaryPosSalt, round, k0, k1);
    launch_sample_boundary(B.cdf.p, B.cdfIds.p, B.host.ns, B.total, B.segAB.p, B.segNormal.p, B.segArc.p, B.segLen.p, N,
                           begin, n, nullptr, cfg.stratified, k0, k1, out->samples.p, g_stream);
    WalkEnv E = make_env(S, pb, cfg.walk, seed, kBoundaryWalkSalt, round);
    uint8_t* failed = ws().get<uint8_t>(kWsFailed, n);
    run_cache_walks(S, R, E, cfg, out->samples.p, n, begin, nullptr, failed, st);
    // deterministic redraw of failed samples (cache.cpp:365-379): a fresh uniform
    // position per (sample, attempt), walks keyed by the redraw salt
    std::vector<uint8_t> hf(n);
    CK(cudaMemcpyAsync(hf.data(), failed, n, cudaMemcpyDeviceToHost, g_stream));
    CK(cudaStreamSynchronize(g_stream));
    std::vector<int> bad;
    for (int i = 0; i < n; ++i) if (hf[i]) bad.push_back(i);
    WalkEnv Er = make_env(S, pb, cfg.walk, seed, kBoundaryRedrawSalt, round);
    for (int guard = 1; !bad.empty(); ++guard) {
        if (guard > 64) throw Error(BVC_ERR_SOLVER, "boundary cache: sample kept failing after 64 redraws");
        int nb = static_cast<int>(bad.size());
        st.resampled += nb;
        std::vector<long long> hc(nb);
        for (int j = 0; j < nb; ++j) hc[j] = (static_cast<long long>(begin) + bad[j]) * 131 + guard;
        long long* dctr = ws().get<long long>(kWsCtr, nb);
        CK(cudaMemcpyAsync(dctr, hc.data(), nb * sizeof(long long), cudaMemcpyHostToDevice, g_stream));
        CacheSample* tmp = ws().get<CacheSample>(kWsSamplesTmp, nb);
        uint32_t r0, r1;
        key_of(seed, kBoundaryRedrawSalt, round, r0, r1);
        launch_sample_boundary(B.cdf.p, B.cdfIds.p, B.host.ns, B.total, B.segAB.p, B.segNormal.p, B.segArc.p,
                               B.segLen.p, N, 0, nb, dctr, 0, r0, r1, tmp, g_stream);
        uint8_t* f2 = ws().get<uint8_t>(kWsSrcFlag, nb);
        run_cache_walks(S, R, Er, cfg, tmp, nb, 0, dctr, f2, st);
        int* didx = ws().get<int>(kWsDIdx + 0, nb);  // reuse after walks are done
        std::vector<int> hb(bad.begin(), bad.end());
        CK(cudaMemcpyAsync(didx, hb.data(), nb * sizeof(int), cudaMemcpyHostToDevice, g_stream));
        redraw_copy_kernel<<<(nb + 127) / 128, 128, 0, g_stream>>>(tmp, didx, nb, out->samples.p);
        count_launch();
        std::vector<uint8_t> hf2(nb);
        CK(cudaMemcpyAsync(hf2.data(), f2, nb, cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
        std::vector<int> still;
        for (int j = 0; j < nb; ++j) if (hf2[j]) still.push_back(bad[j]);
        bad.swap(still);
    }
    // assignVoronoiWeights needs every sample of the round: a shard leaves it to the
    // caller (distributed.py assigns after the all-gather)
    if (cfg.voronoi && begin == 0 && end == N) assign_voronoi(R, out);
}

// RegionSampler::sample (sampling.cpp:62-108): jittered strata over the bounding
// box, rejection by the device inside test; the last pass keeps a random subset
__global__ void region_propose_kernel(int g, double lo0, double lo1, double ex, double ey, int pass, int stratified,
                                      uint32_t k0, uint32_t k1, float insideTol, bvc_dev::SceneView2 S, float* y,
                                      int* ok, unsigned* prio) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= g * g) return;
    bvc_dev::U4 r = bvc_dev::philox4x32_10(bvc_dev::U4{static_cast<uint32_t>(c), static_cast<uint32_t>(pass), 7u, 0u}, k0, k1);
    double ux = (static_cast<double>(r.x >> 5) * 67108864.0 + (r.y >> 6)) * (1.0 / 9007199254740992.0);
    double uy = (static_cast<double>(r.z >> 5) * 67108864.0 + (r.w >> 6)) * (1.0 / 9007199254740992.0);
    double px, py;
    if (stratified) {
        int cx = c % g, cy = c / g;
        px = lo0 + (cx + ux) / g * ex;
        py = lo1 + (cy + uy) / g * ey;
    } else {
        px = lo0 + ux * ex;
        py = lo1 + uy * ey;
    }
    y[2 * c] = static_cast<float>(px);
    y[2 * c + 1] = static_cast<float>(py);
    ok[c] = bvc_dev::inside(S, static_cast<float>(px), static_cast<float>(py), insideTol) ? 1 : 0;
    bvc_dev::U4 q = bvc_dev::philox4x32_10(bvc_dev::U4{static_cast<uint32_t>(c), static_cast<uint32_t>(pass), 9u, 0u}, k0, k1);
    prio[c] = q.x;
}

__global__ void source_emit_kernel(const float* y, const int* idx, int n, int base, float pdf, bvc_dev::DevField f,
                                   SourceSampleDev* out) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int c = idx[j];
    SourceSampleDev s{};
    s.y[0] = y[2 * c];
    s.y[1] = y[2 * c + 1];
    s.pdf = pdf;
    s.f = bvc_dev::field_eval(f, s.y[0], s.y[1]);
    out[base + j] = s;
}

void generate_source(const bvc_problem& pb, bvc_region_s* R, const bvc_cache_config& cfg, uint64_t seed, uint64_t round,
                     bvc_source_cache_s* out) {
    require_device();
    R->upload();
    bvc_scene_s& B = R->boundary;
    if (B.host.dim == 3) {  // no 3D source path (sampleBallGreens is 2D-only, kernels.cpp:98-99)
        out->dim = 3;
        out->area = bvc_host::meshVolume(B.host);
        out->m = 0;
        if (pb.f.kind != BVC_FIELD_NONE) throw Error(BVC_ERR_SOLVER, "3D source caches are not supported");
        return;
    }
    out->dim = 2;
    out->area = bvc_host::loopArea(B.host);
    if (!B.host.closed()) throw Error(BVC_ERR_PARSE, "region sampler requires closed loops");
    if (out->area <= 0.0) throw Error(BVC_ERR_PARSE, "region sampler: non-positive area");
    if (pb.f.kind == BVC_FIELD_NONE) {
        out->m = 0;
        return;
    }
    const int M = std::max(1, cfg.nSource);
    out->m = M;
    out->samples.resize(M);
    int g = std::max(1, static_cast<int>(std::ceil(std::sqrt(static_cast<double>(M)))));
    int cells = cfg.stratified ? g * g : M;
    if (!cfg.stratified) g = static_cast<int>(std::ceil(std::sqrt(static_cast<double>(cells))));
    float* y = ws().get<float>(kWsSrcTmp, 2 * static_cast<size_t>(g) * g);
    int* ok = ws().get<int>(kWsIsD, static_cast<size_t>(g) * g);
    unsigned* prio = ws().get<unsigned>(kWsSortKeysIn, static_cast<size_t>(g) * g);
    int* idx = ws().get<int>(kWsDIdx, static_cast<size_t>(g) * g);
    int* cnt = ws().get<int>(kWsCount, 1);
    uint32_t k0, k1;
    key_of(seed, kSourceSalt, round, k0, k1);
    const auto& h = B.host;
    double ex = h.hi[0] - h.lo[0], ey = h.hi[1] - h.lo[1];
    float tol = static_cast<float>(1e-7 * h.diagonal);
    bvc_dev::SceneView2 SV = B.view();
    bvc_dev::DevField f = to_dev(pb.f);
    long long proposals = 0;
    int accepted = 0;
    for (int pass = 0; accepted < M; ++pass) {
        int nc = g * g;
        region_propose_kernel<<<(nc + 127) / 128, 128, 0, g_stream>>>(g, h.lo[0], h.lo[1], ex, ey, pass,
                                                                      cfg.stratified, k0, k1, tol, SV, y, ok, prio);
        count_launch();
        launch_compact(ok, nc, idx, cnt, g_stream);
        int na = 0;
        CK(cudaMemcpyAsync(&na, cnt, sizeof(int), cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
        proposals += nc;
        if (proposals >= 1000000 && accepted + na < proposals / 10000)
            throw Error(BVC_ERR_PARSE, "degenerate region: rejection acceptance rate below 1e-4");
        int take = std::min(na, M - accepted);
        if (take < na) {  // final pass: a random subset (a shuffled visiting order)
            std::vector<int> hidx(na);
            std::vector<unsigned> hp(static_cast<size_t>(nc));
            CK(cudaMemcpyAsync(hidx.data(), idx, na * sizeof(int), cudaMemcpyDeviceToHost, g_stream));
            CK(cudaMemcpyAsync(hp.data(), prio, nc * sizeof(unsigned), cudaMemcpyDeviceToHost, g_stream));
            CK(cudaStreamSynchronize(g_stream));
            std::stable_sort(hidx.begin(), hidx.end(), [&](int a, int b) { return hp[a] < hp[b]; });
            hidx.resize(take);
            std::sort(hidx.begin(), hidx.end());
            CK(cudaMemcpyAsync(idx, hidx.data(), take * sizeof(int), cudaMemcpyHostToDevice, g_stream));
        }
        source_emit_kernel<<<(take + 127) / 128, 128, 0, g_stream>>>(y, idx, take, accepted, static_cast<float>(1.0 / out->area), f,
                                                                     out->samples.p);
        count_launch();
        accepted += take;
    }
}

int gather_kind(const bvc_kernel_spec& k) {
    bool scr = k.kind == BVC_KERNEL_SCREENED;
    return k.dim == 2 ? (scr ? kScr2 : kLap2) : (scr ? kScr3 : kLap3);
}

// one gather launch over [begin, end) of the active points; mode = SplatMode bits
// (gather.cu) for the clamped / ball-kernel variants (value only)
void splat_launch(bvc_boundary_cache_s* b, bvc_source_cache_s* s, bvc_eval_points_s* P, const bvc_splat_config& cfg,
                  size_t begin, size_t end, bool val, bool grad, int mode, double clamp) {
    int dim = cfg.kernel.dim;
    int N = b ? b->n : 0, M = s ? s->m : 0;
    size_t Ka = static_cast<size_t>(P->active);
    end = std::min(end, Ka);
    if (begin >= end) return;
    int K = static_cast<int>(end - begin);
    int kind = gather_kind(cfg.kernel);
    if (cfg.fp64) {  // FP64 variant (gather64.cu)
        double4* pack64 = ws().get<double4>(kWsPack, 2 * static_cast<size_t>(std::max(N + M, 1)));
        if (N) pack64_boundary(b->samples.p, N, kind, cfg.voronoi, pack64, g_stream);
        if (M) pack64_source(s->samples.p, M, kind, pack64 + 2 * static_cast<size_t>(N), g_stream);
        GatherPlan plan = plan_gather64(kind, K, N, M, val, grad);
        double* part = ws().get<double>(kWsPart, std::max<size_t>(static_cast<size_t>(plan.chunksB + plan.chunksS) * plan.comps * K, 1));
        int* skipB = ws().get<int>(kWsSkipB, K);
        int* skipS = ws().get<int>(kWsSkipS, K);
        CK(cudaMemsetAsync(skipB, 0, K * sizeof(int), g_stream));
        CK(cudaMemsetAsync(skipS, 0, K * sizeof(int), g_stream));
        double* px64 = ws().get<double>(kWsXs64, static_cast<size_t>(dim) * K);
        gather_points64(P->x.p, P->order.p + begin, K, dim, px64, g_stream);
        if (N + M > 0) {
            launch_gather64(kind, plan, pack64, N, M, px64, K, dim, cfg.coincidenceTol, val, grad, part, skipB, skipS,
                            ws().get<unsigned>(kWsUnitCtr, 1), g_stream);
            launch_finalize(part, plan, K, P->order.p + begin, N, M, val, grad, dim, skipB, skipS, P->dev(), g_stream);
        }
        CK(cudaGetLastError());
        return;
    }
    float4* pack = ws().get<float4>(kWsPack, 2 * static_cast<size_t>(std::max(N + M, 1)));
    if (N) pack_boundary(b->samples.p, N, kind, cfg.voronoi, pack, g_stream);
    if (M) pack_source(s->samples.p, M, kind, pack + 2 * static_cast<size_t>(N), g_stream);
    GatherPlan plan = plan_gather(kind, K, N, M, val, grad);
    double* part = ws().get<double>(kWsPart, std::max<size_t>(static_cast<size_t>(plan.chunksB + plan.chunksS) * plan.comps * K, 1));
    int* skipB = ws().get<int>(kWsSkipB, K);
    int* skipS = ws().get<int>(kWsSkipS, K);
    CK(cudaMemsetAsync(skipB, 0, K * sizeof(int), g_stream));
    CK(cudaMemsetAsync(skipS, 0, K * sizeof(int), g_stream));
    float* ballRs = nullptr;
    if (mode & kModeBall) {
        ballRs = ws().get<float>(kWsBallRs, K);
        launch_gather_f32(P->ballR.p, P->order.p + begin, K, ballRs, g_stream);
    }
    if (N + M > 0)
        launch_gather(kind, plan, pack, N, M, P->xs.p + static_cast<size_t>(dim) * begin, K, dim,
                      static_cast<float>(cfg.kernel.sigma), static_cast<float>(cfg.coincidenceTol), val, grad, part,
                      skipB, skipS, ws().get<float4>(kWsTileBox, 2 * static_cast<size_t>((N + 255) / 256 + (M + 255) / 256 + 1)),
                      ws().get<unsigned>(kWsUnitCtr, 1), g_stream, mode, static_cast<float>(clamp), ballRs);
    else
        CK(cudaMemsetAsync(part, 0, sizeof(double), g_stream));
    if (N + M > 0)
        launch_finalize(part, plan, K, P->order.p + begin, N, M, val, grad, dim, skipB, skipS, P->dev(), g_stream);
    CK(cudaGetLastError());
}

// requireBallRadius (cache.cpp:418-423)
void require_ball(bvc_eval_points_s* P) {
    if (!P->ballValid)
        throw Error(BVC_ERR_SOLVER, "ball-kernel mode: evaluation point has no ball radius "
                                    "(markEvaluationPoints not applied)");
}

// splatSolution / splatGradient (cache.cpp:426-497), optionally with the boundary
// dG/dn clamped (mode bits) as in correctedBoundarySplat's first loop
void splat(bvc_boundary_cache_s* b, bvc_source_cache_s* s, bvc_eval_points_s* P, const bvc_splat_config& cfg,
           size_t begin, size_t end, bool val, bool grad, int mode = 0, double clamp = 0.0) {
    require_device();
    need(P != nullptr, "null evaluation points");
    validate_kernel(cfg.kernel);
    int dim = cfg.kernel.dim;
    need(P->dim == dim, "evaluation points and kernel differ in dimension");
    need(!b || b->dim == dim, "boundary cache dimension mismatch");
    need(!s || s->dim == dim, "source cache dimension mismatch");
    if (cfg.useBallGreens && val) {
        if (cfg.kernel.kind != BVC_KERNEL_POISSON || dim != 2)
            throw Error(BVC_ERR_SOLVER, "ball-kernel source mode requires the 2D Poisson kernel");
        mode |= kModeBall;
    }
    if (mode && dim != 2) throw Error(BVC_ERR_INVALID_ARGUMENT, "clamped / ball-kernel splats are 2D (cache.cpp:499-597)");
    if (cfg.fp64 && (cfg.kernel.kind != BVC_KERNEL_POISSON || mode))
        throw Error(BVC_ERR_INVALID_ARGUMENT, "fp64 splats: plain Poisson kernels only");
    ensure_order(P);
    if (mode & kModeBall) require_ball(P);
    if (val && grad && mode) {  // the gradient splat never clamps (cache.cpp:463-497)
        splat_launch(b, s, P, cfg, begin, end, true, false, mode, clamp);
        splat_launch(b, s, P, cfg, begin, end, false, true, 0, 0.0);
    } else {
        splat_launch(b, s, P, cfg, begin, end, val, grad, val ? mode : 0, clamp);
    }
}

// correctedBoundarySplat (cache.cpp:499-553)
void corrected_boundary(bvc_boundary_cache_s* b, bvc_eval_points_s* P, bvc_region_s* R, const bvc_splat_config& cfg,
                        double clamp, int mode, const bvc_boundary_evaluator* ev, uint64_t seed, uint64_t stream) {
    require_device();
    need(P && R, "null argument");
    if (mode == BVC_CLAMP_OFF) throw Error(BVC_ERR_INVALID_ARGUMENT, "corrected splat called with clamping off");
    need(mode == BVC_CLAMP_ONLY || mode == BVC_CLAMP_CORRECT, "unknown clamp mode");
    if (!(clamp > 0.0)) throw Error(BVC_ERR_INVALID_ARGUMENT, "clamp bound must be positive");
    bool haveEval = ev && ev->kind != BVC_EVALUATOR_NONE;
    if (mode == BVC_CLAMP_CORRECT && !haveEval)
        throw Error(BVC_ERR_INVALID_ARGUMENT, "clamp correction needs a boundary evaluator");
    need(cfg.kernel.dim == 2, "clamped splats are 2D (cache.cpp:499)");
    splat(b, nullptr, P, cfg, 0, SIZE_MAX, true, false, kModeClampP, clamp);
    if (mode != BVC_CLAMP_CORRECT) return;
    int K = P->active;
    if (K == 0) return;
    R->upload();
    int N = b ? b->n : 0;
    CorrRayEnv E{};
    E.region = R->boundary.view();
    E.kinds = R->kinds.p;
    E.screened = cfg.kernel.kind == BVC_KERNEL_SCREENED ? 1 : 0;
    E.sqrtSigma = std::sqrt(cfg.kernel.sigma);
    E.clamp = clamp;
    E.tol2 = cfg.coincidenceTol * cfg.coincidenceTol;
    E.nRound = static_cast<double>(N);
    E.insideTol = static_cast<float>(1e-7 * R->boundary.host.diagonal);
    key_of(seed, stream, 0, E.k0, E.k1);
    int* noHit = ws().get<int>(kWsCorrFlag, 1);
    CK(cudaMemsetAsync(noHit, 0, sizeof(int), g_stream));
    auto check_hits = [&]() {
        int h = 0;
        CK(cudaMemcpyAsync(&h, noHit, sizeof(int), cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
        if (h) throw Error(BVC_ERR_SOLVER, "clamp correction: no boundary ray hits from an interior point");
    };
    if (ev->kind == BVC_EVALUATOR_FIELD) {
        E.useField = 1;
        E.field = to_dev(ev->field);
        launch_corr_rays(E, P->x.p, P->order.p, K, nullptr, P->bsum.p, noHit, g_stream);
        check_hits();
        return;
    }
    need(ev->kind == BVC_EVALUATOR_WALKS && ev->scene && ev->problem && ev->cfg,
         "walk evaluator needs scene, problem and cache config");
    need(ev->scene->host.dim == 2, "walk evaluator scene must be 2D");
    // makeDefaultEvaluator (cache.cpp:600-620): correctionWalks WoSt walks per crossing
    WalkEnv W = make_env(ev->scene, *ev->problem, ev->cfg->walk, seed, stream, 1);
    E.eps = W.eps;
    int* counts = ws().get<int>(kWsCorrCounts, K);
    int* offsets = ws().get<int>(kWsCorrOffsets, K);
    launch_corr_rays(E, P->x.p, P->order.p, K, counts, nullptr, noHit, g_stream);
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, counts, offsets, K, g_stream));
    CK(cub::DeviceScan::ExclusiveSum(ws().get<char>(kWsCorrScan, tmp), tmp, counts, offsets, K, g_stream));
    count_launch();
    int last[2] = {0, 0};
    CK(cudaMemcpyAsync(&last[0], offsets + K - 1, sizeof(int), cudaMemcpyDeviceToHost, g_stream));
    CK(cudaMemcpyAsync(&last[1], counts + K - 1, sizeof(int), cudaMemcpyDeviceToHost, g_stream));
    check_hits();
    int H = last[0] + last[1];
    if (H == 0) return;
    float2* starts = ws().get<float2>(kWsCorrStarts, H);
    long long* gid = ws().get<long long>(kWsCorrGid, H);
    double* w = ws().get<double>(kWsCorrW, H);
    launch_corr_emit(E, P->x.p, P->order.p, K, offsets, starts, gid, w, g_stream);
    int nw = std::max(1, ev->cfg->correctionWalks);
    auto* ctr = ws().get<unsigned long long>(kWsCounter, 3);
    CK(cudaMemsetAsync(ctr, 0, 3 * sizeof(unsigned long long), g_stream));
    WalkJob J{};
    J.counter = ctr;
    J.nU = nw;
    J.nPtsU = H;
    J.startU = starts;
    J.gidU = gid;
    J.outU = ws().get<float>(kWsCorrOut, static_cast<size_t>(H) * nw);
    launch_walk_job(W, J, g_stream);
    double* mean = ws().get<double>(kWsCorrMean, H);
    launch_reduce_estimates(J.outU, H, nw, 1, 0, mean, nullptr, g_stream);
    launch_corr_apply(offsets, counts, P->order.p, K, w, mean, E.nRound, P->bsum.p, g_stream);
    CK(cudaGetLastError());
}

// correctedSourceSplat (cache.cpp:555-597)
void corrected_source(bvc_source_cache_s* s, bvc_eval_points_s* P, bvc_region_s* R, const bvc_splat_config& cfg,
                      double clamp, const bvc_field* f, uint64_t seed, uint64_t stream) {
    require_device();
    need(P && R, "null argument");
    if (cfg.kernel.kind != BVC_KERNEL_POISSON || cfg.kernel.dim != 2)
        throw Error(BVC_ERR_SOLVER, "ball-kernel source mode requires the 2D Poisson kernel");
    if (!(clamp > 0.0)) throw Error(BVC_ERR_INVALID_ARGUMENT, "clamp bound must be positive");
    need(P->dim == 2, "evaluation points must be 2D");
    ensure_order(P);
    require_ball(P);
    bvc_splat_config c = cfg;
    c.useBallGreens = 1;
    splat(nullptr, s, P, c, 0, SIZE_MAX, true, false, kModeClampS, clamp);
    int K = P->active;
    if (!(std::isfinite(clamp) && f && f->kind != BVC_FIELD_NONE) || K == 0) return;
    R->upload();
    uint32_t k0, k1;
    key_of(seed, stream, 0, k0, k1);
    launch_ball_corr(R->boundary.view(), static_cast<float>(1e-7 * R->boundary.host.diagonal), P->x.p, P->order.p,
                     P->ballR.p, K, to_dev(*f), clamp, static_cast<double>(s ? s->m : 0), k0, k1, P->ssum.p, g_stream);
    CK(cudaGetLastError());
}

// Andrew's monotone chain; the farthest vertex from any point is a hull vertex
std::vector<double> convex_hull2(const std::vector<double>& v) {
    size_t n = v.size() / 2;
    std::vector<std::pair<double, double>> p(n);
    for (size_t i = 0; i < n; ++i) p[i] = {v[2 * i], v[2 * i + 1]};
    std::sort(p.begin(), p.end());
    p.erase(std::unique(p.begin(), p.end()), p.end());
    if (p.size() < 3) {
        std::vector<double> out;
        for (auto& q : p) { out.push_back(q.first); out.push_back(q.second); }
        return out;
    }
    auto cross = [](const std::pair<double, double>& o, const std::pair<double, double>& a,
                    const std::pair<double, double>& b) {
        return (a.first - o.first) * (b.second - o.second) - (a.second - o.second) * (b.first - o.first);
    };
    std::vector<std::pair<double, double>> h(2 * p.size());
    size_t k = 0;
    for (size_t i = 0; i < p.size(); ++i) {
        while (k >= 2 && cross(h[k - 2], h[k - 1], p[i]) <= 0) --k;
        h[k++] = p[i];
    }
    for (size_t i = p.size() - 1, t = k + 1; i-- > 0;) {
        while (k >= t && cross(h[k - 2], h[k - 1], p[i]) <= 0) --k;
        h[k++] = p[i];
    }
    h.resize(k - 1);
    std::vector<double> out;
    for (auto& q : h) { out.push_back(q.first); out.push_back(q.second); }
    return out;
}

// estimator job over host points (pointwise.h:62-76)
void pointwise(bvc_scene_s* S, const bvc_problem& pb, const double* x, const double* normal, size_t n,
               const bvc_walk_config& cfg, const uint64_t* streams, int mode, double* mean, double* se,
               long long* count, long long* trunc) {
    // mode 0: wos / wost solve, 1: gradient (2 comps), 2: normal derivative
    require_device();
    need(S && x, "null scene or points");
    if (n == 0) return;
    WalkEnv E = make_env(S, pb, cfg, cfg.seed, kPointwiseSalt, 0);
    int nw = std::max(1, cfg.nWalks);
    int ni = static_cast<int>(n);
    std::vector<long long> gid(ni);
    for (int i = 0; i < ni; ++i) {
        uint64_t st = streams ? streams[i] : (ni == 1 ? cfg.stream : bvc_dev::mixKey(cfg.stream, i));
        gid[i] = static_cast<long long>(bvc_dev::mix64(st) >> 1);
    }
    // requireInterior (pointwise.cpp:188-191)
    double* xd = ws().get<double>(kWsEvalIn, 2 * n);
    CK(cudaMemcpyAsync(xd, x, 2 * n * sizeof(double), cudaMemcpyHostToDevice, g_stream));
    if (S->host.closed()) {
        uint8_t* ins = ws().get<uint8_t>(kWsOutside, n);
        launch_inside(E.S, xd, ni, E.insideTol, ins, g_stream);
        std::vector<uint8_t> h(n);
        CK(cudaMemcpyAsync(h.data(), ins, n, cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
        for (size_t i = 0; i < n; ++i)
            if (!h[i]) throw Error(BVC_ERR_SOLVER, "evaluation point lies outside the domain");
    }
    std::vector<float2> hx(n);
    for (size_t i = 0; i < n; ++i) hx[i] = make_float2(static_cast<float>(x[2 * i]), static_cast<float>(x[2 * i + 1]));
    float2* px = ws().get<float2>(kWsStartU, n);
    CK(cudaMemcpyAsync(px, hx.data(), n * sizeof(float2), cudaMemcpyHostToDevice, g_stream));
    long long* dg = ws().get<long long>(kWsGidU, n);
    CK(cudaMemcpyAsync(dg, gid.data(), n * sizeof(long long), cudaMemcpyHostToDevice, g_stream));
    int* tr = ws().get<int>(kWsTruncPt, n);
    CK(cudaMemsetAsync(tr, 0, n * sizeof(int), g_stream));
    auto* ctr = ws().get<unsigned long long>(kWsCounter, 3);
    CK(cudaMemsetAsync(ctr, 0, 3 * sizeof(unsigned long long), g_stream));
    WalkJob J{};
    J.counter = ctr;
    J.steps = ctr + 1;
    J.truncTotal = ctr + 2;
    int comps = 1;
    if (mode == 0) {
        J.nU = nw;
        J.nPtsU = ni;
        J.startU = px;
        J.gidU = dg;
        J.outU = ws().get<float>(kWsOutU, n * nw);
        J.truncU = tr;
    } else {
        // gradientBallRadius: closest point on the whole boundary (pointwise.cpp:217-221)
        double* cpp = ws().get<double>(kWsEvalOut, 2 * n);
        double* cpd = ws().get<double>(kWsMean2, n);
        int* cps = ws().get<int>(kWsSkipB, n);
        double* cpt = ws().get<double>(kWsSe2, n);
        launch_closest(E.S, xd, ni, bvc_dev::kClsAny, cpp, cpd, cps, cpt, g_stream);
        std::vector<double> hd(n);
        CK(cudaMemcpyAsync(hd.data(), cpd, n * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
        std::vector<float> hr(n);
        for (size_t i = 0; i < n; ++i) hr[i] = static_cast<float>(std::max(hd[i], static_cast<double>(E.rmin)));
        float* rD = ws().get<float>(kWsRD, n);
        CK(cudaMemcpyAsync(rD, hr.data(), n * sizeof(float), cudaMemcpyHostToDevice, g_stream));
        J.nD = nw;
        J.nPtsD = ni;
        J.xD = px;
        J.radiusD = rD;
        J.gidD = dg;
        J.truncD = tr;
        if (mode == 2) {
            std::vector<float2> hn(n);
            for (size_t i = 0; i < n; ++i) hn[i] = make_float2(static_cast<float>(normal[2 * i]), static_cast<float>(normal[2 * i + 1]));
            float2* dn = ws().get<float2>(kWsND, n);
            CK(cudaMemcpyAsync(dn, hn.data(), n * sizeof(float2), cudaMemcpyHostToDevice, g_stream));
            J.normalD = dn;
        } else {
            comps = 2;
        }
        J.outD = ws().get<float>(kWsOutD, n * nw * comps);
    }
    launch_walk_job(E, J, g_stream);
    const float* vals = mode == 0 ? J.outU : J.outD;
    double* dm = ws().get<double>(kWsMean, n * comps);
    double* ds = ws().get<double>(kWsSe, n * comps);
    for (int c = 0; c < comps; ++c) launch_reduce_estimates(vals, ni, nw, comps, c, dm + c * n, ds + c * n, g_stream);
    std::vector<double> hm(n * comps), hs(n * comps);
    std::vector<int> ht(n);
    CK(cudaMemcpyAsync(hm.data(), dm, n * comps * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
    CK(cudaMemcpyAsync(hs.data(), ds, n * comps * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
    CK(cudaMemcpyAsync(ht.data(), tr, n * sizeof(int), cudaMemcpyDeviceToHost, g_stream));
    CK(cudaStreamSynchronize(g_stream));
    for (size_t i = 0; i < n; ++i) {
        for (int c = 0; c < comps; ++c) {
            mean[comps * i + c] = hm[c * n + i];
            se[comps * i + c] = hs[c * n + i];
        }
        count[i] = nw;
        trunc[i] = ht[i];
    }
    for (size_t i = 0; i < n * comps; ++i)
        if (!std::isfinite(mean[i])) throw Error(BVC_ERR_SOLVER, "walk cannot terminate: scene has no Dirichlet boundary");
}

// fallback walks of updateSolution (cache.cpp:665-681), accumulated on the device
__global__ void fallback_accumulate_kernel(const int* idx, int n, const double* mean, const double* g0,
                                           const double* g1, int nw, int ngw, const int* trunc, double* walkSum,
                                           long long* walkCount, long long* walkTrunc, double* gws, long long* gwc) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int p = idx[j];
    walkSum[p] += mean[j] * nw;
    walkCount[p] += nw;
    walkTrunc[p] += trunc[j];
    if (g0) {
        gws[2 * p] += g0[j] * ngw;
        gws[2 * p + 1] += g1[j] * ngw;
        gwc[p] += ngw;
    }
}

__global__ void first_ball_radius_kernel(const double* dist, int n, float rmin, float* r) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) r[i] = static_cast<float>(fmax(dist[i], static_cast<double>(rmin)));
}

__global__ void gather_fallback_kernel(const int* idx, int n, const double* x, float2* out, long long* gid) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int p = idx[j];
    out[j] = make_float2(static_cast<float>(x[2 * p]), static_cast<float>(x[2 * p + 1]));
    gid[j] = p;
}

__global__ void gather_fallback3_kernel(const int* idx, int n, const double* x, float4* out, long long* gid,
                                        double* xd) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int p = idx[j];
    out[j] = make_float4(static_cast<float>(x[3 * p]), static_cast<float>(x[3 * p + 1]), static_cast<float>(x[3 * p + 2]), 0.f);
    gid[j] = p;
    xd[3 * j] = x[3 * p];
    xd[3 * j + 1] = x[3 * p + 1];
    xd[3 * j + 2] = x[3 * p + 2];
}

__global__ void radius3_kernel(const double* dist, int n, float rmin, float* r) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) r[j] = fmaxf(static_cast<float>(dist[j]), rmin);
}

__global__ void fallback_accumulate3_kernel(const int* idx, int n, const double* mean, const double* g0,
                                            const double* g1, const double* g2, int nw, const int* trunc,
                                            double* walkSum, long long* walkCount, long long* walkTrunc, double* gws,
                                            long long* gwc) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int p = idx[j];
    walkSum[p] += mean[j] * nw;
    walkCount[p] += nw;
    walkTrunc[p] += trunc[j];
    if (g0) {
        gws[3 * p] += g0[j] * nw;
        gws[3 * p + 1] += g1[j] * nw;
        gws[3 * p + 2] += g2[j] * nw;
        gwc[p] += nw;
    }
}

// fallback-band walks in 3D (the 3D lift of cache.cpp:665-681); the interior check
// runs on the device, failures are reported after the walks
void fallback_walks3(bvc_scene_s* S, const bvc_problem& pb, const bvc_cache_config& cfg, bvc_eval_points_s* P,
                     uint64_t seed, uint64_t round, bool gradients) {
    int nf = static_cast<int>(P->n) - P->active;
    const int* idx = P->order.p + P->active;
    int nw = std::max(1, cfg.walk.nWalks);
    float4* px = ws().get<float4>(kWsStartU, nf);
    long long* gid = ws().get<long long>(kWsGidU, nf);
    double* xd = ws().get<double>(kWsEvalIn, 3 * static_cast<size_t>(nf));
    gather_fallback3_kernel<<<(nf + 127) / 128, 128, 0, g_stream>>>(idx, nf, P->x.p, px, gid, xd);
    count_launch();
    WalkEnv3 E = make_env3(S, pb, cfg.walk, seed, kFallbackSalt, round);
    auto* ctr = ws().get<unsigned long long>(kWsCounter, 3);
    int* tr = ws().get<int>(kWsTruncPt, nf);
    CK(cudaMemsetAsync(tr, 0, nf * sizeof(int), g_stream));
    CK(cudaMemsetAsync(ctr, 0, 3 * sizeof(unsigned long long), g_stream));
    WalkJob3 J{};
    J.counter = ctr;
    J.nU = nw;
    J.nPtsU = nf;
    J.startU = px;
    J.gidU = gid;
    J.outU = ws().get<float>(kWsOutU, static_cast<size_t>(nf) * nw);
    J.truncU = tr;
    launch_walk_job3(E, J, g_stream);
    double* dm = ws().get<double>(kWsMean, nf);
    launch_reduce_estimates(J.outU, nf, nw, 1, 0, dm, nullptr, g_stream);
    double *g0 = nullptr, *g1 = nullptr, *g2 = nullptr;
    if (gradients) {
        WalkEnv3 Eg = make_env3(S, pb, cfg.walk, seed, kFallbackGradSalt, round);
        double* cpp = ws().get<double>(kWsEvalOut, 3 * static_cast<size_t>(nf));
        double* cpd = ws().get<double>(kWsMean2, nf);
        int* cps = ws().get<int>(kWsSkipB, nf);
        launch_closest3(Eg.S, xd, nf, bvc_dev::kClsAny, cpp, cpd, cps, g_stream);
        float* rD = ws().get<float>(kWsRD, nf);
        radius3_kernel<<<(nf + 127) / 128, 128, 0, g_stream>>>(cpd, nf, Eg.rmin, rD);
        count_launch();
        CK(cudaMemsetAsync(ctr, 0, 3 * sizeof(unsigned long long), g_stream));
        WalkJob3 G{};
        G.counter = ctr;
        G.nD = nw;
        G.nPtsD = nf;
        G.xD = px;
        G.radiusD = rD;
        G.gidD = gid;
        G.outD = ws().get<float>(kWsOutD, static_cast<size_t>(nf) * nw * 3);
        launch_walk_job3(Eg, G, g_stream);
        g0 = ws().get<double>(kWsSe, 3 * static_cast<size_t>(nf));
        g1 = g0 + nf;
        g2 = g1 + nf;
        for (int c = 0; c < 3; ++c) launch_reduce_estimates(G.outD, nf, nw, 3, c, g0 + c * nf, nullptr, g_stream);
    }
    fallback_accumulate3_kernel<<<(nf + 127) / 128, 128, 0, g_stream>>>(idx, nf, dm, g0, g1, g2, nw, tr, P->walkSum.p,
                                                                        P->walkCount.p, P->walkTrunc.p,
                                                                        P->gwalkSum.p, P->gwalkCount.p);
    count_launch();
}

void fallback_walks(bvc_scene_s* S, const bvc_problem& pb, const bvc_cache_config& cfg, bvc_eval_points_s* P,
                    uint64_t seed, uint64_t round, bool gradients) {
    ensure_order(P);
    int nf = static_cast<int>(P->n) - P->active;
    if (nf <= 0) return;
    if (S->host.dim == 3) {
        fallback_walks3(S, pb, cfg, P, seed, round, gradients);
        return;
    }
    const int* idx = P->order.p + P->active;
    int nw = std::max(1, cfg.walk.nWalks);
    float2* px = ws().get<float2>(kWsStartU, nf);
    long long* gid = ws().get<long long>(kWsGidU, nf);
    gather_fallback_kernel<<<(nf + 127) / 128, 128, 0, g_stream>>>(idx, nf, P->x.p, px, gid);
    count_launch();
    if (S->host.closed()) {  // requireInterior
        WalkEnv E0 = make_env(S, pb, cfg.walk, seed, kFallbackSalt, round);
        double* xd = ws().get<double>(kWsEvalIn, 2 * static_cast<size_t>(nf));
        gather_points64(P->x.p, idx, nf, 2, xd, g_stream);  // positions of the fallback points
        uint8_t* ins = ws().get<uint8_t>(kWsOutside, nf);
        launch_inside(E0.S, xd, nf, E0.insideTol, ins, g_stream);
        std::vector<uint8_t> h(nf);
        CK(cudaMemcpyAsync(h.data(), ins, nf, cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
        for (int j = 0; j < nf; ++j)
            if (!h[j]) throw Error(BVC_ERR_SOLVER, "evaluation point lies outside the domain");
    }
    auto* ctr = ws().get<unsigned long long>(kWsCounter, 3);
    int* tr = ws().get<int>(kWsTruncPt, nf);
    CK(cudaMemsetAsync(tr, 0, nf * sizeof(int), g_stream));
    CK(cudaMemsetAsync(ctr, 0, 3 * sizeof(unsigned long long), g_stream));
    WalkEnv E = make_env(S, pb, cfg.walk, seed, kFallbackSalt, round);
    WalkJob J{};
    J.counter = ctr;
    J.nU = nw;
    J.nPtsU = nf;
    J.startU = px;
    J.gidU = gid;
    J.outU = ws().get<float>(kWsOutU, static_cast<size_t>(nf) * nw);
    J.truncU = tr;
    launch_walk_job(E, J, g_stream);
    double* dm = ws().get<double>(kWsMean, nf);
    launch_reduce_estimates(J.outU, nf, nw, 1, 0, dm, nullptr, g_stream);
    double *g0 = nullptr, *g1 = nullptr;
    if (gradients) {
        WalkEnv Eg = make_env(S, pb, cfg.walk, seed, kFallbackGradSalt, round);
        double* xd = ws().get<double>(kWsEvalIn, 2 * static_cast<size_t>(nf));
        gather_points64(P->x.p, idx, nf, 2, xd, g_stream);
        double* cpp = ws().get<double>(kWsEvalOut, 2 * static_cast<size_t>(nf));
        double* cpd = ws().get<double>(kWsMean2, nf);
        int* cps = ws().get<int>(kWsSkipB, nf);
        double* cpt = ws().get<double>(kWsSe2, nf);
        launch_closest(Eg.S, xd, nf, bvc_dev::kClsAny, cpp, cpd, cps, cpt, g_stream);
        float* rD = ws().get<float>(kWsRD, nf);
        first_ball_radius_kernel<<<(nf + 127) / 128, 128, 0, g_stream>>>(cpd, nf, Eg.rmin, rD);  // pointwise.cpp:217-221
        count_launch();
        CK(cudaMemsetAsync(ctr, 0, 3 * sizeof(unsigned long long), g_stream));
        WalkJob G{};
        G.counter = ctr;
        G.nD = nw;
        G.nPtsD = nf;
        G.xD = px;
        G.radiusD = rD;
        G.gidD = gid;
        G.outD = ws().get<float>(kWsOutD, static_cast<size_t>(nf) * nw * 2);
        launch_walk_job(Eg, G, g_stream);
        g0 = ws().get<double>(kWsSe, nf);
        g1 = ws().get<double>(kWsMean2, nf);
        launch_reduce_estimates(G.outD, nf, nw, 2, 0, g0, nullptr, g_stream);
        launch_reduce_estimates(G.outD, nf, nw, 2, 1, g1, nullptr, g_stream);
    }
    fallback_accumulate_kernel<<<(nf + 127) / 128, 128, 0, g_stream>>>(idx, nf, dm, g0, g1, nw, nw, tr, P->walkSum.p,
                                                                       P->walkCount.p, P->walkTrunc.p, P->gwalkSum.p,
                                                                       P->gwalkCount.p);
    count_launch();
}

bvc_splat_config make_splat_config(bvc_scene_s* S, const bvc_problem& pb, const bvc_cache_config& cfg) {
    validate_kernel(pb.kernel);
    bvc_splat_config s{};
    s.kernel = pb.kernel;
    s.kernel.scale = S->host.diagonal;
    s.coincidenceTol = 1e-12 * S->host.diagonal;
    s.voronoi = cfg.voronoi;
    s.useBallGreens = cfg.sourceBall;
    if (s.useBallGreens && s.kernel.kind != BVC_KERNEL_POISSON)
        throw Error(BVC_ERR_SOLVER, "ball-kernel source mode requires the Poisson kernel");
    return s;
}

void alloc_points(bvc_eval_points_s* P) {
    size_t n = std::max<size_t>(P->n, 1);
    int d = P->dim;
    P->x.resize(d * n);
    P->fallback.resize(n);
    P->unreliable.resize(n);
    P->bsum.resize(n); P->ssum.resize(n); P->bgsum.resize(d * n); P->sgsum.resize(d * n);
    P->walkSum.resize(n); P->gwalkSum.resize(d * n);
    P->nb.resize(n); P->ms.resize(n); P->nbg.resize(n); P->msg.resize(n);
    P->walkCount.resize(n); P->walkTrunc.resize(n); P->gwalkCount.resize(n); P->skipped.resize(n);
    P->ballR.resize(n);
}

void zero_points(bvc_eval_points_s* P) {
    P->fallback.zero(); P->unreliable.zero();
    P->bsum.zero(); P->ssum.zero(); P->bgsum.zero(); P->sgsum.zero(); P->walkSum.zero(); P->gwalkSum.zero();
    P->nb.zero(); P->ms.zero(); P->nbg.zero(); P->msg.zero(); P->walkCount.zero(); P->walkTrunc.zero();
    P->gwalkCount.zero(); P->skipped.zero();
    P->ballR.zero();
    P->ballValid = false;
}

// EvaluationPoint::solution() / gradient() (cache.h:91-105)
__global__ void solution_kernel(int n, int d, const uint8_t* fb, const double* bsum, const double* ssum,
                                const long long* nb, const long long* ms, const double* bgsum, const double* sgsum,
                                const long long* nbg, const long long* msg, const double* walkSum,
                                const long long* walkCount, const double* gws, const long long* gwc, double* u,
                                double* g) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (fb[i]) {
        u[i] = walkCount[i] > 0 ? walkSum[i] / walkCount[i] : 0.0;
        for (int k = 0; k < d; ++k) g[static_cast<size_t>(d) * i + k] = gwc[i] > 0 ? gws[static_cast<size_t>(d) * i + k] / gwc[i] : 0.0;
        return;
    }
    double v = nb[i] > 0 ? bsum[i] / nb[i] : 0.0;
    if (ms[i] > 0) v += ssum[i] / ms[i];
    u[i] = v;
    for (int k = 0; k < d; ++k) {
        size_t j = static_cast<size_t>(d) * i + k;
        double w = nbg[i] > 0 ? bgsum[j] / nbg[i] : 0.0;
        if (msg[i] > 0) w += sgsum[j] / msg[i];
        g[j] = w;
    }
}

__global__ void mark_kernel(const bvc_dev::SceneView2 scene, const bvc_dev::SceneView2 region, const double* x, int n,
                            float offset, int whole, uint8_t* fb, uint8_t* gu) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float px = static_cast<float>(x[2 * i]), py = static_cast<float>(x[2 * i + 1]);
    // fallbackBand cache.cpp:131-135: whole-domain points within l of the Dirichlet boundary
    // both tests only ask "closer than l": queries bounded by l prune everything farther
    const float l2 = offset * offset;
    uint8_t f = 0;
    if (whole) {
        bvc_dev::Closest c = bvc_dev::closest_point(scene, px, py, bvc_dev::kClsD, l2);
        f = c.seg >= 0 ? 1 : 0;
    }
    bvc_dev::Closest r = bvc_dev::closest_point(region, px, py, bvc_dev::kClsAny, l2);
    fb[i] = f;
    gu[i] = r.seg >= 0 ? 1 : 0;
}


// markEvaluationPoints (cache.cpp:263-276)
void mark_points(bvc_scene_s* s, bvc_region_s* r, const bvc_cache_config& cfg, bvc_eval_points_s* p) {
    require_device();
    need(p->dim == s->host.dim, "markEvaluationPoints: point and scene dimensions differ");
    r->upload();
    if (cfg.sourceBall) {  // cache.cpp:268-274
        need(s->host.dim == 2, "ball-kernel mode is 2D only", BVC_ERR_SOLVER);
        std::vector<double> hull = convex_hull2(r->host.boundary.v);
        double* dh = ws().get<double>(kWsHull, std::max<size_t>(hull.size(), 2));
        CK(cudaMemcpyAsync(dh, hull.data(), hull.size() * sizeof(double), cudaMemcpyHostToDevice, g_stream));
        launch_ball_radius(p->x.p, static_cast<int>(p->n), 2, dh, static_cast<int>(hull.size() / 2), p->ballR.p,
                           g_stream);
        CK(cudaStreamSynchronize(g_stream));  // hull is a pageable host buffer
        p->ballValid = !hull.empty();
    }
    int n = static_cast<int>(p->n);
    if (s->host.dim == 3) {
        const auto& comp = r->boundary.host.component;
        bool single = !comp.empty() && *std::max_element(comp.begin(), comp.end()) == 0;
        launch_mark3(s->view3(), r->boundary.view3(), p->x.p, n, static_cast<float>(r->host.offset),
                     r->host.wholeDomain ? 1 : 0, single ? static_cast<float>(1e-7 * r->boundary.host.diagonal) : -1.f,
                     p->fallback.p, p->unreliable.p, g_stream);
    } else if (n) {
        mark_kernel<<<(n + 127) / 128, 128, 0, g_stream>>>(s->view(), r->boundary.view(), p->x.p, n,
                                                           static_cast<float>(r->host.offset), r->host.wholeDomain ? 1 : 0,
                                                           p->fallback.p, p->unreliable.p);
        count_launch();
    }
    p->orderValid = false;
    CK(cudaGetLastError());
}

std::unique_ptr<bvc_eval_points_s> make_points(const double* x, size_t n, int dim) {
    auto P = std::make_unique<bvc_eval_points_s>();
    P->n = n;
    P->dim = dim;
    alloc_points(P.get());
    P->x.upload(x, dim * n);
    zero_points(P.get());
    return P;
}

// The direction field of runStreamlines (runner.cpp:310-329) for a batch of points:
// status 0 ok (g = unit gradient), 1 outside (not evaluable or in the fallback
// band), 2 zero gradient (|grad u| < 1e-12). The gradient is the splatGradient
// of every retained round's caches accumulated into one EvaluationPoint.
struct StreamCaches {
    std::vector<std::unique_ptr<bvc_boundary_cache_s>> b;
    std::vector<std::unique_ptr<bvc_source_cache_s>> s;
};
void stream_directions(bvc_scene_s* S, bvc_region_s* R, const bvc_cache_config& cfg, const bvc_splat_config& scfg,
                       const StreamCaches& C, const std::vector<double>& x, std::vector<double>& g,
                       std::vector<int>& status) {
    size_t n = x.size() / 2;
    g.assign(2 * n, 0.0);
    status.assign(n, 1);
    if (n == 0) return;
    auto P = make_points(x.data(), n, 2);
    // evaluable (runner.cpp:31-35): inside the scene and, for a subdomain, inside the loop
    float tol = static_cast<float>(1e-7 * S->host.diagonal);
    uint8_t* ins = ws().get<uint8_t>(kWsOutside, 2 * n);
    launch_inside(S->view(), P->x.p, static_cast<int>(n), tol, ins, g_stream);
    if (!R->host.wholeDomain)
        launch_inside(R->boundary.view(), P->x.p, static_cast<int>(n),
                      static_cast<float>(1e-7 * R->boundary.host.diagonal), ins + n, g_stream);
    mark_points(S, R, cfg, P.get());
    std::vector<uint8_t> hin(2 * n, 1), fb(n);
    CK(cudaMemcpyAsync(hin.data(), ins, (R->host.wholeDomain ? 1 : 2) * n, cudaMemcpyDeviceToHost, g_stream));
    P->fallback.download(fb.data(), n);
    CK(cudaStreamSynchronize(g_stream));
    for (size_t i = 0; i < n; ++i) fb[i] = (fb[i] || !hin[i] || !hin[n + i]) ? 1 : 0;
    P->fallback.upload(fb.data(), n);  // excluded from the gather, like the reference's early return
    P->orderValid = false;
    for (size_t r = 0; r < C.b.size(); ++r)
        splat(C.b[r].get(), C.s[r]->m ? C.s[r].get() : nullptr, P.get(), scfg, 0, SIZE_MAX, false, true);
    double* o = ws().get<double>(kWsEvalOut, 3 * n);
    solution_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, g_stream>>>(
        static_cast<int>(n), 2, P->fallback.p, P->bsum.p, P->ssum.p, P->nb.p, P->ms.p, P->bgsum.p, P->sgsum.p,
        P->nbg.p, P->msg.p, P->walkSum.p, P->walkCount.p, P->gwalkSum.p, P->gwalkCount.p, o, o + n);
    count_launch();
    std::vector<double> hg(2 * n);
    CK(cudaMemcpyAsync(hg.data(), o + n, 2 * n * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
    CK(cudaStreamSynchronize(g_stream));
    for (size_t i = 0; i < n; ++i) {
        if (fb[i]) continue;  // outside
        double gx = hg[2 * i], gy = hg[2 * i + 1];
        double nrm = std::sqrt(gx * gx + gy * gy);
        if (nrm < 1e-12) { status[i] = 2; continue; }
        status[i] = 0;
        g[2 * i] = gx / nrm;
        g[2 * i + 1] = gy / nrm;
    }
}

// runStreamlines (runner.cpp:285-373): every seed advances together, so each Heun
// step is two batched gradient gathers (probe and landing) over the retained caches;
// the landing's direction is the next step's k1 (deterministic, so equal to the
// reference's recomputation).
void trace_streamlines(bvc_scene_s* S, const bvc_problem& pb, bvc_region_s* R, const bvc_cache_config& cfg,
                       uint64_t seed, int rounds, const double* seeds, int nSeeds, double h, int steps,
                       double* points, int* counts, int* reasons) {
    require_device();
    need(S->host.dim == 2, "streamlines: 2D scenes only (runner.cpp:285)");
    if (cfg.sourceBall) throw Error(BVC_ERR_INVALID_ARGUMENT, "streamlines: sourceBall mode does not support gradient splats");
    need(nSeeds > 0 && seeds, "streamlines.seeds: required");
    need(h > 0.0, "streamlines.step: expected > 0");
    need(steps >= 1, "streamlines.steps: expected >= 1");
    need(rounds >= 1, "streamlines: rounds must be >= 1");
    bvc_splat_config scfg = make_splat_config(S, pb, cfg);
    StreamCaches C;
    for (int r = 0; r < rounds; ++r) {  // retained caches (runner.cpp:305-308)
        auto b = std::make_unique<bvc_boundary_cache_s>();
        auto s = std::make_unique<bvc_source_cache_s>();
        GenStats st;
        generate_cache(S, pb, R, cfg, seed, r, 0, std::max(1, cfg.nBoundary), b.get(), st);
        generate_source(pb, R, cfg, seed, r, s.get());
        C.b.push_back(std::move(b));
        C.s.push_back(std::move(s));
    }
    const int per = steps + 1;
    std::vector<double> x(seeds, seeds + 2 * static_cast<size_t>(nSeeds)), g;
    std::vector<int> st;
    stream_directions(S, R, cfg, scfg, C, x, g, st);
    std::vector<double> k1(2 * static_cast<size_t>(nSeeds));
    std::vector<int> status(st), active;
    for (int i = 0; i < nSeeds; ++i) {
        counts[i] = 0;
        reasons[i] = BVC_STREAM_OK;
        if (st[i] == 1) { reasons[i] = BVC_STREAM_OUTSIDE; continue; }  // no polyline
        points[2 * static_cast<size_t>(i) * per] = x[2 * i];
        points[2 * static_cast<size_t>(i) * per + 1] = x[2 * i + 1];
        counts[i] = 1;
        k1[2 * i] = g[2 * i];
        k1[2 * i + 1] = g[2 * i + 1];
        active.push_back(i);
    }
    for (int k = 1; k <= steps && !active.empty(); ++k) {
        std::vector<int> go;
        for (int i : active) {
            if (status[i] == 2) reasons[i] = BVC_STREAM_ZERO_GRADIENT;  // k1 = direction(x) failed
            else go.push_back(i);
        }
        if (go.empty()) break;
        std::vector<double> probe(2 * go.size()), gp;
        std::vector<int> sp;
        for (size_t j = 0; j < go.size(); ++j) {
            int i = go[j];
            probe[2 * j] = x[2 * i] + h * k1[2 * i];
            probe[2 * j + 1] = x[2 * i + 1] + h * k1[2 * i + 1];
        }
        stream_directions(S, R, cfg, scfg, C, probe, gp, sp);
        std::vector<double> next(2 * go.size()), gn;
        std::vector<int> sn;
        for (size_t j = 0; j < go.size(); ++j) {
            int i = go[j];
            if (sp[j] == 0) {  // Heun step
                next[2 * j] = x[2 * i] + 0.5 * h * (k1[2 * i] + gp[2 * j]);
                next[2 * j + 1] = x[2 * i + 1] + 0.5 * h * (k1[2 * i + 1] + gp[2 * j + 1]);
            } else {  // the predictor left the region
                next[2 * j] = x[2 * i] + h * k1[2 * i];
                next[2 * j + 1] = x[2 * i + 1] + h * k1[2 * i + 1];
            }
        }
        stream_directions(S, R, cfg, scfg, C, next, gn, sn);
        active.clear();
        for (size_t j = 0; j < go.size(); ++j) {
            int i = go[j];
            if (sn[j] == 1) { reasons[i] = BVC_STREAM_OUTSIDE; continue; }
            x[2 * i] = next[2 * j];
            x[2 * i + 1] = next[2 * j + 1];
            size_t o = 2 * (static_cast<size_t>(i) * per + counts[i]);
            points[o] = x[2 * i];
            points[o + 1] = x[2 * i + 1];
            ++counts[i];
            status[i] = sn[j];
            k1[2 * i] = gn[2 * j];
            k1[2 * i + 1] = gn[2 * j + 1];
            active.push_back(i);
        }
    }
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* bvc_last_error(void) { return g_error.c_str(); }
int bvc_abi_version(void) { return BVC_ABI_VERSION; }
long long bvc_kernel_launch_count(void) { return g_launches.load(); }

int bvc_set_device(int device) { API(require_device(); CK(cudaSetDevice(device))) }
int bvc_set_stream(void* s) { API(g_stream = static_cast<cudaStream_t>(s)) }
int bvc_synchronize(void) { API(require_device(); CK(cudaStreamSynchronize(g_stream))) }

int bvc_scene_create(const double* v, int nv, const int* segs, const int* labels, int ns, bvc_scene* out) {
    API({
        need(out && v && segs && labels, "null argument");
        auto s = std::make_unique<bvc_scene_s>();
        s->host = bvc_host::buildScene2(v, nv, segs, labels, ns);
        *out = s.release();
    })
}
int bvc_scene_create_mesh3(const double* v, int nv, const int* tris, const int* labels, int nt, bvc_scene* out) {
    API({
        need(out && v && tris && labels, "null argument");
        auto s = std::make_unique<bvc_scene_s>();
        s->host = bvc_host::buildMesh3(v, nv, tris, labels, nt);
        *out = s.release();
    })
}
int bvc_scene_destroy(bvc_scene s) { API(delete s) }
int bvc_scene_info(bvc_scene s, int* dim, double* diag, double* lo, double* hi, double* dl, double* nl, int* closed,
                   int* nloops) {
    API({
        need(s, "null scene");
        const auto& h = s->host;
        if (dim) *dim = h.dim;
        if (diag) *diag = h.diagonal;
        for (int k = 0; k < h.dim; ++k) {
            if (lo) lo[k] = h.lo[k];
            if (hi) hi[k] = h.hi[k];
        }
        if (dl) *dl = h.dirichletMeasure;
        if (nl) *nl = h.neumannMeasure;
        if (closed) *closed = h.closed() ? 1 : 0;
        if (nloops) *nloops = static_cast<int>(h.loopLength.size());
    })
}

int bvc_scene_closest_point(bvc_scene s, const double* x, size_t n, int filter, double* point, double* dist, int* seg,
                            double* t) {
    API({
        require_device();
        need(s && x, "null argument");
        if (n == 0) return BVC_OK;
        unsigned mask = filter == BVC_FILTER_DIRICHLET ? bvc_dev::kClsD : filter == BVC_FILTER_NEUMANN ? bvc_dev::kClsNeumann : bvc_dev::kClsAny;
        if (s->host.dim == 3) {  // point: 3n, t: unused (0)
            double* xd3 = ws().get<double>(kWsEvalIn, 3 * n);
            double* o3 = ws().get<double>(kWsEvalOut, 4 * n);
            int* sg3 = ws().get<int>(kWsSkipB, n);
            CK(cudaMemcpyAsync(xd3, x, 3 * n * sizeof(double), cudaMemcpyHostToDevice, g_stream));
            launch_closest3(s->view3(), xd3, static_cast<int>(n), mask, o3, o3 + 3 * n, sg3, g_stream);
            CK(cudaMemcpyAsync(point, o3, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
            CK(cudaMemcpyAsync(dist, o3 + 3 * n, n * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
            CK(cudaMemcpyAsync(seg, sg3, n * sizeof(int), cudaMemcpyDeviceToHost, g_stream));
            CK(cudaStreamSynchronize(g_stream));
            if (t) std::fill(t, t + n, 0.0);
            return BVC_OK;
        }
        double* xd = ws().get<double>(kWsEvalIn, 2 * n);
        double* o = ws().get<double>(kWsEvalOut, 4 * n);
        int* sg = ws().get<int>(kWsSkipB, n);
        CK(cudaMemcpyAsync(xd, x, 2 * n * sizeof(double), cudaMemcpyHostToDevice, g_stream));
        launch_closest(s->view(), xd, static_cast<int>(n), mask, o, o + 2 * n, sg, o + 3 * n, g_stream);
        CK(cudaMemcpyAsync(point, o, 2 * n * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
        CK(cudaMemcpyAsync(dist, o + 2 * n, n * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
        CK(cudaMemcpyAsync(seg, sg, n * sizeof(int), cudaMemcpyDeviceToHost, g_stream));
        CK(cudaMemcpyAsync(t, o + 3 * n, n * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
    })
}
int bvc_scene_silhouette_distance(bvc_scene s, const double* x, size_t n, double* dist) {
    API({
        require_device();
        need(s && x, "null argument");
        if (n == 0) return BVC_OK;
        double* xd = ws().get<double>(kWsEvalIn, 2 * n);
        double* o = ws().get<double>(kWsEvalOut, n);
        CK(cudaMemcpyAsync(xd, x, 2 * n * sizeof(double), cudaMemcpyHostToDevice, g_stream));
        launch_silhouette(s->view(), xd, static_cast<int>(n), o, g_stream);
        CK(cudaMemcpyAsync(dist, o, n * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
    })
}
int bvc_scene_intersect_ray(bvc_scene s, const double* o, const double* d, size_t n, double tMax, int filter,
                            double tMin, double* t, int* seg, double* point, double* sp) {
    API({
        require_device();
        need(s && o && d, "null argument");
        if (n == 0) return BVC_OK;
        unsigned mask = filter == BVC_FILTER_DIRICHLET ? bvc_dev::kClsD : filter == BVC_FILTER_NEUMANN ? bvc_dev::kClsNeumann : bvc_dev::kClsAny;
        double* in = ws().get<double>(kWsEvalIn, 4 * n);
        double* out = ws().get<double>(kWsEvalOut, 4 * n);
        int* sg = ws().get<int>(kWsSkipB, n);
        CK(cudaMemcpyAsync(in, o, 2 * n * sizeof(double), cudaMemcpyHostToDevice, g_stream));
        CK(cudaMemcpyAsync(in + 2 * n, d, 2 * n * sizeof(double), cudaMemcpyHostToDevice, g_stream));
        launch_ray(s->view(), in, in + 2 * n, static_cast<int>(n), tMax, mask, tMin, out, sg, out + n, out + 3 * n, g_stream);
        CK(cudaMemcpyAsync(t, out, n * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
        CK(cudaMemcpyAsync(seg, sg, n * sizeof(int), cudaMemcpyDeviceToHost, g_stream));
        CK(cudaMemcpyAsync(point, out + n, 2 * n * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
        CK(cudaMemcpyAsync(sp, out + 3 * n, n * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
    })
}
int bvc_scene_inside(bvc_scene s, const double* x, size_t n, uint8_t* inside) {
    API({
        require_device();
        need(s && x, "null argument");
        if (n == 0) return BVC_OK;
        int d = s->host.dim;
        double* xd = ws().get<double>(kWsEvalIn, d * n);
        uint8_t* o = ws().get<uint8_t>(kWsOutside, n);
        CK(cudaMemcpyAsync(xd, x, d * n * sizeof(double), cudaMemcpyHostToDevice, g_stream));
        if (d == 3)
            launch_inside3(s->view3(), xd, static_cast<int>(n), static_cast<float>(1e-7 * s->host.diagonal), o, g_stream);
        else
            launch_inside(s->view(), xd, static_cast<int>(n), static_cast<float>(1e-7 * s->host.diagonal), o, g_stream);
        CK(cudaMemcpyAsync(inside, o, n, cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
    })
}

int bvc_region_build(bvc_scene s, const bvc_region_request* req, double eps, bvc_region* out) {
    API({
        need(s && req && out, "null argument");
        auto r = std::make_unique<bvc_region_s>();
        r->host = bvc_host::buildSolveRegion(s->host, req->mode, req->offset, req->subdomain ? &req->subdomain->host : nullptr,
                                             eps);
        r->boundary.host = r->host.boundary;
        *out = r.release();
    })
}
int bvc_region_destroy(bvc_region r) { API(delete r) }
int bvc_region_info(bvc_region r, int* nv, int* ns, double* offset, double* area, int* whole) {
    API({
        need(r, "null region");
        if (nv) *nv = r->host.boundary.nv;
        if (ns) *ns = r->host.boundary.ns;
        if (offset) *offset = r->host.offset;
        if (area) *area = r->host.area;
        if (whole) *whole = r->host.wholeDomain ? 1 : 0;
    })
}
int bvc_region_export(bvc_region r, double* v, int* segs, int* labels, int* kinds, int* src) {
    API({
        need(r, "null region");
        const auto& b = r->host.boundary;
        if (v) std::copy(b.v.begin(), b.v.end(), v);
        if (segs) std::copy(b.idx.begin(), b.idx.end(), segs);
        if (labels) std::copy(b.label.begin(), b.label.end(), labels);
        if (kinds) std::copy(r->host.kinds.begin(), r->host.kinds.end(), kinds);
        if (src) std::copy(r->host.source.begin(), r->host.source.end(), src);
    })
}
bvc_scene bvc_region_boundary(bvc_region r) { return r ? &r->boundary : nullptr; }

int bvc_points_create(const double* x, size_t n, int dim, bvc_eval_points* out) {
    API({
        require_device();
        need(out && (x || n == 0), "null argument");
        need(dim == 2 || dim == 3, "points must be 2D or 3D");
        auto P = std::make_unique<bvc_eval_points_s>();
        P->n = n;
        P->dim = dim;
        alloc_points(P.get());
        P->x.upload(x, dim * n);
        zero_points(P.get());
        CK(cudaStreamSynchronize(g_stream));  // x is read before the call returns (pinned x copies async)
        *out = P.release();
    })
}
int bvc_points_destroy(bvc_eval_points p) { API(delete p) }
int bvc_points_reset(bvc_eval_points p) {
    API({
        require_device();
        need(p, "null points");
        // keep the classification, zero the running sums
        p->bsum.zero(); p->ssum.zero(); p->bgsum.zero(); p->sgsum.zero(); p->walkSum.zero(); p->gwalkSum.zero();
        p->nb.zero(); p->ms.zero(); p->nbg.zero(); p->msg.zero(); p->walkCount.zero(); p->walkTrunc.zero();
        p->gwalkCount.zero(); p->skipped.zero();
    })
}
int bvc_points_download(bvc_eval_points p, bvc_point_state* h) {
    API({
        require_device();
        need(p && h, "null argument");
        size_t n = p->n;
        int d = p->dim;
        h->count = n;
        h->dim = d;
        if (h->x) p->x.download(h->x, static_cast<size_t>(d) * n);
        if (h->fallback) p->fallback.download(h->fallback, n);
        if (h->gradientUnreliable) p->unreliable.download(h->gradientUnreliable, n);
        if (h->boundarySum) p->bsum.download(h->boundarySum, n);
        if (h->sourceSum) p->ssum.download(h->sourceSum, n);
        if (h->nBoundary) p->nb.download(h->nBoundary, n);
        if (h->mSource) p->ms.download(h->mSource, n);
        if (h->boundaryGradSum) p->bgsum.download(h->boundaryGradSum, d * n);
        if (h->sourceGradSum) p->sgsum.download(h->sourceGradSum, d * n);
        if (h->nBoundaryGrad) p->nbg.download(h->nBoundaryGrad, n);
        if (h->mSourceGrad) p->msg.download(h->mSourceGrad, n);
        if (h->walkSum) p->walkSum.download(h->walkSum, n);
        if (h->walkCount) p->walkCount.download(h->walkCount, n);
        if (h->walkTruncated) p->walkTrunc.download(h->walkTruncated, n);
        if (h->gradientWalkSum) p->gwalkSum.download(h->gradientWalkSum, d * n);
        if (h->gradientWalkCount) p->gwalkCount.download(h->gradientWalkCount, n);
        if (h->skipped) p->skipped.download(h->skipped, n);
        if (h->ballRadius) p->ballR.download(h->ballRadius, n);
        CK(cudaStreamSynchronize(g_stream));
    })
}
int bvc_points_solution(bvc_eval_points p, double* u, double* grad) {
    API({
        require_device();
        need(p && (u || grad), "null argument");
        size_t n = p->n;
        if (n == 0) return BVC_OK;
        int d = p->dim;
        double* o = ws().get<double>(kWsEvalOut, (1 + d) * n);
        solution_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, g_stream>>>(
            static_cast<int>(n), d, p->fallback.p, p->bsum.p, p->ssum.p, p->nb.p, p->ms.p, p->bgsum.p, p->sgsum.p,
            p->nbg.p, p->msg.p, p->walkSum.p, p->walkCount.p, p->gwalkSum.p, p->gwalkCount.p, o, o + n);
        count_launch();
        if (u) CK(cudaMemcpyAsync(u, o, n * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
        if (grad) CK(cudaMemcpyAsync(grad, o + n, d * n * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
    })
}

int bvc_points_upload(bvc_eval_points p, const bvc_point_state* h) {
    API({
        require_device();
        need(p && h, "null argument");
        size_t n = p->n;
        int d = p->dim;
        need(h->count == n, "point count mismatch");
        if (h->fallback) { p->fallback.upload(h->fallback, n); p->orderValid = false; }
        if (h->gradientUnreliable) p->unreliable.upload(h->gradientUnreliable, n);
        if (h->boundarySum) p->bsum.upload(h->boundarySum, n);
        if (h->sourceSum) p->ssum.upload(h->sourceSum, n);
        if (h->nBoundary) p->nb.upload(h->nBoundary, n);
        if (h->mSource) p->ms.upload(h->mSource, n);
        if (h->boundaryGradSum) p->bgsum.upload(h->boundaryGradSum, d * n);
        if (h->sourceGradSum) p->sgsum.upload(h->sourceGradSum, d * n);
        if (h->nBoundaryGrad) p->nbg.upload(h->nBoundaryGrad, n);
        if (h->mSourceGrad) p->msg.upload(h->mSourceGrad, n);
        if (h->walkSum) p->walkSum.upload(h->walkSum, n);
        if (h->walkCount) p->walkCount.upload(h->walkCount, n);
        if (h->walkTruncated) p->walkTrunc.upload(h->walkTruncated, n);
        if (h->gradientWalkSum) p->gwalkSum.upload(h->gradientWalkSum, d * n);
        if (h->gradientWalkCount) p->gwalkCount.upload(h->gradientWalkCount, n);
        if (h->skipped) p->skipped.upload(h->skipped, n);
        if (h->ballRadius) {
            p->ballR.upload(h->ballRadius, n);
            // requireBallRadius (cache.cpp:418-423) for every non-fallback point
            std::vector<uint8_t> fb(n);
            p->fallback.download(fb.data(), n);
            CK(cudaStreamSynchronize(g_stream));
            p->ballValid = true;
            for (size_t i = 0; i < n; ++i)
                if (!fb[i] && !(h->ballRadius[i] > 0.0)) p->ballValid = false;
        }
        CK(cudaStreamSynchronize(g_stream));
    })
}
int bvc_mark_evaluation_points(bvc_scene s, bvc_region r, const bvc_cache_config* cfg, bvc_eval_points p) {
    API(need(s && r && cfg && p, "null argument"); mark_points(s, r, *cfg, p))
}

int bvc_trace_streamlines(bvc_scene s, const bvc_problem* pb, bvc_region r, const bvc_cache_config* cfg,
                          uint64_t seed, int rounds, const double* seeds, int nSeeds, double step, int steps,
                          double* points, int* counts, int* reasons) {
    API(need(s && pb && r && cfg && points && counts && reasons, "null argument");
        trace_streamlines(s, *pb, r, *cfg, seed, rounds, seeds, nSeeds, step, steps, points, counts, reasons))
}

int bvc_generate_boundary_cache_shard(bvc_scene s, const bvc_problem* pb, bvc_region r, const bvc_cache_config* cfg,
                                      uint64_t seed, uint64_t round, int begin, int end, bvc_round_stats* stats,
                                      bvc_boundary_cache* out) {
    API({
        need(s && pb && r && cfg && out, "null argument");
        auto c = std::make_unique<bvc_boundary_cache_s>();
        GenStats st;
        generate_cache(s, *pb, r, *cfg, seed, round, begin, end, c.get(), st);
        if (stats) {
            stats->resampled += st.resampled;
            stats->cacheWalks += st.walks;
            stats->cacheTruncated += st.truncated;
            stats->cacheSteps += st.steps;
        }
        *out = c.release();
    })
}
int bvc_generate_boundary_cache(bvc_scene s, const bvc_problem* pb, bvc_region r, const bvc_cache_config* cfg,
                                uint64_t seed, uint64_t round, bvc_round_stats* stats, bvc_boundary_cache* out) {
    return bvc_generate_boundary_cache_shard(s, pb, r, cfg, seed, round, 0, std::max(1, cfg ? cfg->nBoundary : 1), stats,
                                             out);
}
int bvc_generate_source_cache(const bvc_problem* pb, bvc_region r, const bvc_cache_config* cfg, uint64_t seed,
                              uint64_t round, bvc_source_cache* out) {
    API({
        need(pb && r && cfg && out, "null argument");
        auto c = std::make_unique<bvc_source_cache_s>();
        generate_source(*pb, r, *cfg, seed, round, c.get());
        *out = c.release();
    })
}
int bvc_boundary_cache_create(const bvc_boundary_sample* smp, int n, int dim, int voronoi, double length,
                              bvc_boundary_cache* out) {
    API({
        require_device();
        need(out && (smp || n == 0) && n >= 0, "null argument");
        need(dim == 2 || dim == 3, "cache dimension must be 2 or 3");
        auto c = std::make_unique<bvc_boundary_cache_s>();
        c->n = n;
        c->dim = dim;
        c->voronoi = voronoi;
        c->length = length;
        std::vector<CacheSample> h(std::max(n, 1));
        for (int i = 0; i < n; ++i) {
            CacheSample& o = h[i];
            for (int k = 0; k < 3; ++k) {
                o.z[k] = static_cast<float>(smp[i].z[k]);
                o.n[k] = static_cast<float>(smp[i].n[k]);
            }
            if (dim == 2) o.z[2] = o.n[2] = 0.f;
            o.pdf = static_cast<float>(smp[i].pdf);
            o.uHat = static_cast<float>(smp[i].uHat);
            o.dHat = static_cast<float>(smp[i].dHat);
            o.weight = static_cast<float>(smp[i].weight);
            o.arc = static_cast<float>(smp[i].arc);
            o.segment = smp[i].segment;
        }
        c->samples.upload(h.data(), std::max(n, 1));
        *out = c.release();
    })
}
int bvc_boundary_cache_size(bvc_boundary_cache c, int* n, int* dim) {
    API({
        need(c, "null cache");
        if (n) *n = c->n;
        if (dim) *dim = c->dim;
    })
}
int bvc_boundary_cache_download(bvc_boundary_cache c, bvc_boundary_sample* smp) {
    API({
        require_device();
        need(c && smp, "null argument");
        std::vector<CacheSample> h(c->n);
        c->samples.download(h.data(), c->n);
        CK(cudaStreamSynchronize(g_stream));
        for (int i = 0; i < c->n; ++i) {
            bvc_boundary_sample& o = smp[i];
            for (int k = 0; k < 3; ++k) {
                o.z[k] = h[i].z[k];
                o.n[k] = h[i].n[k];
            }
            o.pdf = h[i].pdf;
            o.uHat = h[i].uHat;
            o.dHat = h[i].dHat;
            o.weight = h[i].weight;
            o.segment = h[i].segment;
            o.arc = h[i].arc;
        }
    })
}
int bvc_boundary_cache_packed(bvc_boundary_cache c, void** ptr, size_t* bytes) {
    API({
        need(c && ptr && bytes, "null argument");
        *ptr = c->samples.p;
        *bytes = static_cast<size_t>(c->n) * sizeof(CacheSample);
    })
}
int bvc_boundary_cache_from_packed(const void* ptr, int n, int dim, int voronoi, double length, bvc_boundary_cache* out) {
    API({
        require_device();
        need(out && (ptr || n == 0), "null argument");
        auto c = std::make_unique<bvc_boundary_cache_s>();
        c->n = n;
        c->dim = dim;
        c->voronoi = voronoi;
        c->length = length;
        c->samples.resize(std::max(n, 1));
        if (n) CK(cudaMemcpyAsync(c->samples.p, ptr, n * sizeof(CacheSample), cudaMemcpyDeviceToDevice, g_stream));
        *out = c.release();
    })
}
int bvc_boundary_cache_assign_voronoi(bvc_boundary_cache c, bvc_region r) {
    API(need(c && r, "null argument"); r->upload(); assign_voronoi(r, c))
}
int bvc_boundary_cache_destroy(bvc_boundary_cache c) { API(delete c) }
int bvc_source_cache_create(const bvc_source_sample* smp, int m, int dim, double area, bvc_source_cache* out) {
    API({
        require_device();
        need(out && (smp || m == 0) && m >= 0, "null argument");
        auto c = std::make_unique<bvc_source_cache_s>();
        c->m = m;
        c->dim = dim;
        c->area = area;
        std::vector<SourceSampleDev> h(std::max(m, 1));
        for (int i = 0; i < m; ++i) {
            for (int k = 0; k < 3; ++k) h[i].y[k] = static_cast<float>(smp[i].y[k]);
            if (dim == 2) h[i].y[2] = 0.f;
            h[i].pdf = static_cast<float>(smp[i].pdf);
            h[i].f = static_cast<float>(smp[i].f);
        }
        c->samples.upload(h.data(), std::max(m, 1));
        *out = c.release();
    })
}
int bvc_source_cache_size(bvc_source_cache c, int* m, int* dim) {
    API({
        need(c, "null cache");
        if (m) *m = c->m;
        if (dim) *dim = c->dim;
    })
}
int bvc_source_cache_download(bvc_source_cache c, bvc_source_sample* smp) {
    API({
        require_device();
        need(c && smp, "null argument");
        std::vector<SourceSampleDev> h(std::max(c->m, 1));
        c->samples.download(h.data(), c->m);
        CK(cudaStreamSynchronize(g_stream));
        for (int i = 0; i < c->m; ++i) {
            for (int k = 0; k < 3; ++k) smp[i].y[k] = h[i].y[k];
            smp[i].pdf = h[i].pdf;
            smp[i].f = h[i].f;
        }
    })
}
int bvc_source_cache_destroy(bvc_source_cache c) { API(delete c) }

int bvc_make_splat_config(bvc_scene s, const bvc_problem* pb, const bvc_cache_config* cfg, bvc_splat_config* out) {
    API({
        need(s && pb && cfg && out, "null argument");
        *out = make_splat_config(s, *pb, *cfg);
    })
}
int bvc_splat_solution(bvc_boundary_cache b, bvc_source_cache s, bvc_eval_points p, const bvc_splat_config* cfg) {
    API(need(cfg, "null config"); splat(b, s, p, *cfg, 0, SIZE_MAX, true, false))
}
int bvc_splat_gradient(bvc_boundary_cache b, bvc_source_cache s, bvc_eval_points p, const bvc_splat_config* cfg) {
    API(need(cfg, "null config"); splat(b, s, p, *cfg, 0, SIZE_MAX, false, true))
}
int bvc_splat_solution_gradient(bvc_boundary_cache b, bvc_source_cache s, bvc_eval_points p, const bvc_splat_config* cfg) {
    API(need(cfg, "null config"); splat(b, s, p, *cfg, 0, SIZE_MAX, true, true))
}
int bvc_splat_range(bvc_boundary_cache b, bvc_source_cache s, bvc_eval_points p, const bvc_splat_config* cfg,
                    size_t begin, size_t end, int value, int gradient) {
    API(need(cfg, "null config"); splat(b, s, p, *cfg, begin, end, value != 0, gradient != 0))
}

int bvc_corrected_boundary_splat(bvc_boundary_cache b, bvc_eval_points p, bvc_region r, const bvc_splat_config* cfg,
                                 double clampBound, int clampMode, const bvc_boundary_evaluator* eval, uint64_t seed,
                                 uint64_t stream) {
    API(need(cfg, "null config"); corrected_boundary(b, p, r, *cfg, clampBound, clampMode, eval, seed, stream))
}
int bvc_corrected_source_splat(bvc_source_cache s, bvc_eval_points p, bvc_region r, const bvc_splat_config* cfg,
                               double clampBound, const bvc_field* f, uint64_t seed, uint64_t stream) {
    API(need(cfg, "null config"); corrected_source(s, p, r, *cfg, clampBound, f, seed, stream))
}

int bvc_update_solution(bvc_scene s, const bvc_problem* pb, bvc_region r, const bvc_cache_config* cfg,
                        bvc_eval_points p, uint64_t seed, uint64_t round, int gradients, bvc_round_stats* stats) {
    API({
        require_device();
        need(s && pb && r && cfg && p, "null argument");
        validate_kernel(pb->kernel);
        if (cfg->sourceBall && gradients)
            throw Error(BVC_ERR_SOLVER, "ball-kernel source mode does not support gradient splats");
        bvc_splat_config scfg = make_splat_config(s, *pb, *cfg);
        need(cfg->clampMode >= BVC_CLAMP_OFF && cfg->clampMode <= BVC_CLAMP_CORRECT, "unknown clamp mode");
        cudaEvent_t e0, e1, e2;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventCreate(&e2));
        CK(cudaEventRecord(e0, g_stream));
        bvc_boundary_cache_s bc;
        bvc_source_cache_s sc;
        GenStats st;
        generate_cache(s, *pb, r, *cfg, seed, round, 0, std::max(1, cfg->nBoundary), &bc, st);
        generate_source(*pb, r, *cfg, seed, round, &sc);
        CK(cudaEventRecord(e1, g_stream));
        bool hasSource = pb->f.kind != BVC_FIELD_NONE;
        bvc_source_cache_s* sp = sc.m ? &sc : nullptr;
        // the mode dispatch of updateSolution (cache.cpp:639-662)
        if (cfg->clampMode == BVC_CLAMP_OFF) {
            // ball mode: splatSolution with G^B plus the unclamped (infinite-bound,
            // correction-free) ball source splat, i.e. one ball-kernel splat
            splat(&bc, sp, p, scfg, 0, SIZE_MAX, true, gradients != 0);
        } else {
            double c = cfg->clamp > 0.0 ? cfg->clamp : 10.0 / s->host.diagonal;  // resolvedClamp cache.h:129-131
            bvc_boundary_evaluator ev{};
            ev.kind = BVC_EVALUATOR_WALKS;
            ev.scene = s;
            ev.problem = pb;
            ev.cfg = cfg;
            corrected_boundary(&bc, p, r, scfg, c, cfg->clampMode, &ev, seed, bvc_dev::mixKey(kBoundaryCorrSalt, round));
            if (hasSource) {
                if (cfg->sourceBall) {
                    corrected_source(sp, p, r, scfg, c, &pb->f, seed, bvc_dev::mixKey(kSourceCorrSalt, round));
                } else {
                    splat(nullptr, sp, p, scfg, 0, SIZE_MAX, true, false);
                }
            }
            if (gradients) splat(&bc, sp, p, scfg, 0, SIZE_MAX, false, true);
        }
        fallback_walks(s, *pb, *cfg, p, seed, round, gradients != 0);
        CK(cudaEventRecord(e2, g_stream));
        CK(cudaEventSynchronize(e2));
        if (stats) {
            stats->resampled = st.resampled;
            stats->cacheWalks = st.walks;
            stats->cacheTruncated = st.truncated;
            stats->cacheSteps = st.steps;
            stats->generateSeconds = device_seconds(e0, e1);
            stats->splatSeconds = device_seconds(e1, e2);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaEventDestroy(e2);
    })
}

// the fallback-band loop of updateSolution (cache.cpp:665-681) alone: the sharded
// multi-GPU round runs it for the rank's own points after the exchange and gather
int bvc_fallback_walks(bvc_scene s, const bvc_problem* pb, const bvc_cache_config* cfg, bvc_eval_points p,
                       uint64_t seed, uint64_t round, int gradients) {
    API({
        require_device();
        need(s && pb && cfg && p, "null argument");
        fallback_walks(s, *pb, *cfg, p, seed, round, gradients != 0);
        CK(cudaGetLastError());
    })
}

int bvc_wos_solve(bvc_scene s, const bvc_problem* pb, const double* x, size_t n, const bvc_walk_config* cfg,
                  const uint64_t* streams, bvc_scalar_estimate* out) {
    API({
        need(s && pb && cfg && out, "null argument");
        if (s->host.hasNeumann()) throw Error(BVC_ERR_SOLVER, "wosSolve requires an all-Dirichlet scene");
        std::vector<double> m(n), se(n);
        std::vector<long long> c(n), t(n);
        pointwise(s, *pb, x, nullptr, n, *cfg, streams, 0, m.data(), se.data(), c.data(), t.data());
        for (size_t i = 0; i < n; ++i) out[i] = bvc_scalar_estimate{m[i], se[i], c[i], t[i]};
    })
}
int bvc_wost_solve(bvc_scene s, const bvc_problem* pb, const double* x, size_t n, const bvc_walk_config* cfg,
                   const uint64_t* streams, bvc_scalar_estimate* out) {
    API({
        need(s && pb && cfg && out, "null argument");
        std::vector<double> m(n), se(n);
        std::vector<long long> c(n), t(n);
        pointwise(s, *pb, x, nullptr, n, *cfg, streams, 0, m.data(), se.data(), c.data(), t.data());
        for (size_t i = 0; i < n; ++i) out[i] = bvc_scalar_estimate{m[i], se[i], c[i], t[i]};
    })
}
int bvc_wost_gradient(bvc_scene s, const bvc_problem* pb, const double* x, size_t n, const bvc_walk_config* cfg,
                      const uint64_t* streams, bvc_vector_estimate* out) {
    API({
        need(s && pb && cfg && out, "null argument");
        std::vector<double> m(2 * n), se(2 * n);
        std::vector<long long> c(n), t(n);
        pointwise(s, *pb, x, nullptr, n, *cfg, streams, 1, m.data(), se.data(), c.data(), t.data());
        for (size_t i = 0; i < n; ++i) {
            out[i].mean[0] = m[2 * i];
            out[i].mean[1] = m[2 * i + 1];
            out[i].se[0] = se[2 * i];
            out[i].se[1] = se[2 * i + 1];
            out[i].count = c[i];
            out[i].truncated = t[i];
        }
    })
}
int bvc_wost_normal_derivative(bvc_scene s, const bvc_problem* pb, const double* x, const double* normal, size_t n,
                               const bvc_walk_config* cfg, const uint64_t* streams, bvc_scalar_estimate* out) {
    API({
        need(s && pb && cfg && out && normal, "null argument");
        std::vector<double> m(n), se(n);
        std::vector<long long> c(n), t(n);
        pointwise(s, *pb, x, normal, n, *cfg, streams, 2, m.data(), se.data(), c.data(), t.data());
        for (size_t i = 0; i < n; ++i) out[i] = bvc_scalar_estimate{m[i], se[i], c[i], t[i]};
    })
}

int bvc_walk_traffic_profile(bvc_scene s, const bvc_problem* pb, bvc_region r, const bvc_cache_config* cfg,
                             uint64_t seed, uint64_t round, double* out) {
    API({
        need(s && pb && r && cfg && out, "null argument");
        bvc_boundary_cache_s c;
        GenStats st;
        g_profile = true;
        g_profileTotals[0] = g_profileTotals[1] = 0;
        try {
            generate_cache(s, *pb, r, *cfg, seed, round, 0, std::max(1, cfg->nBoundary), &c, st);
        } catch (...) {
            g_profile = false;
            throw;
        }
        g_profile = false;
        out[0] = static_cast<double>(st.steps);
        out[1] = static_cast<double>(g_profileTotals[0]);
        out[2] = static_cast<double>(g_profileTotals[1]);
        out[3] = static_cast<double>(st.walks);
    })
}

int bvc_eval_kernels(const bvc_kernel_spec* spec, const double* x, const double* y, const double* n, size_t count,
                     double* out) {
    API({
        require_device();
        need(spec && x && y && n && out, "null argument");
        validate_kernel(*spec);
        if (count == 0) return BVC_OK;
        int d = spec->dim;
        double* in = ws().get<double>(kWsEvalIn, 3 * d * count);
        double* o = ws().get<double>(kWsEvalOut, (2 + 2 * d) * count);
        CK(cudaMemcpyAsync(in, x, d * count * sizeof(double), cudaMemcpyHostToDevice, g_stream));
        CK(cudaMemcpyAsync(in + d * count, y, d * count * sizeof(double), cudaMemcpyHostToDevice, g_stream));
        CK(cudaMemcpyAsync(in + 2 * d * count, n, d * count * sizeof(double), cudaMemcpyHostToDevice, g_stream));
        eval_kernels(gather_kind(*spec), in, in + d * count, in + 2 * d * count, static_cast<int>(count), d,
                     static_cast<float>(spec->sigma), o, g_stream);
        CK(cudaMemcpyAsync(out, o, (2 + 2 * d) * count * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
    })
}
int bvc_eval_bessel(int which, const double* t, size_t count, double* out) {
    API({
        require_device();
        need(t && out && which >= 0 && which <= 3, "bad argument");
        if (count == 0) return BVC_OK;
        double* in = ws().get<double>(kWsEvalIn, count);
        double* o = ws().get<double>(kWsEvalOut, count);
        CK(cudaMemcpyAsync(in, t, count * sizeof(double), cudaMemcpyHostToDevice, g_stream));
        eval_bessel(which, in, static_cast<int>(count), o, g_stream);
        CK(cudaMemcpyAsync(out, o, count * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
    })
}

}  // extern "C"
