// capi.cu — the C ABI (include/bvc_b200.h) over the sm_100a BVC kernels: runtime
// state (stream, errors, launch count), scene and region handles, scene queries.
//
// The orchestration of the reference's operator API lives in the capi_*.cu files
// (see capi_common.cuh). Host preprocessing (scene build, solve region, host BVH) is
// host_scene.cpp. There is no CPU fallback: every compute entry point fails with
// BVC_ERR_NO_DEVICE when no CUDA device is present.
#include <atomic>
#include <mutex>

#include <cub/device/device_scan.cuh>

#include "capi_common.cuh"

namespace bvc_capi {

thread_local std::string g_error;
// Runtime state is per host thread and per device: a thread's current stream, its
// scratch workspaces and its side stream. Two threads driving two GPUs (or two
// threads sharing one) never share a stream or a scratch buffer.
__thread cudaStream_t g_stream = nullptr;
thread_local std::function<void()> g_afterWalkLaunch;
__thread bool g_profile = false;
__thread unsigned long long g_profileTotals[2] = {0, 0};

namespace {
std::atomic<long long> g_launches{0};
constexpr int kMaxDevices = 64;
struct DeviceState {
    cudaStream_t stream = nullptr;  // the thread's stream on this device (bvc_set_stream)
    Workspace* work = nullptr;      // main-stream scratch (lives for the process)
    cudaStream_t side = nullptr;    // second stream for work overlapping the cache walks
    Workspace* sideWork = nullptr;  // its own scratch
    cudaEvent_t events[9] = {};     // round_event
    unsigned long long* pinned = nullptr;  // GenStats::snapshot
};
thread_local DeviceState t_dev[kMaxDevices];
thread_local int t_device = -1;  // device g_stream belongs to
int current_device() {
    int d = 0;
    CK(cudaGetDevice(&d));
    need(d >= 0 && d < kMaxDevices, "device index out of range");
    return d;
}
}  // namespace

void require_device() {
    static std::atomic<int> state{-1};  // -1 unknown, 0 none, 1 ok
    if (state.load() < 0) {
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        state.store((e == cudaSuccess && n > 0) ? 1 : 0);
        if (e != cudaSuccess) cudaGetLastError();
    }
    if (!state.load()) throw Error(bvc_host::kNoDevice, "no CUDA device: the BVC path has no CPU fallback");
}

void ensure_pool() {
    static std::once_flag once[kMaxDevices];
    int d = current_device();
    std::call_once(once[d], [d] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    });
}

void bind_device(int device) {
    if (t_device >= 0 && t_device < kMaxDevices) t_dev[t_device].stream = g_stream;
    CK(cudaSetDevice(device));
    t_device = current_device();
    g_stream = t_dev[t_device].stream;
}

void bind_stream(cudaStream_t s) {
    g_stream = s;
    t_device = current_device();
    t_dev[t_device].stream = s;
}

__thread Workspace* g_wsActive = nullptr;
Workspace& ws() {
    if (g_wsActive) return *g_wsActive;
    DeviceState& d = t_dev[current_device()];
    if (!d.work) d.work = new Workspace();  // lives for the process
    return *d.work;
}

namespace {
DeviceState& side_for_device() {
    DeviceState& d = t_dev[current_device()];
    if (!d.side) {
        CK(cudaStreamCreateWithFlags(&d.side, cudaStreamNonBlocking));
        d.sideWork = new Workspace();  // lives for the process, like the main workspace
    }
    return d;
}
}  // namespace

unsigned long long* GenStats::device_counters() {
    if (!dev) {
        dev = ws().get<unsigned long long>(kWsRoundCtr, 4);
        CK(cudaMemsetAsync(dev, 0, 4 * sizeof(unsigned long long), g_stream));
    }
    return dev;
}

void GenStats::snapshot() {
    if (!dev) return;
    DeviceState& d = t_dev[current_device()];
    if (!d.pinned) CK(cudaMallocHost(reinterpret_cast<void**>(&d.pinned), 8 * sizeof(unsigned long long)));
    CK(cudaMemcpyAsync(d.pinned, dev, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, g_stream));
    pinned = d.pinned;
    dev = nullptr;
}

void GenStats::resolve() {
    if (!pinned) return;
    steps += static_cast<long long>(pinned[0]);
    truncated += static_cast<long long>(pinned[1]);
    walks += static_cast<long long>(pinned[2]);
    pinned = nullptr;
}

// One int read back from the device through this thread's pinned scratch. A copy into
// pageable memory blocks inside the driver until the stream reaches it, and other host
// threads' launches queue up behind that call; a pinned copy plus a stream wait does not.
int read_device_int(const int* dev) {
    DeviceState& d = t_dev[current_device()];
    if (!d.pinned) CK(cudaMallocHost(reinterpret_cast<void**>(&d.pinned), 8 * sizeof(unsigned long long)));
    volatile int* slot = reinterpret_cast<volatile int*>(d.pinned + 4);
    CK(cudaMemcpyAsync(const_cast<int*>(slot), dev, sizeof(int), cudaMemcpyDeviceToHost, g_stream));
    CK(cudaStreamSynchronize(g_stream));
    return *slot;
}

cudaEvent_t round_event(int which) {
    need(which >= 0 && which < 9, "round event index");
    DeviceState& d = t_dev[current_device()];
    if (!d.events[which])
        CK(cudaEventCreateWithFlags(&d.events[which], which < 2 ? cudaEventDisableTiming : cudaEventDefault));
    return d.events[which];
}

namespace {
// KernelTimer state: 0 idle, 1 armed, 2 begun, 3 ended, per kind (walk, gather)
thread_local int t_ktState[2] = {0, 0};
thread_local double t_ktLast[2] = {0.0, 0.0};
}  // namespace

void KernelTimer::arm() { t_ktState[0] = t_ktState[1] = 1; }
void KernelTimer::begin(int which) {
    if (t_ktState[which] != 1) return;
    CK(cudaEventRecord(round_event(5 + 2 * which), g_stream));
    t_ktState[which] = 2;
}
void KernelTimer::end(int which) {
    if (t_ktState[which] != 2) return;
    CK(cudaEventRecord(round_event(6 + 2 * which), g_stream));
    t_ktState[which] = 3;
}
void KernelTimer::resolve() {
    for (int k = 0; k < 2; ++k) {
        t_ktLast[k] = 0.0;
        if (t_ktState[k] == 3) {
            CK(cudaEventSynchronize(round_event(6 + 2 * k)));
            t_ktLast[k] = device_seconds(round_event(5 + 2 * k), round_event(6 + 2 * k));
        }
        t_ktState[k] = 0;
    }
}
const double* KernelTimer::last() { return t_ktLast; }

SideScope::SideScope() : stream(side_for_device().side), saved(g_wsActive) { g_wsActive = side_for_device().sideWork; }

int fail(const std::exception& e) {
    g_error = e.what();
    if (auto* be = dynamic_cast<const Error*>(&e)) return be->code;
    if (dynamic_cast<const std::bad_alloc*>(&e)) return BVC_ERR_CUDA;
    return BVC_ERR_SOLVER;
}

int leaf_size(int dim, int ns) {
    const char* e = std::getenv(dim == 2 ? "BVC_LEAF2" : "BVC_LEAF3");
    // measured with the warm-start grid and entry nodes: 3D leaves of 3 (C4 walks -2.5%, C5 -0.3% vs 2),
    // 2D leaves of 2 for 1025-4096 segments (C2; 4 costs +8%) and 4 above (C3 -3.5% vs 2)
    int def = dim == 3 ? 3 : (ns > 4096 ? 4 : (ns > 1024 ? 2 : 4));
    int v = e ? std::atoi(e) : def;
    return v >= 1 && v <= 8 ? v : def;
}

}  // namespace bvc_capi

namespace bvc_impl {
void count_launch(int n) { bvc_capi::g_launches.fetch_add(n, std::memory_order_relaxed); }
int api_fail(const std::exception& e) { return bvc_capi::fail(e); }
}  // namespace bvc_impl

// ---------------------------------------------------------------------------
// bvc_scene_s: device upload and BVH build
// ---------------------------------------------------------------------------
FarField bvc_scene_s::farfield() {
    const char* e = std::getenv("BVC_FARFIELD");
    if (!(e && std::string(e) == "1") || host.hasNeumann()) return FarField{};
    if (ffBuilt) return ff;
    upload();
    std::lock_guard<std::recursive_mutex> lk(lazyMu);
    if (ffBuilt) return ff;
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
    // built once per scene, possibly on another stream than its readers (the round's
    // side stream runs band walks that use it): complete it before publishing it
    CK(cudaStreamSynchronize(g_stream));
    ffBuilt = true;
    return ff;
}


HintGrid bvc_scene_s::hintgrid() {
    const char* e = std::getenv("BVC_HINTGRID");
    if (e && std::string(e) == "0") return HintGrid{};
    if (hgBuilt) return hg;
    upload();
    std::lock_guard<std::recursive_mutex> lk(lazyMu);
    if (hgBuilt) return hg;
    const int dim = host.dim;
    const char* en = std::getenv("BVC_HINTGRID_N");  // vertices along the longest side
    // 3D: cells about the triangle size (1.8 sqrt(triangles) along the longest side, 64-512):
    // a cell's candidate ball is dD(c) + 2 rho, so near the surface smaller cells give deeper
    // entry frontiers. Walk time by vertices along the side (C4 / C5, frontier of 4, 32-byte
    // cell records): 384: 0.327 / 2.467 s, 512: 0.318 / 2.421, 640: 0.310 / 2.384 (one-time build
    // 0.25 / 0.47 / 0.7 s; 1.8 GB at 384^3, 4.3 GB at 512^3, 8.4 GB at 640^3)
    const int n3 = static_cast<int>(std::lround(1.8 * std::sqrt(static_cast<double>(host.ns))));
    // 2D: a quarter of the segment count along the longest side, 1024-4096 (32 B per cell: 34-540 MB).
    // Walk time with frontiers by vertices along the side, C3 (16384 segments): 1024: 93.7 ms, 2048: 89.4,
    // 4096: 86.9 (one entry node per cell: 112.6 at any size); C1 (1024 segments): 1.1 ms at 1024-4096
    const int n2 = std::min(4096, std::max(1024, host.ns / 4));
    const int nLong = en && std::atoi(en) >= 16 ? std::atoi(en) : (dim == 2 ? n2 : std::min(512, std::max(64, n3)));
    double ext = 0.0, lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int k = 0; k < dim; ++k) {
        lo[k] = host.lo[k];
        hi[k] = host.hi[k];
        ext = std::max(ext, hi[k] - lo[k]);
    }
    const double h = std::max(ext, 1e-30) / (nLong - 1);
    int n[3] = {1, 1, 1};
    for (int k = 0; k < dim; ++k) n[k] = static_cast<int>(std::ceil((hi[k] - lo[k]) / h)) + 1;
    hg = HintGrid{};
    hg.lox = static_cast<float>(lo[0]);
    hg.loy = static_cast<float>(lo[1]);
    hg.loz = static_cast<float>(lo[2]);
    hg.h = static_cast<float>(h);
    hg.invH = static_cast<float>(1.0 / h);
    hg.nx = n[0];
    hg.ny = n[1];
    hg.nz = n[2];
    const size_t nv = static_cast<size_t>(n[0]) * n[1] * n[2];
    hgCells.resize(nv);
    // ray lengths are max(R, rMin) with rMin <= eps; a generous 1e-2 diag covers any rMin
    const float rmin = static_cast<float>(1e-2 * host.diagonal);
    const char* ee = std::getenv("BVC_ENTRY");  // 0: queries start at the root
    const char* ef = std::getenv("BVC_FRONT");  // 0: one entry node per cell
    const bool entries = !(ee && std::string(ee) == "0");
    const bool fronts = entries && !(ef && std::string(ef) == "0");
    if (dim == 2) launch_hintgrid2(view(), hg, hgCells.p, entries, fronts, rmin, g_stream);
    else launch_hintgrid3(view3(), hg, hgCells.p, entries, fronts, rmin, g_stream);
    CK(cudaGetLastError());
    // built once per scene, possibly on another stream than its readers (the round's
    // side stream runs band walks that use it): complete it before publishing it
    CK(cudaStreamSynchronize(g_stream));
    hg.cell = hgCells.p;
    hgBuilt = true;
    return hg;
}


std::string bvc_scene_s::builder() const {
    const char* e = std::getenv("BVC_BVH");
    std::string v = e ? e : "";
    if (v == "gpu") v = "lbvh";
    if (v != "sah" && v != "lbvh" && v != "host") v = (host.dim == 3 || host.ns >= 4096) ? "sah" : "host";
    return host.ns > 64 ? v : "host";  // tiny scenes: one host pass
}


namespace {
// Node order for the traversals' caches. The device builders number nodes in the order
// their CTAs finish (atomic counters), so a node's two children land anywhere in the
// array. This relayout numbers them depth first with each node's children in one
// adjacent pair, the pair starting at an even index: for 64-byte 3D nodes a sibling pair
// is one 128-byte line, so the sibling a traversal pops later was fetched with the child
// it descended into, and root-to-leaf paths run forward through memory. Leaf references
// (primitive ranges) are unchanged; the root stays at 0 (index 1 is padding).
template <class Node, class GetL, class GetR, class Set>
void relayout_pairs(DevBuf<Node>& buf, size_t nn, GetL left, GetR right, Set setLinks) {
    if (nn < 3) return;
    std::vector<Node> h(nn);
    buf.download(h.data(), nn);
    CK(cudaStreamSynchronize(g_stream));
    std::vector<int> newId(nn, -1), order;  // order[new] = old
    order.reserve(2 * nn + 2);
    newId[0] = 0;
    order.push_back(0);
    order.push_back(-1);  // padding: pairs start at even indices
    std::vector<int> stack{0};
    while (!stack.empty()) {
        int o = stack.back();
        stack.pop_back();
        int l = left(h[o]), r = right(h[o]);
        int base = static_cast<int>(order.size());
        order.push_back(l >= 0 ? l : -1);
        order.push_back(r >= 0 ? r : -1);
        if (l >= 0) newId[l] = base;
        if (r >= 0) newId[r] = base + 1;
        if (r >= 0) stack.push_back(r);  // left subtree first (it is popped first)
        if (l >= 0) stack.push_back(l);
    }
    std::vector<Node> out(order.size());
    for (size_t k = 0; k < order.size(); ++k) {
        if (order[k] < 0) {
            std::memset(&out[k], 0, sizeof(Node));
            continue;
        }
        Node nd = h[order[k]];
        int l = left(nd), r = right(nd);
        setLinks(nd, l >= 0 ? newId[l] : l, r >= 0 ? newId[r] : r);
        out[k] = nd;
    }
    buf.upload(out.data(), out.size());
}
}  // namespace

void bvc_scene_s::gpu_build(int dim, const float4* a, const float4* b, const float4* c, const int2* sil) {
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
    const char* rl = std::getenv("BVC_RELAYOUT");  // measurement knob: 0 keeps the builder's order
    if (!(rl && std::string(rl) == "0")) {
        if (dim == 3)
            relayout_pairs(nodes3, nn, [](const bvc_dev::Node3& x) { return x.left(); },
                           [](const bvc_dev::Node3& x) { return x.right(); },
                           [](bvc_dev::Node3& x, int l, int r) { x.set_links(l, r, x.mask()); });
        else
            relayout_pairs(nodes, nn, [](const Node2& x) { return x.left; }, [](const Node2& x) { return x.right; },
                           [](Node2& x, int l, int r) { x.left = l; x.right = r; });
    }
}


void bvc_scene_s::upload3() {
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
            hn[i].set_links(bvh.children[2 * i], bvh.children[2 * i + 1], bvh.masks[i]);
        }
        nodes3.upload(hn.data(), nn);
        std::vector<bvc_dev::Prim3> hp(host.ns);
        for (int j = 0; j < host.ns; ++j) {
            int id = bvh.order[j];
            hp[j].a = f4(host.vert(host.idx[3 * id]), int_as_float_host(id));
            hp[j].b = f4(host.vert(host.idx[3 * id + 1]), int_as_float_host(bvc_host::primClass(host, id)));
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
        const double ex = host.sil3B[3 * k] - host.sil3A[3 * k], ey = host.sil3B[3 * k + 1] - host.sil3A[3 * k + 1],
                     ez = host.sil3B[3 * k + 2] - host.sil3A[3 * k + 2], l2 = ex * ex + ey * ey + ez * ez;
        eb[k] = f4(&host.sil3B[3 * k], l2 > 0.0 ? static_cast<float>(1.0 / l2) : 0.f);  // w: 1 / |b - a|^2
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
    if (!host.sil3Always.empty()) build_sil_records();
}


// Silhouette-edge records in leaf order: a star query that reaches a triangle with
// silhouette edges reads them next to the triangle's neighbours in the same leaf,
// without the dependent triSil -> edge-array loads, behind a per-triangle visibility
// pre-test (header; Prim3.c.w = float4 offset << 2 | count).
void bvc_scene_s::build_sil_records() {
    const int n = host.ns;
    DevBuf<int> counts, offsets;
    counts.resize(n);
    offsets.resize(n);
    launch_sil_count3(prims3.p, n, triSil.p, counts.p, g_stream);
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, counts.p, offsets.p, n, g_stream));
    DevBuf<char> scratch;
    scratch.resize(std::max<size_t>(tmp, 1));
    CK(cub::DeviceScan::ExclusiveSum(scratch.p, tmp, counts.p, offsets.p, n, g_stream));
    int last[2] = {0, 0};
    CK(cudaMemcpyAsync(&last[0], offsets.p + (n - 1), sizeof(int), cudaMemcpyDeviceToHost, g_stream));
    CK(cudaMemcpyAsync(&last[1], counts.p + (n - 1), sizeof(int), cudaMemcpyDeviceToHost, g_stream));
    CK(cudaStreamSynchronize(g_stream));
    silRec.resize(static_cast<size_t>(std::max(last[0] + last[1], 1)));  // float4 units
    launch_sil_fill3(prims3.p, n, triSil.p, counts.p, offsets.p, sil3A.p, sil3N1.p, sil3N2.p, sil3B.p, triNormal.p,
                     silRec.p, g_stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(g_stream));
}


bvc_dev::SceneView3 bvc_scene_s::view3() {
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


void bvc_scene_s::upload() {
    if (uploaded) return;
    require_device();
    std::lock_guard<std::recursive_mutex> lk(lazyMu);
    if (uploaded) return;
    if (host.dim == 3) upload3();
    else upload2();
    CK(cudaStreamSynchronize(g_stream));  // published to every thread and stream
    uploaded = true;
}

void bvc_scene_s::upload2() {
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
    std::vector<double4> hab64(host.ns);
    std::vector<float> harc(host.ns), hlen(host.ns);
    for (int i = 0; i < host.ns; ++i) {
        hnrm[i] = make_float2(host.normal[2 * i], host.normal[2 * i + 1]);
        const double *a = host.vert(host.idx[2 * i]), *b = host.vert(host.idx[2 * i + 1]);
        hab[i] = make_float4(a[0], a[1], b[0], b[1]);
        hab64[i] = make_double4(a[0], a[1], b[0], b[1]);
        harc[i] = static_cast<float>(host.arc[i]);
        hlen[i] = static_cast<float>(host.measure[i]);
    }
    segNormal.upload(hnrm.data(), hnrm.size());
    segAB.upload(hab.data(), hab.size());
    segAB64.upload(hab64.data(), hab64.size());
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
    build_runs();
}

// A ray that hits a Neumann segment hits the same point of the line through it, so
// consecutive exactly collinear Neumann segments of a chain can answer the walks' rays
// as one segment (the hit's normal is the run's, and a walker standing on the run
// skips the whole line, which a ray leaving it cannot meet again). A subdivided
// straight wall (C2: 2 x 512 segments) becomes 2 segments, tested in a loop instead of a
// BVH traversal. The same holds for the closest Dirichlet point (the closest point of a
// straight wall is the closest point of its subdivisions) and, with the silhouette
// candidates tested directly, for the star radius. Used only when the runs are few
// (<= 32) and merge >= 4 segments each on average; curved boundaries keep the BVH.
void bvc_scene_s::build_runs() {
    runN = drunN = 0;
    if (const char* e = std::getenv("BVC_RUNS"))  // 0: always query through the BVH (tests, A/B)
        if (std::string(e) == "0") return;
    std::vector<float4> seg[2];
    std::vector<int> ids[2];
    int count[2] = {0, 0};
    for (const auto& L : host.loops) {
        const size_t m = L.size();
        if (m == 0) continue;
        auto dir = [&](int i, double& ex, double& ey) {
            const double *a = host.vert(host.idx[2 * i]), *b = host.vert(host.idx[2 * i + 1]);
            ex = b[0] - a[0];
            ey = b[1] - a[1];
        };
        auto joins = [&](int i, int j) {  // j continues i's straight run of the same label
            if (host.label[i] != host.label[j] || host.idx[2 * i + 1] != host.idx[2 * j]) return false;
            double ax, ay, bx, by;
            dir(i, ax, ay);
            dir(j, bx, by);
            return ax * by - ay * bx == 0.0 && ax * bx + ay * by > 0.0;
        };
        const bool closed = host.loopClosed[host.loop[L[0]]] != 0;
        // start at a segment that does not continue its predecessor's run
        size_t s0 = 0;
        if (closed) {
            size_t k = 0;
            while (k < m && joins(L[(k + m - 1) % m], L[k])) ++k;
            if (k == m) return;  // a closed loop cannot be one straight run
            s0 = k;
        }
        for (size_t c = 0; c < m;) {
            const int first = L[(s0 + c) % m];
            size_t len = 1;
            while (c + len < m && joins(L[(s0 + c + len - 1) % m], L[(s0 + c + len) % m])) ++len;
            const int last = L[(s0 + c + len - 1) % m];
            const double *a = host.vert(host.idx[2 * first]), *b = host.vert(host.idx[2 * last + 1]);
            const int lab = host.label[first] ? 1 : 0;
            seg[lab].push_back(make_float4(a[0], a[1], b[0], b[1]));
            ids[lab].push_back(first);
            count[lab] += static_cast<int>(len);
            c += len;
        }
    }
    // Neumann runs answer the rays; Dirichlet runs (with the silhouette candidates, when
    // few) answer the star and closest-point queries of the walks
    const int nN = static_cast<int>(seg[1].size()), nD = static_cast<int>(seg[0].size());
    if (nN > 0 && nN <= 32 && 4 * nN <= count[1]) {
        runSeg.upload(seg[1].data(), nN);
        runId.upload(ids[1].data(), nN);
        runN = nN;
    }
    const int nSil = static_cast<int>(host.silAlways.size());
    if (nD > 0 && nD <= 32 && 4 * nD <= count[0] && nSil <= 32 && (host.neumannMeasure == 0.0 || runN > 0)) {
        drunSeg.upload(seg[0].data(), nD);
        drunId.upload(ids[0].data(), nD);
        drunN = nD;
    }
}


bvc_dev::SceneView2 bvc_scene_s::view() {
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


extern "C" {

const char* bvc_last_error(void) { return g_error.c_str(); }
int bvc_abi_version(void) { return BVC_ABI_VERSION; }
long long bvc_kernel_launch_count(void) { return bvc_capi::g_launches.load(); }
int bvc_last_round_kernel_seconds(double* walkSeconds, double* gatherSeconds) {
    const double* t = bvc_capi::KernelTimer::last();
    if (walkSeconds) *walkSeconds = t[0];
    if (gatherSeconds) *gatherSeconds = t[1];
    return BVC_OK;
}

int bvc_set_device(int device) { API(require_device(); bind_device(device)) }
int bvc_set_stream(void* s) { API(require_device(); bind_stream(static_cast<cudaStream_t>(s))) }
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
