// capi_points.cu — EvaluationPoint handles (cache.h:73-110) on the device: the
// spatial (Morton) order of the gather, markEvaluationPoints (cache.cpp:263-276) with
// the ball radius of the ball-kernel mode, and the solution readout.
#include <cub/device/device_radix_sort.cuh>

#include "capi_common.cuh"

namespace bvc_capi {

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

// "some segment of the classes in qmask lies at distance < l from x", decided exactly as
// the reference decides it (closestPointOnSegment bvh.h:153-159, then norm() < l, in
// FP64 without contractions, like the host build): the FP32 BVH only proposes the
// candidates — every primitive whose box lies within l + margin, the margin covering
// the FP32 rounding of boxes and of x — and each candidate's distance is FP64.
__device__ bool within_exact(const bvc_dev::SceneView2& S, const double4* ab, double x, double y, unsigned qmask,
                             double l, float margin) {
    const float r = static_cast<float>(l) + margin;
    const float r2 = r * r;
    bool hit = false;
    bvc_dev::traverse_near(
        S, static_cast<float>(x), static_cast<float>(y), qmask,
        [&](const bvc_dev::Prim2& p) {
            if (hit) return;
            const double4 s = ab[p.id];
            const double ux = __dsub_rn(s.z, s.x), uy = __dsub_rn(s.w, s.y);
            const double len2 = __dadd_rn(__dmul_rn(ux, ux), __dmul_rn(uy, uy));
            double t = 0.0;
            if (len2 > 0.0) {
                t = __ddiv_rn(__dadd_rn(__dmul_rn(__dsub_rn(x, s.x), ux), __dmul_rn(__dsub_rn(y, s.y), uy)), len2);
                t = fmin(fmax(t, 0.0), 1.0);
            }
            const double dx = __dsub_rn(__dadd_rn(s.x, __dmul_rn(t, ux)), x);
            const double dy = __dsub_rn(__dadd_rn(s.y, __dmul_rn(t, uy)), y);
            if (__dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy))) < l) hit = true;
        },
        [&]() { return hit ? -1.0f : r2; });
    return hit;
}

__global__ void mark_kernel(const bvc_dev::SceneView2 scene, const double4* sceneAB, const bvc_dev::SceneView2 region,
                            const double4* regionAB, const double* x, int n, double offset, int whole, float margin,
                            uint8_t* fb, uint8_t* gu) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double px = x[2 * i], py = x[2 * i + 1];
    // fallbackBand cache.cpp:131-135: whole-domain points within l of the Dirichlet
    // boundary; gradientUnreliable cache.cpp:270-271: within l of the region boundary
    fb[i] = whole && within_exact(scene, sceneAB, px, py, bvc_dev::kClsD, offset, margin) ? 1 : 0;
    gu[i] = within_exact(region, regionAB, px, py, bvc_dev::kClsAny, offset, margin) ? 1 : 0;
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
        // FP32 boxes and query positions are within ~1e-7 diag of the exact ones
        const float margin = static_cast<float>(1e-5 * std::max(s->host.diagonal, r->boundary.host.diagonal));
        const bvc_dev::SceneView2 sv = s->view(), rv = r->boundary.view();  // uploads both (lazily)
        mark_kernel<<<(n + 127) / 128, 128, 0, g_stream>>>(sv, s->segAB64.p, rv,
                                                           r->boundary.segAB64.p, p->x.p, n, r->host.offset,
                                                           r->host.wholeDomain ? 1 : 0, margin, p->fallback.p,
                                                           p->unreliable.p);
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

void launch_solution(bvc_eval_points_s* P, double* u, double* g) {
    int n = static_cast<int>(P->n);
    solution_kernel<<<(n + 255) / 256, 256, 0, g_stream>>>(
        n, P->dim, P->fallback.p, P->bsum.p, P->ssum.p, P->nb.p, P->ms.p, P->bgsum.p, P->sgsum.p, P->nbg.p, P->msg.p,
        P->walkSum.p, P->walkCount.p, P->gwalkSum.p, P->gwalkCount.p, u, g);
    count_launch();
}

}  // namespace bvc_capi

extern "C" {

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
int bvc_points_set_index_base(bvc_eval_points p, long long base) {
    API({
        need(p, "null points");
        need(base >= 0, "negative index base");
        p->base = base;
    })
}

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
        launch_solution(p, o, o + n);
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

}  // extern "C"
