// correct.cu — the clamped-kernel corrections of the splat.
//
// Reference: correctedBoundarySplat cache.cpp:499-553 (ClampCorrect: one uniform
// ray per point and round; every region-boundary crossing whose |dG/dn| exceeds
// the bound c adds its clipped remainder times a fresh u(z) estimate),
// correctedSourceSplat cache.cpp:555-597 (one ball-kernel sample per point adds
// the clipped mass of G^B), markEvaluationPoints cache.cpp:263-276 (ball radius).
//
// Layout: one thread per active evaluation point (sorted order). The ray pass
// enumerates every crossing of the region BVH; with a walk evaluator it runs
// twice (count, then emit into a compacted hit list at scanned offsets) so the
// correction walks run as one persistent walk job over all saturated hits, and
// an apply pass folds the per-hit means back in fixed hit order (deterministic).
#include <cuda_runtime.h>

#include "gather.h"

namespace bvc_impl {

using namespace bvc_dev;

namespace {

constexpr double kPiD = 3.14159265358979323846;

__device__ __forceinline__ double u01d(uint32_t a, uint32_t b) {  // 53-bit uniform in [0, 1)
    return (static_cast<double>(a >> 5) * 67108864.0 + static_cast<double>(b >> 6)) * (1.0 / 9007199254740992.0);
}

// every crossing of o + t d (t > 0) with the region boundary (Scene::allRayHits
// scene.cpp:230-238), in BVH order; visit(seg, s) with the segment parameter s
template <class Visit>
__device__ void for_each_ray_hit(const SceneView2& S, float ox, float oy, float dx, float dy, Visit&& visit) {
    float idx = 1.0f / dx, idy = 1.0f / dy;
    int stack[kStack];
    int sp = 0, ref = 0;
    for (;;) {
        if (ref >= 0) {
            const Node2 nd = S.nodes[ref];
            bool vl = ray_box(nd.lbox, ox, oy, idx, idy, kFInf);
            bool vr = ray_box(nd.rbox, ox, oy, idx, idy, kFInf);
            if (vl && vr) { stack[sp++] = nd.right; ref = nd.left; continue; }
            if (vl) { ref = nd.left; continue; }
            if (vr) { ref = nd.right; continue; }
        } else {
            int code = ~ref;
            int start = code >> 3, count = (code & 7) + 1;
            for (int i = start; i < start + count; ++i) {
                const Prim2 p = S.prims[i];
                // the watertight side test of intersect_ray (scene_dev.cuh)
                float sa = ray_side(dx, dy, ox, oy, p.seg.x, p.seg.y);
                float sb = ray_side(dx, dy, ox, oy, p.seg.z, p.seg.w);
                if ((sa > 0.0f && sb > 0.0f) || (sa < 0.0f && sb < 0.0f)) continue;
                float den = sa - sb;
                if (den == 0.0f) continue;
                float s = sa / den;
                float px = fmaf(s, p.seg.z - p.seg.x, p.seg.x), py = fmaf(s, p.seg.w - p.seg.y, p.seg.y);
                if ((px - ox) * dx + (py - oy) * dy <= 0.0f) continue;  // t > tMin = 0
                visit(p, s);
            }
        }
        if (sp == 0) return;
        ref = stack[--sp];
    }
}

struct SatHit {
    double zx, zy;  // crossing point
    double w;       // sgn(n.dz) (|P| - c) 2 pi r^2 / |n.dz|  (cache.cpp:547)
    int seg;
};

// ray direction of point p and the saturated crossings along it
template <class Emit>
__device__ int saturated_hits(const CorrRayEnv& E, double x, double y, long long p, Emit&& emit) {
    U4 r = philox4x32_10(U4{static_cast<uint32_t>(p), static_cast<uint32_t>(p >> 32), 0u, 0u}, E.k0, E.k1);
    double theta = 2.0 * kPiD * u01d(r.x, r.y);
    double cd = cos(theta), sd = sin(theta);
    int hits = 0;
    for_each_ray_hit(E.region, static_cast<float>(x), static_cast<float>(y), static_cast<float>(cd),
                     static_cast<float>(sd), [&](const Prim2& pr, float s) {
                         ++hits;
                         double ax = pr.seg.x, ay = pr.seg.y, bx = pr.seg.z, by = pr.seg.w;
                         double zx = ax + s * (bx - ax), zy = ay + s * (by - ay);
                         double dzx = zx - x, dzy = zy - y;
                         double r2 = dzx * dzx + dzy * dzy;
                         if (r2 < E.tol2) return;  // cache.cpp:537
                         float2 n = E.region.segNormal[pr.id];
                         double nd = n.x * dzx + n.y * dzy;
                         double pk = nd / (2.0 * kPiD * r2);
                         if (E.screened) {
                             float t = static_cast<float>(E.sqrtSigma * sqrt(r2));
                             pk *= static_cast<double>(t <= 2.0f ? bessel_tk1_small(t) : t * bessel_k1(t));
                         }
                         double a = fabs(pk);
                         if (!(a > E.clamp)) return;  // unsaturated: nothing clipped
                         double sgn = nd > 0.0 ? 1.0 : -1.0;
                         emit(SatHit{zx, zy, sgn * (a - E.clamp) * 2.0 * kPiD * r2 / fabs(nd), pr.id});
                     });
    return hits;
}

__global__ void corr_rays_kernel(const CorrRayEnv E, const double* x, const int* order, int K, int* counts,
                                 double* bsum, int* noHit) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K) return;
    int p = order[i];
    double px = x[2 * p], py = x[2 * p + 1];
    int nsat = 0;
    double corr = 0.0;
    int hits = saturated_hits(E, px, py, E.base + p, [&](const SatHit& h) {
        ++nsat;
        if (E.useField) corr += h.w * static_cast<double>(field_eval(E.field, static_cast<float>(h.zx), static_cast<float>(h.zy)));
    });
    if (hits == 0 && inside(E.region, static_cast<float>(px), static_cast<float>(py), E.insideTol))
        atomicAdd(noHit, 1);  // cache.cpp:532-534
    if (E.useField) bsum[p] += corr * E.nRound;  // spread over the running /N divisor
    else counts[i] = nsat;
}

__global__ void corr_emit_kernel(const CorrRayEnv E, const double* x, const int* order, int K, const int* offsets,
                                 float2* starts, long long* gid, double* w) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K) return;
    int p = order[i];
    double px = x[2 * p], py = x[2 * p + 1];
    int o = offsets[i], k = 0;
    saturated_hits(E, px, py, E.base + p, [&](const SatHit& h) {
        // makeDefaultEvaluator cache.cpp:608-616: KnownNeumann crossings start eps/2 inside
        double zx = h.zx, zy = h.zy;
        if (E.kinds[h.seg] == 0) {
            float2 n = E.region.segNormal[h.seg];
            zx -= 0.5 * E.eps * n.x;
            zy -= 0.5 * E.eps * n.y;
        }
        starts[o + k] = make_float2(static_cast<float>(zx), static_cast<float>(zy));
        gid[o + k] = (E.base + p) * 4096 + k;
        w[o + k] = h.w;
        ++k;
    });
}

__global__ void corr_apply_kernel(const int* offsets, const int* counts, const int* order, int K, const double* w,
                                  const double* mean, double nRound, double* bsum) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K) return;
    int o = offsets[i], c = counts[i];
    if (!c) return;
    double corr = 0.0;
    for (int k = 0; k < c; ++k) corr += w[o + k] * mean[o + k];
    bsum[order[i]] += corr * nRound;
}

// inverse of the 2D Poisson ball radial CDF F(t) = t^2 (1 - 2 ln t) (kernels.cpp:78-94), FP64
__device__ double invert_ball_cdf_d(double u) {
    if (u <= 0.0) return 0.0;
    if (u >= 1.0) return 1.0;
    double lo = 0.0, hi = 1.0, t = sqrt(u);
    for (int it = 0; it < 60; ++it) {
        double lt = log(t);
        double fv = t * t * (1.0 - 2.0 * lt) - u;
        if (fv > 0.0) hi = t; else lo = t;
        double der = -4.0 * t * lt;
        double nxt = der != 0.0 ? t - fv / der : 0.5 * (lo + hi);
        if (!(nxt > lo && nxt < hi)) nxt = 0.5 * (lo + hi);
        if (fabs(nxt - t) < 1e-15) return nxt;
        t = nxt;
    }
    return t;
}

__global__ void ball_corr_kernel(const SceneView2 region, float insideTol, const double* x, const int* order,
                                 const double* ballR, int K, const DevField f, double clamp, double mRound, uint32_t k0,
                                 uint32_t k1, long long base, double* ssum) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K) return;
    int p = order[i];
    double px = x[2 * p], py = x[2 * p + 1], R = ballR[p];
    const long long gp = base + p;  // global point index: the same stream on any shard
    U4 r = philox4x32_10(U4{static_cast<uint32_t>(gp), static_cast<uint32_t>(gp >> 32), 0u, 0u}, k0, k1);
    // sampleBallGreens kernels.cpp:96-107
    double t = invert_ball_cdf_d(u01d(r.x, r.y));
    double rr = fmax(t * R, 1e-14 * R);
    double theta = 2.0 * kPiD * u01d(r.z, r.w);
    double yx = px + rr * cos(theta), yy = py + rr * sin(theta);
    // cache.cpp:586-591
    double dx = yx - px, dy = yy - py;
    double rc = fmin(sqrt(dx * dx + dy * dy), R);
    double gb = log(fmax(rc, 1e-14 * R) / R) / (2.0 * kPiD);
    double m = fmax(0.0, 1.0 - clamp / fabs(gb));
    if (m > 0.0 && inside(region, static_cast<float>(yx), static_cast<float>(yy), insideTol)) {
        double mass = -R * R / 4.0;  // ballGreensMass kernels.cpp:44-51
        ssum[p] += mass * m * static_cast<double>(field_eval(f, static_cast<float>(yx), static_cast<float>(yy))) * mRound;
    }
}

// markEvaluationPoints cache.cpp:268-274: the farthest region vertex is a hull vertex
__global__ void ball_radius_kernel(const double* x, int n, int dim, const double* hull, int nh, double* R) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double px = x[dim * i], py = x[dim * i + 1], best = 0.0;
    for (int k = 0; k < nh; ++k) {
        double dx = hull[2 * k] - px, dy = hull[2 * k + 1] - py;
        best = fmax(best, sqrt(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy))));  // (v - x).norm(), uncontracted
    }
    R[i] = best;
}

__global__ void gather_f32_kernel(const double* v, const int* order, int K, float* out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < K) out[i] = static_cast<float>(v[order[i]]);
}

inline int blocks(int n) { return (n + 127) / 128; }

}  // namespace

void launch_corr_rays(const CorrRayEnv& E, const double* x, const int* order, int K, int* counts, double* bsum,
                      int* noHit, cudaStream_t st) {
    if (K <= 0) return;
    corr_rays_kernel<<<blocks(K), 128, 0, st>>>(E, x, order, K, counts, bsum, noHit);
    count_launch();
}
void launch_corr_emit(const CorrRayEnv& E, const double* x, const int* order, int K, const int* offsets,
                      float2* starts, long long* gid, double* w, cudaStream_t st) {
    if (K <= 0) return;
    corr_emit_kernel<<<blocks(K), 128, 0, st>>>(E, x, order, K, offsets, starts, gid, w);
    count_launch();
}
void launch_corr_apply(const int* offsets, const int* counts, const int* order, int K, const double* w,
                       const double* mean, double nRound, double* bsum, cudaStream_t st) {
    if (K <= 0) return;
    corr_apply_kernel<<<blocks(K), 128, 0, st>>>(offsets, counts, order, K, w, mean, nRound, bsum);
    count_launch();
}
void launch_ball_corr(const SceneView2& region, float insideTol, const double* x, const int* order,
                      const double* ballR, int K, const DevField& f, double clamp, double mRound, uint32_t k0,
                      uint32_t k1, long long base, double* ssum, cudaStream_t st) {
    if (K <= 0) return;
    ball_corr_kernel<<<blocks(K), 128, 0, st>>>(region, insideTol, x, order, ballR, K, f, clamp, mRound, k0, k1,
                                                 base, ssum);
    count_launch();
}
void launch_ball_radius(const double* x, int n, int dim, const double* hull, int nh, double* R, cudaStream_t st) {
    if (n <= 0) return;
    ball_radius_kernel<<<blocks(n), 128, 0, st>>>(x, n, dim, hull, nh, R);
    count_launch();
}
void launch_gather_f32(const double* v, const int* order, int K, float* out, cudaStream_t st) {
    if (K <= 0) return;
    gather_f32_kernel<<<blocks(K), 128, 0, st>>>(v, order, K, out);
    count_launch();
}

}  // namespace bvc_impl
