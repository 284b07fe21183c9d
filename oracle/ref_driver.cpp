// ref_driver.cpp — extern "C" driver around the REFERENCE's own BVC core.
//
// TEST INFRASTRUCTURE ONLY (see oracle/bvc_oracle.c header). oracle/Makefile
// compiles /root/reference/proj/core/src/{bvh,scene,sampling,kernels,pointwise,
// cache,grid}.cpp unmodified (against oracle/eigen_shim) together with this file
// into oracle/_ref/libbvc_ref.so. It is used to pin the C restatement, to make
// golden vectors, and as the CPU baseline (`cpu_baseline.kind = "reference"`).
// problems.cpp is left out: it needs Eigen/Sparse (fdReference) — the handful of
// scene makers it holds are restated by the Python test helpers instead.
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "bvc/cache.h"
#include "bvc/grid.h"
#include "bvc/kernels.h"
#include "bvc/parallel.h"
#include "bvc/pointwise.h"
#include "bvc/sampling.h"
#include "bvc/scene.h"

extern "C" {
#include "../include/bvc_b200.h"
double or_field_eval(const bvc_field* f, const double* p, int dim, int seg);
}

using namespace bvc;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const KernelSingularity*>(&e)) return BVC_ERR_SINGULARITY;
    if (dynamic_cast<const ParseError*>(&e)) return BVC_ERR_PARSE;
    if (dynamic_cast<const SolverError*>(&e)) return BVC_ERR_SOLVER;
    if (dynamic_cast<const std::invalid_argument*>(&e)) return BVC_ERR_INVALID_ARGUMENT;
    if (dynamic_cast<const std::domain_error*>(&e)) return BVC_ERR_DOMAIN;
    return BVC_ERR_SOLVER;
}

#define GUARD(...)                                   \
    try {                                            \
        __VA_ARGS__;                                 \
        return 0;                                    \
    } catch (const std::exception& e) {              \
        return fail(e);                              \
    }

KernelSpec toSpec(const bvc_kernel_spec& s) {
    KernelSpec k;
    k.kind = s.kind == BVC_KERNEL_SCREENED ? KernelKind::ScreenedPoisson : KernelKind::Poisson;
    k.sigma = s.sigma;
    k.dim = s.dim;
    k.scale = s.scale;
    return k;
}

// bvc_field -> std::function; NONE stays empty exactly like an unset callback
PdeProblem toProblem(const bvc_problem& p) {
    PdeProblem pb;
    pb.kernel = toSpec(p.kernel);
    if (p.f.kind != BVC_FIELD_NONE) {
        bvc_field f = p.f;
        pb.f = [f](const Vector2& x) { double q[2] = {x.x(), x.y()}; return or_field_eval(&f, q, 2, -1); };
    }
    if (p.g.kind != BVC_FIELD_NONE) {
        bvc_field g = p.g;
        pb.g = [g](const Vector2& x, int s) { double q[2] = {x.x(), x.y()}; return or_field_eval(&g, q, 2, s); };
    }
    if (p.h.kind != BVC_FIELD_NONE) {
        bvc_field h = p.h;
        pb.h = [h](const Vector2& x, int s) { double q[2] = {x.x(), x.y()}; return or_field_eval(&h, q, 2, s); };
    }
    return pb;
}

WalkConfig toWalk(const bvc_walk_config& w) {
    WalkConfig c;
    c.epsilon = w.epsilon;
    c.rMin = w.rMin;
    c.maxSteps = w.maxSteps;
    c.nWalks = w.nWalks;
    c.seed = w.seed;
    c.stream = w.stream;
    return c;
}

CacheConfig toCache(const bvc_cache_config& c) {
    CacheConfig k;
    k.nBoundary = c.nBoundary;
    k.nSource = c.nSource;
    k.nWalksNeumann = c.nWalksNeumann;
    k.nWalksDirichlet = c.nWalksDirichlet;
    k.offset = c.offset;
    k.clamp = c.clamp;
    k.clampMode = static_cast<ClampMode>(c.clampMode);
    k.sourceBall = c.sourceBall != 0;
    k.correctionWalks = c.correctionWalks;
    k.voronoi = c.voronoi != 0;
    k.stratified = c.stratified != 0;
    k.walk = toWalk(c.walk);
    k.threads = c.threads;
    return k;
}

QueryFilter toFilter(int f) {
    return f == BVC_FILTER_DIRICHLET ? QueryFilter::DirichletOnly
                                     : f == BVC_FILTER_NEUMANN ? QueryFilter::NeumannOnly
                                                               : QueryFilter::Any;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
uint64_t ref_mixkey(uint64_t key, uint64_t counter) { return mixKey(key, counter); }
uint64_t ref_mix64(uint64_t z) { return mix64(z); }
void ref_rng_uniforms(uint64_t seed, uint64_t stream, int n, double* out) {
    Rng r(seed, stream);
    for (int i = 0; i < n; ++i) out[i] = r.uniform();
}
void ref_rng_key_uniforms(uint64_t key, int n, double* out) {
    Rng r(key);
    for (int i = 0; i < n; ++i) out[i] = r.uniform();
}

// ---- kernels ------------------------------------------------------------------
int ref_bessel(int which, double t, double* out) {
    GUARD(*out = which == 0 ? besselK0(t) : which == 1 ? besselK1(t) : which == 2 ? besselI0(t) : besselI1(t));
}
int ref_eval_kernels(const bvc_kernel_spec* s, const double* x, const double* y, const double* n,
                     size_t count, double* out) {
    GUARD({
        KernelSpec k = toSpec(*s);
        int d = k.dim, stride = 2 + 2 * d;
        for (size_t i = 0; i < count; ++i) {
            double* o = out + stride * i;
            if (d == 2) {
                Vector2 X(x[2 * i], x[2 * i + 1]), Y(y[2 * i], y[2 * i + 1]), N(n[2 * i], n[2 * i + 1]);
                o[0] = greensFree(k, X, Y);
                Vector2 g = greensFreeGradient(k, X, Y);
                o[1] = g.x(); o[2] = g.y();
                o[3] = poissonKernelFree(k, X, Y, N);
                Vector2 pg = poissonKernelGradient(k, X, Y, N);
                o[4] = pg.x(); o[5] = pg.y();
            } else {
                Vector3 X(x[3 * i], x[3 * i + 1], x[3 * i + 2]), Y(y[3 * i], y[3 * i + 1], y[3 * i + 2]),
                    N(n[3 * i], n[3 * i + 1], n[3 * i + 2]);
                o[0] = greensFree(k, X, Y);
                Vector3 g = greensFreeGradient(k, X, Y);
                o[1] = g.x(); o[2] = g.y(); o[3] = g.z();
                o[4] = poissonKernelFree(k, X, Y, N);
                Vector3 pg = poissonKernelGradient(k, X, Y, N);
                o[5] = pg.x(); o[6] = pg.y(); o[7] = pg.z();
            }
        }
    });
}
// which: 0 ballGreens(R, r), 1 ballGreensMass(R), 2 ballSphereWeight(R, r)
int ref_ball(int which, const bvc_kernel_spec* s, double R, double r, double* out) {
    GUARD({
        KernelSpec k = toSpec(*s);
        *out = which == 0 ? ballGreens(k, R, r) : which == 1 ? ballGreensMass(k, R) : ballSphereWeight(k, R, r);
    });
}

// ---- scene ----------------------------------------------------------------------
void* ref_scene_create(const double* v, int nv, const int* segs, const int* labels, int ns) {
    try {
        std::vector<Vector2> verts(nv);
        for (int i = 0; i < nv; ++i) verts[i] = Vector2(v[2 * i], v[2 * i + 1]);
        std::vector<SegmentSpec> specs(ns);
        for (int i = 0; i < ns; ++i)
            specs[i] = {segs[2 * i], segs[2 * i + 1], labels[i] ? BoundaryLabel::Neumann : BoundaryLabel::Dirichlet};
        return new Scene(Scene::build(std::move(verts), specs));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}
void ref_scene_free(void* s) { delete static_cast<Scene*>(s); }
double ref_scene_diagonal(void* s) { return static_cast<Scene*>(s)->diagonal; }
int ref_scene_closed(void* s) { return static_cast<Scene*>(s)->closed(); }
int ref_scene_closest_point(void* sp, const double* x, size_t n, int filter, double* point,
                            double* dist, int* seg, double* t) {
    GUARD({
        const Scene& s = *static_cast<Scene*>(sp);
        for (size_t i = 0; i < n; ++i) {
            ClosestPointResult r = s.closestPoint(Vector2(x[2 * i], x[2 * i + 1]), toFilter(filter));
            point[2 * i] = r.point.x(); point[2 * i + 1] = r.point.y();
            dist[i] = r.dist; seg[i] = r.valid ? r.segment : -1; t[i] = r.t;
        }
    });
}
int ref_scene_silhouette_distance(void* sp, const double* x, size_t n, double* out) {
    GUARD({
        const Scene& s = *static_cast<Scene*>(sp);
        for (size_t i = 0; i < n; ++i) out[i] = s.silhouetteDistance(Vector2(x[2 * i], x[2 * i + 1]));
    });
}
int ref_scene_intersect_ray(void* sp, const double* o, const double* d, size_t n, double tMax,
                            int filter, double tMin, double* t, int* seg, double* point, double* sp_) {
    GUARD({
        const Scene& s = *static_cast<Scene*>(sp);
        for (size_t i = 0; i < n; ++i) {
            auto h = s.intersectRay(Vector2(o[2 * i], o[2 * i + 1]), Vector2(d[2 * i], d[2 * i + 1]), tMax,
                                    toFilter(filter), tMin);
            t[i] = h ? h->t : INFINITY; seg[i] = h ? h->segment : -1;
            point[2 * i] = h ? h->point.x() : 0.0; point[2 * i + 1] = h ? h->point.y() : 0.0;
            sp_[i] = h ? h->s : 0.0;
        }
    });
}
int ref_scene_inside(void* sp, const double* x, size_t n, uint8_t* out) {
    GUARD({
        const Scene& s = *static_cast<Scene*>(sp);
        for (size_t i = 0; i < n; ++i) out[i] = s.inside(Vector2(x[2 * i], x[2 * i + 1]));
    });
}
int ref_boundary_sample(void* sp, int filter, int count, int stratified, uint64_t key, double* p,
                        double* nrm, double* pdf, int* seg, double* arc) {
    GUARD({
        BoundarySampler smp(*static_cast<Scene*>(sp), toFilter(filter));
        Rng rng(key);
        std::vector<BoundaryPointSample> out;
        smp.sample(count, stratified != 0, rng, out);
        for (int i = 0; i < count; ++i) {
            p[2 * i] = out[i].p.x(); p[2 * i + 1] = out[i].p.y();
            nrm[2 * i] = out[i].n.x(); nrm[2 * i + 1] = out[i].n.y();
            pdf[i] = out[i].pdf; seg[i] = out[i].segment; arc[i] = out[i].arc;
        }
    });
}
int ref_region_sample(void* sp, int count, int stratified, uint64_t key, double* p, double* pdf) {
    GUARD({
        RegionSampler smp(*static_cast<Scene*>(sp));
        Rng rng(key);
        std::vector<RegionPointSample> out;
        smp.sample(count, stratified != 0, rng, out);
        for (int i = 0; i < count; ++i) {
            p[2 * i] = out[i].p.x(); p[2 * i + 1] = out[i].p.y(); pdf[i] = out[i].pdf;
        }
    });
}

// ---- region -----------------------------------------------------------------------
void* ref_region_build(void* sp, int mode, double offset, void* sub, double eps) {
    try {
        RegionRequest req;
        req.mode = mode == BVC_REGION_SUBDOMAIN ? RegionRequest::Mode::Subdomain : RegionRequest::Mode::WholeDomain;
        req.offset = offset;
        req.subdomain = static_cast<Scene*>(sub);
        return new SolveRegion(buildSolveRegion(*static_cast<Scene*>(sp), req, eps));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}
void ref_region_free(void* r) { delete static_cast<SolveRegion*>(r); }
void* ref_region_scene(void* r) { return &static_cast<SolveRegion*>(r)->boundary; }
void ref_region_info(void* rp, int* nv, int* ns, double* offset, double* area, int* whole) {
    const SolveRegion& r = *static_cast<SolveRegion*>(rp);
    *nv = static_cast<int>(r.boundary.vertices.size());
    *ns = static_cast<int>(r.boundary.segments.size());
    *offset = r.offset;
    *area = r.area;
    *whole = r.wholeDomain;
}
void ref_region_export(void* rp, double* v, int* segs, int* labels, int* kinds, int* src) {
    const SolveRegion& r = *static_cast<SolveRegion*>(rp);
    for (size_t i = 0; i < r.boundary.vertices.size(); ++i) {
        v[2 * i] = r.boundary.vertices[i].x(); v[2 * i + 1] = r.boundary.vertices[i].y();
    }
    for (size_t i = 0; i < r.boundary.segments.size(); ++i) {
        segs[2 * i] = r.boundary.segments[i].a; segs[2 * i + 1] = r.boundary.segments[i].b;
        labels[i] = static_cast<int>(r.boundary.segments[i].label);
        kinds[i] = static_cast<int>(r.kinds[i]) == 0 ? BVC_SEG_KNOWN_NEUMANN
                   : static_cast<int>(r.kinds[i]) == 1 ? BVC_SEG_ESTIMATED_OFFSET : BVC_SEG_USER_LOOP;
        src[i] = r.sourceSegment[i];
    }
}

// ---- walks -------------------------------------------------------------------------
// kind 0 = wosSolve, 1 = wostSolve; out = mean, se, count, truncated
int ref_solve(void* sp, const bvc_problem* pb, const double* x, const bvc_walk_config* cfg, int kind,
              double* out) {
    GUARD({
        PdeProblem p = toProblem(*pb);
        const Scene& s = *static_cast<Scene*>(sp);
        ScalarEstimate e = kind == 0 ? wosSolve(s, p, Vector2(x[0], x[1]), toWalk(*cfg))
                                     : wostSolve(s, p, Vector2(x[0], x[1]), toWalk(*cfg));
        out[0] = e.mean; out[1] = e.se; out[2] = double(e.count); out[3] = double(e.truncated);
    });
}
// normal == NULL: wostGradient (out mean2, se2, count, truncated) else wostNormalDerivative
int ref_gradient(void* sp, const bvc_problem* pb, const double* x, const double* normal,
                 const bvc_walk_config* cfg, double* out) {
    GUARD({
        PdeProblem p = toProblem(*pb);
        const Scene& s = *static_cast<Scene*>(sp);
        if (normal) {
            ScalarEstimate e = wostNormalDerivative(s, p, Vector2(x[0], x[1]), Vector2(normal[0], normal[1]), toWalk(*cfg));
            out[0] = e.mean; out[1] = e.se; out[2] = double(e.count); out[3] = double(e.truncated);
        } else {
            VectorEstimate e = wostGradient(s, p, Vector2(x[0], x[1]), toWalk(*cfg));
            out[0] = e.mean.x(); out[1] = e.mean.y(); out[2] = e.se.x(); out[3] = e.se.y();
            out[4] = double(e.count); out[5] = double(e.truncated);
        }
    });
}

// generateBoundaryCache; per sample z(2), n(2), pdf, uHat, dHat, weight, segment, arc.
// stats: resampled, cacheWalks, cacheTruncated; seconds: wall time of the call
int ref_generate_boundary_cache(void* sp, const bvc_problem* pb, void* rp, const bvc_cache_config* cfg,
                                uint64_t seed, uint64_t round, double* z, double* nrm, double* pdf,
                                double* uhat, double* dhat, double* w, int* seg, double* arc,
                                long long* stats, double* seconds) {
    GUARD({
        PdeProblem p = toProblem(*pb);
        RoundStats rs;
        auto t0 = std::chrono::steady_clock::now();
        BoundaryCache c = generateBoundaryCache(*static_cast<Scene*>(sp), p, *static_cast<SolveRegion*>(rp),
                                                toCache(*cfg), seed, round, &rs);
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (size_t i = 0; i < c.samples.size(); ++i) {
            const auto& s = c.samples[i];
            z[2 * i] = s.z.x(); z[2 * i + 1] = s.z.y(); nrm[2 * i] = s.n.x(); nrm[2 * i + 1] = s.n.y();
            pdf[i] = s.pdf; uhat[i] = s.uHat; dhat[i] = s.dHat; w[i] = s.weight; seg[i] = s.segment; arc[i] = s.arc;
        }
        stats[0] = rs.resampled; stats[1] = rs.cacheWalks; stats[2] = rs.cacheTruncated;
    });
}
int ref_generate_source_cache(const bvc_problem* pb, void* rp, const bvc_cache_config* cfg, uint64_t seed,
                              uint64_t round, double* y, double* pdf, double* f, int* m) {
    GUARD({
        SourceCache c = generateSourceCache(toProblem(*pb), *static_cast<SolveRegion*>(rp), toCache(*cfg), seed, round);
        *m = static_cast<int>(c.samples.size());
        for (size_t i = 0; i < c.samples.size(); ++i) {
            y[2 * i] = c.samples[i].y.x(); y[2 * i + 1] = c.samples[i].y.y();
            pdf[i] = c.samples[i].pdf; f[i] = c.samples[i].f;
        }
    });
}

// splatSolution (value) and/or splatGradient (gradient) on an identical host cache, 2D.
// Sums accumulate into the given arrays. threads: SplatConfig::threads. seconds: wall time
int ref_splat(const bvc_kernel_spec* spec, double tol, int voronoi, int N, const double* bz,
              const double* bn, const double* bpdf, const double* bu, const double* bd, const double* bw,
              int M, const double* sy, const double* spdf, const double* sf, size_t K, const double* px,
              const uint8_t* fallback, int value, int gradient, int threads, double* bsum, double* ssum,
              long long* nb, long long* ms, double* bgsum, double* sgsum, long long* nbg, long long* msg,
              long long* skipped, double* seconds) {
    GUARD({
        BoundaryCache bc;
        bc.voronoi = voronoi != 0;
        bc.samples.resize(N);
        for (int i = 0; i < N; ++i) {
            auto& s = bc.samples[i];
            s.z = Vector2(bz[2 * i], bz[2 * i + 1]); s.n = Vector2(bn[2 * i], bn[2 * i + 1]);
            s.pdf = bpdf[i]; s.uHat = bu[i]; s.dHat = bd[i]; s.weight = bw ? bw[i] : 0.0;
        }
        SourceCache sc;
        sc.samples.resize(M);
        for (int j = 0; j < M; ++j) sc.samples[j] = {Vector2(sy[2 * j], sy[2 * j + 1]), spdf[j], sf[j]};
        std::vector<EvaluationPoint> pts(K);
        for (size_t k = 0; k < K; ++k) {
            auto& p = pts[k];
            p.x = Vector2(px[2 * k], px[2 * k + 1]);
            p.fallback = fallback ? fallback[k] != 0 : false;
            p.boundarySum = bsum[k]; p.sourceSum = ssum[k]; p.nBoundary = nb[k]; p.mSource = ms[k];
            p.boundaryGradSum = Vector2(bgsum[2 * k], bgsum[2 * k + 1]);
            p.sourceGradSum = Vector2(sgsum[2 * k], sgsum[2 * k + 1]);
            p.nBoundaryGrad = nbg[k]; p.mSourceGrad = msg[k]; p.skipped = skipped[k];
        }
        SplatConfig cfg;
        cfg.kernel = toSpec(*spec);
        cfg.coincidenceTol = tol;
        cfg.voronoi = voronoi != 0;
        cfg.threads = resolveThreadCount(threads);
        auto t0 = std::chrono::steady_clock::now();
        if (value) splatSolution(bc, sc, pts, cfg);
        if (gradient) splatGradient(bc, sc, pts, cfg);
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (size_t k = 0; k < K; ++k) {
            const auto& p = pts[k];
            bsum[k] = p.boundarySum; ssum[k] = p.sourceSum; nb[k] = p.nBoundary; ms[k] = p.mSource;
            bgsum[2 * k] = p.boundaryGradSum.x(); bgsum[2 * k + 1] = p.boundaryGradSum.y();
            sgsum[2 * k] = p.sourceGradSum.x(); sgsum[2 * k + 1] = p.sourceGradSum.y();
            nbg[k] = p.nBoundaryGrad; msg[k] = p.mSourceGrad; skipped[k] = p.skipped;
        }
    });
}

// The 3D splatSolution loop. The reference's solver is 2D-only (pointwise.cpp:23), but its
// kernel templates (kernels.h:78-129) compile for Vector3; this is cache.cpp:426-461 with
// Vector3 points and samples, calling those templates unchanged, parallelised with the
// reference's own parallelFor (parallel.h:25-50). Plain 1/pdf weights (no Voronoi), no
// ball mode. This is the CPU counterpart of the C4/C5 gather (a "port" of the loop, not
// reference code); sums accumulate like EvaluationPoint's.
int ref_splat3(const bvc_kernel_spec* spec, double tol, int N, const double* bz, const double* bn,
               const double* bpdf, const double* bu, const double* bd, size_t K, const double* px,
               int threads, double* bsum, long long* nb, long long* skipped, double* seconds) {
    GUARD({
        struct S3 { Vector3 z, n; double pdf, u, d; };
        std::vector<S3> cache(N);
        for (int i = 0; i < N; ++i)
            cache[i] = {Vector3(bz[3 * i], bz[3 * i + 1], bz[3 * i + 2]),
                        Vector3(bn[3 * i], bn[3 * i + 1], bn[3 * i + 2]), bpdf[i], bu[i], bd[i]};
        KernelSpec k = toSpec(*spec);
        auto t0 = std::chrono::steady_clock::now();
        parallelFor(K, resolveThreadCount(threads), [&](size_t pi) {
            Vector3 x(px[3 * pi], px[3 * pi + 1], px[3 * pi + 2]);
            double sum = 0.0;
            long n = 0, skip = 0;
            for (const auto& s : cache) {
                double r = (x - s.z).norm();
                if (r < tol) {
                    ++skip;
                    continue;
                }
                double val = poissonKernelFree(k, x, s.z, s.n) * s.u - greensFree(k, x, s.z) * s.d;
                sum += val / s.pdf;
                ++n;
            }
            bsum[pi] += sum;
            nb[pi] += n;
            skipped[pi] += skip;
        });
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

// correctedBoundarySplat (ClampOnly) / correctedSourceSplat without the sampled
// terms (empty evaluator / f), or splatSolution, per the mode bits of or_clamped_splat
int ref_clamped_splat(const bvc_kernel_spec* spec, double tol, int voronoi, int N, const double* bz,
                      const double* bn, const double* bpdf, const double* bu, const double* bd,
                      const double* bw, int M, const double* sy, const double* spdf, const double* sf,
                      size_t K, const double* px, int mode, double clamp, const double* ballR, double* bsum,
                      double* ssum, long long* nb, long long* ms, long long* skipped) {
    GUARD({
        BoundaryCache bc;
        bc.voronoi = voronoi != 0;
        bc.samples.resize(N);
        for (int i = 0; i < N; ++i) {
            auto& s = bc.samples[i];
            s.z = Vector2(bz[2 * i], bz[2 * i + 1]); s.n = Vector2(bn[2 * i], bn[2 * i + 1]);
            s.pdf = bpdf[i]; s.uHat = bu[i]; s.dHat = bd[i]; s.weight = bw ? bw[i] : 0.0;
        }
        SourceCache sc;
        sc.samples.resize(M);
        for (int j = 0; j < M; ++j) sc.samples[j] = {Vector2(sy[2 * j], sy[2 * j + 1]), spdf[j], sf[j]};
        std::vector<EvaluationPoint> pts(K);
        for (size_t k = 0; k < K; ++k) {
            pts[k].x = Vector2(px[2 * k], px[2 * k + 1]);
            if (ballR) pts[k].ballRadius = ballR[k];
        }
        SplatConfig cfg;
        cfg.kernel = toSpec(*spec);
        cfg.coincidenceTol = tol;
        cfg.voronoi = voronoi != 0;
        cfg.useBallGreens = (mode & 2) != 0;
        cfg.threads = 1;
        SolveRegion none;  // unused without the sampled corrections
        BoundaryCache noB;
        SourceCache noS;
        if (mode & 1) correctedBoundarySplat(bc, pts, none, cfg, clamp, ClampMode::ClampOnly, {}, 0, 0);
        else splatSolution(bc, noS, pts, cfg);
        if (mode & 4) correctedSourceSplat(sc, pts, none, cfg, clamp, {}, 0, 0);
        else splatSolution(noB, sc, pts, cfg);
        for (size_t k = 0; k < K; ++k) {
            bsum[k] = pts[k].boundarySum; ssum[k] = pts[k].sourceSum; nb[k] = pts[k].nBoundary;
            ms[k] = pts[k].mSource; skipped[k] = pts[k].skipped;
        }
    });
}

// markEvaluationPoints with sourceBall: EvaluationPoint::ballRadius (cache.cpp:268-274)
int ref_ball_radius(void* sp, void* rp, const double* x, size_t n, double* radius) {
    GUARD({
        std::vector<EvaluationPoint> pts(n);
        for (size_t k = 0; k < n; ++k) pts[k].x = Vector2(x[2 * k], x[2 * k + 1]);
        CacheConfig c;
        c.sourceBall = true;
        markEvaluationPoints(*static_cast<Scene*>(sp), *static_cast<SolveRegion*>(rp), c, pts);
        for (size_t k = 0; k < n; ++k) radius[k] = pts[k].ballRadius;
    });
}

// GridField CSV writer and rmse (grid.cpp:22-34, 82-96)
int ref_grid_save_csv(const char* path, double ox, double oy, double h, int nx, int ny, const double* values,
                      const uint8_t* valid) {
    GUARD({
        GridField g = GridField::make(Vector2(ox, oy), h, nx, ny);
        for (size_t i = 0; i < g.values.size(); ++i) {
            g.values[i] = values[i];
            g.valid[i] = valid ? valid[i] != 0 : 1;
        }
        saveGridCsv(g, path);
    });
}
int ref_grid_load_rmse(const char* pathA, const char* pathB, double* out) {
    GUARD({ *out = rmse(loadGridCsv(pathA), loadGridCsv(pathB)); });
}

// markEvaluationPoints: fallback / gradientUnreliable flags
int ref_mark_points(void* sp, void* rp, const bvc_cache_config* cfg, const double* x, size_t n,
                    uint8_t* fallback, uint8_t* unreliable) {
    GUARD({
        std::vector<EvaluationPoint> pts(n);
        for (size_t k = 0; k < n; ++k) pts[k].x = Vector2(x[2 * k], x[2 * k + 1]);
        markEvaluationPoints(*static_cast<Scene*>(sp), *static_cast<SolveRegion*>(rp), toCache(*cfg), pts);
        for (size_t k = 0; k < n; ++k) { fallback[k] = pts[k].fallback; unreliable[k] = pts[k].gradientUnreliable; }
    });
}

// one updateSolution round over fresh points; returns per-point solution (and gradient)
// and the round stats: resampled, cacheWalks, cacheTruncated + generate/splat seconds
int ref_update_solution(void* sp, const bvc_problem* pb, void* rp, const bvc_cache_config* cfg,
                        const double* x, size_t n, uint64_t seed, uint64_t round, int gradients,
                        double* u, double* grad, uint8_t* fallback, long long* stats, double* seconds) {
    GUARD({
        std::vector<EvaluationPoint> pts(n);
        for (size_t k = 0; k < n; ++k) pts[k].x = Vector2(x[2 * k], x[2 * k + 1]);
        const Scene& s = *static_cast<Scene*>(sp);
        const SolveRegion& r = *static_cast<SolveRegion*>(rp);
        CacheConfig c = toCache(*cfg);
        markEvaluationPoints(s, r, c, pts);
        RoundStats rs = updateSolution(s, toProblem(*pb), r, c, pts, seed, round, gradients != 0);
        for (size_t k = 0; k < n; ++k) {
            u[k] = pts[k].solution();
            if (grad) { Vector2 g = pts[k].gradient(); grad[2 * k] = g.x(); grad[2 * k + 1] = g.y(); }
            fallback[k] = pts[k].fallback;
        }
        stats[0] = rs.resampled; stats[1] = rs.cacheWalks; stats[2] = rs.cacheTruncated;
        seconds[0] = rs.generateSeconds; seconds[1] = rs.splatSeconds;
    });
}

int ref_thread_count(int requested) { return resolveThreadCount(requested); }

} // extern "C"
