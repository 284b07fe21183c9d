// gather.h — interface of the splat (gather) kernels in gather.cu.
#pragma once
#include <cmath>

#include "internal.h"

namespace bvc_impl {

enum GatherKind { kLap2 = 0, kScr2 = 1, kLap3 = 2, kScr3 = 3,
                  // screened 3D, values only (C5), evaluated in coordinates scaled by
                  // k = sqrt(sigma) log2(e): gather-internal (pack, tile boxes, points, tolerance)
                  kScr3V = 4 };
// the scale of kScr3V's coordinates
inline float scr3v_scale(double sigma) { return static_cast<float>(std::sqrt(sigma) * 1.4426950408889634074); }

// device pointers of the EvaluationPoint running sums (cache.h:79-89)
struct PointsDev {
    double* bsum;
    double* ssum;
    long long* nb;
    long long* ms;
    double* bgsum;  // dim * n
    double* sgsum;
    long long* nbg;
    long long* msg;
    long long* skipped;
};

struct GatherPlan {
    int tiles = 0, chunk = 0, chunksB = 0, chunksS = 0, grid = 0, comps = 0;
};

GatherPlan plan_gather(int kind, int K, int N, int M, bool val, bool grad);
// the FP32 gather's prologue (gather.cu): pack (k: kScr3V's coordinate scale, 1 for the
// other kinds), per-tile boxes, zeroed skips and unit queue
void launch_prologue(const CacheSample* cs, int N, const SourceSampleDev* ss, int M, int kind, int voronoi, float k,
                     float4* pack, float4* tileBox, unsigned* unitCounter, int* skipB, int* skipS, int K,
                     cudaStream_t st);
void eval_kernels(int kind, const double* x, const double* y, const double* n, int count, int dim, float sigma,
                  double* out, cudaStream_t st);
void eval_bessel(int which, const double* t, int count, double* out, cudaStream_t st);
void gather_points(const double* x, const int* order, int K, int dim, float* out, cudaStream_t st);
void launch_gather(int kind, const GatherPlan& g, const float4* pack, int N, int M, const float* px, int K, int dim,
                   float sigma, float tol, bool val, bool grad, double* part, int* skipB, int* skipS,
                   float4* tileBox, unsigned* unitCounter, cudaStream_t st, int mode = 0, float clamp = 0.f,
                   const float* ballR = nullptr);
// splat modes (gather.cu SplatMode): 1 clamp dG/dn, 2 ball Green's function, 4 clamp source G^B
constexpr int kModeClampP = 1, kModeBall = 2, kModeClampS = 4;

// ray-sampled clamp correction (cache.cpp:526-550) and the ball-source correction
// (cache.cpp:584-592); see correct.cu
struct CorrRayEnv {
    bvc_dev::SceneView2 region;  // region boundary
    const int* kinds;            // region segment kinds (0 = KnownNeumann)
    int screened;
    double sqrtSigma;
    double clamp, tol2, nRound;
    float eps;                   // walk epsilon (Neumann crossings start eps/2 inside)
    float insideTol;
    uint32_t k0, k1;             // ray-direction key (seed, stream)
    long long base;              // global index of the points' first point (sharded point sets)
    int useField;                // 1: u(z) = field(z); 0: counts for the walk evaluator
    bvc_dev::DevField field;
};
void launch_corr_rays(const CorrRayEnv& E, const double* x, const int* order, int K, int* counts, double* bsum,
                      int* noHit, cudaStream_t st);
void launch_corr_emit(const CorrRayEnv& E, const double* x, const int* order, int K, const int* offsets,
                      float2* starts, long long* gid, double* w, cudaStream_t st);
void launch_corr_apply(const int* offsets, const int* counts, const int* order, int K, const double* w,
                       const double* mean, double nRound, double* bsum, cudaStream_t st);
void launch_ball_corr(const bvc_dev::SceneView2& region, float insideTol, const double* x, const int* order,
                      const double* ballR, int K, const bvc_dev::DevField& f, double clamp, double mRound, uint32_t k0,
                      uint32_t k1, long long base, double* ssum, cudaStream_t st);
void launch_ball_radius(const double* x, int n, int dim, const double* hull, int nh, double* R, cudaStream_t st);
void launch_gather_f32(const double* v, const int* order, int K, float* out, cudaStream_t st);
// FP64 variant (gather64.cu): Poisson kernels, exact per-pair coincidence test
void pack64_boundary(const CacheSample* cs, int n, int kind, int voronoi, double4* out, cudaStream_t st);
void pack64_source(const SourceSampleDev* ss, int m, int kind, double4* out, cudaStream_t st);
void gather_points64(const double* x, const int* order, int K, int dim, double* out, cudaStream_t st);
GatherPlan plan_gather64(int kind, int K, int N, int M, bool val, bool grad);
void launch_gather64(int kind, const GatherPlan& g, const double4* pack, int N, int M, const double* px, int K,
                     int dim, double tol, bool val, bool grad, double* part, int* skipB, int* skipS,
                     unsigned* unitCounter, cudaStream_t st);
void launch_finalize(const double* part, const GatherPlan& g, int K, const int* order, int N, int M, bool val,
                     bool grad, int dim, const int* skipB, const int* skipS, const PointsDev& pts, cudaStream_t st);

}  // namespace bvc_impl
