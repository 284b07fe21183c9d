// gather.h — interface of the splat (gather) kernels in gather.cu.
#pragma once
#include "internal.h"

namespace bvc_impl {

enum GatherKind { kLap2 = 0, kScr2 = 1, kLap3 = 2, kScr3 = 3 };

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
void pack_boundary(const CacheSample* cs, int n, int kind, int voronoi, float4* out, cudaStream_t st);
void pack_source(const SourceSampleDev* ss, int m, int kind, float4* out, cudaStream_t st);
void eval_kernels(int kind, const double* x, const double* y, const double* n, int count, int dim, float sigma,
                  double* out, cudaStream_t st);
void eval_bessel(int which, const double* t, int count, double* out, cudaStream_t st);
void gather_points(const double* x, const int* order, int K, int dim, float* out, cudaStream_t st);
void launch_gather(int kind, const GatherPlan& g, const float4* pack, int N, int M, const float* px, int K, int dim,
                   float sigma, float tol, bool val, bool grad, double* part, int* skipB, int* skipS,
                   float4* tileBox, unsigned* unitCounter, cudaStream_t st);
void launch_finalize(const double* part, const GatherPlan& g, int K, const int* order, int N, int M, bool val,
                     bool grad, int dim, const int* skipB, const int* skipS, const PointsDev& pts, cudaStream_t st);

}  // namespace bvc_impl
