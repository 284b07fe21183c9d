// internal.h — types shared by the CUDA translation units of libbvc_b200.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "device_math.cuh"
#include "host_scene.h"
#include "scene3_dev.cuh"
#include "scene_dev.cuh"

namespace bvc_impl {

using bvc_dev::DevField;
using bvc_dev::SceneView2;

// Warm-start grid: for every cell of a uniform grid over the scene box, the Dirichlet
// primitive closest to the cell centre c (2D: segment id; 3D: leaf-order triangle index). A
// walk step at x also seeds its closest-point query with its cell's primitive, whose
// distance is at most d(x) + 2|x - c|: the pruning radius starts near-tight even after a
// long jump, and the result is unchanged (one more candidate of the same minimum).
// BVC_HINTGRID=0 disables it.
//
// The cell also keeps entry refs: with rho its half-diagonal, every Dirichlet or silhouette
// primitive a star / closest-point query at x in the cell can use lies within
// dD(x) <= dD(c) + rho of x, so within r = dD(c) + 2 rho of c; the single entry is the deepest
// BVH node whose subtree holds every primitive box of those classes within r of c, and the
// entry frontier (BVC_FRONT=0 disables it) up to four deeper nodes that together do. A Neumann
// ray of such a step is no longer than dD(x) either, so the ray entry is the same for the
// Neumann classes (kNoEntry: the cell's rays cannot reach any). Queries start there instead
// of the root (BVC_ENTRY=0): the top levels, which every query of the cell would descend
// identically, are skipped, and the result is the same (every candidate is in the subtrees).
// One 32-byte record per cell (one memory sector per walk step): the cell's star /
// closest-point starts (`front`: entry_frontier2 / 3, up to 4 nodes whose subtrees hold every
// usable primitive; front.x alone when frontiers are off; kNoEntry = unused slot), its Neumann
// ray entry, and the Dirichlet primitive closest to the cell centre (the warm start).
struct alignas(32) HintCell {
    int4 front;
    int ray;  // Neumann ray entry node, or kNoEntry
    int id;   // leaf-order (3D) / segment (2D) index of the warm-start primitive, or -1
    int pad0, pad1;
};
static_assert(sizeof(HintCell) == 32, "HintCell layout");
struct HintGrid {
    const HintCell* cell;  // NULL: disabled
    float lox, loy, loz, h, invH;
    int nx, ny, nz;
};
// what a step takes from its cell (roots and no warm start outside the grid)
struct CellHints {
    int4 front;
    int ray, id;
};

// PdeProblem with device field descriptors (pointwise.h:19-26)
struct DevProblem {
    int screened;   // KernelKind::ScreenedPoisson
    float sigma, sqrtSigma;
    int dim;
    DevField f, g, h;
};

// Far-field distance bounds: the exact distance to the whole boundary (any class) at
// the vertices of a uniform grid. At x, d(v) - |x - v| (minus a rounding margin) is a
// lower bound of d(x); when it exceeds tau the step uses it as the ball radius and
// skips the BVH queries (any ball inside the domain keeps walk-on-spheres unbiased;
// near the boundary, where walks terminate, the exact queries run as before).
struct FarField {
    const float* d;  // NULL: disabled
    float lox, loy, loz, h, invH, tau, margin;
    int nx, ny, nz;
};

// WalkContext (pointwise.cpp:11-35) in device form
struct WalkEnv {
    SceneView2 S;
    // Neumann rays against the scene's straight Neumann runs (bvc_scene_s::build_runs):
    // consecutive exactly collinear Neumann segments merged into one; used when there are
    // few (runN > 0), else rays traverse the BVH
    const float4* runSeg;
    const int* runId;  // a segment of the run (its normal is the run's)
    int runN;
    // with Dirichlet runs (drunN > 0) the star / closest-point queries test the runs and
    // the silhouette candidates (S.silP, nSil of them) directly, without the BVH
    const float4* drunSeg;
    const int* drunId;
    int drunN, nSil;
    DevProblem P;
    float eps, rmin, tguard, insideTol, scale, nudge;
    float cx, cy, escape;  // scene box centre and escape half-width
    int maxSteps;
    int hasNeumann, hasSource, hasH, closed;
    uint32_t k0, k1;  // Philox key of the job (seed, salt, round)
    FarField ff;
    HintGrid hg;
};

// A batch of estimator tasks. U tasks: nU plain walks from each U start point.
// D tasks: nD first-ball gradient samples (pointwise.cpp:195-215) at each D point.
// Outputs land in fixed slots, so results do not depend on scheduling.
struct WalkJob {
    int nU;
    int nPtsU;
    const float2* startU;
    const long long* gidU;  // global id per U point (RNG keying; NULL => local index)
    float* outU;            // [pt * nU + k]
    int* truncU;            // per point, may be NULL
    int nD;
    int nPtsD;
    const int* nPtsDdev;    // device count of the D points (then nPtsD is only the capacity), or NULL
    const float2* xD;       // gradient ball center
    const float2* normalD;  // NULL => vector output (wostGradient)
    const float* radiusD;   // first-ball radius
    const long long* gidD;
    float* outD;            // [pt * nD + k] or [2 * (pt * nD + k) + c]
    int* truncD;
    long long gidBaseU;     // global id of U point 0 when gidU is NULL
    unsigned long long* truncTotal;  // total truncated walks (may be NULL)
    unsigned long long* steps;  // total closest-Dirichlet queries (may be NULL)
    unsigned long long* counter; // work-queue head, zeroed by the launcher
    // first-step warm starts (may be NULL): a Dirichlet segment id per U / D point
    const int* hintU;
    const int* hintD;
};

void launch_walk_job(const WalkEnv& env, const WalkJob& job, cudaStream_t st);
// fills the far-field grid (distance to any boundary primitive at every vertex)
void launch_farfield2(const SceneView2& S, const FarField& F, float* d, cudaStream_t st);
void launch_sil_count3(const bvc_dev::Prim3* prims, int n, const int4* triSil, int* counts, cudaStream_t st);
void launch_sil_fill3(bvc_dev::Prim3* prims, int n, const int4* triSil, const int* counts, const int* offsets,
                      const float4* silA, const float4* silN1, const float4* silN2, const float4* silB,
                      const float4* triN, float4* rec, cudaStream_t st);
// entries / fronts false: the records hold the root / the single entry node instead
void launch_hintgrid2(const SceneView2& S, const HintGrid& G, HintCell* cells, bool entries, bool fronts, float rmin,
                      cudaStream_t st);
void launch_hintgrid3(const bvc_dev::SceneView3& S, const HintGrid& G, HintCell* cells, bool entries, bool fronts,
                      float rmin, cudaStream_t st);
void launch_farfield3(const bvc_dev::SceneView3& S, const FarField& F, float* d, cudaStream_t st);

// per-point mean / standard error (runWalks pointwise.cpp:167-186), fixed order
void launch_reduce_estimates(const float* vals, int nPts, int per, int comps, int comp, double* mean,
                             double* se, cudaStream_t st);

// device boundary sampler (BoundarySampler::sample sampling.cpp:37-44)
struct CacheSample {
    float z[3];
    float n[3];
    float pdf, uHat, dHat, weight, arc;
    int segment;
};
static_assert(sizeof(CacheSample) == 48, "packed cache sample is 48 bytes");

struct SourceSampleDev {
    float y[3];
    float pdf, f;
    float pad[3];
};
static_assert(sizeof(SourceSampleDev) == 32, "packed source sample is 32 bytes");

// k-th sample of `count` draws u = stratified ? (k + U)/count : U from Philox
// (key, counter = ctr[j] or begin + j), then the CDF lookup of fromUnit (sampling.cpp:20-35)
void launch_sample_boundary(const double* cdf, const int* ids, int m, double total, const float4* segAB,
                            const float2* segNormal, const float* segArc, const float* segLen, int count,
                            int begin, int n, const long long* ctr, int stratified, uint32_t k0, uint32_t k1,
                            CacheSample* out, cudaStream_t st);

// per-sample preparation for cache generation (cache.cpp:318-352): walk start
// (z, or z - eps/2 n on known-Neumann pieces), D flag, first-ball radius
// (gradientBallRadius pointwise.cpp:217-221), interior check (requireInterior
// pointwise.cpp:188-191) and the exact Neumann data h(z) for Neumann samples
void launch_prepare_samples(const WalkEnv& env, CacheSample* samples, int n, const int* regionKinds,
                            const int* regionSource, float2* startU, int* isD, float* gradR, uint8_t* outside,
                            cudaStream_t st);

// gathers the D points of a cache job from their samples
// nD: the count, or with nDdev (device count) the capacity
void launch_gather_dpoints(const CacheSample* samples, const int* dIdx, int nD, const float* gradR,
                           long long gidBase, const long long* gid, float2* xD, float2* nD_, float* rD,
                           long long* gidD, cudaStream_t st, const int* nDdev = nullptr);

// writes uHat / dHat means into the cache samples and flags non-finite results; with
// nDdev the D-point count is read on the device (nDpts = capacity) and, with walksCtr,
// the job's walk count n nU + nD nDw is added there
void launch_finish_samples(CacheSample* samples, int n, const float* outU, int nU, const int* dIdx, int nDpts,
                           const float* outD, int nD, uint8_t* failed, cudaStream_t st, const int* nDdev = nullptr,
                           unsigned long long* walksCtr = nullptr);
// compaction of nonzero byte flags (failed samples) into indices with a device count
void launch_compact_u8(const uint8_t* flags, int n, int* outIdx, int* outCount, cudaStream_t st);

// single-CTA stream compaction of nonzero flags; writes the count to *outCount
void launch_compact(const int* flags, int n, int* outIdx, int* outCount, cudaStream_t st);

// scene queries for the ABI (batched)
void launch_closest(const SceneView2& S, const double* x, int n, unsigned mask, double* point, double* dist,
                    int* seg, double* t, cudaStream_t st);
void launch_silhouette(const SceneView2& S, const double* x, int n, double* dist, cudaStream_t st);
void launch_ray(const SceneView2& S, const double* o, const double* d, int n, double tMax, unsigned mask,
                double tMin, double* t, int* seg, double* point, double* s, cudaStream_t st);
void launch_inside(const SceneView2& S, const double* x, int n, float tol, uint8_t* out, cudaStream_t st);

// kernel-launch accounting (bench gpu_launches)
void count_launch(int n = 1);
// GPU linear BVH build (lbvh.cu): nodes in Node2/Node3 format, primitives in leaf
// order; returns the tree height, or -1 if n <= leafSize
int build_lbvh(int dim, const float4* a, const float4* b, const float4* c, const int* cls, const int2* sil, int n,
               int leafSize, const double* lo, const double* hi, double pad, int classFirst, void* nodesOut,
               void* primsOut, cudaStream_t st);
// GPU binned-SAH build (sahbvh.cu): nodes plus the leaf order of the ids; returns the
// number of levels, or -1 if n <= leafSize
int build_sah_gpu(int dim, const float4* a, const float4* b, const float4* c, const int* cls, int n, int leafSize,
                  double pad, int classFirst, void* nodesOut, int* idsOut, cudaStream_t st);
// first-step warm starts for cache walks: the scene primitive a sample's region
// segment came from, if Dirichlet (its distance seeds the first closest-point query)
void launch_start_hints(const CacheSample* samples, int n, const int* source, const int* cls, const int* leafOf,
                        const int* dIdx, int nD, int* hintU, int* hintD, cudaStream_t st, const int* nDdev = nullptr);
void launch_leaf_index(int dim, const void* prims, int n, int* leafOf, cudaStream_t st);
void launch_leaf_prims(int dim, const float4* a, const float4* b, const float4* c, const int* cls, const int2* sil,
                       const int* ids, int n, void* primsOut, cudaStream_t st);

// ---------------------------------------------------------------------------
// 3D (triangle meshes; walk3.cu)
// ---------------------------------------------------------------------------
struct WalkEnv3 {
    bvc_dev::SceneView3 S;
    // silhouette-edge blocks in leaf order: per triangle a header (n_t, delta'^2) then its
    // edge records (a, n1, n2, b); Prim3.c.w = float4 offset << 2 | edge count (walk3.cu)
    const float4* silRec;
    const int4* triSil;   // by triangle id: up to 3 silhouette-edge slots
    const float4* silA;   // silhouette edge endpoints
    const float4* silB;
    const float4* silN1;  // adjacent Neumann face normals (silN1.w != 0: open edge)
    const float4* silN2;
    DevProblem P;
    float eps, rmin, tguard, insideTol, scale, nudge;
    float cx, cy, cz, escape;
    int maxSteps;
    int hasNeumann, hasH, closed;
    uint32_t k0, k1;
    FarField ff;
    HintGrid hg;
};

struct WalkJob3 {
    int nU, nPtsU;
    const float4* startU;
    const long long* gidU;
    long long gidBaseU;
    float* outU;
    int* truncU;
    int nD, nPtsD;
    const int* nPtsDdev;  // device count of the D points (then nPtsD is only the capacity), or NULL
    const float4* xD;
    const float4* normalD;  // NULL => vector output (3 components)
    const float* radiusD;
    const long long* gidD;
    float* outD;
    int* truncD;
    unsigned long long* truncTotal;
    unsigned long long* steps;
    unsigned long long* counter;
    // first-step warm starts (may be NULL): leaf index of a Dirichlet triangle per U / D point
    const int* hintU;
    const int* hintD;
};

void launch_walk_job3(const WalkEnv3& env, const WalkJob3& job, cudaStream_t st);
void launch_sample_mesh(const double* cdf, int m, double total, const float4* triA, const float4* triB,
                        const float4* triC, const float4* triN, int count, int begin, int n, const long long* ctr,
                        int stratified, uint32_t k0, uint32_t k1, CacheSample* out, cudaStream_t st);
void launch_prepare3(const WalkEnv3& env, CacheSample* samples, int n, const int* kinds, float4* startU, int* isD,
                     float* gradR, uint8_t* outside, cudaStream_t st);
void launch_gather_dpoints3(const CacheSample* samples, const int* dIdx, int nD, const float* gradR, long long gidBase,
                            const long long* gid, float4* xD, float4* nD_, float* rD, long long* gidD, cudaStream_t st,
                            const int* nDdev = nullptr);
void launch_closest3(const bvc_dev::SceneView3& S, const double* x, int n, unsigned mask, double* point, double* dist,
                     int* tri, cudaStream_t st);
void launch_inside3(const bvc_dev::SceneView3& S, const double* x, int n, float tol, uint8_t* out, cudaStream_t st);
void launch_mark3(const bvc_dev::SceneView3& scene, const bvc_dev::SceneView3& region, const double* x, int n,
                  float offset, int whole, float insideTol, uint8_t* fb, uint8_t* gu, cudaStream_t st);

}  // namespace bvc_impl
