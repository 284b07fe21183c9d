/*
 * bvc_b200.h — C ABI of the B200-native boundary-value-caching (BVC) hot path.
 *
 * Drop-in boundary for the reference's operator API, which is the C++ library
 * API of /root/reference/proj/core (no FFI layer exists upstream).
 * Each entry point below names the reference symbol it replaces (file:line under
 * /root/reference/proj/core). Conventions kept from the reference:
 *   - splats ACCUMULATE into caller-owned evaluation points (cache.cpp:455-459);
 *   - results are deterministic for a fixed (seed, round) and independent of the
 *     launch geometry / GPU count (test_cache.cpp:321-347, 609-621);
 *   - C++ exceptions become status codes + bvc_last_error().
 * No torch types and no CUDA types appear in the signatures: streams are passed
 * as void* (cudaStream_t), device memory is owned by the opaque handles.
 */
#ifndef BVC_B200_H
#define BVC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BVC_ABI_VERSION 3

/* ---- status codes (exception classes of the reference) ------------------- */
typedef enum {
    BVC_OK = 0,
    BVC_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument                   */
    BVC_ERR_PARSE = 2,            /* ParseError           scene.h:14-16      */
    BVC_ERR_SOLVER = 3,           /* SolverError          pointwise.h:13-15  */
    BVC_ERR_SINGULARITY = 4,      /* KernelSingularity    kernels.h:12-14    */
    BVC_ERR_DOMAIN = 5,           /* std::domain_error                       */
    BVC_ERR_CUDA = 6,             /* device / driver failure                 */
    BVC_ERR_NO_DEVICE = 7         /* no CUDA device: there is no CPU fallback */
} bvc_status;

/* ---- enums mirroring the reference ---------------------------------------- */
typedef enum { BVC_DIRICHLET = 0, BVC_NEUMANN = 1 } bvc_label;          /* scene.h:18 */
typedef enum { BVC_FILTER_ANY = 0, BVC_FILTER_DIRICHLET = 1,
               BVC_FILTER_NEUMANN = 2 } bvc_filter;                     /* scene.h:20 */
typedef enum { BVC_KERNEL_POISSON = 0, BVC_KERNEL_SCREENED = 1 } bvc_kernel_kind; /* kernels.h:16 */
typedef enum { BVC_REGION_WHOLE_DOMAIN = 0, BVC_REGION_SUBDOMAIN = 1 } bvc_region_mode; /* cache.h:32 */
typedef enum { BVC_SEG_KNOWN_NEUMANN = 0, BVC_SEG_ESTIMATED_OFFSET = 1,
               BVC_SEG_USER_LOOP = 2 } bvc_region_segment_kind;         /* cache.h:11-15 */
typedef enum { BVC_CLAMP_OFF = 0, BVC_CLAMP_ONLY = 1, BVC_CLAMP_CORRECT = 2 } bvc_clamp_mode; /* cache.h:112 */

/* KernelSpec (kernels.h:25-43) */
typedef struct {
    int kind;      /* bvc_kernel_kind */
    double sigma;  /* 0 iff Poisson */
    int dim;       /* 2 or 3 */
    double scale;  /* scene scale for the singularity guard (kernels.h:56-59) */
} bvc_kernel_spec;

/*
 * Device-evaluable field descriptors. They replace the std::function callbacks
 * of PdeProblem (pointwise.h:19-26), which cannot run on a GPU.
 * Names follow the CLI's named fields (tools/src/fields.cpp:30-72) plus the
 * fields BASELINE.json's configs need. BVC_FIELD_NONE is the empty callback
 * (no source / no Neumann data), distinct from a constant 0.
 */
typedef enum {
    BVC_FIELD_NONE = 0,
    BVC_FIELD_CONSTANT = 1,      /* p[0]                                          */
    BVC_FIELD_LINEAR = 2,        /* p[0]*x + p[1]*y + p[3]*z + p[2]               */
    BVC_FIELD_RADIAL = 3,        /* p[2]*|x - (p0,p1)|^p[3] + p[4]                */
    BVC_FIELD_HARMONIC_POLY = 4, /* p[1]*Re(z^d) + p[2]*Im(z^d), d = (int)p[0]    */
    BVC_FIELD_CHECKERBOARD = 5,  /* origin (p0,p1), cell p2, lo p3, hi p4         */
    BVC_FIELD_SIN_COS = 6,       /* p0*sin(p1*x + p2)*cos(p3*y + p4)              */
    BVC_FIELD_GAUSSIAN_SUM = 7,  /* n terms: sum a_m exp(-|x-c_m|^2 / (2 p0^2));
                                    term m at p[1+4m..4+4m] = (cx, cy, cz, a)     */
    BVC_FIELD_QUADRATIC3 = 8,    /* c + cx x + cy y + cz z + cxx x^2 + cyy y^2 +
                                    czz z^2 + cxy xy + cxz xz + cyz yz (p0..p9)   */
    BVC_FIELD_TRIG3 = 9          /* p0*sin(p1 x) + p2*cos(p3 y) + p4*z + p5       */
} bvc_field_kind;

#define BVC_FIELD_MAX_PARAMS 68
typedef struct {
    int kind;  /* bvc_field_kind */
    int n;     /* term count for GAUSSIAN_SUM (<= 16) */
    double p[BVC_FIELD_MAX_PARAMS];
} bvc_field;

/* PdeProblem (pointwise.h:19-26): Delta u - sigma u = f, u = g on D, du/dn = h on N */
typedef struct {
    bvc_kernel_spec kernel;
    bvc_field f; /* NONE => zero source (hasSource() false) */
    bvc_field g; /* Dirichlet data */
    bvc_field h; /* NONE => zero Neumann data, term skipped (pointwise.cpp:227) */
} bvc_problem;

/* WalkConfig (pointwise.h:28-45) */
typedef struct {
    double epsilon; /* 0 => 1e-3 * scene diagonal */
    double rMin;    /* 0 => epsilon */
    int maxSteps;   /* default 10000 */
    int nWalks;     /* default 128 */
    uint64_t seed;
    uint64_t stream;
} bvc_walk_config;

/* CacheConfig (cache.h:114-132) */
typedef struct {
    int nBoundary;       /* N, default 1024 */
    int nSource;         /* M, default 1024 */
    int nWalksNeumann;   /* u-walk budget, default 16 */
    int nWalksDirichlet; /* du/dn walk budget, default 160 */
    double offset;       /* l; 0 => 5 epsilon */
    double clamp;        /* c; 0 => 10 / diagonal */
    int clampMode;       /* bvc_clamp_mode */
    int sourceBall;      /* ball-kernel source mode (Poisson, 2D) */
    int correctionWalks; /* default 4 */
    int voronoi;         /* Voronoi weights instead of 1/(N pdf) */
    int stratified;      /* default 1 */
    bvc_walk_config walk;
    int threads;         /* ignored: the GPU launch geometry is internal */
} bvc_cache_config;

/* RegionRequest (cache.h:31-36) */
typedef struct bvc_scene_s* bvc_scene;
typedef struct {
    int mode;          /* bvc_region_mode */
    double offset;     /* l; 0 => 5 epsilon */
    bvc_scene subdomain; /* closed user loop for SUBDOMAIN mode */
} bvc_region_request;

/* RoundStats (cache.h:134-140) */
typedef struct {
    long long resampled;
    long long cacheWalks;
    long long cacheTruncated;
    long long cacheSteps;    /* GPU extra: closest-Dirichlet queries (pointwise.cpp:216) */
    double generateSeconds;
    double splatSeconds;
} bvc_round_stats;

/* ScalarEstimate / VectorEstimate (pointwise.h:47-59) */
typedef struct { double mean, se; long long count, truncated; } bvc_scalar_estimate;
typedef struct { double mean[2], se[2]; long long count, truncated; } bvc_vector_estimate;

/* SplatConfig (cache.h:143-149) */
typedef struct {
    bvc_kernel_spec kernel; /* scale = scene diagonal */
    double coincidenceTol;  /* 1e-12 x diagonal */
    int voronoi;
    int useBallGreens;      /* G -> G^B(x, ballRadius) in the d-hat and source terms */
    int fp64;               /* GPU extra: evaluate every pair in FP64 (Poisson kernels; BASELINE C1 fp64) */
} bvc_splat_config;

/* CachedBoundarySample (cache.h:43-52), host AoS exchange format (2D or 3D) */
typedef struct {
    double z[3], n[3];
    double pdf, uHat, dHat, weight;
    int segment;
    double arc;
} bvc_boundary_sample;

/* CachedSourceSample (cache.h:61-65) */
typedef struct { double y[3]; double pdf, f; } bvc_source_sample;

/* EvaluationPoint (cache.h:73-110), host SoA view for download/upload */
typedef struct {
    size_t count;
    int dim;
    double* x;                 /* dim*count */
    uint8_t* fallback;
    uint8_t* gradientUnreliable;
    double* boundarySum;
    double* sourceSum;
    long long* nBoundary;
    long long* mSource;
    double* boundaryGradSum;   /* dim*count */
    double* sourceGradSum;     /* dim*count */
    long long* nBoundaryGrad;
    long long* mSourceGrad;
    double* walkSum;
    long long* walkCount;
    long long* walkTruncated;
    double* gradientWalkSum;   /* dim*count */
    long long* gradientWalkCount;
    long long* skipped;
    double* ballRadius;        /* ball-kernel mode radius (cache.h:77) */
} bvc_point_state;

typedef struct bvc_region_s* bvc_region;
typedef struct bvc_boundary_cache_s* bvc_boundary_cache;
typedef struct bvc_source_cache_s* bvc_source_cache;
typedef struct bvc_eval_points_s* bvc_eval_points;

/* ---- runtime ---------------------------------------------------------------- */
const char* bvc_last_error(void);            /* message of the last failing call on this thread */
int bvc_abi_version(void);
int bvc_set_device(int device);              /* binds the calling thread's device */
int bvc_set_stream(void* cuda_stream);       /* stream for all subsequent launches (NULL = default) */
int bvc_synchronize(void);
/* launches of this library's kernels since process start (bench gpu_launches) */
long long bvc_kernel_launch_count(void);
/* device time (CUDA events on the launching stream) of the main cache-walk launch and the
   main gather launch of this thread's last updateSolution round (plain or sharded), in
   seconds; 0 for a kernel that round did not launch (the rooflines' per-launch durations) */
int bvc_last_round_kernel_seconds(double* walkSeconds, double* gatherSeconds);
/* pipe / cache microbenchmarks behind the rooflines: which = 0 FFMA,
   1 MUFU.LG2, 2 MUFU.RCP, 3 DFMA, 4 MUFU.RSQ, 5 MUFU.EX2 (instructions/s, per GPU),
   6 L2-resident read bandwidth (bytes/s), 7 FFMA / 8 FMUL / 9 FADD with register
   operands only (no immediate or constant-bank operand), 10 packed FFMA2 (FP32 FMAs/s) */
int bvc_pipe_probe(int which, double* opsPerSecond);

/* ---- scene (Scene::build scene.h:84, scene.cpp:11-125) --------------------- */
/* 2D: vertices = 2*nv doubles, segments = 2*ns vertex ids, labels = ns bvc_label */
int bvc_scene_create(const double* vertices, int nv, const int* segments, const int* labels,
                     int ns, bvc_scene* out);
/* 3D triangle mesh / soup (no reference path): tris = 3*nt ids */
int bvc_scene_create_mesh3(const double* vertices, int nv, const int* tris, const int* labels,
                           int nt, bvc_scene* out);
int bvc_scene_destroy(bvc_scene scene);
/* diagonal, bounds lo/hi (dim each), dirichlet/neumann/total measure, closed flag */
int bvc_scene_info(bvc_scene scene, int* dim, double* diagonal, double* lo, double* hi,
                   double* dirichletLength, double* neumannLength, int* closed, int* nLoops);
/* Scene::closestPoint (scene.h:95; bvh.cpp:53-69), batched over n points on the device.
   Outputs are host arrays (point: dim*n, dist, segment, t); segment = -1 if invalid. */
int bvc_scene_closest_point(bvc_scene scene, const double* x, size_t n, int filter,
                            double* point, double* dist, int* segment, double* t);
/* Scene::silhouetteDistance (scene.h:100; scene.cpp:174-185); +inf if none */
int bvc_scene_silhouette_distance(bvc_scene scene, const double* x, size_t n, double* dist);
/* Scene::intersectRay (scene.h:104; scene.cpp:196-208); segment = -1 on a miss */
int bvc_scene_intersect_ray(bvc_scene scene, const double* o, const double* d, size_t n,
                            double tMax, int filter, double tMin, double* t, int* segment,
                            double* point, double* s);
/* Scene::inside (scene.h:117; scene.cpp:240-254) */
int bvc_scene_inside(bvc_scene scene, const double* x, size_t n, uint8_t* inside);

/* ---- solve region (buildSolveRegion cache.h:41; cache.cpp:137-246) ---------- */
int bvc_region_build(bvc_scene scene, const bvc_region_request* request, double epsilon,
                     bvc_region* out);
int bvc_region_destroy(bvc_region region);
/* region boundary as a scene (vertices/segments), per-segment kinds and source ids */
int bvc_region_info(bvc_region region, int* nv, int* ns, double* offset, double* area,
                    int* wholeDomain);
int bvc_region_export(bvc_region region, double* vertices, int* segments, int* labels,
                      int* kinds, int* sourceSegment);
/* the region boundary as a scene handle owned by the region (do not destroy) */
bvc_scene bvc_region_boundary(bvc_region region);

/* ---- evaluation points (EvaluationPoint cache.h:73-110) --------------------- */
int bvc_points_create(const double* x, size_t n, int dim, bvc_eval_points* out);
int bvc_points_destroy(bvc_eval_points pts);
int bvc_points_download(bvc_eval_points pts, bvc_point_state* host); /* fills non-NULL arrays */
int bvc_points_upload(bvc_eval_points pts, const bvc_point_state* host); /* non-NULL arrays */
/* EvaluationPoint::solution() / gradient() (cache.h:91-105) evaluated on the device;
   u: count doubles, grad: dim*count doubles (either may be NULL) */
int bvc_points_solution(bvc_eval_points pts, double* u, double* grad);
int bvc_points_reset(bvc_eval_points pts);  /* zero all running sums */
/* the global index of this point set's first point when it is one shard of a larger
   set (default 0). Per-point random streams (fallback-band walks, clamp corrections)
   are keyed by base + index, so sharded point sets draw exactly what the whole set
   would draw on one device (the reference keys them by point: cache.cpp:665-681) */
int bvc_points_set_index_base(bvc_eval_points pts, long long base);
/* markEvaluationPoints (cache.h:154; cache.cpp:263-276) */
int bvc_mark_evaluation_points(bvc_scene scene, bvc_region region, const bvc_cache_config* cfg,
                               bvc_eval_points pts);

/* ---- caches ----------------------------------------------------------------- */
/* generateBoundaryCache (cache.h:159-161; cache.cpp:301-390) */
int bvc_generate_boundary_cache(bvc_scene scene, const bvc_problem* problem, bvc_region region,
                                const bvc_cache_config* cfg, uint64_t seed, uint64_t round,
                                bvc_round_stats* stats, bvc_boundary_cache* out);
/* shard [begin, end) of the N samples of a round (multi-GPU; RNG keyed by global index) */
int bvc_generate_boundary_cache_shard(bvc_scene scene, const bvc_problem* problem,
                                      bvc_region region, const bvc_cache_config* cfg,
                                      uint64_t seed, uint64_t round, int begin, int end,
                                      bvc_round_stats* stats, bvc_boundary_cache* out);
/* the shard above plus the fallback-band walks of `pts` (cache.cpp:665-681, as
   bvc_fallback_walks) on a second stream while the shard's walks run: a rank's
   cache work and band walks in one call (the sharded multi-GPU round) */
int bvc_generate_boundary_cache_shard_fallback(bvc_scene scene, const bvc_problem* problem,
                                               bvc_region region, const bvc_cache_config* cfg,
                                               uint64_t seed, uint64_t round, int begin, int end,
                                               bvc_eval_points pts, int gradients,
                                               bvc_round_stats* stats, bvc_boundary_cache* out);
/* generateSourceCache (cache.h:163-164; cache.cpp:392-406) */
int bvc_generate_source_cache(const bvc_problem* problem, bvc_region region,
                              const bvc_cache_config* cfg, uint64_t seed, uint64_t round,
                              bvc_source_cache* out);
int bvc_boundary_cache_create(const bvc_boundary_sample* samples, int n, int dim, int voronoi,
                              double boundaryLength, bvc_boundary_cache* out);
int bvc_boundary_cache_size(bvc_boundary_cache c, int* n, int* dim);
int bvc_boundary_cache_download(bvc_boundary_cache c, bvc_boundary_sample* samples);
/* packed device SoA (8 floats/sample) for the NCCL all-gather of cache shards */
int bvc_boundary_cache_packed(bvc_boundary_cache c, void** device_ptr, size_t* bytes);
int bvc_boundary_cache_from_packed(const void* device_ptr, int n, int dim, int voronoi,
                                   double boundaryLength, bvc_boundary_cache* out);
/* assignVoronoiWeights (cache.cpp:280-297) over a whole round's cache: a sharded
   generation skips it, the all-gathered cache gets it once (multi-GPU + voronoi) */
int bvc_boundary_cache_assign_voronoi(bvc_boundary_cache cache, bvc_region region);
int bvc_boundary_cache_destroy(bvc_boundary_cache c);
int bvc_source_cache_create(const bvc_source_sample* samples, int m, int dim, double area,
                            bvc_source_cache* out);
int bvc_source_cache_size(bvc_source_cache c, int* m, int* dim);
int bvc_source_cache_download(bvc_source_cache c, bvc_source_sample* samples);
int bvc_source_cache_destroy(bvc_source_cache c);

/* ---- splats (the dense interior gather) ------------------------------------- */
/* makeSplatConfig (cache.h:151; cache.cpp:248-261) */
int bvc_make_splat_config(bvc_scene scene, const bvc_problem* problem,
                          const bvc_cache_config* cfg, bvc_splat_config* out);
/* splatSolution (cache.h:168-169; cache.cpp:426-461); scache may be NULL */
int bvc_splat_solution(bvc_boundary_cache bcache, bvc_source_cache scache, bvc_eval_points pts,
                       const bvc_splat_config* cfg);
/* splatGradient (cache.h:172-173; cache.cpp:463-497) */
int bvc_splat_gradient(bvc_boundary_cache bcache, bvc_source_cache scache, bvc_eval_points pts,
                       const bvc_splat_config* cfg);
/* fused: both splats in one pass over the cache (same sums as the two calls) */
int bvc_splat_solution_gradient(bvc_boundary_cache bcache, bvc_source_cache scache,
                                bvc_eval_points pts, const bvc_splat_config* cfg);
/* the same, restricted to points [begin, end) (multi-GPU query sharding) */
int bvc_splat_range(bvc_boundary_cache bcache, bvc_source_cache scache, bvc_eval_points pts,
                    const bvc_splat_config* cfg, size_t begin, size_t end, int value,
                    int gradient);

/* BoundaryEvaluator (cache.h:175-176): the u(z) estimate the clamp correction
   multiplies each saturated crossing by. A std::function cannot cross the C ABI or
   run on the device, so it is one of: NONE (the empty callback), FIELD (exact data
   u(z) = field(z), e.g. the tests' constant evaluators), or WALKS (the default
   evaluator of updateSolution, makeDefaultEvaluator cache.cpp:600-620:
   cfg->correctionWalks WoSt walks in `scene` from each crossing, KnownNeumann
   crossings shifted eps/2 inside). */
typedef enum { BVC_EVALUATOR_NONE = 0, BVC_EVALUATOR_FIELD = 1, BVC_EVALUATOR_WALKS = 2 } bvc_evaluator_kind;
typedef struct {
    int kind;                     /* bvc_evaluator_kind */
    bvc_field field;              /* FIELD */
    bvc_scene scene;              /* WALKS */
    const bvc_problem* problem;   /* WALKS */
    const bvc_cache_config* cfg;  /* WALKS: walk settings and correctionWalks */
} bvc_boundary_evaluator;

/* correctedBoundarySplat (cache.h:178-184; cache.cpp:499-553): boundary splat with
   dG/dn clamped to [-c, c]; CLAMP_CORRECT adds one ray-sampled correction per point
   (RNG keyed by (seed, stream, point index)). eval may be NULL for CLAMP_ONLY. */
int bvc_corrected_boundary_splat(bvc_boundary_cache bcache, bvc_eval_points pts, bvc_region region,
                                 const bvc_splat_config* cfg, double clampBound, int clampMode,
                                 const bvc_boundary_evaluator* eval, uint64_t seed, uint64_t stream);
/* correctedSourceSplat (cache.h:186-191; cache.cpp:555-597): source splat through the
   clamped ball kernel G^B plus one ball-sampled correction per point when clampBound
   is finite and f is not NULL / NONE. 2D Poisson only; points need ball radii. */
int bvc_corrected_source_splat(bvc_source_cache scache, bvc_eval_points pts, bvc_region region,
                               const bvc_splat_config* cfg, double clampBound, const bvc_field* f,
                               uint64_t seed, uint64_t stream);

/* ---- one progressive round (updateSolution cache.h:195-198; cache.cpp:622-684) */
int bvc_update_solution(bvc_scene scene, const bvc_problem* problem, bvc_region region,
                        const bvc_cache_config* cfg, bvc_eval_points pts, uint64_t seed,
                        uint64_t round, int gradients, bvc_round_stats* stats);
/* the same with updateSolution's correctionEval argument (cache.h:195-198, used at
   cache.cpp:646-648): the BoundaryEvaluator the ClampCorrect correction multiplies each
   saturated crossing by. NULL or kind NONE = the empty default, i.e. the reference's
   makeDefaultEvaluator (cfg->correctionWalks walks in `scene`, cache.cpp:600-620);
   FIELD = exact data; WALKS = walks in the evaluator's own scene/problem/cfg. */
int bvc_update_solution_with_evaluator(bvc_scene scene, const bvc_problem* problem,
                                       bvc_region region, const bvc_cache_config* cfg,
                                       bvc_eval_points pts, uint64_t seed, uint64_t round,
                                       int gradients, const bvc_boundary_evaluator* correctionEval,
                                       bvc_round_stats* stats);

/* runSolveInMemory's round on host-resident points (runner.cpp:116-169: points built from
   x, markEvaluationPoints, updateSolution, then solution() / gradient() read back). x is
   n points of the scene's dimension; u receives n values, grad (optional, needs
   gradients) n x dim. Equals bvc_points_create + bvc_mark_evaluation_points +
   bvc_update_solution + bvc_points_solution bit for bit; the upload and classification
   of the points overlap the cache walks (second stream). */
int bvc_update_solution_host(bvc_scene scene, const bvc_problem* problem, bvc_region region,
                             const bvc_cache_config* cfg, const double* x, size_t n, uint64_t seed,
                             uint64_t round, int gradients, double* u, double* grad,
                             bvc_round_stats* stats);

/* ---- multi-GPU rounds (the reference's parallelism is parallelFor only,
        parallel.h:25-50) ------------------------------------------------------ */
/* A communicator over the ranks of one job, one GPU per rank (the device current at
   init). NCCL: one rank creates a 128-byte id (bvc_comm_unique_id), the caller's own
   bootstrap (MPI, a TCP store, torch.distributed, ...) sends it to every rank, each
   calls bvc_comm_init_nccl. Callback: a host-staged exchange supplied by the caller
   (gloo, MPI on host buffers, tests): fn(send, recv, bytes, user, stream) is called with
   the library's stream drained and must, before returning, fill the device buffer recv
   (nranks * bytes) with every rank's device send buffer (bytes) in rank order; nonzero
   return = failure. */
typedef struct bvc_comm_s* bvc_comm;
typedef int (*bvc_allgather_fn)(const void* send, void* recv, size_t bytes, void* user, void* stream);
int bvc_comm_unique_id(void* id /* 128 bytes */);
int bvc_comm_init_nccl(const void* id, int nranks, int rank, bvc_comm* out);
int bvc_comm_init_callback(int nranks, int rank, bvc_allgather_fn fn, void* user, bvc_comm* out);
int bvc_comm_info(bvc_comm comm, int* nranks, int* rank);
int bvc_comm_destroy(bvc_comm comm);
/* rank's contiguous share [begin, end) of n units and the padded per-rank count
   ceil(n / nranks) the all-gather moves (host arithmetic, no device needed) */
int bvc_shard_layout(long long n, int nranks, int rank, long long* begin, long long* end,
                     long long* capacity);
/* updateSolution (cache.cpp:622-684) sharded over the communicator: this rank walks
   its share of the round's boundary samples (RNG keyed by global sample index) while
   its fallback-band walks run on a second stream, one all-gather of the 48-byte
   samples assembles the cache on every rank, every rank builds the source cache and
   gathers its own points `pts` (this rank's slice of the job's points, with
   bvc_points_set_index_base = the slice's global offset). Each point's sums equal the
   single-GPU round's bit for bit. stats: this rank's share. */
int bvc_update_solution_sharded(bvc_comm comm, bvc_scene scene, const bvc_problem* problem,
                                bvc_region region, const bvc_cache_config* cfg, bvc_eval_points pts,
                                uint64_t seed, uint64_t round, int gradients, bvc_round_stats* stats);
/* the same on host buffers (bvc_update_solution_host's sharded form): x = this rank's n
   points (global indices indexBase ...), u (n) and grad (n x dim, optional) receive
   their solution() / gradient(); the upload and classification run under the shard's
   walks */
int bvc_update_solution_sharded_host(bvc_comm comm, bvc_scene scene, const bvc_problem* problem,
                                     bvc_region region, const bvc_cache_config* cfg, const double* x,
                                     size_t n, long long indexBase, uint64_t seed, uint64_t round,
                                     int gradients, double* u, double* grad, bvc_round_stats* stats);

/* the fallback-band walks of updateSolution (cache.cpp:665-681) alone, for the
   sharded multi-GPU round (generate shard, all-gather, splat_range, then this) */
int bvc_fallback_walks(bvc_scene scene, const bvc_problem* problem, const bvc_cache_config* cfg,
                       bvc_eval_points pts, uint64_t seed, uint64_t round, int gradients);

/* ---- streamlines (runStreamlines tools/src/runner.cpp:285-373) -------------- */
typedef enum { BVC_STREAM_OK = 0, BVC_STREAM_OUTSIDE = 1, BVC_STREAM_ZERO_GRADIENT = 2 } bvc_stream_reason;
/* Heun tracing along the unit gradient of `rounds` retained cache rounds (seed,
   round 0..rounds-1), all seeds advancing together (two batched gradient gathers
   per step). points: nSeeds * (steps + 1) * 2 doubles, seed s's polyline at
   [s * (steps + 1) * 2 ...], counts[s] points (0 = the seed itself is outside);
   reasons[s] = bvc_stream_reason (why the trace stopped; OK = ran all steps). */
int bvc_trace_streamlines(bvc_scene scene, const bvc_problem* problem, bvc_region region,
                          const bvc_cache_config* cfg, uint64_t seed, int rounds, const double* seeds,
                          int nSeeds, double step, int steps, double* points, int* counts,
                          int* reasons);

/* ---- data formats -------------------------------------------- */
/* GridField CSV `x,y,value,valid`, %.17g, row-major y-rows (grid.h:35-37, grid.cpp:22-80);
   valid may be NULL (all valid). load: call with values = valid = NULL to read the shape. */
int bvc_grid_save_csv(const char* path, double originX, double originY, double spacing, int nx,
                      int ny, const double* values, const uint8_t* valid);
int bvc_grid_load_csv(const char* path, double* originX, double* originY, double* spacing,
                      int* nx, int* ny, double* values, uint8_t* valid, size_t capacity);
/* rmse over jointly valid nodes (grid.cpp:82-96) */
int bvc_grid_rmse(const double* a, const uint8_t* validA, const double* b, const uint8_t* validB,
                  size_t n, double* out);
/* binary PGM (P5) plus the `.txt` legend (tools/src/image.cpp:12-51) */
int bvc_grid_save_pgm(const char* path, int nx, int ny, const double* values, const uint8_t* valid,
                      int autoRange, double lo, double hi);
/* streamline CSV `seed,step,x,y,reason` (runner.cpp:333-369) */
int bvc_streamlines_write_csv(const char* path, const double* seeds, int nSeeds, int steps,
                              const double* points, const int* counts, const int* reasons);

/* ---- pointwise estimators (pointwise.h:62-76), batched over n points -------- */
/* point i uses cfg->stream for i == 0 when n == 1, else streams[i] (NULL => mixKey(stream,i)).
   x (and normal) hold the scene's dimension per point: 2D as the reference, and the 3D
   lift for triangle meshes (bvc_wost_gradient3 for the 3D gradient) */
int bvc_wos_solve(bvc_scene scene, const bvc_problem* problem, const double* x, size_t n,
                  const bvc_walk_config* cfg, const uint64_t* streams, bvc_scalar_estimate* out);
int bvc_wost_solve(bvc_scene scene, const bvc_problem* problem, const double* x, size_t n,
                   const bvc_walk_config* cfg, const uint64_t* streams, bvc_scalar_estimate* out);
int bvc_wost_gradient(bvc_scene scene, const bvc_problem* problem, const double* x, size_t n,
                      const bvc_walk_config* cfg, const uint64_t* streams,
                      bvc_vector_estimate* out);
/* the 3D lift of wostGradient on triangle meshes: mean/se are 3*n (x, y, z per point),
   count / truncated n each (may be NULL) */
int bvc_wost_gradient3(bvc_scene scene, const bvc_problem* problem, const double* x, size_t n,
                       const bvc_walk_config* cfg, const uint64_t* streams, double* mean, double* se,
                       long long* count, long long* truncated);
int bvc_wost_normal_derivative(bvc_scene scene, const bvc_problem* problem, const double* x,
                               const double* normal, size_t n, const bvc_walk_config* cfg,
                               const uint64_t* streams, bvc_scalar_estimate* out);

/* ---- diagnostics ---------------------------------------------------------- */
/* one generateBoundaryCache with per-thread traversal counters (roofline bytes):
   out = [closest-Dirichlet steps, BVH node fetches (48 B), primitive fetches (32 B), walks] */
int bvc_walk_traffic_profile(bvc_scene scene, const bvc_problem* problem, bvc_region region,
                             const bvc_cache_config* cfg, uint64_t seed, uint64_t round, double* out);

/* ---- free-space kernels (kernels.h:78-129) and Bessel functions (kernels.h:46-49),
        evaluated in the device's FP32 arithmetic for parity tests -------------- */
/* out per point: [G, dG/dx (dim), dG/dn_y, d2G/dx dn_y (dim)] = 2 + 2*dim floats */
int bvc_eval_kernels(const bvc_kernel_spec* spec, const double* x, const double* y,
                     const double* n, size_t count, double* out);
/* which: 0 = K0, 1 = K1, 2 = I0, 3 = I1; FP32 device approximations */
int bvc_eval_bessel(int which, const double* t, size_t count, double* out);

#ifdef __cplusplus
}
#endif
#endif /* BVC_B200_H */
