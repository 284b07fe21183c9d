// capi_splat.cu — the dense interior evaluation: splatSolution / splatGradient
// (cache.cpp:426-497), correctedBoundarySplat / correctedSourceSplat (499-597) and
// updateSolution's round with its clamp-mode dispatch (622-684).
#include <cub/device/device_scan.cuh>

#include "capi_common.cuh"

namespace bvc_capi {

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
            KernelTimer::begin(KernelTimer::kGather);
            launch_gather64(kind, plan, pack64, N, M, px64, K, dim, cfg.coincidenceTol, val, grad, part, skipB, skipS,
                            ws().get<unsigned>(kWsUnitCtr, 1), g_stream);
            KernelTimer::end(KernelTimer::kGather);
            launch_finalize(part, plan, K, P->order.p + begin, N, M, val, grad, dim, skipB, skipS, P->dev(), g_stream);
        }
        CK(cudaGetLastError());
        return;
    }
    // screened 3D values gather in scaled coordinates (gather.h kScr3V): one FP32 op less per pair
    if (kind == kScr3 && val && !grad && mode == 0) kind = kScr3V;
    const float k = kind == kScr3V ? scr3v_scale(cfg.kernel.sigma) : 1.0f;
    float4* pack = ws().get<float4>(kWsPack, 2 * static_cast<size_t>(std::max(N + M, 1)));
    GatherPlan plan = plan_gather(kind, K, N, M, val, grad);
    double* part = ws().get<double>(kWsPart, std::max<size_t>(static_cast<size_t>(plan.chunksB + plan.chunksS) * plan.comps * K, 1));
    int* skipB = ws().get<int>(kWsSkipB, K);
    int* skipS = ws().get<int>(kWsSkipS, K);
    float4* tileBox = ws().get<float4>(kWsTileBox, 2 * static_cast<size_t>((N + 255) / 256 + (M + 255) / 256 + 1));
    unsigned* unitCtr = ws().get<unsigned>(kWsUnitCtr, 1);
    // one launch: pack + tile boxes + zeroed skips and unit queue
    launch_prologue(b ? b->samples.p : nullptr, N, s ? s->samples.p : nullptr, M, kind, cfg.voronoi, k, pack, tileBox,
                    unitCtr, skipB, skipS, K, g_stream);
    float* ballRs = nullptr;
    if (mode & kModeBall) {
        ballRs = ws().get<float>(kWsBallRs, K);
        launch_gather_f32(P->ballR.p, P->order.p + begin, K, ballRs, g_stream);
    }
    if (N + M > 0) {
        KernelTimer::begin(KernelTimer::kGather);
        launch_gather(kind, plan, pack, N, M, P->xs.p + static_cast<size_t>(dim) * begin, K, dim,
                      static_cast<float>(cfg.kernel.sigma), static_cast<float>(cfg.coincidenceTol), val, grad, part,
                      skipB, skipS, tileBox, unitCtr, g_stream, mode, static_cast<float>(clamp), ballRs);
        KernelTimer::end(KernelTimer::kGather);
    } else
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
           size_t begin, size_t end, bool val, bool grad, int mode, double clamp) {
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
    E.base = P->base;
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
                     P->ballR.p, K, to_dev(*f), clamp, static_cast<double>(s ? s->m : 0), k0, k1, P->base, P->ssum.p,
                     g_stream);
    CK(cudaGetLastError());
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

// One progressive round (updateSolution cache.cpp:622-684). The fallback-band walks
// (cache.cpp:665-681) do not depend on the cache: they run on a second stream with its
// own workspace, started right after the cache-walk job is enqueued, so they overlap
// the cache walks instead of following the splats (their duration is the longest band
// walk's serial latency, ~0.3 ms on C2, however few band points there are). `points` runs
// first on that stream and returns the evaluation points (the host-buffer round uploads
// and classifies them there). The results equal the sequential order's: the band walks
// and the splats write different fields, with the same per-point RNG streams.
void update_round(bvc_scene_s* s, const bvc_problem& pb, bvc_region_s* r, const bvc_cache_config& cfg,
                  const std::function<bvc_eval_points_s*()>& points, uint64_t seed, uint64_t round, int gradients,
                  bvc_round_stats* stats, const bvc_boundary_evaluator* correctionEval) {
    require_device();
    need(s && r, "null argument");
    validate_kernel(pb.kernel);
    if (cfg.sourceBall && gradients) throw Error(BVC_ERR_SOLVER, "ball-kernel source mode does not support gradient splats");
    make_splat_config(s, pb, cfg);  // validates the mode (cache.cpp:628)
    need(cfg.clampMode >= BVC_CLAMP_OFF && cfg.clampMode <= BVC_CLAMP_CORRECT, "unknown clamp mode");
    s->upload();
    r->upload();
    cudaEvent_t e0 = round_event(2), e1 = round_event(3), e2 = round_event(4);
    cudaEvent_t ready = round_event(0), sideDone = round_event(1);
    KernelTimer::arm();
    CK(cudaEventRecord(e0, g_stream));
    CK(cudaEventRecord(ready, g_stream));  // uploads and earlier rounds precede the side stream's work
    bvc_eval_points_s* p = nullptr;
    bool sideRan = false;
    auto side = [&] {
        SideScope scope;
        CK(cudaStreamWaitEvent(g_stream, ready, 0));
        p = points();
        need(p != nullptr, "null evaluation points");
        fallback_walks(s, pb, cfg, p, seed, round, gradients != 0);
        CK(cudaEventRecord(sideDone, g_stream));
        sideRan = true;
    };
    g_afterWalkLaunch = side;
    bvc_boundary_cache_s bc;
    bvc_source_cache_s sc;
    GenStats st;
    try {
        generate_cache(s, pb, r, cfg, seed, round, 0, std::max(1, cfg.nBoundary), &bc, st);
        if (!sideRan) after_walk_launch();  // no cache-walk job was launched
    } catch (...) {
        g_afterWalkLaunch = nullptr;
        throw;
    }
    g_afterWalkLaunch = nullptr;
    generate_source(pb, r, cfg, seed, round, &sc);
    CK(cudaEventRecord(e1, g_stream));
    CK(cudaStreamWaitEvent(g_stream, sideDone, 0));
    splat_round(s, pb, r, cfg, &bc, sc.m ? &sc : nullptr, p, seed, round, gradients, correctionEval);
    CK(cudaEventRecord(e2, g_stream));
    CK(cudaEventSynchronize(e2));
    KernelTimer::resolve();
    st.resolve();
    if (stats) {
        stats->resampled = st.resampled;
        stats->cacheWalks = st.walks;
        stats->cacheTruncated = st.truncated;
        stats->cacheSteps = st.steps;
        stats->generateSeconds = device_seconds(e0, e1);
        stats->splatSeconds = device_seconds(e1, e2);
    }
}

void splat_round(bvc_scene_s* s, const bvc_problem& pb, bvc_region_s* r, const bvc_cache_config& cfg,
                 bvc_boundary_cache_s* bc, bvc_source_cache_s* sp, bvc_eval_points_s* p, uint64_t seed,
                 uint64_t round, int gradients, const bvc_boundary_evaluator* correctionEval) {
    bvc_splat_config scfg = make_splat_config(s, pb, cfg);
    bool hasSource = pb.f.kind != BVC_FIELD_NONE;
    // the mode dispatch of updateSolution (cache.cpp:639-662)
    if (cfg.clampMode == BVC_CLAMP_OFF) {
        // ball mode: splatSolution with G^B plus the unclamped (infinite-bound,
        // correction-free) ball source splat, i.e. one ball-kernel splat
        splat(bc, sp, p, scfg, 0, SIZE_MAX, true, gradients != 0);
    } else {
        double c = cfg.clamp > 0.0 ? cfg.clamp : 10.0 / s->host.diagonal;  // resolvedClamp cache.h:129-131
        // correctionEval (cache.cpp:646-648): the caller's evaluator, or, when it is
        // empty (NULL / NONE), makeDefaultEvaluator's walks (cache.cpp:600-620)
        bvc_boundary_evaluator ev{};
        if (correctionEval && correctionEval->kind != BVC_EVALUATOR_NONE) {
            ev = *correctionEval;
        } else {
            ev.kind = BVC_EVALUATOR_WALKS;
            ev.scene = s;
            ev.problem = &pb;
            ev.cfg = &cfg;
        }
        corrected_boundary(bc, p, r, scfg, c, cfg.clampMode, &ev, seed, bvc_dev::mixKey(kBoundaryCorrSalt, round));
        if (hasSource) {
            if (cfg.sourceBall) {
                corrected_source(sp, p, r, scfg, c, &pb.f, seed, bvc_dev::mixKey(kSourceCorrSalt, round));
            } else {
                splat(nullptr, sp, p, scfg, 0, SIZE_MAX, true, false);
            }
        }
        if (gradients) splat(bc, sp, p, scfg, 0, SIZE_MAX, false, true);
    }
}

// runSolveInMemory's round on host-resident points (runner.cpp:116-169: build the
// points, markEvaluationPoints, updateSolution, read solution() / gradient()). The
// points' upload, Morton order and classification run on the second stream, with the
// band walks, while the cache walks run; the result equals the handle-based sequence
// bit for bit.
void update_round_host(bvc_scene_s* s, const bvc_problem& pb, bvc_region_s* r, const bvc_cache_config& cfg,
                       const double* x, size_t n, uint64_t seed, uint64_t round, int gradients, double* u, double* grad,
                       bvc_round_stats* stats) {
    require_device();
    need(s && r && (x || n == 0) && (u || n == 0), "null argument");
    need(!grad || gradients, "gradient output requested without gradients");
    s->upload();
    r->upload();
    std::unique_ptr<bvc_eval_points_s> P;
    update_round(s, pb, r, cfg,
                 [&]() -> bvc_eval_points_s* {  // on the side stream
                     P = make_points(x, n, s->host.dim);
                     mark_points(s, r, cfg, P.get());
                     ensure_order(P.get());
                     return P.get();
                 },
                 seed, round, gradients, stats, nullptr);
    if (n == 0) return;
    const int d = P->dim;
    double* o = ws().get<double>(kWsEvalOut, (1 + d) * n);
    launch_solution(P.get(), o, o + n);
    CK(cudaMemcpyAsync(u, o, n * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
    if (grad) CK(cudaMemcpyAsync(grad, o + n, d * n * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
    CK(cudaStreamSynchronize(g_stream));
}

}  // namespace bvc_capi

extern "C" {

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
        need(s && pb && r && cfg && p, "null argument");
        update_round(s, *pb, r, *cfg, [p]() { return p; }, seed, round, gradients, stats, nullptr);
    })
}

int bvc_update_solution_with_evaluator(bvc_scene s, const bvc_problem* pb, bvc_region r,
                                       const bvc_cache_config* cfg, bvc_eval_points p, uint64_t seed,
                                       uint64_t round, int gradients, const bvc_boundary_evaluator* correctionEval,
                                       bvc_round_stats* stats) {
    API({
        need(s && pb && r && cfg && p, "null argument");
        if (correctionEval && correctionEval->kind == BVC_EVALUATOR_WALKS)
            need(correctionEval->scene && correctionEval->problem && correctionEval->cfg, "walk evaluator needs scene, problem and cfg");
        update_round(s, *pb, r, *cfg, [p]() { return p; }, seed, round, gradients, stats, correctionEval);
    })
}

int bvc_update_solution_host(bvc_scene s, const bvc_problem* pb, bvc_region r, const bvc_cache_config* cfg,
                             const double* x, size_t n, uint64_t seed, uint64_t round, int gradients, double* u,
                             double* grad, bvc_round_stats* stats) {
    API({
        need(s && pb && r && cfg, "null argument");
        update_round_host(s, *pb, r, *cfg, x, n, seed, round, gradients, u, grad, stats);
    })
}

}  // extern "C"
