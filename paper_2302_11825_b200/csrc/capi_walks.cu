// capi_walks.cu — the pointwise estimators of pointwise.h:62-76 (wosSolve, wostSolve,
// wostGradient, wostNormalDerivative) and updateSolution's fallback-band walks
// (cache.cpp:665-681), in 2D and the 3D lift.
#include "capi_common.cuh"

namespace bvc_capi {

// the 3D lift of the estimator job (the reference's solver is 2D-only, pointwise.cpp:23):
// solve (mode 0) and normal derivative (mode 2) with the 3D walk kernel; one stream per
// point exactly as in 2D
void pointwise3(bvc_scene_s* S, const bvc_problem& pb, const double* x, const double* normal, size_t n,
                const bvc_walk_config& cfg, const uint64_t* streams, int mode, double* mean, double* se,
                long long* count, long long* trunc) {
    // mode 1: the 3-component gradient (bvc_wost_gradient3)
    WalkEnv3 E = make_env3(S, pb, cfg, cfg.seed, kPointwiseSalt, 0);
    const int nw = std::max(1, cfg.nWalks);
    const int ni = static_cast<int>(n);
    std::vector<long long> gid(ni);
    for (int i = 0; i < ni; ++i) {
        uint64_t st = streams ? streams[i] : (ni == 1 ? cfg.stream : bvc_dev::mixKey(cfg.stream, i));
        gid[i] = static_cast<long long>(bvc_dev::mix64(st) >> 1);
    }
    double* xd = ws().get<double>(kWsEvalIn, 3 * n);
    CK(cudaMemcpyAsync(xd, x, 3 * n * sizeof(double), cudaMemcpyHostToDevice, g_stream));
    if (E.insideTol > 0.f) {  // requireInterior (pointwise.cpp:188-191); meaningless for soups
        uint8_t* ins = ws().get<uint8_t>(kWsOutside, n);
        launch_inside3(E.S, xd, ni, E.insideTol, ins, g_stream);
        std::vector<uint8_t> h(n);
        CK(cudaMemcpyAsync(h.data(), ins, n, cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
        for (size_t i = 0; i < n; ++i)
            if (!h[i]) throw Error(BVC_ERR_SOLVER, "evaluation point lies outside the domain");
    }
    std::vector<float4> hx(n);
    for (size_t i = 0; i < n; ++i)
        hx[i] = make_float4(static_cast<float>(x[3 * i]), static_cast<float>(x[3 * i + 1]),
                            static_cast<float>(x[3 * i + 2]), 0.f);
    float4* px = ws().get<float4>(kWsStartU, n);
    CK(cudaMemcpyAsync(px, hx.data(), n * sizeof(float4), cudaMemcpyHostToDevice, g_stream));
    long long* dg = ws().get<long long>(kWsGidU, n);
    CK(cudaMemcpyAsync(dg, gid.data(), n * sizeof(long long), cudaMemcpyHostToDevice, g_stream));
    int* tr = ws().get<int>(kWsTruncPt, n);
    CK(cudaMemsetAsync(tr, 0, n * sizeof(int), g_stream));
    auto* ctr = ws().get<unsigned long long>(kWsCounter, 3);
    CK(cudaMemsetAsync(ctr, 0, 3 * sizeof(unsigned long long), g_stream));
    WalkJob3 J{};
    J.counter = ctr;
    J.steps = ctr + 1;
    J.truncTotal = ctr + 2;
    if (mode == 0) {
        J.nU = nw;
        J.nPtsU = ni;
        J.startU = px;
        J.gidU = dg;
        J.outU = ws().get<float>(kWsOutU, n * nw);
        J.truncU = tr;
    } else {
        // gradientBallRadius: closest point on the whole boundary (pointwise.cpp:217-221)
        double* cpp = ws().get<double>(kWsEvalOut, 3 * n);
        double* cpd = ws().get<double>(kWsMean2, n);
        int* cps = ws().get<int>(kWsSkipB, n);
        launch_closest3(E.S, xd, ni, bvc_dev::kClsAny, cpp, cpd, cps, g_stream);
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
            std::vector<float4> hn(n);
            for (size_t i = 0; i < n; ++i)
                hn[i] = make_float4(static_cast<float>(normal[3 * i]), static_cast<float>(normal[3 * i + 1]),
                                    static_cast<float>(normal[3 * i + 2]), 0.f);
            float4* dn = ws().get<float4>(kWsND, n);
            CK(cudaMemcpyAsync(dn, hn.data(), n * sizeof(float4), cudaMemcpyHostToDevice, g_stream));
            J.normalD = dn;
        }
        J.outD = ws().get<float>(kWsOutD, n * nw * (mode == 1 ? 3 : 1));
    }
    launch_walk_job3(E, J, g_stream);
    const int comps = mode == 1 ? 3 : 1;
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

// estimator job over host points (pointwise.h:62-76)
void pointwise(bvc_scene_s* S, const bvc_problem& pb, const double* x, const double* normal, size_t n,
               const bvc_walk_config& cfg, const uint64_t* streams, int mode, double* mean, double* se,
               long long* count, long long* trunc) {
    // mode 0: wos / wost solve, 1: gradient (2 comps), 2: normal derivative
    require_device();
    need(S && x, "null scene or points");
    if (n == 0) return;
    if (S->host.dim == 3) {
        pointwise3(S, pb, x, normal, n, cfg, streams, mode, mean, se, count, trunc);
        return;
    }
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

__global__ void gather_fallback_kernel(const int* idx, int n, const double* x, float2* out, long long* gid,
                                       long long base) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int p = idx[j];
    out[j] = make_float2(static_cast<float>(x[2 * p]), static_cast<float>(x[2 * p + 1]));
    gid[j] = base + p;  // global point index: the same walk streams on any shard
}

__global__ void gather_fallback3_kernel(const int* idx, int n, const double* x, float4* out, long long* gid,
                                        double* xd, long long base) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int p = idx[j];
    out[j] = make_float4(static_cast<float>(x[3 * p]), static_cast<float>(x[3 * p + 1]), static_cast<float>(x[3 * p + 2]), 0.f);
    gid[j] = base + p;  // global point index: the same walk streams on any shard
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
    gather_fallback3_kernel<<<(nf + 127) / 128, 128, 0, g_stream>>>(idx, nf, P->x.p, px, gid, xd, P->base);
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
    gather_fallback_kernel<<<(nf + 127) / 128, 128, 0, g_stream>>>(idx, nf, P->x.p, px, gid, P->base);
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

}  // namespace bvc_capi

extern "C" {

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
        need(s->host.dim == 2, "bvc_wost_gradient is the 2D gradient (3D: bvc_wost_gradient3)");
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
int bvc_wost_gradient3(bvc_scene s, const bvc_problem* pb, const double* x, size_t n, const bvc_walk_config* cfg,
                       const uint64_t* streams, double* mean, double* se, long long* count, long long* truncated) {
    API({
        need(s && pb && cfg && mean && se, "null argument");
        need(s->host.dim == 3, "bvc_wost_gradient3 is the 3D gradient (2D: bvc_wost_gradient)");
        std::vector<long long> c(n), t(n);
        pointwise(s, *pb, x, nullptr, n, *cfg, streams, 1, mean, se, c.data(), t.data());
        for (size_t i = 0; i < n; ++i) {
            if (count) count[i] = c[i];
            if (truncated) truncated[i] = t[i];
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

}  // extern "C"
