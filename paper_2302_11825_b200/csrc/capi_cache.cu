// capi_cache.cu — cache construction: generateBoundaryCache (cache.cpp:301-390) with
// its deterministic redraws, assignVoronoiWeights (280-297), generateSourceCache
// (392-406; RegionSampler sampling.cpp:62-108), the walk environments, and the cache
// handle entry points of the C ABI.
#include "capi_common.cuh"

namespace bvc_capi {

WalkEnv make_env(bvc_scene_s* S, const bvc_problem& pb, const bvc_walk_config& wc, uint64_t seed, uint64_t salt,
                 uint64_t round) {
    validate_kernel(pb.kernel);
    if (pb.kernel.dim != 2) throw Error(BVC_ERR_SOLVER, "walk estimators support dim == 2 only");
    WalkEnv E{};
    E.S = S->view();
    E.runSeg = S->runSeg.p;
    E.runId = S->runId.p;
    E.runN = S->runN;
    E.drunSeg = S->drunSeg.p;
    E.drunId = S->drunId.p;
    E.drunN = S->drunN;
    E.nSil = static_cast<int>(S->host.silAlways.size());
    E.P.screened = pb.kernel.kind == BVC_KERNEL_SCREENED;
    E.P.sigma = static_cast<float>(pb.kernel.sigma);
    E.P.sqrtSigma = static_cast<float>(std::sqrt(pb.kernel.sigma));
    E.P.dim = 2;
    E.P.f = to_dev(pb.f);
    E.P.g = to_dev(pb.g);
    E.P.h = to_dev(pb.h);
    double diag = S->host.diagonal;
    double eps = wc.epsilon > 0.0 ? wc.epsilon : 1e-3 * diag;         // pointwise.h:36-38
    double rmin = wc.rMin > 0.0 ? wc.rMin : eps;                        // pointwise.h:39-44
    if (rmin > eps) throw Error(BVC_ERR_INVALID_ARGUMENT, "walk config: r_min must lie in (0, epsilon]");
    E.eps = static_cast<float>(eps);
    E.rmin = static_cast<float>(rmin);
    // the reference's tGuard is 1e-9 diag (pointwise.cpp:115); FP32 positions need a
    // guard above their rounding, and the current segment is skipped explicitly
    E.tguard = static_cast<float>(1e-9 * diag);  // pointwise.cpp:115; the standing segment is skipped
    E.insideTol = S->host.closed() ? static_cast<float>(std::max(1e-9, 1e-7) * diag) : -1.0f;
    E.scale = static_cast<float>(diag);
    E.nudge = static_cast<float>(9.5367431640625e-7 * diag);  // 2^-20 diag, << eps
    E.cx = static_cast<float>(0.5 * (S->host.lo[0] + S->host.hi[0]));
    E.cy = static_cast<float>(0.5 * (S->host.lo[1] + S->host.hi[1]));
    // FP32 safety net: in a closed scene a walker more than one diagonal from the box
    // centre has leaked through the boundary (impossible in exact arithmetic) and ends
    // like a truncated walk. Open scenes (subdomain chains, pointwise solves) keep
    // walking until maxSteps, as the reference does (pointwise.cpp:162-164).
    E.escape = S->host.closed() ? static_cast<float>(diag) : 3.0e38f;
    E.maxSteps = std::max(1, wc.maxSteps);
    E.hasNeumann = S->host.hasNeumann() ? 1 : 0;
    E.hasSource = pb.f.kind != BVC_FIELD_NONE ? 1 : 0;
    E.hasH = pb.h.kind != BVC_FIELD_NONE ? 1 : 0;
    E.closed = S->host.closed() ? 1 : 0;
    if (!(S->host.dirichletMeasure > 0.0))
        throw Error(BVC_ERR_SOLVER, "walk cannot terminate: scene has no Dirichlet boundary");
    key_of(seed, salt, round, E.k0, E.k1);
    E.ff = S->farfield();
    E.hg = S->hintgrid();
    return E;
}

// walks for the samples [0, n) of `samples` (already positioned); writes uHat/dHat
// and returns per-sample failure flags in `failed` (device)
void run_cache_walks(bvc_scene_s* S, bvc_region_s* R, const WalkEnv& E, const bvc_cache_config& cfg,
                     CacheSample* samples, int n, long long gidBase, const long long* gid, uint8_t* failed,
                     GenStats& st) {
    float2* startU = ws().get<float2>(kWsStartU, n);
    int* isD = ws().get<int>(kWsIsD, n);
    float* gradR = ws().get<float>(kWsGradR, n);
    launch_prepare_samples(E, samples, n, R->kinds.p, R->source.p, startU, isD, gradR, failed, g_stream);
    int* dIdx = ws().get<int>(kWsDIdx, n);
    int* cnt = ws().get<int>(kWsCount, 1);
    launch_compact(isD, n, dIdx, cnt, g_stream);
    // the D points stay on the device: buffers sized for all n samples, kernels read the
    // count (no host round trip between the compaction and the walks)
    float2* xD = ws().get<float2>(kWsXD, n);
    float2* nrmD = ws().get<float2>(kWsND, n);
    float* rD = ws().get<float>(kWsRD, n);
    long long* gidD = ws().get<long long>(kWsGidD, n);
    launch_gather_dpoints(samples, dIdx, n, gradR, gidBase, gid, xD, nrmD, rD, gidD, g_stream, cnt);
    int nU = std::max(1, cfg.nWalksNeumann), nDw = std::max(1, cfg.nWalksDirichlet);
    int* hintU = ws().get<int>(kWsHintU, std::max(n, 1));
    int* hintD = ws().get<int>(kWsHintD, std::max(n, 1));
    launch_start_hints(samples, n, R->source.p, S->cls.p, nullptr, dIdx, n, hintU, hintD, g_stream, cnt);
    WalkJob J{};
    J.hintU = hintU;
    J.hintD = hintD;
    J.nU = nU;
    J.nPtsU = n;
    J.startU = startU;
    J.gidU = gid;
    J.gidBaseU = gidBase;
    J.outU = ws().get<float>(kWsOutU, static_cast<size_t>(n) * nU);
    J.nD = nDw;
    J.nPtsD = n;         // capacity
    J.nPtsDdev = cnt;    // count
    J.xD = xD;
    J.normalD = nrmD;
    J.radiusD = rD;
    J.gidD = gidD;
    J.outD = ws().get<float>(kWsOutD, std::max<size_t>(static_cast<size_t>(n) * nDw, 1));
    auto* ctr = ws().get<unsigned long long>(kWsCounter, 1);
    CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), g_stream));
    J.counter = ctr;
    unsigned long long* rc = st.device_counters();  // the generation's steps, truncations, walks
    J.steps = rc;
    J.truncTotal = rc + 1;
    if (g_profile) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        size_t slots = static_cast<size_t>(sms) * 32 * 256 * 2;
        auto* cc = ws().get<unsigned long long>(kWsEvalOut, slots);
        CK(cudaMemsetAsync(cc, 0, slots * sizeof(unsigned long long), g_stream));
        WalkEnv Ec = E;
        Ec.S.counts = cc;
        launch_walk_job(Ec, J, g_stream);
        std::vector<unsigned long long> h(slots);
        CK(cudaMemcpyAsync(h.data(), cc, slots * sizeof(unsigned long long), cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
        for (size_t i = 0; i < slots; ++i) g_profileTotals[i & 1] += h[i];
    } else {
        KernelTimer::begin(KernelTimer::kWalk);
        launch_walk_job(E, J, g_stream);
        KernelTimer::end(KernelTimer::kWalk);
    }
    after_walk_launch();
    launch_finish_samples(samples, n, J.outU, nU, dIdx, n, J.outD, nDw, failed, g_stream, cnt, rc + 2);
}

__global__ void redraw_copy_kernel(const CacheSample* src, const int* idx, int n, CacheSample* dst);

WalkEnv3 make_env3(bvc_scene_s* S, const bvc_problem& pb, const bvc_walk_config& wc, uint64_t seed, uint64_t salt,
                   uint64_t round) {
    validate_kernel(pb.kernel);
    if (pb.kernel.dim != 3) throw Error(BVC_ERR_INVALID_ARGUMENT, "3D scene needs a dim-3 kernel");
    if (pb.f.kind != BVC_FIELD_NONE)
        throw Error(BVC_ERR_SOLVER, "source terms are not supported by the 3D walks (kernels.cpp:98-99 is 2D-only)");
    // the walks' Neumann-data term (neumannTerm pointwise.cpp:52-107, clipped to the ball) has no 3D
    // form here: nonzero data would be dropped silently, so only h = 0 is accepted on Neumann faces
    if (S->host.hasNeumann() && pb.h.kind != BVC_FIELD_NONE && !(pb.h.kind == BVC_FIELD_CONSTANT && pb.h.p[0] == 0.0))
        throw Error(BVC_ERR_SOLVER, "Neumann data h is not supported by the 3D walks: reflecting faces (h = 0) only");
    if (!(S->host.dirichletMeasure > 0.0))
        throw Error(BVC_ERR_SOLVER, "walk cannot terminate: scene has no Dirichlet boundary");
    WalkEnv3 E{};
    E.S = S->view3();
    E.silRec = S->silRec.p;
    E.triSil = S->triSil.p;
    E.silA = S->sil3A.p;
    E.silB = S->sil3B.p;
    E.silN1 = S->sil3N1.p;
    E.silN2 = S->sil3N2.p;
    E.P.screened = pb.kernel.kind == BVC_KERNEL_SCREENED;
    E.P.sigma = static_cast<float>(pb.kernel.sigma);
    E.P.sqrtSigma = static_cast<float>(std::sqrt(pb.kernel.sigma));
    E.P.dim = 3;
    E.P.f = to_dev(pb.f);
    E.P.g = to_dev(pb.g);
    E.P.h = to_dev(pb.h);
    double diag = S->host.diagonal;
    double eps = wc.epsilon > 0.0 ? wc.epsilon : 1e-3 * diag;
    double rmin = wc.rMin > 0.0 ? wc.rMin : eps;
    if (rmin > eps) throw Error(BVC_ERR_INVALID_ARGUMENT, "walk config: r_min must lie in (0, epsilon]");
    E.eps = static_cast<float>(eps);
    E.rmin = static_cast<float>(rmin);
    E.tguard = static_cast<float>(1e-9 * diag);
    E.insideTol = S->host.component.empty() || *std::max_element(S->host.component.begin(), S->host.component.end()) == 0
                      ? static_cast<float>(1e-7 * diag) : -1.0f;  // parity is meaningless for soups
    E.scale = static_cast<float>(diag);
    E.nudge = static_cast<float>(9.5367431640625e-7 * diag);
    E.cx = static_cast<float>(0.5 * (S->host.lo[0] + S->host.hi[0]));
    E.cy = static_cast<float>(0.5 * (S->host.lo[1] + S->host.hi[1]));
    E.cz = static_cast<float>(0.5 * (S->host.lo[2] + S->host.hi[2]));
    E.escape = S->host.closed() ? static_cast<float>(diag) : 3.0e38f;  // meshes are closed soups
    E.maxSteps = std::max(1, wc.maxSteps);
    E.hasNeumann = S->host.hasNeumann() ? 1 : 0;
    E.hasH = pb.h.kind != BVC_FIELD_NONE ? 1 : 0;
    E.closed = E.insideTol > 0.f ? 1 : 0;
    key_of(seed, salt, round, E.k0, E.k1);
    E.ff = S->farfield();
    E.hg = S->hintgrid();
    return E;
}

void run_cache_walks3(bvc_scene_s* S, bvc_region_s* R, const WalkEnv3& E, const bvc_cache_config& cfg,
                      CacheSample* samples, int n, long long gidBase, const long long* gid, uint8_t* failed,
                      GenStats& st) {
    float4* startU = ws().get<float4>(kWsStartU, n);
    int* isD = ws().get<int>(kWsIsD, n);
    float* gradR = ws().get<float>(kWsGradR, n);
    launch_prepare3(E, samples, n, R->kinds.p, startU, isD, gradR, failed, g_stream);
    int* dIdx = ws().get<int>(kWsDIdx, n);
    int* cnt = ws().get<int>(kWsCount, 1);
    launch_compact(isD, n, dIdx, cnt, g_stream);
    // the D points stay on the device: buffers sized for all n samples, kernels read the
    // count (no host round trip between the compaction and the walks)
    float4* xD = ws().get<float4>(kWsXD, n);
    float4* nrmD = ws().get<float4>(kWsND, n);
    float* rD = ws().get<float>(kWsRD, n);
    long long* gidD = ws().get<long long>(kWsGidD, n);
    launch_gather_dpoints3(samples, dIdx, n, gradR, gidBase, gid, xD, nrmD, rD, gidD, g_stream, cnt);
    int nU = std::max(1, cfg.nWalksNeumann), nDw = std::max(1, cfg.nWalksDirichlet);
    int* hintU = ws().get<int>(kWsHintU, std::max(n, 1));
    int* hintD = ws().get<int>(kWsHintD, std::max(n, 1));
    launch_start_hints(samples, n, R->source.p, S->cls.p, S->leafOf.p, dIdx, n, hintU, hintD, g_stream, cnt);
    WalkJob3 J{};
    J.hintU = hintU;
    J.hintD = hintD;
    J.nU = nU;
    J.nPtsU = n;
    J.startU = startU;
    J.gidU = gid;
    J.gidBaseU = gidBase;
    J.outU = ws().get<float>(kWsOutU, static_cast<size_t>(n) * nU);
    J.nD = nDw;
    J.nPtsD = n;         // capacity
    J.nPtsDdev = cnt;    // count
    J.xD = xD;
    J.normalD = nrmD;
    J.radiusD = rD;
    J.gidD = gidD;
    J.outD = ws().get<float>(kWsOutD, std::max<size_t>(static_cast<size_t>(n) * nDw, 1));
    auto* ctr = ws().get<unsigned long long>(kWsCounter, 1);
    CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), g_stream));
    J.counter = ctr;
    unsigned long long* rc = st.device_counters();  // the generation's steps, truncations, walks
    J.steps = rc;
    J.truncTotal = rc + 1;
    if (g_profile) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        size_t slots = static_cast<size_t>(sms) * 32 * 256 * 2;
        auto* cc = ws().get<unsigned long long>(kWsEvalOut, slots);
        CK(cudaMemsetAsync(cc, 0, slots * sizeof(unsigned long long), g_stream));
        WalkEnv3 Ec = E;
        Ec.S.counts = cc;
        launch_walk_job3(Ec, J, g_stream);
        std::vector<unsigned long long> h(slots);
        CK(cudaMemcpyAsync(h.data(), cc, slots * sizeof(unsigned long long), cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
        for (size_t i = 0; i < slots; ++i) g_profileTotals[i & 1] += h[i];
    } else {
        KernelTimer::begin(KernelTimer::kWalk);
        launch_walk_job3(E, J, g_stream);
        KernelTimer::end(KernelTimer::kWalk);
    }
    after_walk_launch();
    launch_finish_samples(samples, n, J.outU, nU, dIdx, n, J.outD, nDw, failed, g_stream, cnt, rc + 2);
}

void generate_cache3(bvc_scene_s* S, const bvc_problem& pb, bvc_region_s* R, const bvc_cache_config& cfg, uint64_t seed,
                     uint64_t round, int begin, int end, bvc_boundary_cache_s* out, GenStats& st) {
    const int N = std::max(1, cfg.nBoundary);
    const int n = end - begin;
    out->n = n;
    out->dim = 3;
    out->voronoi = 0;
    out->length = R->boundary.total;
    out->samples.resize(std::max(n, 1));
    if (n == 0) return;
    if (cfg.voronoi) throw Error(BVC_ERR_INVALID_ARGUMENT, "Voronoi weights are defined for 2D loops only");
    bvc_scene_s& B = R->boundary;
    uint32_t k0, k1;
    key_of(seed, kBoundaryPosSalt, round, k0, k1);
    launch_sample_mesh(B.cdf.p, B.host.ns, B.total, B.triA.p, B.triB.p, B.triC.p, B.triNormal.p, N, begin, n, nullptr,
                       cfg.stratified, k0, k1, out->samples.p, g_stream);
    WalkEnv3 E = make_env3(S, pb, cfg.walk, seed, kBoundaryWalkSalt, round);
    uint8_t* failed = ws().get<uint8_t>(kWsFailed, n);
    run_cache_walks3(S, R, E, cfg, out->samples.p, n, begin, nullptr, failed, st);
    // deterministic redraw of failed samples (cache.cpp:365-379): the failures are
    // compacted on the device and the host reads one 4-byte count (the list only when
    // it is not empty)
    int* badIdx = ws().get<int>(kWsBadIdx, n);
    int* badCnt = ws().get<int>(kWsBadCnt, 1);
    launch_compact_u8(failed, n, badIdx, badCnt, g_stream);
    const int nbad = read_device_int(badCnt);
    std::vector<int> bad(nbad);
    if (nbad) {
        CK(cudaMemcpyAsync(bad.data(), badIdx, nbad * sizeof(int), cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
    }
    WalkEnv3 Er = make_env3(S, pb, cfg.walk, seed, kBoundaryRedrawSalt, round);
    for (int guard = 1; !bad.empty(); ++guard) {
        if (guard > 64) throw Error(BVC_ERR_SOLVER, "boundary cache: sample kept failing after 64 redraws");
        int nb = static_cast<int>(bad.size());
        st.resampled += nb;
        std::vector<long long> hc(nb);
        for (int j = 0; j < nb; ++j) hc[j] = (static_cast<long long>(begin) + bad[j]) * 131 + guard;
        long long* dctr = ws().get<long long>(kWsCtr, nb);
        CK(cudaMemcpyAsync(dctr, hc.data(), nb * sizeof(long long), cudaMemcpyHostToDevice, g_stream));
        CacheSample* tmp = ws().get<CacheSample>(kWsSamplesTmp, nb);
        uint32_t r0, r1;
        key_of(seed, kBoundaryRedrawSalt, round, r0, r1);
        launch_sample_mesh(B.cdf.p, B.host.ns, B.total, B.triA.p, B.triB.p, B.triC.p, B.triNormal.p, N, 0, nb, dctr, 0, r0,
                           r1, tmp, g_stream);
        uint8_t* f2 = ws().get<uint8_t>(kWsSrcFlag, nb);
        run_cache_walks3(S, R, Er, cfg, tmp, nb, 0, dctr, f2, st);
        int* didx = ws().get<int>(kWsDIdx, nb);
        CK(cudaMemcpyAsync(didx, bad.data(), nb * sizeof(int), cudaMemcpyHostToDevice, g_stream));
        redraw_copy_kernel<<<(nb + 127) / 128, 128, 0, g_stream>>>(tmp, didx, nb, out->samples.p);
        count_launch();
        std::vector<uint8_t> hf2(nb);
        CK(cudaMemcpyAsync(hf2.data(), f2, nb, cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
        std::vector<int> still;
        for (int j = 0; j < nb; ++j) if (hf2[j]) still.push_back(bad[j]);
        bad.swap(still);
    }
    st.snapshot();
}

__global__ void redraw_copy_kernel(const CacheSample* src, const int* idx, int n, CacheSample* dst) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) dst[idx[j]] = src[j];
}

// assignVoronoiWeights (cache.cpp:280-297), on the host (rare mode): per region
// loop, each sample's weight is half the arc distance to its two neighbours
void assign_voronoi(bvc_region_s* R, bvc_boundary_cache_s* c) {
    need(c->dim == 2, "Voronoi weights are defined for 2D loops only");
    int n = c->n;
    if (n == 0) return;
    std::vector<CacheSample> hs(n);
    c->samples.download(hs.data(), n);
    CK(cudaStreamSynchronize(g_stream));
    const auto& bh = R->boundary.host;
    std::vector<std::vector<std::pair<double, int>>> per(bh.loopLength.size());
    for (int i = 0; i < n; ++i) per[bh.loop[hs[i].segment]].push_back({hs[i].arc, i});
    for (size_t li = 0; li < per.size(); ++li) {
        auto& e = per[li];
        if (e.empty()) continue;
        std::sort(e.begin(), e.end());
        size_t m = e.size();
        double L = bh.loopLength[li];
        for (size_t k = 0; k < m; ++k) {
            double w;
            if (m == 1) w = L;
            else {
                double prev = k > 0 ? e[k].first - e[k - 1].first : e[0].first + L - e[m - 1].first;
                double next = k + 1 < m ? e[k + 1].first - e[k].first : e[0].first + L - e[m - 1].first;
                w = 0.5 * (prev + next);
            }
            hs[e[k].second].weight = static_cast<float>(w);
        }
    }
    c->samples.upload(hs.data(), n);
    c->voronoi = 1;
}

void generate_cache(bvc_scene_s* S, const bvc_problem& pb, bvc_region_s* R, const bvc_cache_config& cfg, uint64_t seed,
                    uint64_t round, int begin, int end, bvc_boundary_cache_s* out, GenStats& st) {
    require_device();
    need(S && R, "null scene or region");
    R->upload();
    const int N = std::max(1, cfg.nBoundary);
    need(begin >= 0 && begin <= end && end <= N, "shard range outside [0, nBoundary]");
    if (S->host.dim == 3) {
        S->upload();
        generate_cache3(S, pb, R, cfg, seed, round, begin, end, out, st);
        return;
    }
    const int n = end - begin;
    out->n = n;
    out->dim = 2;
    out->voronoi = 0;  // set by assign_voronoi once the whole round is present
    out->length = R->boundary.total;
    out->samples.resize(std::max(n, 1));
    if (n == 0) return;
    bvc_scene_s& B = R->boundary;
    uint32_t k0, k1;
    key_of(seed, kBoundaryPosSalt, round, k0, k1);
    launch_sample_boundary(B.cdf.p, B.cdfIds.p, B.host.ns, B.total, B.segAB.p, B.segNormal.p, B.segArc.p, B.segLen.p, N,
                           begin, n, nullptr, cfg.stratified, k0, k1, out->samples.p, g_stream);
    WalkEnv E = make_env(S, pb, cfg.walk, seed, kBoundaryWalkSalt, round);
    uint8_t* failed = ws().get<uint8_t>(kWsFailed, n);
    run_cache_walks(S, R, E, cfg, out->samples.p, n, begin, nullptr, failed, st);
    // deterministic redraw of failed samples (cache.cpp:365-379): the failures are
    // compacted on the device and the host reads one 4-byte count (the list only when
    // it is not empty)
    int* badIdx = ws().get<int>(kWsBadIdx, n);
    int* badCnt = ws().get<int>(kWsBadCnt, 1);
    launch_compact_u8(failed, n, badIdx, badCnt, g_stream);
    const int nbad = read_device_int(badCnt);
    std::vector<int> bad(nbad);
    if (nbad) {
        CK(cudaMemcpyAsync(bad.data(), badIdx, nbad * sizeof(int), cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
    }
    WalkEnv Er = make_env(S, pb, cfg.walk, seed, kBoundaryRedrawSalt, round);
    for (int guard = 1; !bad.empty(); ++guard) {
        if (guard > 64) throw Error(BVC_ERR_SOLVER, "boundary cache: sample kept failing after 64 redraws");
        int nb = static_cast<int>(bad.size());
        st.resampled += nb;
        std::vector<long long> hc(nb);
        for (int j = 0; j < nb; ++j) hc[j] = (static_cast<long long>(begin) + bad[j]) * 131 + guard;
        long long* dctr = ws().get<long long>(kWsCtr, nb);
        CK(cudaMemcpyAsync(dctr, hc.data(), nb * sizeof(long long), cudaMemcpyHostToDevice, g_stream));
        CacheSample* tmp = ws().get<CacheSample>(kWsSamplesTmp, nb);
        uint32_t r0, r1;
        key_of(seed, kBoundaryRedrawSalt, round, r0, r1);
        launch_sample_boundary(B.cdf.p, B.cdfIds.p, B.host.ns, B.total, B.segAB.p, B.segNormal.p, B.segArc.p,
                               B.segLen.p, N, 0, nb, dctr, 0, r0, r1, tmp, g_stream);
        uint8_t* f2 = ws().get<uint8_t>(kWsSrcFlag, nb);
        run_cache_walks(S, R, Er, cfg, tmp, nb, 0, dctr, f2, st);
        int* didx = ws().get<int>(kWsDIdx + 0, nb);  // reuse after walks are done
        std::vector<int> hb(bad.begin(), bad.end());
        CK(cudaMemcpyAsync(didx, hb.data(), nb * sizeof(int), cudaMemcpyHostToDevice, g_stream));
        redraw_copy_kernel<<<(nb + 127) / 128, 128, 0, g_stream>>>(tmp, didx, nb, out->samples.p);
        count_launch();
        std::vector<uint8_t> hf2(nb);
        CK(cudaMemcpyAsync(hf2.data(), f2, nb, cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
        std::vector<int> still;
        for (int j = 0; j < nb; ++j) if (hf2[j]) still.push_back(bad[j]);
        bad.swap(still);
    }
    // assignVoronoiWeights needs every sample of the round: a shard leaves it to the
    // caller (distributed.py assigns after the all-gather)
    if (cfg.voronoi && begin == 0 && end == N) assign_voronoi(R, out);
    st.snapshot();
}

// RegionSampler::sample (sampling.cpp:62-108): jittered strata over the bounding
// box, rejection by the device inside test; the last pass keeps a random subset
__global__ void region_propose_kernel(int g, double lo0, double lo1, double ex, double ey, int pass, int stratified,
                                      uint32_t k0, uint32_t k1, float insideTol, bvc_dev::SceneView2 S, float* y,
                                      int* ok, unsigned* prio) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= g * g) return;
    bvc_dev::U4 r = bvc_dev::philox4x32_10(bvc_dev::U4{static_cast<uint32_t>(c), static_cast<uint32_t>(pass), 7u, 0u}, k0, k1);
    double ux = (static_cast<double>(r.x >> 5) * 67108864.0 + (r.y >> 6)) * (1.0 / 9007199254740992.0);
    double uy = (static_cast<double>(r.z >> 5) * 67108864.0 + (r.w >> 6)) * (1.0 / 9007199254740992.0);
    double px, py;
    if (stratified) {
        int cx = c % g, cy = c / g;
        px = lo0 + (cx + ux) / g * ex;
        py = lo1 + (cy + uy) / g * ey;
    } else {
        px = lo0 + ux * ex;
        py = lo1 + uy * ey;
    }
    y[2 * c] = static_cast<float>(px);
    y[2 * c + 1] = static_cast<float>(py);
    ok[c] = bvc_dev::inside(S, static_cast<float>(px), static_cast<float>(py), insideTol) ? 1 : 0;
    bvc_dev::U4 q = bvc_dev::philox4x32_10(bvc_dev::U4{static_cast<uint32_t>(c), static_cast<uint32_t>(pass), 9u, 0u}, k0, k1);
    prio[c] = q.x;
}

__global__ void source_emit_kernel(const float* y, const int* idx, int n, int base, float pdf, bvc_dev::DevField f,
                                   SourceSampleDev* out) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int c = idx[j];
    SourceSampleDev s{};
    s.y[0] = y[2 * c];
    s.y[1] = y[2 * c + 1];
    s.pdf = pdf;
    s.f = bvc_dev::field_eval(f, s.y[0], s.y[1]);
    out[base + j] = s;
}

void generate_source(const bvc_problem& pb, bvc_region_s* R, const bvc_cache_config& cfg, uint64_t seed, uint64_t round,
                     bvc_source_cache_s* out) {
    require_device();
    R->upload();
    bvc_scene_s& B = R->boundary;
    if (B.host.dim == 3) {  // no 3D source path (sampleBallGreens is 2D-only, kernels.cpp:98-99)
        out->dim = 3;
        out->area = bvc_host::meshVolume(B.host);
        out->m = 0;
        if (pb.f.kind != BVC_FIELD_NONE) throw Error(BVC_ERR_SOLVER, "3D source caches are not supported");
        return;
    }
    out->dim = 2;
    out->area = bvc_host::loopArea(B.host);
    if (!B.host.closed()) throw Error(BVC_ERR_PARSE, "region sampler requires closed loops");
    if (out->area <= 0.0) throw Error(BVC_ERR_PARSE, "region sampler: non-positive area");
    if (pb.f.kind == BVC_FIELD_NONE) {
        out->m = 0;
        return;
    }
    const int M = std::max(1, cfg.nSource);
    out->m = M;
    out->samples.resize(M);
    int g = std::max(1, static_cast<int>(std::ceil(std::sqrt(static_cast<double>(M)))));
    int cells = cfg.stratified ? g * g : M;
    if (!cfg.stratified) g = static_cast<int>(std::ceil(std::sqrt(static_cast<double>(cells))));
    float* y = ws().get<float>(kWsSrcTmp, 2 * static_cast<size_t>(g) * g);
    int* ok = ws().get<int>(kWsIsD, static_cast<size_t>(g) * g);
    unsigned* prio = ws().get<unsigned>(kWsSortKeysIn, static_cast<size_t>(g) * g);
    int* idx = ws().get<int>(kWsDIdx, static_cast<size_t>(g) * g);
    int* cnt = ws().get<int>(kWsCount, 1);
    uint32_t k0, k1;
    key_of(seed, kSourceSalt, round, k0, k1);
    const auto& h = B.host;
    double ex = h.hi[0] - h.lo[0], ey = h.hi[1] - h.lo[1];
    float tol = static_cast<float>(1e-7 * h.diagonal);
    bvc_dev::SceneView2 SV = B.view();
    bvc_dev::DevField f = to_dev(pb.f);
    long long proposals = 0;
    int accepted = 0;
    for (int pass = 0; accepted < M; ++pass) {
        int nc = g * g;
        region_propose_kernel<<<(nc + 127) / 128, 128, 0, g_stream>>>(g, h.lo[0], h.lo[1], ex, ey, pass,
                                                                      cfg.stratified, k0, k1, tol, SV, y, ok, prio);
        count_launch();
        launch_compact(ok, nc, idx, cnt, g_stream);
        const int na = read_device_int(cnt);
        proposals += nc;
        if (proposals >= 1000000 && accepted + na < proposals / 10000)
            throw Error(BVC_ERR_PARSE, "degenerate region: rejection acceptance rate below 1e-4");
        int take = std::min(na, M - accepted);
        if (take < na) {  // final pass: a random subset (a shuffled visiting order)
            std::vector<int> hidx(na);
            std::vector<unsigned> hp(static_cast<size_t>(nc));
            CK(cudaMemcpyAsync(hidx.data(), idx, na * sizeof(int), cudaMemcpyDeviceToHost, g_stream));
            CK(cudaMemcpyAsync(hp.data(), prio, nc * sizeof(unsigned), cudaMemcpyDeviceToHost, g_stream));
            CK(cudaStreamSynchronize(g_stream));
            std::stable_sort(hidx.begin(), hidx.end(), [&](int a, int b) { return hp[a] < hp[b]; });
            hidx.resize(take);
            std::sort(hidx.begin(), hidx.end());
            CK(cudaMemcpyAsync(idx, hidx.data(), take * sizeof(int), cudaMemcpyHostToDevice, g_stream));
        }
        source_emit_kernel<<<(take + 127) / 128, 128, 0, g_stream>>>(y, idx, take, accepted, static_cast<float>(1.0 / out->area), f,
                                                                     out->samples.p);
        count_launch();
        accepted += take;
    }
}

}  // namespace bvc_capi

namespace bvc_capi {
// a rank's shard [begin, end) of the round's samples with the rank's fallback-band
// walks (cache.cpp:665-681) on the side stream while the shard's walks run; on return
// the main stream waits for both (no host synchronisation). `points` runs on the side
// stream (it may build the points there, as the host-buffer rounds do) and its result
// is returned.
bvc_eval_points_s* generate_shard_with_band(bvc_scene_s* s, const bvc_problem& pb, bvc_region_s* r,
                                           const bvc_cache_config& cfg, uint64_t seed, uint64_t round, int begin,
                                           int end, const std::function<bvc_eval_points_s*()>& points,
                                           bool gradients, bvc_boundary_cache_s* out, GenStats& st) {
    require_device();
    s->upload();
    r->upload();
    cudaEvent_t ready = round_event(0), done = round_event(1);
    CK(cudaEventRecord(ready, g_stream));
    bool ran = false;
    bvc_eval_points_s* p = nullptr;
    auto side = [&] {
        SideScope scope;
        CK(cudaStreamWaitEvent(g_stream, ready, 0));
        p = points();
        need(p != nullptr, "null evaluation points");
        fallback_walks(s, pb, cfg, p, seed, round, gradients);
        CK(cudaEventRecord(done, g_stream));
        ran = true;
    };
    g_afterWalkLaunch = side;
    try {
        generate_cache(s, pb, r, cfg, seed, round, begin, end, out, st);
        if (!ran) after_walk_launch();
    } catch (...) {
        g_afterWalkLaunch = nullptr;
        throw;
    }
    g_afterWalkLaunch = nullptr;
    CK(cudaStreamWaitEvent(g_stream, done, 0));
    return p;
}
}  // namespace bvc_capi

extern "C" {

int bvc_generate_boundary_cache_shard(bvc_scene s, const bvc_problem* pb, bvc_region r, const bvc_cache_config* cfg,
                                      uint64_t seed, uint64_t round, int begin, int end, bvc_round_stats* stats,
                                      bvc_boundary_cache* out) {
    API({
        need(s && pb && r && cfg && out, "null argument");
        auto c = std::make_unique<bvc_boundary_cache_s>();
        GenStats st;
        generate_cache(s, *pb, r, *cfg, seed, round, begin, end, c.get(), st);
        CK(cudaStreamSynchronize(g_stream));
        st.resolve();
        if (stats) {
            stats->resampled += st.resampled;
            stats->cacheWalks += st.walks;
            stats->cacheTruncated += st.truncated;
            stats->cacheSteps += st.steps;
        }
        *out = c.release();
    })
}
int bvc_generate_boundary_cache_shard_fallback(bvc_scene s, const bvc_problem* pb, bvc_region r,
                                               const bvc_cache_config* cfg, uint64_t seed, uint64_t round, int begin,
                                               int end, bvc_eval_points pts, int gradients, bvc_round_stats* stats,
                                               bvc_boundary_cache* out) {
    API({
        need(s && pb && r && cfg && pts && out, "null argument");
        auto c = std::make_unique<bvc_boundary_cache_s>();
        GenStats st;
        generate_shard_with_band(s, *pb, r, *cfg, seed, round, begin, end, [pts]() { return pts; }, gradients != 0,
                                 c.get(), st);
        CK(cudaStreamSynchronize(g_stream));
        st.resolve();
        if (stats) {
            stats->resampled += st.resampled;
            stats->cacheWalks += st.walks;
            stats->cacheTruncated += st.truncated;
            stats->cacheSteps += st.steps;
        }
        *out = c.release();
    })
}
int bvc_generate_boundary_cache(bvc_scene s, const bvc_problem* pb, bvc_region r, const bvc_cache_config* cfg,
                                uint64_t seed, uint64_t round, bvc_round_stats* stats, bvc_boundary_cache* out) {
    return bvc_generate_boundary_cache_shard(s, pb, r, cfg, seed, round, 0, std::max(1, cfg ? cfg->nBoundary : 1), stats,
                                             out);
}
int bvc_generate_source_cache(const bvc_problem* pb, bvc_region r, const bvc_cache_config* cfg, uint64_t seed,
                              uint64_t round, bvc_source_cache* out) {
    API({
        need(pb && r && cfg && out, "null argument");
        auto c = std::make_unique<bvc_source_cache_s>();
        generate_source(*pb, r, *cfg, seed, round, c.get());
        *out = c.release();
    })
}
int bvc_boundary_cache_create(const bvc_boundary_sample* smp, int n, int dim, int voronoi, double length,
                              bvc_boundary_cache* out) {
    API({
        require_device();
        need(out && (smp || n == 0) && n >= 0, "null argument");
        need(dim == 2 || dim == 3, "cache dimension must be 2 or 3");
        auto c = std::make_unique<bvc_boundary_cache_s>();
        c->n = n;
        c->dim = dim;
        c->voronoi = voronoi;
        c->length = length;
        std::vector<CacheSample> h(std::max(n, 1));
        for (int i = 0; i < n; ++i) {
            CacheSample& o = h[i];
            for (int k = 0; k < 3; ++k) {
                o.z[k] = static_cast<float>(smp[i].z[k]);
                o.n[k] = static_cast<float>(smp[i].n[k]);
            }
            if (dim == 2) o.z[2] = o.n[2] = 0.f;
            o.pdf = static_cast<float>(smp[i].pdf);
            o.uHat = static_cast<float>(smp[i].uHat);
            o.dHat = static_cast<float>(smp[i].dHat);
            o.weight = static_cast<float>(smp[i].weight);
            o.arc = static_cast<float>(smp[i].arc);
            o.segment = smp[i].segment;
        }
        c->samples.upload(h.data(), std::max(n, 1));
        *out = c.release();
    })
}
int bvc_boundary_cache_size(bvc_boundary_cache c, int* n, int* dim) {
    API({
        need(c, "null cache");
        if (n) *n = c->n;
        if (dim) *dim = c->dim;
    })
}
int bvc_boundary_cache_download(bvc_boundary_cache c, bvc_boundary_sample* smp) {
    API({
        require_device();
        need(c && smp, "null argument");
        std::vector<CacheSample> h(c->n);
        c->samples.download(h.data(), c->n);
        CK(cudaStreamSynchronize(g_stream));
        for (int i = 0; i < c->n; ++i) {
            bvc_boundary_sample& o = smp[i];
            for (int k = 0; k < 3; ++k) {
                o.z[k] = h[i].z[k];
                o.n[k] = h[i].n[k];
            }
            o.pdf = h[i].pdf;
            o.uHat = h[i].uHat;
            o.dHat = h[i].dHat;
            o.weight = h[i].weight;
            o.segment = h[i].segment;
            o.arc = h[i].arc;
        }
    })
}
int bvc_boundary_cache_packed(bvc_boundary_cache c, void** ptr, size_t* bytes) {
    API({
        need(c && ptr && bytes, "null argument");
        *ptr = c->samples.p;
        *bytes = static_cast<size_t>(c->n) * sizeof(CacheSample);
    })
}
int bvc_boundary_cache_from_packed(const void* ptr, int n, int dim, int voronoi, double length, bvc_boundary_cache* out) {
    API({
        require_device();
        need(out && (ptr || n == 0), "null argument");
        auto c = std::make_unique<bvc_boundary_cache_s>();
        c->n = n;
        c->dim = dim;
        c->voronoi = voronoi;
        c->length = length;
        c->samples.resize(std::max(n, 1));
        if (n) CK(cudaMemcpyAsync(c->samples.p, ptr, n * sizeof(CacheSample), cudaMemcpyDeviceToDevice, g_stream));
        *out = c.release();
    })
}
int bvc_boundary_cache_assign_voronoi(bvc_boundary_cache c, bvc_region r) {
    API(need(c && r, "null argument"); r->upload(); assign_voronoi(r, c))
}
int bvc_boundary_cache_destroy(bvc_boundary_cache c) { API(delete c) }
int bvc_source_cache_create(const bvc_source_sample* smp, int m, int dim, double area, bvc_source_cache* out) {
    API({
        require_device();
        need(out && (smp || m == 0) && m >= 0, "null argument");
        auto c = std::make_unique<bvc_source_cache_s>();
        c->m = m;
        c->dim = dim;
        c->area = area;
        std::vector<SourceSampleDev> h(std::max(m, 1));
        for (int i = 0; i < m; ++i) {
            for (int k = 0; k < 3; ++k) h[i].y[k] = static_cast<float>(smp[i].y[k]);
            if (dim == 2) h[i].y[2] = 0.f;
            h[i].pdf = static_cast<float>(smp[i].pdf);
            h[i].f = static_cast<float>(smp[i].f);
        }
        c->samples.upload(h.data(), std::max(m, 1));
        *out = c.release();
    })
}
int bvc_source_cache_size(bvc_source_cache c, int* m, int* dim) {
    API({
        need(c, "null cache");
        if (m) *m = c->m;
        if (dim) *dim = c->dim;
    })
}
int bvc_source_cache_download(bvc_source_cache c, bvc_source_sample* smp) {
    API({
        require_device();
        need(c && smp, "null argument");
        std::vector<SourceSampleDev> h(std::max(c->m, 1));
        c->samples.download(h.data(), c->m);
        CK(cudaStreamSynchronize(g_stream));
        for (int i = 0; i < c->m; ++i) {
            for (int k = 0; k < 3; ++k) smp[i].y[k] = h[i].y[k];
            smp[i].pdf = h[i].pdf;
            smp[i].f = h[i].f;
        }
    })
}
int bvc_source_cache_destroy(bvc_source_cache c) { API(delete c) }

int bvc_walk_traffic_profile(bvc_scene s, const bvc_problem* pb, bvc_region r, const bvc_cache_config* cfg,
                             uint64_t seed, uint64_t round, double* out) {
    API({
        need(s && pb && r && cfg && out, "null argument");
        bvc_boundary_cache_s c;
        GenStats st;
        g_profile = true;
        g_profileTotals[0] = g_profileTotals[1] = 0;
        try {
            generate_cache(s, *pb, r, *cfg, seed, round, 0, std::max(1, cfg->nBoundary), &c, st);
        } catch (...) {
            g_profile = false;
            throw;
        }
        g_profile = false;
        CK(cudaStreamSynchronize(g_stream));
        st.resolve();
        out[0] = static_cast<double>(st.steps);
        out[1] = static_cast<double>(g_profileTotals[0]);
        out[2] = static_cast<double>(g_profileTotals[1]);
        out[3] = static_cast<double>(st.walks);
    })
}

}  // extern "C"
