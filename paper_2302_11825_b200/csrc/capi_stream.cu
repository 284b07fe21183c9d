// capi_stream.cu — runStreamlines (runner.cpp:285-373) on the device: batched
// gradient gathers over the retained caches, one Heun step for every seed at once.
#include "capi_common.cuh"

namespace bvc_capi {

// The direction field of runStreamlines (runner.cpp:310-329) for a batch of points:
// status 0 ok (g = unit gradient), 1 outside (not evaluable or in the fallback
// band), 2 zero gradient (|grad u| < 1e-12). The gradient is the splatGradient
// of every retained round's caches accumulated into one EvaluationPoint.
struct StreamCaches {
    std::vector<std::unique_ptr<bvc_boundary_cache_s>> b;
    std::vector<std::unique_ptr<bvc_source_cache_s>> s;
};
void stream_directions(bvc_scene_s* S, bvc_region_s* R, const bvc_cache_config& cfg, const bvc_splat_config& scfg,
                       const StreamCaches& C, const std::vector<double>& x, std::vector<double>& g,
                       std::vector<int>& status) {
    size_t n = x.size() / 2;
    g.assign(2 * n, 0.0);
    status.assign(n, 1);
    if (n == 0) return;
    auto P = make_points(x.data(), n, 2);
    // evaluable (runner.cpp:31-35): inside the scene and, for a subdomain, inside the loop
    float tol = static_cast<float>(1e-7 * S->host.diagonal);
    uint8_t* ins = ws().get<uint8_t>(kWsOutside, 2 * n);
    launch_inside(S->view(), P->x.p, static_cast<int>(n), tol, ins, g_stream);
    if (!R->host.wholeDomain)
        launch_inside(R->boundary.view(), P->x.p, static_cast<int>(n),
                      static_cast<float>(1e-7 * R->boundary.host.diagonal), ins + n, g_stream);
    mark_points(S, R, cfg, P.get());
    std::vector<uint8_t> hin(2 * n, 1), fb(n);
    CK(cudaMemcpyAsync(hin.data(), ins, (R->host.wholeDomain ? 1 : 2) * n, cudaMemcpyDeviceToHost, g_stream));
    P->fallback.download(fb.data(), n);
    CK(cudaStreamSynchronize(g_stream));
    for (size_t i = 0; i < n; ++i) fb[i] = (fb[i] || !hin[i] || !hin[n + i]) ? 1 : 0;
    P->fallback.upload(fb.data(), n);  // excluded from the gather, like the reference's early return
    P->orderValid = false;
    for (size_t r = 0; r < C.b.size(); ++r)
        splat(C.b[r].get(), C.s[r]->m ? C.s[r].get() : nullptr, P.get(), scfg, 0, SIZE_MAX, false, true);
    double* o = ws().get<double>(kWsEvalOut, 3 * n);
    launch_solution(P.get(), o, o + n);
    std::vector<double> hg(2 * n);
    CK(cudaMemcpyAsync(hg.data(), o + n, 2 * n * sizeof(double), cudaMemcpyDeviceToHost, g_stream));
    CK(cudaStreamSynchronize(g_stream));
    for (size_t i = 0; i < n; ++i) {
        if (fb[i]) continue;  // outside
        double gx = hg[2 * i], gy = hg[2 * i + 1];
        double nrm = std::sqrt(gx * gx + gy * gy);
        if (nrm < 1e-12) { status[i] = 2; continue; }
        status[i] = 0;
        g[2 * i] = gx / nrm;
        g[2 * i + 1] = gy / nrm;
    }
}

// runStreamlines (runner.cpp:285-373): every seed advances together, so each Heun
// step is two batched gradient gathers (probe and landing) over the retained caches;
// the landing's direction is the next step's k1 (deterministic, so equal to the
// reference's recomputation).
void trace_streamlines(bvc_scene_s* S, const bvc_problem& pb, bvc_region_s* R, const bvc_cache_config& cfg,
                       uint64_t seed, int rounds, const double* seeds, int nSeeds, double h, int steps,
                       double* points, int* counts, int* reasons) {
    require_device();
    need(S->host.dim == 2, "streamlines: 2D scenes only (runner.cpp:285)");
    if (cfg.sourceBall) throw Error(BVC_ERR_INVALID_ARGUMENT, "streamlines: sourceBall mode does not support gradient splats");
    need(nSeeds > 0 && seeds, "streamlines.seeds: required");
    need(h > 0.0, "streamlines.step: expected > 0");
    need(steps >= 1, "streamlines.steps: expected >= 1");
    need(rounds >= 1, "streamlines: rounds must be >= 1");
    bvc_splat_config scfg = make_splat_config(S, pb, cfg);
    StreamCaches C;
    for (int r = 0; r < rounds; ++r) {  // retained caches (runner.cpp:305-308)
        auto b = std::make_unique<bvc_boundary_cache_s>();
        auto s = std::make_unique<bvc_source_cache_s>();
        GenStats st;
        generate_cache(S, pb, R, cfg, seed, r, 0, std::max(1, cfg.nBoundary), b.get(), st);
        generate_source(pb, R, cfg, seed, r, s.get());
        C.b.push_back(std::move(b));
        C.s.push_back(std::move(s));
    }
    const int per = steps + 1;
    std::vector<double> x(seeds, seeds + 2 * static_cast<size_t>(nSeeds)), g;
    std::vector<int> st;
    stream_directions(S, R, cfg, scfg, C, x, g, st);
    std::vector<double> k1(2 * static_cast<size_t>(nSeeds));
    std::vector<int> status(st), active;
    for (int i = 0; i < nSeeds; ++i) {
        counts[i] = 0;
        reasons[i] = BVC_STREAM_OK;
        if (st[i] == 1) { reasons[i] = BVC_STREAM_OUTSIDE; continue; }  // no polyline
        points[2 * static_cast<size_t>(i) * per] = x[2 * i];
        points[2 * static_cast<size_t>(i) * per + 1] = x[2 * i + 1];
        counts[i] = 1;
        k1[2 * i] = g[2 * i];
        k1[2 * i + 1] = g[2 * i + 1];
        active.push_back(i);
    }
    for (int k = 1; k <= steps && !active.empty(); ++k) {
        std::vector<int> go;
        for (int i : active) {
            if (status[i] == 2) reasons[i] = BVC_STREAM_ZERO_GRADIENT;  // k1 = direction(x) failed
            else go.push_back(i);
        }
        if (go.empty()) break;
        std::vector<double> probe(2 * go.size()), gp;
        std::vector<int> sp;
        for (size_t j = 0; j < go.size(); ++j) {
            int i = go[j];
            probe[2 * j] = x[2 * i] + h * k1[2 * i];
            probe[2 * j + 1] = x[2 * i + 1] + h * k1[2 * i + 1];
        }
        stream_directions(S, R, cfg, scfg, C, probe, gp, sp);
        std::vector<double> next(2 * go.size()), gn;
        std::vector<int> sn;
        for (size_t j = 0; j < go.size(); ++j) {
            int i = go[j];
            if (sp[j] == 0) {  // Heun step
                next[2 * j] = x[2 * i] + 0.5 * h * (k1[2 * i] + gp[2 * j]);
                next[2 * j + 1] = x[2 * i + 1] + 0.5 * h * (k1[2 * i + 1] + gp[2 * j + 1]);
            } else {  // the predictor left the region
                next[2 * j] = x[2 * i] + h * k1[2 * i];
                next[2 * j + 1] = x[2 * i + 1] + h * k1[2 * i + 1];
            }
        }
        stream_directions(S, R, cfg, scfg, C, next, gn, sn);
        active.clear();
        for (size_t j = 0; j < go.size(); ++j) {
            int i = go[j];
            if (sn[j] == 1) { reasons[i] = BVC_STREAM_OUTSIDE; continue; }
            x[2 * i] = next[2 * j];
            x[2 * i + 1] = next[2 * j + 1];
            size_t o = 2 * (static_cast<size_t>(i) * per + counts[i]);
            points[o] = x[2 * i];
            points[o + 1] = x[2 * i + 1];
            ++counts[i];
            status[i] = sn[j];
            k1[2 * i] = gn[2 * j];
            k1[2 * i + 1] = gn[2 * j + 1];
            active.push_back(i);
        }
    }
}

}  // namespace bvc_capi

extern "C" {

int bvc_trace_streamlines(bvc_scene s, const bvc_problem* pb, bvc_region r, const bvc_cache_config* cfg,
                          uint64_t seed, int rounds, const double* seeds, int nSeeds, double step, int steps,
                          double* points, int* counts, int* reasons) {
    API(need(s && pb && r && cfg && points && counts && reasons, "null argument");
        trace_streamlines(s, *pb, r, *cfg, seed, rounds, seeds, nSeeds, step, steps, points, counts, reasons))
}

}  // extern "C"
