// integration_example.cpp — INTEGRATION.md's C++ caller, compiled and run by
// tests/test_capi_cpp.py: what runSolveInMemory (runner.cpp:99-207) becomes over the
// C ABI of include/bvc_b200.h. Problem: square-mixed-linear (problems.cpp:94-108 on
// [-1,1]^2): Neumann h = 0 on y = +-1, Dirichlet g = x on x = +-1, exact u = x.
//
//   g++ -std=c++17 -I include tests/cpp/integration_example.cpp
//       -L paper_2302_11825_b200/_build -lbvc_b200 -Wl,-rpath,<that dir> -o example
//   ./example            exit 0: solved within tolerance; 3: no CUDA device (status
//                        BVC_ERR_NO_DEVICE from the first compute call); 1: failure
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <vector>

#include "bvc_b200.h"

struct BvcFailure : std::runtime_error {
    int status;
    BvcFailure(int s, const char* what) : std::runtime_error(what), status(s) {}
};

// the reference throws (SolverError, ParseError, ...); across the C ABI a status code
// plus bvc_last_error() become the exception again
static void check(int status, const char* what) {
    if (status != BVC_OK) throw BvcFailure(status, what);
}

static int run();

int main() {
    try {
        return run();
    } catch (const BvcFailure& e) {
        if (e.status == BVC_ERR_NO_DEVICE) {  // no CPU fallback: the first device call says so
            std::printf("no device: %s (%s)\n", bvc_last_error(), e.what());
            return 3;
        }
        std::fprintf(stderr, "%s: status %d: %s\n", e.what(), e.status, bvc_last_error());
        return 1;
    }
}

static int run() {
    // scene: the same vertex list and (a, b, label) segments Scene::build takes
    const int per = 64;  // segments per side
    std::vector<double> xy;
    std::vector<int> ab, labels;
    const double cx[4] = {-1, 1, 1, -1}, cy[4] = {-1, -1, 1, 1};
    for (int side = 0; side < 4; ++side)
        for (int k = 0; k < per; ++k) {
            double t = static_cast<double>(k) / per;
            xy.push_back(cx[side] + t * (cx[(side + 1) % 4] - cx[side]));
            xy.push_back(cy[side] + t * (cy[(side + 1) % 4] - cy[side]));
        }
    const int nv = 4 * per, ns = 4 * per;
    for (int i = 0; i < ns; ++i) {
        ab.push_back(i);
        ab.push_back((i + 1) % nv);
        labels.push_back((i / per) % 2 == 0 ? BVC_NEUMANN : BVC_DIRICHLET);  // bottom/top Neumann
    }
    bvc_scene scene = nullptr;
    check(bvc_scene_create(xy.data(), nv, ab.data(), labels.data(), ns, &scene), "bvc_scene_create");
    const double eps = 1e-3 * std::sqrt(8.0);
    bvc_region_request req{BVC_REGION_WHOLE_DOMAIN, /*offset l*/ 0.0, nullptr};
    bvc_region region = nullptr;
    check(bvc_region_build(scene, &req, eps, &region), "bvc_region_build");

    bvc_problem pb{};  // PdeProblem
    pb.kernel = {BVC_KERNEL_POISSON, 0.0, 2, std::sqrt(8.0)};
    pb.g.kind = BVC_FIELD_LINEAR;  // g(x, y) = x
    pb.g.p[0] = 1.0;
    bvc_cache_config cfg{/*N*/ 4096, /*M*/ 1024, /*nWalksNeumann*/ 128, /*nWalksDirichlet*/ 256, 0, 0,
                         BVC_CLAMP_OFF, 0, 4, 0, 1, {eps, 0, 10000, 128, 0, 0}, 0};

    // interior grid
    std::vector<double> grid;
    for (int j = 0; j < 16; ++j)
        for (int i = 0; i < 16; ++i) {
            grid.push_back(-0.75 + 1.5 * i / 15.0);
            grid.push_back(-0.75 + 1.5 * j / 15.0);
        }
    const size_t n = grid.size() / 2;
    bvc_eval_points pts = nullptr;
    check(bvc_points_create(grid.data(), n, 2, &pts), "bvc_points_create");
    check(bvc_mark_evaluation_points(scene, region, &cfg, pts), "bvc_mark_evaluation_points");
    const uint64_t seed = 7;
    const int rounds = 8;
    for (uint64_t r = 0; r < static_cast<uint64_t>(rounds); ++r) {
        bvc_round_stats st{};
        check(bvc_update_solution(scene, &pb, region, &cfg, pts, seed, r, /*gradients*/ 1, &st),
              "bvc_update_solution");
    }
    // EvaluationPoint::solution() on the device, then the host view of the sums
    std::vector<double> u(n), g(2 * n);
    check(bvc_points_solution(pts, u.data(), g.data()), "bvc_points_solution");
    std::vector<double> bs(n), ss(n), wsum(n);
    std::vector<long long> nb(n), ms(n), wc(n);
    std::vector<uint8_t> fb(n);
    bvc_point_state hs{};
    hs.count = n;
    hs.dim = 2;
    hs.boundarySum = bs.data();
    hs.sourceSum = ss.data();
    hs.nBoundary = nb.data();
    hs.mSource = ms.data();
    hs.walkSum = wsum.data();
    hs.walkCount = wc.data();
    hs.fallback = fb.data();
    check(bvc_points_download(pts, &hs), "bvc_points_download");
    double maxErr = 0.0, maxGradErr = 0.0, maxRecon = 0.0;
    for (size_t i = 0; i < n; ++i) {
        double x = grid[2 * i];
        maxErr = std::fmax(maxErr, std::fabs(u[i] - x));
        maxGradErr = std::fmax(maxGradErr, std::fabs(g[2 * i] - 1.0) + std::fabs(g[2 * i + 1]));
        // solution() = boundarySum / nBoundary (+ sourceSum / mSource) away from the band
        double v = fb[i] ? (wc[i] ? wsum[i] / wc[i] : 0.0) : (nb[i] ? bs[i] / nb[i] : 0.0) + (ms[i] ? ss[i] / ms[i] : 0.0);
        maxRecon = std::fmax(maxRecon, std::fabs(v - u[i]));
    }

    // one round on host buffers (bvc_update_solution_host, what bench.py times as e2e)
    std::vector<double> u1(n), g1(2 * n);
    bvc_round_stats st{};
    check(bvc_update_solution_host(scene, &pb, region, &cfg, grid.data(), n, seed, 0, 1, u1.data(), g1.data(), &st),
          "bvc_update_solution_host");
    double maxErr1 = 0.0;
    for (size_t i = 0; i < n; ++i) maxErr1 = std::fmax(maxErr1, std::fabs(u1[i] - grid[2 * i]));

    std::printf("{\"points\": %zu, \"rounds\": %d, \"max_abs_err_u\": %.6g, \"max_abs_err_grad\": %.6g, "
                "\"max_solution_reconstruction_err\": %.3g, \"host_round_max_abs_err_u\": %.6g, "
                "\"walks_last_round\": %lld}\n",
                n, rounds, maxErr, maxGradErr, maxRecon, maxErr1, st.cacheWalks);
    bvc_points_destroy(pts);
    bvc_region_destroy(region);
    bvc_scene_destroy(scene);
    // Monte Carlo tolerances: the max over 256 points of errors whose RMS is ~1e-2
    const bool ok = maxErr < 0.06 && maxGradErr < 0.6 && maxRecon < 1e-12 && maxErr1 < 0.12;
    return ok ? 0 : 1;
}
