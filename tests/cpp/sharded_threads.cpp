// sharded_threads.cpp — the multi-GPU round driven from C++ (include/bvc_b200.h), one host
// thread per rank, built and run by tests/test_capi_cpp.py. The ranks exchange their
// cache shards through a host-staged all-gather written here (bvc_comm_init_callback), so
// the program runs wherever the ranks share or own GPUs: with one GPU all ranks share it
// (nothing in a kernel waits on another rank; only the host exchange does). Each rank's
// points get the sums of the single-rank round bit for bit.
//
//   ./sharded_threads [ranks]   exit 0: equal; 3: no CUDA device; 1: failure
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <mutex>
#include <stdexcept>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "bvc_b200.h"

namespace {

struct BvcFailure : std::runtime_error {
    int status;
    BvcFailure(int s, const char* what) : std::runtime_error(what), status(s) {}
};
void check(int status, const char* what) {
    if (status != BVC_OK) throw BvcFailure(status, what);
}

// an in-process all-gather over host memory: every rank copies its device shard to its
// slot, waits for the others, and copies the whole buffer back to its device
struct HostExchange {
    int ranks;
    std::vector<unsigned char> buf;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0, generation = 0, left = 0;
};
struct RankCtx {
    HostExchange* x;
    int rank;
};
int allgather(const void* send, void* recv, size_t bytes, void* user, void* /*stream*/) {
    auto* c = static_cast<RankCtx*>(user);
    HostExchange& x = *c->x;
    std::unique_lock<std::mutex> lk(x.mu);
    x.cv.wait(lk, [&] { return x.left == 0; });  // the previous exchange has been read by all
    if (x.arrived == 0) x.buf.assign(bytes * x.ranks, 0);
    lk.unlock();
    // synchronous copies: the library drained its stream before calling
    std::vector<unsigned char> tmp(bytes);
    if (bytes && cudaMemcpy(tmp.data(), send, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
    lk.lock();
    std::memcpy(x.buf.data() + bytes * c->rank, tmp.data(), bytes);
    const int gen = x.generation;
    if (++x.arrived == x.ranks) {
        x.arrived = 0;
        x.left = x.ranks;
        ++x.generation;
        x.cv.notify_all();
    } else {
        x.cv.wait(lk, [&] { return x.generation != gen; });
    }
    std::vector<unsigned char> all(x.buf);
    if (--x.left == 0) x.cv.notify_all();
    lk.unlock();
    return bytes && cudaMemcpy(recv, all.data(), bytes * x.ranks, cudaMemcpyHostToDevice) != cudaSuccess ? 1 : 0;
}

}  // namespace

static int run(int ranks);

int main(int argc, char** argv) {
    const int ranks = argc > 1 ? std::atoi(argv[1]) : 2;
    try {
        return run(ranks);
    } catch (const BvcFailure& e) {
        if (e.status == BVC_ERR_NO_DEVICE) {
            std::printf("no device: %s\n", bvc_last_error());
            return 3;
        }
        std::fprintf(stderr, "%s: status %d: %s\n", e.what(), e.status, bvc_last_error());
        return 1;
    }
}

static int run(int ranks) {
    // square-mixed-linear on [-1,1]^2 with 64 segments per side
    const int per = 64;
    std::vector<double> xy;
    std::vector<int> ab, labels;
    const double cx[4] = {-1, 1, 1, -1}, cy[4] = {-1, -1, 1, 1};
    for (int side = 0; side < 4; ++side)
        for (int k = 0; k < per; ++k) {
            double t = static_cast<double>(k) / per;
            xy.push_back(cx[side] + t * (cx[(side + 1) % 4] - cx[side]));
            xy.push_back(cy[side] + t * (cy[(side + 1) % 4] - cy[side]));
        }
    for (int i = 0; i < 4 * per; ++i) {
        ab.push_back(i);
        ab.push_back((i + 1) % (4 * per));
        labels.push_back((i / per) % 2 == 0 ? BVC_NEUMANN : BVC_DIRICHLET);
    }
    bvc_scene scene = nullptr;
    check(bvc_scene_create(xy.data(), 4 * per, ab.data(), labels.data(), 4 * per, &scene), "scene");
    bvc_region_request req{BVC_REGION_WHOLE_DOMAIN, 0.02, nullptr};
    bvc_region region = nullptr;
    check(bvc_region_build(scene, &req, 2e-3, &region), "region");
    bvc_problem pb{};
    pb.kernel = {BVC_KERNEL_POISSON, 0.0, 2, 2.828};
    pb.g.kind = BVC_FIELD_LINEAR;
    pb.g.p[0] = 1.0;
    bvc_cache_config cfg{1001, 1024, 32, 64, 0.02, 0, BVC_CLAMP_OFF, 0, 4, 0, 1, {2e-3, 0, 10000, 64, 0, 0}, 0};
    const size_t n = 3000;
    std::vector<double> x(2 * n);
    unsigned s = 12345;
    for (double& v : x) {
        s = s * 1664525u + 1013904223u;
        v = -0.99 + 1.98 * ((s >> 8) / 16777216.0);
    }
    // the single-rank round
    std::vector<double> u1(n), g1(2 * n);
    bvc_round_stats st{};
    check(bvc_update_solution_host(scene, &pb, region, &cfg, x.data(), n, 9, 0, 1, u1.data(), g1.data(), &st), "one");
    // the sharded round, one thread per rank
    HostExchange ex;
    ex.ranks = ranks;
    std::vector<double> u(n), g(2 * n);
    std::vector<int> status(ranks, BVC_OK);
    std::vector<std::thread> th;
    for (int r = 0; r < ranks; ++r)
        th.emplace_back([&, r] {
            long long b = 0, e = 0, cap = 0;
            bvc_shard_layout(static_cast<long long>(n), ranks, r, &b, &e, &cap);
            RankCtx ctx{&ex, r};
            bvc_comm comm = nullptr;
            int rc = bvc_comm_init_callback(ranks, r, allgather, &ctx, &comm);
            if (rc == BVC_OK)
                rc = bvc_update_solution_sharded_host(comm, scene, &pb, region, &cfg, x.data() + 2 * b,
                                                      static_cast<size_t>(e - b), b, 9, 0, 1, u.data() + b,
                                                      g.data() + 2 * b, nullptr);
            if (comm) bvc_comm_destroy(comm);
            status[r] = rc;
        });
    for (auto& t : th) t.join();
    for (int r = 0; r < ranks; ++r) check(status[r], "sharded round");
    const bool same = std::memcmp(u.data(), u1.data(), n * sizeof(double)) == 0 &&
                      std::memcmp(g.data(), g1.data(), 2 * n * sizeof(double)) == 0;
    std::printf("{\"ranks\": %d, \"points\": %zu, \"bitwise_equal\": %s}\n", ranks, n, same ? "true" : "false");
    bvc_region_destroy(region);
    bvc_scene_destroy(scene);
    return same ? 0 : 1;
}
