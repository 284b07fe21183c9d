// gather64.cu — the FP64 variant of the splat gather (BASELINE C1 "u (fp32 and fp64)").
//
// Same decomposition as gather.cu (point tiles x K-independent sample chunks, a
// dynamic unit queue, TMA bulk-copied double-buffered sample tiles, fixed-order
// partials reduced by launch_finalize), but every pair is evaluated in FP64 with
// the reference's exact coincidence test (r < 1e-12 diag, cache.cpp:436-440) on
// each pair, so sums match the reference's double loop to rounding. Poisson
// kernels only (2D and 3D): FP64 has no SFU, so 1/r^2 and 1/r come from the FP32
// MUFU estimate plus two Newton steps and ln r^2 from libdevice's log.
//
// Reference: splatSolution / splatGradient cache.cpp:426-497, kernels.h:78-129.
#include <cuda_runtime.h>

#include "gather.h"
#include "tma.cuh"

namespace bvc_impl {

using namespace bvc_dev;

namespace {

constexpr int kThreads64 = 128;
constexpr int kQ64 = 2;
constexpr int kPT64 = kThreads64 * kQ64;  // points per CTA tile
constexpr int kTS64 = 128;                // samples per shared-memory tile (2 x double4 each)
constexpr double kInv2PiD = 0.15915494309189533577, kInv4PiD = 0.07957747154594766788;

struct Acc64 {
    double v, gx, gy, gz;
};

// 1/r2 to full FP64 accuracy: FP32 MUFU seed (r2 >= tol^2 = 1e-24 diag^2 is a
// normal float) and two Newton steps (error ~1e-28 relative before rounding)
__device__ __forceinline__ double rcp64(double x) {
    double y = static_cast<double>(__frcp_rn(static_cast<float>(x)));
    y = y * fma(-x, y, 2.0);
    return y * fma(-x, y, 2.0);
}
__device__ __forceinline__ double rsqrt64(double x) {
    double y = static_cast<double>(rsqrtf(static_cast<float>(x)));
    y = y * fma(-0.5 * x * y, y, 1.5);
    return y * fma(-0.5 * x * y, y, 1.5);
}

// 2D boundary payload a = (zx, zy, A nx, A ny), b = (Bln, Bg, 0, 0):
//   A = w u / 2pi, Bln = w d / 4pi (G = ln r^2 / 4pi), Bg = w d / 2pi
// 2D source: a = (yx, yy, Cs, Cg), Cs = c / 4pi, Cg = c / 2pi (c = f / pdf)
// 3D boundary: a = (zx, zy, zz, nx), b = (ny, nz, A = w u / 4pi, B = w d / 4pi)
// 3D source: a = (yx, yy, yz, C = c / 4pi)
template <int KIND, bool SRC, bool VAL, bool GRAD>
__device__ __forceinline__ void pair64(const double4& a, const double4& b, double px, double py, double pz,
                                       double tol2, Acc64& acc, int& skip) {
    if constexpr (KIND == kLap2) {
        double dx = a.x - px, dy = a.y - py;
        double r2 = fma(dx, dx, dy * dy);
        if (r2 < tol2) { ++skip; return; }
        double ir2 = rcp64(r2);
        if constexpr (!SRC) {
            double ndA = fma(a.z, dx, a.w * dy);
            if constexpr (VAL) acc.v = fma(ndA, ir2, fma(-b.x, log(r2), acc.v));
            if constexpr (GRAD) {
                double q = fma(2.0 * ndA, ir2, b.y) * ir2;
                acc.gx = fma(q, dx, fma(-ir2, a.z, acc.gx));
                acc.gy = fma(q, dy, fma(-ir2, a.w, acc.gy));
            }
        } else {
            if constexpr (VAL) acc.v = fma(a.z, log(r2), acc.v);
            if constexpr (GRAD) {
                double c = a.w * ir2;
                acc.gx = fma(-c, dx, acc.gx);
                acc.gy = fma(-c, dy, acc.gy);
            }
        }
    } else {
        double dx = a.x - px, dy = a.y - py, dz = a.z - pz;
        double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
        if (r2 < tol2) { ++skip; return; }
        double ir = rsqrt64(r2);
        double ir2 = ir * ir, ir3 = ir2 * ir;
        if constexpr (!SRC) {
            double nd = fma(a.w, dx, fma(b.x, dy, b.y * dz));
            double pn = nd * ir3;
            if constexpr (VAL) acc.v = fma(b.z, pn, fma(b.w, ir, acc.v));
            if constexpr (GRAD) {
                double q = fma(3.0 * b.z, pn * ir2, b.w * ir3);
                double c = b.z * ir3;
                acc.gx = fma(q, dx, fma(-c, a.w, acc.gx));
                acc.gy = fma(q, dy, fma(-c, b.x, acc.gy));
                acc.gz = fma(q, dz, fma(-c, b.y, acc.gz));
            }
        } else {
            if constexpr (VAL) acc.v = fma(-a.w, ir, acc.v);
            if constexpr (GRAD) {
                double c = a.w * ir3;
                acc.gx = fma(-c, dx, acc.gx);
                acc.gy = fma(-c, dy, acc.gy);
                acc.gz = fma(-c, dz, acc.gz);
            }
        }
    }
}

struct Params64 {
    const double4* pack;  // 2 double4 per sample; boundary [0, N), source [N, N+M)
    int N, M;
    const double* px;     // dim * K, sorted order
    int K, dim;
    int chunk, chunksB, chunksS, tiles;
    double tol2;
    double* part;         // [(chunksB + chunksS)][comps][K]
    int comps;
    int* skipB;
    int* skipS;
    unsigned* unitCounter;
};

template <int KIND, bool VAL, bool GRAD>
__global__ void __launch_bounds__(kThreads64) gather64_kernel(const Params64 P) {
    __shared__ __align__(128) double4 sm[2][2 * kTS64];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ int sUnit;
    constexpr bool D3 = KIND == kLap3;
    const int tid = threadIdx.x;
    const int units = P.tiles * (P.chunksB + P.chunksS);
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned phase[2] = {0u, 0u};
    for (int unit = blockIdx.x; unit < units;) {
        const int chunkId = unit % (P.chunksB + P.chunksS);
        const int tile = unit / (P.chunksB + P.chunksS);
        const bool src = chunkId >= P.chunksB;
        const int c0 = src ? P.N + (chunkId - P.chunksB) * P.chunk : chunkId * P.chunk;
        const int cEnd = src ? min(c0 + P.chunk, P.N + P.M) : min(c0 + P.chunk, P.N);
        const int nT = (cEnd - c0 + kTS64 - 1) / kTS64;
        double px[kQ64], py[kQ64], pz[kQ64];
        int pidx[kQ64];
#pragma unroll
        for (int q = 0; q < kQ64; ++q) {
            int i = tile * kPT64 + q * kThreads64 + tid;
            pidx[q] = i;
            bool ok = i < P.K;
            px[q] = ok ? P.px[P.dim * i] : 1e300;
            py[q] = ok ? P.px[P.dim * i + 1] : 1e300;
            pz[q] = (ok && D3) ? P.px[P.dim * i + 2] : 0.0;
        }
        Acc64 acc[kQ64];
        int skips[kQ64];
#pragma unroll
        for (int q = 0; q < kQ64; ++q) { acc[q] = Acc64{0.0, 0.0, 0.0, 0.0}; skips[q] = 0; }
        if (tid == 0) {
#pragma unroll
            for (int st = 0; st < 2; ++st)
                if (st < nT) {
                    int s0 = c0 + st * kTS64, cnt = min(kTS64, cEnd - s0);
                    mbar_expect_tx(&bar[st], cnt * 64u);
                    bulk_g2s(sm[st], P.pack + 2 * static_cast<size_t>(s0), cnt * 64u, &bar[st]);
                }
        }
        for (int it = 0; it < nT; ++it) {
            const int st = it & 1;
            const int s0 = c0 + it * kTS64, cnt = min(kTS64, cEnd - s0);
            mbar_wait(&bar[st], phase[st]);
            phase[st] ^= 1u;
            const double4* S = sm[st];
#pragma unroll 1
            for (int j = 0; j < cnt; ++j) {
                const double4 a = S[2 * j], b = S[2 * j + 1];
#pragma unroll
                for (int q = 0; q < kQ64; ++q) {
                    if (!src) pair64<KIND, false, VAL, GRAD>(a, b, px[q], py[q], pz[q], P.tol2, acc[q], skips[q]);
                    else pair64<KIND, true, VAL, GRAD>(a, b, px[q], py[q], pz[q], P.tol2, acc[q], skips[q]);
                }
            }
            __syncthreads();
            if (tid == 0 && it + 2 < nT) {
                int s2 = c0 + (it + 2) * kTS64, cnt2 = min(kTS64, cEnd - s2);
                mbar_expect_tx(&bar[st], cnt2 * 64u);
                bulk_g2s(sm[st], P.pack + 2 * static_cast<size_t>(s2), cnt2 * 64u, &bar[st]);
            }
        }
        double* out = P.part + static_cast<size_t>(chunkId) * P.comps * P.K;
#pragma unroll
        for (int q = 0; q < kQ64; ++q) {
            int i = pidx[q];
            if (i >= P.K) continue;
            int c = 0;
            if (VAL) out[static_cast<size_t>(c++) * P.K + i] = acc[q].v;
            if (GRAD) {
                out[static_cast<size_t>(c++) * P.K + i] = acc[q].gx;
                out[static_cast<size_t>(c++) * P.K + i] = acc[q].gy;
                if (D3) out[static_cast<size_t>(c++) * P.K + i] = acc[q].gz;
            }
            if (skips[q]) atomicAdd(src ? P.skipS + i : P.skipB + i, skips[q]);
        }
        if (tid == 0) sUnit = static_cast<int>(gridDim.x + atomicAdd(P.unitCounter, 1u));
        __syncthreads();
        unit = sUnit;
        __syncthreads();
    }
}

__global__ void pack64_boundary_kernel(const CacheSample* cs, int n, int kind, int voronoi, double4* out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const CacheSample& s = cs[i];
    double w = voronoi ? static_cast<double>(s.weight) * n : 1.0 / static_cast<double>(s.pdf);
    double u = s.uHat, d = s.dHat;
    if (kind == kLap2) {
        double A = w * u * kInv2PiD;
        out[2 * i] = make_double4(s.z[0], s.z[1], A * s.n[0], A * s.n[1]);
        out[2 * i + 1] = make_double4(w * d * kInv4PiD, w * d * kInv2PiD, 0.0, 0.0);
    } else {
        out[2 * i] = make_double4(s.z[0], s.z[1], s.z[2], s.n[0]);
        out[2 * i + 1] = make_double4(s.n[1], s.n[2], w * u * kInv4PiD, w * d * kInv4PiD);
    }
}

__global__ void pack64_source_kernel(const SourceSampleDev* ss, int m, int kind, double4* out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const SourceSampleDev& s = ss[i];
    double c = static_cast<double>(s.f) / static_cast<double>(s.pdf);
    if (kind == kLap2) out[2 * i] = make_double4(s.y[0], s.y[1], c * kInv4PiD, c * kInv2PiD);
    else out[2 * i] = make_double4(s.y[0], s.y[1], s.y[2], c * kInv4PiD);
    out[2 * i + 1] = make_double4(0.0, 0.0, 0.0, 0.0);
}

__global__ void gather_points64_kernel(const double* x, const int* order, int K, int dim, double* out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K) return;
    int p = order[i];
    for (int d = 0; d < dim; ++d) out[static_cast<size_t>(dim) * i + d] = x[static_cast<size_t>(dim) * p + d];
}

template <int KIND>
void launch64_kind(const Params64& P, bool val, bool grad, int grid, cudaStream_t st) {
    if (val && grad) gather64_kernel<KIND, true, true><<<grid, kThreads64, 0, st>>>(P);
    else if (val) gather64_kernel<KIND, true, false><<<grid, kThreads64, 0, st>>>(P);
    else gather64_kernel<KIND, false, true><<<grid, kThreads64, 0, st>>>(P);
}

template <int KIND>
int occupancy64(bool val, bool grad) {
    int occ = 0;
    if (val && grad) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gather64_kernel<KIND, true, true>, kThreads64, 0);
    else if (val) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gather64_kernel<KIND, true, false>, kThreads64, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gather64_kernel<KIND, false, true>, kThreads64, 0);
    return occ > 0 ? occ : 1;
}

inline int blocks(long long n, int t) { return static_cast<int>((n + t - 1) / t); }

}  // namespace

void pack64_boundary(const CacheSample* cs, int n, int kind, int voronoi, double4* out, cudaStream_t st) {
    if (n <= 0) return;
    pack64_boundary_kernel<<<blocks(n, 256), 256, 0, st>>>(cs, n, kind, voronoi, out);
    count_launch();
}
void pack64_source(const SourceSampleDev* ss, int m, int kind, double4* out, cudaStream_t st) {
    if (m <= 0) return;
    pack64_source_kernel<<<blocks(m, 256), 256, 0, st>>>(ss, m, kind, out);
    count_launch();
}
void gather_points64(const double* x, const int* order, int K, int dim, double* out, cudaStream_t st) {
    if (K <= 0) return;
    gather_points64_kernel<<<blocks(K, 256), 256, 0, st>>>(x, order, K, dim, out);
    count_launch();
}

GatherPlan plan_gather64(int kind, int K, int N, int M, bool val, bool grad) {
    GatherPlan g = plan_gather(kind, K, N, M, val, grad);  // the same K-independent chunks
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int occ = kind == kLap2 ? occupancy64<kLap2>(val, grad) : occupancy64<kLap3>(val, grad);
    g.tiles = (K + kPT64 - 1) / kPT64;
    long long units = static_cast<long long>(g.tiles) * (g.chunksB + g.chunksS);
    long long slots = static_cast<long long>(sms) * occ;
    g.grid = static_cast<int>(units < slots ? units : slots);
    g.grid = g.grid > 0 ? g.grid : 1;
    return g;
}

void launch_gather64(int kind, const GatherPlan& g, const double4* pack, int N, int M, const double* px, int K,
                     int dim, double tol, bool val, bool grad, double* part, int* skipB, int* skipS,
                     unsigned* unitCounter, cudaStream_t st) {
    if (K <= 0 || (N + M) <= 0) return;
    Params64 P;
    P.pack = pack;
    P.N = N;
    P.M = M;
    P.px = px;
    P.K = K;
    P.dim = dim;
    P.chunk = g.chunk;
    P.chunksB = g.chunksB;
    P.chunksS = g.chunksS;
    P.tiles = g.tiles;
    P.tol2 = tol * tol;
    P.part = part;
    P.comps = g.comps;
    P.skipB = skipB;
    P.skipS = skipS;
    P.unitCounter = unitCounter;
    cudaMemsetAsync(unitCounter, 0, sizeof(unsigned), st);
    if (kind == kLap2) launch64_kind<kLap2>(P, val, grad, g.grid, st);
    else launch64_kind<kLap3>(P, val, grad, g.grid, st);
    count_launch();
}

}  // namespace bvc_impl
