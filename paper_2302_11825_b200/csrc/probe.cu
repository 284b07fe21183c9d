// probe.cu — pipe and cache microbenchmarks behind the rooflines (SURVEY §8d asks for
// the FP32 and MUFU issue rates and an L2 bandwidth to be measured, not assumed).
//
// Each probe runs independent dependency chains (8 per thread) so the pipe, not the
// latency, is the limit; times come from CUDA events around one warm launch.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/bvc_b200.h"
#include "internal.h"

namespace bvc_impl {
namespace {

constexpr int kIters = 4096;

template <int OP>
__global__ void __launch_bounds__(256) pipe_kernel(float* out, float seed) {
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = seed + 0.001f * (threadIdx.x + k);
#pragma unroll 16
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if constexpr (OP == 0) v[k] = fmaf(v[k], 0.999f, 0.0001f);
            else if constexpr (OP == 1) { float y; asm volatile("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[k])); v[k] = y; }
            else if constexpr (OP == 2) {  // + c: ptxas folds rcp(rcp(x)) chains away
                float y; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[k])); v[k] = y + 0.5f;
            }
            else if constexpr (OP == 4) { float y; asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[k])); v[k] = y; }
            else { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[k])); v[k] = y; }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
    if (s == 1.2345f) out[threadIdx.x] = s;  // keep the chains alive
}

// register-operand forms (no immediates / constant-bank operands): OP 0 FFMA, 1 FMUL, 2 FADD
template <int OP>
__global__ void __launch_bounds__(256) pipe_reg_kernel(float* out, float seed) {
    float v[8];
    const float m = 0.999f + 1e-9f * threadIdx.x, c = 1e-4f * (1.0f + 1e-9f * threadIdx.x);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = seed + 0.001f * (threadIdx.x + k);
#pragma unroll 16
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if constexpr (OP == 0) v[k] = fmaf(v[k], m, c);
            else if constexpr (OP == 1) v[k] = v[k] * m;
            else v[k] = v[k] + c;
        }
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
    if (s == 1.2345f) out[threadIdx.x] = s;
}

// packed FP32 (FFMA2, sm_100a): each instruction does two FMAs
__global__ void __launch_bounds__(256) ffma2_kernel(float* out, float seed) {
    unsigned long long v[8];
    const float m = 0.999f + 1e-9f * threadIdx.x, c = 1e-4f;
    unsigned long long M, Cc;
    asm("mov.b64 %0, {%1, %2};" : "=l"(M) : "f"(m), "f"(m));
    asm("mov.b64 %0, {%1, %2};" : "=l"(Cc) : "f"(c), "f"(c));
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        float a = seed + 0.001f * (threadIdx.x + k), b = a + 0.5f;
        asm("mov.b64 %0, {%1, %2};" : "=l"(v[k]) : "f"(a), "f"(b));
    }
#pragma unroll 16
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[k]) : "l"(M), "l"(Cc));
    }
    unsigned long long s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s ^= v[k];
    if (s == 12345ull) out[threadIdx.x] = 1.f;
}

__global__ void __launch_bounds__(256) dfma_kernel(double* out, double seed) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = seed + 0.001 * (threadIdx.x + k);
#pragma unroll 16
    for (int i = 0; i < kIters / 4; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = fma(v[k], 0.999, 0.0001);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
    if (s == 1.2345) out[threadIdx.x] = s;
}

// L2-resident read bandwidth: every CTA streams the same 32 MB buffer (< 126 MB L2)
__global__ void __launch_bounds__(256) l2_kernel(const float4* buf, size_t n, int reps, float* out) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (int r = 0; r < reps; ++r)
        for (size_t i = (blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x + r * 977u) % n; ; ) {
            float4 x = __ldcg(buf + i);
            acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
            i += stride;
            if (i >= n) break;
        }
    if (acc.x + acc.y + acc.z + acc.w == 1.2345f) out[threadIdx.x] = acc.x;
}

}  // namespace
}  // namespace bvc_impl

using namespace bvc_impl;

extern "C" int bvc_pipe_probe(int which, double* opsPerSecond) {
    if (!opsPerSecond) return BVC_ERR_INVALID_ARGUMENT;
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return BVC_ERR_NO_DEVICE;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    void* scratch = nullptr;
    cudaMalloc(&scratch, 64 << 20);
    const int grid = sms * 8, threads = 256;
    double ops = 0.0;
    float ms = 0.f;
    if (which == 6) cudaMemset(scratch, 0, 32 << 20);
    for (int pass = 0; pass < 2; ++pass) {  // pass 0 warms up
        cudaEventRecord(a);
        switch (which) {
            case 0: pipe_kernel<0><<<grid, threads>>>(static_cast<float*>(scratch), 1.0f); ops = 1.0; break;
            case 1: pipe_kernel<1><<<grid, threads>>>(static_cast<float*>(scratch), 1.5f); ops = 1.0; break;
            case 2: pipe_kernel<2><<<grid, threads>>>(static_cast<float*>(scratch), 1.5f); ops = 1.0; break;
            case 3: dfma_kernel<<<grid, threads>>>(static_cast<double*>(scratch), 1.0); ops = 0.25; break;
            case 4: pipe_kernel<4><<<grid, threads>>>(static_cast<float*>(scratch), 1.5f); ops = 1.0; break;
            case 5: pipe_kernel<5><<<grid, threads>>>(static_cast<float*>(scratch), 0.5f); ops = 1.0; break;
            case 7: pipe_reg_kernel<0><<<grid, threads>>>(static_cast<float*>(scratch), 1.0f); ops = 1.0; break;
            case 8: pipe_reg_kernel<1><<<grid, threads>>>(static_cast<float*>(scratch), 1.0f); ops = 1.0; break;
            case 9: pipe_reg_kernel<2><<<grid, threads>>>(static_cast<float*>(scratch), 1.0f); ops = 1.0; break;
            case 10: ffma2_kernel<<<grid, threads>>>(static_cast<float*>(scratch), 1.0f); ops = 2.0; break;
            case 6: {
                size_t n = (32u << 20) / sizeof(float4);
                l2_kernel<<<grid, threads>>>(static_cast<const float4*>(scratch), n, 8,
                                             static_cast<float*>(scratch) + (48 << 18));
                ops = 0.0;
                break;
            }
            default: cudaFree(scratch); return BVC_ERR_INVALID_ARGUMENT;
        }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
    }
    count_launch(2);
    double sec = ms * 1e-3;
    if (which == 6) *opsPerSecond = 8.0 * (32u << 20) / sec;  // bytes/s
    else *opsPerSecond = static_cast<double>(grid) * threads * 8.0 * kIters * ops / sec;
    cudaFree(scratch);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return cudaGetLastError() == cudaSuccess ? BVC_OK : BVC_ERR_CUDA;
}
