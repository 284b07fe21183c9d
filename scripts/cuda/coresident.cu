// Co-residency micro-test: a persistent 1-CTA-per-SM kernel A (256 threads, small registers,
// optional local-memory stack) and a 4-CTA-per-SM kernel B (128 threads, ~100 registers, 16 KB
// static shared memory) on two streams. total ~ max(A, B) => the SM hosts both; ~ A + B => not.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o coresident coresident.cu && ./coresident
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <bool LMEM>
__global__ void __launch_bounds__(256, 8) kernelA(long long cycles, int* sink) {
    long long t0 = clock64();
    unsigned long long stack[48];
    int sp = 0, acc = threadIdx.x;
    while (clock64() - t0 < cycles) {
        if (LMEM) {
            stack[sp & 47] = acc;
            sp = (sp * 5 + 1) & 63;
            acc += (int)stack[(sp + acc) & 47];
        } else {
            acc = acc * 3 + 1;
        }
    }
    if (acc == 0x7fffffff) *sink = acc + (LMEM ? (int)stack[3] : 0);
}

__global__ void __launch_bounds__(128, 4) kernelB(long long cycles, float* sink) {
    __shared__ float sm[4096];
    float r[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) r[i] = threadIdx.x + i;
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    long long t0 = clock64();
    while (clock64() - t0 < cycles) {
#pragma unroll
        for (int i = 0; i < 64; ++i) r[i] = fmaf(r[i], 1.0001f, sm[(threadIdx.x + i) & 4095]);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 64; ++i) s += r[i];
    if (s == 1.2345f) *sink = s;
}

static int g_dynA = 0;
static float run(int which, bool lmem, int gridA, long long cyc, cudaStream_t sa, cudaStream_t sb, int* si, float* sf) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaDeviceSynchronize();
    cudaEventRecord(e0, 0);
    cudaStreamWaitEvent(sa, e0, 0); cudaStreamWaitEvent(sb, e0, 0);
    if (which & 1) { if (lmem) kernelA<true><<<gridA, 256, g_dynA, sa>>>(cyc, si); else kernelA<false><<<gridA, 256, g_dynA, sa>>>(cyc, si); }
    if (which & 2) kernelB<<<592, 128, 0, sb>>>(cyc, sf);
    cudaEvent_t ea, eb;
    cudaEventCreate(&ea); cudaEventCreate(&eb);
    cudaEventRecord(ea, sa); cudaEventRecord(eb, sb);
    cudaStreamWaitEvent(0, ea, 0); cudaStreamWaitEvent(0, eb, 0);
    cudaEventRecord(e1, 0);
    cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

int main(int argc, char** argv) {
    const int mode = argc > 1 ? atoi(argv[1]) : 0;
    const int carve = argc > 2 ? atoi(argv[2]) : -1;   // preferred shared-memory carve-out (percent) on both kernels
    const int dynA = argc > 3 ? atoi(argv[3]) : 0;     // dynamic shared memory given to A (bytes)
    g_dynA = dynA;
    if (carve >= 0) {
        cudaFuncSetAttribute(kernelA<true>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
        cudaFuncSetAttribute(kernelA<false>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
        cudaFuncSetAttribute(kernelB, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
    }
    printf("carve %d dynA %d\n", carve, dynA);  // 0: A high priority, 1: equal priorities, 2: A low priority
    int* si; float* sf;
    cudaMalloc(&si, 4); cudaMalloc(&sf, 4);
    cudaStream_t sa, sb;
    int lo, hi; cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&sa, cudaStreamNonBlocking, mode == 0 ? hi : lo);
    cudaStreamCreateWithPriority(&sb, cudaStreamNonBlocking, mode == 2 ? hi : lo);
    printf("mode %d (priority range %d..%d) CUDA_LAUNCH_BLOCKING=%s\n", mode, lo, hi, getenv("CUDA_LAUNCH_BLOCKING") ? getenv("CUDA_LAUNCH_BLOCKING") : "unset");
    cudaFuncAttributes fa, fb;
    cudaFuncGetAttributes(&fa, kernelA<true>); cudaFuncGetAttributes(&fb, kernelB);
    printf("A regs %d lmem %zu; B regs %d smem %zu\n", fa.numRegs, fa.localSizeBytes, fb.numRegs, fb.sharedSizeBytes);
    const long long cyc = 400000000LL;  // ~0.2 s
    for (int lmem = 0; lmem < 2; ++lmem)
        for (int gridA : {148, 1184}) {
            run(3, lmem, gridA, 1000, sa, sb, si, sf);
            float a = run(1, lmem, gridA, cyc, sa, sb, si, sf), b = run(2, lmem, gridA, cyc, sa, sb, si, sf);
            float ab = run(3, lmem, gridA, cyc, sa, sb, si, sf);
            printf("lmem %d gridA %4d: A alone %.1f ms, B alone %.1f ms, together %.1f ms\n", lmem, gridA, a, b, ab);
        }
    return 0;
}
