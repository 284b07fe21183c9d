// Spinning kernels for co-residency probes:
//   spin_launch(stream, grid, threads, cycles, carve_percent)        no shared memory
//   spin_launch_smem(stream, grid, threads, cycles, carve_percent)   16 KB static shared memory, ~100 registers
#include <cuda_runtime.h>
__global__ void spin_kernel(long long cycles, int* sink) {
    long long t0 = clock64();
    int acc = threadIdx.x;
    while (clock64() - t0 < cycles) acc = acc * 3 + 1;
    if (acc == 0x7fffffff) *sink = acc;
}
__global__ void __launch_bounds__(128, 4) spin_smem_kernel(long long cycles, int* sink) {
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
    if (s == 1.2345f) *sink = (int)s;
}
static int* sink_ptr() {
    static int* sink = nullptr;
    if (!sink) cudaMalloc(&sink, 4);
    return sink;
}
extern "C" int spin_launch(void* stream, int grid, int threads, long long cycles, int carve) {
    int* sink = sink_ptr();
    if (carve >= 0) cudaFuncSetAttribute(spin_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
    spin_kernel<<<grid, threads, 0, static_cast<cudaStream_t>(stream)>>>(cycles, sink);
    return static_cast<int>(cudaGetLastError());
}
extern "C" int spin_launch_smem(void* stream, int grid, int threads, long long cycles, int carve) {
    int* sink = sink_ptr();
    if (carve >= 0) cudaFuncSetAttribute(spin_smem_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
    spin_smem_kernel<<<grid, threads, 0, static_cast<cudaStream_t>(stream)>>>(cycles, sink);
    return static_cast<int>(cudaGetLastError());
}
