// sahbvh.cu — binned-SAH BVH construction on the GPU, breadth first.
//
// The same splitting rules as the host builder (host_scene.cpp buildBvh): 32 bins
// per axis over the centroid bounds, cost A(left) N(left) + A(right) N(right); in
// 2D a node holding several primitive classes splits by class first; no valid SAH
// split (coincident centroids) or depth >= 24 splits the range in half. One CTA
// per node of the current level: centroid bounds and bins in shared memory, the
// split chosen by one thread, then a stable in-place partition of the node's
// primitive range with block scans; children at or below the leaf size become
// leaves, the others are appended to the next level. Output: the flattened
// two-child node format the traversals read (Node2 / Node3) and leaf-order ids.
#include <cuda_runtime.h>

#include <cub/block/block_scan.cuh>

#include "internal.h"

namespace bvc_impl {

using namespace bvc_dev;

namespace {

constexpr int kB = 128;    // threads per node CTA
constexpr int kBins = 32;

struct SahIn {
    const float4* a;  // 2D: segment by id; 3D: vertex a
    const float4* b;  // 3D: vertex b
    const float4* c;  // 3D: vertex c
    const int* cls;
    int dim;
};

struct Task {
    int start, count, node, depth;
};

__device__ __forceinline__ void pbox(const SahIn& in, int id, float lo[3], float hi[3]) {
    if (in.dim == 2) {
        float4 s = in.a[id];
        lo[0] = fminf(s.x, s.z); hi[0] = fmaxf(s.x, s.z);
        lo[1] = fminf(s.y, s.w); hi[1] = fmaxf(s.y, s.w);
        lo[2] = hi[2] = 0.f;
    } else {
        float4 a = in.a[id], b = in.b[id], c = in.c[id];
        lo[0] = fminf(a.x, fminf(b.x, c.x)); hi[0] = fmaxf(a.x, fmaxf(b.x, c.x));
        lo[1] = fminf(a.y, fminf(b.y, c.y)); hi[1] = fmaxf(a.y, fmaxf(b.y, c.y));
        lo[2] = fminf(a.z, fminf(b.z, c.z)); hi[2] = fmaxf(a.z, fmaxf(b.z, c.z));
    }
}

// float min/max through ordered-int atomics in shared memory
__device__ __forceinline__ int fkey(float f) { int i = __float_as_int(f); return i >= 0 ? i : i ^ 0x7fffffff; }
__device__ __forceinline__ float fval(int k) { return __int_as_float(k >= 0 ? k : k ^ 0x7fffffff); }

__device__ __forceinline__ float area(const float lo[3], const float hi[3], int dim) {
    if (lo[0] > hi[0]) return 0.f;
    float ex = hi[0] - lo[0], ey = hi[1] - lo[1], ez = hi[2] - lo[2];
    return dim == 2 ? ex + ey : ex * ey + ey * ez + ez * ex;
}

struct Split {
    int mode;        // 0 SAH bin split, 1 class split, 2 half by index
    int axis, bin, cls;
    float clo[3], cext[3];
    int nLeft;
    float lbox[6], rbox[6];
    unsigned lmask, rmask;
};

__global__ void __launch_bounds__(kB) sah_level_kernel(SahIn in, int* ids, int* tmp, const Task* tasks, int nTasks,
                                                      int leafSize, float pad, int classFirst, Task* next,
                                                      int* nextCount, int* nodeCounter, void* nodesOut) {
    using BlockScan = cub::BlockScan<int, kB>;
    __shared__ typename BlockScan::TempStorage scanTmp;
    __shared__ int sLo[3], sHi[3];
    __shared__ int bCnt[3][kBins];
    __shared__ int bLo[3][kBins][3], bHi[3][kBins][3];
    __shared__ unsigned sMask, bMask[3][kBins];
    __shared__ Split sp;
    __shared__ int sRun[2];
    const int t = threadIdx.x;
    const Task task = tasks[blockIdx.x];
    const int s0 = task.start, n = task.count;
    // 1) centroid bounds and the class mask of the node
    if (t < 3) { sLo[t] = fkey(3e38f); sHi[t] = fkey(-3e38f); }
    if (t == 0) sMask = 0;
    __syncthreads();
    float clo[3] = {3e38f, 3e38f, 3e38f}, chi[3] = {-3e38f, -3e38f, -3e38f};
    unsigned mask = 0;
    for (int i = t; i < n; i += kB) {
        int id = ids[s0 + i];
        float lo[3], hi[3];
        pbox(in, id, lo, hi);
        for (int k = 0; k < 3; ++k) {
            float c = 0.5f * (lo[k] + hi[k]);
            clo[k] = fminf(clo[k], c);
            chi[k] = fmaxf(chi[k], c);
        }
        mask |= 1u << in.cls[id];
    }
    for (int k = 0; k < 3; ++k) {
        atomicMin(&sLo[k], fkey(clo[k]));
        atomicMax(&sHi[k], fkey(chi[k]));
    }
    atomicOr(&sMask, mask);
    for (int i = t; i < 3 * kBins; i += kB) {
        int ax = i / kBins, bi = i % kBins;
        bCnt[ax][bi] = 0;
        bMask[ax][bi] = 0;
        for (int k = 0; k < 3; ++k) { bLo[ax][bi][k] = fkey(3e38f); bHi[ax][bi][k] = fkey(-3e38f); }
    }
    __syncthreads();
    const unsigned nodeMask = sMask;
    const bool byClass = classFirst && (nodeMask & (nodeMask - 1));
    float lo0[3], ext[3];
    for (int k = 0; k < 3; ++k) { lo0[k] = fval(sLo[k]); ext[k] = fval(sHi[k]) - lo0[k]; }
    // 2) bins (all axes; the split also needs the class masks and boxes per side)
    if (!byClass) {
        for (int i = t; i < n; i += kB) {
            int id = ids[s0 + i];
            float lo[3], hi[3];
            pbox(in, id, lo, hi);
            for (int ax = 0; ax < in.dim; ++ax) {
                if (!(ext[ax] > 0.f)) continue;
                float c = 0.5f * (lo[ax] + hi[ax]);
                int bi = min(kBins - 1, static_cast<int>((c - lo0[ax]) / ext[ax] * kBins));
                atomicAdd(&bCnt[ax][bi], 1);
                atomicOr(&bMask[ax][bi], 1u << in.cls[id]);
                for (int k = 0; k < 3; ++k) {
                    atomicMin(&bLo[ax][bi][k], fkey(lo[k]));
                    atomicMax(&bHi[ax][bi][k], fkey(hi[k]));
                }
            }
        }
    }
    __syncthreads();
    // 3) choose the split
    if (t == 0) {
        Split s{};
        s.mode = 2;
        s.nLeft = n / 2;
        if (byClass) {
            s.mode = 1;
            s.cls = __ffs(nodeMask) - 1;
        } else if (task.depth < 24) {
            float best = 3.4e38f;
            for (int ax = 0; ax < in.dim; ++ax) {
                if (!(ext[ax] > 0.f)) continue;
                float rA[kBins];
                int rN[kBins];
                float rl[3] = {3e38f, 3e38f, 3e38f}, rh[3] = {-3e38f, -3e38f, -3e38f};
                int cnt = 0;
                for (int bi = kBins - 1; bi > 0; --bi) {
                    for (int k = 0; k < 3; ++k) { rl[k] = fminf(rl[k], fval(bLo[ax][bi][k])); rh[k] = fmaxf(rh[k], fval(bHi[ax][bi][k])); }
                    cnt += bCnt[ax][bi];
                    rA[bi] = area(rl, rh, in.dim);
                    rN[bi] = cnt;
                }
                float ll[3] = {3e38f, 3e38f, 3e38f}, lh[3] = {-3e38f, -3e38f, -3e38f};
                int nl = 0;
                for (int bi = 0; bi < kBins - 1; ++bi) {
                    for (int k = 0; k < 3; ++k) { ll[k] = fminf(ll[k], fval(bLo[ax][bi][k])); lh[k] = fmaxf(lh[k], fval(bHi[ax][bi][k])); }
                    nl += bCnt[ax][bi];
                    if (nl == 0 || rN[bi + 1] == 0) continue;
                    float cost = area(ll, lh, in.dim) * nl + rA[bi + 1] * rN[bi + 1];
                    if (cost < best) { best = cost; s.mode = 0; s.axis = ax; s.bin = bi; s.nLeft = nl; }
                }
            }
        }
        for (int k = 0; k < 3; ++k) { s.clo[k] = lo0[k]; s.cext[k] = ext[k]; }
        sp = s;
        sRun[0] = 0;
        sRun[1] = 0;
    }
    __syncthreads();
    const Split s = sp;
    // 4) stable partition into tmp, left part first; side boxes and masks on the fly
    int nLeftTotal = s.nLeft;  // bin and half modes know it; the class mode counts it
    if (s.mode == 1) {
        int nl = 0, dummy;
        for (int i = t; i < n; i += kB) nl += in.cls[ids[s0 + i]] == s.cls ? 1 : 0;
        BlockScan(scanTmp).ExclusiveSum(nl, dummy, nLeftTotal);
        __syncthreads();
    }
    float blo[2][3], bhi[2][3];
    unsigned bm[2] = {0u, 0u};
    for (int k = 0; k < 3; ++k) { blo[0][k] = blo[1][k] = 3e38f; bhi[0][k] = bhi[1][k] = -3e38f; }
    for (int base = 0; base < n; base += kB) {
        int i = base + t;
        int id = i < n ? ids[s0 + i] : 0;
        int left = 0;
        float lo[3], hi[3];
        if (i < n) {
            pbox(in, id, lo, hi);
            if (s.mode == 0) {
                float c = 0.5f * (lo[s.axis] + hi[s.axis]);
                int bi = min(kBins - 1, static_cast<int>((c - s.clo[s.axis]) / s.cext[s.axis] * kBins));
                left = bi <= s.bin;
            } else if (s.mode == 1) {
                left = in.cls[id] == s.cls;
            } else {
                left = i < s.nLeft;
            }
            int side = left ? 0 : 1;
            for (int k = 0; k < 3; ++k) { blo[side][k] = fminf(blo[side][k], lo[k]); bhi[side][k] = fmaxf(bhi[side][k], hi[k]); }
            bm[side] |= 1u << in.cls[id];
        }
        int lRank, lTot;
        BlockScan(scanTmp).ExclusiveSum(left, lRank, lTot);
        __syncthreads();
        if (i < n) {
            int rRank = (i - base) - lRank;  // rank among this chunk's right elements
            int pos = left ? sRun[0] + lRank : nLeftTotal + sRun[1] + rRank;
            tmp[s0 + pos] = id;
        }
        __syncthreads();
        if (t == 0) {
            int chunk = min(kB, n - base);
            sRun[0] += lTot;
            sRun[1] += chunk - lTot;
        }
        __syncthreads();
    }
    for (int i = t; i < n; i += kB) ids[s0 + i] = tmp[s0 + i];
    // side boxes / masks: block reductions through the shared bin arrays (reused)
    __syncthreads();
    if (t < 2) {
        for (int k = 0; k < 3; ++k) { bLo[0][t][k] = fkey(3e38f); bHi[0][t][k] = fkey(-3e38f); }
        bMask[0][t] = 0;
    }
    __syncthreads();
    for (int side = 0; side < 2; ++side) {
        for (int k = 0; k < 3; ++k) {
            atomicMin(&bLo[0][side][k], fkey(blo[side][k]));
            atomicMax(&bHi[0][side][k], fkey(bhi[side][k]));
        }
        atomicOr(&bMask[0][side], bm[side]);
    }
    __syncthreads();
    // 5) emit this node and the child tasks
    if (t == 0) {
        int nl = nLeftTotal, nr = n - nLeftTotal;
        if (nl == 0 || nr == 0) { nl = n / 2; nr = n - nl; }  // cannot happen for valid splits; stay safe
        int ref[2];
        int cnts[2] = {nl, nr}, starts[2] = {s0, s0 + nl};
        for (int side = 0; side < 2; ++side) {
            if (cnts[side] <= leafSize) {
                ref[side] = ~((starts[side] << 3) | (cnts[side] - 1));
            } else {
                int node = atomicAdd(nodeCounter, 1);
                ref[side] = node;
                int slot = atomicAdd(nextCount, 1);
                next[slot] = Task{starts[side], cnts[side], node, task.depth + 1};
            }
        }
        float bx[2][6];
        for (int side = 0; side < 2; ++side)
            for (int k = 0; k < 3; ++k) {
                bx[side][k] = fval(bLo[0][side][k]) - pad;
                bx[side][3 + k] = fval(bHi[0][side][k]) + pad;
            }
        unsigned m = bMask[0][0] | (bMask[0][1] << 3);
        if (in.dim == 2) {
            Node2 o;
            o.lbox = make_float4(bx[0][0], bx[0][1], bx[0][3], bx[0][4]);
            o.rbox = make_float4(bx[1][0], bx[1][1], bx[1][3], bx[1][4]);
            o.left = ref[0];
            o.right = ref[1];
            o.mask = m;
            o.pad = 0;
            static_cast<Node2*>(nodesOut)[task.node] = o;
        } else {
            Node3 o;
            o.llo = make_float4(bx[0][0], bx[0][1], bx[0][2], 0.f);
            o.lhi = make_float4(bx[0][3], bx[0][4], bx[0][5], 0.f);
            o.rlo = make_float4(bx[1][0], bx[1][1], bx[1][2], 0.f);
            o.rhi = make_float4(bx[1][3], bx[1][4], bx[1][5], 0.f);
            o.set_links(ref[0], ref[1], m);
            static_cast<Node3*>(nodesOut)[task.node] = o;
        }
    }
}

__global__ void iota_kernel(int* v, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = i;
}

}  // namespace

// Returns the tree depth (levels), or -1 if n <= leafSize. `idsOut` receives the
// leaf order (n ints, device); nodesOut needs n - 1 nodes of capacity.
int build_sah_gpu(int dim, const float4* a, const float4* b, const float4* c, const int* cls, int n, int leafSize,
                  double pad, int classFirst, void* nodesOut, int* idsOut, cudaStream_t st) {
    if (n <= leafSize) return -1;
    SahIn in{a, b, c, cls, dim};
    int *tmp, *counts;
    Task *cur, *nxt;
    cudaMallocAsync(&tmp, n * sizeof(int), st);
    cudaMallocAsync(&cur, n * sizeof(Task), st);
    cudaMallocAsync(&nxt, n * sizeof(Task), st);
    cudaMallocAsync(&counts, 2 * sizeof(int), st);  // [0] next-level task count, [1] node counter
    iota_kernel<<<(n + 255) / 256, 256, 0, st>>>(idsOut, n);
    Task root{0, n, 0, 0};
    cudaMemcpyAsync(cur, &root, sizeof(Task), cudaMemcpyHostToDevice, st);
    const int init[2] = {0, 1};  // next-level task count, node counter (the root is node 0)
    cudaMemcpyAsync(counts, init, 2 * sizeof(int), cudaMemcpyHostToDevice, st);
    int nTasks = 1, levels = 0;
    while (nTasks > 0) {
        cudaMemsetAsync(counts, 0, sizeof(int), st);
        sah_level_kernel<<<nTasks, kB, 0, st>>>(in, idsOut, tmp, cur, nTasks, leafSize, static_cast<float>(pad),
                                                classFirst, nxt, counts, counts + 1, nodesOut);
        ++levels;
        int h[2];
        cudaMemcpyAsync(h, counts, 2 * sizeof(int), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        nTasks = h[0];
        std::swap(cur, nxt);
        if (levels > 60) break;
    }
    count_launch(levels + 1);
    cudaFreeAsync(tmp, st);
    cudaFreeAsync(cur, st);
    cudaFreeAsync(nxt, st);
    cudaFreeAsync(counts, st);
    return levels;
}

}  // namespace bvc_impl
