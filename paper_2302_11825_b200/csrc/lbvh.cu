// lbvh.cu — BVH construction on the GPU (north star: "a GPU-built BVH").
//
// Linear BVH (Karras, HPG 2012): 64-bit Morton keys of the primitive centroids
// (2D: the primitive class in the top bits, so the tree splits Dirichlet /
// Neumann / silhouette primitives apart first, as the host builder does), one CUB
// radix sort, one thread per internal node to find its key range and split from
// common-prefix lengths, subtrees of <= leafSize primitives collapsed into leaves,
// and a bottom-up pass (atomic arrival counters) for the child boxes, class masks
// and heights. The output is the same flattened two-child node format the
// traversals read (Node2 / Node3), with primitives in leaf order.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include "internal.h"

namespace bvc_impl {

using namespace bvc_dev;

namespace {

__device__ __forceinline__ unsigned long long spread2(unsigned long long v) {  // 31 bits -> even bits
    v &= 0x7fffffffULL;
    v = (v | (v << 16)) & 0x0000ffff0000ffffULL;
    v = (v | (v << 8)) & 0x00ff00ff00ff00ffULL;
    v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0fULL;
    v = (v | (v << 2)) & 0x3333333333333333ULL;
    v = (v | (v << 1)) & 0x5555555555555555ULL;
    return v;
}
__device__ __forceinline__ unsigned long long spread3(unsigned long long v) {  // 21 bits -> every third bit
    v &= 0x1fffffULL;
    v = (v | (v << 32)) & 0x1f00000000ffffULL;
    v = (v | (v << 16)) & 0x1f0000ff0000ffULL;
    v = (v | (v << 8)) & 0x100f00f00f00f00fULL;
    v = (v | (v << 4)) & 0x10c30c30c30c30c3ULL;
    v = (v | (v << 2)) & 0x1249249249249249ULL;
    return v;
}

struct PrimIn {
    const float4* a;  // 2D: segment (a.xy, b.xy) by id; 3D: vertex a by id
    const float4* b;  // 3D: vertex b
    const float4* c;  // 3D: vertex c
    const int* cls;   // class by id
    const int2* sil;  // 2D: silhouette slots by id
    int dim;
};

__device__ __forceinline__ void prim_box(const PrimIn& in, int id, float lo[3], float hi[3]) {
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

__global__ void keys_kernel(PrimIn in, int n, float3 lo, float3 inv, int classFirst, unsigned long long* keys,
                            int* ids) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float bl[3], bh[3];
    prim_box(in, i, bl, bh);
    float cx = 0.5f * (bl[0] + bh[0]), cy = 0.5f * (bl[1] + bh[1]), cz = 0.5f * (bl[2] + bh[2]);
    unsigned long long k;
    if (in.dim == 2) {
        const float q = 1073741823.0f;  // 30 bits per axis, 2 class bits on top
        unsigned long long x = static_cast<unsigned long long>(fminf(fmaxf((cx - lo.x) * inv.x, 0.f), 1.f) * q);
        unsigned long long y = static_cast<unsigned long long>(fminf(fmaxf((cy - lo.y) * inv.y, 0.f), 1.f) * q);
        k = spread2(x) | (spread2(y) << 1);
        if (classFirst) k |= static_cast<unsigned long long>(in.cls[i] & 3) << 62;
    } else {
        const float q = 2097151.0f;  // 21 bits per axis
        unsigned long long x = static_cast<unsigned long long>(fminf(fmaxf((cx - lo.x) * inv.x, 0.f), 1.f) * q);
        unsigned long long y = static_cast<unsigned long long>(fminf(fmaxf((cy - lo.y) * inv.y, 0.f), 1.f) * q);
        unsigned long long z = static_cast<unsigned long long>(fminf(fmaxf((cz - lo.z) * inv.z, 0.f), 1.f) * q);
        k = spread3(x) | (spread3(y) << 1) | (spread3(z) << 2);
    }
    keys[i] = k;
    ids[i] = i;
}

// common prefix length of sorted keys i and j, ties broken by index (Karras 2012)
__device__ __forceinline__ int delta(const unsigned long long* k, int n, int i, int j) {
    if (j < 0 || j >= n) return -1;
    unsigned long long a = k[i], b = k[j];
    if (a == b) return 64 + __clz(static_cast<unsigned>(i ^ j));
    return __clzll(a ^ b);
}

struct Tmp {
    int lo, hi;     // leaf-order primitive range
    int left, right;  // child refs in the output encoding
    int parent;     // parent internal node (-1 for the root)
};

__global__ void radix_tree_kernel(const unsigned long long* k, int n, int leafSize, Tmp* t) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    int d = (delta(k, n, i, i + 1) - delta(k, n, i, i - 1)) >= 0 ? 1 : -1;
    int dmin = delta(k, n, i, i - d);
    int lmax = 2;
    while (delta(k, n, i, i + lmax * d) > dmin) lmax <<= 1;
    int l = 0;
    for (int s = lmax >> 1; s >= 1; s >>= 1)
        if (delta(k, n, i, i + (l + s) * d) > dmin) l += s;
    int j = i + l * d;
    int dnode = delta(k, n, i, j);
    int s = 0;
    int len = l;
    for (int step = (len + 1) >> 1;; step = (step + 1) >> 1) {
        if (delta(k, n, i, i + (s + step) * d) > dnode) s += step;
        if (step <= 1) break;
    }
    int g = i + s * d + min(d, 0);
    int lo = min(i, j), hi = max(i, j);
    Tmp r;
    r.lo = lo;
    r.hi = hi;
    int nl = g - lo + 1, nr = hi - g;
    r.left = nl <= leafSize ? ~((lo << 3) | (nl - 1)) : g;
    r.right = nr <= leafSize ? ~(((g + 1) << 3) | (nr - 1)) : g + 1;
    t[i].lo = r.lo;
    t[i].hi = r.hi;
    t[i].left = r.left;
    t[i].right = r.right;
    if (r.left >= 0) t[r.left].parent = i;
    if (r.right >= 0) t[r.right].parent = i;
    if (i == 0) t[0].parent = -1;
}

// per-node output while building: child boxes (lo xyz, hi xyz) and masks
struct Build {
    float box[2][6];
    unsigned mask[2];
    int height[2];
};

__device__ void leaf_summary(const PrimIn& in, const int* ids, int start, int count, float* box, unsigned& mask) {
    float lo[3] = {3e38f, 3e38f, 3e38f}, hi[3] = {-3e38f, -3e38f, -3e38f};
    mask = 0;
    for (int p = start; p < start + count; ++p) {
        int id = ids[p];
        float bl[3], bh[3];
        prim_box(in, id, bl, bh);
        for (int c = 0; c < 3; ++c) { lo[c] = fminf(lo[c], bl[c]); hi[c] = fmaxf(hi[c], bh[c]); }
        mask |= 1u << in.cls[id];
    }
    for (int c = 0; c < 3; ++c) { box[c] = lo[c]; box[3 + c] = hi[c]; }
}

__global__ void bottom_up_kernel(PrimIn in, const int* ids, int n, int leafSize, const Tmp* t, Build* b,
                                 unsigned* arrive) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    Tmp me = t[i];
    if (me.hi - me.lo + 1 <= leafSize && i != 0) return;  // inside a collapsed leaf: unreachable
    int done = 0;
    if (me.left < 0) {
        int code = ~me.left;
        leaf_summary(in, ids, code >> 3, (code & 7) + 1, b[i].box[0], b[i].mask[0]);
        b[i].height[0] = 0;
        ++done;
    }
    if (me.right < 0) {
        int code = ~me.right;
        leaf_summary(in, ids, code >> 3, (code & 7) + 1, b[i].box[1], b[i].mask[1]);
        b[i].height[1] = 0;
        ++done;
    }
    if (!done) return;
    __threadfence();
    int node = i;
    unsigned prev = atomicAdd(&arrive[node], static_cast<unsigned>(done));
    while (prev + done == 2) {  // both child slots of `node` are written: summarise it into its parent
        int parent = t[node].parent;
        if (parent < 0) return;
        volatile Build* vb = b + node;
        float box[6];
        for (int c = 0; c < 3; ++c) {
            box[c] = fminf(vb->box[0][c], vb->box[1][c]);
            box[3 + c] = fmaxf(vb->box[0][3 + c], vb->box[1][3 + c]);
        }
        unsigned mask = vb->mask[0] | vb->mask[1];
        int h = 1 + max(vb->height[0], vb->height[1]);
        int side = t[parent].left == node ? 0 : 1;
        for (int c = 0; c < 6; ++c) b[parent].box[side][c] = box[c];
        b[parent].mask[side] = mask;
        b[parent].height[side] = h;
        __threadfence();
        node = parent;
        done = 1;
        prev = atomicAdd(&arrive[node], 1u);
    }
}

__global__ void emit2_kernel(const Tmp* t, const Build* b, int nInternal, float pad, Node2* out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nInternal) return;
    const Build& q = b[i];
    Node2 o;
    o.lbox = make_float4(q.box[0][0] - pad, q.box[0][1] - pad, q.box[0][3] + pad, q.box[0][4] + pad);
    o.rbox = make_float4(q.box[1][0] - pad, q.box[1][1] - pad, q.box[1][3] + pad, q.box[1][4] + pad);
    o.left = t[i].left;
    o.right = t[i].right;
    o.mask = q.mask[0] | (q.mask[1] << 3);
    o.pad = 0;
    out[i] = o;
}
__global__ void emit3_kernel(const Tmp* t, const Build* b, int nInternal, float pad, Node3* out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nInternal) return;
    const Build& q = b[i];
    Node3 o;
    o.llo = make_float4(q.box[0][0] - pad, q.box[0][1] - pad, q.box[0][2] - pad, 0.f);
    o.lhi = make_float4(q.box[0][3] + pad, q.box[0][4] + pad, q.box[0][5] + pad, 0.f);
    o.rlo = make_float4(q.box[1][0] - pad, q.box[1][1] - pad, q.box[1][2] - pad, 0.f);
    o.rhi = make_float4(q.box[1][3] + pad, q.box[1][4] + pad, q.box[1][5] + pad, 0.f);
    o.set_links(t[i].left, t[i].right, q.mask[0] | (q.mask[1] << 3));
    out[i] = o;
}
__global__ void prims2_kernel(PrimIn in, const int* ids, int n, Prim2* out) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int id = ids[j];
    Prim2 p;
    p.seg = in.a[id];
    p.id = id;
    p.label = in.cls[id];
    int2 s = in.sil[id];
    p.sil0 = s.x;
    p.sil1 = s.y;
    out[j] = p;
}
__global__ void prims3_kernel(PrimIn in, const int* ids, int n, Prim3* out) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int id = ids[j];
    float4 a = in.a[id], b = in.b[id], c = in.c[id];
    Prim3 p;
    p.a = make_float4(a.x, a.y, a.z, __int_as_float(id));
    p.b = make_float4(b.x, b.y, b.z, __int_as_float(in.cls[id]));
    p.c = make_float4(c.x, c.y, c.z, 0.f);
    out[j] = p;
}
__global__ void root_height_kernel(const Build* b, int* h) { *h = 1 + max(b[0].height[0], b[0].height[1]); }

inline int blocks(long long n, int t) { return static_cast<int>((n + t - 1) / t); }

}  // namespace

// Returns the tree height (root = 1) or -1 when the scene is too small for an
// internal node (n <= leafSize: the caller hangs one leaf on a root node).
int build_lbvh(int dim, const float4* a, const float4* b, const float4* c, const int* cls, const int2* sil, int n,
               int leafSize, const double* lo, const double* hi, double pad, int classFirst, void* nodesOut,
               void* primsOut, cudaStream_t st) {
    if (n <= leafSize) return -1;
    PrimIn in{a, b, c, cls, sil, dim};
    unsigned long long *kin, *kout;
    int *vin, *vout, *h;
    Tmp* t;
    Build* bb;
    unsigned* arrive;
    cudaMallocAsync(&kin, n * sizeof(unsigned long long), st);
    cudaMallocAsync(&kout, n * sizeof(unsigned long long), st);
    cudaMallocAsync(&vin, n * sizeof(int), st);
    cudaMallocAsync(&vout, n * sizeof(int), st);
    cudaMallocAsync(&t, n * sizeof(Tmp), st);
    cudaMallocAsync(&bb, n * sizeof(Build), st);
    cudaMallocAsync(&arrive, n * sizeof(unsigned), st);
    cudaMallocAsync(&h, sizeof(int), st);
    cudaMemsetAsync(arrive, 0, n * sizeof(unsigned), st);
    float3 flo = make_float3(static_cast<float>(lo[0]), static_cast<float>(lo[1]), dim == 3 ? static_cast<float>(lo[2]) : 0.f);
    auto inv = [&](int k) { double e = hi[k] - lo[k]; return static_cast<float>(e > 0 ? 1.0 / e : 1.0); };
    float3 finv = make_float3(inv(0), inv(1), dim == 3 ? inv(2) : 1.f);
    keys_kernel<<<blocks(n, 256), 256, 0, st>>>(in, n, flo, finv, classFirst, kin, vin);
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, n, 0, 64, st);
    void* tbuf;
    cudaMallocAsync(&tbuf, tmp, st);
    cub::DeviceRadixSort::SortPairs(tbuf, tmp, kin, kout, vin, vout, n, 0, 64, st);
    radix_tree_kernel<<<blocks(n - 1, 256), 256, 0, st>>>(kout, n, leafSize, t);
    bottom_up_kernel<<<blocks(n - 1, 256), 256, 0, st>>>(in, vout, n, leafSize, t, bb, arrive);
    if (dim == 2) {
        emit2_kernel<<<blocks(n - 1, 256), 256, 0, st>>>(t, bb, n - 1, static_cast<float>(pad), static_cast<Node2*>(nodesOut));
        prims2_kernel<<<blocks(n, 256), 256, 0, st>>>(in, vout, n, static_cast<Prim2*>(primsOut));
    } else {
        emit3_kernel<<<blocks(n - 1, 256), 256, 0, st>>>(t, bb, n - 1, static_cast<float>(pad), static_cast<Node3*>(nodesOut));
        prims3_kernel<<<blocks(n, 256), 256, 0, st>>>(in, vout, n, static_cast<Prim3*>(primsOut));
    }
    root_height_kernel<<<1, 1, 0, st>>>(bb, h);
    count_launch(8);
    int height = 0;
    cudaMemcpyAsync(&height, h, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    for (void* p : {static_cast<void*>(kin), static_cast<void*>(kout), static_cast<void*>(vin), static_cast<void*>(vout),
                    static_cast<void*>(t), static_cast<void*>(bb), static_cast<void*>(arrive), static_cast<void*>(h), tbuf})
        cudaFreeAsync(p, st);
    return height;
}

// primitives in leaf order from a permutation of ids (shared with sahbvh.cu)
void launch_leaf_prims(int dim, const float4* a, const float4* b, const float4* c, const int* cls, const int2* sil,
                       const int* ids, int n, void* primsOut, cudaStream_t st) {
    PrimIn in{a, b, c, cls, sil, dim};
    if (dim == 2) prims2_kernel<<<blocks(n, 256), 256, 0, st>>>(in, ids, n, static_cast<Prim2*>(primsOut));
    else prims3_kernel<<<blocks(n, 256), 256, 0, st>>>(in, ids, n, static_cast<Prim3*>(primsOut));
    count_launch();
}

}  // namespace bvc_impl
