// scene3_dev.cuh — device triangle-mesh scene and BVH queries (3D).
//
// The reference's solver core is 2D-only (pointwise.cpp:23); 3D exists there only
// as kernel templates (kernels.h:78-129). BASELINE configs 4-5 are triangle
// meshes, so this is the 3D lift of scene_dev.cuh: closest point on a triangle,
// best-first traversal, and a watertight ray parity test for `inside`.
#pragma once
#include "scene_dev.cuh"

namespace bvc_dev {

// 64 bytes: one node is half a 128-byte line (4 x LDG.128). The
// child refs and the class masks live in the w slots of the boxes.
struct alignas(16) Node3 {  // 64 B; device arrays are 256-B aligned, and an over-aligned device local (a 128-B node) miscompiled
    float4 llo;  // left box lo (xyz), w = left child ref (int bits)
    float4 lhi;  // left box hi, w = right child ref
    float4 rlo;  // right box lo, w = class masks as Node2 (left | right << 3)
    float4 rhi;  // right box hi, w unused
    BVC_HD int left() const { return float_bits(llo.w); }
    BVC_HD int right() const { return float_bits(lhi.w); }
    BVC_HD unsigned mask() const { return static_cast<unsigned>(float_bits(rlo.w)); }
    BVC_HD void set_links(int l, int r, unsigned m) {
        llo.w = bits_float(l);
        lhi.w = bits_float(r);
        rlo.w = bits_float(static_cast<int>(m));
        rhi.w = 0.0f;
    }
};
static_assert(sizeof(Node3) == 64, "Node3 layout");

struct alignas(16) Prim3 {
    float4 a;  // a.xyz, w = id (as int bits)
    float4 b;  // b.xyz, w = class (as int bits)
    float4 c;  // c.xyz
};
static_assert(sizeof(Prim3) == 48, "Prim3 layout");

struct SceneView3 {
    const Node3* nodes;
    const Prim3* prims;
    const float4* triNormal;  // by triangle id: outward unit normal
    int nt;
    float diagonal;
    unsigned long long* counts;  // diagnostic traversal counters (as SceneView2)
};

template <bool COUNT = false>
__device__ __forceinline__ void count_fetch3(const SceneView3& S, int which) {
    if constexpr (COUNT) {
        if (S.counts) S.counts[2 * (blockIdx.x * blockDim.x + threadIdx.x) + which] += 1;
    }
}

__device__ __forceinline__ float box3_dist2(const float4& lo, const float4& hi, float x, float y, float z) {
    float dx = fmaxf(fmaxf(lo.x - x, 0.0f), x - hi.x);
    float dy = fmaxf(fmaxf(lo.y - y, 0.0f), y - hi.y);
    float dz = fmaxf(fmaxf(lo.z - z, 0.0f), z - hi.z);
    return dx * dx + dy * dy + dz * dz;
}
// the same with (x, y) packed: the x and y differences are two FADD2
__device__ __forceinline__ float box3_dist2(const float4& lo, const float4& hi, F2 pxy, float z) {
    float ax, ay, cx, cy;
    upk(sub2(pk(lo.x, lo.y), pxy), ax, ay);
    upk(sub2(pxy, pk(hi.x, hi.y)), cx, cy);
    float dx = fmaxf(fmaxf(ax, 0.0f), cx);
    float dy = fmaxf(fmaxf(ay, 0.0f), cy);
    float dz = fmaxf(fmaxf(lo.z - z, 0.0f), z - hi.z);
    return dx * dx + dy * dy + dz * dz;
}

// closest point on triangle abc to p (Ericson, Real-Time Collision Detection 5.1.5)
__device__ __forceinline__ float tri_closest(const Prim3& t, float px, float py, float pz, float& qx, float& qy,
                                             float& qz) {
    float ax = t.a.x, ay = t.a.y, az = t.a.z;
    float abx = t.b.x - ax, aby = t.b.y - ay, abz = t.b.z - az;
    float acx = t.c.x - ax, acy = t.c.y - ay, acz = t.c.z - az;
    float apx = px - ax, apy = py - ay, apz = pz - az;
    float d1 = abx * apx + aby * apy + abz * apz, d2 = acx * apx + acy * apy + acz * apz;
    float v, w;
    if (d1 <= 0.0f && d2 <= 0.0f) { qx = ax; qy = ay; qz = az; }
    else {
        float bpx = px - t.b.x, bpy = py - t.b.y, bpz = pz - t.b.z;
        float d3 = abx * bpx + aby * bpy + abz * bpz, d4 = acx * bpx + acy * bpy + acz * bpz;
        if (d3 >= 0.0f && d4 <= d3) { qx = t.b.x; qy = t.b.y; qz = t.b.z; }
        else {
            float vc = d1 * d4 - d3 * d2;
            if (vc <= 0.0f && d1 >= 0.0f && d3 <= 0.0f) {
                v = __fdividef(d1, d1 - d3);
                qx = ax + v * abx; qy = ay + v * aby; qz = az + v * abz;
            } else {
                float cpx = px - t.c.x, cpy = py - t.c.y, cpz = pz - t.c.z;
                float d5 = abx * cpx + aby * cpy + abz * cpz, d6 = acx * cpx + acy * cpy + acz * cpz;
                if (d6 >= 0.0f && d5 <= d6) { qx = t.c.x; qy = t.c.y; qz = t.c.z; }
                else {
                    float vb = d5 * d2 - d1 * d6;
                    if (vb <= 0.0f && d2 >= 0.0f && d6 <= 0.0f) {
                        w = __fdividef(d2, d2 - d6);
                        qx = ax + w * acx; qy = ay + w * acy; qz = az + w * acz;
                    } else {
                        float va = d3 * d6 - d5 * d4;
                        if (va <= 0.0f && (d4 - d3) >= 0.0f && (d5 - d6) >= 0.0f) {
                            w = __fdividef(d4 - d3, (d4 - d3) + (d5 - d6));
                            qx = t.b.x + w * (t.c.x - t.b.x); qy = t.b.y + w * (t.c.y - t.b.y); qz = t.b.z + w * (t.c.z - t.b.z);
                        } else {
                            float denom = __frcp_rn(va + vb + vc);
                            v = vb * denom;
                            w = vc * denom;
                            qx = ax + abx * v + acx * w; qy = ay + aby * v + acy * w; qz = az + abz * v + acz * w;
                        }
                    }
                }
            }
        }
    }
    float dx = qx - px, dy = qy - py, dz = qz - pz;
    return dx * dx + dy * dy + dz * dz;
}

// "while-while" structure (Aila & Laine, HPG 2009): each lane descends inner nodes
// in one loop and handles leaves in the next, so the warp switches between the two
// code paths once per leaf instead of once per node visit
// Entry frontiers (HintCell::front): up to 4 starts per grid cell whose subtrees together
// hold every primitive a query from the cell can need (kNoEntry = unused slot).
// `starts`: the query cell's frontier; starts.x is the first node visited, the others are
// stacked at distance 0 and visited after it. kRootStart: the whole tree.
template <bool COUNT = false, class Visit, class Thr>
__device__ __forceinline__ void traverse_near3(const SceneView3& S, float x, float y, float z, unsigned qmask,
                                               Visit&& visit, Thr&& threshold, const int4 starts = kRootStart) {
    unsigned long long stack[kStack];  // (distance bits << 32 | ref): one local load per pop
    int sp = 0;
    if (starts.w != kNoEntry) stack[sp++] = static_cast<unsigned>(starts.w);
    if (starts.z != kNoEntry) stack[sp++] = static_cast<unsigned>(starts.z);
    if (starts.y != kNoEntry) stack[sp++] = static_cast<unsigned>(starts.y);
    const int start = starts.x;
    if (start == kNoEntry) return;
    int ref = start;
    const F2 pxy = pk(x, y);
    auto pop = [&]() -> bool {  // next entry still within the pruning radius; false when empty
        for (;;) {
            if (sp == 0) return false;
            unsigned long long e = stack[--sp];
            if (__uint_as_float(static_cast<unsigned>(e >> 32)) <= threshold()) {
                ref = static_cast<int>(static_cast<unsigned>(e));
                return true;
            }
        }
    };
    for (;;) {
        while (ref >= 0) {
            const Node3 nd = S.nodes[ref];
            count_fetch3<COUNT>(S, 0);
            float thr = threshold();
            float dl = (nd.mask() & qmask) ? box3_dist2(nd.llo, nd.lhi, pxy, z) : kFInf;
            float dr = ((nd.mask() >> 3) & qmask) ? box3_dist2(nd.rlo, nd.rhi, pxy, z) : kFInf;
            bool vl = dl <= thr, vr = dr <= thr;
            if (vl && vr) {
                bool lfirst = dl <= dr;
                stack[sp++] = (static_cast<unsigned long long>(__float_as_uint(fmaxf(dl, dr))) << 32) |
                              static_cast<unsigned>(lfirst ? nd.right() : nd.left());
                ref = lfirst ? nd.left() : nd.right();
            } else if (vl) {
                ref = nd.left();
            } else if (vr) {
                ref = nd.right();
            } else if (!pop()) {
                return;
            }
        }
        int code = ~ref;
        int first = code >> 3, count = (code & 7) + 1;
        for (int i = first; i < first + count; ++i) {
            const Prim3 p = S.prims[i];
            count_fetch3<COUNT>(S, 1);
            if ((1u << __float_as_int(p.b.w)) & qmask) visit(p, i);
        }
        if (!pop()) return;
    }
}

struct Closest3 {
    float d2, px, py, pz;
    int tri;
    int prim;  // leaf-order index of the triangle (a warm-start hint for the next query)
};

// closest point on the primitive at leaf-order index `prim` (a traversal warm start)
__device__ __forceinline__ Closest3 closest_on3(const SceneView3& S, int prim, float x, float y, float z) {
    const Prim3 p = S.prims[prim];
    Closest3 c;
    c.d2 = tri_closest(p, x, y, z, c.px, c.py, c.pz);
    c.tri = __float_as_int(p.a.w);
    c.prim = prim;
    return c;
}

// hint >= 0: leaf-order index of a primitive of the queried classes whose distance
// seeds the pruning radius (the walker's previous closest triangle)
template <bool COUNT = false>
__device__ __forceinline__ Closest3 closest_point3(const SceneView3& S, float x, float y, float z, unsigned qmask,
                                                   float maxD2 = kFInf, int hint = -1, int hint2 = -1,
                                                   const int4 starts = kRootStart) {
    Closest3 c{maxD2, 0.f, 0.f, 0.f, -1, -1};
    if (hint >= 0) {
        Closest3 h = closest_on3(S, hint, x, y, z);
        if (h.d2 < c.d2) c = h;
    }
    if (hint2 >= 0 && hint2 != hint) {  // a second seed (the warm-start grid's)
        Closest3 h = closest_on3(S, hint2, x, y, z);
        if (h.d2 < c.d2) c = h;
    }
    traverse_near3<COUNT>(
        S, x, y, z, qmask,
        [&](const Prim3& p, int i) {
            float qx, qy, qz;
            float d2 = tri_closest(p, x, y, z, qx, qy, qz);
            if (d2 < c.d2) c = Closest3{d2, qx, qy, qz, __float_as_int(p.a.w), i};
        },
        [&]() { return c.d2; }, starts);
    return c;
}

// ray (o + t d, t in (0, tMax]) vs triangle: Moller-Trumbore with the edge tests
// on signed volumes computed identically for shared edges (watertight enough for
// parity counting; an exact hit on an edge counts for one of the two triangles)
__device__ __forceinline__ bool ray_tri(const Prim3& t, float ox, float oy, float oz, float dx, float dy, float dz,
                                        float tMax, float& tHit) {
    float e1x = t.b.x - t.a.x, e1y = t.b.y - t.a.y, e1z = t.b.z - t.a.z;
    float e2x = t.c.x - t.a.x, e2y = t.c.y - t.a.y, e2z = t.c.z - t.a.z;
    float px = dy * e2z - dz * e2y, py = dz * e2x - dx * e2z, pz = dx * e2y - dy * e2x;
    float det = e1x * px + e1y * py + e1z * pz;
    if (det == 0.0f) return false;
    float inv = 1.0f / det;
    float sx = ox - t.a.x, sy = oy - t.a.y, sz = oz - t.a.z;
    float u = (sx * px + sy * py + sz * pz) * inv;
    if (u < 0.0f || u > 1.0f) return false;
    float qx = sy * e1z - sz * e1y, qy = sz * e1x - sx * e1z, qz = sx * e1y - sy * e1x;
    float v = (dx * qx + dy * qy + dz * qz) * inv;
    if (v < 0.0f || u + v > 1.0f) return false;
    float tt = (e2x * qx + e2y * qy + e2z * qz) * inv;
    if (tt <= 0.0f || tt > tMax) return false;
    tHit = tt;
    return true;
}

__device__ __forceinline__ bool ray_box3(const float4& lo, const float4& hi, float ox, float oy, float oz, float idx,
                                         float idy, float idz, float tMax) {
    float t0 = 0.0f, t1 = tMax;
    float tn = (lo.x - ox) * idx, tf = (hi.x - ox) * idx;
    t0 = fmaxf(t0, fminf(tn, tf)); t1 = fminf(t1, fmaxf(tn, tf));
    tn = (lo.y - oy) * idy; tf = (hi.y - oy) * idy;
    t0 = fmaxf(t0, fminf(tn, tf)); t1 = fminf(t1, fmaxf(tn, tf));
    tn = (lo.z - oz) * idz; tf = (hi.z - oz) * idz;
    t0 = fmaxf(t0, fminf(tn, tf)); t1 = fminf(t1, fmaxf(tn, tf));
    return t0 <= t1;
}

// the same slab test, returning the entry distance (kFInf on a miss)
// oxi = ox * idx etc. (see ray_box_t in scene_dev.cuh): one FFMA per slab bound
__device__ __forceinline__ float ray_box3_t(const float4& lo, const float4& hi, F2 noixy, float nozi, F2 idxy, float idz,
                                            float tMax) {
    float tnx, tny, tfx, tfy;
    upk(fma2(pk(lo.x, lo.y), idxy, noixy), tnx, tny);
    upk(fma2(pk(hi.x, hi.y), idxy, noixy), tfx, tfy);
    float tnz = fmaf(lo.z, idz, nozi), tfz = fmaf(hi.z, idz, nozi);
    float t0 = fmaxf(fmaxf(fminf(tnx, tfx), fminf(tny, tfy)), fmaxf(fminf(tnz, tfz), 0.0f));
    float t1 = fminf(fminf(fmaxf(tnx, tfx), fmaxf(tny, tfy)), fminf(fmaxf(tnz, tfz), tMax));
    return t0 <= t1 ? t0 : kFInf;
}

// entry_node (scene_dev.cuh) on the 3D tree
__device__ __forceinline__ int entry_node3(const SceneView3& S, float x, float y, float z, float r2, unsigned qmask) {
    int ref = 0;
    while (ref >= 0) {
        const Node3 nd = S.nodes[ref];
        const bool vl = (nd.mask() & qmask) && box3_dist2(nd.llo, nd.lhi, x, y, z) <= r2;
        const bool vr = ((nd.mask() >> 3) & qmask) && box3_dist2(nd.rlo, nd.rhi, x, y, z) <= r2;
        if (vl && vr) return ref;
        if (vl) ref = nd.left();
        else if (vr) ref = nd.right();
        else return kNoEntry;
    }
    return ref;
}

// Up to 4 nodes whose subtrees together hold every primitive of qmask within
// sqrt(r2) of p: entry_node3's node, then, while there is room, a frontier node whose two
// children both qualify is replaced by them (single qualifying children are descended
// into, nodes with none dropped). A cell straddling a high split of the tree gets deep
// starts on both sides instead of their common ancestor. f[0] == kNoEntry: none.
__device__ __forceinline__ void entry_frontier3(const SceneView3& S, float x, float y, float z, float r2,
                                                unsigned qmask, int (&f)[4]) {
    for (int k = 0; k < 4; ++k) f[k] = kNoEntry;
    f[0] = entry_node3(S, x, y, z, r2, qmask);
    int nf = f[0] == kNoEntry ? 0 : 1;
    for (int guard = 0; guard < 1024; ++guard) {
        bool changed = false;
        for (int i = 0; i < nf; ++i) {
            const int ref = f[i];
            if (ref < 0) continue;  // a leaf
            const Node3 nd = S.nodes[ref];
            const bool vl = (nd.mask() & qmask) && box3_dist2(nd.llo, nd.lhi, x, y, z) <= r2;
            const bool vr = ((nd.mask() >> 3) & qmask) && box3_dist2(nd.rlo, nd.rhi, x, y, z) <= r2;
            if (vl && vr) {
                if (nf < 4) {
                    f[i] = nd.left();
                    f[nf++] = nd.right();
                    changed = true;
                }
            } else if (vl || vr) {
                f[i] = vl ? nd.left() : nd.right();
                changed = true;
            } else {
                f[i] = f[--nf];
                f[nf] = kNoEntry;
                changed = true;
                --i;
            }
        }
        if (!changed) break;
    }
}

// inside: boundary-inclusive within tol, then ray-crossing parity along a fixed
// irrational direction (avoids axis-aligned edge degeneracies of meshes)
__device__ __forceinline__ bool inside3(const SceneView3& S, float x, float y, float z, float tol) {
    Closest3 c = closest_point3(S, x, y, z, kClsAny, tol * tol);
    if (c.tri >= 0) return true;
    const float dx = 0.57735027f * 1.0000193f, dy = 0.57735027f * 0.9999871f, dz = 0.57735027f;
    float n = rsqrtf(dx * dx + dy * dy + dz * dz);
    float rx = dx * n, ry = dy * n, rz = dz * n;
    float idx = 1.0f / rx, idy = 1.0f / ry, idz = 1.0f / rz;
    bool in = false;
    int stack[kStack];
    int sp = 0, ref = 0;
    for (;;) {
        if (ref >= 0) {
            const Node3 nd = S.nodes[ref];
            bool vl = (nd.mask() & 7u) && ray_box3(nd.llo, nd.lhi, x, y, z, idx, idy, idz, kFInf);
            bool vr = ((nd.mask() >> 3) & 7u) && ray_box3(nd.rlo, nd.rhi, x, y, z, idx, idy, idz, kFInf);
            if (vl && vr) { stack[sp++] = nd.right(); ref = nd.left(); continue; }
            if (vl) { ref = nd.left(); continue; }
            if (vr) { ref = nd.right(); continue; }
        } else {
            int code = ~ref;
            int start = code >> 3, count = (code & 7) + 1;
            for (int i = start; i < start + count; ++i) {
                float th;
                if (ray_tri(S.prims[i], x, y, z, rx, ry, rz, kFInf, th)) in = !in;
            }
        }
        if (sp == 0) return in;
        ref = stack[--sp];
    }
}

}  // namespace bvc_dev
