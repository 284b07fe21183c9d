// scene_dev.cuh — device scene layout and BVH traversals (2D segments).
//
// Replaces the reference's recursive AoS double-precision BVH queries
// (bvh.h:107-146, bvh.cpp:53-83, scene.cpp:133-254) with stack-based FP32
// traversals over a flattened binary BVH whose nodes hold both child boxes
// (one 48-byte node fetch orders and prunes both children).
#pragma once
#include <cstdint>

#include "device_math.cuh"

namespace bvc_dev {

constexpr float kFInf = __builtin_huge_valf();

struct alignas(16) Node2 {
    float4 lbox;  // lo.x, lo.y, hi.x, hi.y
    float4 rbox;
    int left, right;  // >= 0 internal node; < 0 leaf: ~((start << 3) | (count - 1))
    unsigned mask;    // left class mask | right class mask << 3 (classes: host_scene.h primClass)
    int pad;
};

struct alignas(16) Prim2 {
    float4 seg;      // a.x, a.y, b.x, b.y
    int id;          // caller-side segment index
    int label;       // class: 0 Dirichlet, 1 Neumann, 2 Neumann with silhouette candidates
    int sil0, sil1;  // silhouette candidate slots (-1 none)
};

struct SceneView2 {
    const Node2* nodes;
    const Prim2* prims;        // leaf order
    const float2* segNormal;   // by segment id: unit outward normal
    const float4* segAB;       // by segment id: a.x, a.y, b.x, b.y
    const float2* silP;        // silhouette vertex
    const float4* silN;        // n1, n2
    const int* silAlways;
    int ns;
    float diagonal;
    // diagnostic traversal counters (NULL in production launches): per thread,
    // [2 t] node fetches (48 B each), [2 t + 1] primitive fetches (32 B each)
    unsigned long long* counts;
};

// compiled in only for the instrumented launch (bvc_walk_traffic_profile)
template <bool COUNT>
__device__ __forceinline__ void count_fetch(const SceneView2& S, int which) {
    if constexpr (COUNT) {
        if (S.counts) S.counts[2 * (blockIdx.x * blockDim.x + threadIdx.x) + which] += 1;
    }
}

__device__ __forceinline__ float box_dist2(const float4& b, float x, float y) {
    float dx = fmaxf(fmaxf(b.x - x, 0.0f), x - b.z);
    float dy = fmaxf(fmaxf(b.y - y, 0.0f), y - b.w);
    return dx * dx + dy * dy;
}
// the same with p = (x, y) packed: the four differences are two FADD2
__device__ __forceinline__ float box_dist2(const float4& b, F2 p) {
    float ax, ay, cx, cy;
    upk(sub2(pk(b.x, b.y), p), ax, ay);
    upk(sub2(p, pk(b.z, b.w)), cx, cy);
    float dx = fmaxf(fmaxf(ax, 0.0f), cx);
    float dy = fmaxf(fmaxf(ay, 0.0f), cy);
    return dx * dx + dy * dy;
}

// closest point on a segment (bvh.h:153-159); returns squared distance
__device__ __forceinline__ float seg_closest(const float4& s, float x, float y, float& px, float& py, float& t) {
    float ux = s.z - s.x, uy = s.w - s.y;
    float l2 = ux * ux + uy * uy;
    // fast division: t only places the closest point, and the distance is
    // stationary in t there, so a 2-ulp quotient moves d^2 at second order
    float tt = l2 > 0.0f ? __fdividef((x - s.x) * ux + (y - s.y) * uy, l2) : 0.0f;
    tt = fminf(fmaxf(tt, 0.0f), 1.0f);
    px = fmaf(tt, ux, s.x);
    py = fmaf(tt, uy, s.y);
    t = tt;
    float dx = px - x, dy = py - y;
    return dx * dx + dy * dy;
}

constexpr int kStack = 48;
// primitive class masks (host_scene.h primClass)
constexpr unsigned kClsD = 1u, kClsN = 2u, kClsSil = 4u;
constexpr unsigned kClsNeumann = kClsN | kClsSil, kClsAny = kClsD | kClsN | kClsSil;

// Generic best-first traversal. visit(prim) handles one primitive of a visited
// leaf; threshold() returns the current squared pruning radius. "While-while"
// structure (Aila & Laine, HPG 2009): inner nodes in one loop, leaves in the next.
// Entry refs (HintGrid): a traversal may start at a subtree known to hold every
// primitive that can matter for the query (start = 0: the root); kNoEntry = none.
constexpr int kNoEntry = -2147483647 - 1;
// starts of a traversal (HintCell::front): .x first, the others stacked; kRootStart: the whole tree
#define kRootStart make_int4(0, kNoEntry, kNoEntry, kNoEntry)

template <bool COUNT = false, class Visit, class Thr>
__device__ __forceinline__ void traverse_near(const SceneView2& S, float x, float y, unsigned qmask, Visit&& visit,
                                              Thr&& threshold, const int4 starts = kRootStart) {
    // (distance bits << 32 | ref) per entry: one local load per pop
    unsigned long long stack[kStack];
    int sp = 0;
    // the cell's entry frontier (entry_frontier2): starts 2-4 stacked at distance 0
    if (starts.w != kNoEntry) stack[sp++] = static_cast<unsigned>(starts.w);
    if (starts.z != kNoEntry) stack[sp++] = static_cast<unsigned>(starts.z);
    if (starts.y != kNoEntry) stack[sp++] = static_cast<unsigned>(starts.y);
    const int start = starts.x;
    if (start == kNoEntry) return;
    int ref = start;
    const F2 p2 = pk(x, y);
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
            const Node2 nd = S.nodes[ref];
            count_fetch<COUNT>(S, 0);
            float thr = threshold();
            float dl = (nd.mask & qmask) ? box_dist2(nd.lbox, p2) : kFInf;
            float dr = ((nd.mask >> 3) & qmask) ? box_dist2(nd.rbox, p2) : kFInf;
            bool vl = dl <= thr, vr = dr <= thr;
            if (vl && vr) {
                int nearRef = dl <= dr ? nd.left : nd.right;
                int farRef = dl <= dr ? nd.right : nd.left;
                stack[sp++] = (static_cast<unsigned long long>(__float_as_uint(fmaxf(dl, dr))) << 32) |
                              static_cast<unsigned>(farRef);
                ref = nearRef;
            } else if (vl) {
                ref = nd.left;
            } else if (vr) {
                ref = nd.right;
            } else if (!pop()) {
                return;
            }
        }
        int code = ~ref;
        int first = code >> 3, count = (code & 7) + 1;
        for (int i = first; i < first + count; ++i) {
            const Prim2 p = S.prims[i];
            count_fetch<COUNT>(S, 1);
            if ((1u << p.label) & qmask) visit(p);
        }
        if (!pop()) return;
    }
}

struct Closest {
    float d2;
    float px, py, t;
    int seg;
};

// closest point of one segment (by id) as a traversal warm start
__device__ __forceinline__ Closest closest_on(const SceneView2& S, int seg, float x, float y) {
    Closest c;
    c.d2 = seg_closest(S.segAB[seg], x, y, c.px, c.py, c.t);
    c.seg = seg;
    return c;
}

// Scene::closestPoint (scene.cpp:133-144; bvh.cpp:53-69). hint >= 0: a segment of
// the queried classes whose distance seeds the pruning radius (the walker's
// previous closest segment), so far subtrees are never pushed.
template <bool COUNT = false>
__device__ __forceinline__ Closest closest_point(const SceneView2& S, float x, float y, unsigned qmask,
                                                 float maxD2 = kFInf, int hint = -1, int hint2 = -1,
                                                 const int4 starts = kRootStart) {
    Closest c{maxD2, 0.0f, 0.0f, 0.0f, -1};
    if (hint >= 0) {
        Closest h = closest_on(S, hint, x, y);
        if (h.d2 < c.d2) c = h;
    }
    if (hint2 >= 0 && hint2 != hint) {  // a second seed (the warm-start grid's)
        Closest h = closest_on(S, hint2, x, y);
        if (h.d2 < c.d2) c = h;
    }
    traverse_near<COUNT>(
        S, x, y, qmask,
        [&](const Prim2& p) {
            float px, py, t;
            float d2 = seg_closest(p.seg, x, y, px, py, t);
            if (d2 < c.d2) { c.d2 = d2; c.px = px; c.py = py; c.t = t; c.seg = p.id; }
        },
        [&]() { return c.d2; }, starts);
    return c;
}

// silhouetteTest (scene.cpp:166-172)
__device__ __forceinline__ bool silhouette_ok(const SceneView2& S, int k, float x, float y, float& d2) {
    float2 p = S.silP[k];
    float dx = p.x - x, dy = p.y - y;
    d2 = dx * dx + dy * dy;
    if (S.silAlways[k]) return true;
    float4 n = S.silN[k];
    float d1 = n.x * dx + n.y * dy, d2n = n.z * dx + n.w * dy;
    return d1 * d2n <= 0.0f;
}

// Scene::silhouetteDistance (scene.cpp:174-185); returns squared distance
template <bool COUNT = false>
__device__ __forceinline__ float silhouette_dist2(const SceneView2& S, float x, float y) {
    float best = kFInf;
    traverse_near<COUNT>(
        S, x, y, kClsSil,
        [&](const Prim2& p) {
            float d2;
            if (p.sil0 >= 0 && silhouette_ok(S, p.sil0, x, y, d2) && d2 < best) best = d2;
            if (p.sil1 >= 0 && silhouette_ok(S, p.sil1, x, y, d2) && d2 < best) best = d2;
        },
        [&]() { return best; });
    return best;
}

// One WoSt step's geometry in a single traversal: the closest Dirichlet point and
// the closest visible Neumann silhouette vertex (pointwise.cpp:216-222). Pruning
// uses max(min(bestD, bestS), eps): everything the reference's two separate
// queries would decide on (termination within eps; R = min(dD, dS)) is exact.
struct StarQuery {
    Closest D;
    float s2;
};
template <bool COUNT = false>
__device__ __forceinline__ StarQuery star_query(const SceneView2& S, float x, float y, float eps2, int hint = -1,
                                                int hint2 = -1, const int4 starts = kRootStart) {
    StarQuery q;
    q.D = hint >= 0 ? closest_on(S, hint, x, y) : Closest{kFInf, 0.0f, 0.0f, 0.0f, -1};
    if (hint2 >= 0 && hint2 != hint) {
        Closest h = closest_on(S, hint2, x, y);
        if (h.d2 < q.D.d2) q.D = h;
    }
    q.s2 = kFInf;
    traverse_near<COUNT>(
        S, x, y, kClsD | kClsSil,
        [&](const Prim2& p) {
            if (p.label == 0) {
                float px, py, t;
                float d2 = seg_closest(p.seg, x, y, px, py, t);
                if (d2 < q.D.d2) { q.D.d2 = d2; q.D.px = px; q.D.py = py; q.D.t = t; q.D.seg = p.id; }
            } else {
                // a silhouette no closer than the closest Dirichlet point cannot shorten
                // R = min(dD, dS) (pointwise.cpp:136-138) nor the pruning radius
                float d2;
                if (p.sil0 >= 0 && silhouette_ok(S, p.sil0, x, y, d2) && d2 < fminf(q.s2, q.D.d2)) q.s2 = d2;
                if (p.sil1 >= 0 && silhouette_ok(S, p.sil1, x, y, d2) && d2 < fminf(q.s2, q.D.d2)) q.s2 = d2;
            }
        },
        [&]() { return fmaxf(fminf(q.D.d2, q.s2), eps2); }, starts);
    return q;
}

// slab test against o + t d, t in [0, tMax] (bvh.h:32-43)
__device__ __forceinline__ bool ray_box(const float4& b, float ox, float oy, float idx, float idy, float tMax) {
    float t0 = 0.0f, t1 = tMax;
    float tn = (b.x - ox) * idx, tf = (b.z - ox) * idx;
    if (tn > tf) { float s = tn; tn = tf; tf = s; }
    t0 = fmaxf(t0, tn);
    t1 = fminf(t1, tf);
    if (t0 > t1) return false;
    tn = (b.y - oy) * idy;
    tf = (b.w - oy) * idy;
    if (tn > tf) { float s = tn; tn = tf; tf = s; }
    t0 = fmaxf(t0, tn);
    t1 = fminf(t1, tf);
    return t0 <= t1;
}

// the same slab test, returning the entry distance (kFInf on a miss). Takes the
// origin premultiplied by the reciprocal direction (oxi = ox * idx), so each slab
// bound is one FFMA; the rounding of oxi moves a slab by about ulp(ox) in position,
// far inside the boxes' padding. An axis with idx = inf yields NaN bounds, which
// fminf / fmaxf drop: that axis then does not constrain (conservative).
__device__ __forceinline__ float ray_box_t(const float4& b, F2 noi, F2 id, float tMax) {  // noi = -(ox idx, oy idy)
    float tnx, tny, tfx, tfy;
    upk(fma2(pk(b.x, b.y), id, noi), tnx, tny);
    upk(fma2(pk(b.z, b.w), id, noi), tfx, tfy);
    float t0 = fmaxf(fmaxf(fminf(tnx, tfx), fminf(tny, tfy)), 0.0f);
    float t1 = fminf(fminf(fmaxf(tnx, tfx), fmaxf(tny, tfy)), tMax);
    return t0 <= t1 ? t0 : kFInf;
}

// side of v relative to the ray o + t d; explicit roundings (no FMA contraction)
// so a vertex shared by two segments is classified identically for both
__device__ __forceinline__ float ray_side(float dx, float dy, float ox, float oy, float vx, float vy) {
    return __fsub_rn(__fmul_rn(dx, __fsub_rn(vy, oy)), __fmul_rn(dy, __fsub_rn(vx, ox)));
}

struct RayHit {
    float t, s, px, py;
    int seg;
};

// Scene::intersectRay (scene.cpp:196-208; raySegment bvh.cpp:71-83): first hit
// with t in (tMin, tMax] among the filtered segments, skipping `skipSeg` (the
// segment the walk currently stands on: a ray leaving a straight segment cannot
// hit it again, and skipping it keeps FP32 re-hits out).
// one segment against the ray o + t d (unit d), keeping the nearest hit with
// tMin < t <= limit in h (limit shrinks to it). Watertight crossing test: each endpoint
// is classified by its side of the ray; a vertex shared by two segments gets the same
// sign in both, so a ray can never slip between them (raySegment bvh.cpp:71-83 decides
// via s in [0,1], which FP32 cancellation breaks near vertices).
__device__ __forceinline__ void ray_segment_hit(const float4 seg, int id, float ox, float oy, float dx, float dy,
                                                float tMin, float& limit, RayHit& h) {
    float sa = ray_side(dx, dy, ox, oy, seg.x, seg.y);
    float sb = ray_side(dx, dy, ox, oy, seg.z, seg.w);
    if ((sa > 0.0f && sb > 0.0f) || (sa < 0.0f && sb < 0.0f)) return;
    float den = sa - sb;  // = cross(d, e) with e = b - a, up to sign convention
    if (den == 0.0f) return;  // parallel / collinear: miss
    float s = sa / den;
    float ex = seg.z - seg.x, ey = seg.w - seg.y;
    float px = fmaf(s, ex, seg.x), py = fmaf(s, ey, seg.y);
    float t = (px - ox) * dx + (py - oy) * dy;  // unit direction: distance along the ray
    if (t <= 0.0f || t > limit) return;
    if (t > tMin && t < h.t) {
        h.t = t; h.s = s; h.seg = id;
        h.px = px; h.py = py;
        limit = t;
    }
}

template <bool COUNT = false>
__device__ __forceinline__ RayHit intersect_ray(const SceneView2& S, float ox, float oy, float dx, float dy,
                                                float tMax, unsigned qmask, float tMin, int skipSeg, int start = 0) {
    RayHit h{kFInf, 0.0f, 0.0f, 0.0f, -1};
    if (start == kNoEntry) return h;
    float idx = f_rcp(dx), idy = f_rcp(dy);  // slab tests on padded boxes: an approximate reciprocal suffices
    const F2 id2 = pk(idx, idy), noi2 = pk(-(ox * idx), -(oy * idy));
    float limit = tMax;
    // nearer child first (entry distance), the other pushed with its entry distance and
    // dropped at pop time once a hit closer than it is known; while-while structure
    unsigned long long stack[kStack];
    int sp = 0, ref = start;
    auto pop = [&]() -> bool {
        for (;;) {
            if (sp == 0) return false;
            unsigned long long e = stack[--sp];
            if (__uint_as_float(static_cast<unsigned>(e >> 32)) <= limit) {
                ref = static_cast<int>(static_cast<unsigned>(e));
                return true;
            }
        }
    };
    for (;;) {
        while (ref >= 0) {
            const Node2 nd = S.nodes[ref];
            count_fetch<COUNT>(S, 0);
            float tl = (nd.mask & qmask) ? ray_box_t(nd.lbox, noi2, id2, limit) : kFInf;
            float tr = ((nd.mask >> 3) & qmask) ? ray_box_t(nd.rbox, noi2, id2, limit) : kFInf;
            bool vl = tl != kFInf, vr = tr != kFInf;
            if (vl && vr) {
                bool lf = tl <= tr;
                stack[sp++] = (static_cast<unsigned long long>(__float_as_uint(lf ? tr : tl)) << 32) |
                              static_cast<unsigned>(lf ? nd.right : nd.left);
                ref = lf ? nd.left : nd.right;
            } else if (vl) {
                ref = nd.left;
            } else if (vr) {
                ref = nd.right;
            } else if (!pop()) {
                return h;
            }
        }
        int code = ~ref;
        int start = code >> 3, count = (code & 7) + 1;
        for (int i = start; i < start + count; ++i) {
            const Prim2 p = S.prims[i];
            count_fetch<COUNT>(S, 1);
            if (!((1u << p.label) & qmask) || p.id == skipSeg) continue;
            ray_segment_hit(p.seg, p.id, ox, oy, dx, dy, tMin, limit, h);
        }
        if (!pop()) return h;
    }
}

// the deepest node whose subtree holds every primitive of the classes in qmask whose
// box lies within sqrt(r2) of (x, y): descend while exactly one child qualifies
// (a leaf ref when it narrows to one leaf; kNoEntry when nothing qualifies)
__device__ __forceinline__ int entry_node(const SceneView2& S, float x, float y, float r2, unsigned qmask) {
    int ref = 0;
    while (ref >= 0) {
        const Node2 nd = S.nodes[ref];
        const bool vl = (nd.mask & qmask) && box_dist2(nd.lbox, x, y) <= r2;
        const bool vr = ((nd.mask >> 3) & qmask) && box_dist2(nd.rbox, x, y) <= r2;
        if (vl && vr) return ref;
        if (vl) ref = nd.left;
        else if (vr) ref = nd.right;
        else return kNoEntry;
    }
    return ref;
}

// Up to 4 nodes whose subtrees together hold every primitive of qmask within sqrt(r2) of
// (x, y): entry_node's node, then, while there is room, a frontier node whose two children
// both qualify is replaced by them (single qualifying children are descended into, nodes
// with none dropped). f[0] == kNoEntry: none. (The 2D form of entry_frontier3.)
__device__ __forceinline__ void entry_frontier2(const SceneView2& S, float x, float y, float r2, unsigned qmask,
                                                int (&f)[4]) {
    for (int k = 0; k < 4; ++k) f[k] = kNoEntry;
    f[0] = entry_node(S, x, y, r2, qmask);
    int nf = f[0] == kNoEntry ? 0 : 1;
    for (int guard = 0; guard < 1024; ++guard) {
        bool changed = false;
        for (int i = 0; i < nf; ++i) {
            const int ref = f[i];
            if (ref < 0) continue;  // a leaf
            const Node2 nd = S.nodes[ref];
            const bool vl = (nd.mask & qmask) && box_dist2(nd.lbox, x, y) <= r2;
            const bool vr = ((nd.mask >> 3) & qmask) && box_dist2(nd.rbox, x, y) <= r2;
            if (vl && vr) {
                if (nf < 4) {
                    f[i] = nd.left;
                    f[nf++] = nd.right;
                    changed = true;
                }
            } else if (vl || vr) {
                f[i] = vl ? nd.left : nd.right;
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

// Scene::inside (scene.cpp:240-254): boundary-inclusive within tol, then crossing
// parity along +x with the straddle form; only leaves whose box spans x.y and
// reaches past x.x are visited.
template <bool COUNT = false>
__device__ __forceinline__ bool inside(const SceneView2& S, float x, float y, float tol) {
    Closest c = closest_point<COUNT>(S, x, y, kClsAny, tol * tol);
    if (c.seg >= 0) return true;
    bool in = false;
    int stack[kStack];
    int sp = 0, ref = 0;
    for (;;) {
        if (ref >= 0) {
            const Node2 nd = S.nodes[ref];
            count_fetch<COUNT>(S, 0);
            bool vl = (nd.mask & 7u) && nd.lbox.y <= y && nd.lbox.w >= y && nd.lbox.z > x;
            bool vr = ((nd.mask >> 3) & 7u) && nd.rbox.y <= y && nd.rbox.w >= y && nd.rbox.z > x;
            if (vl && vr) { stack[sp++] = nd.right; ref = nd.left; continue; }
            if (vl) { ref = nd.left; continue; }
            if (vr) { ref = nd.right; continue; }
        } else {
            int code = ~ref;
            int start = code >> 3, count = (code & 7) + 1;
            for (int i = start; i < start + count; ++i) {
                const float4 s = S.prims[i].seg;
                count_fetch<COUNT>(S, 1);
                if ((s.y > y) == (s.w > y)) continue;
                float xc = s.x + (y - s.y) / (s.w - s.y) * (s.z - s.x);
                if (x < xc) in = !in;
            }
        }
        if (sp == 0) return in;
        ref = stack[--sp];
    }
}

}  // namespace bvc_dev
