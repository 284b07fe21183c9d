// walk3.cu — 3D walk-on-spheres / walk-on-stars on triangle meshes (sm_100a).
//
// The reference solver throws for dim != 2 (pointwise.cpp:23); BASELINE configs 4
// and 5 are 3D triangle meshes, so this is the 3D lift of walk.cu with the same
// execution model (warp-refilled lanes, Philox keyed by global task id, fixed
// output slots). The estimator follows walkSampleImpl (pointwise.cpp:125-165):
//   * star radius R = min(dist to Dirichlet, dist to visible Neumann silhouette
//     EDGES), floored at rMin; termination within eps at g(closest point);
//   * directions uniform on S^2, or on the hemisphere about the inward normal
//     after a Neumann hit; Neumann hits by a first-hit ray query within R;
//   * screened weight per step: ballSphereWeight 3D (kernels.cpp:63-65).
// Gradient samples (the 3D gradientSample): v = (3/R) u(z) dir on the first ball,
// plus, for screened kernels, grad G^B(x,R,y) sigma u(y) / pdf(y) with y drawn
// from |G^B| of the 3D Poisson ball (radial CDF F(t) = 3t^2 - 2t^3) and u(y)
// from a nested walk. Source terms (f) are not supported in 3D (the reference's
// sampleBallGreens is 2D-only, kernels.cpp:98-99).
#include <cuda_runtime.h>

#include <cstdlib>

#include "internal.h"
#include "scene3_dev.cuh"

namespace bvc_impl {

using namespace bvc_dev;

namespace {

constexpr int kThreads3 = 256;
constexpr int kChunk3 = 64;

__device__ __forceinline__ float g3(const WalkEnv3& E, const Closest3& c) { return field_eval(E.P.g, c.px, c.py, c.pz); }

// Silhouette edge visible from x (the 3D analogue of scene.cpp:166-172) and closer than
// `bound` (squared); rec = its leaf-order record (a, n1, n2, b) in WalkEnv3::silRec, d2 =
// squared distance. Visibility is tested first (the first endpoint and the two face
// normals), so an edge hidden from x never loads its second endpoint or computes the
// distance; n1.w != 0 marks an open boundary edge (a silhouette from
// everywhere), b.w = 1 / |b - a|^2.
__device__ __forceinline__ bool sil_rec_ok(const float4* rec, float x, float y, float z, float bound, float& d2) {
    const float4 a = rec[0], n1 = rec[1];
    const float ax = a.x - x, ay = a.y - y, az = a.z - z;
    if (n1.w == 0.f) {
        const float4 n2 = rec[2];
        const float s1 = n1.x * ax + n1.y * ay + n1.z * az, s2 = n2.x * ax + n2.y * ay + n2.z * az;
        if (s1 * s2 > 0.0f) return false;
    }
    const float4 b = rec[3];
    const float ux = b.x - a.x, uy = b.y - a.y, uz = b.z - a.z;
    float tt = -(ax * ux + ay * uy + az * uz) * b.w;
    tt = fminf(fmaxf(tt, 0.f), 1.f);
    const float qx = fmaf(tt, ux, ax), qy = fmaf(tt, uy, ay), qz = fmaf(tt, uz, az);
    d2 = qx * qx + qy * qy + qz * qz;
    return d2 < bound;
}

struct Star3 {
    Closest3 D;
    float s2;
};

template <bool COUNT>
__device__ __forceinline__ Star3 star_query3(const WalkEnv3& E, float x, float y, float z, int hint, int hint2,
                                             const int4 starts) {
    Star3 q{hint >= 0 ? closest_on3(E.S, hint, x, y, z) : Closest3{kFInf, 0.f, 0.f, 0.f, -1, -1}, kFInf};
    if (hint2 >= 0 && hint2 != hint) {
        Closest3 h = closest_on3(E.S, hint2, x, y, z);
        if (h.d2 < q.D.d2) q.D = h;
    }
    float eps2 = E.eps * E.eps;
    traverse_near3<COUNT>(
        E.S, x, y, z, kClsD | kClsSil,
        [&](const Prim3& p, int i) {
            if (__float_as_int(p.b.w) == 0) {
                float qx, qy, qz;
                float d2 = tri_closest(p, x, y, z, qx, qy, qz);
                if (d2 < q.D.d2) q.D = Closest3{d2, qx, qy, qz, __float_as_int(p.a.w), i};
            } else {
                const int code = __float_as_int(p.c.w);
                const int cnt = code & 3;
                if (cnt) {
                    // triangle-level pre-test (sil_fill3_kernel): x strictly on one side of
                    // both faces of every edge of this triangle => no silhouette here
                    const float4* blk = E.silRec + (code >> 2);
                    const float4 h = blk[0];
                    const float ax = p.a.x - x, ay = p.a.y - y, az = p.a.z - z;
                    const float st = fmaf(h.x, ax, fmaf(h.y, ay, h.z * az));
                    const float bx = p.b.x - x, by = p.b.y - y, bz = p.b.z - z;
                    const float cx = p.c.x - x, cy = p.c.y - y, cz = p.c.z - z;
                    const float R2 = fmaxf(fmaf(ax, ax, fmaf(ay, ay, az * az)),
                                           fmaxf(fmaf(bx, bx, fmaf(by, by, bz * bz)), fmaf(cx, cx, fmaf(cy, cy, cz * cz))));
                    if (st * st <= h.w * R2) {
                        // a silhouette no closer than the closest Dirichlet point cannot shorten
                        // R = min(dD, dS) (pointwise.cpp:136-138) nor the pruning radius
                        float d2;
                        for (int k = 0; k < cnt; ++k)
                            if (sil_rec_ok(blk + 1 + 4 * k, x, y, z, fminf(q.s2, q.D.d2), d2)) q.s2 = d2;
                    }
                }
            }
        },
        [&]() { return fmaxf(fminf(q.D.d2, q.s2), eps2); }, starts);
    return q;
}

struct Hit3 {
    float t;
    int tri;
};

template <bool COUNT>
__device__ __forceinline__ Hit3 ray_neumann3(const WalkEnv3& E, float ox, float oy, float oz, float dx, float dy,
                                             float dz, float tMax, int skip, int start) {
    Hit3 h{kFInf, -1};
    if (start == kNoEntry) return h;
    float idx = f_rcp(dx), idy = f_rcp(dy), idz = f_rcp(dz);  // slab tests on padded boxes
    const F2 idxy = pk(idx, idy), noixy = pk(-(ox * idx), -(oy * idy));
    const float nozi = -(oz * idz);
    float limit = tMax;
    // nearer child first, the other pushed with its entry distance (dropped at pop once
    // a closer hit is known); while-while structure
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
            const Node3 nd = E.S.nodes[ref];
            count_fetch3<COUNT>(E.S, 0);
            float tl = (nd.mask() & kClsNeumann) ? ray_box3_t(nd.llo, nd.lhi, noixy, nozi, idxy, idz, limit) : kFInf;
            float tr = ((nd.mask() >> 3) & kClsNeumann) ? ray_box3_t(nd.rlo, nd.rhi, noixy, nozi, idxy, idz, limit)
                                                      : kFInf;
            bool vl = tl != kFInf, vr = tr != kFInf;
            if (vl && vr) {
                bool lf = tl <= tr;
                stack[sp++] = (static_cast<unsigned long long>(__float_as_uint(lf ? tr : tl)) << 32) |
                              static_cast<unsigned>(lf ? nd.right() : nd.left());
                ref = lf ? nd.left() : nd.right();
            } else if (vl) {
                ref = nd.left();
            } else if (vr) {
                ref = nd.right();
            } else if (!pop()) {
                return h;
            }
        }
        int code = ~ref;
        int start = code >> 3, count = (code & 7) + 1;
        for (int i = start; i < start + count; ++i) {
            const Prim3 p = E.S.prims[i];
            count_fetch3<COUNT>(E.S, 1);
            int cls = __float_as_int(p.b.w), id = __float_as_int(p.a.w);
            if (!((1u << cls) & kClsNeumann) || id == skip) continue;
            float th;
            if (ray_tri(p, ox, oy, oz, dx, dy, dz, limit, th) && th > E.tguard && th < h.t) {
                h = Hit3{th, id};
                limit = th;
            }
        }
        if (!pop()) return h;
    }
}

// uniform direction on S^2, or on the hemisphere about axis n (unit)
__device__ __forceinline__ void sphere_dir(float u1, float u2, float& dx, float& dy, float& dz) {
    float zc = 1.0f - 2.0f * u1;
    float r = sqrtf(fmaxf(0.f, 1.f - zc * zc));
    float s, c;
    __sincosf(kTwoPi * u2, &s, &c);
    dx = r * c; dy = r * s; dz = zc;
}
__device__ __forceinline__ void hemi_dir(float u1, float u2, float nx, float ny, float nz, float& dx, float& dy,
                                         float& dz) {
    float ct = u1;  // uniform solid angle on the hemisphere: cos(theta) uniform in [0, 1)
    float st = sqrtf(fmaxf(0.f, 1.f - ct * ct));
    float s, c;
    __sincosf(kTwoPi * u2, &s, &c);
    // orthonormal basis about n (Frisvad / Duff et al.)
    float sign = copysignf(1.0f, nz);
    float a = -1.0f / (sign + nz), b = nx * ny * a;
    float t1x = 1.0f + sign * nx * nx * a, t1y = sign * b, t1z = -sign * nx;
    float t2x = b, t2y = sign + ny * ny * a, t2z = -ny;
    dx = st * (c * t1x + s * t2x) + ct * nx;
    dy = st * (c * t1y + s * t2y) + ct * ny;
    dz = st * (c * t1z + s * t2z) + ct * nz;
}

// 3D ballSphereWeight (kernels.cpp:63-65); (tR) / sinh(tR) on the sphere
__device__ __forceinline__ float sphere_weight3(float s, float R, float rHit) {
    float tR = R * s;
    float a = (R - rHit) * s;
    float e = __expf(-tR);
    float shR = 0.5f * (1.0f - e * e);  // sinh(tR) e^{-tR}
    float ea = __expf(a - tR);
    float ch = 0.5f * (ea + __expf(-a - tR)), sh = 0.5f * (ea - __expf(-a - tR));  // cosh(a), sinh(a) times e^{-tR}
    return (rHit * s * ch + sh) / shR;
}

// what a step at x takes from its grid cell (HintCell): one 32-byte record, read as a
// streaming load (one cell per step out of gigabytes: evict-first). Outside the grid, or
// without one: the root for both queries and no warm start.
__device__ __forceinline__ CellHints cell_hints3(const HintGrid& G, float x, float y, float z) {
    CellHints c{kRootStart, 0, -1};
    if (!G.cell) return c;
    const int ix = __float2int_rd((x - G.lox) * G.invH), iy = __float2int_rd((y - G.loy) * G.invH),
              iz = __float2int_rd((z - G.loz) * G.invH);
    if (static_cast<unsigned>(ix) >= static_cast<unsigned>(G.nx) || static_cast<unsigned>(iy) >= static_cast<unsigned>(G.ny) ||
        static_cast<unsigned>(iz) >= static_cast<unsigned>(G.nz))
        return c;
    const int4* rec = reinterpret_cast<const int4*>(G.cell + (static_cast<size_t>(iz) * G.ny + iy) * G.nx + ix);
    c.front = __ldcs(rec);
    const int4 t = __ldcs(rec + 1);
    c.ray = t.x;
    c.id = t.y;
    return c;
}

struct Walk3 {
    float x, y, z, weight;
    float inx, iny, inz;
    int onN, prevTri, step;
    int lastD;  // leaf-order index of the previous closest Dirichlet triangle (warm start)
};

__device__ __forceinline__ void walk3_start(Walk3& w, float x, float y, float z) {
    w.x = x; w.y = y; w.z = z; w.weight = 1.f; w.inx = w.iny = w.inz = 0.f; w.onN = 0; w.prevTri = -1; w.step = 0;
    w.lastD = -1;
}

// far-field lower bound of the distance to the boundary at x, or -1 (FarField)
__device__ __forceinline__ float farfield_bound3(const FarField& F, float x, float y, float z) {
    int ix = __float2int_rn((x - F.lox) * F.invH), iy = __float2int_rn((y - F.loy) * F.invH),
        iz = __float2int_rn((z - F.loz) * F.invH);
    if (ix < 0 || iy < 0 || iz < 0 || ix >= F.nx || iy >= F.ny || iz >= F.nz) return -1.0f;
    float dx = x - fmaf(static_cast<float>(ix), F.h, F.lox), dy = y - fmaf(static_cast<float>(iy), F.h, F.loy),
          dz = z - fmaf(static_cast<float>(iz), F.h, F.loz);
    return __ldg(F.d + (static_cast<size_t>(iz) * F.ny + iy) * F.nx + ix) - sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz))) -
           F.margin;
}

template <bool NEU, bool SCR, bool COUNT>
__device__ __forceinline__ bool walk3_step(const WalkEnv3& E, Walk3& w, U4 rnd, float& value, int& trunc,
                                           unsigned long long& steps) {
    ++steps;
    Closest3 cp;
    float R;
    // far field: a ball from the distance grid, no BVH queries (FarField)
    const float lb = E.ff.d ? farfield_bound3(E.ff, w.x, w.y, w.z) : -1.0f;
    const bool far = lb >= E.ff.tau;
    const CellHints cell = far ? CellHints{kRootStart, 0, -1} : cell_hints3(E.hg, w.x, w.y, w.z);
    if (far) {
        R = lb;
    } else {
        if constexpr (NEU) {
            Star3 q = star_query3<COUNT>(E, w.x, w.y, w.z, w.lastD, cell.id, cell.front);
            cp = q.D;
            float dD = sqrtf(cp.d2);
            if (dD <= E.eps) { value = w.weight * g3(E, cp); return true; }
            R = fminf(dD, sqrtf(q.s2));
        } else {
            cp = closest_point3<COUNT>(E.S, w.x, w.y, w.z, kClsD, kFInf, w.lastD, cell.id, cell.front);
            float dD = sqrtf(cp.d2);
            if (dD <= E.eps) { value = w.weight * g3(E, cp); return true; }
            R = dD;
        }
        w.lastD = cp.prim;
    }
    R = fmaxf(R, E.rmin);
    float dx, dy, dz;
    if (w.onN) hemi_dir(u01(rnd.x), u01(rnd.y), w.inx, w.iny, w.inz, dx, dy, dz);
    else sphere_dir(u01(rnd.x), u01(rnd.y), dx, dy, dz);
    float travel = R;
    bool hit = false;
    if (NEU && !far) {
        Hit3 h = ray_neumann3<COUNT>(E, w.x, w.y, w.z, dx, dy, dz, R, w.onN ? w.prevTri : -1, cell.ray);
        if (h.tri >= 0) {
            hit = true;
            travel = h.t;
            float4 n = E.S.triNormal[h.tri];
            if (E.closed || n.x * dx + n.y * dy + n.z * dz > 0.f) { w.inx = -n.x; w.iny = -n.y; w.inz = -n.z; }
            else { w.inx = n.x; w.iny = n.y; w.inz = n.z; }
            w.x = fmaf(h.t, dx, w.x) + E.nudge * w.inx;
            w.y = fmaf(h.t, dy, w.y) + E.nudge * w.iny;
            w.z = fmaf(h.t, dz, w.z) + E.nudge * w.inz;
            w.onN = 1;
            w.prevTri = h.tri;
        }
    }
    if (!hit) {
        w.x = fmaf(R, dx, w.x);
        w.y = fmaf(R, dy, w.y);
        w.z = fmaf(R, dz, w.z);
        w.onN = 0;
        w.prevTri = -1;
    }
    if constexpr (SCR) w.weight *= sphere_weight3(E.P.sqrtSigma, R, travel);
    bool escaped = fabsf(w.x - E.cx) > E.escape || fabsf(w.y - E.cy) > E.escape || fabsf(w.z - E.cz) > E.escape;
    if (++w.step >= E.maxSteps || escaped) {
        trunc = 1;
        Closest3 c = closest_point3(E.S, w.x, w.y, w.z, kClsD);
        value = w.weight * g3(E, c);
        return true;
    }
    return false;
}

// radial CDF of |G^B| in the 3D Poisson ball: F(t) = 3 t^2 - 2 t^3
__device__ __forceinline__ float invert_ball_cdf3(float u) {
    float t = sqrtf(u / 3.0f) * 1.2f;
    t = fminf(fmaxf(t, 1e-6f), 1.0f);
#pragma unroll 1
    for (int it = 0; it < 30; ++it) {
        float f = t * t * (3.0f - 2.0f * t) - u, d = 6.0f * t * (1.0f - t);
        float nt = d > 0.f ? t - f / d : t;
        nt = fminf(fmaxf(nt, 0.5f * t), fminf(1.0f, 1.5f * t + 1e-6f));
        if (fabsf(nt - t) < 1e-7f) return nt;
        t = nt;
    }
    return t;
}

struct Task3 {
    long long id;
    unsigned long long rid;
    int role, pt, phase;
    uint32_t draw;
    float R, dx, dy, dz, vx, vy, vz, cx, cy, cz, y2x, y2y, y2z;
    int trunc;
};

__device__ __forceinline__ U4 draw3(const WalkEnv3& E, Task3& t) {
    U4 c{static_cast<uint32_t>(t.rid), static_cast<uint32_t>(t.rid >> 32), t.draw++, static_cast<uint32_t>(t.role)};
    return philox4x32_10(c, E.k0, E.k1);
}

// A task's start (a U walk from its point, or a D task's first-ball walk) and what
// follows the end of one of its walks (the U value, the D phase change or its
// gradient): shared by the persistent kernel and the wavefront step kernel, so both
// compute every walk bit for bit alike.
template <bool SCR>
__device__ __forceinline__ void task3_begin(const WalkEnv3& E, const WalkJob3& J, long long nUtot, long long id,
                                            Task3& t, Walk3& w) {
    t.id = id;
    t.draw = 0;
    t.phase = 0;
    t.trunc = 0;
    if (id < nUtot) {
        t.role = 0;
        t.pt = id < 0x7fffffffLL ? static_cast<int>(static_cast<unsigned>(id) / static_cast<unsigned>(J.nU))
                                 : static_cast<int>(id / J.nU);
        int k = static_cast<int>(id - static_cast<long long>(t.pt) * J.nU);
        long long g = J.gidU ? J.gidU[t.pt] : J.gidBaseU + t.pt;
        t.rid = static_cast<unsigned long long>(g) * J.nU + k;
        float4 s = J.startU[t.pt];
        walk3_start(w, s.x, s.y, s.z);
        if (J.hintU) w.lastD = J.hintU[t.pt];
    } else {
        long long d = id - nUtot;
        t.role = 1;
        t.pt = d < 0x7fffffffLL ? static_cast<int>(static_cast<unsigned>(d) / static_cast<unsigned>(J.nD))
                                : static_cast<int>(d / J.nD);
        int k = static_cast<int>(d - static_cast<long long>(t.pt) * J.nD);
        long long g = J.gidD ? J.gidD[t.pt] : t.pt;
        t.rid = static_cast<unsigned long long>(g) * J.nD + k;
        float4 c = J.xD[t.pt];
        t.R = J.radiusD[t.pt];
        U4 r0 = draw3(E, t);
        U4 r1 = draw3(E, t);
        sphere_dir(u01(r0.x), u01(r0.y), t.dx, t.dy, t.dz);
        t.vx = t.vy = t.vz = 0.f;
        if (SCR && E.P.sigma > 0.f) {
            // y ~ |G^B| in the Poisson ball, grad G^B (kernels.cpp:68-75, 3D) sigma / pdf
            float tt = invert_ball_cdf3(u01(r0.z));
            float r = fmaxf(tt * t.R, 1e-6f * t.R);
            float ex, ey, ez;
            sphere_dir(u01(r0.w), u01(r1.x), ex, ey, ez);
            float gb = (1.0f / t.R - 1.0f / r) * kInv4Pi;            // G^B 3D
            float pdf = gb / (-t.R * t.R / 6.0f);                     // / mass
            float gf = (1.0f / (t.R * t.R * t.R) - 1.0f / (r * r * r)) * kInv4Pi * (E.P.sigma / pdf);
            t.cx = r * ex * gf; t.cy = r * ey * gf; t.cz = r * ez * gf;
            t.y2x = c.x + r * ex; t.y2y = c.y + r * ey; t.y2z = c.z + r * ez;
        }
        float rr = t.R * 0.99999952f;
        walk3_start(w, fmaf(rr, t.dx, c.x), fmaf(rr, t.dy, c.y), fmaf(rr, t.dz, c.z));
        if (J.hintD) w.lastD = J.hintD[t.pt];
    }
}

// returns whether the task continues (a screened D task's nested walk)
template <bool SCR>
__device__ __forceinline__ bool task3_walk_done(const WalkEnv3& E, const WalkJob3& J, long long nUtot, Task3& t,
                                                Walk3& w, float value) {
    bool active = true;
    if (t.role == 0) {
        J.outU[t.id] = value;
        if (t.trunc && J.truncU) atomicAdd(J.truncU + t.pt, 1);
        if (t.trunc && J.truncTotal) atomicAdd(J.truncTotal, 1ull);
        active = false;
    } else if (t.phase == 0) {
        float s = (3.0f / t.R) * value;
        t.vx = fmaf(s, t.dx, t.vx);
        t.vy = fmaf(s, t.dy, t.vy);
        t.vz = fmaf(s, t.dz, t.vz);
        if (SCR && E.P.sigma > 0.f) {
            t.phase = 1;
            walk3_start(w, t.y2x, t.y2y, t.y2z);
            if (J.hintD) w.lastD = J.hintD[t.pt];
        } else {
            active = false;
        }
    } else {
        t.vx = fmaf(t.cx, value, t.vx);
        t.vy = fmaf(t.cy, value, t.vy);
        t.vz = fmaf(t.cz, value, t.vz);
        active = false;
    }
    if (!active && t.role == 1) {
        long long slot = t.id - nUtot;
        if (J.normalD) {
            float4 n = J.normalD[t.pt];
            J.outD[slot] = n.x * t.vx + n.y * t.vy + n.z * t.vz;
        } else {
            J.outD[3 * slot] = t.vx;
            J.outD[3 * slot + 1] = t.vy;
            J.outD[3 * slot + 2] = t.vz;
        }
        if (t.trunc && J.truncD) atomicAdd(J.truncD + t.pt, 1);
        if (t.trunc && J.truncTotal) atomicAdd(J.truncTotal, 1ull);
    }
    return active;
}

// resident blocks per SM: Neumann scenes 8 (32 registers, spilling; C5: 3.54 s at 8, 3.60 s
// at 6), Dirichlet-only 6 (40 registers; C4 walks 435 ms at 6, 469 at 5, 521 at 4, 477 at 8)
template <bool NEU, bool SCR, bool COUNT, int MINB = NEU ? 8 : 6>
__global__ void __launch_bounds__(kThreads3, MINB) walk3_kernel(const WalkEnv3 E, const WalkJob3 J) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const long long nUtot = static_cast<long long>(J.nPtsU) * J.nU;
    const long long total = nUtot + static_cast<long long>(J.nPtsDdev ? *J.nPtsDdev : J.nPtsD) * J.nD;
    long long qNext = 0, qEnd = 0;
    bool exhausted = false, active = false;
    Task3 t;
    Walk3 w;
    unsigned long long steps = 0;
    for (;;) {
        unsigned need = __ballot_sync(0xffffffffu, !active);
        while (need && !exhausted) {
            if (qNext >= qEnd) {
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(J.counter, static_cast<unsigned long long>(kChunk3));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (static_cast<long long>(base) >= total) { exhausted = true; break; }
                qNext = static_cast<long long>(base);
                qEnd = min(qNext + kChunk3, total);
            }
            int take = static_cast<int>(min(static_cast<long long>(__popc(need)), qEnd - qNext));
            int rank = __popc(need & lt);
            if (((need >> lane) & 1u) && rank < take) {
                task3_begin<SCR>(E, J, nUtot, qNext + rank, t, w);
                active = true;
            }
            qNext += take;
            need = __ballot_sync(0xffffffffu, !active);
        }
        if (__ballot_sync(0xffffffffu, active) == 0u) break;
        if (active) {
            U4 rnd = draw3(E, t);
            float value;
            if (walk3_step<NEU, SCR, COUNT>(E, w, rnd, value, t.trunc, steps))
                active = task3_walk_done<SCR>(E, J, nUtot, t, w, value);
        }
    }
    if (J.steps) {
        for (int o = 16; o > 0; o >>= 1) steps += __shfl_xor_sync(0xffffffffu, steps, o);
        if (lane == 0) atomicAdd(J.steps, steps);
    }
}

// area-uniform boundary samples (the 3D BoundarySampler): the stratified CDF
// coordinate picks the triangle, its in-triangle remainder and a second
// uniform give uniform barycentrics
__global__ void sample_mesh_kernel(const double* cdf, int m, double total, const float4* triA, const float4* triB,
                                   const float4* triC, const float4* triN, int count, int begin, int n,
                                   const long long* ctr, int stratified, uint32_t k0, uint32_t k1, CacheSample* out) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    long long k = ctr ? ctr[j] : static_cast<long long>(begin) + j;
    U4 r = philox4x32_10(U4{static_cast<uint32_t>(k), static_cast<uint32_t>(k >> 32), 0u, 0u}, k0, k1);
    double U = (static_cast<double>(r.x >> 5) * 67108864.0 + static_cast<double>(r.y >> 6)) * (1.0 / 9007199254740992.0);
    double u = stratified ? (static_cast<double>(k) + U) / count : U;
    double target = u * total;
    int lo = 0, hi = m;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (cdf[mid] < target) lo = mid + 1; else hi = mid;
    }
    int id = lo >= m ? m - 1 : lo;
    double prev = id > 0 ? cdf[id - 1] : 0.0;
    double f = fmin(fmax((target - prev) / (cdf[id] - prev), 0.0), 1.0);
    float r1 = sqrtf(static_cast<float>(f)), r2 = u01(r.z);
    float wa = 1.f - r1, wb = r1 * (1.f - r2), wc = r1 * r2;
    float4 a = triA[id], b = triB[id], c = triC[id], nn = triN[id];
    CacheSample o;
    o.z[0] = wa * a.x + wb * b.x + wc * c.x;
    o.z[1] = wa * a.y + wb * b.y + wc * c.y;
    o.z[2] = wa * a.z + wb * b.z + wc * c.z;
    o.n[0] = nn.x; o.n[1] = nn.y; o.n[2] = nn.z;
    o.pdf = static_cast<float>(1.0 / total);
    o.uHat = 0.f; o.dHat = 0.f; o.weight = 0.f; o.arc = 0.f;
    o.segment = id;
    out[j] = o;
}

__global__ void prepare3_kernel(const WalkEnv3 E, CacheSample* samples, int n, const int* kinds, float4* startU,
                                int* isD, float* gradR, uint8_t* outside) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    CacheSample s = samples[i];
    float x = s.z[0], y = s.z[1], z = s.z[2];
    if (kinds[s.segment] == 0) {  // known Neumann: half a shell inside, d = h(z)
        x -= 0.5f * E.eps * s.n[0];
        y -= 0.5f * E.eps * s.n[1];
        z -= 0.5f * E.eps * s.n[2];
        samples[i].dHat = E.hasH ? field_eval(E.P.h, s.z[0], s.z[1], s.z[2]) : 0.f;
        isD[i] = 0;
        gradR[i] = 0.f;
    } else {
        isD[i] = 1;
        Closest3 c = closest_point3(E.S, x, y, z, kClsAny);
        gradR[i] = fmaxf(sqrtf(c.d2), E.rmin);
    }
    startU[i] = make_float4(x, y, z, 0.f);
    outside[i] = (E.insideTol < 0.f || inside3(E.S, x, y, z, E.insideTol)) ? 0 : 1;
}

__global__ void gather_dpoints3_kernel(const CacheSample* samples, const int* dIdx, int nD, const float* gradR,
                                       long long gidBase, const long long* gid, float4* xD, float4* nD_, float* rD,
                                       long long* gidD, const int* nDdev) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= (nDdev ? *nDdev : nD)) return;
    int i = dIdx[j];
    CacheSample s = samples[i];
    xD[j] = make_float4(s.z[0], s.z[1], s.z[2], 0.f);
    nD_[j] = make_float4(s.n[0], s.n[1], s.n[2], 0.f);
    rD[j] = gradR[i];
    gidD[j] = gid ? gid[i] : gidBase + i;
}

__global__ void closest3_kernel(const SceneView3 S, const double* x, int n, unsigned mask, double* point, double* dist,
                                int* tri) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Closest3 c = closest_point3(S, static_cast<float>(x[3 * i]), static_cast<float>(x[3 * i + 1]),
                                static_cast<float>(x[3 * i + 2]), mask);
    point[3 * i] = c.px; point[3 * i + 1] = c.py; point[3 * i + 2] = c.pz;
    dist[i] = c.tri >= 0 ? sqrt(static_cast<double>(c.d2)) : INFINITY;
    tri[i] = c.tri;
}

__global__ void inside3_kernel(const SceneView3 S, const double* x, int n, float tol, uint8_t* out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = inside3(S, static_cast<float>(x[3 * i]), static_cast<float>(x[3 * i + 1]), static_cast<float>(x[3 * i + 2]),
                     tol) ? 1 : 0;
}

// fallback band in 3D: within l of the Dirichlet boundary (cache.cpp:131-135) or, for a
// closed region mesh, outside it — the vertex-normal offset surface is not exactly at
// distance l, and a point outside the region would get the exterior value of the BIE
__global__ void mark3_kernel(const SceneView3 scene, const SceneView3 region, const double* x, int n, float offset,
                             int whole, float insideTol, uint8_t* fb, uint8_t* gu) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float px = static_cast<float>(x[3 * i]), py = static_cast<float>(x[3 * i + 1]), pz = static_cast<float>(x[3 * i + 2]);
    const float l2 = offset * offset;  // bounded queries: only "closer than l" matters
    uint8_t f = 0;
    if (whole) {
        Closest3 c = closest_point3(scene, px, py, pz, kClsD, l2);
        f = c.tri >= 0 ? 1 : 0;
        if (!f && insideTol > 0.f && !inside3(region, px, py, pz, insideTol)) f = 1;
    }
    Closest3 r = closest_point3(region, px, py, pz, kClsAny, l2);
    fb[i] = f;
    gu[i] = r.tri >= 0 ? 1 : 0;
}

inline int blocks(long long n, int t) { return static_cast<int>((n + t - 1) / t); }

}  // namespace

__global__ void farfield3_kernel(const SceneView3 S, const FarField F, float* d) {
    long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<long long>(F.nx) * F.ny * F.nz) return;
    int ix = static_cast<int>(i % F.nx), iy = static_cast<int>((i / F.nx) % F.ny), iz = static_cast<int>(i / (static_cast<long long>(F.nx) * F.ny));
    float x = fmaf(static_cast<float>(ix), F.h, F.lox), y = fmaf(static_cast<float>(iy), F.h, F.loy),
          z = fmaf(static_cast<float>(iz), F.h, F.loz);
    d[i] = sqrtf(closest_point3(S, x, y, z, kClsAny).d2);
}

template <bool NEU, bool SCR, bool COUNT>
void launch_walk3_t(const WalkEnv3& env, const WalkJob3& job, long long total, cudaStream_t st) {
    int dev = 0, sms = 148, perSm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&perSm, walk3_kernel<NEU, SCR, COUNT>, kThreads3, 0);
    perSm = perSm > 0 ? perSm : 1;
    if (const char* e = std::getenv("BVC_WALK_OCC")) {  // co-residency experiments: blocks per SM cap
        int v = std::atoi(e);
        if (v >= 1 && v < perSm) perSm = v;
    }
    long long want = (total + kThreads3 - 1) / kThreads3;
    int grid = static_cast<int>(want < static_cast<long long>(sms) * perSm ? want : static_cast<long long>(sms) * perSm);
    if (const char* e = std::getenv("BVC_WALK_CARVEOUT"))  // co-residency experiments: shared-memory carve-out, percent
        cudaFuncSetAttribute(walk3_kernel<NEU, SCR, COUNT>, cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(e));
    walk3_kernel<NEU, SCR, COUNT><<<grid, kThreads3, 0, st>>>(env, job);
}

__global__ void hintgrid3_kernel(const SceneView3 S, const HintGrid G, HintCell* cells, int entries, int fronts,
                                 float rmin) {
    long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<long long>(G.nx) * G.ny * G.nz) return;
    int ix = static_cast<int>(i % G.nx), iy = static_cast<int>((i / G.nx) % G.ny), iz = static_cast<int>(i / (static_cast<long long>(G.nx) * G.ny));
    // cell [v, v + h)^3: centre c, half-diagonal rho; r = dD(c) + 2 rho plus FP32 slack
    const float cx = fmaf(static_cast<float>(ix) + 0.5f, G.h, G.lox), cy = fmaf(static_cast<float>(iy) + 0.5f, G.h, G.loy),
                cz = fmaf(static_cast<float>(iz) + 0.5f, G.h, G.loz), rho = 0.8660254f * G.h;
    const Closest3 c = closest_point3(S, cx, cy, cz, kClsD);
    HintCell out;
    out.id = c.prim;  // at x in the cell its distance is at most d(x) + 2 |x - c|
    out.pad0 = out.pad1 = 0;
    out.front = kRootStart;
    out.ray = 0;
    if (entries) {
        const float r = sqrtf(c.d2) + 2.0f * rho + 1e-5f * S.diagonal;
        const float rr = r + rmin;
        out.ray = entry_node3(S, cx, cy, cz, rr * rr, kClsNeumann);
        int f[4] = {kNoEntry, kNoEntry, kNoEntry, kNoEntry};
        if (fronts) entry_frontier3(S, cx, cy, cz, r * r, kClsD | kClsSil, f);
        else f[0] = entry_node3(S, cx, cy, cz, r * r, kClsD | kClsSil);
        if (f[0] == kNoEntry) f[0] = 0;  // cannot happen for a star query (the closest Dirichlet primitive qualifies)
        out.front = make_int4(f[0], f[1], f[2], f[3]);
    }
    cells[i] = out;
}

void launch_hintgrid3(const SceneView3& S, const HintGrid& G, HintCell* cells, bool entries, bool fronts, float rmin,
                      cudaStream_t st) {
    hintgrid3_kernel<<<blocks(static_cast<long long>(G.nx) * G.ny * G.nz, 128), 128, 0, st>>>(S, G, cells, entries ? 1 : 0,
                                                                                            fronts ? 1 : 0, rmin);
    count_launch();
}

// per triangle: the float4 count of its record block (a header plus 4 per edge), or 0
__global__ void sil_count3_kernel(const Prim3* prims, int n, const int4* triSil, int* counts) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const int4 sl = triSil[__float_as_int(prims[j].a.w)];
    const int k = (sl.x >= 0) + (sl.y >= 0) + (sl.z >= 0);
    counts[j] = k ? 1 + 4 * k : 0;
}
// A triangle's block: header (n_t, delta'^2), then its edges' records (a, n1, n2, b).
// The header is the triangle-level visibility pre-test of star_query3: every edge of
// the triangle has the triangle's plane through it, so s_t = n_t.(a - x) is the same for
// all of them, and the other face's s_o = n_o.(a_e - x) differs from s_t by at most
// |n_o - n_t| |a_e - x| <= delta R (R = the farthest vertex from x). |s_t| > delta' R
// therefore proves every edge of the triangle invisible from x (s_t s_o > 0) without
// reading its records. delta' = delta (1 + 1e-5) + 4e-6 covers the FP32 rounding of
// both tests (|s| errors ~4e-7 R), so the pre-test never rejects an edge that
// sil_rec_ok would accept; an open (always-silhouette) edge makes delta' infinite.
__global__ void sil_fill3_kernel(Prim3* prims, int n, const int4* triSil, const int* counts, const int* offsets,
                                 const float4* silA, const float4* silN1, const float4* silN2, const float4* silB,
                                 const float4* triN, float4* rec) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const int id = __float_as_int(prims[j].a.w);
    const int4 sl = triSil[id];
    const int e[3] = {sl.x, sl.y, sl.z};
    const int off = offsets[j];
    int k = 0;
    float delta = 0.f;
    bool always = false;
    for (int r = 0; r < 3; ++r) {
        if (e[r] < 0) continue;
        float4* o = rec + off + 1 + 4 * static_cast<size_t>(k++);
        const float4 n1 = silN1[e[r]], n2 = silN2[e[r]];
        o[0] = silA[e[r]];
        o[1] = n1;
        o[2] = n2;
        o[3] = silB[e[r]];
        always |= n1.w != 0.f;
        const float dx = n1.x - n2.x, dy = n1.y - n2.y, dz = n1.z - n2.z;
        delta = fmaxf(delta, sqrtf(dx * dx + dy * dy + dz * dz));
    }
    if (k) {
        const float4 nt = triN[id];
        const float dp = fmaf(delta, 1.00001f, 4e-6f);
        rec[off] = make_float4(nt.x, nt.y, nt.z, always ? kFInf : dp * dp);
    }
    prims[j].c.w = __int_as_float((off << 2) | k);
}

void launch_sil_count3(const Prim3* prims, int n, const int4* triSil, int* counts, cudaStream_t st) {
    if (n <= 0) return;
    sil_count3_kernel<<<blocks(n, 256), 256, 0, st>>>(prims, n, triSil, counts);
    count_launch();
}

void launch_sil_fill3(Prim3* prims, int n, const int4* triSil, const int* counts, const int* offsets,
                      const float4* silA, const float4* silN1, const float4* silN2, const float4* silB,
                      const float4* triN, float4* rec, cudaStream_t st) {
    if (n <= 0) return;
    sil_fill3_kernel<<<blocks(n, 256), 256, 0, st>>>(prims, n, triSil, counts, offsets, silA, silN1, silN2, silB, triN,
                                                      rec);
    count_launch();
}

void launch_farfield3(const SceneView3& S, const FarField& F, float* d, cudaStream_t st) {
    long long n = static_cast<long long>(F.nx) * F.ny * F.nz;
    farfield3_kernel<<<blocks(n, 128), 128, 0, st>>>(S, F, d);
    count_launch();
}

void launch_walk_job3(const WalkEnv3& env, const WalkJob3& job, cudaStream_t st) {
    long long total = static_cast<long long>(job.nPtsU) * job.nU + static_cast<long long>(job.nPtsD) * job.nD;
    if (total <= 0) return;
    cudaMemsetAsync(job.counter, 0, sizeof(unsigned long long), st);
    const int code = (env.hasNeumann ? 1 : 0) | (env.P.screened ? 2 : 0) | (env.S.counts ? 4 : 0);
    switch (code) {
        case 0: launch_walk3_t<false, false, false>(env, job, total, st); break;
        case 1: launch_walk3_t<true, false, false>(env, job, total, st); break;
        case 2: launch_walk3_t<false, true, false>(env, job, total, st); break;
        case 3: launch_walk3_t<true, true, false>(env, job, total, st); break;
        case 4: launch_walk3_t<false, false, true>(env, job, total, st); break;
        case 5: launch_walk3_t<true, false, true>(env, job, total, st); break;
        case 6: launch_walk3_t<false, true, true>(env, job, total, st); break;
        default: launch_walk3_t<true, true, true>(env, job, total, st); break;
    }
    count_launch();
}

void launch_sample_mesh(const double* cdf, int m, double total, const float4* triA, const float4* triB,
                        const float4* triC, const float4* triN, int count, int begin, int n, const long long* ctr,
                        int stratified, uint32_t k0, uint32_t k1, CacheSample* out, cudaStream_t st) {
    if (n <= 0) return;
    sample_mesh_kernel<<<blocks(n, 256), 256, 0, st>>>(cdf, m, total, triA, triB, triC, triN, count, begin, n, ctr,
                                                      stratified, k0, k1, out);
    count_launch();
}

void launch_prepare3(const WalkEnv3& env, CacheSample* samples, int n, const int* kinds, float4* startU, int* isD,
                     float* gradR, uint8_t* outside, cudaStream_t st) {
    if (n <= 0) return;
    prepare3_kernel<<<blocks(n, 128), 128, 0, st>>>(env, samples, n, kinds, startU, isD, gradR, outside);
    count_launch();
}

void launch_gather_dpoints3(const CacheSample* samples, const int* dIdx, int nD, const float* gradR, long long gidBase,
                            const long long* gid, float4* xD, float4* nD_, float* rD, long long* gidD, cudaStream_t st,
                            const int* nDdev) {
    if (nD <= 0) return;
    gather_dpoints3_kernel<<<blocks(nD, 256), 256, 0, st>>>(samples, dIdx, nD, gradR, gidBase, gid, xD, nD_, rD, gidD,
                                                             nDdev);
    count_launch();
}

void launch_closest3(const SceneView3& S, const double* x, int n, unsigned mask, double* point, double* dist, int* tri,
                     cudaStream_t st) {
    if (n <= 0) return;
    closest3_kernel<<<blocks(n, 128), 128, 0, st>>>(S, x, n, mask, point, dist, tri);
    count_launch();
}

void launch_inside3(const SceneView3& S, const double* x, int n, float tol, uint8_t* out, cudaStream_t st) {
    if (n <= 0) return;
    inside3_kernel<<<blocks(n, 128), 128, 0, st>>>(S, x, n, tol, out);
    count_launch();
}

void launch_mark3(const SceneView3& scene, const SceneView3& region, const double* x, int n, float offset, int whole,
                  float insideTol, uint8_t* fb, uint8_t* gu, cudaStream_t st) {
    if (n <= 0) return;
    mark3_kernel<<<blocks(n, 128), 128, 0, st>>>(scene, region, x, n, offset, whole, insideTol, fb, gu);
    count_launch();
}

}  // namespace bvc_impl
