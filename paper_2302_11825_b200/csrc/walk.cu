// walk.cu — cache-construction walks (WoS / WoSt) and their helpers on sm_100a.
//
// Reference: walkSampleImpl pointwise.cpp:125-165, runWalks 167-186,
// gradientSample 195-215, sourceTerm 110-121, neumannTerm 52-107,
// generateBoundaryCache cache.cpp:301-390.
//
// Execution model: one lane = one walk. Each warp owns a small queue of task ids
// (refilled 64 at a time from one global counter) and hands a new task to every
// lane whose walk terminated, so all 32 lanes keep stepping until the queue
// drains (heavy-tailed walk lengths would otherwise idle most of a warp). Task
// outputs are written to fixed slots and reduced in a fixed order afterwards,
// so results are independent of scheduling, launch geometry and GPU count.
#include <cuda_runtime.h>

#include <cstdlib>

#include "internal.h"

namespace bvc_impl {

using namespace bvc_dev;

namespace {

constexpr int kWalkThreads = 256;
constexpr int kChunk = 64;

// --- ball kernels (kernels.cpp:31-107), 2D ---------------------------------
__device__ __forceinline__ float ball_greens_poisson(float R, float r) { return f_ln(r / R) * kInv2Pi; }

// screened G^B (kernels.cpp:36-40) with exponentially scaled Bessel functions
__device__ __forceinline__ float ball_greens_screened(float s, float R, float r) {
    float tR = R * s, tr = r * s;
    float ratioTerm = bessel_i0e(tr) * bessel_k0e(tR) / bessel_i0e(tR) * f_exp(tr - 2.0f * tR);
    return -(bessel_k0(tr) - ratioTerm) * kInv2Pi;
}

// WoSt recursion weight (ballSphereWeight kernels.cpp:55-66); 1/I0(tR) on the sphere
__device__ __forceinline__ float ball_sphere_weight(float s, float R, float rHit) {
    float tR = R * s, tr = rHit * s;
    if (rHit >= R) return f_exp(-tR) / bessel_i0e(tR);
    float k1 = tr <= 2.0f ? bessel_tk1_small(tr) : tr * bessel_k1(tr);
    return k1 + tr * bessel_i1e(tr) * bessel_k0e(tR) / bessel_i0e(tR) * f_exp(tr - 2.0f * tR);
}

// inverse of the radial CDF F(t) = t^2 (1 - 2 ln t) (kernels.cpp:78-94)
__device__ __forceinline__ float invert_ball_cdf(float u) {
    if (u <= 0.0f) return 1e-8f;
    if (u >= 1.0f) return 1.0f;
    // start near the root: F ~ 1 - 2 (1 - t)^2 at t -> 1 (double root of F - 1),
    // sqrt(u) elsewhere; safeguarded Newton with the SFU log
    float lo = 0.0f, hi = 1.0f, t = u > 0.9f ? 1.0f - sqrtf(0.5f * (1.0f - u)) : sqrtf(u);
#pragma unroll 1
    for (int it = 0; it < 16; ++it) {
        float lt = f_ln(t);
        float fv = t * t * (1.0f - 2.0f * lt) - u;
        if (fv > 0.0f) hi = t; else lo = t;
        float der = -4.0f * t * lt;
        float nxt = der != 0.0f ? t - __fdividef(fv, der) : 0.5f * (lo + hi);
        if (!(nxt > lo && nxt < hi)) nxt = 0.5f * (lo + hi);
        if (fabsf(nxt - t) < 2e-7f) return nxt;
        t = nxt;
    }
    return t;
}

struct BallSample {
    float x, y, r, pdf;
};
// sampleBallGreens kernels.cpp:96-107 (2D Poisson ball around c)
__device__ __forceinline__ BallSample sample_ball(float cx, float cy, float R, float u1, float u2) {
    float t = invert_ball_cdf(u1);
    float r = fmaxf(t * R, 1e-14f * R);
    float sn, cs;
    __sincosf(kTwoPi * u2, &sn, &cs);
    BallSample b;
    b.x = cx + r * cs;
    b.y = cy + r * sn;
    b.r = r;
    b.pdf = ball_greens_poisson(R, r) / (-0.25f * R * R);
    return b;
}

__device__ __forceinline__ float g_value(const WalkEnv& E, const Closest& c) {
    return field_eval(E.P.g, c.px, c.py);
}

// sourceTerm pointwise.cpp:110-121
__device__ float source_term(const WalkEnv& E, float x, float y, float R, float u1, float u2) {
    BallSample b = sample_ball(x, y, R, u1, u2);
    float fy = field_eval(E.P.f, b.x, b.y);
    if (fy == 0.0f) return 0.0f;
    if (E.hasNeumann && !inside(E.S, b.x, b.y, E.insideTol)) return 0.0f;
    float contrib = fy * (-0.25f * R * R);
    if (E.P.screened) {
        float r = fminf(fmaxf(b.r, 1e-13f * E.scale), R);
        contrib *= ball_greens_screened(E.P.sqrtSigma, R, r) / ball_greens_poisson(R, r);
    }
    return contrib;
}

// neumannTerm / clipNeumann pointwise.cpp:52-107: Neumann boundary clipped to the
// ball, one point drawn by length. Two passes over the Neumann leaves near x.
__device__ float neumann_term(const WalkEnv& E, float x, float y, float R, float u) {
    const SceneView2& S = E.S;
    float total = 0.0f;
    auto clip = [&](const Prim2& p, float& t0, float& t1) -> bool {
        float ux = p.seg.z - p.seg.x, uy = p.seg.w - p.seg.y, qx = p.seg.x - x, qy = p.seg.y - y;
        float A = ux * ux + uy * uy, B = 2.0f * (qx * ux + qy * uy), C = qx * qx + qy * qy - R * R;
        float disc = B * B - 4.0f * A * C;
        if (!(disc > 0.0f) || A <= 0.0f) return false;
        float sq = sqrtf(disc);
        t0 = fmaxf(0.0f, (-B - sq) / (2.0f * A));
        t1 = fminf(1.0f, (-B + sq) / (2.0f * A));
        return t1 > t0;
    };
    float R2 = R * R;
    traverse_near(
        S, x, y, kClsNeumann,
        [&](const Prim2& p) {
            float t0, t1;
            if (clip(p, t0, t1)) {
                float ux = p.seg.z - p.seg.x, uy = p.seg.w - p.seg.y;
                total += (t1 - t0) * sqrtf(ux * ux + uy * uy);
            }
        },
        [&]() { return R2; });
    if (total <= 0.0f) return 0.0f;
    float target = u * total, run = 0.0f;
    float bx = x, by = y;
    bool done = false;
    traverse_near(
        S, x, y, kClsNeumann,
        [&](const Prim2& p) {
            if (done) return;
            float t0, t1;
            if (!clip(p, t0, t1)) return;
            float ux = p.seg.z - p.seg.x, uy = p.seg.w - p.seg.y;
            float len = (t1 - t0) * sqrtf(ux * ux + uy * uy);
            float local = fminf(fmaxf((target - run) / len, 0.0f), 1.0f);
            float t = t0 + (t1 - t0) * local;
            bx = p.seg.x + t * ux;
            by = p.seg.y + t * uy;
            if (target <= run + len) done = true;
            run += len;
        },
        [&]() { return R2; });
    float dx = bx - x, dy = by - y;
    float r = fminf(fmaxf(sqrtf(dx * dx + dy * dy), 1e-12f * E.scale), R);
    float hv = field_eval(E.P.h, bx, by);
    float gb = E.P.screened ? ball_greens_screened(E.P.sqrtSigma, R, r) : ball_greens_poisson(R, r);
    return -gb * hv * total;
}

// far-field lower bound of the distance to the boundary at (x, y), or -1 (FarField)
__device__ __forceinline__ float farfield_bound(const FarField& F, float x, float y) {
    float gx = (x - F.lox) * F.invH, gy = (y - F.loy) * F.invH;
    int ix = __float2int_rn(gx), iy = __float2int_rn(gy);
    if (ix < 0 || iy < 0 || ix >= F.nx || iy >= F.ny) return -1.0f;
    float dx = x - fmaf(static_cast<float>(ix), F.h, F.lox), dy = y - fmaf(static_cast<float>(iy), F.h, F.loy);
    return __ldg(F.d + static_cast<size_t>(iy) * F.nx + ix) - sqrtf(fmaf(dx, dx, dy * dy)) - F.margin;
}

// what a step at (x, y) takes from its grid cell (HintCell): one 32-byte record, read as a
// streaming load. Outside the grid, or without one: the root for both queries and no warm start.
__device__ __forceinline__ CellHints cell_hints(const HintGrid& G, float x, float y) {
    CellHints c{kRootStart, 0, -1};
    if (!G.cell) return c;
    const int ix = __float2int_rd((x - G.lox) * G.invH), iy = __float2int_rd((y - G.loy) * G.invH);
    if (static_cast<unsigned>(ix) >= static_cast<unsigned>(G.nx) || static_cast<unsigned>(iy) >= static_cast<unsigned>(G.ny))
        return c;
    const int4* rec = reinterpret_cast<const int4*>(G.cell + static_cast<size_t>(iy) * G.nx + ix);
    c.front = __ldcs(rec);
    const int4 t = __ldcs(rec + 1);
    c.ray = t.x;
    c.id = t.y;
    return c;
}

// per-lane walk state
struct Walk {
    float x, y, acc, weight, inx, iny;
    int onN, prevSeg, step;
    int lastD;  // previous step's closest Dirichlet segment: the next query's warm start
};

__device__ __forceinline__ void walk_start(Walk& w, float x, float y) {
    w.x = x; w.y = y; w.acc = 0.0f; w.weight = 1.0f; w.inx = 0.0f; w.iny = 0.0f;
    w.onN = 0; w.prevSeg = -1; w.step = 0; w.lastD = -1;
}

// star query against the straight Dirichlet runs and the silhouette candidates
// (WalkEnv::drunSeg): the closest Dirichlet point of the runs (the closest point of a
// straight wall is that of its subdivisions) and the closest visible silhouette nearer
// than it (pointwise.cpp:136-138), as star_query returns them
__device__ __forceinline__ StarQuery star_runs(const WalkEnv& E, float x, float y, bool sil) {
    StarQuery q;
    q.D = Closest{kFInf, 0.0f, 0.0f, 0.0f, -1};
    q.s2 = kFInf;
    for (int i = 0; i < E.drunN; ++i) {
        float px, py, t;
        const float d2 = seg_closest(__ldg(E.drunSeg + i), x, y, px, py, t);
        if (d2 < q.D.d2) q.D = Closest{d2, px, py, t, __ldg(E.drunId + i)};
    }
    if (sil) {
        for (int k = 0; k < E.nSil; ++k) {
            float d2;
            if (silhouette_ok(E.S, k, x, y, d2) && d2 < fminf(q.s2, q.D.d2)) q.s2 = d2;
        }
    }
    return q;
}

// Neumann ray against the straight Neumann runs (WalkEnv::runSeg): the first hit within
// (tguard, R], the same point as on the run's own segments; no run is reachable from a
// cell without a ray entry node (HintGrid)
__device__ __forceinline__ RayHit ray_runs(const WalkEnv& E, float ox, float oy, float dx, float dy, float tMax,
                                           int skip, int entry) {
    RayHit h{kFInf, 0.0f, 0.0f, 0.0f, -1};
    if (entry == kNoEntry) return h;
    float limit = tMax;
    for (int i = 0; i < E.runN; ++i) {
        const int id = __ldg(E.runId + i);
        if (id != skip) ray_segment_hit(__ldg(E.runSeg + i), id, ox, oy, dx, dy, E.tguard, limit, h);
    }
    return h;
}

// One iteration of walkSampleImpl's loop (pointwise.cpp:130-161). Returns true
// when the walk terminated; then *value holds its estimate. The scene traits
// (Neumann boundary, screening, source) and the traffic counters are
// compile-time, so each configuration runs only its own code.
template <bool NEU, bool SCR, bool SRC, bool COUNT>
__device__ __forceinline__ bool walk_step(const WalkEnv& E, Walk& w, U4 rnd, float& value, int& trunc,
                                          unsigned long long& steps) {
    Closest cp;
    float R;
    ++steps;
    // far field: a ball from the distance grid, no BVH query (FarField); such a ball
    // holds no boundary point, so no Neumann crossing and no Neumann-data term either
    const float lb = E.ff.d ? farfield_bound(E.ff, w.x, w.y) : -1.0f;
    const bool far = lb >= E.ff.tau;
    const CellHints cell = (far || E.drunN) ? CellHints{kRootStart, 0, -1} : cell_hints(E.hg, w.x, w.y);
    if (far) {
        R = lb;
    } else if (E.drunN) {  // straight-run scene: no BVH (bvc_scene_s::build_runs)
        StarQuery q = star_runs(E, w.x, w.y, NEU);
        cp = q.D;
        float dD = sqrtf(cp.d2);
        if (dD <= E.eps) { value = w.acc + w.weight * g_value(E, cp); return true; }
        R = NEU ? fminf(dD, sqrtf(q.s2)) : dD;
        w.lastD = cp.seg;
    } else {
        // (scenes without Dirichlet segments are rejected on the host, pointwise.cpp:217-218)
        if constexpr (NEU) {
            // a Dirichlet segment farther than the closest visible silhouette may be
            // pruned (q.D.seg < 0, d2 = inf): R is then the silhouette distance
            StarQuery q = star_query<COUNT>(E.S, w.x, w.y, E.eps * E.eps, w.lastD, cell.id, cell.front);
            cp = q.D;
            float dD = sqrtf(cp.d2);
            if (dD <= E.eps) { value = w.acc + w.weight * g_value(E, cp); return true; }
            R = fminf(dD, sqrtf(q.s2));
        } else {
            cp = closest_point<COUNT>(E.S, w.x, w.y, kClsD, kFInf, w.lastD, cell.id, cell.front);
            float dD = sqrtf(cp.d2);
            if (dD <= E.eps) { value = w.acc + w.weight * g_value(E, cp); return true; }
            R = dD;
        }
        w.lastD = cp.seg;
    }
    R = fmaxf(R, E.rmin);
    float factor = w.onN ? 2.0f : 1.0f;
    if constexpr (SRC) w.acc += w.weight * factor * source_term(E, w.x, w.y, R, u01(rnd.y), u01(rnd.z));
    if (NEU && E.hasH && !far) w.acc += w.weight * factor * neumann_term(E, w.x, w.y, R, u01(rnd.w));
    // direction: full circle, or the half circle around the inward normal on Neumann
    float dx, dy;
    if (w.onN) {
        float sn, cs;
        __sincosf(kPi * (u01(rnd.x) - 0.5f), &sn, &cs);
        dx = w.inx * cs - w.iny * sn;
        dy = w.inx * sn + w.iny * cs;
    } else {
        __sincosf(kTwoPi * u01(rnd.x), &dy, &dx);
    }
    float travel = R;
    bool hit = false;
    if (NEU && !far) {
        RayHit h = E.runN ? ray_runs(E, w.x, w.y, dx, dy, R, w.onN ? w.prevSeg : -1, cell.ray)
                          : intersect_ray<COUNT>(E.S, w.x, w.y, dx, dy, R, kClsNeumann, E.tguard,
                                                 w.onN ? w.prevSeg : -1, cell.ray);
        if (h.seg >= 0) {
            hit = true;
            travel = h.t;
            float2 n = E.S.segNormal[h.seg];
            // pointwise.cpp:157 picks the side the ray came from; in a closed scene
            // every Neumann segment bounds the domain with outward n, so the walker's
            // side is -n (a walker that rounded onto the far side is pulled back)
            if (E.closed || n.x * dx + n.y * dy > 0.0f) { w.inx = -n.x; w.iny = -n.y; } else { w.inx = n.x; w.iny = n.y; }
            // FP32 hit points can round to the far side of the wall, where a later
            // ray would re-enter through a neighbouring segment and trap the walk
            // outside; keep the walker nudge (~2^-20 diag) on the side it came from
            w.x = fmaf(E.nudge, w.inx, h.px);
            w.y = fmaf(E.nudge, w.iny, h.py);
            w.onN = 1;
            w.prevSeg = h.seg;
        }
    }
    if (!hit) {
        w.x = fmaf(R, dx, w.x);
        w.y = fmaf(R, dy, w.y);
        w.onN = 0;
        w.prevSeg = -1;
    }
    if constexpr (SCR) w.weight *= ball_sphere_weight(E.P.sqrtSigma, R, travel);
    // safety net: a walker that left the scene's neighbourhood (impossible in exact
    // arithmetic) ends like a truncated walk instead of wandering to maxSteps
    bool escaped = fabsf(w.x - E.cx) > E.escape || fabsf(w.y - E.cy) > E.escape;
    if (++w.step >= E.maxSteps || escaped) {  // truncation: g at the closest Dirichlet point (pointwise.cpp:162-164)
        trunc = 1;
        Closest c = E.drunN ? star_runs(E, w.x, w.y, false).D : closest_point(E.S, w.x, w.y, kClsD);
        value = w.acc + w.weight * g_value(E, c);
        return true;
    }
    return false;
}

// task-level state: which estimator a lane serves and its accumulators
struct Task {
    long long id;     // local task index
    unsigned long long rid;  // RNG id (global point id * per + k)
    int role;         // 0 = U, 1 = D
    int pt, k;
    int phase;        // D: 0 = walk from the first-ball sphere, 1 = nested screened walk
    uint32_t draw;    // Philox draw counter
    float R, dirx, diry, vx, vy, cyx, cyy, y2x, y2y;
    int trunc;
};

__device__ __forceinline__ U4 draw4(const WalkEnv& E, Task& t) {
    U4 c{static_cast<uint32_t>(t.rid), static_cast<uint32_t>(t.rid >> 32), t.draw++,
         static_cast<uint32_t>(t.role)};
    return philox4x32_10(c, E.k0, E.k1);
}

// resident blocks per SM (registers per thread = 64K / (256 x MINB)), measured on
// C1-C3: Neumann scenes 4 (C2: 6.36 ms vs 6.72 at 6), screened 8 (C3: 148 vs 155 ms
// at 6), plain Laplace 6 (C1: 1.29 vs 1.40 ms at 8)
#ifndef BVC_W2_MINB_NEU
#define BVC_W2_MINB_NEU 4
#endif
#ifndef BVC_W2_MINB_SCR
#define BVC_W2_MINB_SCR 8
#endif
#ifndef BVC_W2_MINB_DIR
#define BVC_W2_MINB_DIR 6
#endif
template <bool NEU, bool SCR, bool SRC, bool COUNT,
          int MINB = NEU ? BVC_W2_MINB_NEU : (SCR ? BVC_W2_MINB_SCR : BVC_W2_MINB_DIR)>
__global__ void __launch_bounds__(kWalkThreads, MINB) walk_kernel(const WalkEnv E, const WalkJob J) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const long long nUtot = static_cast<long long>(J.nPtsU) * J.nU;
    const long long total = nUtot + static_cast<long long>(J.nPtsDdev ? *J.nPtsDdev : J.nPtsD) * J.nD;
    long long qNext = 0, qEnd = 0;
    bool exhausted = false;
    bool active = false;
    Task t;
    Walk w;
    unsigned long long steps = 0;
    for (;;) {
        unsigned need = __ballot_sync(0xffffffffu, !active);
        while (need && !exhausted) {
            if (qNext >= qEnd) {
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(J.counter, static_cast<unsigned long long>(kChunk));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (static_cast<long long>(base) >= total) { exhausted = true; break; }
                qNext = static_cast<long long>(base);
                qEnd = min(qNext + kChunk, total);
            }
            int take = static_cast<int>(min(static_cast<long long>(__popc(need)), qEnd - qNext));
            int rank = __popc(need & lt);
            if (((need >> lane) & 1u) && rank < take) {
                long long id = qNext + rank;
                t.id = id;
                t.draw = 0;
                t.phase = 0;
                t.trunc = 0;
                if (id < nUtot) {
                    t.role = 0;
                    t.pt = id < 0x7fffffffLL ? static_cast<int>(static_cast<unsigned>(id) / static_cast<unsigned>(J.nU))
                                             : static_cast<int>(id / J.nU);
                    t.k = static_cast<int>(id - static_cast<long long>(t.pt) * J.nU);
                    long long g = J.gidU ? J.gidU[t.pt] : J.gidBaseU + t.pt;
                    t.rid = static_cast<unsigned long long>(g) * J.nU + t.k;
                    float2 s = J.startU[t.pt];
                    walk_start(w, s.x, s.y);
                    if (J.hintU) w.lastD = J.hintU[t.pt];
                } else {
                    long long d = id - nUtot;
                    t.role = 1;
                    t.pt = d < 0x7fffffffLL ? static_cast<int>(static_cast<unsigned>(d) / static_cast<unsigned>(J.nD))
                                            : static_cast<int>(d / J.nD);
                    t.k = static_cast<int>(d - static_cast<long long>(t.pt) * J.nD);
                    long long g = J.gidD ? J.gidD[t.pt] : t.pt;
                    t.rid = static_cast<unsigned long long>(g) * J.nD + t.k;
                    // gradientSample (pointwise.cpp:195-215): sphere point, source and nested draws
                    float2 c = J.xD[t.pt];
                    t.R = J.radiusD[t.pt];
                    U4 r0 = draw4(E, t);
                    U4 r1 = draw4(E, t);
                    __sincosf(kTwoPi * u01(r0.x), &t.diry, &t.dirx);
                    t.vx = 0.0f;
                    t.vy = 0.0f;
                    if constexpr (SRC) {
                        BallSample b = sample_ball(c.x, c.y, t.R, u01(r0.y), u01(r0.z));
                        float fy = field_eval(E.P.f, b.x, b.y);
                        if (fy != 0.0f) {
                            float ddx = b.x - c.x, ddy = b.y - c.y;
                            float gf = (1.0f / (t.R * t.R) - 1.0f / (ddx * ddx + ddy * ddy)) * kInv2Pi * (fy / b.pdf);
                            t.vx += ddx * gf;
                            t.vy += ddy * gf;
                        }
                    }
                    if (SCR && E.P.sigma > 0.0f) {
                        BallSample b = sample_ball(c.x, c.y, t.R, u01(r0.w), u01(r1.x));
                        float ddx = b.x - c.x, ddy = b.y - c.y;
                        float gf = (1.0f / (t.R * t.R) - 1.0f / (ddx * ddx + ddy * ddy)) * kInv2Pi *
                                   (E.P.sigma / b.pdf);
                        t.cyx = ddx * gf;
                        t.cyy = ddy * gf;
                        t.y2x = b.x;
                        t.y2y = b.y;
                    }
                    // the first ball touches the boundary: start a hair inside it
                    float rr = t.R * 0.99999952f;
                    walk_start(w, fmaf(rr, t.dirx, c.x), fmaf(rr, t.diry, c.y));
                    if (J.hintD) w.lastD = J.hintD[t.pt];
                }
                active = true;
            }
            qNext += take;
            need = __ballot_sync(0xffffffffu, !active);
        }
        if (__ballot_sync(0xffffffffu, active) == 0u) break;
        if (active) {
            U4 rnd = draw4(E, t);
            float value;
            if (walk_step<NEU, SCR, SRC, COUNT>(E, w, rnd, value, t.trunc, steps)) {
                if (t.role == 0) {
                    J.outU[t.id] = value;
                    if (t.trunc && J.truncU) atomicAdd(J.truncU + t.pt, 1);
                    if (t.trunc && J.truncTotal) atomicAdd(J.truncTotal, 1ull);
                    active = false;
                } else if (t.phase == 0) {
                    float s = (2.0f / t.R) * value;
                    t.vx = fmaf(s, t.dirx, t.vx);
                    t.vy = fmaf(s, t.diry, t.vy);
                    if (SCR && E.P.sigma > 0.0f) {
                        t.phase = 1;
                        walk_start(w, t.y2x, t.y2y);
                        if (J.hintD) w.lastD = J.hintD[t.pt];
                    } else {
                        active = false;
                    }
                } else {
                    t.vx = fmaf(t.cyx, value, t.vx);
                    t.vy = fmaf(t.cyy, value, t.vy);
                    active = false;
                }
                if (!active && t.role == 1) {
                    long long slot = t.id - nUtot;
                    if (J.normalD) {
                        float2 n = J.normalD[t.pt];
                        J.outD[slot] = n.x * t.vx + n.y * t.vy;
                    } else {
                        J.outD[2 * slot] = t.vx;
                        J.outD[2 * slot + 1] = t.vy;
                    }
                    if (t.trunc && J.truncD) atomicAdd(J.truncD + t.pt, 1);
                    if (t.trunc && J.truncTotal) atomicAdd(J.truncTotal, 1ull);
                }
            }
        }
    }
    if (J.steps) {
        for (int o = 16; o > 0; o >>= 1) steps += __shfl_xor_sync(0xffffffffu, steps, o);
        if (lane == 0) atomicAdd(J.steps, steps);
    }
}

// fixed-order per-point mean and standard error (runWalks pointwise.cpp:175-185)
__global__ void reduce_kernel(const float* vals, int nPts, int per, int comps, int comp, double* mean,
                              double* se) {
    int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (warp >= nPts) return;
    double s = 0.0, q = 0.0;
    const float* v = vals + static_cast<long long>(warp) * per * comps;
    for (int k = lane; k < per; k += 32) {
        double x = v[static_cast<long long>(k) * comps + comp];
        s += x;
        q += x * x;
    }
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        q += __shfl_xor_sync(0xffffffffu, q, o);
    }
    if (lane == 0) {
        double m = s / per;
        double var = fmax(0.0, q / per - m * m);
        mean[warp] = m;
        if (se) se[warp] = per > 1 ? sqrt(var / (per - 1)) : 0.0;
    }
}

__global__ void sample_boundary_kernel(const double* cdf, const int* ids, int m, double total,
                                       const float4* segAB, const float2* segNormal, const float* segArc,
                                       const float* segLen, int count, int begin, int n, const long long* ctr,
                                       int stratified, uint32_t k0, uint32_t k1, CacheSample* out) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    long long k = ctr ? ctr[j] : static_cast<long long>(begin) + j;
    U4 r = philox4x32_10(U4{static_cast<uint32_t>(k), static_cast<uint32_t>(k >> 32), 0u, 0u}, k0, k1);
    // 53-bit uniform from two words, like the reference's double draws
    double U = (static_cast<double>(r.x >> 5) * 67108864.0 + static_cast<double>(r.y >> 6)) * (1.0 / 9007199254740992.0);
    double u = stratified ? (static_cast<double>(k) + U) / count : U;
    double target = u * total;
    int lo = 0, hi = m;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (cdf[mid] < target) lo = mid + 1; else hi = mid;
    }
    int idx = lo >= m ? m - 1 : lo;
    int sid = ids[idx];
    double within = target - (idx > 0 ? cdf[idx - 1] : 0.0);
    double tt = within / segLen[sid];
    tt = fmin(fmax(tt, 0.0), 1.0);
    float4 s = segAB[sid];
    CacheSample o;
    o.z[0] = static_cast<float>(s.x + tt * (static_cast<double>(s.z) - s.x));
    o.z[1] = static_cast<float>(s.y + tt * (static_cast<double>(s.w) - s.y));
    o.z[2] = 0.0f;
    float2 nn = segNormal[sid];
    o.n[0] = nn.x;
    o.n[1] = nn.y;
    o.n[2] = 0.0f;
    o.pdf = static_cast<float>(1.0 / total);
    o.uHat = 0.0f;
    o.dHat = 0.0f;
    o.weight = 0.0f;
    o.arc = static_cast<float>(segArc[sid] + tt * segLen[sid]);
    o.segment = sid;
    out[j] = o;
}

__global__ void prepare_kernel(const WalkEnv E, CacheSample* samples, int n, const int* kinds, const int* source,
                               float2* startU, int* isD, float* gradR, uint8_t* outside) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    CacheSample s = samples[i];
    float x = s.z[0], y = s.z[1];
    int kind = kinds[s.segment];
    if (kind == 0) {  // known Neumann: walk from half a shell inside, d = h(z) exactly
        x -= 0.5f * E.eps * s.n[0];
        y -= 0.5f * E.eps * s.n[1];
        samples[i].dHat = E.hasH ? field_eval(E.P.h, s.z[0], s.z[1]) : 0.0f;
        isD[i] = 0;
        gradR[i] = 0.0f;
    } else {
        isD[i] = 1;
        Closest c = closest_point(E.S, x, y, kClsAny);
        gradR[i] = fmaxf(sqrtf(c.d2), E.rmin);
    }
    (void)source;
    startU[i] = make_float2(x, y);
    outside[i] = (E.insideTol < 0.0f || inside(E.S, x, y, E.insideTol)) ? 0 : 1;
}

__global__ void gather_dpoints_kernel(const CacheSample* samples, const int* dIdx, int nD, const float* gradR,
                                      long long gidBase, const long long* gid, float2* xD, float2* nD_, float* rD,
                                      long long* gidD, const int* nDdev) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= (nDdev ? *nDdev : nD)) return;
    int i = dIdx[j];
    CacheSample s = samples[i];
    xD[j] = make_float2(s.z[0], s.z[1]);
    nD_[j] = make_float2(s.n[0], s.n[1]);
    rD[j] = gradR[i];
    gidD[j] = gid ? gid[i] : gidBase + i;
}

__global__ void finish_kernel(CacheSample* samples, int n, const float* outU, int nU, const int* dIdx, int nDcap,
                              const float* outD, int nD, uint8_t* failed, const int* nDdev,
                              unsigned long long* walksCtr) {
    int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    const int nDpts = nDdev ? *nDdev : nDcap;
    if (walksCtr && warp == 0 && lane == 0)
        atomicAdd(walksCtr, static_cast<unsigned long long>(n) * nU + static_cast<unsigned long long>(nDpts) * nD);
    if (warp >= n + nDpts) return;
    const float* v;
    int per, i;
    if (warp < n) { i = warp; v = outU + static_cast<long long>(i) * nU; per = nU; }
    else { int j = warp - n; i = dIdx[j]; v = outD + static_cast<long long>(j) * nD; per = nD; }
    double s = 0.0;
    for (int k = lane; k < per; k += 32) s += v[k];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
        float m = static_cast<float>(s / per);
        if (warp < n) samples[i].uHat = m; else samples[i].dHat = m;
        if (!isfinite(s)) failed[i] = 1;
    }
}
__global__ void compact_u8_kernel(const uint8_t* flags, int n, int* outIdx, int* outCount) {
    __shared__ int sums[1024];
    int tid = threadIdx.x, nt = blockDim.x;
    int chunk = (n + nt - 1) / nt;
    int b = tid * chunk, e = min(n, b + chunk);
    int c = 0;
    for (int i = b; i < e; ++i) c += flags[i] != 0;
    sums[tid] = c;
    __syncthreads();
    for (int off = 1; off < nt; off <<= 1) {
        int v = tid >= off ? sums[tid - off] : 0;
        __syncthreads();
        sums[tid] += v;
        __syncthreads();
    }
    int pos = sums[tid] - c;
    for (int i = b; i < e; ++i)
        if (flags[i]) outIdx[pos++] = i;
    if (tid == nt - 1) *outCount = sums[tid];
}

// single-CTA compaction: each thread scans a contiguous chunk
__global__ void compact_kernel(const int* flags, int n, int* outIdx, int* outCount) {
    __shared__ int sums[1024];
    int tid = threadIdx.x, nt = blockDim.x;
    int chunk = (n + nt - 1) / nt;
    int b = tid * chunk, e = min(n, b + chunk);
    int c = 0;
    for (int i = b; i < e; ++i) c += flags[i] != 0;
    sums[tid] = c;
    __syncthreads();
    for (int off = 1; off < nt; off <<= 1) {
        int v = tid >= off ? sums[tid - off] : 0;
        __syncthreads();
        sums[tid] += v;
        __syncthreads();
    }
    int pos = sums[tid] - c;
    for (int i = b; i < e; ++i)
        if (flags[i]) outIdx[pos++] = i;
    if (tid == nt - 1) *outCount = sums[tid];
}

__global__ void closest_kernel(const SceneView2 S, const double* x, int n, unsigned mask, double* point,
                               double* dist, int* seg, double* t) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Closest c = closest_point(S, static_cast<float>(x[2 * i]), static_cast<float>(x[2 * i + 1]), mask);
    point[2 * i] = c.px;
    point[2 * i + 1] = c.py;
    dist[i] = c.seg >= 0 ? sqrt(static_cast<double>(c.d2)) : INFINITY;
    seg[i] = c.seg;
    t[i] = c.t;
}

__global__ void silhouette_kernel(const SceneView2 S, const double* x, int n, double* dist) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float d2 = silhouette_dist2(S, static_cast<float>(x[2 * i]), static_cast<float>(x[2 * i + 1]));
    dist[i] = sqrt(static_cast<double>(d2));
}

__global__ void ray_kernel(const SceneView2 S, const double* o, const double* d, int n, float tMax, unsigned mask,
                           float tMin, double* t, int* seg, double* point, double* s) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    RayHit h = intersect_ray(S, static_cast<float>(o[2 * i]), static_cast<float>(o[2 * i + 1]),
                             static_cast<float>(d[2 * i]), static_cast<float>(d[2 * i + 1]), tMax, mask, tMin, -1);
    t[i] = h.seg >= 0 ? h.t : INFINITY;
    seg[i] = h.seg;
    point[2 * i] = h.px;
    point[2 * i + 1] = h.py;
    s[i] = h.s;
}

__global__ void inside_kernel(const SceneView2 S, const double* x, int n, float tol, uint8_t* out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = inside(S, static_cast<float>(x[2 * i]), static_cast<float>(x[2 * i + 1]), tol) ? 1 : 0;
}

inline int blocks(long long n, int t) { return static_cast<int>((n + t - 1) / t); }

__global__ void farfield2_kernel(const SceneView2 S, const FarField F, float* d) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= F.nx * F.ny) return;
    int ix = i % F.nx, iy = i / F.nx;
    float x = fmaf(static_cast<float>(ix), F.h, F.lox), y = fmaf(static_cast<float>(iy), F.h, F.loy);
    d[i] = sqrtf(closest_point(S, x, y, kClsAny).d2);
}

__global__ void hintgrid2_kernel(const SceneView2 S, const HintGrid G, HintCell* cells, int entries, int fronts,
                                 float rmin) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= G.nx * G.ny) return;
    int ix = i % G.nx, iy = i / G.nx;
    // cell [v, v + h)^2: centre c, half-diagonal rho; r = dD(c) + 2 rho plus FP32 slack
    const float cx = fmaf(static_cast<float>(ix) + 0.5f, G.h, G.lox), cy = fmaf(static_cast<float>(iy) + 0.5f, G.h, G.loy),
                rho = 0.70710678f * G.h;
    const Closest c = closest_point(S, cx, cy, kClsD);
    HintCell out;
    out.id = c.seg;  // at x in the cell its distance is at most d(x) + 2 |x - c|
    out.pad0 = out.pad1 = 0;
    out.front = kRootStart;
    out.ray = 0;
    if (entries) {
        const float r = sqrtf(c.d2) + 2.0f * rho + 1e-5f * S.diagonal;
        const float rr = r + rmin;
        out.ray = entry_node(S, cx, cy, rr * rr, kClsNeumann);
        int f[4] = {kNoEntry, kNoEntry, kNoEntry, kNoEntry};
        if (fronts) entry_frontier2(S, cx, cy, r * r, kClsD | kClsSil, f);
        else f[0] = entry_node(S, cx, cy, r * r, kClsD | kClsSil);
        if (f[0] == kNoEntry) f[0] = 0;  // cannot happen for a star query (the closest Dirichlet primitive qualifies)
        out.front = make_int4(f[0], f[1], f[2], f[3]);
    }
    cells[i] = out;
}


__global__ void start_hints_kernel(const CacheSample* samples, int n, const int* source, const int* cls,
                                   const int* leafOf, const int* dIdx, int nD, int* hintU, int* hintD,
                                   const int* nDdev) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (nDdev) nD = *nDdev;
    auto hint = [&](int k) {
        int seg = samples[k].segment;
        int src = source ? (seg >= 0 ? source[seg] : -1) : seg;
        if (src < 0 || cls[src] != 0) return -1;  // only a Dirichlet primitive may seed the D distance
        return leafOf ? leafOf[src] : src;
    };
    if (i < n) hintU[i] = hint(i);
    if (i < nD) hintD[i] = hint(dIdx[i]);
}

__global__ void leaf_index_kernel(int dim, const void* prims, int n, int* leafOf) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int id = dim == 2 ? static_cast<const Prim2*>(prims)[j].id
                      : __float_as_int(static_cast<const bvc_dev::Prim3*>(prims)[j].a.w);
    leafOf[id] = j;
}

}  // namespace

template <bool NEU, bool SCR, bool SRC, bool COUNT>
void launch_walk_t(const WalkEnv& env, const WalkJob& job, long long total, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int perSm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&perSm, walk_kernel<NEU, SCR, SRC, COUNT>, kWalkThreads, 0);
    perSm = perSm > 0 ? perSm : 1;
    if (const char* e = std::getenv("BVC_WALK_OCC")) {  // co-residency experiments: blocks per SM cap
        int v = std::atoi(e);
        if (v >= 1 && v < perSm) perSm = v;
    }
    long long want = (total + kWalkThreads - 1) / kWalkThreads;
    int grid = static_cast<int>(want < static_cast<long long>(sms) * perSm ? want : static_cast<long long>(sms) * perSm);
    walk_kernel<NEU, SCR, SRC, COUNT><<<grid, kWalkThreads, 0, st>>>(env, job);
}

void launch_farfield2(const SceneView2& S, const FarField& F, float* d, cudaStream_t st) {
    farfield2_kernel<<<blocks(static_cast<long long>(F.nx) * F.ny, 128), 128, 0, st>>>(S, F, d);
    count_launch();
}

void launch_hintgrid2(const SceneView2& S, const HintGrid& G, HintCell* cells, bool entries, bool fronts, float rmin,
                      cudaStream_t st) {
    hintgrid2_kernel<<<blocks(static_cast<long long>(G.nx) * G.ny, 128), 128, 0, st>>>(S, G, cells, entries ? 1 : 0,
                                                                                   fronts ? 1 : 0, rmin);
    count_launch();
}

void launch_start_hints(const CacheSample* samples, int n, const int* source, const int* cls, const int* leafOf,
                        const int* dIdx, int nD, int* hintU, int* hintD, cudaStream_t st, const int* nDdev) {
    int m = n > nD ? n : nD;
    if (m <= 0) return;
    start_hints_kernel<<<blocks(m, 256), 256, 0, st>>>(samples, n, source, cls, leafOf, dIdx, nD, hintU, hintD, nDdev);
    count_launch();
}
void launch_leaf_index(int dim, const void* prims, int n, int* leafOf, cudaStream_t st) {
    if (n <= 0) return;
    leaf_index_kernel<<<blocks(n, 256), 256, 0, st>>>(dim, prims, n, leafOf);
    count_launch();
}

void launch_walk_job(const WalkEnv& env, const WalkJob& job, cudaStream_t st) {
    long long total = static_cast<long long>(job.nPtsU) * job.nU + static_cast<long long>(job.nPtsD) * job.nD;
    if (total <= 0) return;
    cudaMemsetAsync(job.counter, 0, sizeof(unsigned long long), st);
    const int code = (env.hasNeumann ? 1 : 0) | (env.P.screened ? 2 : 0) | (env.hasSource ? 4 : 0) |
                     (env.S.counts ? 8 : 0);
    switch (code) {
#define BVC_WALK_CASE(c) \
    case c: launch_walk_t<(c & 1) != 0, (c & 2) != 0, (c & 4) != 0, (c & 8) != 0>(env, job, total, st); break;
        BVC_WALK_CASE(0) BVC_WALK_CASE(1) BVC_WALK_CASE(2) BVC_WALK_CASE(3)
        BVC_WALK_CASE(4) BVC_WALK_CASE(5) BVC_WALK_CASE(6) BVC_WALK_CASE(7)
        BVC_WALK_CASE(8) BVC_WALK_CASE(9) BVC_WALK_CASE(10) BVC_WALK_CASE(11)
        BVC_WALK_CASE(12) BVC_WALK_CASE(13) BVC_WALK_CASE(14) BVC_WALK_CASE(15)
#undef BVC_WALK_CASE
    }
    count_launch();
}

void launch_reduce_estimates(const float* vals, int nPts, int per, int comps, int comp, double* mean, double* se,
                             cudaStream_t st) {
    if (nPts <= 0) return;
    reduce_kernel<<<blocks(static_cast<long long>(nPts) * 32, 256), 256, 0, st>>>(vals, nPts, per, comps, comp, mean, se);
    count_launch();
}

void launch_sample_boundary(const double* cdf, const int* ids, int m, double total, const float4* segAB,
                            const float2* segNormal, const float* segArc, const float* segLen, int count, int begin,
                            int n, const long long* ctr, int stratified, uint32_t k0, uint32_t k1, CacheSample* out,
                            cudaStream_t st) {
    if (n <= 0) return;
    sample_boundary_kernel<<<blocks(n, 256), 256, 0, st>>>(cdf, ids, m, total, segAB, segNormal, segArc, segLen, count,
                                                          begin, n, ctr, stratified, k0, k1, out);
    count_launch();
}

void launch_prepare_samples(const WalkEnv& env, CacheSample* samples, int n, const int* regionKinds,
                            const int* regionSource, float2* startU, int* isD, float* gradR, uint8_t* outside,
                            cudaStream_t st) {
    if (n <= 0) return;
    prepare_kernel<<<blocks(n, 128), 128, 0, st>>>(env, samples, n, regionKinds, regionSource, startU, isD, gradR,
                                                   outside);
    count_launch();
}

void launch_gather_dpoints(const CacheSample* samples, const int* dIdx, int nD, const float* gradR, long long gidBase,
                           const long long* gid, float2* xD, float2* nD_, float* rD, long long* gidD,
                           cudaStream_t st, const int* nDdev) {
    if (nD <= 0) return;
    gather_dpoints_kernel<<<blocks(nD, 256), 256, 0, st>>>(samples, dIdx, nD, gradR, gidBase, gid, xD, nD_, rD, gidD,
                                                            nDdev);
    count_launch();
}

void launch_finish_samples(CacheSample* samples, int n, const float* outU, int nU, const int* dIdx, int nDpts,
                           const float* outD, int nD, uint8_t* failed, cudaStream_t st, const int* nDdev,
                           unsigned long long* walksCtr) {
    long long warps = static_cast<long long>(n) + nDpts;
    if (warps <= 0) return;
    finish_kernel<<<blocks(warps * 32, 256), 256, 0, st>>>(samples, n, outU, nU, dIdx, nDpts, outD, nD, failed, nDdev,
                                                           walksCtr);
    count_launch();
}

void launch_compact_u8(const uint8_t* flags, int n, int* outIdx, int* outCount, cudaStream_t st) {
    compact_u8_kernel<<<1, 1024, 0, st>>>(flags, n, outIdx, outCount);
    count_launch();
}

void launch_compact(const int* flags, int n, int* outIdx, int* outCount, cudaStream_t st) {
    compact_kernel<<<1, 1024, 0, st>>>(flags, n, outIdx, outCount);
    count_launch();
}

void launch_closest(const SceneView2& S, const double* x, int n, unsigned mask, double* point, double* dist, int* seg,
                    double* t, cudaStream_t st) {
    if (n <= 0) return;
    closest_kernel<<<blocks(n, 128), 128, 0, st>>>(S, x, n, mask, point, dist, seg, t);
    count_launch();
}

void launch_silhouette(const SceneView2& S, const double* x, int n, double* dist, cudaStream_t st) {
    if (n <= 0) return;
    silhouette_kernel<<<blocks(n, 128), 128, 0, st>>>(S, x, n, dist);
    count_launch();
}

void launch_ray(const SceneView2& S, const double* o, const double* d, int n, double tMax, unsigned mask, double tMin,
                double* t, int* seg, double* point, double* s, cudaStream_t st) {
    if (n <= 0) return;
    float tm = static_cast<float>(fmin(tMax, 3.0e38));
    ray_kernel<<<blocks(n, 128), 128, 0, st>>>(S, o, d, n, tm, mask, static_cast<float>(tMin), t, seg, point, s);
    count_launch();
}

void launch_inside(const SceneView2& S, const double* x, int n, float tol, uint8_t* out, cudaStream_t st) {
    if (n <= 0) return;
    inside_kernel<<<blocks(n, 128), 128, 0, st>>>(S, x, n, tol, out);
    count_launch();
}

}  // namespace bvc_impl
