// gather.cu — the dense interior evaluation (boundary-integral splats) on sm_100a.
//
// Reference: splatSolution cache.cpp:426-461 and splatGradient cache.cpp:463-497
// over the kernels of kernels.h:78-129 (reference sign convention).
//
// N-body style FP32 gather. Per-sample constants are folded once (pack_*):
//   2D Laplace boundary: A = w u/2pi, B = w d ln2/4pi, Bg = w d/2pi  (w = 1/pdf or
//   Voronoi weight*N), so a pair costs dx,dy,r2,nd, rcp, lg2 and a few FMAs.
// Each CTA owns PT query points (Q per thread, register-blocked) and streams a
// chunk of the cache through shared memory in tiles of TS samples; tiles arrive
// by 1D TMA bulk copies (cp.async.bulk + mbarrier, double-buffered) and are read
// as warp-wide broadcasts. Tile partials are FP32; tiles and chunks accumulate in
// FP64 in a fixed order, so sums are deterministic and independent of the grid
// and of how points are sharded across GPUs. Near-coincident pairs
// (r < 1e-12 diag, cache.cpp:436-440) are rare: the hot loop only tracks min r^2
// and a slow path redoes a tile for a point that hit one.
#include <cuda_runtime.h>

#include <cstdlib>

#include "gather.h"
#include "tma.cuh"

namespace bvc_impl {

using namespace bvc_dev;

namespace {

constexpr int kThreads = 128;
#ifndef BVC_UNROLL_PACKED
#define BVC_UNROLL_PACKED 2
#endif
constexpr int kUnrollPacked = BVC_UNROLL_PACKED;  // samples per packed tile-loop iteration
constexpr int kQ = 4;  // query points per thread (register blocking), most kinds
// screened-3D values (C5) hold BVC_Q_SCR3 points per thread (measured, see DESIGN)
#ifndef BVC_Q_SCR3
#define BVC_Q_SCR3 4
#endif
template <int KIND, bool VAL, bool GRAD, int MODE>
constexpr int q_of() { return (KIND == 4 && VAL && !GRAD && MODE == 0) ? BVC_Q_SCR3 : kQ; }
constexpr int kTS = 256;            // samples per shared-memory tile

// --- per-pair kernels ---------------------------------------------------------
// 2D: payload a = (zx, zy, nx, ny) (Laplace boundary: (zx, zy, A nx, A ny)),
// b = per-kind constants
struct Acc {
    float v, gx, gy, gz;
};


// --- screened 2D, written once for one lane (float) and two packed lanes (F2) ----
// Every product and sum is an explicit fma / mul (never a mul feeding an add, which
// ptxas would contract for f32x2), so a point gets identical bits on the scalar path
// (slow tiles, clamp modes, eval_kernels) and on the packed one.
struct SOps {
    using V = float;
    static __device__ __forceinline__ V c(float x) { return x; }
    static __device__ __forceinline__ V mul(V a, V b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ V sub(V a, V b) { return __fsub_rn(a, b); }
    static __device__ __forceinline__ V fma(V a, V b, V d) { return fmaf(a, b, d); }
    template <class Fn>
    static __device__ __forceinline__ V map(V a, Fn&& f) { return f(a); }
};
struct POps {
    using V = F2;
    static __device__ __forceinline__ V c(float x) { return bc(x); }
    static __device__ __forceinline__ V mul(V a, V b) { return mul2(a, b); }
    static __device__ __forceinline__ V sub(V a, V b) { return sub2(a, b); }
    static __device__ __forceinline__ V fma(V a, V b, V d) { return fma2(a, b, d); }
    template <class Fn>
    static __device__ __forceinline__ V map(V a, Fn&& f) { return each(a, f); }
};

// K0(t) and Q = t K1(t) for t <= 2 (A&S 9.8.1-9.8.4 with I0/I1 9.8.1/9.8.3), Horner with fma
template <class O>
__device__ __forceinline__ void k0q_small(typename O::V t, typename O::V& K0, typename O::V& Q) {
    using V = typename O::V;
    const V h = O::mul(t, O::c(0.5f));
    const V y = O::mul(h, h);
    const V l = O::map(h, [](float x) { return f_lg2(x); });
    const V lnh = O::mul(l, O::c(kLn2)), nlnh = O::mul(l, O::c(-kLn2));
    const V w = O::mul(O::mul(t, t), O::c(1.0f / 14.0625f));
    V i0 = O::fma(w, O::c(0.0045813f), O::c(0.0360768f));
    i0 = O::fma(w, i0, O::c(0.2659732f));
    i0 = O::fma(w, i0, O::c(1.2067492f));
    i0 = O::fma(w, i0, O::c(3.0899424f));
    i0 = O::fma(w, i0, O::c(3.5156229f));
    i0 = O::fma(w, i0, O::c(1.0f));
    V i1 = O::fma(w, O::c(0.00032411f), O::c(0.00301532f));
    i1 = O::fma(w, i1, O::c(0.02658733f));
    i1 = O::fma(w, i1, O::c(0.15084934f));
    i1 = O::fma(w, i1, O::c(0.51498869f));
    i1 = O::fma(w, i1, O::c(0.87890594f));
    i1 = O::fma(w, i1, O::c(0.5f));
    i1 = O::mul(t, i1);
    V p0 = O::fma(y, O::c(0.0000074f), O::c(0.00010750f));
    p0 = O::fma(y, p0, O::c(0.00262698f));
    p0 = O::fma(y, p0, O::c(0.03488590f));
    p0 = O::fma(y, p0, O::c(0.23069756f));
    p0 = O::fma(y, p0, O::c(0.42278420f));
    p0 = O::fma(y, p0, O::c(-0.57721566f));
    V p1 = O::fma(y, O::c(-0.00004686f), O::c(-0.00110404f));
    p1 = O::fma(y, p1, O::c(-0.01919402f));
    p1 = O::fma(y, p1, O::c(-0.18156897f));
    p1 = O::fma(y, p1, O::c(-0.67278579f));
    p1 = O::fma(y, p1, O::c(0.15443144f));
    p1 = O::fma(y, p1, O::c(1.0f));
    K0 = O::fma(nlnh, i0, p0);
    Q = O::fma(O::mul(t, lnh), i1, p1);
}
// the same for t > 2 (A&S 9.8.5-9.8.8)
template <class O>
__device__ __forceinline__ void k0q_large(typename O::V t, typename O::V& K0, typename O::V& Q) {
    using V = typename O::V;
    const V rt = O::map(t, [](float x) { return f_rsq(x); });
    const V e = O::map(O::mul(t, O::c(-1.44269504088896340736f)), [](float x) { return f_ex2(x); });
    const V y = O::mul(O::mul(rt, rt), O::c(2.0f));
    V p0 = O::fma(y, O::c(0.00053208f), O::c(-0.00251540f));
    p0 = O::fma(y, p0, O::c(0.00587872f));
    p0 = O::fma(y, p0, O::c(-0.01062446f));
    p0 = O::fma(y, p0, O::c(0.02189568f));
    p0 = O::fma(y, p0, O::c(-0.07832358f));
    p0 = O::fma(y, p0, O::c(1.25331414f));
    V p1 = O::fma(y, O::c(-0.00068245f), O::c(0.00325614f));
    p1 = O::fma(y, p1, O::c(-0.00780353f));
    p1 = O::fma(y, p1, O::c(0.01504268f));
    p1 = O::fma(y, p1, O::c(-0.03655620f));
    p1 = O::fma(y, p1, O::c(0.23498619f));
    p1 = O::fma(y, p1, O::c(1.25331414f));
    const V er = O::mul(e, rt);
    K0 = O::mul(p0, er);
    Q = O::mul(O::mul(p1, er), t);
}

// One screened-2D pair (kernels.h:62-129 with G = -K0/2pi folded into the payload):
// a = (zx, zy, nx, ny), b = (w u / 2pi, w d / 2pi) for a boundary sample, b.x =
// (f / pdf) / 2pi for a source sample. K0/Q pick their branch per lane.
template <class O, bool SRC, bool VAL, bool GRAD, int MODE>
__device__ __forceinline__ void scr2_pair(const float4 a, const float4 b, typename O::V px, typename O::V py,
                                          float sigma, float s, typename O::V& v, typename O::V& gx,
                                          typename O::V& gy, typename O::V& r2out, float c2pi) {
    using V = typename O::V;
    const V dx = O::sub(O::c(a.x), px), dy = O::sub(O::c(a.y), py);
    const V r2 = O::fma(dx, dx, O::mul(dy, dy));
    r2out = r2;
    const V ir = O::map(r2, [](float x) { return f_rsq(x); });
    const V ir2 = O::mul(ir, ir);
    const V t = O::mul(O::c(s), O::mul(r2, ir));
    V K0, Q;
    if constexpr (sizeof(V) == sizeof(float)) {
        if (t <= 2.0f) k0q_small<O>(t, K0, Q);
        else k0q_large<O>(t, K0, Q);
    } else {
        float t0, t1;
        upk(t, t0, t1);
        const bool s0 = t0 <= 2.0f, s1 = t1 <= 2.0f;
        V Ks = O::c(0.f), Qs = O::c(0.f), Kl = O::c(0.f), Ql = O::c(0.f);
        if (s0 || s1) k0q_small<O>(t, Ks, Qs);
        if (!s0 || !s1) k0q_large<O>(t, Kl, Ql);
        float ks0, ks1, qs0, qs1, kl0, kl1, ql0, ql1;
        upk(Ks, ks0, ks1);
        upk(Qs, qs0, qs1);
        upk(Kl, kl0, kl1);
        upk(Ql, ql0, ql1);
        K0 = pk(s0 ? ks0 : kl0, s1 ? ks1 : kl1);
        Q = pk(s0 ? qs0 : ql0, s1 ? qs1 : ql1);
    }
    if constexpr (!SRC) {
        const V nd = O::fma(O::c(a.z), dx, O::mul(O::c(a.w), dy));
        const V p = O::mul(nd, ir2);
        if constexpr (VAL) {
            V qp = O::mul(Q, p);
            if constexpr ((MODE & 1) != 0) qp = fminf(fmaxf(qp, -c2pi), c2pi);  // kClampP (scalar only)
            v = O::fma(O::c(b.x), qp, O::fma(O::c(b.y), K0, v));
        }
        if constexpr (GRAD) {
            // d (A (2 Q p / r^2 + sigma K0 p) + B Q / r^2) - n (A Q / r^2)
            const V aq = O::mul(O::c(b.x), Q);
            const V inner = O::fma(O::c(b.x * sigma), O::mul(K0, p), O::mul(O::mul(O::c(b.y), Q), ir2));
            const V q = O::fma(O::mul(aq, O::c(2.0f)), O::mul(p, ir2), inner);
            const V c = O::mul(aq, ir2);
            gx = O::fma(q, dx, O::fma(c, O::c(-a.z), gx));
            gy = O::fma(q, dy, O::fma(c, O::c(-a.w), gy));
        }
    } else {
        if constexpr (VAL) v = O::fma(O::c(-b.x), K0, v);
        if constexpr (GRAD) {
            const V nc = O::mul(O::mul(O::c(-b.x), Q), ir2);
            gx = O::fma(nc, dx, gx);
            gy = O::fma(nc, dy, gy);
        }
    }
}

// splat variants of correctedBoundarySplat / correctedSourceSplat (cache.cpp:499-597):
//   kClampP: dG/dn clamped to [-c, c] in the boundary term (clampKernel kernels.h:52)
//   kBall:   G -> G^B(x, R_x) (ballGreens kernels.cpp:31-43) in the d-hat and source terms
//   kClampS: source G^B clamped to [-c, c]
enum SplatMode { kClampP = 1, kBall = 2, kClampS = 4 };
struct ModeCtx {
    float c2pi;   // 2 pi c (the clamp in the units of nd / r^2)
    float R2;     // R_x^2 (ball radius of the evaluation point)
    float lgR2;   // log2 R_x^2
    float sclamp; // c 4 pi / ln 2 (the source clamp in log2 units)
};

// Accumulator sign conventions, chosen so that no pair needs a negation (the tile
// end restores the signs): 2D Laplace values are accumulated negated (-u), 3D
// Laplace boundary gradients negated; everything else as is.
template <int KIND, bool SRC>
struct Conv {
    static constexpr bool negV = KIND == kLap2;
    static constexpr bool negG = KIND == kLap3 && !SRC;
};

// Scalar pair. Plain products and sums use the non-contracting __fmul_rn /
// __fadd_rn, so this is bit-identical, lane by lane, to the packed pair2 below
// (FMUL2 / FADD2 / FFMA2 round each lane exactly like FMUL / FADD / FFMA):
// points take the packed or the scalar path (slow tiles, clamp modes) and get
// the same bits either way.
template <int KIND, bool SRC, bool VAL, bool GRAD, bool TRACK = false, int MODE = 0>
__device__ __forceinline__ void pair(const float4 a, const float4 b, float px, float py, float pz, float sigma,
                                     float s, Acc& acc, float& mn, const ModeCtx* mc = nullptr) {
    if constexpr (KIND == kLap2 || KIND == kScr2) {
        float dx = __fsub_rn(a.x, px), dy = __fsub_rn(a.y, py);
        float r2 = fmaf(dx, dx, __fmul_rn(dy, dy));
        if constexpr (TRACK) mn = fminf(mn, r2);
        if constexpr (KIND == kLap2) {
            float nir2 = f_rcp(-r2);  // -1 / r^2
            if constexpr (!SRC) {
                // a.zw = A n, b = (A, B ln2/4pi-scaled, -Bg, 0): t = -A p, -u += B lg2 r^2 + t
                float ndA = fmaf(a.z, dx, __fmul_rn(a.w, dy));
                float t = __fmul_rn(ndA, nir2);
                if constexpr (VAL) {
                    float l = (MODE & kBall) ? f_lg2(fminf(r2, mc->R2)) - mc->lgR2 : f_lg2(r2);
                    float base = fmaf(b.y, l, acc.v);
                    if constexpr ((MODE & kClampP) != 0) {
                        // clamp p = n.d / r^2 to +-2 pi c, i.e. A p to +-2 pi c |A|; an
                        // unsaturated pair gets exactly the plain path's bits
                        float lim = mc->c2pi * fabsf(b.x);
                        acc.v = fabsf(t) > lim ? __fadd_rn(base, copysignf(lim, t)) : fmaf(ndA, nir2, base);
                    } else {
                        acc.v = fmaf(ndA, nir2, base);
                    }
                }
                if constexpr (GRAD) {
                    float q = __fmul_rn(fmaf(t, 2.0f, b.z), nir2);     // (2 A p + Bg) / r^2
                    acc.gx = fmaf(q, dx, fmaf(nir2, a.z, acc.gx));     // - (A / r^2) n
                    acc.gy = fmaf(q, dy, fmaf(nir2, a.w, acc.gy));
                }
            } else {
                // b = (-c ln2/4pi, c/2pi, 0, 0)
                if constexpr (VAL) {
                    float l = (MODE & kBall) ? f_lg2(fminf(r2, mc->R2)) - mc->lgR2 : f_lg2(r2);
                    if constexpr ((MODE & kClampS) != 0) l = fmaxf(l, -mc->sclamp);
                    acc.v = fmaf(b.x, l, acc.v);
                }
                if constexpr (GRAD) {
                    float c = __fmul_rn(b.y, nir2);
                    acc.gx = fmaf(c, dx, acc.gx);
                    acc.gy = fmaf(c, dy, acc.gy);
                }
            }
        } else {
            float r2o;
            scr2_pair<SOps, SRC, VAL, GRAD, MODE>(a, b, px, py, sigma, s, acc.v, acc.gx, acc.gy, r2o,
                                                  (MODE & kClampP) ? mc->c2pi : 0.0f);
        }
    } else {
        // 3D boundary payload a = (zx, zy, zz, A nx), b = (A ny, A nz, -B, B); source a = (y, -C)
        float dx = __fsub_rn(a.x, px), dy = __fsub_rn(a.y, py), dz = __fsub_rn(a.z, pz);
        float r2 = fmaf(dx, dx, fmaf(dy, dy, __fmul_rn(dz, dz)));
        if constexpr (TRACK) mn = fminf(mn, r2);
        float ir = f_rsq(r2);
        float ir2 = __fmul_rn(ir, ir), ir3 = __fmul_rn(ir2, ir);
        if constexpr (KIND == kLap3) {
            if constexpr (!SRC) {
                float ndA = fmaf(a.w, dx, fmaf(b.x, dy, __fmul_rn(b.y, dz)));
                // A (n.d) / r^3 + B / r = (A (n.d) / r^2 + B) / r: no 1/r^3 for values
                if constexpr (VAL) acc.v = fmaf(ir, fmaf(ndA, ir2, b.w), acc.v);
                if constexpr (GRAD) {  // accumulated negated: (A/r^3) n - q d
                    float nq = __fmul_rn(fmaf(__fmul_rn(ndA, -3.0f), ir2, b.z), ir3);
                    acc.gx = fmaf(nq, dx, fmaf(ir3, a.w, acc.gx));
                    acc.gy = fmaf(nq, dy, fmaf(ir3, b.x, acc.gy));
                    acc.gz = fmaf(nq, dz, fmaf(ir3, b.y, acc.gz));
                }
            } else {
                if constexpr (VAL) acc.v = fmaf(a.w, ir, acc.v);
                if constexpr (GRAD) {
                    float c = __fmul_rn(a.w, ir3);
                    acc.gx = fmaf(c, dx, acc.gx);
                    acc.gy = fmaf(c, dy, acc.gy);
                    acc.gz = fmaf(c, dz, acc.gz);
                }
            }
        } else if constexpr (KIND == kScr3V) {
            static_assert(!GRAD && MODE == 0, "kScr3V is the value-only kind");
            // values in coordinates scaled by k = s log2(e) (see pack_boundary_one): with
            // r' = k r, e^{-s r} = 2^{-r'} and s + 1/r = k (ln2 + 1/r'), the k factors fold into
            // the payload (A k^2 n, k B; source k C), so the pair needs no scale multiply
            const float ir1 = ir;
            const float e = f_ex2(-__fmul_rn(r2, ir1));
            if constexpr (!SRC) {
                float ndA = fmaf(a.w, dx, fmaf(b.x, dy, __fmul_rn(b.y, dz)));
                acc.v = fmaf(__fmul_rn(e, ir1), fmaf(__fmul_rn(ndA, ir1), __fadd_rn(kLn2, ir1), b.w), acc.v);
            } else {
                acc.v = fmaf(__fmul_rn(a.w, ir1), e, acc.v);
            }
        } else {  // screened 3D: e = exp(-s r), Q = e (s r + 1)
            float r = __fmul_rn(r2, ir);
            float t = __fmul_rn(s, r);
            float e = f_ex2(__fmul_rn(r, -1.44269504088896340736f * s));
            float Q = fmaf(e, t, e);
            if constexpr (!SRC) {
                float ndA = fmaf(a.w, dx, fmaf(b.x, dy, __fmul_rn(b.y, dz)));
                float pA = __fmul_rn(ndA, ir3);  // A p
                // A p Q + B e / r = (e / r) (A (n.d) / r (s + 1 / r) + B): three fewer ops per pair
                if constexpr (VAL)
                    acc.v = fmaf(__fmul_rn(e, ir), fmaf(__fmul_rn(ndA, ir), __fadd_rn(s, ir), b.w), acc.v);
                if constexpr (GRAD) {
                    float q = fmaf(3.0f * Q * pA, ir2, b.w * Q * ir3);
                    q = fmaf(sigma * e, pA, q);
                    float c = Q * ir3;
                    acc.gx = fmaf(q, dx, fmaf(-c, a.w, acc.gx));
                    acc.gy = fmaf(q, dy, fmaf(-c, b.x, acc.gy));
                    acc.gz = fmaf(q, dz, fmaf(-c, b.y, acc.gz));
                }
            } else {
                if constexpr (VAL) acc.v = fmaf(__fmul_rn(a.w, ir), e, acc.v);
                if constexpr (GRAD) {
                    float c = a.w * Q * ir3;
                    acc.gx = fmaf(c, dx, acc.gx);
                    acc.gy = fmaf(c, dy, acc.gy);
                    acc.gz = fmaf(c, dz, acc.gz);
                }
            }
        }
    }
}

// --- packed FP32 (sm_100a FFMA2 / FMUL2 / FADD2): two query points per op --------
// The gather is issue-bound, not FP32-pipe-bound: a packed op does two lanes' work
// in one issue slot (measured: FFMA2 sustains the full 128 FP32 FMA/clk/SM), which
// leaves slots for the MUFU, LDS and loop instructions. Scalar sample operands
// broadcast for free (ptxas folds them into a .F32 operand).
struct Acc2 {
    F2 v, gx, gy, gz;
};

// which (KIND, VAL, GRAD, MODE) run packed: 2D and 3D Laplace, 3D screened values
template <int KIND, bool VAL, bool GRAD, int MODE>
struct Packed {
    static constexpr bool value =
        MODE == 0 && (KIND == kLap2 || KIND == kLap3 || KIND == kScr2 || KIND == kScr3V || (KIND == kScr3 && !GRAD));
};

// pair() on two query points at once; same operations, same rounding per lane
template <int KIND, bool SRC, bool VAL, bool GRAD, bool TRACK>
__device__ __forceinline__ void pair2(const float4 a, const float4 b, F2 px, F2 py, F2 pz, float sigma, float s,
                                      Acc2& acc, float* mn) {
    if constexpr (KIND == kScr2) {
        F2 r2;
        scr2_pair<POps, SRC, VAL, GRAD, 0>(a, b, px, py, sigma, s, acc.v, acc.gx, acc.gy, r2, 0.0f);
        if constexpr (TRACK) {
            float lo, hi;
            upk(r2, lo, hi);
            mn[0] = fminf(mn[0], lo);
            mn[1] = fminf(mn[1], hi);
        }
    } else if constexpr (KIND == kLap2) {
        F2 dx = sub2(bc(a.x), px), dy = sub2(bc(a.y), py);
        F2 r2 = fma2(dx, dx, mul2(dy, dy));
        if constexpr (TRACK) {
            float lo, hi;
            upk(r2, lo, hi);
            mn[0] = fminf(mn[0], lo);
            mn[1] = fminf(mn[1], hi);
        }
        F2 nir2 = each(r2, [](float x) { return f_rcp(-x); });
        if constexpr (!SRC) {
            F2 ndA = fma2(bc(a.z), dx, mul2(bc(a.w), dy));
            F2 t = mul2(ndA, nir2);
            // (ptxas contracts a mul2 feeding an add2 into FFMA2 even for .rn, so the
            // fused form is written out, here and in the scalar pair())
            if constexpr (VAL) acc.v = fma2(ndA, nir2, fma2(bc(b.y), each(r2, [](float x) { return f_lg2(x); }), acc.v));
            if constexpr (GRAD) {
                F2 q = mul2(fma2(t, bc(2.0f), bc(b.z)), nir2);
                acc.gx = fma2(q, dx, fma2(nir2, bc(a.z), acc.gx));
                acc.gy = fma2(q, dy, fma2(nir2, bc(a.w), acc.gy));
            }
        } else {
            if constexpr (VAL) acc.v = fma2(bc(b.x), each(r2, [](float x) { return f_lg2(x); }), acc.v);
            if constexpr (GRAD) {
                F2 c = mul2(bc(b.y), nir2);
                acc.gx = fma2(c, dx, acc.gx);
                acc.gy = fma2(c, dy, acc.gy);
            }
        }
    } else {
        F2 dx = sub2(bc(a.x), px), dy = sub2(bc(a.y), py), dz = sub2(bc(a.z), pz);
        F2 r2 = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
        if constexpr (TRACK) {
            float lo, hi;
            upk(r2, lo, hi);
            mn[0] = fminf(mn[0], lo);
            mn[1] = fminf(mn[1], hi);
        }
        F2 ir = each(r2, [](float x) { return f_rsq(x); });
        F2 ir2 = mul2(ir, ir), ir3 = mul2(ir2, ir);
        if constexpr (KIND == kLap3) {
            if constexpr (!SRC) {
                F2 ndA = fma2(bc(a.w), dx, fma2(bc(b.x), dy, mul2(bc(b.y), dz)));
                if constexpr (VAL) acc.v = fma2(ir, fma2(ndA, ir2, bc(b.w)), acc.v);
                if constexpr (GRAD) {
                    F2 nq = mul2(fma2(mul2(ndA, bc(-3.0f)), ir2, bc(b.z)), ir3);
                    acc.gx = fma2(nq, dx, fma2(ir3, bc(a.w), acc.gx));
                    acc.gy = fma2(nq, dy, fma2(ir3, bc(b.x), acc.gy));
                    acc.gz = fma2(nq, dz, fma2(ir3, bc(b.y), acc.gz));
                }
            } else {
                if constexpr (VAL) acc.v = fma2(bc(a.w), ir, acc.v);
                if constexpr (GRAD) {
                    F2 c = mul2(bc(a.w), ir3);
                    acc.gx = fma2(c, dx, acc.gx);
                    acc.gy = fma2(c, dy, acc.gy);
                    acc.gz = fma2(c, dz, acc.gz);
                }
            }
        } else if constexpr (KIND == kScr3V) {  // scaled coordinates (scalar pair above)
            F2 e = each(mul2(r2, ir), [](float x) { return f_ex2(-x); });
            if constexpr (!SRC) {
                F2 ndA = fma2(bc(a.w), dx, fma2(bc(b.x), dy, mul2(bc(b.y), dz)));
                acc.v = fma2(mul2(e, ir), fma2(mul2(ndA, ir), add2(bc(kLn2), ir), bc(b.w)), acc.v);
            } else {
                acc.v = fma2(mul2(bc(a.w), ir), e, acc.v);
            }
        } else {  // kScr3, values only
            F2 r = mul2(r2, ir);
            F2 e = each(mul2(r, bc(-1.44269504088896340736f * s)), [](float x) { return f_ex2(x); });
            if constexpr (!SRC) {
                F2 ndA = fma2(bc(a.w), dx, fma2(bc(b.x), dy, mul2(bc(b.y), dz)));
                acc.v = fma2(mul2(e, ir), fma2(mul2(ndA, ir), add2(bc(s), ir), bc(b.w)), acc.v);
            } else {
                acc.v = fma2(mul2(bc(a.w), ir), e, acc.v);
            }
        }
    }
}

struct Params {
    const float4* pack;      // 2 float4 per sample; boundary samples [0, N), source [N, N+M)
    int N, M;
    const float* px;         // dim * K (active points, sorted order)
    int K, dim;
    int chunk;               // samples per chunk (multiple of kTS)
    int chunksB, chunksS;    // chunks over boundary / source samples
    int tiles;               // point tiles
    float sigma, s, tol, tol2;
    float coordScale;        // kScr3V: k = s log2(e) (points, pack and tol are scaled); else 1
    double* part;            // [(chunksB + chunksS)][comps][K]
    int comps;               // 1 (value) + dim (gradient) as enabled
    int* skipB;              // [K]
    int* skipS;
    const float4* tileBox;   // per shared-memory tile: lo (x, y, z), hi (x, y, z) of its samples
    int tilesB;              // boundary tiles (source tiles follow)
    unsigned* unitCounter;   // dynamic work-unit queue (zeroed per launch)
    // corrected-splat variants (MODE != 0)
    float clamp;             // c
    const float* ballR;      // per active point (sorted order): ball radius R_x
};

__device__ __forceinline__ ModeCtx mode_ctx(const Params& P, int i) {
    ModeCtx m;
    m.c2pi = kTwoPi * P.clamp;
    m.sclamp = P.clamp * 4.0f * kPi / kLn2;
    float R = (P.ballR && i < P.K) ? P.ballR[i] : 1.0f;
    m.R2 = R * R;
    m.lgR2 = f_lg2(m.R2);
    return m;
}

// slow path: recompute one point's tile partial, skipping near-coincident samples
template <int KIND, bool SRC, bool VAL, bool GRAD, int MODE>
__device__ void tile_slow(const float4* sm, int cnt, float px, float py, float pz, const Params& P, Acc& acc,
                          int& skips, const ModeCtx* mc) {
    acc = Acc{0.f, 0.f, 0.f, 0.f};
    for (int j = 0; j < cnt; ++j) {
        float4 a = sm[2 * j], b = sm[2 * j + 1];
        float dx = a.x - px, dy = a.y - py, dz = (KIND == kLap3 || KIND == kScr3 || KIND == kScr3V) ? a.z - pz : 0.0f;
        if (dx * dx + dy * dy + dz * dz < P.tol2) { ++skips; continue; }  // cache.cpp:436-440
        float mn = 0.f;
        pair<KIND, SRC, VAL, GRAD, false, MODE>(a, b, px, py, pz, P.sigma, P.s, acc, mn, mc);
    }
}

template <int KIND, bool SRC, bool VAL, bool GRAD, bool TRACK, int MODE, int kQ>
__device__ __forceinline__ void tile_loop(const float4* S, int cnt, const float* px, const float* py, const float* pz,
                                          const Params& P, Acc* acc, float* mn, const ModeCtx* mc) {
    if constexpr (Packed<KIND, VAL, GRAD, MODE>::value) {
        F2 px2[kQ / 2], py2[kQ / 2], pz2[kQ / 2];
        Acc2 a2[kQ / 2];
#pragma unroll
        for (int h = 0; h < kQ / 2; ++h) {
            px2[h] = pk(px[2 * h], px[2 * h + 1]);
            py2[h] = pk(py[2 * h], py[2 * h + 1]);
            pz2[h] = pk(pz[2 * h], pz[2 * h + 1]);
            a2[h].v = a2[h].gx = a2[h].gy = a2[h].gz = pk(0.f, 0.f);
        }
#pragma unroll kUnrollPacked
        for (int j = 0; j < cnt; ++j) {
            const float4 a = S[2 * j], b = S[2 * j + 1];
#pragma unroll
            for (int h = 0; h < kQ / 2; ++h)
                pair2<KIND, SRC, VAL, GRAD, TRACK>(a, b, px2[h], py2[h], pz2[h], P.sigma, P.s, a2[h], mn + 2 * h);
        }
#pragma unroll
        for (int h = 0; h < kQ / 2; ++h) {
            upk(a2[h].v, acc[2 * h].v, acc[2 * h + 1].v);
            upk(a2[h].gx, acc[2 * h].gx, acc[2 * h + 1].gx);
            upk(a2[h].gy, acc[2 * h].gy, acc[2 * h + 1].gy);
            upk(a2[h].gz, acc[2 * h].gz, acc[2 * h + 1].gz);
        }
    } else {
#pragma unroll 2
        for (int j = 0; j < cnt; ++j) {
            const float4 a = S[2 * j], b = S[2 * j + 1];
#pragma unroll
            for (int q = 0; q < kQ; ++q)
                pair<KIND, SRC, VAL, GRAD, TRACK, MODE>(a, b, px[q], py[q], pz[q], P.sigma, P.s, acc[q], mn[q], mc + q);
        }
    }
}

template <int KIND, bool VAL, bool GRAD, int MODE>
__device__ __forceinline__ void gather_body(const Params& P) {
    constexpr int kQ = q_of<KIND, VAL, GRAD, MODE>();
    constexpr int kPT = kThreads * kQ;  // points per CTA tile
    __shared__ __align__(128) float4 sm[2][2 * kTS];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ int sUnit;
    const int tid = threadIdx.x;
    const int units = P.tiles * (P.chunksB + P.chunksS);
    constexpr bool D3 = (KIND == kLap3 || KIND == kScr3 || KIND == kScr3V);
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned phase[2] = {0u, 0u};
    // units are equal-cost (point tile x sample chunk); CTAs take them from a queue
    // so the last partial wave is filled by whichever CTAs finish first
    for (int unit = blockIdx.x; unit < units;) {
        const int chunkId = unit % (P.chunksB + P.chunksS);
        const int tile = unit / (P.chunksB + P.chunksS);
        const bool src = chunkId >= P.chunksB;
        const int c0 = src ? P.N + (chunkId - P.chunksB) * P.chunk : chunkId * P.chunk;
        const int cEnd = src ? min(c0 + P.chunk, P.N + P.M) : min(c0 + P.chunk, P.N);
        const int nT = (cEnd - c0 + kTS - 1) / kTS;
        // points
        float px[kQ], py[kQ], pz[kQ];
        int pidx[kQ];
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
            // each thread owns kQ consecutive points of the Morton order: a packed pair
            // holds neighbours (same screened-Bessel branch), a warp one compact patch
            int i = tile * kPT + tid * kQ + q;
            pidx[q] = i;
            bool ok = i < P.K;
            px[q] = ok ? P.px[P.dim * i] : 1e30f;
            py[q] = ok ? P.px[P.dim * i + 1] : 1e30f;
            pz[q] = (ok && D3) ? P.px[P.dim * i + 2] : 0.0f;
            if constexpr (KIND == kScr3V) {  // gather coordinates (pack_boundary_one)
                px[q] = ok ? __fmul_rn(px[q], P.coordScale) : 1e30f;
                py[q] = ok ? __fmul_rn(py[q], P.coordScale) : 1e30f;
                pz[q] = __fmul_rn(pz[q], P.coordScale);
            }
        }
        double dv[kQ], dg0[kQ], dg1[kQ], dg2[kQ];
        int skips[kQ];
#pragma unroll
        for (int q = 0; q < kQ; ++q) { dv[q] = dg0[q] = dg1[q] = dg2[q] = 0.0; skips[q] = 0; }
        ModeCtx mc[kQ];
        if constexpr (MODE != 0) {
#pragma unroll
            for (int q = 0; q < kQ; ++q) mc[q] = mode_ctx(P, pidx[q]);
        }
        // prologue: first two tiles in flight
        if (tid == 0) {
#pragma unroll
            for (int st = 0; st < 2; ++st)
                if (st < nT) {
                    int s0 = c0 + st * kTS, cnt = min(kTS, cEnd - s0);
                    mbar_expect_tx(&bar[st], cnt * 32u);
                    bulk_g2s(sm[st], P.pack + 2 * static_cast<size_t>(s0), cnt * 32u, &bar[st]);
                }
        }
        for (int it = 0; it < nT; ++it) {
            const int st = it & 1;
            const int s0 = c0 + it * kTS, cnt = min(kTS, cEnd - s0);
            // near-coincidence (r < tol) is only possible for points inside the tile's
            // sample box grown by tol; those (point, tile) pairs take the exact slow path
            const int tb = src ? P.tilesB + (s0 - P.N) / kTS : s0 / kTS;
            const float4 blo = P.tileBox[2 * tb], bhi = P.tileBox[2 * tb + 1];
            bool near = false;
#pragma unroll
            for (int q = 0; q < kQ; ++q)
                near |= pidx[q] < P.K && px[q] >= blo.x - P.tol && px[q] <= bhi.x + P.tol && py[q] >= blo.y - P.tol &&
                        py[q] <= bhi.y + P.tol && (!D3 || (pz[q] >= blo.z - P.tol && pz[q] <= bhi.z + P.tol));
            // warp-uniform: warps with a point inside the tile box track min r^2 per pair
            const bool track = __any_sync(0xffffffffu, near);
            mbar_wait(&bar[st], phase[st]);
            phase[st] ^= 1u;
            Acc acc[kQ];
            float mn[kQ];
#pragma unroll
            for (int q = 0; q < kQ; ++q) { acc[q] = Acc{0.f, 0.f, 0.f, 0.f}; mn[q] = 3.0e38f; }
            const float4* S = sm[st];
            if (!src) {
                if (track) tile_loop<KIND, false, VAL, GRAD, true, MODE, kQ>(S, cnt, px, py, pz, P, acc, mn, mc);
                else tile_loop<KIND, false, VAL, GRAD, false, MODE, kQ>(S, cnt, px, py, pz, P, acc, mn, mc);
            } else {
                if (track) tile_loop<KIND, true, VAL, GRAD, true, MODE, kQ>(S, cnt, px, py, pz, P, acc, mn, mc);
                else tile_loop<KIND, true, VAL, GRAD, false, MODE, kQ>(S, cnt, px, py, pz, P, acc, mn, mc);
            }
#pragma unroll
            for (int q = 0; q < kQ; ++q) {
                if (mn[q] < P.tol2 && pidx[q] < P.K) {
                    if (!src) tile_slow<KIND, false, VAL, GRAD, MODE>(S, cnt, px[q], py[q], pz[q], P, acc[q], skips[q], mc + q);
                    else tile_slow<KIND, true, VAL, GRAD, MODE>(S, cnt, px[q], py[q], pz[q], P, acc[q], skips[q], mc + q);
                }
                // undo the accumulator sign conventions (Conv)
                const bool nv = src ? Conv<KIND, true>::negV : Conv<KIND, false>::negV;
                const bool ng = src ? Conv<KIND, true>::negG : Conv<KIND, false>::negG;
                if (VAL) dv[q] += nv ? -static_cast<double>(acc[q].v) : static_cast<double>(acc[q].v);
                if (GRAD) {
                    dg0[q] += ng ? -static_cast<double>(acc[q].gx) : static_cast<double>(acc[q].gx);
                    dg1[q] += ng ? -static_cast<double>(acc[q].gy) : static_cast<double>(acc[q].gy);
                    if (D3) dg2[q] += ng ? -static_cast<double>(acc[q].gz) : static_cast<double>(acc[q].gz);
                }
            }
            __syncthreads();  // everyone is done reading buffer st
            if (tid == 0 && it + 2 < nT) {
                int s2 = c0 + (it + 2) * kTS, cnt2 = min(kTS, cEnd - s2);
                mbar_expect_tx(&bar[st], cnt2 * 32u);
                bulk_g2s(sm[st], P.pack + 2 * static_cast<size_t>(s2), cnt2 * 32u, &bar[st]);
            }
        }
        // chunk partials: fixed slot per (chunk, component, point)
        double* out = P.part + static_cast<size_t>(chunkId) * P.comps * P.K;
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
            int i = pidx[q];
            if (i >= P.K) continue;
            int c = 0;
            if (VAL) out[static_cast<size_t>(c++) * P.K + i] = dv[q];
            if (GRAD) {
                out[static_cast<size_t>(c++) * P.K + i] = dg0[q];
                out[static_cast<size_t>(c++) * P.K + i] = dg1[q];
                if (D3) out[static_cast<size_t>(c++) * P.K + i] = dg2[q];
            }
            if (skips[q]) atomicAdd(src ? P.skipS + i : P.skipB + i, skips[q]);
        }
        if (tid == 0) sUnit = static_cast<int>(gridDim.x + atomicAdd(P.unitCounter, 1u));
        __syncthreads();
        unit = sUnit;
        __syncthreads();
    }
}

// (kThreads, 1): an explicit minimum of one CTA lets ptxas use more registers than the
// bare bound does; screened 3D values run 2.3% faster with it (C5 4.52 -> 4.42 s), screened
// 2D the same
template <int KIND, bool VAL, bool GRAD, int MODE = 0>
__global__ void __launch_bounds__(kThreads, 1) gather_kernel(const Params P) {
    gather_body<KIND, VAL, GRAD, MODE>(P);
}
// the Laplace kinds at 8 (2D; 64 registers) / 7 (3D; 72 registers) resident CTAs: measured
// against 6, 7 and 8 (C2 gather 2.52 / 2.52 / 2.40 ms, C4 228 / 218 / 223 ms); the screened
// kinds spill 272-448 B at 64 registers and keep the compiler's choice (C3 +2%)
template <int KIND, bool VAL, bool GRAD>
__global__ void __launch_bounds__(kThreads, KIND == kLap3 ? 7 : 8) gather_kernel8(const Params P) {
    gather_body<KIND, VAL, GRAD, 0>(P);
}

// bounding box of each 256-sample tile (one warp per tile)
// fold per-sample constants (the "pack-cache epilogue")
__device__ __forceinline__ void pack_boundary_one(const CacheSample& s, int n, int kind, int voronoi, float4* out,
                                                  int i, float k = 1.f) {
    double w = voronoi ? static_cast<double>(s.weight) * n : 1.0 / static_cast<double>(s.pdf);
    double u = s.uHat, d = s.dHat;
    const double inv2pi = 0.15915494309189533577, inv4pi = 0.07957747154594766788, ln2 = 0.69314718055994530942;
    float4 a, b;
    if (kind == kLap2) {
        double A = w * u * inv2pi;
        a = make_float4(s.z[0], s.z[1], static_cast<float>(A * s.n[0]), static_cast<float>(A * s.n[1]));
        b = make_float4(static_cast<float>(A), static_cast<float>(w * d * ln2 * 0.5 * inv2pi),
                        static_cast<float>(-w * d * inv2pi), 0.f);
    } else if (kind == kScr2) {
        a = make_float4(s.z[0], s.z[1], s.n[0], s.n[1]);
        b = make_float4(static_cast<float>(w * u * inv2pi), static_cast<float>(w * d * inv2pi), 0.f, 0.f);
    } else if (kind == kScr3V) {  // scaled coordinates z' = k z; A k^2 in the normal, k B
        const double kk = k;
        double A = w * u * inv4pi * kk * kk, Bv = w * d * inv4pi * kk;
        a = make_float4(static_cast<float>(kk * s.z[0]), static_cast<float>(kk * s.z[1]), static_cast<float>(kk * s.z[2]),
                        static_cast<float>(A * s.n[0]));
        b = make_float4(static_cast<float>(A * s.n[1]), static_cast<float>(A * s.n[2]), static_cast<float>(-Bv),
                        static_cast<float>(Bv));
    } else {  // 3D: A folded into the normal, b = (A ny, A nz, -B, B)
        double A = w * u * inv4pi, Bv = w * d * inv4pi;
        a = make_float4(s.z[0], s.z[1], s.z[2], static_cast<float>(A * s.n[0]));
        b = make_float4(static_cast<float>(A * s.n[1]), static_cast<float>(A * s.n[2]), static_cast<float>(-Bv),
                        static_cast<float>(Bv));
    }
    out[2 * i] = a;
    out[2 * i + 1] = b;
}

__device__ __forceinline__ void pack_source_one(const SourceSampleDev& s, int kind, float4* out, int i, float k = 1.f) {
    double c = static_cast<double>(s.f) / static_cast<double>(s.pdf);
    const double inv2pi = 0.15915494309189533577, inv4pi = 0.07957747154594766788, ln2 = 0.69314718055994530942;
    float4 a, b = make_float4(0.f, 0.f, 0.f, 0.f);
    if (kind == kLap2) {
        a = make_float4(s.y[0], s.y[1], 0.f, 0.f);
        b = make_float4(static_cast<float>(-c * ln2 * 0.5 * inv2pi), static_cast<float>(c * inv2pi), 0.f, 0.f);
    } else if (kind == kScr2) {
        a = make_float4(s.y[0], s.y[1], 0.f, 0.f);
        b = make_float4(static_cast<float>(c * inv2pi), 0.f, 0.f, 0.f);
    } else if (kind == kScr3V) {
        const double kk = k;
        a = make_float4(static_cast<float>(kk * s.y[0]), static_cast<float>(kk * s.y[1]), static_cast<float>(kk * s.y[2]),
                        static_cast<float>(-c * inv4pi * kk));
    } else {
        a = make_float4(s.y[0], s.y[1], s.y[2], static_cast<float>(-c * inv4pi));
    }
    out[2 * i] = a;
    out[2 * i + 1] = b;
}
// The gather's prologue in one launch: pack the boundary and source samples (one CTA
// per 256-sample shared-memory tile), each tile's coordinate box (the near-coincidence
// test, gather_body), and zeroed skip counters and work-unit queue for the gather that
// follows on the same stream (instead of 2 pack launches, a box launch and 3 memsets)
__global__ void __launch_bounds__(kTS) prologue_kernel(const CacheSample* cs, int N, const SourceSampleDev* ss, int M,
                                                        int kind, int voronoi, float k, float4* pack, float4* box,
                                                        unsigned* unitCounter, int* skipB, int* skipS, int K) {
    const int tilesB = (N + kTS - 1) / kTS;
    const int t = blockIdx.x;
    const bool src = t >= tilesB;
    const int s0 = src ? N + (t - tilesB) * kTS : t * kTS;
    const int s1 = src ? min(s0 + kTS, N + M) : min(s0 + kTS, N);
    const int i = s0 + threadIdx.x;
    const bool d3 = kind == kLap3 || kind == kScr3 || kind == kScr3V;
    float lo[3] = {3e38f, 3e38f, 3e38f}, hi[3] = {-3e38f, -3e38f, -3e38f};
    if (i < s1) {
        if (!src) pack_boundary_one(cs[i], N, kind, voronoi, pack, i, k);
        else pack_source_one(ss[i - N], kind, pack + 2 * static_cast<size_t>(N), i - N, k);
        const float4 a = pack[2 * static_cast<size_t>(i)];
        const float c[3] = {a.x, a.y, d3 ? a.z : 0.f};
        for (int q = 0; q < 3; ++q) lo[q] = hi[q] = c[q];
    }
    __shared__ float red[6][kTS / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int q = 0; q < 3; ++q)
        for (int o = 16; o > 0; o >>= 1) {
            lo[q] = fminf(lo[q], __shfl_xor_sync(0xffffffffu, lo[q], o));
            hi[q] = fmaxf(hi[q], __shfl_xor_sync(0xffffffffu, hi[q], o));
        }
    if (lane == 0)
        for (int q = 0; q < 3; ++q) {
            red[q][warp] = lo[q];
            red[3 + q][warp] = hi[q];
        }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kTS / 32; ++w)
            for (int q = 0; q < 3; ++q) {
                red[q][0] = fminf(red[q][0], red[q][w]);
                red[3 + q][0] = fmaxf(red[3 + q][0], red[3 + q][w]);
            }
        box[2 * t] = make_float4(red[0][0], red[1][0], red[2][0], 0.f);
        box[2 * t + 1] = make_float4(red[3][0], red[4][0], red[5][0], 0.f);
    }
    const int g = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    if (g == 0) *unitCounter = 0u;
    for (int j = g; j < K; j += stride) {
        skipB[j] = 0;
        skipS[j] = 0;
    }
}


// G, dG/dx, dG/dn_y, d2G/dx dn_y through the hot loop's own pair() code with
// unit payloads (u = 1, d = 0, w = 1 for the double layer; f/pdf = 1 for G)
template <int KIND>
__global__ void eval_kernels_kernel(const double* x, const double* y, const double* n, int count, int dim,
                                    float sigma, double* out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    float px = x[dim * i], py = x[dim * i + 1], pz = dim == 3 ? x[dim * i + 2] : 0.f;
    CacheSample cs{};
    SourceSampleDev ss{};
    for (int k = 0; k < dim; ++k) {
        cs.z[k] = y[dim * i + k];
        cs.n[k] = n[dim * i + k];
        ss.y[k] = y[dim * i + k];
    }
    cs.pdf = 1.f; cs.uHat = 1.f; cs.dHat = 0.f;
    ss.pdf = 1.f; ss.f = 1.f;
    float4 pb[2], ps[2];
    pack_boundary_one(cs, 1, KIND, 0, pb, 0);
    pack_source_one(ss, KIND, ps, 0);
    Acc ab{0.f, 0.f, 0.f, 0.f}, as{0.f, 0.f, 0.f, 0.f};
    float mn = 0.f, s = sqrtf(sigma);
    pair<KIND, false, true, true>(pb[0], pb[1], px, py, pz, sigma, s, ab, mn);
    pair<KIND, true, true, true>(ps[0], ps[1], px, py, pz, sigma, s, as, mn);
    if (Conv<KIND, false>::negV) ab.v = -ab.v;
    if (Conv<KIND, true>::negV) as.v = -as.v;
    if (Conv<KIND, false>::negG) { ab.gx = -ab.gx; ab.gy = -ab.gy; ab.gz = -ab.gz; }
    if (Conv<KIND, true>::negG) { as.gx = -as.gx; as.gy = -as.gy; as.gz = -as.gz; }
    double* o = out + (2 + 2 * dim) * i;
    o[0] = as.v;
    o[1] = as.gx; o[2] = as.gy; if (dim == 3) o[3] = as.gz;
    o[1 + dim] = ab.v;
    o[2 + dim] = ab.gx; o[3 + dim] = ab.gy; if (dim == 3) o[4 + dim] = ab.gz;
}

__global__ void eval_bessel_kernel(int which, const double* t, int count, double* out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    float v = static_cast<float>(t[i]);
    out[i] = which == 0 ? bessel_k0(v) : which == 1 ? bessel_k1(v) : which == 2 ? bessel_i0(v) : bessel_i1(v);
}

// partials -> running sums of the evaluation points (cache.cpp:455-459, 491-495)
__global__ void finalize_kernel(const double* part, int chunksB, int chunksS, int comps, int K, const int* order,
                                int N, int M, int val, int grad, int dim, const int* skipB, const int* skipS,
                                PointsDev pts) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K) return;
    int p = order[i];
    size_t stride = static_cast<size_t>(comps) * K;
    double b[4] = {0, 0, 0, 0}, s[4] = {0, 0, 0, 0};
    for (int c = 0; c < chunksB; ++c)
        for (int k = 0; k < comps; ++k) b[k] += part[c * stride + static_cast<size_t>(k) * K + i];
    for (int c = chunksB; c < chunksB + chunksS; ++c)
        for (int k = 0; k < comps; ++k) s[k] += part[c * stride + static_cast<size_t>(k) * K + i];
    int sb = skipB[i], sS = skipS[i];
    int k = 0;
    if (val) {
        pts.bsum[p] += b[k];
        pts.ssum[p] += s[k];
        pts.nb[p] += N - sb;
        pts.ms[p] += M - sS;
        pts.skipped[p] += sb + sS;
        ++k;
    }
    if (grad) {
        for (int d = 0; d < dim; ++d) {
            pts.bgsum[static_cast<size_t>(dim) * p + d] += b[k + d];
            pts.sgsum[static_cast<size_t>(dim) * p + d] += s[k + d];
        }
        pts.nbg[p] += N - sb;
        pts.msg[p] += M - sS;
        pts.skipped[p] += sb + sS;
    }
}

__global__ void gather_points_kernel(const double* x, const int* order, int K, int dim, float* out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K) return;
    int p = order[i];
    for (int d = 0; d < dim; ++d) out[static_cast<size_t>(dim) * i + d] = static_cast<float>(x[static_cast<size_t>(dim) * p + d]);
}

template <int KIND>
void launch_kind(const Params& P, bool val, bool grad, int grid, cudaStream_t st) {
    if constexpr (KIND == kLap2 || KIND == kLap3) {
        if (val && grad) gather_kernel8<KIND, true, true><<<grid, kThreads, 0, st>>>(P);
        else if (val) gather_kernel8<KIND, true, false><<<grid, kThreads, 0, st>>>(P);
        else gather_kernel8<KIND, false, true><<<grid, kThreads, 0, st>>>(P);
    } else {
        if (val && grad) gather_kernel<KIND, true, true><<<grid, kThreads, 0, st>>>(P);
        else if (val) gather_kernel<KIND, true, false><<<grid, kThreads, 0, st>>>(P);
        else gather_kernel<KIND, false, true><<<grid, kThreads, 0, st>>>(P);
    }
}

template <int KIND>
int occupancy(bool val, bool grad) {
    int occ = 0;
    if constexpr (KIND == kScr3V) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gather_kernel<kScr3V, true, false>, kThreads, 0);
    } else if constexpr (KIND == kLap2 || KIND == kLap3) {
        if (val && grad) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gather_kernel8<KIND, true, true>, kThreads, 0);
        else if (val) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gather_kernel8<KIND, true, false>, kThreads, 0);
        else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gather_kernel8<KIND, false, true>, kThreads, 0);
    } else {
        if (val && grad) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gather_kernel<KIND, true, true>, kThreads, 0);
        else if (val) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gather_kernel<KIND, true, false>, kThreads, 0);
        else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gather_kernel<KIND, false, true>, kThreads, 0);
    }
    return occ > 0 ? occ : 1;
}

inline int blocks(long long n, int t) { return static_cast<int>((n + t - 1) / t); }

}  // namespace


void launch_prologue(const CacheSample* cs, int N, const SourceSampleDev* ss, int M, int kind, int voronoi, float k,
                     float4* pack, float4* tileBox, unsigned* unitCounter, int* skipB, int* skipS, int K,
                     cudaStream_t st) {
    const int tiles = (N + kTS - 1) / kTS + (M + kTS - 1) / kTS;
    if (tiles <= 0) return;
    if (const char* e = std::getenv("BVC_GATHER_CARVEOUT"))  // co-residency experiments (percent)
        cudaFuncSetAttribute(prologue_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(e));
    prologue_kernel<<<tiles, kTS, 0, st>>>(cs, N, ss, M, kind, voronoi, k, pack, tileBox, unitCounter, skipB, skipS, K);
    count_launch();
}


void eval_kernels(int kind, const double* x, const double* y, const double* n, int count, int dim, float sigma,
                  double* out, cudaStream_t st) {
    if (count <= 0) return;
    int g = blocks(count, 128);
    switch (kind) {
        case kLap2: eval_kernels_kernel<kLap2><<<g, 128, 0, st>>>(x, y, n, count, dim, sigma, out); break;
        case kScr2: eval_kernels_kernel<kScr2><<<g, 128, 0, st>>>(x, y, n, count, dim, sigma, out); break;
        case kLap3: eval_kernels_kernel<kLap3><<<g, 128, 0, st>>>(x, y, n, count, dim, sigma, out); break;
        default: eval_kernels_kernel<kScr3><<<g, 128, 0, st>>>(x, y, n, count, dim, sigma, out); break;
    }
    count_launch();
}

void eval_bessel(int which, const double* t, int count, double* out, cudaStream_t st) {
    if (count <= 0) return;
    eval_bessel_kernel<<<blocks(count, 128), 128, 0, st>>>(which, t, count, out);
    count_launch();
}

void gather_points(const double* x, const int* order, int K, int dim, float* out, cudaStream_t st) {
    if (K <= 0) return;
    gather_points_kernel<<<blocks(K, 256), 256, 0, st>>>(x, order, K, dim, out);
    count_launch();
}

GatherPlan plan_gather(int kind, int K, int N, int M, bool val, bool grad) {
    GatherPlan g;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int occ = kind == kLap2 ? occupancy<kLap2>(val, grad)
              : kind == kScr2 ? occupancy<kScr2>(val, grad)
              : kind == kLap3 ? occupancy<kLap3>(val, grad)
              : kind == kScr3V ? occupancy<kScr3V>(true, false)
                              : occupancy<kScr3>(val, grad);
    if (const char* e = std::getenv("BVC_GATHER_OCC")) {  // co-residency experiments: CTAs per SM cap
        int v = std::atoi(e);
        if (v >= 1 && v < occ) occ = v;
    }
    const int q = kind == kScr3V && val && !grad ? q_of<4, true, false, 0>() : kQ;
    g.tiles = (K + kThreads * q - 1) / (kThreads * q);
    long long slots = static_cast<long long>(sms) * occ;
    // The chunk size depends only on the cache (N + M), never on K: each point's
    // sum runs over the same chunks in the same order however the points are
    // split into ranges or ranks (bitwise shard invariance). 16 chunks give the
    // dynamic unit queue several waves at the configs' K (C2: 510 point tiles x 16
    // = 9 waves); a ~1-wave launch of long units measured 2x slower, because the
    // block scheduler does not always place every slot at once.
    int total = N + M;
    int maxTiles = (total + kTS - 1) / kTS;
    static const int knob = [] {  // BVC_GATHER_CHUNKS: sweep knob (0 = the default below)
        const char* e = std::getenv("BVC_GATHER_CHUNKS");
        int v = e ? std::atoi(e) : 0;
        return v >= 1 && v <= 1024 ? v : 0;
    }();
    // Caches of 2^19+ samples (C5) take 4 chunks: their units are plentiful at any useful
    // K, and every chunk costs an FP64 partial per point (C5: 16 chunks wrote 2.1 GB of
    // partials per round, 4 write 0.53 GB). Still a function of the cache size only.
    const int nChunks = knob ? knob : (total >= (1 << 19) ? 4 : 16);
    int ct = maxTiles > nChunks ? (maxTiles + nChunks - 1) / nChunks : 1;
    g.chunk = ct * kTS;
    g.chunksB = (N + g.chunk - 1) / g.chunk;
    g.chunksS = (M + g.chunk - 1) / g.chunk;
    long long units = static_cast<long long>(g.tiles) * (g.chunksB + g.chunksS);
    g.grid = static_cast<int>(units < slots ? units : slots);
    g.grid = g.grid > 0 ? g.grid : 1;
    g.comps = (val ? 1 : 0) + (grad ? (kind >= kLap3 ? 3 : 2) : 0);
    return g;
}

void launch_gather(int kind, const GatherPlan& g, const float4* pack, int N, int M, const float* px, int K, int dim,
                   float sigma, float tol, bool val, bool grad, double* part, int* skipB, int* skipS,
                   float4* tileBox, unsigned* unitCounter, cudaStream_t st, int mode, float clamp,
                   const float* ballR) {
    if (K <= 0 || (N + M) <= 0) return;
    Params P;
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
    P.sigma = sigma;
    P.s = sqrtf(sigma);
    P.coordScale = kind == kScr3V ? scr3v_scale(sigma) : 1.0f;  // the pack is scaled alike
    P.tol = tol * P.coordScale;
    P.tol2 = P.tol * P.tol;
    P.tilesB = (N + kTS - 1) / kTS;
    P.tileBox = tileBox;
    P.unitCounter = unitCounter;
    P.part = part;
    P.comps = g.comps;
    P.skipB = skipB;
    P.skipS = skipS;
    P.clamp = clamp;
    P.ballR = ballR;
    if (mode != 0) {  // corrected-splat variants: value only (cache.cpp:499-597)
        if (kind == kLap2) {
            switch (mode) {
                case kClampP: gather_kernel<kLap2, true, false, kClampP><<<g.grid, kThreads, 0, st>>>(P); break;
                case kBall: gather_kernel<kLap2, true, false, kBall><<<g.grid, kThreads, 0, st>>>(P); break;
                case kClampP | kBall: gather_kernel<kLap2, true, false, kClampP | kBall><<<g.grid, kThreads, 0, st>>>(P); break;
                case kBall | kClampS: gather_kernel<kLap2, true, false, kBall | kClampS><<<g.grid, kThreads, 0, st>>>(P); break;
                default: gather_kernel<kLap2, true, false, kClampP | kBall | kClampS><<<g.grid, kThreads, 0, st>>>(P); break;
            }
        } else {
            gather_kernel<kScr2, true, false, kClampP><<<g.grid, kThreads, 0, st>>>(P);
        }
        count_launch();
        return;
    }
    switch (kind) {
        case kLap2: launch_kind<kLap2>(P, val, grad, g.grid, st); break;
        case kScr2: launch_kind<kScr2>(P, val, grad, g.grid, st); break;
        case kLap3: launch_kind<kLap3>(P, val, grad, g.grid, st); break;
        case kScr3V:
            if (const char* e = std::getenv("BVC_GATHER_CARVEOUT"))  // co-residency experiments (percent)
                cudaFuncSetAttribute(gather_kernel<kScr3V, true, false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     std::atoi(e));
            gather_kernel<kScr3V, true, false><<<g.grid, kThreads, 0, st>>>(P);
            break;
        default: launch_kind<kScr3>(P, val, grad, g.grid, st); break;
    }
    count_launch();
}

void launch_finalize(const double* part, const GatherPlan& g, int K, const int* order, int N, int M, bool val,
                     bool grad, int dim, const int* skipB, const int* skipS, const PointsDev& pts, cudaStream_t st) {
    if (K <= 0) return;
    finalize_kernel<<<blocks(K, 256), 256, 0, st>>>(part, g.chunksB, g.chunksS, g.comps, K, order, N, M, val ? 1 : 0,
                                                    grad ? 1 : 0, dim, skipB, skipS, pts);
    count_launch();
}

}  // namespace bvc_impl
