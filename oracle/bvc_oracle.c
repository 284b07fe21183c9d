/*
 * bvc_oracle.c — CPU restatement of the reference's BVC hot path, in plain C.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only as the
 * checker or the timed CPU baseline — never as the product path.
 *
 * Every function follows a reference function, cited as file:line under
 * /root/reference/proj/core. Double precision throughout, like the reference.
 * Pinned by tests/test_oracle_pin.py against (a) the reference itself compiled
 * from its own sources into oracle/_ref (oracle/Makefile) and (b) the golden
 * vectors/known answers of the reference's tests (tests/golden/).
 *
 * Scope: RNG, Bessel functions, free-space and ball kernels, 2D scene queries
 * (brute-force twins), boundary/region samplers, WoS/WoSt walks and the
 * gradient estimator, boundary-cache generation, and the u / grad-u splats in
 * 2D and 3D. Region construction (buildSolveRegion) is host preprocessing and is
 * checked product-vs-reference directly; it is not restated here.
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/bvc_b200.h"

#define OR_PI 3.14159265358979323846
#define OR_INF (1.0 / 0.0)

/* ------------------------------------------------------------------------- */
/* RNG — rng.h:8-59 (SplitMix64 mixing, xoshiro256++, 53-bit uniforms)       */
/* ------------------------------------------------------------------------- */
uint64_t or_mix64(uint64_t z) { /* rng.h:8-13 */
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
uint64_t or_mixkey(uint64_t key, uint64_t counter) { /* rng.h:16-18 */
    return or_mix64(key ^ (counter + 0x9e3779b97f4a7c15ull));
}
typedef struct { uint64_t s[4]; } or_rng;
static void rng_from_key(or_rng* r, uint64_t key) { /* rng.h:25-31 */
    uint64_t z = key;
    for (int i = 0; i < 4; i++) { z += 0x9e3779b97f4a7c15ull; r->s[i] = or_mix64(z); }
}
static void rng_init(or_rng* r, uint64_t seed, uint64_t stream) { /* rng.h:33 */
    rng_from_key(r, or_mixkey(or_mix64(seed), stream));
}
static inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static uint64_t rng_next(or_rng* r) { /* rng.h:35-45 */
    uint64_t* s = r->s;
    const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}
static double rng_uniform(or_rng* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; } /* rng.h:48 */
static double rng_uniform_ab(or_rng* r, double a, double b) { return a + (b - a) * rng_uniform(r); }
static uint64_t rng_below(or_rng* r, uint64_t n) { return rng_next(r) % n; } /* rng.h:54 */

/* exported for pinning: n uniforms from Rng(seed, stream) */
void or_rng_uniforms(uint64_t seed, uint64_t stream, int n, double* out) {
    or_rng r; rng_init(&r, seed, stream);
    for (int i = 0; i < n; i++) out[i] = rng_uniform(&r);
}
void or_rng_key_uniforms(uint64_t key, int n, double* out) {
    or_rng r; rng_from_key(&r, key);
    for (int i = 0; i < n; i++) out[i] = rng_uniform(&r);
}

/* ------------------------------------------------------------------------- */
/* Bessel functions — kernels.cpp:7-29. The reference calls libstdc++'s       */
/* std::cyl_bessel_k/i; this restates them from the power series (t <= 2) and */
/* the integral K_nu(t) = int_0^inf exp(-t cosh s) cosh(nu s) ds (t > 2),    */
/* whose trapezoid rule converges geometrically (tests/support/oracles.h:19). */
/* ------------------------------------------------------------------------- */
static double bessel_i_series(int nu, double t) {
    double q = 0.25 * t * t, term = 1.0, sum = 0.0;
    for (int k = 1; k <= nu; k++) term *= 0.5 * t / k;
    for (int k = 0; k < 2000; k++) {
        sum += term;
        term *= q / ((k + 1.0) * (k + 1.0 + nu));
        if (term < 1e-18 * sum) break;
    }
    return sum;
}
static double bessel_k_quad(int nu, double t) {
    double h = 0.0625, sum = 0.5 * exp(-t);
    for (int k = 1; k < 100000; k++) {
        double s = k * h, e = -t * cosh(s);
        if (e < -745.0) break;
        double v = exp(e) * (nu ? cosh(s) : 1.0);
        sum += v;
        if (v < 1e-19 * sum) break;
    }
    return h * sum;
}
static const double OR_EULER = 0.57721566490153286061;
double or_bessel_i0(double t) { /* kernels.cpp:19-23 */
    if (t >= 700.0) return OR_INF;
    return bessel_i_series(0, t);
}
double or_bessel_i1(double t) { /* kernels.cpp:25-29 */
    if (t >= 700.0) return OR_INF;
    return bessel_i_series(1, t);
}
double or_bessel_k0(double t) { /* kernels.cpp:7-11 */
    if (!(t > 0.0)) return NAN;
    if (t >= 740.0) return 0.0;
    if (t > 2.0) return bessel_k_quad(0, t);
    double q = 0.25 * t * t, term = 1.0, H = 0.0, sum = 0.0;
    for (int k = 1; k < 200; k++) {
        term *= q / ((double)k * k);
        H += 1.0 / k;
        sum += term * H;
        if (term * H < 1e-18 * fabs(sum)) break;
    }
    return -(log(0.5 * t) + OR_EULER) * bessel_i_series(0, t) + sum;
}
double or_bessel_k1(double t) { /* kernels.cpp:13-17 */
    if (!(t > 0.0)) return NAN;
    if (t >= 740.0) return 0.0;
    if (t > 2.0) return bessel_k_quad(1, t);
    /* K1 = 1/t + ln(t/2) I1 - (t/4) sum_k [psi(k+1)+psi(k+2)] q^k / (k!(k+1)!) */
    double q = 0.25 * t * t, term = 1.0, sum = 0.0;
    double psi1 = -OR_EULER, psi2 = 1.0 - OR_EULER;
    for (int k = 0; k < 200; k++) {
        double v = (psi1 + psi2) * term;
        sum += v;
        term *= q / ((k + 1.0) * (k + 2.0));
        psi1 += 1.0 / (k + 1.0);
        psi2 += 1.0 / (k + 2.0);
        if (fabs(v) < 1e-18 * fabs(sum) && k > 2) break;
    }
    return 1.0 / t + log(0.5 * t) * bessel_i_series(1, t) - 0.25 * t * sum;
}

/* ------------------------------------------------------------------------- */
/* Free-space kernels — kernels.h:56-129 (reference sign convention)         */
/* ------------------------------------------------------------------------- */
static int guard_radius(const bvc_kernel_spec* s, double r) { /* kernels.h:56-59 */
    return (r >= 1e-12 * s->scale) ? 0 : BVC_ERR_SINGULARITY;
}
static double screened_q(const bvc_kernel_spec* s, double r) { /* kernels.h:62-66 */
    if (s->kind == BVC_KERNEL_POISSON) return 1.0;
    double t = r * sqrt(s->sigma);
    return s->dim == 2 ? or_bessel_k1(t) * t : exp(-t) * (t + 1.0);
}
static double screened_qprime(const bvc_kernel_spec* s, double r) { /* kernels.h:69-73 */
    if (s->kind == BVC_KERNEL_POISSON) return 0.0;
    double t = r * sqrt(s->sigma);
    return s->dim == 2 ? -s->sigma * or_bessel_k0(t) : -s->sigma * exp(-t);
}
static double vdot(const double* a, const double* b, int d) {
    double s = 0; for (int i = 0; i < d; i++) s += a[i] * b[i]; return s;
}
static double vdist(const double* a, const double* b, int d) {
    double s = 0; for (int i = 0; i < d; i++) { double t = a[i] - b[i]; s += t * t; } return sqrt(s);
}
/* greensFree kernels.h:78-86 */
int or_greens(const bvc_kernel_spec* s, const double* x, const double* y, double* out) {
    double r = vdist(x, y, s->dim);
    if (guard_radius(s, r)) return BVC_ERR_SINGULARITY;
    if (s->kind == BVC_KERNEL_POISSON)
        *out = s->dim == 2 ? log(r) / (2.0 * OR_PI) : -1.0 / (4.0 * OR_PI * r);
    else {
        double t = r * sqrt(s->sigma);
        *out = s->dim == 2 ? -or_bessel_k0(t) / (2.0 * OR_PI) : -exp(-t) / (4.0 * OR_PI * r);
    }
    return 0;
}
/* greensFreeGradient kernels.h:89-97 */
int or_greens_gradient(const bvc_kernel_spec* s, const double* x, const double* y, double* out) {
    int d = s->dim;
    double r = vdist(x, y, d);
    if (guard_radius(s, r)) return BVC_ERR_SINGULARITY;
    double r2 = r * r, q = screened_q(s, r);
    for (int i = 0; i < d; i++) {
        double p = d == 2 ? (x[i] - y[i]) / (2.0 * OR_PI * r2) : (x[i] - y[i]) / (4.0 * OR_PI * r2 * r);
        out[i] = q * p;
    }
    return 0;
}
/* poissonKernelFree kernels.h:100-108 */
int or_poisson_kernel(const bvc_kernel_spec* s, const double* x, const double* y, const double* n,
                      double* out) {
    int d = s->dim;
    double r = vdist(x, y, d);
    if (guard_radius(s, r)) return BVC_ERR_SINGULARITY;
    double ym[3]; for (int i = 0; i < d; i++) ym[i] = y[i] - x[i];
    double r2 = r * r;
    double p = d == 2 ? vdot(n, ym, d) / (2.0 * OR_PI * r2) : vdot(n, ym, d) / (4.0 * OR_PI * r2 * r);
    *out = screened_q(s, r) * p;
    return 0;
}
/* poissonKernelGradient kernels.h:111-129 */
int or_poisson_kernel_gradient(const bvc_kernel_spec* s, const double* x, const double* y,
                               const double* n, double* out) {
    int d = s->dim;
    double r = vdist(x, y, d);
    if (guard_radius(s, r)) return BVC_ERR_SINGULARITY;
    double ym[3]; for (int i = 0; i < d; i++) ym[i] = y[i] - x[i];
    double r2 = r * r, dot = vdot(n, ym, d), pv;
    double pg[3];
    if (d == 2) {
        for (int i = 0; i < 2; i++)
            pg[i] = 2.0 * dot / (2.0 * OR_PI * r2 * r2) * ym[i] - n[i] / (2.0 * OR_PI * r2);
        pv = dot / (2.0 * OR_PI * r2);
    } else {
        for (int i = 0; i < 3; i++)
            pg[i] = 3.0 * dot / (4.0 * OR_PI * r2 * r2 * r) * ym[i] - n[i] / (4.0 * OR_PI * r2 * r);
        pv = dot / (4.0 * OR_PI * r2 * r);
    }
    double q = screened_q(s, r), qp = screened_qprime(s, r);
    for (int i = 0; i < d; i++) out[i] = q * pg[i] + pv * qp * (x[i] - y[i]);
    return 0;
}
/* all four at once (mirror of bvc_eval_kernels): [G, dG/dx, dG/dn, d2G/dxdn] */
int or_eval_kernels(const bvc_kernel_spec* s, const double* x, const double* y, const double* n,
                    size_t count, double* out) {
    int d = s->dim, stride = 2 + 2 * d;
    for (size_t i = 0; i < count; i++) {
        const double *xi = x + d * i, *yi = y + d * i, *ni = n + d * i;
        double* o = out + stride * i;
        int e = or_greens(s, xi, yi, o);
        if (!e) e = or_greens_gradient(s, xi, yi, o + 1);
        if (!e) e = or_poisson_kernel(s, xi, yi, ni, o + 1 + d);
        if (!e) e = or_poisson_kernel_gradient(s, xi, yi, ni, o + 2 + d);
        if (e) return e;
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Ball kernels — kernels.cpp:31-107 (2D walks only need these)              */
/* ------------------------------------------------------------------------- */
double or_ball_greens(const bvc_kernel_spec* s, double R, double r) { /* kernels.cpp:31-43 */
    if (s->kind == BVC_KERNEL_POISSON)
        return s->dim == 2 ? log(r / R) / (2.0 * OR_PI) : (1.0 / R - 1.0 / r) / (4.0 * OR_PI);
    double q = sqrt(s->sigma);
    if (s->dim == 2) {
        double ratio = or_bessel_k0(R * q) / or_bessel_i0(R * q);
        return -(or_bessel_k0(r * q) - or_bessel_i0(r * q) * ratio) / (2.0 * OR_PI);
    }
    return -sinh((R - r) * q) / (4.0 * OR_PI * r * sinh(R * q));
}
double or_ball_sphere_weight(const bvc_kernel_spec* s, double R, double rHit) { /* kernels.cpp:55-66 */
    if (s->kind == BVC_KERNEL_POISSON) return 1.0;
    double q = sqrt(s->sigma);
    if (s->dim == 2) {
        double tR = R * q, tr = rHit * q;
        double i0 = or_bessel_i0(tR);
        if (!isfinite(i0)) return 0.0;
        return tr * (or_bessel_k1(tr) + or_bessel_i1(tr) * or_bessel_k0(tR) / i0);
    }
    double a = (R - rHit) * q;
    return (rHit * q * cosh(a) + sinh(a)) / sinh(R * q);
}
double or_ball_greens_mass(const bvc_kernel_spec* s, double R) { /* kernels.cpp:46-52 */
    if (s->kind == BVC_KERNEL_POISSON) return s->dim == 2 ? -R * R / 4.0 : -R * R / 6.0;
    double c = or_ball_sphere_weight(s, R, R);
    return (c - 1.0) / s->sigma;
}
static double invert_ball_radial_cdf(double u) { /* kernels.cpp:78-94 */
    if (u <= 0.0) return 1e-8;
    if (u >= 1.0) return 1.0;
    double lo = 0.0, hi = 1.0, t = sqrt(u);
    for (int it = 0; it < 100; it++) {
        double lt = log(t);
        double fv = t * t * (1.0 - 2.0 * lt) - u;
        if (fv > 0.0) hi = t; else lo = t;
        double deriv = -4.0 * t * lt;
        double step = deriv != 0.0 ? fv / deriv : 0.0;
        double next = t - step;
        if (!(next > lo && next < hi)) next = 0.5 * (lo + hi);
        if (fabs(next - t) < 1e-15) return next;
        t = next;
    }
    return t;
}
/* sampleBallGreens kernels.cpp:96-107 (2D Poisson ball) */
static void sample_ball_greens(double scale, const double* c, double R, or_rng* rng, double* p,
                               double* pdf) {
    bvc_kernel_spec ps = {BVC_KERNEL_POISSON, 0.0, 2, scale};
    double t = invert_ball_radial_cdf(rng_uniform(rng));
    double r = fmax(t * R, 1e-14 * R);
    double th = rng_uniform_ab(rng, 0.0, 2.0 * OR_PI);
    p[0] = c[0] + r * cos(th);
    p[1] = c[1] + r * sin(th);
    *pdf = or_ball_greens(&ps, R, r) / or_ball_greens_mass(&ps, R);
}
/* ballGreensGradient kernels.cpp:68-75 (Poisson) */
static void ball_greens_gradient2(const double* x, double R, const double* y, double* out) {
    double d0 = y[0] - x[0], d1 = y[1] - x[1];
    double r2 = d0 * d0 + d1 * d1;
    double f = (1.0 / (R * R) - 1.0 / r2) / (2.0 * OR_PI);
    out[0] = d0 * f; out[1] = d1 * f;
}

/* ------------------------------------------------------------------------- */
/* Fields — the device descriptor set (include/bvc_b200.h), evaluated in      */
/* double as the reference's std::function callbacks would (fields.cpp:30-72) */
/* ------------------------------------------------------------------------- */
double or_field_eval(const bvc_field* f, const double* p, int dim, int seg) {
    (void)seg;
    double x = p[0], y = p[1], z = dim == 3 ? p[2] : 0.0;
    const double* q = f->p;
    switch (f->kind) {
        case BVC_FIELD_NONE: return 0.0;
        case BVC_FIELD_CONSTANT: return q[0];
        case BVC_FIELD_LINEAR: return q[0] * x + q[1] * y + q[3] * z + q[2];
        case BVC_FIELD_RADIAL: {
            double dx = x - q[0], dy = y - q[1];
            return q[2] * pow(sqrt(dx * dx + dy * dy), q[3]) + q[4];
        }
        case BVC_FIELD_HARMONIC_POLY: { /* Re/Im of (x + iy)^d, fields.cpp:49-58 */
            int d = (int)q[0];
            double re = 1.0, im = 0.0;
            for (int k = 0; k < d; k++) { double t = re * x - im * y; im = re * y + im * x; re = t; }
            return q[1] * re + q[2] * im;
        }
        case BVC_FIELD_CHECKERBOARD: {
            long ix = (long)floor((x - q[0]) / q[2]), iy = (long)floor((y - q[1]) / q[2]);
            return ((ix + iy) & 1) == 0 ? q[3] : q[4];
        }
        case BVC_FIELD_SIN_COS: return q[0] * sin(q[1] * x + q[2]) * cos(q[3] * y + q[4]);
        case BVC_FIELD_GAUSSIAN_SUM: {
            double s = 0.0, inv = 1.0 / (2.0 * q[0] * q[0]);
            for (int m = 0; m < f->n; m++) {
                const double* t = q + 1 + 4 * m;
                double dx = x - t[0], dy = y - t[1], dz = z - t[2];
                s += t[3] * exp(-(dx * dx + dy * dy + dz * dz) * inv);
            }
            return s;
        }
        case BVC_FIELD_QUADRATIC3:
            return q[0] + q[1] * x + q[2] * y + q[3] * z + q[4] * x * x + q[5] * y * y +
                   q[6] * z * z + q[7] * x * y + q[8] * x * z + q[9] * y * z;
        case BVC_FIELD_TRIG3: return q[0] * sin(q[1] * x) + q[2] * cos(q[3] * y) + q[4] * z + q[5];
    }
    return 0.0;
}

/* ------------------------------------------------------------------------- */
/* 2D scene — Scene::build scene.cpp:11-125 and the brute-force query twins   */
/* (closestPointBrute 146-164, silhouetteDistanceBrute 187-194,               */
/*  intersectRayBrute 210-228, inside 240-254)                                */
/* ------------------------------------------------------------------------- */
typedef struct {
    int nv, ns;
    double* v;      /* 2*nv */
    int *a, *b, *label, *loop;
    double *nx, *ny, *len, *arc;
    int nsil;
    double *sil_p, *sil_n1, *sil_n2; /* 2*nsil each */
    int* sil_always;
    int* seg_sil;   /* 2*ns */
    int nloops;
    double* loop_len;
    int* loop_closed;
    double lo[2], hi[2], diagonal, dlen, nlen, tlen;
} or_scene;

void or_scene_free(or_scene* s) {
    if (!s) return;
    free(s->v); free(s->a); free(s->b); free(s->label); free(s->loop);
    free(s->nx); free(s->ny); free(s->len); free(s->arc);
    free(s->sil_p); free(s->sil_n1); free(s->sil_n2); free(s->sil_always); free(s->seg_sil);
    free(s->loop_len); free(s->loop_closed);
    free(s);
}

or_scene* or_scene_create(const double* v, int nv, const int* segs, const int* labels, int ns) {
    if (nv <= 0 || ns <= 0) return NULL;
    or_scene* s = (or_scene*)calloc(1, sizeof(or_scene));
    s->nv = nv; s->ns = ns;
    s->v = (double*)malloc(sizeof(double) * 2 * nv); memcpy(s->v, v, sizeof(double) * 2 * nv);
    s->a = (int*)malloc(sizeof(int) * ns); s->b = (int*)malloc(sizeof(int) * ns);
    s->label = (int*)malloc(sizeof(int) * ns); s->loop = (int*)malloc(sizeof(int) * ns);
    s->nx = (double*)malloc(sizeof(double) * ns); s->ny = (double*)malloc(sizeof(double) * ns);
    s->len = (double*)malloc(sizeof(double) * ns); s->arc = (double*)malloc(sizeof(double) * ns);
    s->lo[0] = s->lo[1] = OR_INF; s->hi[0] = s->hi[1] = -OR_INF;
    for (int i = 0; i < nv; i++) for (int k = 0; k < 2; k++) {
        s->lo[k] = fmin(s->lo[k], v[2 * i + k]); s->hi[k] = fmax(s->hi[k], v[2 * i + k]);
    }
    s->diagonal = hypot(s->hi[0] - s->lo[0], s->hi[1] - s->lo[1]);
    double floor_len = 1e-12 * fmax(s->diagonal, 1.0);
    for (int i = 0; i < ns; i++) { /* scene.cpp:22-38 */
        int a = segs[2 * i], b = segs[2 * i + 1];
        if (a < 0 || a >= nv || b < 0 || b >= nv) { or_scene_free(s); return NULL; }
        double dx = v[2 * b] - v[2 * a], dy = v[2 * b + 1] - v[2 * a + 1];
        double L = sqrt(dx * dx + dy * dy);
        if (L <= floor_len) { or_scene_free(s); return NULL; }
        s->a[i] = a; s->b[i] = b; s->label[i] = labels[i]; s->len[i] = L;
        s->nx[i] = dy / L; s->ny[i] = -dx / L; /* outwardNormal vec.h:21-23 */
        if (labels[i] == BVC_DIRICHLET) s->dlen += L; else s->nlen += L;
        s->tlen += L;
    }
    int *out_seg = (int*)malloc(sizeof(int) * nv), *in_seg = (int*)malloc(sizeof(int) * nv);
    for (int i = 0; i < nv; i++) out_seg[i] = in_seg[i] = -1;
    for (int i = 0; i < ns; i++) { /* scene.cpp:42-51 */
        if (out_seg[s->a[i]] >= 0 || in_seg[s->b[i]] >= 0) {
            free(out_seg); free(in_seg); or_scene_free(s); return NULL;
        }
        out_seg[s->a[i]] = i; in_seg[s->b[i]] = i;
    }
    /* loop tracing scene.cpp:54-83 */
    char* visited = (char*)calloc(ns, 1);
    s->loop_len = (double*)malloc(sizeof(double) * ns);
    s->loop_closed = (int*)malloc(sizeof(int) * ns);
    for (int pass = 0; pass < 2; pass++) {
        for (int i = 0; i < ns; i++) {
            if (visited[i] || (pass == 0 && in_seg[s->a[i]] >= 0)) continue;
            int id = s->nloops++, cur = i, closed = 0;
            double arc = 0.0;
            while (cur >= 0 && !visited[cur]) {
                visited[cur] = 1; s->loop[cur] = id; s->arc[cur] = arc; arc += s->len[cur];
                cur = out_seg[s->b[cur]];
                if (cur == i) { closed = 1; break; }
            }
            s->loop_len[id] = arc; s->loop_closed[id] = closed;
        }
    }
    free(visited);
    /* silhouette candidates scene.cpp:85-114 */
    s->seg_sil = (int*)malloc(sizeof(int) * 2 * ns);
    for (int i = 0; i < 2 * ns; i++) s->seg_sil[i] = -1;
    s->sil_p = (double*)malloc(sizeof(double) * 2 * nv);
    s->sil_n1 = (double*)malloc(sizeof(double) * 2 * nv);
    s->sil_n2 = (double*)malloc(sizeof(double) * 2 * nv);
    s->sil_always = (int*)malloc(sizeof(int) * nv);
    for (int vi = 0; vi < nv; vi++) {
        int sin_ = in_seg[vi], sout = out_seg[vi];
        int nin = sin_ >= 0 && s->label[sin_] == BVC_NEUMANN;
        int nout = sout >= 0 && s->label[sout] == BVC_NEUMANN;
        if (!nin && !nout) continue;
        int k = s->nsil, always = 0;
        double n1x = 0, n1y = 0, n2x = 0, n2y = 0;
        if (nin && nout) { n1x = s->nx[sin_]; n1y = s->ny[sin_]; n2x = s->nx[sout]; n2y = s->ny[sout]; }
        else if ((nin && sout < 0) || (nout && sin_ < 0)) always = 1;
        else continue;
        s->sil_p[2 * k] = v[2 * vi]; s->sil_p[2 * k + 1] = v[2 * vi + 1];
        s->sil_n1[2 * k] = n1x; s->sil_n1[2 * k + 1] = n1y;
        s->sil_n2[2 * k] = n2x; s->sil_n2[2 * k + 1] = n2y;
        s->sil_always[k] = always;
        s->nsil++;
        if (nin) { int* sl = s->seg_sil + 2 * sin_; if (sl[0] < 0) sl[0] = k; else sl[1] = k; }
        if (nout) { int* sl = s->seg_sil + 2 * sout; if (sl[0] < 0) sl[0] = k; else sl[1] = k; }
    }
    free(out_seg); free(in_seg);
    return s;
}

int or_scene_closed(const or_scene* s) { /* scene.cpp:127-131 */
    for (int i = 0; i < s->nloops; i++) if (!s->loop_closed[i]) return 0;
    return s->nloops > 0;
}
double or_scene_diagonal(const or_scene* s) { return s->diagonal; }
int or_scene_has_neumann(const or_scene* s) { return s->nlen > 0.0; }

static unsigned filter_mask(int f) { /* scene.h:22-28 */
    return f == BVC_FILTER_DIRICHLET ? 1u : f == BVC_FILTER_NEUMANN ? 2u : ~0u;
}
typedef struct { int valid; double p[2], dist, t; int seg; } or_cp;
/* closestPointBrute scene.cpp:146-164 with closestPointOnSegment bvh.h:153-159 */
static or_cp closest_point(const or_scene* s, const double* x, int filter) {
    or_cp r = {0, {0, 0}, OR_INF, 0.0, -1};
    unsigned mask = filter_mask(filter);
    for (int i = 0; i < s->ns; i++) {
        if (((1u << s->label[i]) & mask) == 0) continue;
        const double *a = s->v + 2 * s->a[i], *b = s->v + 2 * s->b[i];
        double ux = b[0] - a[0], uy = b[1] - a[1], l2 = ux * ux + uy * uy;
        double t = l2 > 0.0 ? ((x[0] - a[0]) * ux + (x[1] - a[1]) * uy) / l2 : 0.0;
        t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
        double px = a[0] + t * ux, py = a[1] + t * uy;
        double d = hypot(px - x[0], py - x[1]);
        if (d < r.dist) { r.valid = 1; r.p[0] = px; r.p[1] = py; r.dist = d; r.seg = i; r.t = t; }
    }
    return r;
}
void or_scene_closest_point(const or_scene* s, const double* x, size_t n, int filter,
                            double* point, double* dist, int* seg, double* t) {
    for (size_t i = 0; i < n; i++) {
        or_cp c = closest_point(s, x + 2 * i, filter);
        point[2 * i] = c.p[0]; point[2 * i + 1] = c.p[1];
        dist[i] = c.dist; seg[i] = c.valid ? c.seg : -1; t[i] = c.t;
    }
}
/* silhouetteTest scene.cpp:166-172 + silhouetteDistanceBrute 187-194 */
static double silhouette_distance(const or_scene* s, const double* x) {
    double best = OR_INF;
    for (int k = 0; k < s->nsil; k++) {
        const double* p = s->sil_p + 2 * k;
        double d = hypot(p[0] - x[0], p[1] - x[1]);
        if (!(d < best)) continue;
        int ok = s->sil_always[k];
        if (!ok) {
            double d1 = s->sil_n1[2 * k] * (p[0] - x[0]) + s->sil_n1[2 * k + 1] * (p[1] - x[1]);
            double d2 = s->sil_n2[2 * k] * (p[0] - x[0]) + s->sil_n2[2 * k + 1] * (p[1] - x[1]);
            ok = d1 * d2 <= 0.0;
        }
        if (ok) best = d;
    }
    return best;
}
void or_scene_silhouette_distance(const or_scene* s, const double* x, size_t n, double* out) {
    for (size_t i = 0; i < n; i++) out[i] = silhouette_distance(s, x + 2 * i);
}
/* raySegment bvh.cpp:71-83 */
static int ray_segment(const double* o, const double* d, const double* a, const double* b,
                       double tMax, double* t_out, double* s_out) {
    double ex = b[0] - a[0], ey = b[1] - a[1];
    double denom = d[0] * ey - d[1] * ex;
    if (fabs(denom) < 1e-300) return 0;
    double aox = a[0] - o[0], aoy = a[1] - o[1];
    double t = (aox * ey - aoy * ex) / denom;
    double s = (aox * d[1] - aoy * d[0]) / denom;
    if (t <= 0.0 || t > tMax || s < 0.0 || s > 1.0) return 0;
    *t_out = t; *s_out = s;
    return 1;
}
typedef struct { int hit; double t, s, p[2]; int seg; } or_hit;
/* intersectRayBrute scene.cpp:210-228 */
static or_hit intersect_ray(const or_scene* s, const double* o, const double* d, double tMax,
                            int filter, double tMin) {
    or_hit best = {0, OR_INF, 0.0, {0, 0}, -1};
    unsigned mask = filter_mask(filter);
    for (int i = 0; i < s->ns; i++) {
        if (((1u << s->label[i]) & mask) == 0) continue;
        double t, sp;
        if (ray_segment(o, d, s->v + 2 * s->a[i], s->v + 2 * s->b[i], tMax, &t, &sp) &&
            t > tMin && t < best.t) {
            best.hit = 1; best.t = t; best.s = sp; best.seg = i;
            best.p[0] = o[0] + t * d[0]; best.p[1] = o[1] + t * d[1];
        }
    }
    return best;
}
void or_scene_intersect_ray(const or_scene* s, const double* o, const double* d, size_t n,
                            double tMax, int filter, double tMin, double* t, int* seg,
                            double* point, double* sp) {
    for (size_t i = 0; i < n; i++) {
        or_hit h = intersect_ray(s, o + 2 * i, d + 2 * i, tMax, filter, tMin);
        t[i] = h.hit ? h.t : OR_INF; seg[i] = h.hit ? h.seg : -1;
        point[2 * i] = h.p[0]; point[2 * i + 1] = h.p[1]; sp[i] = h.s;
    }
}
/* inside scene.cpp:240-254 */
static int scene_inside(const or_scene* s, const double* x) {
    or_cp cp = closest_point(s, x, BVC_FILTER_ANY);
    if (cp.valid && cp.dist <= 1e-9 * s->diagonal) return 1;
    int in = 0;
    for (int i = 0; i < s->ns; i++) {
        const double *a = s->v + 2 * s->a[i], *b = s->v + 2 * s->b[i];
        if ((a[1] > x[1]) == (b[1] > x[1])) continue;
        double xc = a[0] + (x[1] - a[1]) / (b[1] - a[1]) * (b[0] - a[0]);
        if (x[0] < xc) in = !in;
    }
    return in;
}
void or_scene_inside(const or_scene* s, const double* x, size_t n, uint8_t* out) {
    for (size_t i = 0; i < n; i++) out[i] = (uint8_t)scene_inside(s, x + 2 * i);
}

/* ------------------------------------------------------------------------- */
/* Samplers — sampling.cpp:8-108                                             */
/* ------------------------------------------------------------------------- */
/* BoundarySampler::sample sampling.cpp:37-44 with fromUnit 20-35.
   out per sample: p(2), n(2), pdf, segment, arc */
int or_boundary_sample(const or_scene* s, int filter, int count, int stratified, uint64_t key,
                       int use_key, uint64_t seed, uint64_t stream, double* p, double* nrm,
                       double* pdf, int* seg, double* arc) {
    unsigned mask = filter_mask(filter);
    int* ids = (int*)malloc(sizeof(int) * s->ns);
    double* cdf = (double*)malloc(sizeof(double) * s->ns);
    int m = 0;
    double L = 0.0;
    for (int i = 0; i < s->ns; i++) {
        if (((1u << s->label[i]) & mask) == 0) continue;
        ids[m] = i; L += s->len[i]; cdf[m] = L; m++;
    }
    if (m == 0) { free(ids); free(cdf); return BVC_ERR_PARSE; }
    or_rng rng;
    if (use_key) rng_from_key(&rng, key); else rng_init(&rng, seed, stream);
    for (int k = 0; k < count; k++) {
        double u = stratified ? (k + rng_uniform(&rng)) / count : rng_uniform(&rng);
        double target = u * L;
        int lo = 0, hi = m; /* lower_bound */
        while (lo < hi) { int mid = (lo + hi) / 2; if (cdf[mid] < target) lo = mid + 1; else hi = mid; }
        int idx = lo >= m ? m - 1 : lo;
        int sid = ids[idx];
        double within = target - (idx > 0 ? cdf[idx - 1] : 0.0);
        double t = within / s->len[sid];
        t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
        const double *a = s->v + 2 * s->a[sid], *b = s->v + 2 * s->b[sid];
        p[2 * k] = a[0] + t * (b[0] - a[0]); p[2 * k + 1] = a[1] + t * (b[1] - a[1]);
        nrm[2 * k] = s->nx[sid]; nrm[2 * k + 1] = s->ny[sid];
        pdf[k] = 1.0 / L; seg[k] = sid; arc[k] = s->arc[sid] + t * s->len[sid];
    }
    free(ids); free(cdf);
    return 0;
}
/* loopArea sampling.cpp:46-54 */
double or_loop_area(const or_scene* s) {
    double area = 0.0;
    for (int i = 0; i < s->ns; i++) {
        const double *a = s->v + 2 * s->a[i], *b = s->v + 2 * s->b[i];
        area += 0.5 * (a[0] * b[1] - a[1] * b[0]);
    }
    return area;
}
/* RegionSampler::sample sampling.cpp:62-108 (stratified: shuffled jittered strata) */
int or_region_sample(const or_scene* s, int count, int stratified, uint64_t seed, uint64_t stream,
                     int use_key, uint64_t key, double* p, double* pdf) {
    double area = or_loop_area(s);
    if (!or_scene_closed(s) || area <= 0.0) return BVC_ERR_PARSE;
    or_rng rng;
    if (use_key) rng_from_key(&rng, key); else rng_init(&rng, seed, stream);
    double ex = s->hi[0] - s->lo[0], ey = s->hi[1] - s->lo[1], pd = 1.0 / area;
    long proposals = 0, accepted = 0;
    if (!stratified) {
        while (accepted < count) {
            proposals++;
            if (proposals >= 1000000 && accepted < proposals / 10000) return BVC_ERR_PARSE;
            /* Vector2(u*ex, u*ey): g++ evaluates the constructor arguments right to
               left, so the reference draws y first (sampling.cpp:86) */
            double q[2];
            q[1] = s->lo[1] + rng_uniform(&rng) * ey;
            q[0] = s->lo[0] + rng_uniform(&rng) * ex;
            if (scene_inside(s, q)) { p[2 * accepted] = q[0]; p[2 * accepted + 1] = q[1]; pdf[accepted] = pd; accepted++; }
        }
        return 0;
    }
    int g = (int)ceil(sqrt((double)count));
    if (g < 1) g = 1;
    int* order = (int*)malloc(sizeof(int) * (size_t)g * g);
    for (int i = 0; i < g * g; i++) order[i] = i;
    while (accepted < count) {
        for (size_t i = (size_t)g * g; i > 1; i--) {
            size_t j = rng_below(&rng, i);
            int tmp = order[i - 1]; order[i - 1] = order[j]; order[j] = tmp;
        }
        for (int c = 0; c < g * g; c++) {
            if (accepted >= count) break;
            proposals++;
            if (proposals >= 1000000 && accepted < proposals / 10000) { free(order); return BVC_ERR_PARSE; }
            int cx = order[c] % g, cy = order[c] / g;
            double q[2];
            q[1] = s->lo[1] + (cy + rng_uniform(&rng)) / g * ey; /* y first, as above */
            q[0] = s->lo[0] + (cx + rng_uniform(&rng)) / g * ex;
            if (scene_inside(s, q)) { p[2 * accepted] = q[0]; p[2 * accepted + 1] = q[1]; pdf[accepted] = pd; accepted++; }
        }
    }
    free(order);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Walks — pointwise.cpp:11-288                                              */
/* ------------------------------------------------------------------------- */
typedef struct {
    const or_scene* scene;
    const bvc_problem* problem;
    bvc_kernel_spec kernel, poisson;
    double eps, rmin, tguard;
    int max_steps, has_neumann, screened;
} or_ctx;

static int make_ctx(const or_scene* s, const bvc_problem* pb, const bvc_walk_config* c,
                    or_ctx* ctx) { /* makeContext pointwise.cpp:23-35 */
    if (pb->kernel.dim != 2) return BVC_ERR_SOLVER;
    ctx->scene = s; ctx->problem = pb;
    ctx->kernel = pb->kernel; ctx->kernel.scale = s->diagonal;
    bvc_kernel_spec ps = {BVC_KERNEL_POISSON, 0.0, 2, s->diagonal};
    ctx->poisson = ps;
    ctx->eps = c->epsilon > 0.0 ? c->epsilon : 1e-3 * s->diagonal; /* pointwise.h:36-38 */
    ctx->rmin = c->rMin > 0.0 ? c->rMin : ctx->eps;                /* pointwise.h:39-44 */
    if (ctx->rmin > ctx->eps) return BVC_ERR_INVALID_ARGUMENT;
    ctx->tguard = 1e-9 * s->diagonal;
    ctx->max_steps = c->maxSteps > 1 ? c->maxSteps : 1;
    ctx->has_neumann = s->nlen > 0.0;
    ctx->screened = pb->kernel.kind == BVC_KERNEL_SCREENED;
    return 0;
}
static double g_value(const or_ctx* c, const or_cp* cp) { /* pointwise.cpp:37-39 */
    return c->problem->g.kind != BVC_FIELD_NONE ? or_field_eval(&c->problem->g, cp->p, 2, cp->seg) : 0.0;
}
/* neumannTerm/clipNeumann pointwise.cpp:61-107 */
static double neumann_term(const or_ctx* c, const double* x, double R, or_rng* rng,
                           int* pseg, double* pt0, double* pt1, double* plen) {
    const or_scene* s = c->scene;
    int np = 0;
    double total = 0.0;
    for (int i = 0; i < s->ns; i++) {
        if (s->label[i] != BVC_NEUMANN) continue;
        const double *a = s->v + 2 * s->a[i], *b = s->v + 2 * s->b[i];
        double ux = b[0] - a[0], uy = b[1] - a[1], qx = a[0] - x[0], qy = a[1] - x[1];
        double A = ux * ux + uy * uy, B = 2.0 * (qx * ux + qy * uy), C = qx * qx + qy * qy - R * R;
        double disc = B * B - 4.0 * A * C;
        if (!(disc > 0.0) || A <= 0.0) continue;
        double sq = sqrt(disc);
        double t0 = fmax(0.0, (-B - sq) / (2.0 * A)), t1 = fmin(1.0, (-B + sq) / (2.0 * A));
        if (t1 <= t0) continue;
        double len = (t1 - t0) * s->len[i];
        pseg[np] = i; pt0[np] = t0; pt1[np] = t1; plen[np] = len; np++;
        total += len;
    }
    if (total <= 0.0) return 0.0;
    double target = rng_uniform(rng) * total, run = 0.0, local = 0.5;
    int ch = np - 1;
    for (int k = 0; k < np; k++) {
        if (target <= run + plen[k] || k == np - 1) {
            ch = k;
            local = (target - run) / plen[k];
            local = local < 0.0 ? 0.0 : (local > 1.0 ? 1.0 : local);
            break;
        }
        run += plen[k];
    }
    double t = pt0[ch] + (pt1[ch] - pt0[ch]) * local;
    int sid = pseg[ch];
    const double *a = s->v + 2 * s->a[sid], *b = s->v + 2 * s->b[sid];
    double y[2] = {a[0] + t * (b[0] - a[0]), a[1] + t * (b[1] - a[1])};
    double r = hypot(y[0] - x[0], y[1] - x[1]);
    double lo = 1e-12 * c->kernel.scale;
    r = r < lo ? lo : (r > R ? R : r);
    double hv = or_field_eval(&c->problem->h, y, 2, sid);
    return -or_ball_greens(&c->kernel, R, r) * hv * total;
}
/* sourceTerm pointwise.cpp:110-121 */
static double source_term(const or_ctx* c, const double* x, double R, or_rng* rng) {
    double y[2], pdf;
    sample_ball_greens(c->scene->diagonal, x, R, rng, y, &pdf);
    double fy = or_field_eval(&c->problem->f, y, 2, -1);
    if (fy == 0.0) return 0.0;
    if (c->has_neumann && !scene_inside(c->scene, y)) return 0.0;
    double contrib = fy * or_ball_greens_mass(&c->poisson, R);
    if (c->screened) {
        double r = hypot(y[0] - x[0], y[1] - x[1]);
        double lo = 1e-13 * c->kernel.scale;
        r = r < lo ? lo : (r > R ? R : r);
        contrib *= or_ball_greens(&c->kernel, R, r) / or_ball_greens(&c->poisson, R, r);
    }
    return contrib;
}
/* walkSampleImpl pointwise.cpp:125-165; *steps counts closest-Dirichlet queries */
static double walk_sample(const or_ctx* c, const double* x0, or_rng* rng, int* truncated,
                          long* steps, int* scratch_i, double* scratch_d) {
    double x[2] = {x0[0], x0[1]}, acc = 0.0, weight = 1.0, inward[2] = {0, 0};
    int on_neumann = 0;
    const or_scene* s = c->scene;
    for (int step = 0; step < c->max_steps; step++) {
        or_cp cpD = closest_point(s, x, BVC_FILTER_DIRICHLET);
        if (steps) (*steps)++;
        if (!cpD.valid) return NAN; /* SolverError: no Dirichlet boundary */
        if (cpD.dist <= c->eps) return acc + weight * g_value(c, &cpD);
        double R = cpD.dist;
        if (c->has_neumann) R = fmin(R, silhouette_distance(s, x));
        R = fmax(R, c->rmin);
        double factor = on_neumann ? 2.0 : 1.0;
        if (c->problem->f.kind != BVC_FIELD_NONE) acc += weight * factor * source_term(c, x, R, rng);
        if (c->has_neumann && c->problem->h.kind != BVC_FIELD_NONE)
            acc += weight * factor *
                   neumann_term(c, x, R, rng, scratch_i, scratch_d, scratch_d + s->ns, scratch_d + 2 * s->ns);
        double th; /* sampleDirection pointwise.cpp:42-49 */
        if (on_neumann) th = atan2(inward[1], inward[0]) + rng_uniform_ab(rng, -0.5 * OR_PI, 0.5 * OR_PI);
        else th = rng_uniform_ab(rng, 0.0, 2.0 * OR_PI);
        double d[2] = {cos(th), sin(th)};
        double travel = R;
        or_hit hit = {0};
        if (c->has_neumann) hit = intersect_ray(s, x, d, R, BVC_FILTER_NEUMANN, c->tguard);
        if (hit.hit) {
            x[0] = hit.p[0]; x[1] = hit.p[1];
            travel = hit.t;
            double nx = s->nx[hit.seg], ny = s->ny[hit.seg];
            if (nx * d[0] + ny * d[1] > 0.0) { inward[0] = -nx; inward[1] = -ny; }
            else { inward[0] = nx; inward[1] = ny; }
            on_neumann = 1;
        } else {
            x[0] += R * d[0]; x[1] += R * d[1];
            on_neumann = 0;
        }
        if (c->screened) weight *= or_ball_sphere_weight(&c->kernel, R, travel);
    }
    *truncated = 1;
    or_cp cp = closest_point(s, x, BVC_FILTER_DIRICHLET);
    return acc + weight * g_value(c, &cp);
}
/* gradientSample pointwise.cpp:195-215 */
static void gradient_sample(const or_ctx* c, const double* x, double R, or_rng* rng, int* trunc,
                            long* steps, int* si, double* sd, double* v) {
    double th = rng_uniform_ab(rng, 0.0, 2.0 * OR_PI);
    double dir[2] = {cos(th), sin(th)};
    double z[2] = {x[0] + R * dir[0], x[1] + R * dir[1]};
    double uz = walk_sample(c, z, rng, trunc, steps, si, sd);
    v[0] = (2.0 / R) * uz * dir[0];
    v[1] = (2.0 / R) * uz * dir[1];
    if (c->problem->f.kind != BVC_FIELD_NONE) {
        double y[2], pdf, g[2];
        sample_ball_greens(c->scene->diagonal, x, R, rng, y, &pdf);
        double fy = or_field_eval(&c->problem->f, y, 2, -1);
        if (fy != 0.0) {
            ball_greens_gradient2(x, R, y, g);
            v[0] += g[0] * (fy / pdf); v[1] += g[1] * (fy / pdf);
        }
    }
    if (c->screened && c->kernel.sigma > 0.0) {
        double y[2], pdf, g[2];
        sample_ball_greens(c->scene->diagonal, x, R, rng, y, &pdf);
        double uy = walk_sample(c, y, rng, trunc, steps, si, sd);
        ball_greens_gradient2(x, R, y, g);
        v[0] += g[0] * (c->kernel.sigma * uy / pdf);
        v[1] += g[1] * (c->kernel.sigma * uy / pdf);
    }
}

/* runWalks pointwise.cpp:167-186 / wostSolve 233-238 (requireInterior 188-191).
   kind: 0 = wos (rejects Neumann scenes), 1 = wost. out: mean, se, count, truncated, steps */
int or_solve(const or_scene* s, const bvc_problem* pb, const double* x, const bvc_walk_config* cfg,
             int kind, double* out) {
    if (kind == 0 && s->nlen > 0.0) return BVC_ERR_SOLVER;
    or_ctx c;
    int e = make_ctx(s, pb, cfg, &c);
    if (e) return e;
    if (or_scene_closed(s) && !scene_inside(s, x)) return BVC_ERR_SOLVER;
    int n = cfg->nWalks > 1 ? cfg->nWalks : 1;
    int* si = (int*)malloc(sizeof(int) * s->ns);
    double* sd = (double*)malloc(sizeof(double) * 3 * s->ns);
    double sum = 0.0, sq = 0.0;
    long trunc = 0, steps = 0;
    for (int k = 0; k < n; k++) {
        or_rng rng; rng_init(&rng, cfg->seed, or_mixkey(cfg->stream, (uint64_t)k));
        int t = 0;
        double v = walk_sample(&c, x, &rng, &t, &steps, si, sd);
        if (isnan(v)) { free(si); free(sd); return BVC_ERR_SOLVER; }
        sum += v; sq += v * v; trunc += t;
    }
    free(si); free(sd);
    double mean = sum / n, var = fmax(0.0, sq / n - mean * mean);
    out[0] = mean; out[1] = n > 1 ? sqrt(var / (n - 1)) : 0.0;
    out[2] = n; out[3] = (double)trunc; out[4] = (double)steps;
    return 0;
}
/* gradientBallRadius 217-221 + wostGradient 240-263 (normal == NULL) or
   wostNormalDerivative 265-288. out: mean[2], se[2], count, truncated, steps (gradient) or
   mean, se, count, truncated, steps (normal derivative) */
int or_gradient(const or_scene* s, const bvc_problem* pb, const double* x, const double* normal,
                const bvc_walk_config* cfg, double* out) {
    or_ctx c;
    int e = make_ctx(s, pb, cfg, &c);
    if (e) return e;
    if (or_scene_closed(s) && !scene_inside(s, x)) return BVC_ERR_SOLVER;
    or_cp cp = closest_point(s, x, BVC_FILTER_ANY);
    if (!cp.valid) return BVC_ERR_SOLVER;
    double R = fmax(cp.dist, c.rmin);
    int n = cfg->nWalks > 1 ? cfg->nWalks : 1;
    int* si = (int*)malloc(sizeof(int) * s->ns);
    double* sd = (double*)malloc(sizeof(double) * 3 * s->ns);
    double sum[2] = {0, 0}, sq[2] = {0, 0};
    long trunc = 0, steps = 0;
    for (int k = 0; k < n; k++) {
        or_rng rng; rng_init(&rng, cfg->seed, or_mixkey(cfg->stream, (uint64_t)k));
        int t = 0;
        double v[2];
        gradient_sample(&c, x, R, &rng, &t, &steps, si, sd, v);
        if (normal) { v[0] = normal[0] * v[0] + normal[1] * v[1]; v[1] = 0.0; }
        for (int i = 0; i < 2; i++) { sum[i] += v[i]; sq[i] += v[i] * v[i]; }
        trunc += t;
    }
    free(si); free(sd);
    if (normal) {
        double mean = sum[0] / n, var = fmax(0.0, sq[0] / n - mean * mean);
        out[0] = mean; out[1] = n > 1 ? sqrt(var / (n - 1)) : 0.0;
        out[2] = n; out[3] = (double)trunc; out[4] = (double)steps;
    } else {
        for (int i = 0; i < 2; i++) {
            double mean = sum[i] / n, var = fmax(0.0, sq[i] / n - mean * mean);
            out[i] = mean; out[2 + i] = n > 1 ? sqrt(var / (n - 1)) : 0.0;
        }
        out[4] = n; out[5] = (double)trunc; out[6] = (double)steps;
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* generateBoundaryCache cache.cpp:301-390 (region given as a scene + kinds)  */
/* out per sample: z(2), n(2), pdf, uHat, dHat, segment, arc. stats[0..2]:     */
/* resampled, cacheWalks, cacheTruncated; stats[3] = steps (not in reference)  */
/* ------------------------------------------------------------------------- */
int or_generate_boundary_cache(const or_scene* scene, const bvc_problem* pb,
                               const or_scene* region, const int* kinds, const int* source_seg,
                               const bvc_cache_config* cfg, uint64_t seed, uint64_t round,
                               int begin, int end, double* z, double* nrm, double* pdf,
                               double* uhat, double* dhat, int* seg, double* arc, long* stats) {
    int N = cfg->nBoundary > 1 ? cfg->nBoundary : 1;
    double* p = (double*)malloc(sizeof(double) * 2 * N);
    double* nn = (double*)malloc(sizeof(double) * 2 * N);
    double* pd = (double*)malloc(sizeof(double) * N);
    int* sg = (int*)malloc(sizeof(int) * N);
    double* ar = (double*)malloc(sizeof(double) * N);
    /* positions: Rng(seed, mixKey(0x1001, round)) cache.cpp:309-311 */
    int e = or_boundary_sample(region, BVC_FILTER_ANY, N, cfg->stratified, 0, 0, seed,
                               or_mixkey(0x1001, round), p, nn, pd, sg, ar);
    if (e) goto done;
    double eps = cfg->walk.epsilon > 0.0 ? cfg->walk.epsilon : 1e-3 * scene->diagonal;
    if (end > N || end <= 0) end = N;
    for (int i = begin; i < end; i++) {
        int o = i - begin;
        uint64_t tag = or_mixkey(or_mixkey(0x1002, round), (uint64_t)i); /* cache.cpp:361 */
        z[2 * o] = p[2 * i]; z[2 * o + 1] = p[2 * i + 1];
        nrm[2 * o] = nn[2 * i]; nrm[2 * o + 1] = nn[2 * i + 1];
        pdf[o] = pd[i]; seg[o] = sg[i]; arc[o] = ar[i];
        bvc_walk_config wc = cfg->walk;
        wc.seed = seed;
        double r[7];
        if (kinds[sg[i]] == BVC_SEG_KNOWN_NEUMANN) { /* cache.cpp:329-339 */
            int src = source_seg[sg[i]];
            dhat[o] = pb->h.kind != BVC_FIELD_NONE ? or_field_eval(&pb->h, p + 2 * i, 2, src) : 0.0;
            wc.nWalks = cfg->nWalksNeumann;
            wc.stream = or_mixkey(tag, 1);
            double x[2] = {p[2 * i] - 0.5 * eps * nn[2 * i], p[2 * i + 1] - 0.5 * eps * nn[2 * i + 1]};
            e = or_solve(scene, pb, x, &wc, 1, r);
            if (e) goto done; /* the reference redraws; the oracle reports */
            uhat[o] = r[0]; stats[1] += (long)r[2]; stats[2] += (long)r[3]; stats[3] += (long)r[4];
        } else { /* cache.cpp:341-352 */
            wc.nWalks = cfg->nWalksNeumann;
            wc.stream = or_mixkey(tag, 1);
            e = or_solve(scene, pb, p + 2 * i, &wc, 1, r);
            if (e) goto done;
            uhat[o] = r[0]; stats[1] += (long)r[2]; stats[2] += (long)r[3]; stats[3] += (long)r[4];
            wc.nWalks = cfg->nWalksDirichlet;
            wc.stream = or_mixkey(tag, 2);
            e = or_gradient(scene, pb, p + 2 * i, nn + 2 * i, &wc, r);
            if (e) goto done;
            dhat[o] = r[0]; stats[1] += (long)r[2]; stats[2] += (long)r[3]; stats[3] += (long)r[4];
        }
    }
done:
    free(p); free(nn); free(pd); free(sg); free(ar);
    return e;
}

/* generateSourceCache cache.cpp:392-406: y(2), pdf, f */
int or_generate_source_cache(const bvc_problem* pb, const or_scene* region,
                             const bvc_cache_config* cfg, uint64_t seed, uint64_t round,
                             double* y, double* pdf, double* f) {
    int M = cfg->nSource > 1 ? cfg->nSource : 1;
    int e = or_region_sample(region, M, cfg->stratified, seed, or_mixkey(0x1004, round), 0, 0, y, pdf);
    if (e) return e;
    for (int i = 0; i < M; i++) f[i] = or_field_eval(&pb->f, y + 2 * i, 2, -1);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Splats — splatSolution cache.cpp:426-461 and splatGradient 463-497, for    */
/* 2D and 3D (the 3D loop restates the same code with the reference's own 3D */
/* kernel templates, kernels.h:78-129; there is no reference 3D splat path).  */
/* Arrays: bz/bn dim*N, bpdf/bu/bd/bw N; sy dim*M, spdf/sf M; px dim*K;        */
/* sums accumulate (+=) like the reference.                                    */
/* ------------------------------------------------------------------------- */
int or_splat(const bvc_kernel_spec* spec, double coincidence_tol, int voronoi, int N,
             const double* bz, const double* bn, const double* bpdf, const double* bu,
             const double* bd, const double* bw, int M, const double* sy, const double* spdf,
             const double* sf, size_t K, const double* px, const uint8_t* fallback, int value,
             int gradient, double* bsum, double* ssum, long long* nb, long long* ms,
             double* bgsum, double* sgsum, long long* nbg, long long* msg, long long* skipped) {
    int d = spec->dim;
    for (size_t k = 0; k < K; k++) {
        if (fallback && fallback[k]) continue; /* cache.cpp:431 */
        const double* x = px + d * k;
        if (value) {
            double b = 0.0, s = 0.0;
            long long bn_ = 0, mn = 0, skip = 0;
            for (int i = 0; i < N; i++) {
                if (vdist(x, bz + d * i, d) < coincidence_tol) { skip++; continue; }
                double P, G;
                int e = or_poisson_kernel(spec, x, bz + d * i, bn + d * i, &P);
                if (!e) e = or_greens(spec, x, bz + d * i, &G);
                if (e) return e;
                double val = P * bu[i] - G * bd[i];
                b += voronoi ? val * bw[i] * N : val / bpdf[i];
                bn_++;
            }
            for (int j = 0; j < M; j++) {
                if (vdist(x, sy + d * j, d) < coincidence_tol) { skip++; continue; }
                double G;
                int e = or_greens(spec, x, sy + d * j, &G);
                if (e) return e;
                s += G * sf[j] / spdf[j];
                mn++;
            }
            bsum[k] += b; nb[k] += bn_; ssum[k] += s; ms[k] += mn; skipped[k] += skip;
        }
        if (gradient) {
            double b[3] = {0, 0, 0}, s[3] = {0, 0, 0};
            long long bn_ = 0, mn = 0, skip = 0;
            for (int i = 0; i < N; i++) {
                if (vdist(x, bz + d * i, d) < coincidence_tol) { skip++; continue; }
                double PG[3], GG[3];
                int e = or_poisson_kernel_gradient(spec, x, bz + d * i, bn + d * i, PG);
                if (!e) e = or_greens_gradient(spec, x, bz + d * i, GG);
                if (e) return e;
                for (int c = 0; c < d; c++) {
                    double val = PG[c] * bu[i] - GG[c] * bd[i];
                    b[c] += voronoi ? val * bw[i] * N : val / bpdf[i];
                }
                bn_++;
            }
            for (int j = 0; j < M; j++) {
                if (vdist(x, sy + d * j, d) < coincidence_tol) { skip++; continue; }
                double GG[3];
                int e = or_greens_gradient(spec, x, sy + d * j, GG);
                if (e) return e;
                for (int c = 0; c < d; c++) s[c] += GG[c] * (sf[j] / spdf[j]);
                mn++;
            }
            for (int c = 0; c < d; c++) { bgsum[d * k + c] += b[c]; sgsum[d * k + c] += s[c]; }
            nbg[k] += bn_; msg[k] += mn; skipped[k] += skip;
        }
    }
    return 0;
}

/* The clamped and ball-kernel splat loops, value only, 2D (mode bits as the GPU's
   gather.cu SplatMode):
     1  dG/dn clamped to [-c, c]  correctedBoundarySplat cache.cpp:512-524 (kernels.h:52)
     2  G -> G^B(x, R_x)           greensValue cache.cpp:410-416 (ballGreens kernels.cpp:31-43)
     4  source G^B clamped         correctedSourceSplat cache.cpp:573-582
   The sampled correction terms (cache.cpp:526-550, 584-592) are random and are
   checked statistically against closed forms instead. */
int or_clamped_splat(const bvc_kernel_spec* spec, double tol, int voronoi, int N, const double* bz,
                     const double* bn, const double* bpdf, const double* bu, const double* bd,
                     const double* bw, int M, const double* sy, const double* spdf, const double* sf,
                     size_t K, const double* px, const uint8_t* fallback, int mode, double clamp,
                     const double* ballR, double* bsum, double* ssum, long long* nb, long long* ms,
                     long long* skipped) {
    if (spec->dim != 2) return 1;
    bvc_kernel_spec ball = {BVC_KERNEL_POISSON, 0.0, 2, spec->scale};
    for (size_t k = 0; k < K; k++) {
        if (fallback && fallback[k]) continue;
        const double* x = px + 2 * k;
        double R = ballR ? ballR[k] : 0.0;
        if ((mode & 6) && !(R > 0.0)) return 2; /* requireBallRadius cache.cpp:418-423 */
        double b = 0.0, s = 0.0;
        long long bn_ = 0, mn = 0, skip = 0;
        for (int i = 0; i < N; i++) {
            double r = vdist(x, bz + 2 * i, 2);
            if (r < tol) { skip++; continue; }
            double P, G;
            int e = or_poisson_kernel(spec, x, bz + 2 * i, bn + 2 * i, &P);
            if (e) return e;
            if (mode & 1) P = fmax(-clamp, fmin(clamp, P));
            if (mode & 2) G = or_ball_greens(&ball, R, fmin(r, R));
            else if ((e = or_greens(spec, x, bz + 2 * i, &G))) return e;
            double val = P * bu[i] - G * bd[i];
            b += voronoi ? val * bw[i] * N : val / bpdf[i];
            bn_++;
        }
        for (int j = 0; j < M; j++) {
            double r = vdist(x, sy + 2 * j, 2);
            if (r < tol) { skip++; continue; }
            double G;
            if (mode & 2) {
                G = or_ball_greens(&ball, R, fmin(r, R));
                if (mode & 4) G = fmax(-clamp, fmin(clamp, G));
            } else {
                int e = or_greens(spec, x, sy + 2 * j, &G);
                if (e) return e;
            }
            s += G * sf[j] / spdf[j];
            mn++;
        }
        bsum[k] += b; nb[k] += bn_; ssum[k] += s; ms[k] += mn; skipped[k] += skip;
    }
    return 0;
}
