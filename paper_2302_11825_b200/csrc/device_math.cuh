// device_math.cuh — FP32 device math for the BVC hot path on sm_100a.
//
//  * Philox4x32-10 counter-based RNG (the north star replaces the reference's
//    xoshiro256++ streams, rng.h:21-59; walk parity is therefore statistical).
//  * FP32 modified Bessel functions I0/I1/K0/K1 (replacing std::cyl_bessel_k/i
//    of kernels.cpp:7-29) from the Abramowitz & Stegun 9.8.1-9.8.8 polynomial
//    fits, with exponentially scaled variants for the ball kernels.
//  * device-evaluable field descriptors (replacing the std::function callbacks of
//    PdeProblem, pointwise.h:19-26; names follow tools/src/fields.cpp:30-72).
#pragma once
#include <cstdint>
#include <cstring>

#ifndef BVC_HD
#define BVC_HD __host__ __device__ __forceinline__
#endif

namespace bvc_dev {

constexpr float kPi = 3.14159265358979323846f;
constexpr float kTwoPi = 6.28318530717958647692f;
constexpr float kInv2Pi = 0.15915494309189533577f;
constexpr float kInv4Pi = 0.07957747154594766788f;
constexpr float kLn2 = 0.69314718055994530942f;

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11). counter (x,y,z,w), key (x,y)
// ---------------------------------------------------------------------------
BVC_HD void mulhilo32(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
#ifdef __CUDA_ARCH__
    lo = a * b;
    hi = __umulhi(a, b);
#else
    uint64_t p = static_cast<uint64_t>(a) * b;
    lo = static_cast<uint32_t>(p);
    hi = static_cast<uint32_t>(p >> 32);
#endif
}

struct U4 { uint32_t x, y, z, w; };

BVC_HD U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0, lo0, hi1, lo1;
        mulhilo32(0xD2511F53u, c.x, hi0, lo0);
        mulhilo32(0xCD9E8D57u, c.z, hi1, lo1);
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// uniform in [0, 1) from the top 24 bits
BVC_HD float u01(uint32_t v) { return static_cast<float>(v >> 8) * 5.9604644775390625e-8f; }

// SplitMix64 mixing (the reference's rng.h:8-18), used only to derive Philox keys
BVC_HD uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
BVC_HD uint64_t mixKey(uint64_t key, uint64_t counter) {
    return mix64(key ^ (counter + 0x9e3779b97f4a7c15ull));
}

// float <-> int bit casts usable on both sides (node links stored in float slots)
BVC_HD int float_bits(float f) {
#ifdef __CUDA_ARCH__
    return __float_as_int(f);
#else
    int i;
    std::memcpy(&i, &f, sizeof i);
    return i;
#endif
}
BVC_HD float bits_float(int i) {
#ifdef __CUDA_ARCH__
    return __int_as_float(i);
#else
    float f;
    std::memcpy(&f, &i, sizeof f);
    return f;
#endif
}

// ---------------------------------------------------------------------------
// fast SFU wrappers
// ---------------------------------------------------------------------------
#ifdef __CUDA_ARCH__
__device__ __forceinline__ float f_lg2(float x) { float y; asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float f_ex2(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float f_rcp(float x) { float y; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float f_rsq(float x) { float y; asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
#else
inline float f_lg2(float x) { return std::log2(x); }
inline float f_ex2(float x) { return std::exp2(x); }
inline float f_rcp(float x) { return 1.0f / x; }
inline float f_rsq(float x) { return 1.0f / std::sqrt(x); }
#endif
// packed FP32 pairs (sm_100a FFMA2 / FMUL2 / FADD2): one instruction, two lanes,
// each lane rounded exactly like the scalar FFMA / FMUL / FADD
struct F2 {
    unsigned long long v;
};
__device__ __forceinline__ F2 pk(float lo, float hi) {
    F2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ F2 bc(float x) { return pk(x, x); }
__device__ __forceinline__ void upk(F2 a, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a.v)); }
__device__ __forceinline__ F2 add2(F2 a, F2 b) { F2 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v)); return r; }
__device__ __forceinline__ F2 sub2(F2 a, F2 b) { F2 r; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v)); return r; }
__device__ __forceinline__ F2 mul2(F2 a, F2 b) { F2 r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v)); return r; }
__device__ __forceinline__ F2 fma2(F2 a, F2 b, F2 c) {
    F2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
    return r;
}
template <class Fn>
__device__ __forceinline__ F2 each(F2 a, Fn&& f) {
    float lo, hi;
    upk(a, lo, hi);
    return pk(f(lo), f(hi));
}
BVC_HD float f_ln(float x) { return f_lg2(x) * kLn2; }
BVC_HD float f_exp(float x) { return f_ex2(x * 1.44269504088896340736f); }

// ---------------------------------------------------------------------------
// Bessel functions, FP32 (A&S 9.8.1-9.8.8; |rel err| ~< 3e-7)
// "e" variants are exponentially scaled: I0e = e^-t I0, K0e = e^t K0.
// ---------------------------------------------------------------------------
BVC_HD float bessel_i0_small(float t) {  // |t| <= 3.75
    float y = t * (1.0f / 3.75f); y *= y;
    return 1.0f + y * (3.5156229f + y * (3.0899424f + y * (1.2067492f + y * (0.2659732f + y * (0.0360768f + y * 0.0045813f)))));
}
BVC_HD float bessel_i1_small(float t) {  // |t| <= 3.75, returns I1
    float y = t * (1.0f / 3.75f); y *= y;
    return t * (0.5f + y * (0.87890594f + y * (0.51498869f + y * (0.15084934f + y * (0.02658733f + y * (0.00301532f + y * 0.00032411f))))));
}
BVC_HD float bessel_i0e_large(float t) {  // t >= 3.75: e^-t I0(t)
    float y = 3.75f * f_rcp(t);
    float p = 0.39894228f + y * (0.01328592f + y * (0.00225319f + y * (-0.00157565f + y * (0.00916281f + y * (-0.02057706f + y * (0.02635537f + y * (-0.01647633f + y * 0.00392377f)))))));
    return p * f_rsq(t);
}
BVC_HD float bessel_i1e_large(float t) {  // t >= 3.75: e^-t I1(t)
    float y = 3.75f * f_rcp(t);
    float p = 0.39894228f + y * (-0.03988024f + y * (-0.00362018f + y * (0.00163801f + y * (-0.01031555f + y * (0.02282967f + y * (-0.02895312f + y * (0.01787654f - y * 0.00420059f)))))));
    return p * f_rsq(t);
}
BVC_HD float bessel_i0e(float t) { return t <= 3.75f ? bessel_i0_small(t) * f_exp(-t) : bessel_i0e_large(t); }
BVC_HD float bessel_i1e(float t) { return t <= 3.75f ? bessel_i1_small(t) * f_exp(-t) : bessel_i1e_large(t); }
BVC_HD float bessel_i0(float t) { return t <= 3.75f ? bessel_i0_small(t) : bessel_i0e_large(t) * f_exp(t); }
BVC_HD float bessel_i1(float t) { return t <= 3.75f ? bessel_i1_small(t) : bessel_i1e_large(t) * f_exp(t); }

// K0 on (0, 2]
BVC_HD float bessel_k0_small(float t) {
    float h = 0.5f * t, y = h * h;
    float p = -0.57721566f + y * (0.42278420f + y * (0.23069756f + y * (0.03488590f + y * (0.00262698f + y * (0.00010750f + y * 0.0000074f)))));
    return -f_ln(h) * bessel_i0_small(t) + p;
}
// t K1 on (0, 2]
BVC_HD float bessel_tk1_small(float t) {
    float h = 0.5f * t, y = h * h;
    float p = 1.0f + y * (0.15443144f + y * (-0.67278579f + y * (-0.18156897f + y * (-0.01919402f + y * (-0.00110404f - y * 0.00004686f)))));
    return t * f_ln(h) * bessel_i1_small(t) + p;
}
// sqrt(t) e^t K0(t) and sqrt(t) e^t K1(t) on [2, inf)
BVC_HD float bessel_k0_large_poly(float t) {
    float y = 2.0f * f_rcp(t);
    return 1.25331414f + y * (-0.07832358f + y * (0.02189568f + y * (-0.01062446f + y * (0.00587872f + y * (-0.00251540f + y * 0.00053208f)))));
}
BVC_HD float bessel_k1_large_poly(float t) {
    float y = 2.0f * f_rcp(t);
    return 1.25331414f + y * (0.23498619f + y * (-0.03655620f + y * (0.01504268f + y * (-0.00780353f + y * (0.00325614f - y * 0.00068245f)))));
}
BVC_HD float bessel_k0(float t) {
    return t <= 2.0f ? bessel_k0_small(t) : bessel_k0_large_poly(t) * f_rsq(t) * f_exp(-t);
}
BVC_HD float bessel_k1(float t) {
    return t <= 2.0f ? bessel_tk1_small(t) * f_rcp(t) : bessel_k1_large_poly(t) * f_rsq(t) * f_exp(-t);
}
BVC_HD float bessel_k0e(float t) {  // e^t K0(t)
    return t <= 2.0f ? bessel_k0_small(t) * f_exp(t) : bessel_k0_large_poly(t) * f_rsq(t);
}
BVC_HD float bessel_k1e(float t) {
    return t <= 2.0f ? bessel_tk1_small(t) * f_rcp(t) * f_exp(t) : bessel_k1_large_poly(t) * f_rsq(t);
}

// ---------------------------------------------------------------------------
// field descriptors (bvc_field in include/bvc_b200.h), evaluated in FP32
// ---------------------------------------------------------------------------
constexpr int kFieldMaxParams = 68;
struct DevField {
    int kind;
    int n;
    float p[kFieldMaxParams];
};

BVC_HD float field_eval(const DevField& f, float x, float y, float z = 0.0f) {
    const float* q = f.p;
    switch (f.kind) {
        case 0: return 0.0f;
        case 1: return q[0];
        case 2: return q[0] * x + q[1] * y + q[3] * z + q[2];
        case 3: {
            float dx = x - q[0], dy = y - q[1];
            float r = sqrtf(dx * dx + dy * dy);
            return q[2] * powf(r, q[3]) + q[4];
        }
        case 4: {
            int d = static_cast<int>(q[0]);
            float re = 1.0f, im = 0.0f;
            for (int k = 0; k < d; ++k) { float t = re * x - im * y; im = re * y + im * x; re = t; }
            return q[1] * re + q[2] * im;
        }
        case 5: {
            long ix = static_cast<long>(floorf((x - q[0]) / q[2]));
            long iy = static_cast<long>(floorf((y - q[1]) / q[2]));
            return ((ix + iy) & 1) == 0 ? q[3] : q[4];
        }
        case 6: return q[0] * sinf(q[1] * x + q[2]) * cosf(q[3] * y + q[4]);
        case 7: {
            float s = 0.0f, inv = 1.0f / (2.0f * q[0] * q[0]);
            for (int m = 0; m < f.n; ++m) {
                const float* t = q + 1 + 4 * m;
                float dx = x - t[0], dy = y - t[1], dz = z - t[2];
                s += t[3] * expf(-(dx * dx + dy * dy + dz * dz) * inv);
            }
            return s;
        }
        case 8:
            return q[0] + q[1] * x + q[2] * y + q[3] * z + q[4] * x * x + q[5] * y * y + q[6] * z * z +
                   q[7] * x * y + q[8] * x * z + q[9] * y * z;
        case 9: return q[0] * sinf(q[1] * x) + q[2] * cosf(q[3] * y) + q[4] * z + q[5];
    }
    return 0.0f;
}

}  // namespace bvc_dev
