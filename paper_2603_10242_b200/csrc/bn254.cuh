// BN254 field arithmetic for sm_100a: 8 x 32-bit limbs (little-endian),
// Montgomery form (R = 2^256), CIOS multiplication as PTX carry chains
// (mad.lo.cc / madc.hi.cc on the IMAD pipe). Fq = base field p, Fr = scalar
// field r. The reference has no BN254 code;
// parity is against the from-scratch CPU oracle (oracle/bn254_oracle.c).
//
// Bounds: both moduli are < 2^254, so the CIOS accumulator stays < 2p + p*2^32
// < 2^288 (nine limbs, no tenth) and results are fully reduced to [0, m).
#pragma once
#include <cstdint>

namespace ace_gpu {
namespace bn {

struct FqCfg {
    static constexpr uint32_t M[8] = {0xd87cfd47u, 0x3c208c16u, 0x6871ca8du, 0x97816a91u,
                                      0x8181585du, 0xb85045b6u, 0xe131a029u, 0x30644e72u};
    static constexpr uint32_t ONE[8] = {0xc58f0d9du, 0xd35d438du, 0xf5c70b3du, 0x0a78eb28u,
                                        0x7879462cu, 0x666ea36fu, 0x9a07df2fu, 0x0e0a77c1u};
    static constexpr uint32_t R2[8] = {0x538afa89u, 0xf32cfc5bu, 0xd44501fbu, 0xb5e71911u,
                                       0x0a417ff6u, 0x47ab1effu, 0xcab8351fu, 0x06d89f71u};
    static constexpr uint32_t N0 = 0xe4866389u;
};

struct FrCfg {
    static constexpr uint32_t M[8] = {0xf0000001u, 0x43e1f593u, 0x79b97091u, 0x2833e848u,
                                      0x8181585du, 0xb85045b6u, 0xe131a029u, 0x30644e72u};
    static constexpr uint32_t ONE[8] = {0x4ffffffbu, 0xac96341cu, 0x9f60cd29u, 0x36fc7695u,
                                        0x7879462eu, 0x666ea36fu, 0x9a07df2fu, 0x0e0a77c1u};
    static constexpr uint32_t R2[8] = {0xae216da7u, 0x1bb8e645u, 0xe35c59e3u, 0x53fe3ab1u,
                                       0x53bb8085u, 0x8c49833du, 0x7f4e44a5u, 0x0216d0b1u};
    static constexpr uint32_t N0 = 0xefffffffu;
};

// Limb accessors usable in device code with run-time indices (a static
// constexpr member array may not be odr-used on the device).
template <class C>
__device__ __forceinline__ uint32_t mod_limb(int i) {
    constexpr uint32_t a[8] = {C::M[0], C::M[1], C::M[2], C::M[3],
                               C::M[4], C::M[5], C::M[6], C::M[7]};
    return a[i];
}
template <class C>
__device__ __forceinline__ uint32_t one_limb(int i) {
    constexpr uint32_t a[8] = {C::ONE[0], C::ONE[1], C::ONE[2], C::ONE[3],
                               C::ONE[4], C::ONE[5], C::ONE[6], C::ONE[7]};
    return a[i];
}
template <class C>
__device__ __forceinline__ uint32_t r2_limb(int i) {
    constexpr uint32_t a[8] = {C::R2[0], C::R2[1], C::R2[2], C::R2[3],
                               C::R2[4], C::R2[5], C::R2[6], C::R2[7]};
    return a[i];
}

template <class C>
struct Fp {
    uint32_t v[8];

    __device__ __forceinline__ static Fp zero() {
        Fp r;
#pragma unroll
        for (int i = 0; i < 8; ++i) r.v[i] = 0;
        return r;
    }
    __device__ __forceinline__ static Fp one() {
        Fp r;
#pragma unroll
        for (int i = 0; i < 8; ++i) r.v[i] = one_limb<C>(i);
        return r;
    }
    __device__ __forceinline__ bool is_zero() const {
        uint32_t x = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) x |= v[i];
        return x == 0;
    }
    __device__ __forceinline__ bool operator==(const Fp& o) const {
        uint32_t x = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) x |= v[i] ^ o.v[i];
        return x == 0;
    }
};

using Fq = Fp<FqCfg>;
using Fr = Fp<FrCfg>;

// t (9 limbs) -> t - m if t >= m (t < 2m guaranteed).
template <class C>
__device__ __forceinline__ void final_sub(uint32_t t[9], uint32_t r[8]) {
    uint32_t s[8], br;
    asm("sub.cc.u32  %0, %9,  %17;\n\t"
        "subc.cc.u32 %1, %10, %18;\n\t"
        "subc.cc.u32 %2, %11, %19;\n\t"
        "subc.cc.u32 %3, %12, %20;\n\t"
        "subc.cc.u32 %4, %13, %21;\n\t"
        "subc.cc.u32 %5, %14, %22;\n\t"
        "subc.cc.u32 %6, %15, %23;\n\t"
        "subc.cc.u32 %7, %16, %24;\n\t"
        "subc.u32    %8, %25, 0;"
        : "=r"(s[0]), "=r"(s[1]), "=r"(s[2]), "=r"(s[3]), "=r"(s[4]), "=r"(s[5]), "=r"(s[6]),
          "=r"(s[7]), "=r"(br)
        : "r"(t[0]), "r"(t[1]), "r"(t[2]), "r"(t[3]), "r"(t[4]), "r"(t[5]), "r"(t[6]), "r"(t[7]),
          "n"(C::M[0]), "n"(C::M[1]), "n"(C::M[2]), "n"(C::M[3]), "n"(C::M[4]), "n"(C::M[5]),
          "n"(C::M[6]), "n"(C::M[7]), "r"(t[8]));
    // br == 0xffffffff iff t < m (borrow out of the 9-limb subtraction)
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = br ? t[i] : s[i];
}

// CIOS Montgomery multiplication: r = a * b * 2^-256 mod m.
template <class C>
__device__ __forceinline__ Fp<C> mul_cios(const Fp<C>& a, const Fp<C>& b) {
    uint32_t t0 = 0, t1 = 0, t2 = 0, t3 = 0, t4 = 0, t5 = 0, t6 = 0, t7 = 0, t8 = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t bi = b.v[i];
        // t += a * b_i : low halves into t0..t7 (carry into t8 = 0), high halves into t1..t8.
        asm("mad.lo.cc.u32  %0, %9,  %17, %0;\n\t"
            "madc.lo.cc.u32 %1, %10, %17, %1;\n\t"
            "madc.lo.cc.u32 %2, %11, %17, %2;\n\t"
            "madc.lo.cc.u32 %3, %12, %17, %3;\n\t"
            "madc.lo.cc.u32 %4, %13, %17, %4;\n\t"
            "madc.lo.cc.u32 %5, %14, %17, %5;\n\t"
            "madc.lo.cc.u32 %6, %15, %17, %6;\n\t"
            "madc.lo.cc.u32 %7, %16, %17, %7;\n\t"
            "addc.u32       %8, 0, 0;"
            : "+r"(t0), "+r"(t1), "+r"(t2), "+r"(t3), "+r"(t4), "+r"(t5), "+r"(t6), "+r"(t7),
              "=r"(t8)
            : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]),
              "r"(a.v[6]), "r"(a.v[7]), "r"(bi));
        asm("mad.hi.cc.u32  %0, %8,  %16, %0;\n\t"
            "madc.hi.cc.u32 %1, %9,  %16, %1;\n\t"
            "madc.hi.cc.u32 %2, %10, %16, %2;\n\t"
            "madc.hi.cc.u32 %3, %11, %16, %3;\n\t"
            "madc.hi.cc.u32 %4, %12, %16, %4;\n\t"
            "madc.hi.cc.u32 %5, %13, %16, %5;\n\t"
            "madc.hi.cc.u32 %6, %14, %16, %6;\n\t"
            "madc.hi.u32    %7, %15, %16, %7;"
            : "+r"(t1), "+r"(t2), "+r"(t3), "+r"(t4), "+r"(t5), "+r"(t6), "+r"(t7), "+r"(t8)
            : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]),
              "r"(a.v[6]), "r"(a.v[7]), "r"(bi));
        const uint32_t m = t0 * C::N0;
        // t += m * M, then t >>= 32 (t0 becomes 0 and is dropped).
        asm("mad.lo.cc.u32  %0, %9,  %10, %0;\n\t"
            "madc.lo.cc.u32 %1, %9,  %11, %1;\n\t"
            "madc.lo.cc.u32 %2, %9,  %12, %2;\n\t"
            "madc.lo.cc.u32 %3, %9,  %13, %3;\n\t"
            "madc.lo.cc.u32 %4, %9,  %14, %4;\n\t"
            "madc.lo.cc.u32 %5, %9,  %15, %5;\n\t"
            "madc.lo.cc.u32 %6, %9,  %16, %6;\n\t"
            "madc.lo.cc.u32 %7, %9,  %17, %7;\n\t"
            "addc.u32       %8, %8, 0;"
            : "+r"(t0), "+r"(t1), "+r"(t2), "+r"(t3), "+r"(t4), "+r"(t5), "+r"(t6), "+r"(t7),
              "+r"(t8)
            : "r"(m), "n"(C::M[0]), "n"(C::M[1]), "n"(C::M[2]), "n"(C::M[3]), "n"(C::M[4]),
              "n"(C::M[5]), "n"(C::M[6]), "n"(C::M[7]));
        asm("mad.hi.cc.u32  %0, %8,  %9,  %0;\n\t"
            "madc.hi.cc.u32 %1, %8,  %10, %1;\n\t"
            "madc.hi.cc.u32 %2, %8,  %11, %2;\n\t"
            "madc.hi.cc.u32 %3, %8,  %12, %3;\n\t"
            "madc.hi.cc.u32 %4, %8,  %13, %4;\n\t"
            "madc.hi.cc.u32 %5, %8,  %14, %5;\n\t"
            "madc.hi.cc.u32 %6, %8,  %15, %6;\n\t"
            "madc.hi.u32    %7, %8,  %16, %7;"
            : "+r"(t1), "+r"(t2), "+r"(t3), "+r"(t4), "+r"(t5), "+r"(t6), "+r"(t7), "+r"(t8)
            : "r"(m), "n"(C::M[0]), "n"(C::M[1]), "n"(C::M[2]), "n"(C::M[3]), "n"(C::M[4]),
              "n"(C::M[5]), "n"(C::M[6]), "n"(C::M[7]));
        t0 = t1; t1 = t2; t2 = t3; t3 = t4; t4 = t5; t5 = t6; t6 = t7; t7 = t8; t8 = 0;
    }
    uint32_t t[9] = {t0, t1, t2, t3, t4, t5, t6, t7, t8};
    Fp<C> r;
    final_sub<C>(t, r.v);
    return r;
}

// ---- FP64 (DFMA) Montgomery product ----------------------------------------
// On sm_100a IMAD, IMAD.HI and DFMA share one issue pipe: IMAD costs 2
// cycles per warp, IMAD.HI 4, IMAD.WIDE 6, DFMA 2 (tools/int_pipes.cu). A
// 32x32-bit product (lo + hi) therefore costs 6 pipe cycles for 1,024 bits^2
// while a 52x52-bit DFMA split (3 FP64 ops) costs 6 for 2,704: the product
// below does the multiplications in FP64 and the column sums on the integer
// ALU pipe. Radix 2^52, 5 limbs, R' = 2^260, used as a drop-in for the
// R = 2^256 product: MM'(16a, b) = a b 2^-256 mod m, bit-identical results.
// Split of x*y (x, y < 2^52): t = fma_rz(x, y, 2^104) = 2^104 + hi 2^52,
// s = (2^104 + 2^52) - t (exact), l = fma(x, y, s) = 2^52 + lo; hi and lo
// are the low mantissa bits of t and l, accumulated as raw bit patterns in
// 64-bit columns that start from minus the exponent bits they will collect.
namespace f64 {
constexpr uint64_t kM52 = (1ull << 52) - 1;
constexpr uint64_t kB52 = 0x4330000000000000ull;   // bits(2^52)
constexpr uint64_t kB104 = 0x4670000000000000ull;  // bits(2^104)
constexpr double kC1 = 20282409603651670423947251286016.0;                       // 2^104
constexpr double kC2 = 20282409603651670423947251286016.0 + 4503599627370496.0;  // + 2^52
constexpr double kT52 = 4503599627370496.0;                                      // 2^52
template <class C>
constexpr uint64_t limb52(int k) {  // bits [52k, 52k + 52) of the modulus
    uint64_t r = 0;
    for (int b = 0; b < 52; ++b) {
        const int i = 52 * k + b;
        if (i < 256 && ((C::M[i >> 5] >> (i & 31)) & 1)) r |= 1ull << b;
    }
    return r;
}
template <class C>
constexpr uint64_t nprime52() {  // -m^-1 mod 2^52 (Newton)
    const uint64_t m0 = (uint64_t)C::M[0] | ((uint64_t)C::M[1] << 32);
    uint64_t x = m0;  // correct to 3 bits
    for (int i = 0; i < 5; ++i) x *= 2 - m0 * x;
    return (0ull - x) & kM52;
}
// column bias: minus the exponent bits of the lo / hi patterns column k collects
constexpr uint64_t bias(int k) {
    uint64_t s = 0;
    for (int i = 0; i < 5; ++i)
        for (int j = 0; j < 5; ++j) {
            if (i + j == k) s += kB52;      // a_i b_j lo
            if (i + j + 1 == k) s += kB104;  // a_i b_j hi
            if (j > 0 && i + j == k) s += kB52;  // m_i p_j lo (j = 0: carried, not added)
            if (i + j + 1 == k) s += kB104;      // m_i p_j hi
        }
    return 0ull - s;
}
__device__ __forceinline__ uint64_t bits(double x) { return (uint64_t)__double_as_longlong(x); }
__device__ __forceinline__ double to_d(uint64_t x52) {  // exact for x < 2^52
    return __dsub_rn(__longlong_as_double((long long)(x52 | kB52)), kT52);
}
__device__ __forceinline__ void split_acc(double x, double y, uint64_t& clo, uint64_t& chi) {
    const double t = __fma_rz(x, y, kC1);
    const double l = __fma_rn(x, y, __dsub_rn(kC2, t));
    clo += bits(l);
    chi += bits(t);
}
// 8 x 32-bit limbs -> 5 x 52-bit doubles of (a << SH); a << SH < 2^260
template <int SH>
__device__ __forceinline__ void to52(const uint32_t v[8], double d[5]) {
    const uint64_t w0 = ((uint64_t)v[1] << 32) | v[0], w1 = ((uint64_t)v[3] << 32) | v[2],
                   w2 = ((uint64_t)v[5] << 32) | v[4], w3 = ((uint64_t)v[7] << 32) | v[6];
    d[0] = to_d((w0 << SH) & kM52);
    d[1] = to_d(((w0 >> (52 - SH)) | (w1 << (12 + SH))) & kM52);
    d[2] = to_d(((w1 >> (40 - SH)) | (w2 << (24 + SH))) & kM52);
    d[3] = to_d(((w2 >> (28 - SH)) | (w3 << (36 + SH))) & kM52);
    d[4] = to_d((w3 >> (16 - SH)) & kM52);
}
}  // namespace f64

// r = a b 2^-256 mod m (a, b < m), fully reduced: identical to mul().
template <class C>
__device__ __forceinline__ Fp<C> mul_f64(const Fp<C>& a, const Fp<C>& b) {
    using namespace f64;
    double x[5], y[5];
    to52<4>(a.v, x);
    to52<0>(b.v, y);
    uint64_t c[10];
#pragma unroll
    for (int k = 0; k < 10; ++k) c[k] = bias(k);
#pragma unroll
    for (int i = 0; i < 5; ++i)
#pragma unroll
        for (int j = 0; j < 5; ++j) split_acc(x[i], y[j], c[i + j], c[i + j + 1]);
    constexpr double NP = (double)nprime52<C>();
    constexpr double P[5] = {(double)limb52<C>(0), (double)limb52<C>(1), (double)limb52<C>(2),
                             (double)limb52<C>(3), (double)limb52<C>(4)};
    uint64_t carry = 0;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const uint64_t s = c[i] + carry;
        const uint64_t v = s & kM52;
        carry = (s >> 52) + (v != 0);  // v + lo(m p_0) is 0 or 2^52
        const double vd = to_d(v);
        const double t = __fma_rz(vd, NP, kC1);
        const double md = __dsub_rn(__fma_rn(vd, NP, __dsub_rn(kC2, t)), kT52);  // lo52(v n')
        c[i + 1] += bits(__fma_rz(md, P[0], kC1));
#pragma unroll
        for (int j = 1; j < 5; ++j) split_acc(md, P[j], c[i + j], c[i + j + 1]);
    }
    uint64_t r[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const uint64_t s = c[5 + k] + carry;
        r[k] = s & kM52;
        carry = s >> 52;
    }
    // result < 2^255: r[4] < 2^47, no carry out
    const uint64_t w0 = r[0] | (r[1] << 52), w1 = (r[1] >> 12) | (r[2] << 40),
                   w2 = (r[2] >> 24) | (r[3] << 28), w3 = (r[3] >> 36) | (r[4] << 16);
    uint32_t t9[9] = {(uint32_t)w0, (uint32_t)(w0 >> 32), (uint32_t)w1, (uint32_t)(w1 >> 32),
                      (uint32_t)w2, (uint32_t)(w2 >> 32), (uint32_t)w3, (uint32_t)(w3 >> 32), 0u};
    Fp<C> out;
    final_sub<C>(t9, out.v);
    return out;
}

#ifndef ACEGPU_F64MUL
#define ACEGPU_F64MUL 1  // 0: every mul() through the IMAD CIOS product (mul_cios)
#endif
template <class C>
__device__ __forceinline__ Fp<C> mul(const Fp<C>& a, const Fp<C>& b) {
    if constexpr (ACEGPU_F64MUL) return mul_f64(a, b);
    else return mul_cios(a, b);
}

// ---- lazy reduction in the FP64 domain ------------------------------------
// W10: a 520-bit value X = sum_k c[k] 2^(52 k) as ten SIGNED 64-bit columns
// (not normalised), holding 16 a b of the product (the R' = 2^260 scaling of
// mul_f64), so sums and differences of products are column-wise integer adds
// and one redc10 per output does the Montgomery reduction: X 2^-260 mod m =
// (a b + ...) 2^-256, the R = 2^256 Montgomery form of the rest of the code.
// Column magnitudes stay below 2^60 (sums of at most a few dozen 52-bit parts).
struct W10 {
    int64_t c[10];
};
namespace f64 {
constexpr uint64_t bias_ab(int k) {  // exponent bits the 25 products leave in column k
    uint64_t s = 0;
    for (int i = 0; i < 5; ++i)
        for (int j = 0; j < 5; ++j) {
            if (i + j == k) s += kB52;
            if (i + j + 1 == k) s += kB104;
        }
    return 0ull - s;
}
constexpr uint64_t bias_red(int k) {  // ... and the reduction's 5 x (1 + 4 x 2) parts
    uint64_t s = 0;
    for (int i = 0; i < 5; ++i)
        for (int j = 0; j < 5; ++j) {
            if (j > 0 && i + j == k) s += kB52;
            if (i + j + 1 == k) s += kB104;
        }
    return 0ull - s;
}
}  // namespace f64

// w = 16 a b as true column values (a < 2^256, b < 2^256).
template <class C>
__device__ __forceinline__ void mul_wide10(const Fp<C>& a, const Fp<C>& b, W10& w) {
    using namespace f64;
    double x[5], y[5];
    to52<4>(a.v, x);
    to52<0>(b.v, y);
    uint64_t c[10];
#pragma unroll
    for (int k = 0; k < 10; ++k) c[k] = bias_ab(k);
#pragma unroll
    for (int i = 0; i < 5; ++i)
#pragma unroll
        for (int j = 0; j < 5; ++j) split_acc(x[i], y[j], c[i + j], c[i + j + 1]);
#pragma unroll
    for (int k = 0; k < 10; ++k) w.c[k] = (int64_t)c[k];
}
__device__ __forceinline__ void w10_sub(W10& w, const W10& o) {
#pragma unroll
    for (int k = 0; k < 10; ++k) w.c[k] -= o.c[k];
}
__device__ __forceinline__ void w10_add(W10& w, const W10& o) {
#pragma unroll
    for (int k = 0; k < 10; ++k) w.c[k] += o.c[k];
}
__device__ __forceinline__ void w10_shl1(W10& w) {
#pragma unroll
    for (int k = 0; k < 10; ++k) w.c[k] *= 2;
}
// w += m 2^260 (m's 52-bit limbs in columns 5..9): lifts a difference of
// products |X| < m 2^260 into [0, 2 m 2^260)
template <class C>
__device__ __forceinline__ void w10_add_m260(W10& w) {
    // compile-time limbs (C::M may not be read on the device at run time)
    constexpr int64_t L[5] = {(int64_t)f64::limb52<C>(0), (int64_t)f64::limb52<C>(1),
                              (int64_t)f64::limb52<C>(2), (int64_t)f64::limb52<C>(3),
                              (int64_t)f64::limb52<C>(4)};
#pragma unroll
    for (int k = 0; k < 5; ++k) w.c[5 + k] += L[k];
}
// X 2^-260 mod m for 0 <= X < 2 m 2^260, fully reduced (result < 3m before
// the two conditional subtractions).
template <class C>
__device__ __forceinline__ Fp<C> redc10(const W10& w) {
    using namespace f64;
    constexpr double NP = (double)nprime52<C>();
    constexpr double P[5] = {(double)limb52<C>(0), (double)limb52<C>(1), (double)limb52<C>(2),
                             (double)limb52<C>(3), (double)limb52<C>(4)};
    uint64_t c[10];
#pragma unroll
    for (int k = 0; k < 10; ++k) c[k] = (uint64_t)w.c[k] + bias_red(k);
    int64_t carry = 0;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const int64_t s = (int64_t)c[i] + carry;  // column i is complete (true value)
        const uint64_t v = (uint64_t)s & kM52;
        carry = (s >> 52) + (v != 0);
        const double vd = to_d(v);
        const double t = __fma_rz(vd, NP, kC1);
        const double md = __dsub_rn(__fma_rn(vd, NP, __dsub_rn(kC2, t)), kT52);
        c[i + 1] += bits(__fma_rz(md, P[0], kC1));
#pragma unroll
        for (int j = 1; j < 5; ++j) split_acc(md, P[j], c[i + j], c[i + j + 1]);
    }
    uint64_t r[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int64_t s = (int64_t)c[5 + k] + carry;
        r[k] = (uint64_t)s & kM52;
        carry = s >> 52;
    }
    // value < 3 m < 2^256: r[4] < 2^48
    const uint64_t w0 = r[0] | (r[1] << 52), w1 = (r[1] >> 12) | (r[2] << 40),
                   w2 = (r[2] >> 24) | (r[3] << 28), w3 = (r[3] >> 36) | (r[4] << 16);
    uint32_t t9[9] = {(uint32_t)w0, (uint32_t)(w0 >> 32), (uint32_t)w1, (uint32_t)(w1 >> 32),
                      (uint32_t)w2, (uint32_t)(w2 >> 32), (uint32_t)w3, (uint32_t)(w3 >> 32), 0u};
    Fp<C> o1, out;
    final_sub<C>(t9, o1.v);  // < 2m
    uint32_t u9[9];
#pragma unroll
    for (int i = 0; i < 8; ++i) u9[i] = o1.v[i];
    u9[8] = 0;
    final_sub<C>(u9, out.v);  // < m
    return out;
}

// ---- lazy reduction: 512-bit products, one Montgomery reduction per sum ----
// A Montgomery product is half schoolbook product (128 IMAD) and half
// reduction (136). Sums/differences of products (Karatsuba Fq2, x*y - z*w)
// are formed on the 512-bit products and reduced once.

// w = a * b (16 limbs). a, b < 2^256 (unreduced sums of two elements are fine).
template <class C>
__device__ __forceinline__ void mul_wide(const Fp<C>& a, const Fp<C>& b, uint32_t w[16]) {
    uint32_t t0 = 0, t1 = 0, t2 = 0, t3 = 0, t4 = 0, t5 = 0, t6 = 0, t7 = 0, t8 = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t bi = b.v[i];
        asm("mad.lo.cc.u32  %0, %9,  %17, %0;\n\t"
            "madc.lo.cc.u32 %1, %10, %17, %1;\n\t"
            "madc.lo.cc.u32 %2, %11, %17, %2;\n\t"
            "madc.lo.cc.u32 %3, %12, %17, %3;\n\t"
            "madc.lo.cc.u32 %4, %13, %17, %4;\n\t"
            "madc.lo.cc.u32 %5, %14, %17, %5;\n\t"
            "madc.lo.cc.u32 %6, %15, %17, %6;\n\t"
            "madc.lo.cc.u32 %7, %16, %17, %7;\n\t"
            "addc.u32       %8, %8, 0;"
            : "+r"(t0), "+r"(t1), "+r"(t2), "+r"(t3), "+r"(t4), "+r"(t5), "+r"(t6), "+r"(t7),
              "+r"(t8)
            : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]),
              "r"(a.v[6]), "r"(a.v[7]), "r"(bi));
        asm("mad.hi.cc.u32  %0, %8,  %16, %0;\n\t"
            "madc.hi.cc.u32 %1, %9,  %16, %1;\n\t"
            "madc.hi.cc.u32 %2, %10, %16, %2;\n\t"
            "madc.hi.cc.u32 %3, %11, %16, %3;\n\t"
            "madc.hi.cc.u32 %4, %12, %16, %4;\n\t"
            "madc.hi.cc.u32 %5, %13, %16, %5;\n\t"
            "madc.hi.cc.u32 %6, %14, %16, %6;\n\t"
            "madc.hi.u32    %7, %15, %16, %7;"
            : "+r"(t1), "+r"(t2), "+r"(t3), "+r"(t4), "+r"(t5), "+r"(t6), "+r"(t7), "+r"(t8)
            : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]),
              "r"(a.v[6]), "r"(a.v[7]), "r"(bi));
        w[i] = t0;  // final: later rows start one limb higher
        t0 = t1; t1 = t2; t2 = t3; t3 = t4; t4 = t5; t5 = t6; t6 = t7; t7 = t8; t8 = 0;
    }
    w[8] = t0; w[9] = t1; w[10] = t2; w[11] = t3;
    w[12] = t4; w[13] = t5; w[14] = t6; w[15] = t7;
}

// w = a^2 (16 limbs): 28 off-diagonal products (lo + hi), doubled by a
// funnel shift, plus the 8 diagonal squares: 72 IMAD instead of 128.
template <class C>
__device__ __forceinline__ void sqr_wide(const Fp<C>& x, uint32_t t[16]) {
    const uint32_t* a = x.v;
#pragma unroll
    for (int k = 0; k < 16; ++k) t[k] = 0;
    asm("mad.lo.cc.u32  %0, %8, %9, %0;\n\t"
        "madc.lo.cc.u32 %1, %8, %10, %1;\n\t"
        "madc.lo.cc.u32 %2, %8, %11, %2;\n\t"
        "madc.lo.cc.u32 %3, %8, %12, %3;\n\t"
        "madc.lo.cc.u32 %4, %8, %13, %4;\n\t"
        "madc.lo.cc.u32 %5, %8, %14, %5;\n\t"
        "madc.lo.cc.u32 %6, %8, %15, %6;\n\t"
        "addc.u32       %7, %7, 0;"
        : "+r"(t[1]), "+r"(t[2]), "+r"(t[3]), "+r"(t[4]), "+r"(t[5]), "+r"(t[6]), "+r"(t[7]), "+r"(t[8])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
    asm("mad.hi.cc.u32  %0, %7, %8, %0;\n\t"
        "madc.hi.cc.u32 %1, %7, %9, %1;\n\t"
        "madc.hi.cc.u32 %2, %7, %10, %2;\n\t"
        "madc.hi.cc.u32 %3, %7, %11, %3;\n\t"
        "madc.hi.cc.u32 %4, %7, %12, %4;\n\t"
        "madc.hi.cc.u32 %5, %7, %13, %5;\n\t"
        "madc.hi.u32    %6, %7, %14, %6;"
        : "+r"(t[2]), "+r"(t[3]), "+r"(t[4]), "+r"(t[5]), "+r"(t[6]), "+r"(t[7]), "+r"(t[8])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
    asm("mad.lo.cc.u32  %0, %7, %8, %0;\n\t"
        "madc.lo.cc.u32 %1, %7, %9, %1;\n\t"
        "madc.lo.cc.u32 %2, %7, %10, %2;\n\t"
        "madc.lo.cc.u32 %3, %7, %11, %3;\n\t"
        "madc.lo.cc.u32 %4, %7, %12, %4;\n\t"
        "madc.lo.cc.u32 %5, %7, %13, %5;\n\t"
        "addc.u32       %6, %6, 0;"
        : "+r"(t[3]), "+r"(t[4]), "+r"(t[5]), "+r"(t[6]), "+r"(t[7]), "+r"(t[8]), "+r"(t[9])
        : "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
    asm("mad.hi.cc.u32  %0, %6, %7, %0;\n\t"
        "madc.hi.cc.u32 %1, %6, %8, %1;\n\t"
        "madc.hi.cc.u32 %2, %6, %9, %2;\n\t"
        "madc.hi.cc.u32 %3, %6, %10, %3;\n\t"
        "madc.hi.cc.u32 %4, %6, %11, %4;\n\t"
        "madc.hi.u32    %5, %6, %12, %5;"
        : "+r"(t[4]), "+r"(t[5]), "+r"(t[6]), "+r"(t[7]), "+r"(t[8]), "+r"(t[9])
        : "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
    asm("mad.lo.cc.u32  %0, %6, %7, %0;\n\t"
        "madc.lo.cc.u32 %1, %6, %8, %1;\n\t"
        "madc.lo.cc.u32 %2, %6, %9, %2;\n\t"
        "madc.lo.cc.u32 %3, %6, %10, %3;\n\t"
        "madc.lo.cc.u32 %4, %6, %11, %4;\n\t"
        "addc.u32       %5, %5, 0;"
        : "+r"(t[5]), "+r"(t[6]), "+r"(t[7]), "+r"(t[8]), "+r"(t[9]), "+r"(t[10])
        : "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
    asm("mad.hi.cc.u32  %0, %5, %6, %0;\n\t"
        "madc.hi.cc.u32 %1, %5, %7, %1;\n\t"
        "madc.hi.cc.u32 %2, %5, %8, %2;\n\t"
        "madc.hi.cc.u32 %3, %5, %9, %3;\n\t"
        "madc.hi.u32    %4, %5, %10, %4;"
        : "+r"(t[6]), "+r"(t[7]), "+r"(t[8]), "+r"(t[9]), "+r"(t[10])
        : "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
    asm("mad.lo.cc.u32  %0, %5, %6, %0;\n\t"
        "madc.lo.cc.u32 %1, %5, %7, %1;\n\t"
        "madc.lo.cc.u32 %2, %5, %8, %2;\n\t"
        "madc.lo.cc.u32 %3, %5, %9, %3;\n\t"
        "addc.u32       %4, %4, 0;"
        : "+r"(t[7]), "+r"(t[8]), "+r"(t[9]), "+r"(t[10]), "+r"(t[11])
        : "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
    asm("mad.hi.cc.u32  %0, %4, %5, %0;\n\t"
        "madc.hi.cc.u32 %1, %4, %6, %1;\n\t"
        "madc.hi.cc.u32 %2, %4, %7, %2;\n\t"
        "madc.hi.u32    %3, %4, %8, %3;"
        : "+r"(t[8]), "+r"(t[9]), "+r"(t[10]), "+r"(t[11])
        : "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
    asm("mad.lo.cc.u32  %0, %4, %5, %0;\n\t"
        "madc.lo.cc.u32 %1, %4, %6, %1;\n\t"
        "madc.lo.cc.u32 %2, %4, %7, %2;\n\t"
        "addc.u32       %3, %3, 0;"
        : "+r"(t[9]), "+r"(t[10]), "+r"(t[11]), "+r"(t[12])
        : "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
    asm("mad.hi.cc.u32  %0, %3, %4, %0;\n\t"
        "madc.hi.cc.u32 %1, %3, %5, %1;\n\t"
        "madc.hi.u32    %2, %3, %6, %2;"
        : "+r"(t[10]), "+r"(t[11]), "+r"(t[12])
        : "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
    asm("mad.lo.cc.u32  %0, %3, %4, %0;\n\t"
        "madc.lo.cc.u32 %1, %3, %5, %1;\n\t"
        "addc.u32       %2, %2, 0;"
        : "+r"(t[11]), "+r"(t[12]), "+r"(t[13])
        : "r"(a[5]), "r"(a[6]), "r"(a[7]));
    asm("mad.hi.cc.u32  %0, %2, %3, %0;\n\t"
        "madc.hi.u32    %1, %2, %4, %1;"
        : "+r"(t[12]), "+r"(t[13])
        : "r"(a[5]), "r"(a[6]), "r"(a[7]));
    asm("mad.lo.cc.u32  %0, %2, %3, %0;\n\t"
        "addc.u32       %1, %1, 0;"
        : "+r"(t[13]), "+r"(t[14])
        : "r"(a[6]), "r"(a[7]));
    asm("mad.hi.u32     %0, %1, %2, %0;"
        : "+r"(t[14])
        : "r"(a[6]), "r"(a[7]));
#pragma unroll
    for (int k = 15; k > 0; --k) t[k] = __funnelshift_l(t[k - 1], t[k], 1);
    t[0] <<= 1;
    asm("mad.lo.cc.u32  %0, %16, %16, %0;\n\t"
        "madc.hi.cc.u32 %1, %16, %16, %1;\n\t"
        "madc.lo.cc.u32 %2, %17, %17, %2;\n\t"
        "madc.hi.cc.u32 %3, %17, %17, %3;\n\t"
        "madc.lo.cc.u32 %4, %18, %18, %4;\n\t"
        "madc.hi.cc.u32 %5, %18, %18, %5;\n\t"
        "madc.lo.cc.u32 %6, %19, %19, %6;\n\t"
        "madc.hi.cc.u32 %7, %19, %19, %7;\n\t"
        "madc.lo.cc.u32 %8, %20, %20, %8;\n\t"
        "madc.hi.cc.u32 %9, %20, %20, %9;\n\t"
        "madc.lo.cc.u32 %10, %21, %21, %10;\n\t"
        "madc.hi.cc.u32 %11, %21, %21, %11;\n\t"
        "madc.lo.cc.u32 %12, %22, %22, %12;\n\t"
        "madc.hi.cc.u32 %13, %22, %22, %13;\n\t"
        "madc.lo.cc.u32 %14, %23, %23, %14;\n\t"
        "madc.hi.u32    %15, %23, %23, %15;"
        : "+r"(t[0]), "+r"(t[1]), "+r"(t[2]), "+r"(t[3]), "+r"(t[4]), "+r"(t[5]), "+r"(t[6]), "+r"(t[7]), "+r"(t[8]), "+r"(t[9]), "+r"(t[10]), "+r"(t[11]), "+r"(t[12]), "+r"(t[13]), "+r"(t[14]), "+r"(t[15])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
}


// w -= x (16 limbs); returns the borrow mask (0xffffffff when w < x).
__device__ __forceinline__ uint32_t sub_wide(uint32_t w[16], const uint32_t x[16]) {
    uint32_t br;
    asm("sub.cc.u32  %0, %0, %17;\n\t"
        "subc.cc.u32 %1, %1, %18;\n\t"
        "subc.cc.u32 %2, %2, %19;\n\t"
        "subc.cc.u32 %3, %3, %20;\n\t"
        "subc.cc.u32 %4, %4, %21;\n\t"
        "subc.cc.u32 %5, %5, %22;\n\t"
        "subc.cc.u32 %6, %6, %23;\n\t"
        "subc.cc.u32 %7, %7, %24;\n\t"
        "subc.cc.u32 %8, %8, %25;\n\t"
        "subc.cc.u32 %9, %9, %26;\n\t"
        "subc.cc.u32 %10, %10, %27;\n\t"
        "subc.cc.u32 %11, %11, %28;\n\t"
        "subc.cc.u32 %12, %12, %29;\n\t"
        "subc.cc.u32 %13, %13, %30;\n\t"
        "subc.cc.u32 %14, %14, %31;\n\t"
        "subc.cc.u32 %15, %15, %32;\n\t"
        "subc.u32    %16, 0, 0;"
        : "+r"(w[0]), "+r"(w[1]), "+r"(w[2]), "+r"(w[3]), "+r"(w[4]), "+r"(w[5]), "+r"(w[6]),
          "+r"(w[7]), "+r"(w[8]), "+r"(w[9]), "+r"(w[10]), "+r"(w[11]), "+r"(w[12]),
          "+r"(w[13]), "+r"(w[14]), "+r"(w[15]), "=r"(br)
        : "r"(x[0]), "r"(x[1]), "r"(x[2]), "r"(x[3]), "r"(x[4]), "r"(x[5]), "r"(x[6]),
          "r"(x[7]), "r"(x[8]), "r"(x[9]), "r"(x[10]), "r"(x[11]), "r"(x[12]), "r"(x[13]),
          "r"(x[14]), "r"(x[15]));
    return br;
}

// w += m * 2^256 where mask is all-ones (mod 2^512): brings a negative
// difference of two products back into [0, m * 2^256).
template <class C>
__device__ __forceinline__ void add_mR_masked(uint32_t w[16], uint32_t mask) {
    asm("add.cc.u32  %0, %0, %8;\n\t"
        "addc.cc.u32 %1, %1, %9;\n\t"
        "addc.cc.u32 %2, %2, %10;\n\t"
        "addc.cc.u32 %3, %3, %11;\n\t"
        "addc.cc.u32 %4, %4, %12;\n\t"
        "addc.cc.u32 %5, %5, %13;\n\t"
        "addc.cc.u32 %6, %6, %14;\n\t"
        "addc.u32    %7, %7, %15;"
        : "+r"(w[8]), "+r"(w[9]), "+r"(w[10]), "+r"(w[11]), "+r"(w[12]), "+r"(w[13]),
          "+r"(w[14]), "+r"(w[15])
        : "r"(C::M[0] & mask), "r"(C::M[1] & mask), "r"(C::M[2] & mask), "r"(C::M[3] & mask),
          "r"(C::M[4] & mask), "r"(C::M[5] & mask), "r"(C::M[6] & mask), "r"(C::M[7] & mask));
}

// Montgomery reduction of a 512-bit w < m * 2^256: returns w * 2^-256 mod m,
// fully reduced. Reduces the low half (u = (w_lo + q m) / 2^256 <= m), then
// u + w_hi < 2m takes one conditional subtraction.
template <class C>
__device__ __forceinline__ Fp<C> redc_wide(const uint32_t w[16]) {
    uint32_t t0 = w[0], t1 = w[1], t2 = w[2], t3 = w[3], t4 = w[4], t5 = w[5], t6 = w[6],
             t7 = w[7], t8 = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t m = t0 * C::N0;
        asm("mad.lo.cc.u32  %0, %9,  %10, %0;\n\t"
            "madc.lo.cc.u32 %1, %9,  %11, %1;\n\t"
            "madc.lo.cc.u32 %2, %9,  %12, %2;\n\t"
            "madc.lo.cc.u32 %3, %9,  %13, %3;\n\t"
            "madc.lo.cc.u32 %4, %9,  %14, %4;\n\t"
            "madc.lo.cc.u32 %5, %9,  %15, %5;\n\t"
            "madc.lo.cc.u32 %6, %9,  %16, %6;\n\t"
            "madc.lo.cc.u32 %7, %9,  %17, %7;\n\t"
            "addc.u32       %8, %8, 0;"
            : "+r"(t0), "+r"(t1), "+r"(t2), "+r"(t3), "+r"(t4), "+r"(t5), "+r"(t6), "+r"(t7),
              "+r"(t8)
            : "r"(m), "n"(C::M[0]), "n"(C::M[1]), "n"(C::M[2]), "n"(C::M[3]), "n"(C::M[4]),
              "n"(C::M[5]), "n"(C::M[6]), "n"(C::M[7]));
        asm("mad.hi.cc.u32  %0, %8,  %9,  %0;\n\t"
            "madc.hi.cc.u32 %1, %8,  %10, %1;\n\t"
            "madc.hi.cc.u32 %2, %8,  %11, %2;\n\t"
            "madc.hi.cc.u32 %3, %8,  %12, %3;\n\t"
            "madc.hi.cc.u32 %4, %8,  %13, %4;\n\t"
            "madc.hi.cc.u32 %5, %8,  %14, %5;\n\t"
            "madc.hi.cc.u32 %6, %8,  %15, %6;\n\t"
            "madc.hi.u32    %7, %8,  %16, %7;"
            : "+r"(t1), "+r"(t2), "+r"(t3), "+r"(t4), "+r"(t5), "+r"(t6), "+r"(t7), "+r"(t8)
            : "r"(m), "n"(C::M[0]), "n"(C::M[1]), "n"(C::M[2]), "n"(C::M[3]), "n"(C::M[4]),
              "n"(C::M[5]), "n"(C::M[6]), "n"(C::M[7]));
        t0 = t1; t1 = t2; t2 = t3; t3 = t4; t4 = t5; t5 = t6; t6 = t7; t7 = t8; t8 = 0;
    }
    uint32_t t[9];
    asm("add.cc.u32  %0, %9,  %17;\n\t"
        "addc.cc.u32 %1, %10, %18;\n\t"
        "addc.cc.u32 %2, %11, %19;\n\t"
        "addc.cc.u32 %3, %12, %20;\n\t"
        "addc.cc.u32 %4, %13, %21;\n\t"
        "addc.cc.u32 %5, %14, %22;\n\t"
        "addc.cc.u32 %6, %15, %23;\n\t"
        "addc.cc.u32 %7, %16, %24;\n\t"
        "addc.u32    %8, 0, 0;"
        : "=r"(t[0]), "=r"(t[1]), "=r"(t[2]), "=r"(t[3]), "=r"(t[4]), "=r"(t[5]), "=r"(t[6]),
          "=r"(t[7]), "=r"(t[8])
        : "r"(t0), "r"(t1), "r"(t2), "r"(t3), "r"(t4), "r"(t5), "r"(t6), "r"(t7), "r"(w[8]),
          "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]));
    Fp<C> r;
    final_sub<C>(t, r.v);
    return r;
}

// Montgomery squaring: sqr_wide + one reduction (208 IMAD vs 264).
template <class C>
__device__ __forceinline__ Fp<C> sqr(const Fp<C>& a) {
    uint32_t w[16];
    sqr_wide(a, w);
    return redc_wide<C>(w);
}

// a + b without reduction (a, b < m < 2^254: the sum fits 8 limbs).
template <class C>
__device__ __forceinline__ Fp<C> add_raw(const Fp<C>& a, const Fp<C>& b) {
    Fp<C> r;
    asm("add.cc.u32  %0, %8,  %16;\n\t"
        "addc.cc.u32 %1, %9,  %17;\n\t"
        "addc.cc.u32 %2, %10, %18;\n\t"
        "addc.cc.u32 %3, %11, %19;\n\t"
        "addc.cc.u32 %4, %12, %20;\n\t"
        "addc.cc.u32 %5, %13, %21;\n\t"
        "addc.cc.u32 %6, %14, %22;\n\t"
        "addc.u32    %7, %15, %23;"
        : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]),
          "=r"(r.v[6]), "=r"(r.v[7])
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]),
          "r"(a.v[6]), "r"(a.v[7]), "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]),
          "r"(b.v[4]), "r"(b.v[5]), "r"(b.v[6]), "r"(b.v[7]));
    return r;
}

// a * b - c * d (a..d reduced): two products, one reduction.
template <class C>
__device__ __forceinline__ Fp<C> mul_sub_mul(const Fp<C>& a, const Fp<C>& b, const Fp<C>& c,
                                             const Fp<C>& d) {
    uint32_t w[16], x[16];
    mul_wide(a, b, w);
    mul_wide(c, d, x);
    add_mR_masked<C>(w, sub_wide(w, x));  // (-m^2, m^2) -> [0, m * 2^256)
    return redc_wide<C>(w);
}

template <class C>
__device__ __forceinline__ Fp<C> add(const Fp<C>& a, const Fp<C>& b) {
    uint32_t t[9];
    asm("add.cc.u32  %0, %9,  %17;\n\t"
        "addc.cc.u32 %1, %10, %18;\n\t"
        "addc.cc.u32 %2, %11, %19;\n\t"
        "addc.cc.u32 %3, %12, %20;\n\t"
        "addc.cc.u32 %4, %13, %21;\n\t"
        "addc.cc.u32 %5, %14, %22;\n\t"
        "addc.cc.u32 %6, %15, %23;\n\t"
        "addc.cc.u32 %7, %16, %24;\n\t"
        "addc.u32    %8, 0, 0;"
        : "=r"(t[0]), "=r"(t[1]), "=r"(t[2]), "=r"(t[3]), "=r"(t[4]), "=r"(t[5]), "=r"(t[6]),
          "=r"(t[7]), "=r"(t[8])
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]),
          "r"(a.v[6]), "r"(a.v[7]), "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]),
          "r"(b.v[4]), "r"(b.v[5]), "r"(b.v[6]), "r"(b.v[7]));
    Fp<C> r;
    final_sub<C>(t, r.v);
    return r;
}

template <class C>
__device__ __forceinline__ Fp<C> sub(const Fp<C>& a, const Fp<C>& b) {
    uint32_t t[8], br;
    asm("sub.cc.u32  %0, %9,  %17;\n\t"
        "subc.cc.u32 %1, %10, %18;\n\t"
        "subc.cc.u32 %2, %11, %19;\n\t"
        "subc.cc.u32 %3, %12, %20;\n\t"
        "subc.cc.u32 %4, %13, %21;\n\t"
        "subc.cc.u32 %5, %14, %22;\n\t"
        "subc.cc.u32 %6, %15, %23;\n\t"
        "subc.cc.u32 %7, %16, %24;\n\t"
        "subc.u32    %8, 0, 0;"
        : "=r"(t[0]), "=r"(t[1]), "=r"(t[2]), "=r"(t[3]), "=r"(t[4]), "=r"(t[5]), "=r"(t[6]),
          "=r"(t[7]), "=r"(br)
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]),
          "r"(a.v[6]), "r"(a.v[7]), "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]),
          "r"(b.v[4]), "r"(b.v[5]), "r"(b.v[6]), "r"(b.v[7]));
    // add back m & borrow-mask
    Fp<C> r;
    asm("add.cc.u32  %0, %8,  %16;\n\t"
        "addc.cc.u32 %1, %9,  %17;\n\t"
        "addc.cc.u32 %2, %10, %18;\n\t"
        "addc.cc.u32 %3, %11, %19;\n\t"
        "addc.cc.u32 %4, %12, %20;\n\t"
        "addc.cc.u32 %5, %13, %21;\n\t"
        "addc.cc.u32 %6, %14, %22;\n\t"
        "addc.u32    %7, %15, %23;"
        : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]),
          "=r"(r.v[6]), "=r"(r.v[7])
        : "r"(t[0]), "r"(t[1]), "r"(t[2]), "r"(t[3]), "r"(t[4]), "r"(t[5]), "r"(t[6]), "r"(t[7]),
          "r"(C::M[0] & br), "r"(C::M[1] & br), "r"(C::M[2] & br), "r"(C::M[3] & br),
          "r"(C::M[4] & br), "r"(C::M[5] & br), "r"(C::M[6] & br), "r"(C::M[7] & br));
    return r;
}

template <class C>
__device__ __forceinline__ Fp<C> neg(const Fp<C>& a) {
    return a.is_zero() ? a : sub(Fp<C>::zero(), a);
}

template <class C>
__device__ __forceinline__ Fp<C> dbl(const Fp<C>& a) { return add(a, a); }

// Standard (canonical, little-endian limbs) <-> Montgomery.
template <class C>
__device__ __forceinline__ Fp<C> to_mont(const Fp<C>& a) {
    Fp<C> r2;
#pragma unroll
    for (int i = 0; i < 8; ++i) r2.v[i] = r2_limb<C>(i);
    return mul(a, r2);
}

template <class C>
__device__ __forceinline__ Fp<C> from_mont(const Fp<C>& a) {
    Fp<C> one;
#pragma unroll
    for (int i = 0; i < 8; ++i) one.v[i] = i == 0 ? 1u : 0u;
    return mul(a, one);
}

// a^e for a small public exponent given as 8 limbs (square-and-multiply).
template <class C>
__device__ Fp<C> pow(const Fp<C>& a, const uint32_t e[8]) {
    Fp<C> r = Fp<C>::one(), b = a;
    for (int i = 0; i < 256; ++i) {
        if ((e[i >> 5] >> (i & 31)) & 1) r = mul(r, b);
        b = sqr(b);
    }
    return r;
}

// Fermat inverse a^(m-2).
template <class C>
__device__ Fp<C> inv(const Fp<C>& a) {
    uint32_t e[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) e[i] = mod_limb<C>(i);
    e[0] -= 2;
    return pow(a, e);
}

// Binary extended-Euclid inverse (variable time; the operands here are
// public curve coordinates): ~2*254 shift/subtract steps on 8 limbs instead
// of Fermat's 254 squarings + multiplications. Montgomery in, Montgomery out:
// t = (aR)^-1 as an integer, then t * R^2 via two Montgomery products.
namespace detail {
__device__ __forceinline__ bool limbs_is_one(const uint32_t x[8]) {
    uint32_t o = x[0] ^ 1u;
#pragma unroll
    for (int i = 1; i < 8; ++i) o |= x[i];
    return o == 0;
}
__device__ __forceinline__ bool limbs_geq(const uint32_t a[8], const uint32_t b[8]) {
#pragma unroll
    for (int i = 7; i >= 0; --i)
        if (a[i] != b[i]) return a[i] > b[i];
    return true;
}
__device__ __forceinline__ void limbs_sub(uint32_t a[8], const uint32_t b[8]) {
    uint32_t br = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        uint64_t d = (uint64_t)a[i] - b[i] - br;
        a[i] = (uint32_t)d;
        br = (uint32_t)(d >> 63);
    }
}
__device__ __forceinline__ void limbs_add(uint32_t a[8], const uint32_t b[8]) {
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        uint64_t s = (uint64_t)a[i] + b[i] + c;
        a[i] = (uint32_t)s;
        c = (uint32_t)(s >> 32);
    }
}
__device__ __forceinline__ void limbs_shr1(uint32_t a[8]) {
#pragma unroll
    for (int i = 0; i < 7; ++i) a[i] = __funnelshift_r(a[i], a[i + 1], 1);
    a[7] >>= 1;
}
// x = x/2 mod m (x < m, m odd)
template <class C>
__device__ __forceinline__ void half_mod(uint32_t x[8]) {
    if (x[0] & 1) {
        uint32_t m[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) m[i] = mod_limb<C>(i);
        limbs_add(x, m);  // < 2m < 2^255: no overflow
    }
    limbs_shr1(x);
}
// x = x - y mod m
template <class C>
__device__ __forceinline__ void sub_mod(uint32_t x[8], const uint32_t y[8]) {
    if (limbs_geq(x, y)) {
        limbs_sub(x, y);
    } else {
        uint32_t m[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) m[i] = mod_limb<C>(i);
        limbs_add(x, m);
        limbs_sub(x, y);
    }
}
}  // namespace detail

template <class C>
__device__ Fp<C> inv_fast(const Fp<C>& a) {
    using namespace detail;
    if (a.is_zero()) return a;
    uint32_t u[8], v[8], x1[8], x2[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        u[i] = a.v[i];
        v[i] = mod_limb<C>(i);
        x1[i] = i == 0;
        x2[i] = 0;
    }
    while (!limbs_is_one(u) && !limbs_is_one(v)) {
        while (!(u[0] & 1)) {
            limbs_shr1(u);
            half_mod<C>(x1);
        }
        while (!(v[0] & 1)) {
            limbs_shr1(v);
            half_mod<C>(x2);
        }
        if (limbs_geq(u, v)) {
            limbs_sub(u, v);
            sub_mod<C>(x1, x2);
        } else {
            limbs_sub(v, u);
            sub_mod<C>(x2, x1);
        }
    }
    Fp<C> t, r2;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        t.v[i] = limbs_is_one(u) ? x1[i] : x2[i];
        r2.v[i] = r2_limb<C>(i);
    }
    return mul(mul(t, r2), r2);
}

// 16-B vector loads / stores of one element (32 B, 16-B aligned).
template <class C>
__device__ __forceinline__ Fp<C> load(const void* p) {
    const uint4* q = static_cast<const uint4*>(p);
    uint4 x = q[0], y = q[1];
    Fp<C> r;
    r.v[0] = x.x; r.v[1] = x.y; r.v[2] = x.z; r.v[3] = x.w;
    r.v[4] = y.x; r.v[5] = y.y; r.v[6] = y.z; r.v[7] = y.w;
    return r;
}
template <class C>
__device__ __forceinline__ void store(void* p, const Fp<C>& a) {
    uint4* q = static_cast<uint4*>(p);
    q[0] = make_uint4(a.v[0], a.v[1], a.v[2], a.v[3]);
    q[1] = make_uint4(a.v[4], a.v[5], a.v[6], a.v[7]);
}

}  // namespace bn
}  // namespace ace_gpu
