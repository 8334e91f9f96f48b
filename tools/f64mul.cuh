// FP64 (DFMA) Montgomery product for BN254 Fq (tools probe).
// Radix 2^52 (5 limbs), R = 2^260, as a drop-in for mul():
// MM260(16a, b) = a b 2^-256 mod p. Each 52x52 limb product is split exactly:
// t = fma_rz(x, y, 2^104) (hi in t's mantissa), s = (2^104 + 2^52) - t,
// l = fma(x, y, s) = lo + 2^52 (lo in l's mantissa); hi and lo are accumulated
// as raw bit patterns in 64-bit integer columns (ALU pipe), the exponent bits
// removed by a per-column bias the columns start from.
#pragma once
#include "bn254.cuh"

namespace f64m {
using namespace ace_gpu::bn;
constexpr uint64_t M52 = (1ull << 52) - 1;
constexpr uint64_t B52 = 0x4330000000000000ull;   // bits(2^52)
constexpr uint64_t B104 = 0x4670000000000000ull;  // bits(2^104)
constexpr double C1 = 20282409603651670423947251286016.0;                       // 2^104
constexpr double C2 = 20282409603651670423947251286016.0 + 4503599627370496.0;  // 2^104 + 2^52
constexpr double T52 = 4503599627370496.0;
constexpr double P0 = (double)0x8c16d87cfd47ull, P1 = (double)0x916871ca8d3c2ull,
                 P2 = (double)0x181585d97816aull, P3 = (double)0xa029b85045b68ull,
                 P4 = (double)0x30644e72e131ull;
constexpr double NP = (double)0x20782e4866389ull;
__device__ __forceinline__ double pl(int j) {
    return j == 0 ? P0 : j == 1 ? P1 : j == 2 ? P2 : j == 3 ? P3 : P4;
}
// bias of column k: -(#lo * B52 + #hi * B104) over the ab products and the
// reduction products (the j = 0 lo of m p_0 is not accumulated)
constexpr uint64_t bias(int k) {
    uint64_t s = 0;
    for (int i = 0; i < 5; ++i)
        for (int j = 0; j < 5; ++j) {
            if (i + j == k) s += B52;
            if (i + j + 1 == k) s += B104;
        }
    for (int i = 0; i < 5; ++i)
        for (int j = 0; j < 5; ++j) {
            if (j > 0 && i + j == k) s += B52;
            if (i + j + 1 == k) s += B104;
        }
    return 0ull - s;
}
__device__ __forceinline__ uint64_t bits(double x) { return (uint64_t)__double_as_longlong(x); }
__device__ __forceinline__ double to_d(uint64_t x52) {  // x < 2^52
    return __dsub_rn(__longlong_as_double((long long)(x52 | B52)), T52);
}
__device__ __forceinline__ void split_acc(double x, double y, uint64_t& clo, uint64_t& chi) {
    const double t = __fma_rz(x, y, C1);
    const double s = __dsub_rn(C2, t);
    const double l = __fma_rn(x, y, s);
    clo += bits(l);
    chi += bits(t);
}
// 8 x 32-bit limbs -> 5 x 52-bit doubles of (a << SH), SH in {0, 4}
template <int SH>
__device__ __forceinline__ void to52(const uint32_t v[8], double d[5]) {
    const uint64_t w0 = ((uint64_t)v[1] << 32) | v[0], w1 = ((uint64_t)v[3] << 32) | v[2],
                   w2 = ((uint64_t)v[5] << 32) | v[4], w3 = ((uint64_t)v[7] << 32) | v[6];
    d[0] = to_d((w0 << SH) & M52);
    d[1] = to_d(((w0 >> (52 - SH)) | (w1 << (12 + SH))) & M52);
    d[2] = to_d(((w1 >> (40 - SH)) | (w2 << (24 + SH))) & M52);
    d[3] = to_d(((w2 >> (28 - SH)) | (w3 << (36 + SH))) & M52);
    d[4] = to_d((w3 >> (16 - SH)) & M52);
}

__device__ __forceinline__ Fq mul_f64(const Fq& a, const Fq& b) {
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
    uint64_t carry = 0;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const uint64_t s = c[i] + carry;
        const uint64_t v = s & M52;
        carry = (s >> 52) + (v != 0);
        const double vd = to_d(v);
        const double t = __fma_rz(vd, NP, C1);
        const double l = __fma_rn(vd, NP, __dsub_rn(C2, t));
        const double md = __dsub_rn(l, T52);  // m = lo52(v n')
        c[i + 1] += bits(__fma_rz(md, P0, C1));
#pragma unroll
        for (int j = 1; j < 5; ++j) split_acc(md, pl(j), c[i + j], c[i + j + 1]);
    }
    uint64_t r[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const uint64_t s = c[5 + k] + carry;
        r[k] = s & M52;
        carry = s >> 52;
    }
    r[4] += carry << 52;
    const uint64_t w0 = r[0] | (r[1] << 52), w1 = (r[1] >> 12) | (r[2] << 40),
                   w2 = (r[2] >> 24) | (r[3] << 28), w3 = (r[3] >> 36) | (r[4] << 16);
    uint32_t t9[9] = {(uint32_t)w0, (uint32_t)(w0 >> 32), (uint32_t)w1, (uint32_t)(w1 >> 32),
                      (uint32_t)w2, (uint32_t)(w2 >> 32), (uint32_t)w3, (uint32_t)(w3 >> 32),
                      (uint32_t)(r[4] >> 48)};
    Fq out;
    final_sub<FqCfg>(t9, out.v);
    return out;
}
}  // namespace f64m
