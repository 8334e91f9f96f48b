// Optimal ate pairing on BN254 for sm_100a: the Groth16 verifier of the
// north-star block path (verify_finality_certificate with
// real Groth16 in a few pairings instead of an O(N) recompute).
//
// Tower (same as the CPU oracle, oracle/bn254_oracle.c):
//   Fq2 = Fq[u]/(u^2+1), Fq6 = Fq2[v]/(v^3 - xi), xi = 9+u, Fq12 = Fq6[w]/(w^2 - v).
// G2 lives on the D-type twist y^2 = x^3 + 3/xi, untwisted by (x w^2, y w^3).
// Miller loop over 6x+2 (x = 4965661367192848881) in homogeneous projective
// coordinates, no inversions; each line is scaled by an Fq2 factor (killed by
// the final exponentiation):
//   doubling T=(X,Y,Z):  W = 3X^2, S = YZ, B = XYS, H = W^2 - 8B,
//        2T = (2HS, W(4B - H) - 8Y^2S^2, 8S^3),
//        line = 2YZ^2 yP  + (-3X^2 Z) xP w + (3X^3 - 2Y^2 Z) w^3
//   addition T + (x2, y2):  N = y2 Z - Y, D = x2 Z - X, A = N^2 Z - D^3 - 2D^2 X,
//        T' = (D A, N(D^2 X - A) - D^3 Y, D^3 Z),
//        line = D yP + (-N) xP w + (N x2 - D y2) w^3
// (derivations in DESIGN.md §6). Final exponentiation: (p^6-1)(p^2+1) by
// conjugation / inversion / Frobenius, then the hard part with the
// Devegili-Scott-Dahab chain (three exponentiations by x and Frobenius maps).
#pragma once
#include "curve.cuh"

namespace ace_gpu {
namespace bn {

struct Fq6 {
    Fq2 c0, c1, c2;
};
struct Fq12 {
    Fq6 c0, c1;
};

// gamma[k-1][i] = xi^(i (p^k - 1) / 6), standard form (Frobenius^k of w^i).
__device__ __constant__ static const uint32_t kFrobGamma[18][2][8] = {
    {{0x00000001u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u},
     {0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u}},  // k=1 i=0
    {{0xdcc9e470u, 0xd60b35dau, 0x292f2176u, 0x5c521e08u, 0x76e68b60u, 0xe8b99fddu, 0x2865a7dfu, 0x1284b71cu},
     {0x80f362acu, 0xca5cf05fu, 0x8eeec7e5u, 0x74799277u, 0x12150b8eu, 0xa6327cfeu, 0xb4fae7e6u, 0x246996f3u}},  // k=1 i=1
    {{0x176f553du, 0x99e39557u, 0xc2c3330cu, 0xb78cc310u, 0xf559b143u, 0x4c0bec3cu, 0x4f7911f7u, 0x2fb34798u},
     {0x640fcba2u, 0x1665d51cu, 0x0b7c9dceu, 0x32ae2a1du, 0xd75a0794u, 0x4ba4cc8bu, 0x61ebae20u, 0x16c9e550u}},  // k=1 i=2
    {{0x71a0135au, 0xdc540146u, 0xa9c95998u, 0xdbaae0edu, 0xb6e2f9b9u, 0xdc5ec698u, 0x489af5dcu, 0x063cf305u},
     {0x2623b0e3u, 0x82d37f63u, 0x8fa25bd2u, 0x21807dc9u, 0xec796f2bu, 0x0704b5a7u, 0xac41049au, 0x07c03cbcu}},  // k=1 i=3
    {{0x921ea762u, 0x848a1f55u, 0xbe94ec72u, 0xd33365f7u, 0x5a181e84u, 0x80f3c0b7u, 0x64eea801u, 0x05b54f5eu},
     {0xcd2b8126u, 0xc13b4711u, 0x1bdec763u, 0x3685d2eau, 0x3b0b1c92u, 0x9f3a80b0u, 0xe7fd8aeeu, 0x2c145edbu}},  // k=1 i=4
    {{0xeab7692fu, 0x2ea2c810u, 0x55aa1bd3u, 0x425c459bu, 0xa4353ff4u, 0xe93a3661u, 0x4f798649u, 0x0183c1e7u},
     {0x6e0c2c4bu, 0x24c6b8eeu, 0x678e2ac0u, 0xb080cb99u, 0xc7729f7du, 0xa27fb246u, 0x76fd0675u, 0x12acf2cau}},  // k=1 i=5
    {{0x00000001u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u},
     {0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u}},  // k=2 i=0
    {{0x607cfd49u, 0xe4bd44e5u, 0xbb966e3du, 0xc28f069fu, 0xe0acccb0u, 0x5e6dd9e7u, 0xe131a029u, 0x30644e72u},
     {0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u}},  // k=2 i=1
    {{0x607cfd48u, 0xe4bd44e5u, 0xbb966e3du, 0xc28f069fu, 0xe0acccb0u, 0x5e6dd9e7u, 0xe131a029u, 0x30644e72u},
     {0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u}},  // k=2 i=2
    {{0xd87cfd46u, 0x3c208c16u, 0x6871ca8du, 0x97816a91u, 0x8181585du, 0xb85045b6u, 0xe131a029u, 0x30644e72u},
     {0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u}},  // k=2 i=3
    {{0x77fffffeu, 0x57634731u, 0xacdb5c4fu, 0xd4f263f1u, 0xa0d48bacu, 0x59e26bceu, 0x00000000u, 0x00000000u},
     {0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u}},  // k=2 i=4
    {{0x77ffffffu, 0x57634731u, 0xacdb5c4fu, 0xd4f263f1u, 0xa0d48bacu, 0x59e26bceu, 0x00000000u, 0x00000000u},
     {0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u}},  // k=2 i=5
    {{0x00000001u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u},
     {0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u}},  // k=3 i=0
    {{0x1ed4a67fu, 0xe86f7d39u, 0xbe55d24au, 0x894cb38du, 0xd0acaa90u, 0xefe9608cu, 0xcc82e4bbu, 0x19dc81cfu},
     {0xf4c0c101u, 0x7694aa2bu, 0x97d439ecu, 0x7f03a5e3u, 0x3576139du, 0x06cbeee3u, 0x0be77d73u, 0x00abf8b6u}},  // k=3 i=1
    {{0x7bdcfb6du, 0x7b746ee8u, 0x5d6942d3u, 0x805ffd3du, 0x959f25acu, 0xbaff1c77u, 0xb755ef0au, 0x0856e078u},
     {0xaaa586deu, 0x380cab2bu, 0x98ff2631u, 0x0fdf31bfu, 0xec26094fu, 0xa9f30e6du, 0xb3d1766fu, 0x04f1de41u}},  // k=3 i=2
    {{0x66dce9edu, 0x5fcc8ad0u, 0xbea870f4u, 0xbbd689a3u, 0xca9e5ea3u, 0xdbf17f1du, 0x9896aa4cu, 0x2a275b6du},
     {0xb2594c64u, 0xb94d0cb3u, 0xd8cf6ebau, 0x7600ecc7u, 0x9507e932u, 0xb14b900eu, 0x34f09b8fu, 0x28a411b6u}},  // k=3 i=3
    {{0x3ccbf066u, 0x0e1a92bcu, 0x75b06bcbu, 0xe6330945u, 0xb5b2444eu, 0x19bee0f7u, 0x11c08dabu, 0x0bc58c66u},
     {0x730c239fu, 0x5fe3ed9du, 0x737f96e5u, 0xa44a9e08u, 0x0cd21d04u, 0xfeb0f6efu, 0xe1910a12u, 0x23d5e999u}},  // k=3 i=4
    {{0x76261b43u, 0xebde8470u, 0x967c84a5u, 0x2ed68098u, 0x3b4d3f69u, 0x711699fau, 0x952c0905u, 0x13c49044u},
     {0x84282499u, 0x1f250413u, 0x20028021u, 0x3e2ddaeau, 0x2a48633du, 0x9fb1b228u, 0x59b1dd0bu, 0x16db366au}},  // k=3 i=5
};

__device__ __forceinline__ Fq2 f2_neg(const Fq2& a) { return {neg(a.c0), neg(a.c1)}; }
__device__ __forceinline__ Fq2 f2_conj(const Fq2& a) { return {a.c0, neg(a.c1)}; }
__device__ __forceinline__ Fq2 f2_mul_fq(const Fq2& a, const Fq& s) {
    return {fq_mul_call(a.c0, s), fq_mul_call(a.c1, s)};
}
__device__ __forceinline__ Fq f_x9(const Fq& a) {  // 9a
    Fq a2 = add(a, a), a4 = add(a2, a2), a8 = add(a4, a4);
    return add(a8, a);
}
__device__ __forceinline__ Fq2 f2_mul_xi(const Fq2& a) {  // (a0 + a1 u)(9 + u)
    return {sub(f_x9(a.c0), a.c1), add(a.c0, f_x9(a.c1))};
}
__device__ __forceinline__ Fq2 f2_inv(const Fq2& a) {
    const Fq n = add(fq_mul_call(a.c0, a.c0), fq_mul_call(a.c1, a.c1));
    const Fq ni = inv_fast(n);
    return {fq_mul_call(a.c0, ni), neg(fq_mul_call(a.c1, ni))};
}
__device__ __forceinline__ Fq2 f2_gamma(int k, int i) {
    Fq2 g;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        g.c0.v[j] = kFrobGamma[6 * (k - 1) + i][0][j];
        g.c1.v[j] = kFrobGamma[6 * (k - 1) + i][1][j];
    }
    return {to_mont(g.c0), to_mont(g.c1)};
}

// ---- Fq6 ------------------------------------------------------------------
__device__ __forceinline__ Fq6 f6_add(const Fq6& a, const Fq6& b) {
    return {fadd(a.c0, b.c0), fadd(a.c1, b.c1), fadd(a.c2, b.c2)};
}
__device__ __forceinline__ Fq6 f6_sub(const Fq6& a, const Fq6& b) {
    return {fsub(a.c0, b.c0), fsub(a.c1, b.c1), fsub(a.c2, b.c2)};
}
__device__ __forceinline__ Fq6 f6_neg(const Fq6& a) { return {f2_neg(a.c0), f2_neg(a.c1), f2_neg(a.c2)}; }
__device__ __forceinline__ Fq6 f6_mul_v(const Fq6& a) { return {f2_mul_xi(a.c2), a.c0, a.c1}; }

// Karatsuba-style (6 Fq2 products).
static __device__ __noinline__ Fq6 f6_mul(const Fq6& a, const Fq6& b) {
    const Fq2 t0 = fmul(a.c0, b.c0), t1 = fmul(a.c1, b.c1), t2 = fmul(a.c2, b.c2);
    const Fq2 c0 = fadd(t0, f2_mul_xi(fsub(fsub(fmul(fadd(a.c1, a.c2), fadd(b.c1, b.c2)), t1), t2)));
    const Fq2 c1 = fadd(fsub(fsub(fmul(fadd(a.c0, a.c1), fadd(b.c0, b.c1)), t0), t1), f2_mul_xi(t2));
    const Fq2 c2 = fadd(fsub(fsub(fmul(fadd(a.c0, a.c2), fadd(b.c0, b.c2)), t0), t2), t1);
    return {c0, c1, c2};
}
static __device__ __noinline__ Fq6 f6_inv(const Fq6& a) {
    const Fq2 t0 = fsub(fsqr(a.c0), f2_mul_xi(fmul(a.c1, a.c2)));
    const Fq2 t1 = fsub(f2_mul_xi(fsqr(a.c2)), fmul(a.c0, a.c1));
    const Fq2 t2 = fsub(fsqr(a.c1), fmul(a.c0, a.c2));
    const Fq2 d = fadd(fmul(a.c0, t0), f2_mul_xi(fadd(fmul(a.c2, t1), fmul(a.c1, t2))));
    const Fq2 di = f2_inv(d);
    return {fmul(t0, di), fmul(t1, di), fmul(t2, di)};
}

// ---- Fq12 -----------------------------------------------------------------
__device__ __forceinline__ Fq12 f12_one() {
    Fq12 r;
    fset_one(r.c0.c0);
    fset_zero(r.c0.c1);
    fset_zero(r.c0.c2);
    fset_zero(r.c1.c0);
    fset_zero(r.c1.c1);
    fset_zero(r.c1.c2);
    return r;
}
static __device__ __noinline__ Fq12 f12_mul(const Fq12& a, const Fq12& b) {
    const Fq6 t0 = f6_mul(a.c0, b.c0), t1 = f6_mul(a.c1, b.c1);
    const Fq6 c1 = f6_sub(f6_sub(f6_mul(f6_add(a.c0, a.c1), f6_add(b.c0, b.c1)), t0), t1);
    return {f6_add(t0, f6_mul_v(t1)), c1};
}
// (a0 + a1 w)^2 = a0^2 + a1^2 v + 2 a0 a1 w, via (a0 + a1)(a0 + a1 v).
static __device__ __noinline__ Fq12 f12_sqr(const Fq12& a) {
    const Fq6 ab = f6_mul(a.c0, a.c1);
    const Fq6 t = f6_mul(f6_add(a.c0, a.c1), f6_add(a.c0, f6_mul_v(a.c1)));
    const Fq6 c0 = f6_sub(f6_sub(t, ab), f6_mul_v(ab));
    return {c0, f6_add(ab, ab)};
}
__device__ __forceinline__ Fq12 f12_conj(const Fq12& a) { return {a.c0, f6_neg(a.c1)}; }

// a * (b0 + b1 v): 5 Fq2 products (Karatsuba on the two non-zero terms).
static __device__ __noinline__ Fq6 f6_mul_01(const Fq6& a, const Fq2& b0, const Fq2& b1) {
    const Fq2 v0 = fmul(a.c0, b0), v1 = fmul(a.c1, b1);
    const Fq2 c1 = fsub(fsub(fmul(fadd(a.c0, a.c1), fadd(b0, b1)), v0), v1);
    return {fadd(v0, f2_mul_xi(fmul(a.c2, b1))), c1, fadd(v1, fmul(a.c2, b0))};
}
// f * line, line = l0 + (l1 + l2 v) w (the Miller-loop line shape): 13 Fq2
// products instead of the dense 18.
static __device__ __noinline__ Fq12 f12_mul_line(const Fq12& f, const Fq2& l0, const Fq2& l1,
                                                 const Fq2& l2) {
    const Fq6 t0 = {fmul(f.c0.c0, l0), fmul(f.c0.c1, l0), fmul(f.c0.c2, l0)};
    const Fq6 t1 = f6_mul_01(f.c1, l1, l2);
    const Fq6 t2 = f6_mul_01(f6_add(f.c0, f.c1), fadd(l0, l1), l2);
    return {f6_add(t0, f6_mul_v(t1)), f6_sub(f6_sub(t2, t0), t1)};
}
// Squaring in the cyclotomic subgroup (Granger-Scott): the three Fq4
// squarings (z0,z1) = (c0.c0, c1.c1), (z2,z3) = (c1.c0, c0.c2),
// (z4,z5) = (c0.c1, c1.c2) over y^2 = xi; 6 Fq2 products instead of 12.
static __device__ __noinline__ Fq12 f12_cyc_sqr(const Fq12& a) {
    auto fq4 = [](const Fq2& x, const Fq2& y, Fq2& s0, Fq2& s1) {  // (x + y t)^2, t^2 = xi
        const Fq2 xy = fmul(x, y);
        s0 = fsub(fsub(fmul(fadd(x, y), fadd(x, f2_mul_xi(y))), xy), f2_mul_xi(xy));
        s1 = fadd(xy, xy);
    };
    Fq2 t0, t1, t2, t3, t4, t5;
    fq4(a.c0.c0, a.c1.c1, t0, t1);
    fq4(a.c1.c0, a.c0.c2, t2, t3);
    fq4(a.c0.c1, a.c1.c2, t4, t5);
    auto tw = [](const Fq2& t, const Fq2& z, bool plus) {  // 3t -+ 2z
        const Fq2 d = plus ? fadd(t, z) : fsub(t, z);
        return fadd(fadd(d, d), t);
    };
    Fq12 r;
    r.c0.c0 = tw(t0, a.c0.c0, false);
    r.c1.c1 = tw(t1, a.c1.c1, true);
    r.c1.c0 = tw(f2_mul_xi(t5), a.c1.c0, true);
    r.c0.c2 = tw(t4, a.c0.c2, false);
    r.c0.c1 = tw(t2, a.c0.c1, false);
    r.c1.c2 = tw(t3, a.c1.c2, true);
    return r;
}
static __device__ __noinline__ Fq12 f12_inv(const Fq12& a) {
    const Fq6 d = f6_sub(f6_mul(a.c0, a.c0), f6_mul_v(f6_mul(a.c1, a.c1)));
    const Fq6 di = f6_inv(d);
    return {f6_mul(a.c0, di), f6_neg(f6_mul(a.c1, di))};
}
// Frobenius^k: coefficient of w^i -> conj^k(c_i) * gamma[k][i]; w^i order
// (a0, b0, a1, b1, a2, b2) for a + b w, a = a0 + a1 v + a2 v^2.
static __device__ __noinline__ Fq12 f12_frob(const Fq12& a, int k) {
    auto cj = [k](const Fq2& x) { return (k & 1) ? f2_conj(x) : x; };
    Fq12 r;
    r.c0.c0 = cj(a.c0.c0);
    r.c1.c0 = fmul(cj(a.c1.c0), f2_gamma(k, 1));
    r.c0.c1 = fmul(cj(a.c0.c1), f2_gamma(k, 2));
    r.c1.c1 = fmul(cj(a.c1.c1), f2_gamma(k, 3));
    r.c0.c2 = fmul(cj(a.c0.c2), f2_gamma(k, 4));
    r.c1.c2 = fmul(cj(a.c1.c2), f2_gamma(k, 5));
    return r;
}
__device__ __forceinline__ bool f12_is_one(const Fq12& a) {
    const Fq12 o = f12_one();
    return feq(a.c0.c0, o.c0.c0) && fzero(a.c0.c1) && fzero(a.c0.c2) && fzero(a.c1.c0) &&
           fzero(a.c1.c1) && fzero(a.c1.c2);
}

// a^x, x = 4965661367192848881 (63 bits); a in the cyclotomic subgroup.
__device__ __forceinline__ Fq12 f12_pow_x(const Fq12& a) {
    const uint64_t x = 4965661367192848881ull;
    Fq12 r = f12_one();
    for (int i = 62; i >= 0; --i) {
        r = f12_cyc_sqr(r);
        if ((x >> i) & 1) r = f12_mul(r, a);
    }
    return r;
}

// ---- Miller loop ----------------------------------------------------------
struct G2Proj {
    Fq2 X, Y, Z;
};

// Line (cy * yP) + (cx * xP) w + c3 w^3 = l0 + (l1 + l2 v) w.
struct Line {
    Fq2 l0, l1, l2;
};
__device__ __forceinline__ Line make_line(const Fq2& cy, const Fq2& cx, const Fq2& c3,
                                          const Fq& xP, const Fq& yP) {
    return {f2_mul_fq(cy, yP), f2_mul_fq(cx, xP), c3};
}
__device__ __forceinline__ Fq12 f12_mul_line(const Fq12& f, const Line& l) {
    return f12_mul_line(f, l.l0, l.l1, l.l2);
}

static __device__ __noinline__ Line dbl_step(G2Proj& T, const Fq& xP, const Fq& yP) {
    const Fq2 X2 = fsqr(T.X), Y2 = fsqr(T.Y);
    const Fq2 W = fadd(fadd(X2, X2), X2);
    const Fq2 S = fmul(T.Y, T.Z);
    const Fq2 B = fmul(fmul(T.X, T.Y), S);
    const Fq2 B4 = fadd(fadd(B, B), fadd(B, B));
    const Fq2 H = fsub(fsqr(W), fadd(B4, B4));
    const Fq2 S2 = fsqr(S);
    // line (before T changes)
    const Fq2 YZ2 = fmul(S, T.Z);                       // Y Z^2
    const Fq2 cy = fadd(YZ2, YZ2);                      // 2 Y Z^2
    const Fq2 cx = f2_neg(fmul(W, T.Z));                // -3 X^2 Z
    const Fq2 Y2Z = fmul(Y2, T.Z);
    const Fq2 c3 = fsub(fmul(W, T.X), fadd(Y2Z, Y2Z));  // 3X^3 - 2Y^2 Z
    const Fq2 HS = fmul(H, S);
    const Fq2 Y2S2 = fmul(Y2, S2);
    const Fq2 Y2S2x8 = fadd(fadd(fadd(Y2S2, Y2S2), fadd(Y2S2, Y2S2)),
                            fadd(fadd(Y2S2, Y2S2), fadd(Y2S2, Y2S2)));
    const Fq2 S3 = fmul(S2, S);
    const Fq2 S3x2 = fadd(S3, S3), S3x4 = fadd(S3x2, S3x2);
    T.X = fadd(HS, HS);
    T.Y = fsub(fmul(W, fsub(B4, H)), Y2S2x8);
    T.Z = fadd(S3x4, S3x4);
    return make_line(cy, cx, c3, xP, yP);
}

static __device__ __noinline__ Line add_step(G2Proj& T, const Fq2& x2, const Fq2& y2, const Fq& xP,
                                            const Fq& yP) {
    const Fq2 N = fsub(fmul(y2, T.Z), T.Y);
    const Fq2 D = fsub(fmul(x2, T.Z), T.X);
    const Fq2 cy = D;
    const Fq2 cx = f2_neg(N);
    const Fq2 c3 = fsub(fmul(N, x2), fmul(D, y2));
    const Fq2 D2 = fsqr(D), D3 = fmul(D2, D);
    const Fq2 D2X = fmul(D2, T.X);
    const Fq2 A = fsub(fsub(fmul(fsqr(N), T.Z), D3), fadd(D2X, D2X));
    const Fq2 X3 = fmul(D, A);
    const Fq2 Y3 = fsub(fmul(N, fsub(D2X, A)), fmul(D3, T.Y));
    const Fq2 Z3 = fmul(D3, T.Z);
    T.X = X3;
    T.Y = Y3;
    T.Z = Z3;
    return make_line(cy, cx, c3, xP, yP);
}

// pi(Q) on the twist: (conj(x) gamma_{1,2}, conj(y) gamma_{1,3}).
__device__ __forceinline__ void frob_twist(Fq2& x, Fq2& y) {
    x = fmul(f2_conj(x), f2_gamma(1, 2));
    y = fmul(f2_conj(y), f2_gamma(1, 3));
}

// f_{6x+2,Q}(P) * l_{T,pi(Q)}(P) * l_{T',-pi^2(Q)}(P); Q, P affine, not infinity.
static __device__ __noinline__ Fq12 miller_loop(const Fq& xP, const Fq& yP, const Fq2& xQ,
                                                const Fq2& yQ) {
    const uint64_t loop_lo = 0x9d797039be763ba8ull;  // 6x+2 = 2^64 + loop_lo
    Fq12 f = f12_one();
    G2Proj T;
    T.X = xQ;
    T.Y = yQ;
    fset_one(T.Z);
    for (int i = 63; i >= 0; --i) {
        f = f12_sqr(f);
        f = f12_mul_line(f, dbl_step(T, xP, yP));
        if ((loop_lo >> i) & 1) f = f12_mul_line(f, add_step(T, xQ, yQ, xP, yP));
    }
    Fq2 x1 = xQ, y1 = yQ;
    frob_twist(x1, y1);
    Fq2 x2 = x1, y2 = y1;
    frob_twist(x2, y2);
    f = f12_mul_line(f, add_step(T, x1, y1, xP, yP));
    f = f12_mul_line(f, add_step(T, x2, f2_neg(y2), xP, yP));
    return f;
}

// The Miller loop split over four warps of one CTA for up to 32 pairs (one
// per lane): warp 3 walks T and produces the lines (dbl_step, add_step),
// handing them over in shared memory double-buffered by iteration parity with
// one __syncthreads per iteration, so T's doubling overlaps f's squaring;
// warps 0-2 share f's squaring (two Fq6 products) and each line product (the
// three parts of f12_mul_line) through shared memory and a named barrier
// (bar.sync 1, 96). Same operations in the same order as miller_loop, so f
// is bit-identical. All 128 threads call it; f is valid in warps 0-2.
struct LinePair {
    Line d, a;
};

struct MillerSmem {
    LinePair lines[2][32];
    Fq6 xs[3][32];
};
__device__ __forceinline__ void f_bar() { asm volatile("bar.sync 1, 96;" ::: "memory"); }
__device__ __forceinline__ Fq12 f12_sqr_3w(const Fq12& a, Fq6 (*xs)[32], int w, int lane,
                                           bool active) {
    if (active && w < 2)
        xs[w][lane] = w == 0 ? f6_mul(a.c0, a.c1)
                             : f6_mul(f6_add(a.c0, a.c1), f6_add(a.c0, f6_mul_v(a.c1)));
    f_bar();
    const Fq6 ab = xs[0][lane], t = xs[1][lane];
    f_bar();
    return {f6_sub(f6_sub(t, ab), f6_mul_v(ab)), f6_add(ab, ab)};
}
__device__ __forceinline__ Fq12 f12_mul_line_3w(const Fq12& f, const Line& l, Fq6 (*xs)[32], int w,
                                                int lane, bool active) {
    if (active) {
        if (w == 0) xs[0][lane] = {fmul(f.c0.c0, l.l0), fmul(f.c0.c1, l.l0), fmul(f.c0.c2, l.l0)};
        else if (w == 1) xs[1][lane] = f6_mul_01(f.c1, l.l1, l.l2);
        else xs[2][lane] = f6_mul_01(f6_add(f.c0, f.c1), fadd(l.l0, l.l1), l.l2);
    }
    f_bar();
    const Fq6 t0 = xs[0][lane], t1 = xs[1][lane], t2 = xs[2][lane];
    f_bar();
    return {f6_add(t0, f6_mul_v(t1)), f6_sub(f6_sub(t2, t0), t1)};
}
__device__ __forceinline__ Fq12 miller_loop_4w(const Fq& xP, const Fq& yP, const Fq2& xQ,
                                               const Fq2& yQ, bool active, MillerSmem& sm) {
    const uint64_t loop_lo = 0x9d797039be763ba8ull;  // 6x+2 = 2^64 + loop_lo
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    Fq12 f = f12_one();
    G2Proj T;
    T.X = xQ;
    T.Y = yQ;
    fset_one(T.Z);
    for (int i = 63; i >= 0; --i) {
        const int par = i & 1;
        const bool bit = (loop_lo >> i) & 1;
        if (w == 3) {
            if (active) {
                sm.lines[par][lane].d = dbl_step(T, xP, yP);
                if (bit) sm.lines[par][lane].a = add_step(T, xQ, yQ, xP, yP);
            }
        } else {
            f = f12_sqr_3w(f, sm.xs, w, lane, active);
        }
        __syncthreads();
        if (w < 3) {
            f = f12_mul_line_3w(f, sm.lines[par][lane].d, sm.xs, w, lane, active);
            if (bit) f = f12_mul_line_3w(f, sm.lines[par][lane].a, sm.xs, w, lane, active);
        }
    }
    if (w == 3 && active) {  // lines[1] was last read before the i = 0 barrier
        Fq2 x1 = xQ, y1 = yQ;
        frob_twist(x1, y1);
        Fq2 x2 = x1, y2 = y1;
        frob_twist(x2, y2);
        sm.lines[1][lane].d = add_step(T, x1, y1, xP, yP);
        sm.lines[1][lane].a = add_step(T, x2, f2_neg(y2), xP, yP);
    }
    __syncthreads();
    if (w < 3) {
        f = f12_mul_line_3w(f, sm.lines[1][lane].d, sm.xs, w, lane, active);
        f = f12_mul_line_3w(f, sm.lines[1][lane].a, sm.xs, w, lane, active);
    }
    return f;
}

// Hard part ^((p^4 - p^2 + 1) / r) of an element of the cyclotomic subgroup.
static __device__ __noinline__ Fq12 final_exp_hard(const Fq12& t1) {
    const Fq12 fp = f12_frob(t1, 1), fp2 = f12_frob(t1, 2), fp3 = f12_frob(fp2, 1);
    const Fq12 fu = f12_pow_x(t1), fu2 = f12_pow_x(fu), fu3 = f12_pow_x(fu2);
    Fq12 y3 = f12_frob(fu, 1);
    const Fq12 fu2p = f12_frob(fu2, 1), fu3p = f12_frob(fu3, 1), y2 = f12_frob(fu2, 2);
    const Fq12 y0 = f12_mul(f12_mul(fp, fp2), fp3);
    const Fq12 y1 = f12_conj(t1);
    const Fq12 y5 = f12_conj(fu2);
    y3 = f12_conj(y3);
    const Fq12 y4 = f12_conj(f12_mul(fu, fu2p));
    const Fq12 y6 = f12_conj(f12_mul(fu3, fu3p));
    Fq12 t0 = f12_mul(f12_mul(f12_cyc_sqr(y6), y4), y5);
    Fq12 u1 = f12_mul(f12_mul(y3, y5), t0);
    t0 = f12_mul(t0, y2);
    u1 = f12_cyc_sqr(f12_mul(f12_cyc_sqr(u1), t0));
    t0 = f12_mul(u1, y1);
    u1 = f12_mul(u1, y0);
    t0 = f12_mul(f12_cyc_sqr(t0), u1);
    return t0;
}

// f^((p^12 - 1) / r).
static __device__ __noinline__ Fq12 final_exp(const Fq12& in) {
    Fq12 t1 = f12_mul(f12_conj(in), f12_inv(in));  // ^(p^6 - 1)
    t1 = f12_mul(t1, f12_frob(t1, 2));             // ^(p^2 + 1)
    return final_exp_hard(t1);
}


// ---- the final exponentiation on one warp, lane-parallel --------------------
// All 32 lanes hold the operands; lanes 0-17 each compute ONE of the 18 Fq2
// products of an Fq12 product (3 Karatsuba Fq6 products x 6 Fq2 products),
// or lanes 0-5 the 6 products of a cyclotomic squaring — the same product
// code on different data, so an Fq12 product costs one Fq2 product of
// latency. Products meet in a per-warp shared buffer; every lane then forms
// the (exact, order-independent) sums. Bit-identical to the serial forms.
struct WarpProducts {
    Fq2 p[32];
};
__device__ __forceinline__ Fq6 f6_from_products(const Fq2* p) {
    const Fq2 t0 = p[0], t1 = p[1], t2 = p[2];
    return {fadd(t0, f2_mul_xi(fsub(fsub(p[3], t1), t2))), fadd(fsub(fsub(p[4], t0), t1), f2_mul_xi(t2)),
            fadd(fsub(fsub(p[5], t0), t2), t1)};
}
static __device__ __noinline__ Fq12 f12_mul_warp(const Fq12& a, const Fq12& b, WarpProducts& ws) {
    const int lane = threadIdx.x & 31;
    const int which = lane < 18 ? lane / 6 : 0, j = lane % 6;
    const Fq6 x6 = which == 0 ? a.c0 : which == 1 ? a.c1 : f6_add(a.c0, a.c1);
    const Fq6 y6 = which == 0 ? b.c0 : which == 1 ? b.c1 : f6_add(b.c0, b.c1);
    Fq2 x, y;
    if (j < 3) {
        x = j == 0 ? x6.c0 : j == 1 ? x6.c1 : x6.c2;
        y = j == 0 ? y6.c0 : j == 1 ? y6.c1 : y6.c2;
    } else if (j == 3) {
        x = fadd(x6.c1, x6.c2);
        y = fadd(y6.c1, y6.c2);
    } else if (j == 4) {
        x = fadd(x6.c0, x6.c1);
        y = fadd(y6.c0, y6.c1);
    } else {
        x = fadd(x6.c0, x6.c2);
        y = fadd(y6.c0, y6.c2);
    }
    const Fq2 pr = fmul(x, y);
    if (lane < 18) ws.p[lane] = pr;
    __syncwarp();
    const Fq6 t0 = f6_from_products(ws.p), t1 = f6_from_products(ws.p + 6),
              t2 = f6_from_products(ws.p + 12);
    __syncwarp();
    return {f6_add(t0, f6_mul_v(t1)), f6_sub(f6_sub(t2, t0), t1)};
}
static __device__ __noinline__ Fq12 f12_cyc_sqr_warp(const Fq12& a, WarpProducts& ws) {
    const int lane = threadIdx.x & 31;
    const int w = lane < 6 ? lane >> 1 : 0;
    const Fq2 x = w == 0 ? a.c0.c0 : w == 1 ? a.c1.c0 : a.c0.c1;
    const Fq2 y = w == 0 ? a.c1.c1 : w == 1 ? a.c0.c2 : a.c1.c2;
    const Fq2 pr = (lane & 1) ? fmul(fadd(x, y), fadd(x, f2_mul_xi(y))) : fmul(x, y);
    if (lane < 6) ws.p[lane] = pr;
    __syncwarp();
    Fq2 t[6];
#pragma unroll
    for (int k = 0; k < 3; ++k) {  // (x + y t)^2 = ((x+y)(x+xi y) - xy - xi xy) + 2xy t
        const Fq2 xy = ws.p[2 * k];
        t[2 * k] = fsub(fsub(ws.p[2 * k + 1], xy), f2_mul_xi(xy));
        t[2 * k + 1] = fadd(xy, xy);
    }
    __syncwarp();
    auto tw = [](const Fq2& tt, const Fq2& z, bool plus) {  // 3t -+ 2z
        const Fq2 d = plus ? fadd(tt, z) : fsub(tt, z);
        return fadd(fadd(d, d), tt);
    };
    Fq12 r;
    r.c0.c0 = tw(t[0], a.c0.c0, false);
    r.c1.c1 = tw(t[1], a.c1.c1, true);
    r.c1.c0 = tw(f2_mul_xi(t[5]), a.c1.c0, true);
    r.c0.c2 = tw(t[4], a.c0.c2, false);
    r.c0.c1 = tw(t[2], a.c0.c1, false);
    r.c1.c2 = tw(t[3], a.c1.c2, true);
    return r;
}
__device__ __forceinline__ Fq12 f12_pow_x_warp(const Fq12& a, WarpProducts& ws) {
    const uint64_t x = 4965661367192848881ull;
    Fq12 r = f12_one();
    for (int i = 62; i >= 0; --i) {
        r = f12_cyc_sqr_warp(r, ws);
        if ((x >> i) & 1) r = f12_mul_warp(r, a, ws);
    }
    return r;
}
// Every lane of ONE warp calls it; the result is replicated in all lanes.
static __device__ __noinline__ Fq12 final_exp_warp(const Fq12& in, WarpProducts& ws) {
    Fq12 t1 = f12_mul_warp(f12_conj(in), f12_inv(in), ws);  // ^(p^6 - 1)
    t1 = f12_mul_warp(t1, f12_frob(t1, 2), ws);             // ^(p^2 + 1)
    const Fq12 fp = f12_frob(t1, 1), fp2 = f12_frob(t1, 2), fp3 = f12_frob(fp2, 1);
    const Fq12 fu = f12_pow_x_warp(t1, ws), fu2 = f12_pow_x_warp(fu, ws),
               fu3 = f12_pow_x_warp(fu2, ws);
    Fq12 y3 = f12_frob(fu, 1);
    const Fq12 fu2p = f12_frob(fu2, 1), fu3p = f12_frob(fu3, 1), y2 = f12_frob(fu2, 2);
    const Fq12 y0 = f12_mul_warp(f12_mul_warp(fp, fp2, ws), fp3, ws);
    const Fq12 y1 = f12_conj(t1);
    const Fq12 y5 = f12_conj(fu2);
    y3 = f12_conj(y3);
    const Fq12 y4 = f12_conj(f12_mul_warp(fu, fu2p, ws));
    const Fq12 y6 = f12_conj(f12_mul_warp(fu3, fu3p, ws));
    Fq12 t0 = f12_mul_warp(f12_mul_warp(f12_cyc_sqr_warp(y6, ws), y4, ws), y5, ws);
    Fq12 u1 = f12_mul_warp(f12_mul_warp(y3, y5, ws), t0, ws);
    t0 = f12_mul_warp(t0, y2, ws);
    u1 = f12_cyc_sqr_warp(f12_mul_warp(f12_cyc_sqr_warp(u1, ws), t0, ws), ws);
    t0 = f12_mul_warp(u1, y1, ws);
    u1 = f12_mul_warp(u1, y0, ws);
    return f12_mul_warp(f12_cyc_sqr_warp(t0, ws), u1, ws);
}

}  // namespace bn
}  // namespace ace_gpu
