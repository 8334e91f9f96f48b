// BN254 G1 (y^2 = x^3 + 3 over Fq) and G2 (y^2 = x^3 + 3/(9+u) over
// Fq2 = Fq[u]/(u^2 + 1)) for sm_100a. Bucket accumulators use XYZZ
// coordinates (x = X/ZZ, y = Y/ZZZ; ZZ = 0 is the point at infinity) with the
// madd-2008-s / add-2008-s / dbl-2008-s-1 formulas (a = 0): a mixed add costs
// 8M + 2S, a general add 12M + 2S. Fq2 multiplication is Karatsuba (3 Fq muls).
#pragma once
#include "bn254.cuh"

namespace ace_gpu {
namespace bn {

struct Fq2 {
    Fq c0, c1;
};

// ---- uniform field interface (Fq and Fq2) ---------------------------------
// The Fq multiplication is ~530 SASS instructions; curve formulas call it a
// dozen times per point operation, so it is an out-of-line call here
// (inlined, a bucket kernel's body exceeded 1 MB of code and thrashed the
// instruction caches; see profiles/). NTT kernels keep the inline `mul`.
#ifndef ACEGPU_FQ2_SHARED
#define ACEGPU_FQ2_SHARED 1  // Fq2 units call one shared 512-bit product / reduction body
#endif
struct W16 {
    uint32_t v[16];
};
#if ACEGPU_FQ2_SHARED
// The G2 bucket loop was instruction-fetch bound with the products inlined
// into each Fq2 unit (ncu: stalled_no_instruction ~1 per issue); one
// out-of-line body each keeps the loop's code small.
static __device__ __noinline__ W16 fq_mul_wide_call(const Fq a, const Fq b) {
    W16 w;
    mul_wide(a, b, w.v);
    return w;
}
static __device__ __noinline__ Fq fq_redc_call(const W16 w) { return redc_wide<FqCfg>(w.v); }
#ifndef ACEGPU_REDC2
#define ACEGPU_REDC2 1
#endif
#if ACEGPU_REDC2
// Both coordinates' reductions in one body: two independent carry chains the
// scheduler interleaves (ILP for the low-occupancy G2 loop).
struct Fq2Pair {
    Fq a, b;
};
static __device__ __noinline__ Fq2Pair fq_redc2_call(const W16 x, const W16 y) {
    return {redc_wide<FqCfg>(x.v), redc_wide<FqCfg>(y.v)};
}
#define ACE_REDC2(x, y) ([&] { const Fq2Pair r_ = fq_redc2_call(x, y); return Fq2{r_.a, r_.b}; }())
#ifndef ACEGPU_WIDE2
#define ACEGPU_WIDE2 0  // 1: two 512-bit products per call (measured chunk 50.4 vs 49.4 ms)
#endif
struct W16Pair {
    W16 x, y;
};
static __device__ __noinline__ W16Pair fq_mul_wide2_call(const Fq a, const Fq b, const Fq c,
                                                         const Fq d) {
    W16Pair r;
    mul_wide(a, b, r.x.v);
    mul_wide(c, d, r.y.v);
    return r;
}
#else
#define ACE_REDC2(x, y) (Fq2{fq_redc_call(x), fq_redc_call(y)})
#endif
#else
__device__ __forceinline__ W16 fq_mul_wide_call(const Fq& a, const Fq& b) {
    W16 w;
    mul_wide(a, b, w.v);
    return w;
}
__device__ __forceinline__ Fq fq_redc_call(const W16& w) { return redc_wide<FqCfg>(w.v); }
#endif
#ifndef ACEGPU_ONE_BODY
#define ACEGPU_ONE_BODY 0  // 1: G1 products through the G2 bodies too (measured 51.0 vs 50.7 ms chunk)
#endif
#if ACEGPU_ONE_BODY && ACEGPU_FQ2_SHARED
static __device__ __noinline__ Fq fq_mul_call(const Fq a, const Fq b) {
    return fq_redc_call(fq_mul_wide_call(a, b));
}
#else
static __device__ __noinline__ Fq fq_mul_call(const Fq a, const Fq b) { return mul(a, b); }
#endif
__device__ __forceinline__ Fq fmul(const Fq& a, const Fq& b) { return fq_mul_call(a, b); }
#ifndef ACEGPU_G1_MUL2
#define ACEGPU_G1_MUL2 0  // 1: G1 products two per call (measured slower: G1 2^20 4.37 vs 4.23 ms)
#endif
struct FqPair2 {
    Fq a, b;
};
// two independent products in one body: the scheduler interleaves the chains
static __device__ __noinline__ FqPair2 fq_mul2_call(const Fq a, const Fq b, const Fq c,
                                                    const Fq d) {
    return {mul(a, b), mul(c, d)};
}
// (A dedicated out-of-line squaring, 208 IMAD, measured slower in the bucket
// loop than reusing the one product routine: a second 500-instruction body.)
__device__ __forceinline__ Fq fsqr(const Fq& a) { return fq_mul_call(a, a); }
__device__ __forceinline__ Fq fadd(const Fq& a, const Fq& b) { return add(a, b); }
__device__ __forceinline__ Fq fsub(const Fq& a, const Fq& b) { return sub(a, b); }
__device__ __forceinline__ bool fzero(const Fq& a) { return a.is_zero(); }
__device__ __forceinline__ void fset_one(Fq& a) { a = Fq::one(); }
__device__ __forceinline__ void fset_zero(Fq& a) { a = Fq::zero(); }
__device__ __forceinline__ bool feq(const Fq& a, const Fq& b) { return a == b; }

// Fq2 products: Karatsuba over out-of-line Fq products. (Inlining the three
// Fq products into one out-of-line Fq2 unit measured 8 % slower.)
#ifndef ACEGPU_LAZY
#define ACEGPU_LAZY 1  // lazy-reduced Karatsuba / product differences (0: one reduction per product)
#endif
#if ACEGPU_LAZY
// Karatsuba on 512-bit products: c0 = a0 b0 - a1 b1 in [0, p 2^256),
// c1 = (a0 + a1)(b0 + b1) - a0 b0 - a1 b1 = a0 b1 + a1 b0 in [0, 2p^2):
// three products, two reductions (656 IMAD vs 792).
__device__ __forceinline__ void fq2_mul_wide(const Fq2& a, const Fq2& b, W16& c0, W16& c1) {
#if ACEGPU_REDC2 && ACEGPU_WIDE2
    const W16Pair p01 = fq_mul_wide2_call(a.c0, b.c0, a.c1, b.c1);  // two chains interleaved
    c0 = p01.x;
    const W16 w1 = p01.y;
#else
    c0 = fq_mul_wide_call(a.c0, b.c0);
    const W16 w1 = fq_mul_wide_call(a.c1, b.c1);
#endif
    c1 = fq_mul_wide_call(add_raw(a.c0, a.c1), add_raw(b.c0, b.c1));
    sub_wide(c1.v, c0.v);
    sub_wide(c1.v, w1.v);
    add_mR_masked<FqCfg>(c0.v, sub_wide(c0.v, w1.v));
}
#ifndef ACEGPU_G2_F64
#define ACEGPU_G2_F64 1  // Fq2 products through the FP64 wide product (W10) + one redc10 each
#endif
#if ACEGPU_G2_F64
// FP64-domain Karatsuba: three 16 a b column products, sums / differences
// column-wise, two reductions (bn254.cuh W10 / redc10).
static __device__ __noinline__ W10 fq_mulw10_call(const Fq a, const Fq b) {
    W10 w;
    mul_wide10(a, b, w);
    return w;
}
static __device__ __noinline__ Fq2Pair fq_redc10x2_call(const W10 x, const W10 y) {
    return {redc10<FqCfg>(x), redc10<FqCfg>(y)};
}
// c0 = 16 (a0 b0 - a1 b1) (signed), c1 = 16 (a0 b1 + a1 b0) >= 0
__device__ __forceinline__ void fq2_mul_wide10(const Fq2& a, const Fq2& b, W10& c0, W10& c1) {
    c0 = fq_mulw10_call(a.c0, b.c0);
    const W10 t1 = fq_mulw10_call(a.c1, b.c1);
    c1 = fq_mulw10_call(add_raw(a.c0, a.c1), add_raw(b.c0, b.c1));
    w10_sub(c1, c0);
    w10_sub(c1, t1);
    w10_sub(c0, t1);
}
static __device__ __noinline__ Fq2 fq2_mul_call(const Fq2 a, const Fq2 b) {
    W10 c0, c1;
    fq2_mul_wide10(a, b, c0, c1);
    w10_add_m260<FqCfg>(c0);
    const Fq2Pair r = fq_redc10x2_call(c0, c1);
    return {r.a, r.b};
}
// a b - c d over Fq2: six products, two reductions.
static __device__ __noinline__ Fq2 fq2_mul_sub_call(const Fq2 a, const Fq2 b, const Fq2 c,
                                                    const Fq2 d) {
    W10 x0, x1, y0, y1;
    fq2_mul_wide10(a, b, x0, x1);
    fq2_mul_wide10(c, d, y0, y1);
    w10_sub(x0, y0);
    w10_sub(x1, y1);
    w10_add_m260<FqCfg>(x0);
    w10_add_m260<FqCfg>(x1);
    const Fq2Pair r = fq_redc10x2_call(x0, x1);
    return {r.a, r.b};
}
#else
static __device__ __noinline__ Fq2 fq2_mul_call(const Fq2 a, const Fq2 b) {
    W16 c0, c1;
    fq2_mul_wide(a, b, c0, c1);
    return ACE_REDC2(c0, c1);
}
// a b - c d over Fq2: six products, two reductions.
static __device__ __noinline__ Fq2 fq2_mul_sub_call(const Fq2 a, const Fq2 b, const Fq2 c,
                                                    const Fq2 d) {
    W16 x0, x1, y0, y1;
    fq2_mul_wide(a, b, x0, x1);
    fq2_mul_wide(c, d, y0, y1);
    add_mR_masked<FqCfg>(x0.v, sub_wide(x0.v, y0.v));
    add_mR_masked<FqCfg>(x1.v, sub_wide(x1.v, y1.v));
    return ACE_REDC2(x0, x1);
}
#endif
#if ACEGPU_ONE_BODY && ACEGPU_FQ2_SHARED
__device__ __forceinline__ Fq fq_mul_sub_call(const Fq& a, const Fq& b, const Fq& c, const Fq& d) {
    W16 w = fq_mul_wide_call(a, b);
    const W16 x = fq_mul_wide_call(c, d);
    add_mR_masked<FqCfg>(w.v, sub_wide(w.v, x.v));
    return fq_redc_call(w);
}
#elif ACEGPU_G2_F64 && !ACEGPU_G1_MULSUB_CIOS
// a b - c d: two FP64 wide products, one reduction (|16 (ab - cd)| < p 2^260)
static __device__ __noinline__ Fq fq_mul_sub_call(const Fq a, const Fq b, const Fq c, const Fq d) {
    W10 w, x;
    mul_wide10(a, b, w);
    mul_wide10(c, d, x);
    w10_sub(w, x);
    w10_add_m260<FqCfg>(w);
    return redc10<FqCfg>(w);
}
#else
static __device__ __noinline__ Fq fq_mul_sub_call(const Fq a, const Fq b, const Fq c, const Fq d) {
    return mul_sub_mul(a, b, c, d);
}
#endif
__device__ __forceinline__ Fq2 fmul(const Fq2& a, const Fq2& b) { return fq2_mul_call(a, b); }
__device__ __forceinline__ Fq fmul_sub(const Fq& a, const Fq& b, const Fq& c, const Fq& d) {
    return fq_mul_sub_call(a, b, c, d);
}
__device__ __forceinline__ Fq2 fmul_sub(const Fq2& a, const Fq2& b, const Fq2& c, const Fq2& d) {
    return fq2_mul_sub_call(a, b, c, d);
}
#else
__device__ __forceinline__ Fq2 fmul(const Fq2& a, const Fq2& b) {
    Fq t0 = fq_mul_call(a.c0, b.c0), t1 = fq_mul_call(a.c1, b.c1);
    Fq t2 = fq_mul_call(add(a.c0, a.c1), add(b.c0, b.c1));
    return {sub(t0, t1), sub(sub(t2, t0), t1)};
}
#endif
#if ACEGPU_G2_F64
// (c0 + c1 u)^2 = (c0 + c1)(c0 - c1) + 2 c0 c1 u: two FP64 wide products
// (both non-negative, below 32 p^2), two reductions.
__device__ __forceinline__ Fq2 fsqr(const Fq2& a) {
    W10 t = fq_mulw10_call(a.c0, a.c1);
    const W10 u = fq_mulw10_call(add_raw(a.c0, a.c1), sub(a.c0, a.c1));
    w10_shl1(t);
    const Fq2Pair r = fq_redc10x2_call(u, t);
    return {r.a, r.b};
}
#elif ACEGPU_LAZY && ACEGPU_FQ2_SHARED
// (c0 + c1 u)^2 = (c0 + c1)(c0 - c1) + 2 c0 c1 u through the shared wide
// bodies: (c0 + c1) unreduced times (c0 - c1) mod p < 2p^2, and 2 c0 c1 <
// 2p^2 (a one-bit shift of the 512-bit product), both below p 2^256.
__device__ __forceinline__ Fq2 fsqr(const Fq2& a) {
#if ACEGPU_REDC2 && ACEGPU_WIDE2
    const W16Pair p = fq_mul_wide2_call(a.c0, a.c1, add_raw(a.c0, a.c1), sub(a.c0, a.c1));
    W16 t = p.x;
    const W16 u = p.y;
#else
    W16 t = fq_mul_wide_call(a.c0, a.c1);
    const W16 u = fq_mul_wide_call(add_raw(a.c0, a.c1), sub(a.c0, a.c1));
#endif
#pragma unroll
    for (int k = 15; k > 0; --k) t.v[k] = __funnelshift_l(t.v[k - 1], t.v[k], 1);
    t.v[0] <<= 1;
    return ACE_REDC2(u, t);
}
#else
__device__ __forceinline__ Fq2 fsqr(const Fq2& a) {
    // (c0 + c1 u)^2 = (c0 + c1)(c0 - c1) + 2 c0 c1 u
    Fq t = fq_mul_call(a.c0, a.c1);
    return {fq_mul_call(add(a.c0, a.c1), sub(a.c0, a.c1)), add(t, t)};
}
#endif

// Selectable inlining: the G1 bucket-accumulation loop inlines its Fq
// multiplications (one madd body, ILP across independent products).
template <bool INL>
__device__ __forceinline__ Fq fmul_s(const Fq& a, const Fq& b) {
    if constexpr (INL) return mul(a, b);
    else return fq_mul_call(a, b);
}
template <bool INL>
__device__ __forceinline__ Fq2 fmul_s(const Fq2& a, const Fq2& b) { return fmul(a, b); }
__device__ __forceinline__ Fq2 fadd(const Fq2& a, const Fq2& b) {
    return {add(a.c0, b.c0), add(a.c1, b.c1)};
}
__device__ __forceinline__ Fq2 fsub(const Fq2& a, const Fq2& b) {
    return {sub(a.c0, b.c0), sub(a.c1, b.c1)};
}
#if !ACEGPU_LAZY
template <class F>
__device__ __forceinline__ F fmul_sub(const F& a, const F& b, const F& c, const F& d) {
    return fsub(fmul(a, b), fmul(c, d));
}
#endif
__device__ __forceinline__ bool fzero(const Fq2& a) { return a.c0.is_zero() && a.c1.is_zero(); }
__device__ __forceinline__ void fset_one(Fq2& a) { a.c0 = Fq::one(); a.c1 = Fq::zero(); }
__device__ __forceinline__ void fset_zero(Fq2& a) { a.c0 = Fq::zero(); a.c1 = Fq::zero(); }
__device__ __forceinline__ bool feq(const Fq2& a, const Fq2& b) { return a.c0 == b.c0 && a.c1 == b.c1; }

template <class F>
struct Affine {
    F x, y;  // infinity encoded by the caller (all-zero record)
};

template <class F>
struct XYZZ {
    F X, Y, ZZ, ZZZ;

    __device__ __forceinline__ static XYZZ inf() {
        XYZZ p;
        fset_one(p.X);
        fset_one(p.Y);
        fset_zero(p.ZZ);
        fset_zero(p.ZZZ);
        return p;
    }
    __device__ __forceinline__ bool is_inf() const { return fzero(ZZ); }
};

// dbl-2008-s-1 on an XYZZ point (a = 0).
template <class F>
__device__ __forceinline__ XYZZ<F> xyzz_dbl(const XYZZ<F>& p) {
    if (p.is_inf()) return p;
    F U = fadd(p.Y, p.Y);
    F V = fsqr(U);
    F W = fmul(U, V);
    F S = fmul(p.X, V);
    F X2 = fsqr(p.X);
    F M = fadd(fadd(X2, X2), X2);
    XYZZ<F> r;
    r.X = fsub(fsub(fsqr(M), S), S);
    r.Y = fmul_sub(M, fsub(S, r.X), W, p.Y);
    r.ZZ = fmul(V, p.ZZ);
    r.ZZZ = fmul(W, p.ZZZ);
    return r;
}

// mdbl: double an affine point into XYZZ.
template <class F>
__device__ __forceinline__ XYZZ<F> xyzz_mdbl(const F& x, const F& y) {
    F U = fadd(y, y);
    F V = fsqr(U);
    F W = fmul(U, V);
    F S = fmul(x, V);
    F X2 = fsqr(x);
    F M = fadd(fadd(X2, X2), X2);
    XYZZ<F> r;
    r.X = fsub(fsub(fsqr(M), S), S);
    r.Y = fmul_sub(M, fsub(S, r.X), W, y);
    r.ZZ = V;
    r.ZZZ = W;
    return r;
}

// madd-2008-s: p + (x, y) with (x, y) affine, not infinity. INL inlines the
// ten Fq products (independent pairs interleave); the rare doubling path
// stays out of line.
template <class F, bool INL = false>
__device__ __forceinline__ XYZZ<F> xyzz_madd(const XYZZ<F>& p, const F& x, const F& y) {
    if (p.is_inf()) {
        XYZZ<F> r;
        r.X = x;
        r.Y = y;
        fset_one(r.ZZ);
        fset_one(r.ZZZ);
        return r;
    }
#if ACEGPU_G1_MUL2
    if constexpr (sizeof(F) == sizeof(Fq) && !INL) {
        // G1: the ten products as four independent pairs + the lazy Y3
        const FqPair2 us = fq_mul2_call(x, p.ZZ, y, p.ZZZ);
        const F P = fsub(us.a, p.X);
        const F R = fsub(us.b, p.Y);
        if (fzero(P)) {
            if (fzero(R)) return xyzz_mdbl(x, y);
            return XYZZ<F>::inf();
        }
        const FqPair2 sq = fq_mul2_call(P, P, R, R);  // PP, R^2
        const FqPair2 pq = fq_mul2_call(P, sq.a, p.X, sq.a);  // PPP, Q
        XYZZ<F> r;
        r.X = fsub(fsub(fsub(sq.b, pq.a), pq.b), pq.b);
        const FqPair2 zz = fq_mul2_call(p.ZZ, sq.a, p.ZZZ, pq.a);
        r.ZZ = zz.a;
        r.ZZZ = zz.b;
        r.Y = fmul_sub(R, fsub(pq.b, r.X), p.Y, pq.a);
        return r;
    }
#endif
    F U2 = fmul_s<INL>(x, p.ZZ);
    F S2 = fmul_s<INL>(y, p.ZZZ);
    F P = fsub(U2, p.X);
    F R = fsub(S2, p.Y);
    if (fzero(P)) {
        if (fzero(R)) return xyzz_mdbl(x, y);
        return XYZZ<F>::inf();
    }
    F PP = fsqr(P);
    F PPP = fmul_s<INL>(P, PP);
    F Q = fmul_s<INL>(p.X, PP);
    F R2 = fsqr(R);
    XYZZ<F> r;
    r.ZZ = fmul_s<INL>(p.ZZ, PP);
    r.ZZZ = fmul_s<INL>(p.ZZZ, PPP);
    r.X = fsub(fsub(fsub(R2, PPP), Q), Q);
    r.Y = fmul_sub(R, fsub(Q, r.X), p.Y, PPP);
    return r;
}

// add-2008-s: general XYZZ + XYZZ.
template <class F>
__device__ __forceinline__ XYZZ<F> xyzz_add(const XYZZ<F>& p, const XYZZ<F>& q) {
    if (p.is_inf()) return q;
    if (q.is_inf()) return p;
    F U1 = fmul(p.X, q.ZZ);
    F U2 = fmul(q.X, p.ZZ);
    F S1 = fmul(p.Y, q.ZZZ);
    F S2 = fmul(q.Y, p.ZZZ);
    F P = fsub(U2, U1);
    F R = fsub(S2, S1);
    if (fzero(P)) {
        if (fzero(R)) return xyzz_dbl(p);
        return XYZZ<F>::inf();
    }
    F PP = fsqr(P);
    F PPP = fmul(P, PP);
    F Q = fmul(U1, PP);
    XYZZ<F> r;
    r.X = fsub(fsub(fsub(fsqr(R), PPP), Q), Q);
    r.Y = fmul_sub(R, fsub(Q, r.X), S1, PPP);
    r.ZZ = fmul(fmul(p.ZZ, q.ZZ), PP);
    r.ZZZ = fmul(fmul(p.ZZZ, q.ZZZ), PPP);
    return r;
}

template <class F>
__device__ __forceinline__ XYZZ<F> xyzz_neg(const XYZZ<F>& p) {
    XYZZ<F> r = p;
    F z;
    fset_zero(z);
    r.Y = fsub(z, p.Y);
    return r;
}

// k * p for a small scalar k (double-and-add, MSB first, from k's top bit:
// the bucket weights of a reduction are < 2^20, so 12+ doublings of the
// point at infinity are skipped).
template <class F>
__device__ XYZZ<F> xyzz_mul_small(const XYZZ<F>& p, uint32_t k) {
    if (!k) return XYZZ<F>::inf();
    XYZZ<F> r = p;
    for (int b = 30 - __clz(k); b >= 0; --b) {
        r = xyzz_dbl(r);
        if ((k >> b) & 1) r = xyzz_add(r, p);
    }
    return r;
}

// ---- element / point I/O (Montgomery form in memory, 16-B aligned) --------
__device__ __forceinline__ void fload(Fq& a, const uint8_t* p) { a = load<FqCfg>(p); }
__device__ __forceinline__ void fload(Fq2& a, const uint8_t* p) {
    a.c0 = load<FqCfg>(p);
    a.c1 = load<FqCfg>(p + 32);
}
__device__ __forceinline__ void fstore(uint8_t* p, const Fq& a) { store<FqCfg>(p, a); }
__device__ __forceinline__ void fstore(uint8_t* p, const Fq2& a) {
    store<FqCfg>(p, a.c0);
    store<FqCfg>(p + 32, a.c1);
}
template <class F>
constexpr int felem_bytes() { return sizeof(F) == sizeof(Fq) ? 32 : 64; }

}  // namespace bn
}  // namespace ace_gpu
