// Fr NTT / iNTT / coset-NTT for sm_100a (north-star row a21; the reference
// has none). Natural order in and out.
//
// Four-step decomposition n = n1 * n2 (n1 = 2^L1, n2 = 2^L2, L2 = ceil(L/2)):
//   i = i1 + n1*i2, k = k2 + n2*k1
//   pass A: for each column i1, the size-n2 DFT over i2 of a[i1 + n1*i2],
//           times the twiddle w^(i1*k2), stored at i1 + n1*k2 (scratch);
//   pass C: for each k2, the size-n1 DFT over i1 of that row, stored at
//           X[k2 + n2*k1] (natural order).
// Each CTA owns R adjacent columns (pass A) / rows (pass C) so global
// accesses are R*32-B contiguous; the sub-DFT runs entirely in shared memory
// (bit-reversed load + radix-2 DIT stages), twiddles from small L1-resident
// tables. Coset scaling (g^i on input) and the inverse's n^-1 (and g^-k) are
// fused into the loads / stores. Compute: log2(n)/2 + 2 Fr muls per element,
// IMAD-pipe bound (NTT at 2^21-2^22 is ~8x above the HBM ridge).
//
// Above 2^22 (a whole block's domain, up to 2^28 = 8.6 GB per vector) pass A's
// column DFT of length n2 = p q no longer fits shared memory and is itself
// split (n = nC p q, i = i1 + nC (u + p v), k2 = s + q t):
//   pass B1: for each (i1, u), the q-point DFT over v, times w^(nC u s),
//            written back in place (the CTA rewrites exactly what it read);
//   pass B2: for each (i1, s), the p-point DFT over u, times w^(i1 k2), to
//            i1 + nC k2 (scratch) — pass A's output;
//   pass C : as above with n1 = nC. Twiddle / coset tables are split lo/hi
//            (the n-entry tables would be 8.6 GB each at 2^28).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "bn254.cuh"
#include "ntt.cuh"

namespace ace_gpu {
namespace bn {

namespace {

__device__ __forceinline__ Fr ld(const Fr* p) { return load<FrCfg>(p); }
__device__ __forceinline__ void st(Fr* p, const Fr& x) { store<FrCfg>(p, x); }

// Pass kernels' occupancy: the FP64 product needs ~84 registers; the passes
// are sized so several CTAs share an SM (loads of one CTA overlap another's
// butterflies). ACEGPU_NTT_CIOS=1 uses the IMAD product (fewer registers)
// inside the NTT instead.
// Passes A / C run 256-thread CTAs, three per SM (the 64 KB sub-DFT of
// 2^21-2^22 allows three): 80 registers without spills, against 512 x 2 at
// 64 registers with 150-200 B of spills (2^21 forward 0.631 -> 0.564 ms,
// 2^22 1.261 -> 1.124, 2^26 23.6 -> 22.2; 256 x 2 and 256 x 4 in between).
#ifndef ACEGPU_NTT_AC_THREADS
#define ACEGPU_NTT_AC_THREADS 256
#endif
#ifndef ACEGPU_NTT_AC_MINB
#define ACEGPU_NTT_AC_MINB 3
#endif
#ifndef ACEGPU_NTT_CIOS
#define ACEGPU_NTT_CIOS 0
#endif
#if ACEGPU_NTT_CIOS
__device__ __forceinline__ Fr mul(const Fr& a, const Fr& b) { return mul_cios(a, b); }
#endif

// Shared-memory sub-DFT arrays are planar: the low and high 16 B of element
// i live at plane 0 / plane 1 index i, so a warp's 16-B accesses to
// consecutive elements are contiguous (4 wavefronts, no bank conflicts)
// instead of 32-B strided (8 wavefronts; ncu: 61 % of the shared wavefronts
// were conflicts with the interleaved layout).
#ifndef ACEGPU_NTT_PLANAR
#define ACEGPU_NTT_PLANAR 1
#endif
struct SmemFr {
    uint4* base;
    uint32_t n;  // elements
    __device__ __forceinline__ Fr get(uint32_t i) const {
        if constexpr (ACEGPU_NTT_PLANAR) {
            const uint4 lo = base[i], hi = base[n + i];
            Fr r;
            r.v[0] = lo.x; r.v[1] = lo.y; r.v[2] = lo.z; r.v[3] = lo.w;
            r.v[4] = hi.x; r.v[5] = hi.y; r.v[6] = hi.z; r.v[7] = hi.w;
            return r;
        } else {
            return ld(reinterpret_cast<const Fr*>(base) + i);
        }
    }
    __device__ __forceinline__ void put(uint32_t i, const Fr& x) const {
        if constexpr (ACEGPU_NTT_PLANAR) {
            base[i] = make_uint4(x.v[0], x.v[1], x.v[2], x.v[3]);
            base[n + i] = make_uint4(x.v[4], x.v[5], x.v[6], x.v[7]);
        } else {
            st(reinterpret_cast<Fr*>(base) + i, x);
        }
    }
};

__device__ __forceinline__ uint32_t bitrev(uint32_t x, int bits) {
    return __brev(x) >> (32 - bits);
}

// Shared-memory sub-DFT of size 2^m over R interleaved batches:
// element (r, j) lives at s[j * R + r]. In: bit-reversed; out: natural.
template <int R>  // compile-time: the index arithmetic divides by it
__device__ __forceinline__ void smem_dit(const SmemFr& s, int m, const Fr* __restrict__ w) {
    const int half_n = 1 << (m - 1);
    const int total = half_n * R;
    for (int stage = 0; stage < m; ++stage) {
        const int half = 1 << stage;
        const int tw_shift = m - 1 - stage;  // w_sub^(j << tw_shift)
        for (int b = threadIdx.x; b < total; b += blockDim.x) {
            const int r = b % R;
            const int bf = b / R;
            const int j = bf & (half - 1);
            const int base = ((bf >> stage) << (stage + 1)) + j;
            const uint32_t iu = base * R + r, iv = (base + half) * R + r;
            Fr u = s.get(iu), v = s.get(iv);
            if (j) v = mul(v, ld(&w[j << tw_shift]));
            s.put(iu, add(u, v));
            s.put(iv, sub(u, v));
        }
        __syncthreads();
    }
}

struct PassArgs {
    const uint8_t* in;
    uint8_t* out;
    int L, L1, L2, R;
    const Fr* w_sub;     // roots of the sub-DFT (size 2^(m-1))
    const Fr* tw_lo;     // pass A: w^e for e < n2 ; pass C: unused
    const Fr* tw_hi;     // pass A: w^(n2*e) for e < n1
    const Fr* tw_full;   // pass A: w^e for e < n (replaces tw_lo * tw_hi when present)
    const Fr* pre_full;  // pass A coset: g^idx (replaces pre_lo * pre_hi)
    const Fr* post_full; // pass C coset: n^-1 g^-idx (replaces post_lo * post_hi)
    const Fr* pre_lo;    // pass A coset: g^i1 (n1) ; single: g^i (n)
    const Fr* pre_hi;    // pass A coset: g^(n1*i2) (n2)
    const Fr* post_lo;   // pass C: scale_k2 (n2), e.g. n^-1 g^-k2
    const Fr* post_hi;   // pass C: g^(-n2*k1) (n1)
    const Fr* scale;     // uniform output scale (n^-1) when post tables are absent
    uint64_t bstride;    // batch (blockIdx.y): elements between transforms (pass A / C)
};

// Pass A: columns i1 in [cb*R, cb*R+R), DFT length n2 over i2.
__global__ void __launch_bounds__(ACEGPU_NTT_AC_THREADS, ACEGPU_NTT_AC_MINB) ntt_pass_a(PassArgs a) {
    extern __shared__ uint4 smem_raw[];
    const int n1 = 1 << a.L1, n2 = 1 << a.L2;
    constexpr int R = kNttR;
    const SmemFr s{smem_raw, uint32_t(n2 * R)};
    const int i1_0 = blockIdx.x * R;
    const uint8_t* in = a.in + 32 * a.bstride * blockIdx.y;
    uint8_t* out = a.out + 32 * a.bstride * blockIdx.y;
    for (int e = threadIdx.x; e < n2 * R; e += blockDim.x) {
        const int r = e % R, i2 = e / R;
        const int i1 = i1_0 + r;
        const uint64_t idx = i1 + (uint64_t)n1 * i2;
        Fr x = load<FrCfg>(in + 32 * idx);
        if (a.pre_full) x = mul(x, ld(&a.pre_full[idx]));
        else if (a.pre_lo) x = mul(x, mul(ld(&a.pre_lo[i1]), ld(&a.pre_hi[i2])));
        s.put(bitrev(i2, a.L2) * R + r, x);
    }
    __syncthreads();
    smem_dit<R>(s, a.L2, a.w_sub);
    for (int e = threadIdx.x; e < n2 * R; e += blockDim.x) {
        const int r = e % R, k2 = e / R;
        const int i1 = i1_0 + r;
        Fr x = s.get(k2 * R + r);
        // twiddle w^(i1*k2), exponent < n, split as lo (L2 bits) + hi
        const uint64_t ex = (uint64_t)i1 * k2;
        if (a.tw_full) {
            if (ex) x = mul(x, ld(&a.tw_full[ex]));
        } else {
            const uint32_t lo = ex & (n2 - 1), hi = ex >> a.L2;
            if (ex) x = mul(x, mul(ld(&a.tw_lo[lo]), ld(&a.tw_hi[hi])));
        }
        store<FrCfg>(out + 32 * (i1 + (uint64_t)n1 * k2), x);
    }
}

// Pass C: rows k2 in [rb*R, rb*R+R), DFT length n1 over i1; natural output.
__global__ void __launch_bounds__(ACEGPU_NTT_AC_THREADS, ACEGPU_NTT_AC_MINB) ntt_pass_c(PassArgs a) {
    extern __shared__ uint4 smem_raw[];
    const int n1 = 1 << a.L1, n2 = 1 << a.L2;
    constexpr int R = kNttR;
    const SmemFr s{smem_raw, uint32_t(n1 * R)};
    const int k2_0 = blockIdx.x * R;
    const uint8_t* in = a.in + 32 * a.bstride * blockIdx.y;
    uint8_t* out = a.out + 32 * a.bstride * blockIdx.y;
    for (int e = threadIdx.x; e < n1 * R; e += blockDim.x) {
        const int r = e % R, i1 = e / R;
        const uint64_t idx = i1 + (uint64_t)n1 * (k2_0 + r);
        s.put(bitrev(i1, a.L1) * R + r, load<FrCfg>(in + 32 * idx));
    }
    __syncthreads();
    smem_dit<R>(s, a.L1, a.w_sub);
    for (int e = threadIdx.x; e < n1 * R; e += blockDim.x) {
        const int r = e % R, k1 = e / R;
        const int k2 = k2_0 + r;
        Fr x = s.get(k1 * R + r);
        if (a.post_full) x = mul(x, ld(&a.post_full[k2 + (uint64_t)n2 * k1]));
        else if (a.post_lo) x = mul(x, mul(ld(&a.post_lo[k2]), ld(&a.post_hi[k1])));
        else if (a.scale) x = mul(x, ld(a.scale));
        store<FrCfg>(out + 32 * (k2 + (uint64_t)n2 * k1), x);
    }
}

// Passes B1 / B2 of the three-pass transform: CTA b handles column i1 =
// b mod nC (adjacent CTAs read adjacent 32-B elements) and sub-DFT x =
// b / nC: element j at in_base + in_stride j, result k at out_base +
// out_stride k times w^(tw_a (tw_b + tw_k k)).
struct PassB {
    const uint8_t* in;
    uint8_t* out;
    int LC, m, L2;           // log2 nC, log2 of this pass's sub-DFT, log2 n2 (lo/hi split)
    uint64_t in_xmul, in_stride, out_xmul, out_stride;  // strides in elements
    int tw_mode;             // 1: exponent nC x k (B1); 2: i1 (x + q k) (B2)
    uint32_t q;              // B2: q
    const Fr* w_sub;
    const Fr* tw_lo;         // w^e, e < n2
    const Fr* tw_hi;         // w^(n2 e), e < n / n2
    const Fr* pre_lo;        // coset (B1 of a forward coset transform): g^i1 (nC)
    const Fr* pre_hi;        // g^(nC i2) (n2)
    const Fr* tw_b;          // B1: w^(nC e), e < p q (one product instead of lo * hi)
};
// Pass B CTAs have at most 256 threads (m <= 9 for n <= 2^28): bounds
// (256, 3) give it 80 registers instead of 64 with 200 B of spills (2^26
// forward 24.2 -> 23.7 ms, 2^28 107.7 -> 105.4 ms; (256, 2): 118 registers,
// slower at 24.8 / 115.2 ms).
#ifndef ACEGPU_NTT_B_THREADS
#define ACEGPU_NTT_B_THREADS 256
#endif
#ifndef ACEGPU_NTT_B_MINB
#define ACEGPU_NTT_B_MINB 3
#endif
__global__ void __launch_bounds__(ACEGPU_NTT_B_THREADS, ACEGPU_NTT_B_MINB) ntt_pass_b(PassB a) {
    extern __shared__ uint4 smem_raw[];
    const uint32_t M = 1u << a.m;
    const SmemFr s{smem_raw, M};
    const uint64_t nC = 1ull << a.LC;
    const uint64_t i1 = blockIdx.x & (nC - 1), x = blockIdx.x >> a.LC;
    const uint64_t ib = i1 + nC * x * a.in_xmul, ob = i1 + nC * x * a.out_xmul;
    for (uint32_t j = threadIdx.x; j < M; j += blockDim.x) {
        const uint64_t idx = ib + a.in_stride * j;
        Fr v = load<FrCfg>(a.in + 32 * idx);
        if (a.pre_lo) v = mul(v, mul(ld(&a.pre_lo[i1]), ld(&a.pre_hi[idx >> a.LC])));
        s.put(bitrev(j, a.m), v);
    }
    __syncthreads();
    smem_dit<1>(s, a.m, a.w_sub);
    const uint64_t n2m = (1ull << a.L2) - 1;
    for (uint32_t k = threadIdx.x; k < M; k += blockDim.x) {
        Fr v = s.get(k);
        if (a.tw_mode == 1) {
            const uint64_t e = x * k;  // w^(nC u s), u s < p q
            if (e) v = mul(v, ld(&a.tw_b[e]));
        } else {
            const uint64_t ex = i1 * (x + (uint64_t)a.q * k);
            if (ex) v = mul(v, mul(ld(&a.tw_lo[ex & n2m]), ld(&a.tw_hi[ex >> a.L2])));
        }
        store<FrCfg>(a.out + 32 * (ob + a.out_stride * k), v);
    }
}

// Whole transform in one CTA (n <= 2^12): pre table g^i (n), post table
// scale*g^-k (n) or uniform scale.
__global__ void __launch_bounds__(512) ntt_single(PassArgs a) {
    extern __shared__ uint4 smem_raw[];
    const int n = 1 << a.L;
    const SmemFr s{smem_raw, uint32_t(n)};
    const uint64_t off = (uint64_t)blockIdx.x * n;  // batch of independent transforms
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        Fr x = load<FrCfg>(a.in + 32 * (off + i));
        if (a.pre_lo) x = mul(x, ld(&a.pre_lo[i]));
        s.put(a.L ? bitrev(i, a.L) : 0, x);
    }
    __syncthreads();
    if (a.L) smem_dit<1>(s, a.L, a.w_sub);
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        Fr x = s.get(k);
        if (a.post_lo) x = mul(x, ld(&a.post_lo[k]));
        else if (a.scale) x = mul(x, ld(a.scale));
        store<FrCfg>(a.out + 32 * (off + k), x);
    }
}

// table[k] = base^(k * step) for k < n (each thread: square-and-multiply).
__global__ void powers_kernel(const Fr* base, uint32_t step, uint32_t n, const Fr* scale,
                              Fr* table) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    uint64_t e = (uint64_t)k * step;
    Fr r = Fr::one(), b = *base;
    while (e) {
        if (e & 1) r = mul(r, b);
        b = sqr(b);
        e >>= 1;
    }
    if (scale) r = mul(r, *scale);
    table[k] = r;
}

// Scalars: w = 5^((r-1)/2^L) (inverse: its inverse), g = 5, n^-1.
__global__ void roots_kernel(int L, Fr* out /* [0]=w [1]=w^-1 [2]=g [3]=g^-1 [4]=n^-1 */) {
    if (threadIdx.x || blockIdx.x) return;
    // e = (r - 1) >> L
    uint32_t e[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) e[i] = mod_limb<FrCfg>(i);
    e[0] -= 1;
    for (int s = 0; s < L; ++s) {
        for (int i = 0; i < 8; ++i) e[i] = (e[i] >> 1) | (i < 7 ? (e[i + 1] << 31) : 0u);
    }
    Fr five = Fr::zero();
    five.v[0] = 5;
    five = to_mont(five);
    Fr w = pow(five, e);
    out[0] = w;
    out[1] = inv(w);
    out[2] = five;
    out[3] = inv(five);
    Fr n = Fr::zero();
    if (L < 32) n.v[0] = 1u << L;
    out[4] = inv(to_mont(n));
}

__global__ void convert_kernel(uint8_t* data, uint64_t n, int to) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    Fr x = load<FrCfg>(data + 32 * i);
    store<FrCfg>(data + 32 * i, to ? to_mont(x) : from_mont(x));
}

// ---- mixed radix 3 * 2^k --------------------------------------------------
// w3 = w_N^(N/3) and its inverse: 3 * 2^k roots (r - 1 = 2^28 3^2 ...);
// c: [0] w_N [1] w_N^-1 [2] w3 [3] w3^-1 [4] 3^-1 [5] g [6] g^-1
__global__ void roots3_kernel(int k, Fr* out) {
    if (threadIdx.x || blockIdx.x) return;
    uint32_t e[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) e[i] = mod_limb<FrCfg>(i);
    e[0] -= 1;
    for (int s = 0; s < k; ++s)
        for (int i = 0; i < 8; ++i) e[i] = (e[i] >> 1) | (i < 7 ? (e[i + 1] << 31) : 0u);
    uint64_t rem = 0;  // e /= 3
    for (int i = 7; i >= 0; --i) {
        const uint64_t cur = (rem << 32) | e[i];
        e[i] = (uint32_t)(cur / 3);
        rem = cur % 3;
    }
    Fr five = Fr::zero();
    five.v[0] = 5;
    five = to_mont(five);
    const Fr w = pow(five, e);
    out[0] = w;
    out[1] = inv(w);
    uint32_t m[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // N / 3 = 2^k
    m[k >> 5] = 1u << (k & 31);
    out[2] = pow(w, m);
    out[3] = inv(out[2]);
    Fr three = Fr::zero();
    three.v[0] = 3;
    out[4] = inv(to_mont(three));
    out[5] = five;
    out[6] = inv(five);
}

__device__ __forceinline__ Fr split_pow(const Fr* lo, const Fr* hi, uint64_t e, int S) {
    return mul(ld(&lo[e & ((1ull << S) - 1)]), ld(&hi[e >> S]));
}

// Y_i1[i2] = x[i1 + 3 i2] (times g^(i1 + 3 i2) for a forward coset
// transform); thread i2 reads its three contiguous elements (one 96-B run:
// reading the groups in separate threads pulled every line from DRAM three
// times) and writes one element of each sub-vector.
__global__ void deint3_kernel(const uint8_t* in, uint8_t* y, uint64_t M, const Fr* g_lo,
                              const Fr* g_hi, int S) {
    const uint64_t i2 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i2 >= M) return;
#pragma unroll
    for (int i1 = 0; i1 < 3; ++i1) {
        const uint64_t src = i1 + 3 * i2;
        Fr v = load<FrCfg>(in + 32 * src);
        if (g_lo) v = mul(v, split_pow(g_lo, g_hi, src, S));
        store<FrCfg>(y + 32 * (M * i1 + i2), v);
    }
}

// X[k2 + M k1] = sum_i1 w_N^(i1 k2) w3^(i1 k1) Y_i1[k2], with 1 + w3 + w3^2 = 0:
// X0 = y0 + t1 + t2, X1 = y0 - t2 + w3 (t1 - t2), X2 = y0 - t1 - w3 (t1 - t2).
// Inverse: w^-1 roots, times 3^-1 (the sub-NTTs applied 2^-k), coset g^-k.
__global__ void combine3_kernel(const uint8_t* y, uint8_t* out, uint64_t M, const Fr* c,
                                const Fr* w_lo, const Fr* w_hi, int inverse, const Fr* gi_lo,
                                const Fr* gi_hi, int S) {
    const uint64_t k2 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k2 >= M) return;
    const Fr y0 = load<FrCfg>(y + 32 * k2), y1 = load<FrCfg>(y + 32 * (M + k2)),
             y2 = load<FrCfg>(y + 32 * (2 * M + k2));
    Fr t1 = y1, t2 = y2;
    if (k2) {
        const Fr tw = split_pow(w_lo, w_hi, k2, S);
        t1 = mul(y1, tw);
        t2 = mul(y2, sqr(tw));
    }
    const Fr d = mul(ld(&c[inverse ? 3 : 2]), sub(t1, t2));
    Fr x[3] = {add(add(y0, t1), t2), add(sub(y0, t2), d), sub(sub(y0, t1), d)};
#pragma unroll
    for (int k1 = 0; k1 < 3; ++k1) {
        const uint64_t k = k2 + M * k1;
        Fr v = x[k1];
        if (inverse) {
            v = mul(v, ld(&c[4]));
            if (gi_lo) v = mul(v, split_pow(gi_lo, gi_hi, k, S));
        }
        store<FrCfg>(out + 32 * k, v);
    }
}

}  // namespace

// ------------------------------------------------------------------ host side
int ntt3_tables(Ntt3Tables& t, int k, cudaStream_t s) {
    if (t.k == k && t.consts) return 0;
    t.release();
    if (k < 0 || k > kNtt3MaxLog) return -1;
    t.k = k;
    const uint64_t M = 1ull << k, N = 3 * M;
    t.S = (k + 2) / 2;  // lo tables 2^S entries
    const uint64_t lo = 1ull << t.S, hi_w = (M + lo - 1) / lo, hi_g = (N + lo - 1) / lo;
    auto alloc = [&](Fr** p, size_t cnt) { return cudaMalloc(p, sizeof(Fr) * (cnt ? cnt : 1)); };
    if (alloc(&t.consts, 8)) return -1;
    roots3_kernel<<<1, 1, 0, s>>>(k, t.consts);
    auto pw = [&](Fr** dst, const Fr* base, uint32_t step, uint64_t cnt) {
        if (alloc(dst, cnt)) return -1;
        powers_kernel<<<(unsigned)((cnt + 255) / 256), 256, 0, s>>>(base, step, (uint32_t)cnt,
                                                                    nullptr, *dst);
        return 0;
    };
    const uint32_t step = (uint32_t)lo;
    if (pw(&t.wn_lo, t.consts + 0, 1, lo) || pw(&t.wn_hi, t.consts + 0, step, hi_w) ||
        pw(&t.wni_lo, t.consts + 1, 1, lo) || pw(&t.wni_hi, t.consts + 1, step, hi_w) ||
        pw(&t.g_lo, t.consts + 5, 1, lo) || pw(&t.g_hi, t.consts + 5, step, hi_g) ||
        pw(&t.gi_lo, t.consts + 6, 1, lo) || pw(&t.gi_hi, t.consts + 6, step, hi_g))
        return -1;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

void Ntt3Tables::release() {
    Fr** all[] = {&consts, &wn_lo, &wn_hi, &wni_lo, &wni_hi, &g_lo, &g_hi, &gi_lo, &gi_hi};
    for (Fr** p : all) {
        if (*p) cudaFree(*p);
        *p = nullptr;
    }
    k = -1;
}

int ntt3_run(const Ntt3Tables& t, const NttTables& tM, const uint8_t* in, uint8_t* out,
             uint8_t* ybuf, uint8_t* scratch, int inverse, int coset, cudaStream_t s) {
    if (t.k < 0 || tM.L != t.k) return -1;
    const uint64_t M = 1ull << t.k;
    const unsigned g1 = (unsigned)((M + 255) / 256);
    deint3_kernel<<<g1, 256, 0, s>>>(in, ybuf, M, (coset && !inverse) ? t.g_lo : nullptr, t.g_hi,
                                     t.S);
    if (t.k <= kNttTwoPassMax) {  // the three sub-NTTs as one batch (scratch: 3 x 2^k)
        if (ntt_run(tM, ybuf, ybuf, scratch, inverse, 0, 3, s)) return -1;
    } else {
        for (int i1 = 0; i1 < 3; ++i1)
            if (ntt_run(tM, ybuf + 32 * M * i1, ybuf + 32 * M * i1, scratch, inverse, 0, 1, s))
                return -1;
    }
    combine3_kernel<<<g1, 256, 0, s>>>(ybuf, out, M, t.consts, inverse ? t.wni_lo : t.wn_lo,
                                       inverse ? t.wni_hi : t.wn_hi, inverse,
                                       (coset && inverse) ? t.gi_lo : nullptr, t.gi_hi, t.S);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// (power-of-two tables)
int ntt_tables(NttTables& t, int L, cudaStream_t s) {
    if (t.L == L && t.w_a) return 0;
    t.release();
    t.L = L;
    const int L2 = (L + 1) / 2, L1 = L - L2;
    t.L1 = L1;
    t.L2 = L2;
    const uint32_t n = 1u << L, n1 = 1u << L1, n2 = 1u << L2;
    auto alloc = [&](Fr** p, size_t cnt) { return cudaMalloc(p, sizeof(Fr) * (cnt ? cnt : 1)); };
    if (alloc(&t.consts, 8)) return -1;
    roots_kernel<<<1, 1, 0, s>>>(L, t.consts);
    Fr* w = t.consts + 0;
    Fr* wi = t.consts + 1;
    Fr* g = t.consts + 2;
    Fr* gi = t.consts + 3;
    Fr* ninv = t.consts + 4;
    auto pw = [&](Fr** dst, const Fr* base, uint32_t step, uint32_t cnt, const Fr* scale) {
        if (alloc(dst, cnt)) return -1;
        powers_kernel<<<(cnt + 255) / 256, 256, 0, s>>>(base, step, cnt, scale, *dst);
        return 0;
    };
    if (L <= kNttSingleMax) {
        // single-CTA transform: sub-DFT roots of size n, coset tables of size n
        if (pw(&t.w_a, w, 1, n / 2 ? n / 2 : 1, nullptr) || pw(&t.wi_a, wi, 1, n / 2 ? n / 2 : 1, nullptr) ||
            pw(&t.g_lo, g, 1, n, nullptr) || pw(&t.gi_post_lo, gi, 1, n, ninv))
            return -1;
        return cudaGetLastError() == cudaSuccess ? 0 : -1;
    }
    if (L > kNttTwoPassMax) {
        // three passes: nC = 2^LC (pass C), p = 2^LP (B2), q = 2^LQ (B1); the
        // lo/hi split of twiddles and coset factors is at n2 = p q
        t.LQ = L / 3;
        t.LP = L / 3;
        t.LC = L - t.LP - t.LQ;
        t.L1 = t.LC;
        t.L2 = L - t.LC;
        const uint32_t nc = 1u << t.LC, m2 = 1u << t.L2, p = 1u << t.LP, q = 1u << t.LQ;
        if (pw(&t.w_q, w, n / q, q / 2, nullptr) || pw(&t.wi_q, wi, n / q, q / 2, nullptr) ||
            pw(&t.w_p, w, n / p, p / 2, nullptr) || pw(&t.wi_p, wi, n / p, p / 2, nullptr) ||
            pw(&t.w_c, w, m2, nc / 2, nullptr) || pw(&t.wi_c, wi, m2, nc / 2, nullptr) ||
            pw(&t.tw_lo, w, 1, m2, nullptr) || pw(&t.tw_hi, w, m2, nc, nullptr) ||
            pw(&t.twi_lo, wi, 1, m2, nullptr) || pw(&t.twi_hi, wi, m2, nc, nullptr) ||
            pw(&t.g_lo, g, 1, nc, nullptr) || pw(&t.g_hi, g, nc, m2, nullptr) ||
            pw(&t.gi_post_lo, gi, 1, m2, ninv) || pw(&t.gi_post_hi, gi, m2, nc, nullptr) ||
            pw(&t.tw_full, w, nc, m2, nullptr) || pw(&t.twi_full, wi, nc, m2, nullptr))
            return -1;
        t.w_a = t.w_q;  // marks the tables built
        return cudaGetLastError() == cudaSuccess ? 0 : -1;
    }
    // pass A: sub-DFT of size n2 -> root w^n1 ; pass C: size n1 -> root w^n2
    if (pw(&t.w_a, w, n1, n2 / 2, nullptr) || pw(&t.wi_a, wi, n1, n2 / 2, nullptr) ||
        pw(&t.w_c, w, n2, n1 / 2, nullptr) || pw(&t.wi_c, wi, n2, n1 / 2, nullptr) ||
        pw(&t.tw_lo, w, 1, n2, nullptr) || pw(&t.tw_hi, w, n2, n1, nullptr) ||
        pw(&t.twi_lo, wi, 1, n2, nullptr) || pw(&t.twi_hi, wi, n2, n1, nullptr) ||
        pw(&t.g_lo, g, 1, n1, nullptr) || pw(&t.g_hi, g, n1, n2, nullptr) ||
        pw(&t.gi_post_lo, gi, 1, n2, ninv) || pw(&t.gi_post_hi, gi, n2, n1, nullptr) ||
        pw(&t.tw_full, w, 1, n, nullptr) || pw(&t.twi_full, wi, 1, n, nullptr) ||
        pw(&t.g_full, g, 1, n, nullptr) || pw(&t.gi_post_full, gi, 1, n, ninv))
        return -1;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

void NttTables::release() {
    if (w_a == w_q) w_a = nullptr;  // three-pass tables alias w_a to w_q
    Fr** all[] = {&consts, &w_a, &wi_a, &w_c, &wi_c, &tw_lo, &tw_hi, &twi_lo, &twi_hi,
                  &g_lo, &g_hi, &gi_post_lo, &gi_post_hi, &tw_full, &twi_full, &g_full,
                  &gi_post_full, &w_q, &wi_q, &w_p, &wi_p};
    for (Fr** p : all) {
        if (*p) cudaFree(*p);
        *p = nullptr;
    }
    LC = LP = LQ = 0;
    L = -1;
}

int ntt_run(const NttTables& t, const uint8_t* in, uint8_t* out, uint8_t* scratch, int inverse,
            int coset, int batch, cudaStream_t s) {
    const int L = t.L;
    PassArgs a{};
    a.L = L;
    a.L1 = t.L1;
    a.L2 = t.L2;
    a.scale = nullptr;
    if (L <= kNttSingleMax) {
        a.in = in;
        a.out = out;
        a.w_sub = inverse ? t.wi_a : t.w_a;
        a.pre_lo = (coset && !inverse) ? t.g_lo : nullptr;
        a.post_lo = (coset && inverse) ? t.gi_post_lo : nullptr;
        if (inverse && !coset) a.scale = t.consts + 4;
        const size_t smem = sizeof(Fr) << L;
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(ntt_single, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        ntt_single<<<batch, 512, smem, s>>>(a);
        return cudaGetLastError() == cudaSuccess ? 0 : -1;
    }
    const int n1 = 1 << t.L1, n2 = 1 << t.L2;
    if (L > kNttTwoPassMax) {
        // B1: in -> out (in place per CTA), B2: out -> scratch, C: scratch -> out
        const uint64_t nc = 1ull << t.LC, p = 1ull << t.LP, q = 1ull << t.LQ;
        PassB b{};
        b.LC = t.LC;
        b.L2 = t.L2;
        b.tw_lo = inverse ? t.twi_lo : t.tw_lo;
        b.tw_hi = inverse ? t.twi_hi : t.tw_hi;
        b.in = in;
        b.out = out;
        b.m = t.LQ;
        b.in_xmul = 1, b.in_stride = nc * p, b.out_xmul = 1, b.out_stride = nc * p;
        b.tw_mode = 1;
        b.w_sub = inverse ? t.wi_q : t.w_q;
        b.pre_lo = (coset && !inverse) ? t.g_lo : nullptr;
        b.pre_hi = (coset && !inverse) ? t.g_hi : nullptr;
        b.tw_b = inverse ? t.twi_full : t.tw_full;  // three-pass: w^(nC e), e < p q
        size_t sm = sizeof(Fr) << t.LQ;
        cudaFuncSetAttribute(ntt_pass_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        // one butterfly per thread and stage: M / 2 threads
        auto thr = [](int m) { return std::max(32, std::min(512, 1 << (m - 1))); };
        ntt_pass_b<<<(unsigned)(nc * p), thr(t.LQ), sm, s>>>(b);
        PassB b2 = b;
        b2.in = out;
        b2.out = scratch;
        b2.m = t.LP;
        b2.in_xmul = p, b2.in_stride = nc, b2.out_xmul = 1, b2.out_stride = nc * q;
        b2.tw_mode = 2;
        b2.q = (uint32_t)q;
        b2.w_sub = inverse ? t.wi_p : t.w_p;
        b2.pre_lo = b2.pre_hi = nullptr;
        sm = sizeof(Fr) << t.LP;
        ntt_pass_b<<<(unsigned)(nc * q), thr(t.LP), sm, s>>>(b2);
        PassArgs c{};
        c.L = L;
        c.L1 = t.L1;
        c.L2 = t.L2;
        c.R = kNttR;
        c.in = scratch;
        c.out = out;
        c.w_sub = inverse ? t.wi_c : t.w_c;
        c.post_lo = (coset && inverse) ? t.gi_post_lo : nullptr;
        c.post_hi = (coset && inverse) ? t.gi_post_hi : nullptr;
        if (inverse && !coset) c.scale = t.consts + 4;
        c.bstride = 0;
        sm = sizeof(Fr) * (size_t)n1 * kNttR;
        cudaFuncSetAttribute(ntt_pass_c, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        ntt_pass_c<<<(unsigned)(n2 / kNttR), ACEGPU_NTT_AC_THREADS, sm, s>>>(c);
        return cudaGetLastError() == cudaSuccess ? 0 : -1;
    }
    // pass A: in -> scratch
    a.in = in;
    a.out = scratch;
    a.R = kNttR;
    a.w_sub = inverse ? t.wi_a : t.w_a;
    a.tw_lo = inverse ? t.twi_lo : t.tw_lo;
    a.tw_hi = inverse ? t.twi_hi : t.tw_hi;
    static const bool full = !getenv("ACEGPU_NTT_SPLIT_TW");
    a.tw_full = full ? (inverse ? t.twi_full : t.tw_full) : nullptr;
    a.pre_lo = (coset && !inverse) ? t.g_lo : nullptr;
    a.pre_hi = (coset && !inverse) ? t.g_hi : nullptr;
    a.pre_full = (full && coset && !inverse) ? t.g_full : nullptr;
    // batch > 1: contiguous transforms (scratch holds batch x n)
    a.bstride = 1ull << L;
    size_t smem = sizeof(Fr) * (size_t)n2 * kNttR;
    cudaFuncSetAttribute(ntt_pass_a, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    ntt_pass_a<<<dim3(n1 / kNttR, batch), ACEGPU_NTT_AC_THREADS, smem, s>>>(a);
    // pass C: scratch -> out
    PassArgs c = a;
    c.in = scratch;
    c.out = out;
    c.w_sub = inverse ? t.wi_c : t.w_c;
    c.pre_lo = c.pre_hi = nullptr;
    c.post_lo = (coset && inverse) ? t.gi_post_lo : nullptr;
    c.post_hi = (coset && inverse) ? t.gi_post_hi : nullptr;
    c.pre_full = nullptr;
    c.post_full = (full && coset && inverse) ? t.gi_post_full : nullptr;
 if (inverse && !coset) c.scale = t.consts + 4;
    smem = sizeof(Fr) * (size_t)n1 * kNttR;
    cudaFuncSetAttribute(ntt_pass_c, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    ntt_pass_c<<<dim3(n2 / kNttR, batch), ACEGPU_NTT_AC_THREADS, smem, s>>>(c);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

void launch_fr_convert(uint8_t* data, uint64_t n, int to_mont, cudaStream_t s) {
    if (n) convert_kernel<<<(n + 255) / 256, 256, 0, s>>>(data, n, to_mont);
}

}  // namespace bn
}  // namespace ace_gpu
