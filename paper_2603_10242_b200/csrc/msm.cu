// Pippenger multi-scalar multiplication over BN254 G1 and G2 for sm_100a
// (north-star row a21: K8/K9 of SURVEY §2b; the reference has none).
//
// Fixed-base form: the proving key's bases are fixed, so `msm_prepare`
// stores table[w][i] = 2^(c w) P_i once (affine, c = kMsmC = 17 -> 15
// windows). A run then needs no doublings between windows: every
// (window, point) pair with a non-zero signed c-bit digit d lands in one of
// 2^(c-1) buckets |d| of a single bucket set, and the result is
// sum_k k * B_k.
//
//   1. count     : signed digits of each scalar -> bucket histogram (atomics)
//   2. scan      : exclusive prefix sum -> bucket offsets
//   3. scatter   : (window*n + i | sign) into bucket order
//   4. accumulate: each thread mixed-adds kMsmSeg (fewer for small MSMs)
//                  consecutive sorted entries
//                  (XYZZ, 8M + 2S, lazy-reduced Y); a bucket wholly inside
//                  the segment is written directly, the first/last runs that
//                  cross a segment edge go to two partial slots
//   5. fixup     : one thread per bucket crossing segments sums its partials
//                  (and writes infinity for empty buckets)
//   6. reduce    : sum_k k*B_k by per-segment running sums + small scalar
//                  multiples, per-CTA trees, then one CTA and affine.
// Bound: IMAD pipe (Fq mul = CIOS carry chains). Work ~ (W*n) mixed adds.
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>
#include <algorithm>
#include <cstdlib>

#include "curve.cuh"
#include "msm.cuh"

namespace ace_gpu {
namespace bn {

namespace {

__device__ __forceinline__ Fq finv(const Fq& a) { return inv_fast(a); }
__device__ __forceinline__ Fq2 finv(const Fq2& a) {
    Fq n = add(fmul(a.c0, a.c0), fmul(a.c1, a.c1));
    Fq ni = inv_fast(n);
    return {fmul(a.c0, ni), neg(fmul(a.c1, ni))};
}
__device__ __forceinline__ Fq fneg(const Fq& a) { return neg(a); }
__device__ __forceinline__ Fq2 fneg(const Fq2& a) { return {neg(a.c0), neg(a.c1)}; }

#ifndef ACEGPU_G2_ACC_MINB
#define ACEGPU_G2_ACC_MINB 1  // measured (paper-size chunk): 1 -> 60.1 ms, 3 -> 61.4, 4 -> 61.1
#endif
#ifndef ACEGPU_G1_ACC_MINB
#define ACEGPU_G1_ACC_MINB 4  // 128 registers, 4 CTAs/SM: G1 2^20 4.65 -> 4.36 ms, chunk 46.9 -> 44.9 ms
#endif
template <class F>
struct Lay {
    static constexpr int EB = felem_bytes<F>();
    static constexpr int AFF = 2 * EB;
    static constexpr int XZ = 4 * EB;
    // accumulate_kernel min CTAs/SM (register cap): G2's Fq2 temporaries
    // fill 255 registers (and spill 172 B) -> 2 CTAs (8 warps) per SM;
    // capping them lower spills more and measured slower
    static constexpr int ACC_MIN_CTAS = EB == 32 ? ACEGPU_G1_ACC_MINB : ACEGPU_G2_ACC_MINB;
};

// Window configuration: c-bit signed digits, W windows, NB buckets per
// window, reduction segments. Fixed base uses c = kMsmC (17); variable base
// (block-size keys) uses kMsmVbC: with 2^26-point sub-ranges the 2^19
// buckets of c = 20 cost ~2 % and save 2 of 15 windows.
// NARROW: the last NARROW windows are one bit narrower (widths C ... C,
// C-1 ... C-1 summing to >= 255), so the top window is nearly full — with
// uniform 20-bit windows the top one holds 14 bits, 2^13 buckets of 2^13
// entries each at 2^26 points: all "heavy".
template <int C, int NARROW = 0, int RED_THREADS = 0>
struct Win {
    static constexpr int c = C;
    static constexpr int W = (255 + NARROW + C - 1) / C;
    static constexpr int NB = 1 << (C - 1);
    __host__ __device__ static constexpr int width(int w) { return w < W - NARROW ? C : C - 1; }
    __host__ __device__ static constexpr int off(int w) {
        return w <= W - NARROW ? C * w : C * (W - NARROW) + (C - 1) * (w - (W - NARROW));
    }
    static_assert(C * (W - NARROW) + (C - 1) * NARROW >= 255, "windows cover 255 bits");
#ifndef ACEGPU_RED_THREADS
#define ACEGPU_RED_THREADS 8192
#endif
    // buckets per reduction thread: NB / ACEGPU_RED_THREADS, at least 2
    static constexpr int RT = RED_THREADS ? RED_THREADS : ACEGPU_RED_THREADS;
    static constexpr int RedSeg = NB / RT > 2 ? NB / RT : 2;
    static constexpr int RedThreads = NB / RedSeg;
    static_assert(RedThreads / 128 <= 1024, "reduce_final partials");
};
using WinFixed = Win<kMsmC>;
#ifndef ACEGPU_MSM_VB_NARROW
#define ACEGPU_MSM_VB_NARROW 5  // c = 20: 8 x 20 + 5 x 19 = 255 bits (13 windows)
#endif
#ifndef ACEGPU_VB_RED_THREADS
#define ACEGPU_VB_RED_THREADS 8192
#endif
using WinVb = Win<kMsmVbC, ACEGPU_MSM_VB_NARROW, ACEGPU_VB_RED_THREADS>;
using WinMid = Win<19, 11>;  // 3 x 19 + 11 x 18 = 255 bits, 14 windows x 2^18 buckets

template <class F>
__device__ __forceinline__ bool load_affine(const uint8_t* p, F& x, F& y) {
    fload(x, p);
    fload(y, p + Lay<F>::EB);
    return !(fzero(x) && fzero(y));  // all-zero record = infinity
}

template <class F>
__device__ __forceinline__ void store_affine(uint8_t* p, const F& x, const F& y) {
    fstore(p, x);
    fstore(p + Lay<F>::EB, y);
}

template <class F>
__device__ __forceinline__ void store_xyzz(uint8_t* p, const XYZZ<F>& a) {
    constexpr int E = Lay<F>::EB;
    fstore(p, a.X);
    fstore(p + E, a.Y);
    fstore(p + 2 * E, a.ZZ);
    fstore(p + 3 * E, a.ZZZ);
}

template <class F>
__device__ __forceinline__ XYZZ<F> load_xyzz(const uint8_t* p) {
    constexpr int E = Lay<F>::EB;
    XYZZ<F> a;
    fload(a.X, p);
    fload(a.Y, p + E);
    fload(a.ZZ, p + 2 * E);
    fload(a.ZZZ, p + 3 * E);
    return a;
}

template <class F>
__device__ __forceinline__ void to_affine(const XYZZ<F>& a, F& x, F& y) {
    if (a.is_inf()) {
        fset_zero(x);
        fset_zero(y);
        return;
    }
    F t = finv(fmul(a.ZZ, a.ZZZ));
    x = fmul(a.X, fmul(t, a.ZZZ));  // X / ZZ
    y = fmul(a.Y, fmul(t, a.ZZ));   // Y / ZZZ
}

// ---- prepare: table[w*n + i] = 2^(c w) P_i ----------------------------------
template <class F>
__global__ void prepare_kernel(const uint8_t* bases, uint64_t n, uint8_t* table) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    constexpr int A = Lay<F>::AFF;
    F x, y;
    const bool fin = load_affine<F>(bases + A * i, x, y);
    store_affine(table + A * i, x, y);
    for (int w = 1; w < kMsmWindows; ++w) {
        if (fin) {
            XYZZ<F> q;
            q.X = x;
            q.Y = y;
            fset_one(q.ZZ);
            fset_one(q.ZZZ);
            for (int d = 0; d < kMsmC; ++d) q = xyzz_dbl(q);
            to_affine(q, x, y);
        }
        store_affine(table + A * ((uint64_t)w * n + i), x, y);
    }
}

// Signed base-2^c digits of a canonical scalar < r < 2^254: window w reads
// bits [c w, c w + c) (a 64-bit window over two limbs); raw values above
// 2^(c-1) become raw - 2^c with a carry into the next window. The top window
// holds < 2^(254 - c (W-1)) <= 2^(c-1), so no carry leaves it.
template <class Wn = WinFixed>
__device__ __forceinline__ void digits(const uint8_t* s, int32_t d[Wn::W]) {
    const uint4* q = reinterpret_cast<const uint4*>(s);
    uint4 a = q[0], b = q[1];
    const uint32_t limb[9] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, 0u};
    uint32_t carry = 0;
#pragma unroll
    for (int w = 0; w < Wn::W; ++w) {
        const int kC = Wn::width(w);
        const int bit = Wn::off(w), lo = bit >> 5, sh = bit & 31;
        const uint64_t v = ((uint64_t)limb[lo + 1] << 32) | limb[lo];
        const uint32_t raw = (uint32_t)(v >> sh) & ((1u << kC) - 1u);
        const uint32_t t = raw + carry;
        if (t > (1u << (kC - 1))) {
            d[w] = (int32_t)t - (1 << kC);
            carry = 1;
        } else {
            d[w] = (int32_t)t;
            carry = 0;
        }
    }
}

// Histogram / scatter with warp-aggregated atomics: lanes whose digit lands
// in the same bucket elect one lane for the atomic (__match_any_sync), so a
// hot bucket (a 0/1 witness sends every point to bucket 1) costs one atomic
// per warp instead of 32 serialised ones. Lanes past n take part with a
// bucket no real digit uses.
#ifndef ACEGPU_SORT_AGG
#define ACEGPU_SORT_AGG 1
#endif
#if !ACEGPU_SORT_AGG
template <bool VB, class Wn = WinFixed>
__global__ void count_kernel(const uint8_t* scalars, uint64_t n, uint32_t* hist) {
    static_assert(!VB, "variable-base MSM needs ACEGPU_SORT_AGG");
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t d[kMsmWindows];
    digits(scalars + 32 * i, d);
#pragma unroll
    for (int w = 0; w < kMsmWindows; ++w)
        if (d[w]) atomicAdd(&hist[abs(d[w]) - 1], 1u);
}
template <bool VB, class Wn = WinFixed>
__global__ void scatter_kernel(const uint8_t* scalars, uint64_t n, uint32_t* cursor,
                               uint32_t* sorted) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t d[kMsmWindows];
    digits(scalars + 32 * i, d);
#pragma unroll
    for (int w = 0; w < kMsmWindows; ++w) {
        if (!d[w]) continue;
        const uint32_t pos = atomicAdd(&cursor[abs(d[w]) - 1], 1u);
        sorted[pos] = (uint32_t)(w * n + i) | (d[w] < 0 ? 0x80000000u : 0u);
    }
}
#else
// VB (variable base, no window tables): bucket key w * kMsmBuckets + |d| - 1
// (one bucket set per window) and entry = the point index; fixed base: key
// |d| - 1 and entry = the table row w n + i.
template <bool VB, class Wn>
__device__ __forceinline__ uint32_t bucket_key(int w, int32_t d) {
    return VB ? (uint32_t)(w * Wn::NB + abs(d) - 1) : (uint32_t)(abs(d) - 1);
}
template <bool VB, class Wn = WinFixed>
__global__ void count_kernel(const uint8_t* scalars, uint64_t n, uint32_t* hist) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    int32_t d[Wn::W];
    if (i < n) digits<Wn>(scalars + 32 * i, d);
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int w = 0; w < Wn::W; ++w) {
        const uint32_t key = (i < n && d[w]) ? bucket_key<VB, Wn>(w, d[w]) : 0xFFFFFFFFu;
        const uint32_t peers = __match_any_sync(0xffffffffu, key);
        if (key != 0xFFFFFFFFu && lane == __ffs(peers) - 1) atomicAdd(&hist[key], __popc(peers));
    }
}

template <bool VB, class Wn = WinFixed>
__global__ void scatter_kernel(const uint8_t* scalars, uint64_t n, uint32_t* cursor,
                               uint32_t* sorted) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    int32_t d[Wn::W];
    if (i < n) digits<Wn>(scalars + 32 * i, d);
    const int lane = threadIdx.x & 31;
    const uint32_t below = (1u << lane) - 1u;
#pragma unroll
    for (int w = 0; w < Wn::W; ++w) {
        const uint32_t key = (i < n && d[w]) ? bucket_key<VB, Wn>(w, d[w]) : 0xFFFFFFFFu;
        const uint32_t peers = __match_any_sync(0xffffffffu, key);
        const int leader = __ffs(peers) - 1;
        uint32_t base = 0;
        if (key != 0xFFFFFFFFu && lane == leader) base = atomicAdd(&cursor[key], __popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (key != 0xFFFFFFFFu)
            sorted[base + __popc(peers & below)] =
                (uint32_t)(VB ? i : w * n + i) | (d[w] < 0 ? 0x80000000u : 0u);
    }
}
#endif

// Large variable-base sorts in window passes: the digits once into a
// window-major key array (coalesced), the bucket histogram alongside; then,
// per window and bucket range, a scatter whose destinations span a region
// the L2 can hold — one pass over all windows at once scatters 4-B entries
// over the whole sorted array, and every partial-sector write becomes a DRAM
// read-modify-write (ncu at 2^26 points: 27.5 GB read + 30.4 GB written for
// 3.5 GB of entries).
template <class Wn>
__global__ void digits_keys_kernel(const uint8_t* scalars, uint64_t n, uint32_t* keys,
                                   uint32_t* hist) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    int32_t d[Wn::W];
    if (i < n) digits<Wn>(scalars + 32 * i, d);
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int w = 0; w < Wn::W; ++w) {
        const uint32_t key = (i < n && d[w]) ? bucket_key<true, Wn>(w, d[w]) : 0xFFFFFFFFu;
        if (i < n)
            keys[(uint64_t)w * n + i] =
                d[w] ? (uint32_t)(abs(d[w]) - 1) | (d[w] < 0 ? 0x80000000u : 0u) : 0xFFFFFFFFu;
        const uint32_t peers = __match_any_sync(0xffffffffu, key);
        if (key != 0xFFFFFFFFu && lane == __ffs(peers) - 1) atomicAdd(&hist[key], __popc(peers));
    }
}
__global__ void scatter_range_kernel(const uint32_t* keys_w, uint64_t n, uint32_t lo, uint32_t hi,
                                     uint32_t* cursor_w, uint32_t* sorted) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t k = keys_w[i];
    const uint32_t b = k & 0x7FFFFFFFu;
    if (k == 0xFFFFFFFFu || b < lo || b >= hi) return;
    sorted[atomicAdd(&cursor_w[b], 1u)] = (uint32_t)i | (k & 0x80000000u);
}

// The non-empty bucket b with offs[b] <= pos < offs[b + 1] (NB buckets).
template <int NB = kMsmBuckets>
__device__ __forceinline__ int bucket_of(const uint32_t* offs, uint32_t pos) {
    int lo = 0, hi = NB;
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (offs[mid] <= pos) lo = mid;
        else hi = mid;
    }
    return lo;
}

template <class F>
__device__ __forceinline__ void store_inf(uint8_t* p) {
    store_xyzz(p, XYZZ<F>::inf());
}

// One thread per segment of segsz consecutive sorted entries. Runs of one
// bucket: a run that is the whole bucket is stored to buckets[b]; a run cut
// by the segment edge is stored to partials[2 seg] (first run of the
// segment) or partials[2 seg + 1] (a later run).
template <class F, int NB>
__global__ void __launch_bounds__(128, Lay<F>::ACC_MIN_CTAS) accumulate_kernel(const uint8_t* table,
                                                         const uint32_t* sorted,
                                                         const uint32_t* offs,
                                                         uint8_t* buckets,
                                                         uint8_t* partials, uint32_t segsz) {
    const uint32_t seg = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t total = offs[NB];
    const uint32_t p0 = seg * segsz;
    if (p0 >= total) return;
    constexpr int A = Lay<F>::AFF, X = Lay<F>::XZ;
    const uint32_t p1 = min(total, p0 + segsz);
    int b = bucket_of<NB>(offs, p0);
    uint32_t bs = offs[b], be = offs[b + 1];
    int slot = 0;
    XYZZ<F> acc = XYZZ<F>::inf();
    uint32_t v = sorted[p0];
    for (uint32_t pos = p0; pos < p1; ++pos) {
        const uint32_t nv = pos + 1 < p1 ? sorted[pos + 1] : 0u;  // prefetch the next index
        F x, y;
        if (load_affine<F>(table + (uint64_t)A * (v & 0x7FFFFFFFu), x, y)) {  // skip infinity
            if (v >> 31) y = fneg(y);
            acc = xyzz_madd<F>(acc, x, y);  // out-of-line Fq products (inlining measured slower)
        }
        v = nv;
        if (pos + 1 == be || pos + 1 == p1) {  // the run of bucket b ends here
            if (bs >= p0 && be <= p1) store_xyzz(buckets + (uint64_t)X * b, acc);
            else store_xyzz(partials + (uint64_t)X * (2ull * seg + slot), acc);
            slot = 1;
            acc = XYZZ<F>::inf();
            if (pos + 1 < p1) {
                do {  // next non-empty bucket
                    ++b;
                    bs = be;
                    be = offs[b + 1];
                } while (be == bs);
            }
        }
    }
}

template <class F>
__device__ __forceinline__ XYZZ<F> shfl_xyzz(const XYZZ<F>& a, int src_lane_delta) {
    XYZZ<F> r;
    const uint32_t* in = reinterpret_cast<const uint32_t*>(&a);
    uint32_t* out = reinterpret_cast<uint32_t*>(&r);
#pragma unroll
    for (int k = 0; k < (int)(sizeof(XYZZ<F>) / 4); ++k)
        out[k] = __shfl_down_sync(0xffffffffu, in[k], src_lane_delta);
    return r;
}

// Sum of a 128-thread CTA's values (result valid in thread 0).
template <class F>
__device__ __forceinline__ XYZZ<F> cta_sum128(XYZZ<F> v) {
    constexpr int X = Lay<F>::XZ;
    if constexpr (sizeof(F) > sizeof(Fq)) {
        // G2: a shared-memory tree (shuffling 64-word XYZZ values spilled)
        __shared__ __align__(16) uint8_t buf[128 * sizeof(XYZZ<F>)];
        const int t = threadIdx.x;
        store_xyzz(buf + X * t, v);
        __syncthreads();
#pragma unroll 1
        for (int st = 64; st >= 1; st >>= 1) {
            if (t < st) {
                v = xyzz_add(v, load_xyzz<F>(buf + X * (t + st)));
                store_xyzz(buf + X * t, v);
            }
            __syncthreads();
        }
        return v;
    }
    __shared__ __align__(16) uint8_t sm[4 * sizeof(XYZZ<F>)];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        XYZZ<F> o = shfl_xyzz(v, d);
        if (lane < d) v = xyzz_add(v, o);
    }
    if (lane == 0) store_xyzz(sm + X * warp, v);
    __syncthreads();
    if (threadIdx.x == 0)
        for (int w = 1; w < 4; ++w) v = xyzz_add(v, load_xyzz<F>(sm + X * w));
    return v;
}

constexpr uint32_t kHeavySpan = 64;  // segments; longer buckets go to heavy_kernel

// One thread per bucket: empty -> infinity; a bucket spanning segments
// s0 < s1 sums its run partials (slot 0 or 1 in s0, slot 0 after). Buckets
// spanning more than kHeavySpan segments (skewed digits, e.g. a witness of
// 0/1 values) are queued for heavy_kernel instead of one serial thread.
template <class F, int NB>
__global__ void __launch_bounds__(128) fixup_kernel(const uint32_t* offs, const uint8_t* partials,
                                                    uint8_t* buckets, uint32_t* heavy,
                                                    uint32_t segsz) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= NB) return;
    constexpr int X = Lay<F>::XZ;
    const uint32_t s = offs[b], e = offs[b + 1];
    if (s == e) {
        store_inf<F>(buckets + (uint64_t)X * b);
        return;
    }
    const uint32_t s0 = s / segsz, s1 = (e - 1) / segsz;
    if (s0 == s1) return;
    if (s1 - s0 > kHeavySpan) {
        heavy[1 + atomicAdd(&heavy[0], 1u)] = b;
        return;
    }
    XYZZ<F> acc = load_xyzz<F>(partials + (uint64_t)X * (2ull * s0 + (s == s0 * segsz ? 0 : 1)));
    for (uint32_t sg = s0 + 1; sg <= s1; ++sg)
        acc = xyzz_add(acc, load_xyzz<F>(partials + (uint64_t)X * (2ull * sg)));
    store_xyzz(buckets + (uint64_t)X * b, acc);
}

// Heavy buckets in two passes: the segment partials of every queued bucket
// are cut into slices of kHeavySlice segments, one CTA per slice (grid-
// stride over all slices of all heavy buckets) sums its slice into
// heavy_part; then one CTA per heavy bucket sums its slice sums. A 0/1
// witness sends ~a million entries (16k segments) to one bucket: one CTA
// walking them was the longest kernel of such a proof.
constexpr uint32_t kHeavySlice = 256;  // segments per slice (2 per thread)
// slices of heavy bucket h, and the first slice index of h (nh is small)
__device__ __forceinline__ uint32_t heavy_slices(const uint32_t* offs, const uint32_t* heavy,
                                                 uint32_t h, uint32_t segsz) {
    const int b = heavy[1 + h];
    const uint32_t s0 = offs[b] / segsz, s1 = (offs[b + 1] - 1) / segsz;
    return (s1 - s0 + kHeavySlice) / kHeavySlice;  // segments s0..s1
}
template <class F>
__global__ void __launch_bounds__(128) heavy_slice_kernel(const uint32_t* offs,
                                                          const uint8_t* partials,
                                                          const uint32_t* heavy, uint32_t segsz,
                                                          uint8_t* heavy_part) {
    constexpr int X = Lay<F>::XZ;
    const uint32_t nh = heavy[0];
    uint32_t h = 0, first = 0;  // the bucket of the current item and its first slice
    for (uint32_t it = blockIdx.x;; it += gridDim.x) {
        while (h < nh && it >= first + heavy_slices(offs, heavy, h, segsz)) {
            first += heavy_slices(offs, heavy, h, segsz);
            ++h;
        }
        if (h >= nh) return;
        const int b = heavy[1 + h];
        const uint32_t s = offs[b];
        const uint32_t s0 = s / segsz, s1 = (offs[b + 1] - 1) / segsz;
        const uint32_t lo = s0 + (it - first) * kHeavySlice;
        const uint32_t hi = min(s1, lo + kHeavySlice - 1);
        XYZZ<F> acc = XYZZ<F>::inf();
        for (uint32_t sg = lo + threadIdx.x; sg <= hi; sg += blockDim.x) {
            // the bucket's first segment holds its run in slot 0 only if the
            // bucket starts the segment, else in slot 1
            const uint32_t slot = (sg == s0 && s != s0 * segsz) ? 1 : 0;
            acc = xyzz_add(acc, load_xyzz<F>(partials + (uint64_t)X * (2ull * sg + slot)));
        }
        acc = cta_sum128(acc);
        if (threadIdx.x == 0) store_xyzz(heavy_part + (uint64_t)X * it, acc);
        __syncthreads();
    }
}
template <class F>
__global__ void __launch_bounds__(128) heavy_final_kernel(const uint32_t* offs,
                                                          const uint32_t* heavy, uint32_t segsz,
                                                          const uint8_t* heavy_part,
                                                          uint8_t* buckets) {
    constexpr int X = Lay<F>::XZ;
    const uint32_t nh = heavy[0];
    uint32_t first = 0, h0 = 0;
    for (uint32_t h = blockIdx.x; h < nh; h += gridDim.x) {
        for (; h0 < h; ++h0) first += heavy_slices(offs, heavy, h0, segsz);
        const uint32_t ns = heavy_slices(offs, heavy, h, segsz);
        XYZZ<F> acc = XYZZ<F>::inf();
        for (uint32_t k = threadIdx.x; k < ns; k += blockDim.x)
            acc = xyzz_add(acc, load_xyzz<F>(heavy_part + (uint64_t)X * (first + k)));
        acc = cta_sum128(acc);
        if (threadIdx.x == 0) store_xyzz(buckets + (uint64_t)X * heavy[1 + h], acc);
        __syncthreads();
    }
}


// Segment j covers bucket indices [a, a+kRedSeg), weights a+1 .. a+kRedSeg:
// sum = tot + a*run with running sums from the top; one partial per CTA.
// (A work-efficient multi-level recursion on the run_j measured 2.7x slower
// here: every level pays a serial chain of point additions.)
// (blockIdx.y: the window's bucket set in a variable-base run)
template <class F, class Wn>
__global__ void __launch_bounds__(128) reduce_seg_kernel(const uint8_t* buckets, uint8_t* segsum) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    constexpr int X = Lay<F>::XZ;
    constexpr int kRedSeg = Wn::RedSeg, kRedThreads = Wn::RedThreads;
    buckets += (uint64_t)X * Wn::NB * blockIdx.y;
    segsum += (uint64_t)X * gridDim.x * blockIdx.y;
    XYZZ<F> tot = XYZZ<F>::inf();
    if (j < kRedThreads) {
        const int a = j * kRedSeg;
        XYZZ<F> run = XYZZ<F>::inf();
        for (int k = a + kRedSeg - 1; k >= a; --k) {
            run = xyzz_add(run, load_xyzz<F>(buckets + (uint64_t)X * k));
            tot = xyzz_add(tot, run);
        }
        if (a) tot = xyzz_add(tot, xyzz_mul_small(run, (uint32_t)a));
    }
    tot = cta_sum128(tot);
    if (threadIdx.x == 0) store_xyzz(segsum + (uint64_t)X * blockIdx.x, tot);
}

// Sum the per-CTA partials of reduce_seg (kRedThreads / 128 <= 64) and
// write the affine result.
// (blockIdx.x: the window in a variable-base run -> out[window])
template <class F, class Wn>
__global__ void __launch_bounds__(64) reduce_final_kernel(const uint8_t* segsum, uint8_t* out) {
    constexpr int X = Lay<F>::XZ;
    constexpr int kParts = Wn::RedThreads / 128;
    segsum += (uint64_t)X * kParts * blockIdx.x;
    out += (uint64_t)Lay<F>::AFF * blockIdx.x;
    __shared__ __align__(16) uint8_t sm[2 * sizeof(XYZZ<F>)];
    XYZZ<F> acc = XYZZ<F>::inf();
    for (int p = threadIdx.x; p < kParts; p += 64)
        acc = xyzz_add(acc, load_xyzz<F>(segsum + (uint64_t)X * p));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        XYZZ<F> o = shfl_xyzz(acc, d);
        if (lane < d) acc = xyzz_add(acc, o);
    }
    if (lane == 0) store_xyzz(sm + X * warp, acc);
    __syncthreads();
    if (threadIdx.x == 0) {
        XYZZ<F> r = xyzz_add(load_xyzz<F>(sm), load_xyzz<F>(sm + X));
        F x, y;
        to_affine(r, x, y);
        store_affine(out, x, y);
    }
}

// ---- batch-affine bucket levels (G1) ---------------------------------------
// Alternative to accumulate/fixup: each level adds the entries of every
// bucket pairwise in AFFINE coordinates, (x1,y1) + (x2,y2) with
// lambda = num / den (den = x2 - x1, or 2y for a doubling), 3 products + one
// shared inversion. The inversions of a warp's 32 x kAffK additions are
// batched (Montgomery's trick: prefix products per lane, a product scan
// across lanes, ONE binary-EEA inversion on lane 0 — ALU work, off the
// saturated IMAD pipe), so an addition costs ~6 products + 12/kAffK
// instead of the mixed XYZZ add's 8 products + a lazy difference. After
// ~log2(entries / buckets) levels the few points left per bucket are summed
// in XYZZ. EXPERIMENTAL, off by default (-DACEGPU_MSM_AFFINE=1 builds it in;
// ACEGPU_MSM_AFFINE=0 in the environment then selects XYZZ at run time):
// correct (the MSM tests pass on it) but G1 2^20 takes 8.6 ms vs 5.0 ms —
// each level re-gathers its input pairs in the back-substitution pass (DRAM
// 3.9 GB at level 0), 168 registers leave 12 warps/SM for random gathers,
// and the per-warp inversion puts a ~130 us latency floor under each level.
// A version staging the pairs in shared memory with a larger batch is the
// round-2 candidate (DESIGN.md round log).
#ifndef ACEGPU_MSM_AFFINE
#define ACEGPU_MSM_AFFINE 0
#endif
#ifndef ACEGPU_AFF_K
#define ACEGPU_AFF_K 8
#endif
constexpr int kAffK = ACEGPU_AFF_K;
inline bool affine_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("ACEGPU_MSM_AFFINE");
        return !e || e[0] != '0';
    }();
    return on;
}

// out[b] = ceil(size_b / 2), out[NB] = 0 (for the exclusive scan)
__global__ void halve_counts_kernel(const uint32_t* in_offs, uint32_t* cnt) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b > kMsmBuckets) return;
    cnt[b] = b < kMsmBuckets ? (in_offs[b + 1] - in_offs[b] + 1) / 2 : 0u;
}

__device__ __forceinline__ Fq shfl_fq(const Fq& a, int lane_or_delta, int mode) {
    Fq r;
#pragma unroll
    for (int k = 0; k < 8; ++k)
        r.v[k] = mode == 0 ? __shfl_sync(0xffffffffu, a.v[k], lane_or_delta)
                 : mode == 1 ? __shfl_up_sync(0xffffffffu, a.v[k], lane_or_delta)
                             : __shfl_down_sync(0xffffffffu, a.v[k], lane_or_delta);
    return r;
}

template <bool FIRST>
__device__ __forceinline__ bool aff_load(const uint8_t* table, const uint32_t* sorted,
                                         const uint8_t* pts, uint32_t i, Fq& x, Fq& y) {
    if (FIRST) {
        const uint32_t v = sorted[i];
        const bool fin = load_affine<Fq>(table + 64ull * (v & 0x7FFFFFFFu), x, y);
        if (fin && (v >> 31)) y = neg(y);
        return fin;
    }
    return load_affine<Fq>(pts + 64ull * i, x, y);
}

// Slot j of bucket b: its input pair, the case and (num, den).
// kind: 0 = copy P1, 1 = copy P2, 2 = infinity, 3 = add (num / den)
template <bool FIRST>
__device__ __forceinline__ int aff_pair(const uint8_t* table, const uint32_t* sorted,
                                        const uint8_t* pts, const uint32_t* in_offs,
                                        const uint32_t* out_offs, int b, uint32_t j, Fq& x1,
                                        Fq& y1, Fq& x2, Fq& y2, Fq& num, Fq& den) {
    const uint32_t i0 = in_offs[b] + 2 * (j - out_offs[b]);
    const bool f1 = aff_load<FIRST>(table, sorted, pts, i0, x1, y1);
    const bool f2 = i0 + 1 < in_offs[b + 1] && aff_load<FIRST>(table, sorted, pts, i0 + 1, x2, y2);
    den = Fq::one();
    if (!f2) return f1 ? 0 : 2;
    if (!f1) return 1;
    if (x1 == x2) {
        if (!(y1 == y2)) return 2;  // P + (-P)
        const Fq xx = fsqr(x1);
        num = add(add(xx, xx), xx);  // doubling: 3x^2 / 2y (no 2-torsion in G1)
        den = add(y1, y1);
        return 3;
    }
    num = sub(y2, y1);
    den = sub(x2, x1);
    return 3;
}

// One level: output slot j = pair (2(j - out_offs[b]), +1) of bucket b's
// input run. Every lane of a warp takes part in the scans (no early exit).
template <bool FIRST>
__global__ void __launch_bounds__(128) affine_level_kernel(const uint8_t* table,
                                                           const uint32_t* sorted,
                                                           const uint8_t* in_pts,
                                                           const uint32_t* in_offs,
                                                           const uint32_t* out_offs,
                                                           uint8_t* out_pts) {
    const uint32_t total = out_offs[kMsmBuckets];
    const uint32_t j0 = (blockIdx.x * blockDim.x + threadIdx.x) * kAffK;
    const int lane = threadIdx.x & 31;
    int bs[kAffK];
    Fq pre[kAffK];
    Fq run = Fq::one();
    int b = j0 < total ? bucket_of(out_offs, j0) : 0;
#pragma unroll
    for (int s = 0; s < kAffK; ++s) {
        const uint32_t j = j0 + s;
        Fq den = Fq::one();
        if (j < total) {
            while (out_offs[b + 1] <= j) ++b;
            Fq x1, y1, x2, y2, num;
            aff_pair<FIRST>(table, sorted, in_pts, in_offs, out_offs, b, j, x1, y1, x2, y2, num,
                            den);
        }
        bs[s] = b;
        run = fmul(run, den);
        pre[s] = run;
    }
    // inclusive prefix and suffix products of the lane totals across the warp
    Fq q = run, sx = run;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const Fq o = shfl_fq(q, d, 1), u = shfl_fq(sx, d, 2);
        if (lane >= d) q = fmul(q, o);
        if (lane + d < 32) sx = fmul(sx, u);
    }
    Fq inv = shfl_fq(q, 31, 0);
    if (lane == 0) inv = finv(inv);
    inv = shfl_fq(inv, 0, 0);
    Fq pe = shfl_fq(q, 1, 1), se = shfl_fq(sx, 1, 2);
    if (lane == 0) pe = Fq::one();
    if (lane == 31) se = Fq::one();
    Fq inv_run = fmul(fmul(inv, pe), se);  // 1 / (this lane's product)
#pragma unroll
    for (int s = kAffK - 1; s >= 0; --s) {
        const uint32_t j = j0 + s;
        if (j >= total) continue;
        Fq x1, y1, x2, y2, num, den;
        const int kind = aff_pair<FIRST>(table, sorted, in_pts, in_offs, out_offs, bs[s], j, x1, y1,
                                         x2, y2, num, den);
        const Fq inv_den = s > 0 ? fmul(inv_run, pre[s - 1]) : inv_run;
        inv_run = fmul(inv_run, den);
        uint8_t* o = out_pts + 64ull * j;
        if (kind == 3) {
            const Fq lam = fmul(num, inv_den);
            const Fq x3 = sub(sub(fsqr(lam), x1), x2);
            store_affine(o, x3, sub(fmul(lam, sub(x1, x3)), y1));
        } else if (kind == 0) {
            store_affine(o, x1, y1);
        } else if (kind == 1) {
            store_affine(o, x2, y2);
        } else {
            store_affine(o, Fq::zero(), Fq::zero());
        }
    }
}

// After the levels: one thread per bucket sums its (few) remaining affine
// points into XYZZ; long runs (skewed digits) go to the heavy queue.
__global__ void __launch_bounds__(128) affine_finish_kernel(const uint8_t* pts,
                                                            const uint32_t* offs,
                                                            uint8_t* buckets, uint32_t* heavy) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= kMsmBuckets) return;
    const uint32_t s = offs[b], e = offs[b + 1];
    if (e - s > 64) {
        heavy[1 + atomicAdd(&heavy[0], 1u)] = b;
        return;
    }
    XYZZ<Fq> acc = XYZZ<Fq>::inf();
    for (uint32_t i = s; i < e; ++i) {
        Fq x, y;
        if (load_affine<Fq>(pts + 64ull * i, x, y)) acc = xyzz_madd<Fq>(acc, x, y);
    }
    store_xyzz(buckets + 128ull * b, acc);
}

__global__ void __launch_bounds__(128) affine_heavy_kernel(const uint8_t* pts, const uint32_t* offs,
                                                           uint8_t* buckets, const uint32_t* heavy) {
    const uint32_t nh = heavy[0];
    for (uint32_t h = blockIdx.x; h < nh; h += gridDim.x) {
        const int b = heavy[1 + h];
        XYZZ<Fq> acc = XYZZ<Fq>::inf();
        for (uint32_t i = offs[b] + threadIdx.x; i < offs[b + 1]; i += blockDim.x) {
            Fq x, y;
            if (load_affine<Fq>(pts + 64ull * i, x, y)) acc = xyzz_madd<Fq>(acc, x, y);
        }
        acc = cta_sum128(acc);
        if (threadIdx.x == 0) store_xyzz(buckets + 128ull * b, acc);
        __syncthreads();
    }
}

// Variable-base result: win[r * W + w] = the window-w sum of sub-range r
// (affine); out = sum_w 2^(c w) sum_r win[r W + w] (Horner from the top).
template <class F, class Wn>
__global__ void combine_windows_kernel(const uint8_t* win, uint32_t nsub, uint8_t* out) {
    if (threadIdx.x || blockIdx.x) return;
    constexpr int A = Lay<F>::AFF;
    XYZZ<F> acc = XYZZ<F>::inf();
    for (int w = Wn::W - 1; w >= 0; --w) {
        for (int d = 0; d < Wn::width(w); ++d) acc = xyzz_dbl(acc);
        for (uint32_t r = 0; r < nsub; ++r) {
            F x, y;
            if (load_affine<F>(win + (uint64_t)A * (r * Wn::W + w), x, y))
                acc = xyzz_madd<F>(acc, x, y);
        }
    }
    F x, y;
    to_affine(acc, x, y);
    store_affine(out, x, y);
}

__global__ void points_convert_kernel(uint8_t* pts, uint64_t n_elems, int to) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n_elems) return;
    Fq x = load<FqCfg>(pts + 32 * i);
    store<FqCfg>(pts + 32 * i, to ? to_mont(x) : from_mont(x));
}

template <class F>
int prepare_t(const uint8_t* bases, uint64_t n, uint8_t* table, cudaStream_t s) {
    prepare_kernel<F><<<(n + 127) / 128, 128, 0, s>>>(bases, n, table);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// One Pippenger pass. Fixed base (VB = false): table = the window tables,
// out = the affine result. Variable base (VB = true): table = the n bases
// themselves, one bucket set per window, out = the kMsmWindows affine window
// sums (combine_windows_kernel weights them).
// Phase 1 of a Pippenger pass: the scalars' signed digits sorted into bucket
// order (sc.offs, sc.sorted); several tables over the same scalars share it.
// The segment size for n scalars, and the scratch grown to hold them.
template <bool VB, class Wn>
int ensure_core(uint64_t n, MsmScratch& sc, cudaStream_t s, uint32_t& segsz_out,
                uint64_t& nseg_out) {
    constexpr int NB = VB ? Wn::W * Wn::NB : Wn::NB;
    const uint64_t cap = (uint64_t)Wn::W * n;
    // segment length: kMsmSeg, shorter for small MSMs (>= ~19k threads, so a
    // verifier-size MSM is not a few hundred threads of 64 serial adds)
    uint32_t segsz = kMsmSeg;
    while (segsz > 4 && cap / segsz < 148ull * 128) segsz >>= 1;
    const uint64_t nseg = (cap + segsz - 1) / segsz;
    if (sc.cap_entries < cap || sc.cap_segs < nseg || sc.cap_buckets < (uint64_t)NB || !sc.hist) {
        const uint64_t keep = std::max<uint64_t>(cap, sc.cap_entries);
        const uint64_t keep_segs = std::max<uint64_t>(nseg, sc.cap_segs);
        const uint64_t nbk = std::max<uint64_t>(NB, sc.cap_buckets);
        uint8_t* win = sc.win;  // the variable-base window sums survive the regrow
        const uint64_t win_cap = sc.win_cap;
        sc.win = nullptr;
        sc.release();
        sc.win = win;
        sc.win_cap = win_cap;
        if (cudaMalloc(&sc.hist, 4 * (nbk + 1)) || cudaMalloc(&sc.offs, 4 * (nbk + 1)) ||
            cudaMalloc(&sc.cursor, 4 * nbk) || cudaMalloc(&sc.sorted, 4 * keep) ||
            cudaMalloc(&sc.partials, (size_t)256 * 2 * keep_segs) ||  // G2 size: scratch shared
            cudaMalloc(&sc.buckets, (size_t)256 * nbk) ||
            cudaMalloc(&sc.segsum, (size_t)256 * 1024 * std::max<uint64_t>(Wn::W, 16)) ||
            cudaMalloc(&sc.heavy, 4 * (nbk + 1)) ||
            // slices: <= nseg / kHeavySlice + one partial slice per heavy bucket
            // (each spans > kHeavySpan segments)
            cudaMalloc(&sc.heavy_part,
                       (size_t)256 * (keep_segs / kHeavySlice + keep_segs / kHeavySpan + 16)))
            return -1;
        cub::DeviceScan::ExclusiveSum(nullptr, sc.scan_bytes, sc.hist, sc.offs, (int)nbk + 1, s);
        if (cudaMalloc(&sc.scan_tmp, sc.scan_bytes)) return -1;
        sc.cap_entries = keep;
        sc.cap_segs = keep_segs;
        sc.cap_buckets = nbk;
    }
    segsz_out = segsz;
    nseg_out = nseg;
    return 0;
}

template <bool VB, class Wn>
int sort_core(uint64_t n, const uint8_t* scalars, MsmScratch& sc, cudaStream_t s,
              uint32_t& segsz_out, uint64_t& nseg_out) {
    constexpr int NB = VB ? Wn::W * Wn::NB : Wn::NB;
    uint32_t segsz;
    uint64_t nseg;
    if (ensure_core<VB, Wn>(n, sc, s, segsz, nseg)) return -1;
    cudaMemsetAsync(sc.hist, 0, 4 * (NB + 1), s);
    const unsigned gb = (unsigned)((n + 255) / 256);
    // large variable-base sorts: window passes over a key array (see
    // digits_keys_kernel); ACEGPU_SORT_SPLIT = bucket ranges per window (0: off)
    static const int split = [] {
        const char* e = std::getenv("ACEGPU_SORT_SPLIT");
        return e ? std::atoi(e) : 2;
    }();
    if (VB && split > 0 && n >= (1ull << 22)) {
        if (sc.keys_cap < (uint64_t)Wn::W * n) {
            if (sc.keys) cudaFree(sc.keys);
            sc.keys = nullptr;
            sc.keys_cap = 0;
            if (cudaMalloc(&sc.keys, 4ull * Wn::W * n)) return -1;
            sc.keys_cap = (uint64_t)Wn::W * n;
        }
        digits_keys_kernel<Wn><<<gb, 256, 0, s>>>(scalars, n, sc.keys, sc.hist);
        size_t scan_bytes = sc.scan_bytes;
        if (cub::DeviceScan::ExclusiveSum(sc.scan_tmp, scan_bytes, sc.hist, sc.offs, NB + 1, s) !=
            cudaSuccess)
            return -1;
        cudaMemcpyAsync(sc.cursor, sc.offs, 4 * NB, cudaMemcpyDeviceToDevice, s);
        for (int w = 0; w < Wn::W; ++w) {
            const uint32_t nbw = 1u << (Wn::width(w) - 1);  // buckets this window uses
            for (int r = 0; r < split; ++r) {
                const uint32_t lo = (uint32_t)((uint64_t)nbw * r / split),
                               hi = (uint32_t)((uint64_t)nbw * (r + 1) / split);
                scatter_range_kernel<<<gb, 256, 0, s>>>(sc.keys + (uint64_t)w * n, n, lo, hi,
                                                        sc.cursor + (uint64_t)w * Wn::NB,
                                                        sc.sorted);
            }
        }
        segsz_out = segsz;
        nseg_out = nseg;
        return cudaGetLastError() == cudaSuccess ? 0 : -1;
    }
    count_kernel<VB, Wn><<<gb, 256, 0, s>>>(scalars, n, sc.hist);
    // offs = exclusive scan of hist[0..NB] (hist[NB] = 0 -> offs[NB] = total)
    size_t scan_bytes = sc.scan_bytes;
    if (cub::DeviceScan::ExclusiveSum(sc.scan_tmp, scan_bytes, sc.hist, sc.offs, NB + 1, s) !=
        cudaSuccess)
        return -1;
    cudaMemcpyAsync(sc.cursor, sc.offs, 4 * NB, cudaMemcpyDeviceToDevice, s);
    scatter_kernel<VB, Wn><<<gb, 256, 0, s>>>(scalars, n, sc.cursor, sc.sorted);
    segsz_out = segsz;
    nseg_out = nseg;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// Phase 2: bucket accumulation of `table` over the sorted entries, fixup,
// heavy buckets, reduction -> out (fixed base: the affine result; variable
// base: the W window sums).
// (srt: the scratch holding the sorted entries when another stream's scratch
// sorted them; sc: this accumulation's buckets, partials and reductions)
template <class F, bool VB, class Wn>
int acc_core(const uint8_t* table, uint64_t n, MsmScratch& sc, uint32_t segsz, uint64_t nseg,
             uint8_t* out, cudaStream_t s, const MsmScratch* srt = nullptr) {
    constexpr int X = Lay<F>::XZ;
    constexpr int NB = VB ? Wn::W * Wn::NB : Wn::NB;
    const uint64_t cap = (uint64_t)Wn::W * n;
    const uint32_t* sorted = srt ? srt->sorted : sc.sorted;
    const uint32_t* offs = srt ? srt->offs : sc.offs;
    cudaMemsetAsync(sc.heavy, 0, 4, s);
    bool affine = false;
    if constexpr (sizeof(F) == sizeof(Fq) && !VB) affine = ACEGPU_MSM_AFFINE && affine_enabled();
    if (affine) {
        // levels until ~1 point per bucket remains for uniform digits (the
        // finish kernel sums what is left); output-slot upper bounds size the
        // grids without a host sync
        uint64_t U = cap, ub[24];
        int L = 0;
        do {
            U = U / 2 + kMsmBuckets;
            ub[L++] = U;
        } while ((cap >> L) > (uint64_t)kMsmBuckets && L < 20);
        if (sc.aff_cap < ub[0]) {
            for (void* p : {(void*)sc.aff_pts[0], (void*)sc.aff_pts[1]})
                if (p) cudaFree(p);
            if (cudaMalloc(&sc.aff_pts[0], 64 * ub[0]) || cudaMalloc(&sc.aff_pts[1], 64 * ub[0]))
                return -1;
            sc.aff_cap = ub[0];
        }
        if (!sc.aff_offs[0] &&
            (cudaMalloc(&sc.aff_offs[0], 4 * (kMsmBuckets + 1)) ||
             cudaMalloc(&sc.aff_offs[1], 4 * (kMsmBuckets + 1)) ||
             cudaMalloc(&sc.aff_cnt, 4 * (kMsmBuckets + 1))))
            return -1;
        const uint32_t* in_offs = sc.offs;
        const uint8_t* in_pts = nullptr;
        for (int l = 0; l < L; ++l) {
            uint32_t* out_offs = sc.aff_offs[l & 1];
            uint8_t* out_pts = sc.aff_pts[l & 1];
            halve_counts_kernel<<<kMsmBuckets / 128 + 1, 128, 0, s>>>(in_offs, sc.aff_cnt);
            if (cub::DeviceScan::ExclusiveSum(sc.scan_tmp, sc.scan_bytes, sc.aff_cnt, out_offs,
                                              kMsmBuckets + 1, s) != cudaSuccess)
                return -1;
            const unsigned grid = (unsigned)((ub[l] + 128ull * kAffK - 1) / (128ull * kAffK));
            if (l == 0)
                affine_level_kernel<true><<<grid, 128, 0, s>>>(table, sc.sorted, nullptr, in_offs,
                                                               out_offs, out_pts);
            else
                affine_level_kernel<false><<<grid, 128, 0, s>>>(nullptr, nullptr, in_pts, in_offs,
                                                                out_offs, out_pts);
            in_offs = out_offs;
            in_pts = out_pts;
        }
        affine_finish_kernel<<<kMsmBuckets / 128, 128, 0, s>>>(in_pts, in_offs, sc.buckets,
                                                               sc.heavy);
        affine_heavy_kernel<<<148, 128, 0, s>>>(in_pts, in_offs, sc.buckets, sc.heavy);
    } else {
        accumulate_kernel<F, NB><<<(unsigned)((nseg + 127) / 128), 128, 0, s>>>(
            table, sorted, offs, sc.buckets, sc.partials, segsz);
        fixup_kernel<F, NB><<<NB / 128, 128, 0, s>>>(offs, sc.partials, sc.buckets, sc.heavy,
                                                     segsz);
        heavy_slice_kernel<F><<<4 * 148, 128, 0, s>>>(offs, sc.partials, sc.heavy, segsz,
                                                        sc.heavy_part);
        heavy_final_kernel<F><<<148, 128, 0, s>>>(offs, sc.heavy, segsz, sc.heavy_part,
                                                  sc.buckets);
    }
    constexpr unsigned nw = VB ? Wn::W : 1;
    reduce_seg_kernel<F, Wn><<<dim3(Wn::RedThreads / 128, nw), 128, 0, s>>>(sc.buckets, sc.segsum);
    reduce_final_kernel<F, Wn><<<nw, 64, 0, s>>>(sc.segsum, out);
    (void)X;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

template <class F, bool VB, class Wn>
int run_core(const uint8_t* table, uint64_t n, const uint8_t* scalars, MsmScratch& sc,
             uint8_t* out, cudaStream_t s) {
    uint32_t segsz;
    uint64_t nseg;
    if (sort_core<VB, Wn>(n, scalars, sc, s, segsz, nseg)) return -1;
    return acc_core<F, VB, Wn>(table, n, sc, segsz, nseg, out, s);
}

template <bool VB, class Wn>
int acc_any(int group, const uint8_t* table, uint64_t n, MsmScratch& sc, uint32_t segsz,
            uint64_t nseg, uint8_t* out, cudaStream_t s) {
    return group == 2 ? acc_core<Fq2, VB, Wn>(table, n, sc, segsz, nseg, out, s)
                      : acc_core<Fq, VB, Wn>(table, n, sc, segsz, nseg, out, s);
}

template <class F>
int run_t(const uint8_t* table, uint64_t n, const uint8_t* scalars, MsmScratch& sc, uint8_t* out,
          cudaStream_t s) {
    return run_core<F, false, WinFixed>(table, n, scalars, sc, out, s);
}

// Variable base: sub-ranges of <= sub points (their W x sub sorted entries
// stay below 2^32), W window sums each, then one Horner combination; k
// tables (G1 or G2) over the same scalars share each sub-range's sort.
template <class Wn>
int run_vb_multi_t(int k, const int* groups, const uint8_t* const* bases, uint64_t n,
                   const uint8_t* scalars, MsmScratch& sc, uint8_t* const* outs, uint64_t sub,
                   cudaStream_t s) {
    if (!sub || sub > kMsmVbSubMax) sub = kMsmVbSubMax;
    uint64_t nsub = n ? (n + sub - 1) / sub : 1;
    // balanced sub-ranges (each pays its own per-window reductions and
    // fixups: 140 M points as 2 x 70 M instead of 67 + 67 + 6 M)
    if (n) sub = (n + nsub - 1) / nsub;
    const uint64_t per = (uint64_t)256 * Wn::W * nsub;  // one table's window sums
    if (sc.win_cap < k * nsub) {
        if (sc.win) cudaFree(sc.win);
        sc.win = nullptr;
        sc.win_cap = 0;
        if (cudaMalloc(&sc.win, per * k)) return -1;
        sc.win_cap = k * nsub;
    }
    if (!n) cudaMemsetAsync(sc.win, 0, per * k, s);
    for (uint64_t r = 0; r < n; r += sub) {
        const uint64_t len = std::min<uint64_t>(sub, n - r);
        uint32_t segsz;
        uint64_t nseg;
        if (sort_core<true, Wn>(len, scalars + 32 * r, sc, s, segsz, nseg)) return -1;
        for (int i = 0; i < k; ++i) {
            const uint64_t A = 64ull * groups[i];
            if (acc_any<true, Wn>(groups[i], bases[i] + A * r, len, sc, segsz, nseg,
                                  sc.win + per * i + A * Wn::W * (r / sub), s))
                return -1;
        }
    }
    for (int i = 0; i < k; ++i) {
        if (groups[i] == 2)
            combine_windows_kernel<Fq2, Wn><<<1, 32, 0, s>>>(sc.win + per * i, (uint32_t)nsub, outs[i]);
        else
            combine_windows_kernel<Fq, Wn><<<1, 32, 0, s>>>(sc.win + per * i, (uint32_t)nsub, outs[i]);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// Window size by size: c = 20 (13 windows x 2^19 buckets) pays off over
// 2^26-point sub-ranges; up to ACEGPU_MSM_VB_SMALL points (small split slices)
// c = 17 (15 x 2^16 buckets): 15 % more bucket entries but a fraction of
// the per-window reductions and fixups.
#ifndef ACEGPU_MSM_VB_SMALL
#define ACEGPU_MSM_VB_SMALL (1ull << 24)
#endif
#ifndef ACEGPU_MSM_VB_MID
#define ACEGPU_MSM_VB_MID 0  // c = 19 tier off: measured within noise (8 ranks -1 %, 4 ranks +2 %)
#endif
int run_vb_multi(int k, const int* groups, const uint8_t* const* bases, uint64_t n,
                 const uint8_t* scalars, MsmScratch& sc, uint8_t* const* outs, uint64_t sub,
                 cudaStream_t s) {
    const char* e = std::getenv("ACEGPU_MSM_VB_SMALL");  // per call: tests force either form
    const uint64_t small = e ? std::strtoull(e, nullptr, 0) : (uint64_t)ACEGPU_MSM_VB_SMALL;
    const char* em = std::getenv("ACEGPU_MSM_VB_MID");   // c = 19 up to this size
    const uint64_t mid = em ? std::strtoull(em, nullptr, 0) : (uint64_t)ACEGPU_MSM_VB_MID;
    if (n <= small) return run_vb_multi_t<WinFixed>(k, groups, bases, n, scalars, sc, outs, sub, s);
    if (n <= mid) return run_vb_multi_t<WinMid>(k, groups, bases, n, scalars, sc, outs, sub, s);
    return run_vb_multi_t<WinVb>(k, groups, bases, n, scalars, sc, outs, sub, s);
}

}  // namespace

void MsmScratch::release() {
    void* ps[] = {hist, offs, cursor, sorted, partials, buckets, segsum, scan_tmp, heavy,
                  aff_pts[0], aff_pts[1], aff_offs[0], aff_offs[1], aff_cnt, win, keys};
    keys = nullptr;
    keys_cap = 0;
    win = nullptr;
    win_cap = 0;
    cap_buckets = 0;
    for (void* p : ps)
        if (p) cudaFree(p);
    aff_pts[0] = aff_pts[1] = nullptr;
    aff_offs[0] = aff_offs[1] = aff_cnt = nullptr;
    aff_cap = 0;
    cap_segs = 0;
    hist = offs = cursor = sorted = heavy = nullptr;
    if (heavy_part) cudaFree(heavy_part);
    heavy_part = nullptr;
    partials = buckets = segsum = nullptr;
    scan_tmp = nullptr;
    scan_bytes = 0;
    cap_entries = 0;
}

int msm_prepare(int group, const uint8_t* bases, uint64_t n, uint8_t* table, cudaStream_t s) {
    return group == 2 ? prepare_t<Fq2>(bases, n, table, s) : prepare_t<Fq>(bases, n, table, s);
}

int msm_run(int group, const uint8_t* table, uint64_t n, const uint8_t* scalars, MsmScratch& sc,
            uint8_t* out, cudaStream_t s) {
    return group == 2 ? run_t<Fq2>(table, n, scalars, sc, out, s)
                      : run_t<Fq>(table, n, scalars, sc, out, s);
}

int msm_run_vb(int group, const uint8_t* bases, uint64_t n, const uint8_t* scalars,
               MsmScratch& sc, uint8_t* out, cudaStream_t s, uint64_t sub) {
    return run_vb_multi(1, &group, &bases, n, scalars, sc, &out, sub, s);
}

int msm_run_vb_multi(int k, const int* groups, const uint8_t* const* bases, uint64_t n,
                     const uint8_t* scalars, MsmScratch& sc, uint8_t* const* outs, cudaStream_t s,
                     uint64_t sub) {
    return run_vb_multi(k, groups, bases, n, scalars, sc, outs, sub, s);
}

int msm_sort(uint64_t n, const uint8_t* scalars, MsmScratch& sc, MsmSorted& info,
             cudaStream_t s) {
    info.n = n;
    return sort_core<false, WinFixed>(n, scalars, sc, s, info.segsz, info.nseg);
}

int msm_accumulate(int group, const uint8_t* table, const MsmScratch& srt, const MsmSorted& info,
                   MsmScratch& acc, uint8_t* out, cudaStream_t s) {
    uint32_t segsz;
    uint64_t nseg;
    if (ensure_core<false, WinFixed>(info.n, acc, s, segsz, nseg)) return -1;
    return group == 2 ? acc_core<Fq2, false, WinFixed>(table, info.n, acc, info.segsz, info.nseg,
                                                       out, s, &srt)
                      : acc_core<Fq, false, WinFixed>(table, info.n, acc, info.segsz, info.nseg,
                                                      out, s, &srt);
}

int msm_run_multi(int k, const int* groups, const uint8_t* const* tables, uint64_t n,
                  const uint8_t* scalars, MsmScratch& sc, uint8_t* const* outs, cudaStream_t s) {
    uint32_t segsz;
    uint64_t nseg;
    if (sort_core<false, WinFixed>(n, scalars, sc, s, segsz, nseg)) return -1;
    for (int i = 0; i < k; ++i)
        if (acc_any<false, WinFixed>(groups[i], tables[i], n, sc, segsz, nseg, outs[i], s))
            return -1;
    return 0;
}

void launch_points_convert(int group, uint8_t* pts, uint64_t n, int to_mont, cudaStream_t s) {
    launch_fq_convert(pts, n * 2 * group, to_mont, s);
}

void launch_fq_convert(uint8_t* elems, uint64_t n, int to_mont, cudaStream_t s) {
    if (n) points_convert_kernel<<<(n + 255) / 256, 256, 0, s>>>(elems, n, to_mont);
}

}  // namespace bn
}  // namespace ace_gpu
