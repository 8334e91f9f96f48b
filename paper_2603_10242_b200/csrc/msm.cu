// Pippenger multi-scalar multiplication over BN254 G1 and G2 for sm_100a
// (north-star row a21: K8/K9 of SURVEY §2b; the reference has none).
//
// Fixed-base form: the proving key's bases are fixed, so `msm_prepare`
// stores table[w][i] = 2^(16 w) P_i once (affine). A run then needs no
// doublings between windows: every (window, point) pair with a non-zero
// signed 16-bit digit d lands in one of 2^15 buckets |d| of a single bucket
// set, and the result is sum_k k * B_k.
//
//   1. count    : signed digits of each scalar -> bucket histogram (atomics)
//   2. scan     : exclusive prefix sum -> bucket offsets
//   3. scatter  : (window*n + i | sign) into bucket order
//   4. accumulate: each thread adds kMsmSeg sorted entries (mixed XYZZ adds,
//                 8M + 2S each), finished buckets written directly, the
//                 first/last (split) buckets of a segment as partials
//   5. fixup    : one warp per split bucket sums its partials (shuffles)
//   6. reduce   : sum_k k*B_k by per-segment running sums + small scalar
//                 multiples, then a block reduction, then affine.
// Bound: IMAD pipe (Fq mul = CIOS carry chains). Work ~ (W*n) mixed adds.
#include <cuda_runtime.h>

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
#ifndef ACEGPU_RED_SEG
#define ACEGPU_RED_SEG 4
#endif
template <class F>
struct Lay {
    static constexpr int EB = felem_bytes<F>();
    static constexpr int AFF = 2 * EB;
    static constexpr int XZ = 4 * EB;
    // accumulate_kernel min CTAs/SM (register cap): G2's Fq2 temporaries
    // take 216 registers -> 2 CTAs (8 warps) per SM; capping them spills
    // and measured slower
    static constexpr int ACC_MIN_CTAS = EB == 32 ? 1 : ACEGPU_G2_ACC_MINB;
};

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

// ---- prepare: table[w*n + i] = 2^(16w) P_i ----------------------------------
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

// Signed base-2^16 digits of a canonical scalar < r < 2^254 (16 windows).
__device__ __forceinline__ void digits16(const uint8_t* s, int32_t d[kMsmWindows]) {
    const uint4* q = reinterpret_cast<const uint4*>(s);
    uint4 a = q[0], b = q[1];
    const uint32_t limb[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t carry = 0;
#pragma unroll
    for (int w = 0; w < kMsmWindows; ++w) {
        uint32_t raw = ((limb[w >> 1] >> (16 * (w & 1))) & 0xFFFFu) + carry;
        if (raw > (1u << (kMsmC - 1))) {
            d[w] = (int32_t)raw - (1 << kMsmC);
            carry = 1;
        } else {
            d[w] = (int32_t)raw;
            carry = 0;
        }
    }
}

__global__ void count_kernel(const uint8_t* scalars, uint64_t n, uint32_t* hist) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t d[kMsmWindows];
    digits16(scalars + 32 * i, d);
#pragma unroll
    for (int w = 0; w < kMsmWindows; ++w)
        if (d[w]) atomicAdd(&hist[abs(d[w]) - 1], 1u);
}

// Exclusive scans (one CTA of 1024 threads) of the bucket sizes -> entry
// offsets, and of the per-bucket chunk counts ceil(size / kMsmSeg) -> chunk
// offsets. Chunks never straddle buckets.
__global__ void __launch_bounds__(1024) scan_kernel(const uint32_t* hist, uint32_t* offs,
                                                    uint32_t* cursor, uint32_t* coffs) {
    __shared__ uint32_t part[1024], cpart[1024];
    constexpr int per = kMsmBuckets / 1024;
    const int t = threadIdx.x;
    uint32_t loc[per], cloc[per], sum = 0, csum = 0;
#pragma unroll
    for (int k = 0; k < per; ++k) {
        const uint32_t h = hist[t * per + k];
        loc[k] = sum;
        cloc[k] = csum;
        sum += h;
        csum += (h + kMsmSeg - 1) / kMsmSeg;
    }
    part[t] = sum;
    cpart[t] = csum;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        uint32_t v = t >= off ? part[t - off] : 0;
        uint32_t cv = t >= off ? cpart[t - off] : 0;
        __syncthreads();
        part[t] += v;
        cpart[t] += cv;
        __syncthreads();
    }
    const uint32_t base = t ? part[t - 1] : 0, cbase = t ? cpart[t - 1] : 0;
#pragma unroll
    for (int k = 0; k < per; ++k) {
        offs[t * per + k] = base + loc[k];
        cursor[t * per + k] = base + loc[k];
        coffs[t * per + k] = cbase + cloc[k];
    }
    if (t == 1023) {
        offs[kMsmBuckets] = part[1023];
        coffs[kMsmBuckets] = cpart[1023];
    }
}

__global__ void scatter_kernel(const uint8_t* scalars, uint64_t n, uint32_t* cursor,
                               uint32_t* sorted) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t d[kMsmWindows];
    digits16(scalars + 32 * i, d);
#pragma unroll
    for (int w = 0; w < kMsmWindows; ++w) {
        if (!d[w]) continue;
        const uint32_t pos = atomicAdd(&cursor[abs(d[w]) - 1], 1u);
        sorted[pos] = (uint32_t)(w * n + i) | (d[w] < 0 ? 0x80000000u : 0u);
    }
}

__device__ __forceinline__ int bucket_of(const uint32_t* offs, uint32_t pos) {
    int lo = 0, hi = kMsmBuckets;  // offs[lo] <= pos < offs[hi]
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (offs[mid] <= pos) lo = mid;
        else hi = mid;
    }
    return lo;
}

// One thread per chunk (<= kMsmSeg entries of one bucket): mixed-add the
// chunk's bases into one XYZZ partial.
template <class F>
__global__ void __launch_bounds__(128, Lay<F>::ACC_MIN_CTAS) accumulate_kernel(const uint8_t* table,
                                                         const uint32_t* sorted,
                                                         const uint32_t* offs,
                                                         const uint32_t* coffs,
                                                         uint8_t* partials) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= coffs[kMsmBuckets]) return;
    constexpr int A = Lay<F>::AFF, X = Lay<F>::XZ;
    const int b = bucket_of(coffs, c);
    const uint32_t p0 = offs[b] + (c - coffs[b]) * kMsmSeg;
    const uint32_t p1 = min(offs[b + 1], p0 + kMsmSeg);
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
    }
    store_xyzz(partials + (uint64_t)X * c, acc);
}

// One thread per bucket: sum its chunk partials (infinity when empty).
template <class F>
__global__ void __launch_bounds__(128) bucket_sum_kernel(const uint32_t* coffs,
                                                         const uint8_t* partials,
                                                         uint8_t* buckets) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= kMsmBuckets) return;
    constexpr int X = Lay<F>::XZ;
    XYZZ<F> acc = XYZZ<F>::inf();
    for (uint32_t c = coffs[b]; c < coffs[b + 1]; ++c)
        acc = xyzz_add(acc, load_xyzz<F>(partials + (uint64_t)X * c));
    store_xyzz(buckets + (uint64_t)X * b, acc);
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

constexpr int kRedSeg = ACEGPU_RED_SEG;              // buckets per reducing thread
constexpr int kRedThreads = kMsmBuckets / kRedSeg;  // 4096

// Segment j covers bucket indices [a, a+kRedSeg), weights a+1 .. a+kRedSeg:
// sum = tot + a*run with running sums from the top.
template <class F>
__global__ void __launch_bounds__(128) reduce_seg_kernel(const uint8_t* buckets, uint8_t* segsum) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    constexpr int X = Lay<F>::XZ;
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
    // one partial per CTA: warp shuffles, then the 4 warp sums
    __shared__ __align__(16) uint8_t sm[4 * sizeof(XYZZ<F>)];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        XYZZ<F> o = shfl_xyzz(tot, d);
        if (lane < d) tot = xyzz_add(tot, o);
    }
    if (lane == 0) store_xyzz(sm + X * warp, tot);
    __syncthreads();
    if (threadIdx.x == 0) {
        XYZZ<F> r = load_xyzz<F>(sm);
        for (int w = 1; w < 4; ++w) r = xyzz_add(r, load_xyzz<F>(sm + X * w));
        store_xyzz(segsum + (uint64_t)X * blockIdx.x, r);
    }
}

// Sum the kRedThreads segment sums in one CTA and write the affine result.
template <class F>
// Sum the per-CTA partials of reduce_seg (kRedThreads / 128 <= 64) and
// write the affine result.
__global__ void __launch_bounds__(64) reduce_final_kernel(const uint8_t* segsum, uint8_t* out) {
    constexpr int X = Lay<F>::XZ;
    constexpr int kParts = kRedThreads / 128;
    __shared__ __align__(16) uint8_t sm[2 * sizeof(XYZZ<F>)];
    XYZZ<F> acc = threadIdx.x < kParts ? load_xyzz<F>(segsum + (uint64_t)X * threadIdx.x)
                                       : XYZZ<F>::inf();
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

template <class F>
int run_t(const uint8_t* table, uint64_t n, const uint8_t* scalars, MsmScratch& sc, uint8_t* out,
          cudaStream_t s) {
    constexpr int X = Lay<F>::XZ;
    const uint64_t cap = (uint64_t)kMsmWindows * n;
    if (sc.cap_entries < cap || !sc.hist) {
        sc.release();
        const uint64_t chunks = (cap + kMsmSeg - 1) / kMsmSeg + kMsmBuckets;
        if (cudaMalloc(&sc.hist, 4 * (kMsmBuckets + 1)) || cudaMalloc(&sc.offs, 4 * (kMsmBuckets + 1)) ||
            cudaMalloc(&sc.coffs, 4 * (kMsmBuckets + 1)) ||
            cudaMalloc(&sc.cursor, 4 * kMsmBuckets) || cudaMalloc(&sc.sorted, 4 * cap) ||
            cudaMalloc(&sc.partials, (size_t)256 * chunks) ||
            cudaMalloc(&sc.buckets, (size_t)256 * kMsmBuckets) ||
            cudaMalloc(&sc.segsum, (size_t)256 * kRedThreads))
            return -1;
        sc.cap_entries = cap;
    }
    cudaMemsetAsync(sc.hist, 0, 4 * (kMsmBuckets + 1), s);
    const unsigned gb = (unsigned)((n + 255) / 256);
    count_kernel<<<gb, 256, 0, s>>>(scalars, n, sc.hist);
    scan_kernel<<<1, 1024, 0, s>>>(sc.hist, sc.offs, sc.cursor, sc.coffs);
    scatter_kernel<<<gb, 256, 0, s>>>(scalars, n, sc.cursor, sc.sorted);
    const uint64_t chunks = (cap + kMsmSeg - 1) / kMsmSeg + kMsmBuckets;  // upper bound
    accumulate_kernel<F><<<(unsigned)((chunks + 127) / 128), 128, 0, s>>>(
        table, sc.sorted, sc.offs, sc.coffs, sc.partials);
    bucket_sum_kernel<F><<<kMsmBuckets / 128, 128, 0, s>>>(sc.coffs, sc.partials, sc.buckets);
    reduce_seg_kernel<F><<<kRedThreads / 128, 128, 0, s>>>(sc.buckets, sc.segsum);
    static_assert(kRedThreads / 128 <= 64, "reduce_final holds one partial per thread");
    reduce_final_kernel<F><<<1, 64, 0, s>>>(sc.segsum, out);
    (void)X;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace

void MsmScratch::release() {
    void* ps[] = {hist, offs, coffs, cursor, sorted, partials, buckets, segsum};
    coffs = nullptr;
    for (void* p : ps)
        if (p) cudaFree(p);
    hist = offs = cursor = sorted = nullptr;
    partials = buckets = segsum = nullptr;
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

void launch_points_convert(int group, uint8_t* pts, uint64_t n, int to_mont, cudaStream_t s) {
    launch_fq_convert(pts, n * 2 * group, to_mont, s);
}

void launch_fq_convert(uint8_t* elems, uint64_t n, int to_mont, cudaStream_t s) {
    if (n) points_convert_kernel<<<(n + 255) / 256, 256, 0, s>>>(elems, n, to_mont);
}

}  // namespace bn
}  // namespace ace_gpu
