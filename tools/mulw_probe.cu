// Multiplier probe (tools only): the current CIOS Montgomery product
// (mad.lo.cc / madc.hi.cc chains -> IMAD + IMAD.HI + IADD3.X) against
// variants built on mul.wide.u32 / mad.wide.u32 (IMAD.WIDE.U32: one
// instruction per 32x32->64 half-product pair), for BN254 Fq.
// Checks every variant bit-exact against the current product on random
// inputs, then measures products/s with 4 independent chains per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2603_10242_b200/csrc tools/mulw_probe.cu -o /tmp/mulw_probe
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include "bn254.cuh"
#include "f64mul.cuh"

using namespace ace_gpu::bn;

namespace {

__device__ __forceinline__ void wide(uint32_t a, uint32_t b, uint32_t& lo, uint32_t& hi) {
    uint64_t p;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a), "r"(b));
    lo = (uint32_t)p;
    hi = (uint32_t)(p >> 32);
}
__device__ __forceinline__ void wide_add(uint32_t a, uint32_t b, uint32_t c, uint32_t& lo,
                                         uint32_t& hi) {
    uint64_t p;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(p) : "r"(a), "r"(b), "l"((uint64_t)c));
    lo = (uint32_t)p;
    hi = (uint32_t)(p >> 32);
}

// t[0..8] += x[0..7] (columns 0..7, carry into t8)
__device__ __forceinline__ void acc_lo(uint32_t t[9], const uint32_t x[8]) {
    asm("add.cc.u32  %0, %0, %9;\n\t"
        "addc.cc.u32 %1, %1, %10;\n\t"
        "addc.cc.u32 %2, %2, %11;\n\t"
        "addc.cc.u32 %3, %3, %12;\n\t"
        "addc.cc.u32 %4, %4, %13;\n\t"
        "addc.cc.u32 %5, %5, %14;\n\t"
        "addc.cc.u32 %6, %6, %15;\n\t"
        "addc.cc.u32 %7, %7, %16;\n\t"
        "addc.u32    %8, %8, 0;"
        : "+r"(t[0]), "+r"(t[1]), "+r"(t[2]), "+r"(t[3]), "+r"(t[4]), "+r"(t[5]), "+r"(t[6]),
          "+r"(t[7]), "+r"(t[8])
        : "r"(x[0]), "r"(x[1]), "r"(x[2]), "r"(x[3]), "r"(x[4]), "r"(x[5]), "r"(x[6]),
          "r"(x[7]));
}
// t[1..8] += x[0..7]
__device__ __forceinline__ void acc_hi(uint32_t t[9], const uint32_t x[8]) {
    asm("add.cc.u32  %0, %0, %8;\n\t"
        "addc.cc.u32 %1, %1, %9;\n\t"
        "addc.cc.u32 %2, %2, %10;\n\t"
        "addc.cc.u32 %3, %3, %11;\n\t"
        "addc.cc.u32 %4, %4, %12;\n\t"
        "addc.cc.u32 %5, %5, %13;\n\t"
        "addc.cc.u32 %6, %6, %14;\n\t"
        "addc.u32    %7, %7, %15;"
        : "+r"(t[1]), "+r"(t[2]), "+r"(t[3]), "+r"(t[4]), "+r"(t[5]), "+r"(t[6]), "+r"(t[7]),
          "+r"(t[8])
        : "r"(x[0]), "r"(x[1]), "r"(x[2]), "r"(x[3]), "r"(x[4]), "r"(x[5]), "r"(x[6]),
          "r"(x[7]));
}

// W1: CIOS with mul.wide (no addend); per row two add chains for the
// product and two for the reduction.
template <class C>
__device__ __forceinline__ Fp<C> mul_w1(const Fp<C>& a, const Fp<C>& b) {
    uint32_t t[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        uint32_t lo[8], hi[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) wide(a.v[j], b.v[i], lo[j], hi[j]);
        acc_lo(t, lo);
        acc_hi(t, hi);
        const uint32_t m = t[0] * C::N0;
#pragma unroll
        for (int j = 0; j < 8; ++j) wide(m, mod_limb<C>(j), lo[j], hi[j]);
        acc_lo(t, lo);
        acc_hi(t, hi);
#pragma unroll
        for (int j = 0; j < 8; ++j) t[j] = t[j + 1];
        t[8] = 0;
    }
    Fp<C> r;
    final_sub<C>(t, r.v);
    return r;
}

// W2: CIOS with mad.wide (t_j folded in as the addend): p_j = a_j b_i + t_j
// fits 64 bits; new t_j = lo(p_j) + hi(p_{j-1}) as one add chain.
template <class C>
__device__ __forceinline__ void row_w2(uint32_t t[9], const uint32_t a[8], uint32_t bi) {
    uint32_t lo[8], hi[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) wide_add(a[j], bi, t[j], lo[j], hi[j]);
    // t0 = lo0; t_j = lo_j + hi_{j-1}; t8 += hi7
    t[0] = lo[0];
    asm("add.cc.u32  %0, %8, %15;\n\t"
        "addc.cc.u32 %1, %9, %16;\n\t"
        "addc.cc.u32 %2, %10, %17;\n\t"
        "addc.cc.u32 %3, %11, %18;\n\t"
        "addc.cc.u32 %4, %12, %19;\n\t"
        "addc.cc.u32 %5, %13, %20;\n\t"
        "addc.cc.u32 %6, %14, %21;\n\t"
        "addc.u32    %7, %7, %22;"
        : "=r"(t[1]), "=r"(t[2]), "=r"(t[3]), "=r"(t[4]), "=r"(t[5]), "=r"(t[6]), "=r"(t[7]),
          "+r"(t[8])
        : "r"(lo[1]), "r"(lo[2]), "r"(lo[3]), "r"(lo[4]), "r"(lo[5]), "r"(lo[6]), "r"(lo[7]),
          "r"(hi[0]), "r"(hi[1]), "r"(hi[2]), "r"(hi[3]), "r"(hi[4]), "r"(hi[5]), "r"(hi[6]),
          "r"(hi[7]));
}
template <class C>
__device__ __forceinline__ Fp<C> mul_w2(const Fp<C>& a, const Fp<C>& b) {
    uint32_t t[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t M[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) M[j] = mod_limb<C>(j);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        row_w2<C>(t, a.v, b.v[i]);
        const uint32_t m = t[0] * C::N0;
        row_w2<C>(t, M, m);
#pragma unroll
        for (int j = 0; j < 8; ++j) t[j] = t[j + 1];
        t[8] = 0;
    }
    Fp<C> r;
    final_sub<C>(t, r.v);
    return r;
}

// W3: SOS — full 512-bit product by rows of mad.wide (operand scanning,
// carry word per row), then 8 reduction rows the same way.
template <class C>
__device__ __forceinline__ Fp<C> mul_w3(const Fp<C>& a, const Fp<C>& b) {
    uint32_t w[17];
#pragma unroll
    for (int k = 0; k < 17; ++k) w[k] = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        uint32_t c = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            uint64_t p;
            asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(p) : "r"(a.v[j]), "r"(b.v[i]),
                "l"((uint64_t)w[i + j]));
            asm("add.u64 %0, %0, %1;" : "+l"(p) : "l"((uint64_t)c));
            w[i + j] = (uint32_t)p;
            c = (uint32_t)(p >> 32);
        }
        w[i + 8] = c;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t m = w[i] * C::N0;
        uint32_t c = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            uint64_t p;
            asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(p) : "r"(m), "r"(mod_limb<C>(j)),
                "l"((uint64_t)w[i + j]));
            asm("add.u64 %0, %0, %1;" : "+l"(p) : "l"((uint64_t)c));
            w[i + j] = (uint32_t)p;
            c = (uint32_t)(p >> 32);
        }
        // propagate c into w[i+8..16]
        asm("add.cc.u32 %0, %0, %1;" : "+r"(w[i + 8]) : "r"(c));
#pragma unroll
        for (int k = i + 9; k < 17; ++k) asm("addc.cc.u32 %0, %0, 0;" : "+r"(w[k]));
        asm("addc.u32 %0, 0, 0;" : "=r"(c));  // unused (w < 2^513 impossible)
    }
    uint32_t t[9] = {w[8], w[9], w[10], w[11], w[12], w[13], w[14], w[15], w[16]};
    Fp<C> r;
    final_sub<C>(t, r.v);
    return r;
}

template <int V>
__device__ __forceinline__ Fq mulv(const Fq& a, const Fq& b) {
    if (V == 0) return mul(a, b);
    if (V == 1) return mul_w1(a, b);
    if (V == 2) return mul_w2(a, b);
    if (V == 4) return f64m::mul_f64(a, b);
    return mul_w3(a, b);
}

template <int V>
__global__ void check_kernel(const Fq* a, const Fq* b, uint32_t n, uint32_t* bad) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Fq x = mulv<0>(a[i], b[i]), y = mulv<V>(a[i], b[i]);
    // chain a few to exercise non-trivial inputs
    for (int k = 0; k < 4; ++k) {
        x = mulv<0>(x, b[i]);
        y = mulv<V>(y, b[i]);
    }
    if (!(x == y)) atomicAdd(bad, 1u);
}

template <int V>
__global__ void rate_kernel(uint32_t* sink, uint32_t iters) {
    Fq x[4], y = Fq::one();
    y.v[0] ^= blockIdx.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        x[k] = Fq::one();
        x[k].v[1] ^= threadIdx.x + k;
    }
    for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 4; ++k) x[k] = mulv<V>(x[k], y);
    }
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) acc ^= x[k].v[0];
    if (acc == 0x1234567u) sink[0] = acc;
}

template <int V>
void run(const Fq* a, const Fq* b, uint32_t n, uint32_t* bad, uint32_t* sink, int sms) {
    cudaMemset(bad, 0, 4);
    check_kernel<V><<<(n + 255) / 256, 256>>>(a, b, n, bad);
    uint32_t hb = 0;
    cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
    for (int threads : {128, 256}) {
        for (int per_sm : {2, 4, 8}) {
            const int blocks = sms * per_sm;
            const uint32_t iters = 512;
            rate_kernel<V><<<blocks, threads>>>(sink, 8);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            rate_kernel<V><<<blocks, threads>>>(sink, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("V%d threads=%d ctas/sm=%d: %.2f G mul/s  (mismatches %u / %u)  %s\n", V, threads,
                   per_sm, double(blocks) * threads * iters * 4 / (ms * 1e-3) / 1e9, hb, n,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
}

}  // namespace

int main2();
int main(int argc, char**) {
    if (argc > 1) return main2();
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint32_t n = 1 << 16;
    uint32_t* h = (uint32_t*)malloc(2ull * n * 32);
    uint64_t s = 0x9E3779B97F4A7C15ull;
    for (uint64_t i = 0; i < 2ull * n * 8; ++i) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        h[i] = (uint32_t)s;
    }
    for (uint64_t i = 0; i < 2ull * n; ++i) h[i * 8 + 7] &= 0x1fffffffu;  // < p
    Fq *a, *b;
    uint32_t *bad, *sink;
    cudaMalloc(&a, n * 32);
    cudaMalloc(&b, n * 32);
    cudaMalloc(&bad, 4);
    cudaMalloc(&sink, 4);
    cudaMemcpy(a, h, n * 32, cudaMemcpyHostToDevice);
    cudaMemcpy(b, h + n * 8, n * 32, cudaMemcpyHostToDevice);
    run<0>(a, b, n, bad, sink, sms);
    run<1>(a, b, n, bad, sink, sms);
    run<2>(a, b, n, bad, sink, sms);
    run<3>(a, b, n, bad, sink, sms);
    run<4>(a, b, n, bad, sink, sms);
    return 0;
}

// ---- call-shape probe: the MSM calls its products out of line, one at a time
namespace callshape {
__device__ __noinline__ Fq mul1_call(const Fq a, const Fq b) { return f64m::mul_f64(a, b); }
struct Fq2v { Fq a, b; };
__device__ __noinline__ Fq2v mul2_call(const Fq a, const Fq b, const Fq c, const Fq d) {
    return {f64m::mul_f64(a, b), f64m::mul_f64(c, d)};
}
__device__ __noinline__ Fq cios1_call(const Fq a, const Fq b) { return mul(a, b); }

template <int MODE>  // 0: f64 1 chain/call, 1: f64 2 chains/call, 2: cios 1 chain/call
__global__ void __launch_bounds__(128) k(uint32_t* sink, uint32_t iters) {
    Fq x = Fq::one(), z = Fq::one(), y = Fq::one();
    y.v[0] ^= blockIdx.x;
    x.v[1] ^= threadIdx.x;
    z.v[2] ^= threadIdx.x;
    for (uint32_t it = 0; it < iters; ++it) {
        if (MODE == 0) { x = mul1_call(x, y); z = mul1_call(z, y); }
        if (MODE == 1) { Fq2v r = mul2_call(x, y, z, y); x = r.a; z = r.b; }
        if (MODE == 2) { x = cios1_call(x, y); z = cios1_call(z, y); }
    }
    if ((x.v[0] ^ z.v[0]) == 0x1234567u) sink[0] = 1;
}
template <int MODE>
void run(uint32_t* sink, int sms) {
    for (int per_sm : {2, 4, 8, 16}) {
        const int blocks = sms * per_sm;
        const uint32_t iters = 256;
        k<MODE><<<blocks, 128>>>(sink, 4);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k<MODE><<<blocks, 128>>>(sink, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("callshape %d ctas/sm=%2d (128 thr): %.2f G mul/s\n", MODE, per_sm,
               double(blocks) * 128 * iters * 2 / (ms * 1e-3) / 1e9);
    }
}
}  // namespace callshape

int main2() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* sink;
    cudaMalloc(&sink, 4);
    callshape::run<0>(sink, sms);
    callshape::run<1>(sink, sms);
    callshape::run<2>(sink, sms);
    return 0;
}
