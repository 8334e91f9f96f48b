// Integer-pipe microbenchmark (tools only): IMAD vs IMAD.WIDE vs IMAD.HI vs
// IADD3 throughput on sm_100a, to size the Fq multiplier design.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(uint32_t* sink, uint32_t iters) {
    uint32_t a[8];
    uint64_t w[8];
    double dd[8];
    for (int j = 0; j < 8; ++j) { a[j] = threadIdx.x * 7 + j; w[j] = a[j]; dd[j] = a[j]; }
    const uint32_t m = blockIdx.x | 0x9E3779B1u;
    for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (MODE == 0) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(m), "r"(it));
                if (MODE == 1) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[j]) : "r"((uint32_t)(w[j] >> 7)), "r"(m));
                if (MODE == 2) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(m), "r"(it));
                if (MODE == 3) asm volatile("add.u32 %0, %0, %1;" : "+r"(a[j]) : "r"(m));
                if (MODE == 5) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(dd[j]) : "d"(1.0000001), "d"(1e-9));
                if (MODE == 6) {  // even warps DFMA, odd warps IMAD
                    if ((threadIdx.x >> 5) & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(m), "r"(it));
                    else asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(dd[j]) : "d"(1.0000001), "d"(1e-9));
                }
                if (MODE == 7) {  // even warps DFMA, odd warps IMAD.HI
                    if ((threadIdx.x >> 5) & 1) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(m), "r"(it));
                    else asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(dd[j]) : "d"(1.0000001), "d"(1e-9));
                }
                if (MODE == 8) {  // even warps FFMA, odd warps IMAD.HI
                    if ((threadIdx.x >> 5) & 1) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(m), "r"(it));
                    else asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(0x3f800001u), "r"(0x3000000u));
                }
                if (MODE == 9) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(0x3f800001u), "r"(0x3000000u));
                if (MODE == 4) asm volatile("{.reg .u32 t; mad.lo.cc.u32 %0, %0, %1, %2; madc.hi.u32 t, %0, %1, 0; add.u32 %0, %0, t;}" : "+r"(a[j]) : "r"(m), "r"(it));
            }
        }
    }
    uint64_t x = 0;
    for (int j = 0; j < 8; ++j) x ^= a[j] ^ w[j] ^ (uint64_t)dd[j];
    if (x == 0x1234567ull) sink[0] = (uint32_t)x;
}

template <int MODE>
double run(uint32_t* sink) {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256;
    const uint32_t iters = 2048;
    k<MODE><<<blocks, threads>>>(sink, 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE><<<blocks, threads>>>(sink, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return double(blocks) * threads * iters * 16 * 8 / (ms * 1e-3);
}

int main() {
    uint32_t* sink;
    cudaMalloc(&sink, 16);
    printf("mad.lo.u32   %.3e /s\n", run<0>(sink));
    printf("mad.wide.u32 %.3e /s\n", run<1>(sink));
    printf("mad.hi.u32   %.3e /s\n", run<2>(sink));
    printf("add.u32      %.3e /s\n", run<3>(sink));
    printf("lo.cc+hi chain(3 ops) %.3e /s\n", run<4>(sink));
    printf("fma.rn.f64   %.3e /s\n", run<5>(sink));
    printf("DFMA|IMAD warps %.3e /s (sum of both)\n", run<6>(sink));
    printf("DFMA|IMAD.HI warps %.3e /s (sum of both)\n", run<7>(sink));
    printf("FFMA|IMAD.HI warps %.3e /s (sum of both)\n", run<8>(sink));
    printf("fma.rn.f32   %.3e /s\n", run<9>(sink));
    return 0;
}
