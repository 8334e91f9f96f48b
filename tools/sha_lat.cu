// Single-warp SHA-256 compression LATENCY probe (the narrow tree levels are a
// serial chain of 11 compressions per level). Variants:
//   full     sha256_compress (unrolled, schedule inline)
//   compact  sha256_compress_c
//   rnd_smem sha256_rounds, W+K from shared memory (the level_kernel<8> path)
//   rndc_smem sha256_rounds_c, W+K from shared memory
//   rnd_fast reassociated rounds (d+h+W+K formed 3 rounds ahead), W+K from smem
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2603_10242_b200/csrc
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "sha256.cuh"

using namespace ace_gpu;

// Reassociated rounds: at round t, h_t = e_{t-3} and d_t = a_{t-3} are known
// three rounds early, so hk = h + WK and dhk = d + h + WK are off the chain;
// e' = dhk + S1 + Ch (one IADD3 after Sigma1), a' = (hk + S1 + Ch) + S0 + Maj.
template <class WK>
__device__ __forceinline__ void sha256_rounds_fast(uint32_t s[8], WK wk) {
    uint32_t a = s[0], b = s[1], c = s[2], d = s[3], e = s[4], f = s[5], g = s[6], h = s[7];
#pragma unroll
    for (int i = 0; i < 64; ++i) {
        const uint32_t hk = h + wk(i);
        const uint32_t dhk = d + hk;
        const uint32_t S1 = rotr32(e, 6) ^ rotr32(e, 11) ^ rotr32(e, 25);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t S0 = rotr32(a, 2) ^ rotr32(a, 13) ^ rotr32(a, 22);
        const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        const uint32_t ne = dhk + S1 + ch;
        const uint32_t na = hk + S1 + ch + S0 + mj;
        h = g; g = f; f = e; e = ne; d = c; c = b; b = a; a = na;
    }
    s[0] += a; s[1] += b; s[2] += c; s[3] += d;
    s[4] += e; s[5] += f; s[6] += g; s[7] += h;
}

// Pipe-balanced compression: part of the additions as IMAD (x * kOne + y)
// with a constant-bank multiplier ptxas cannot fold, so they issue on the FMA
// pipe instead of the (saturated) integer ALU pipe.
__device__ __constant__ uint32_t kOne = 1;
__device__ __forceinline__ uint32_t madd(uint32_t x, uint32_t y) { return x * kOne + y; }

template <int MODE>
__device__ __forceinline__ void sha256_compress_bal(uint32_t s[8], uint32_t w[16]) {
    constexpr uint32_t K[64] = ACE_K256;
    uint32_t a = s[0], b = s[1], c = s[2], d = s[3], e = s[4], f = s[5], g = s[6], h = s[7];
#pragma unroll
    for (int i = 0; i < 64; ++i) {
        uint32_t wi;
        if (i < 16) {
            wi = w[i];
        } else {
            uint32_t w15 = w[(i - 15) & 15], w2 = w[(i - 2) & 15];
            uint32_t s0 = rotr32(w15, 7) ^ rotr32(w15, 18) ^ (w15 >> 3);
            uint32_t s1 = rotr32(w2, 17) ^ rotr32(w2, 19) ^ (w2 >> 10);
            if (MODE & 1) wi = w[i & 15] = madd(w[i & 15] + s0, w[(i - 7) & 15] + s1);
            else wi = w[i & 15] = w[i & 15] + s0 + w[(i - 7) & 15] + s1;
        }
        uint32_t S1 = rotr32(e, 6) ^ rotr32(e, 11) ^ rotr32(e, 25);
        uint32_t ch = (e & f) ^ (~e & g);
        uint32_t S0 = rotr32(a, 2) ^ rotr32(a, 13) ^ rotr32(a, 22);
        uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        uint32_t hk = (MODE & 2) ? madd(h, K[i] + wi) : h + K[i] + wi;
        uint32_t t1 = hk + S1 + ch;
        h = g;
        g = f;
        f = e;
        e = (MODE & 4) ? madd(d, t1) : d + t1;
        d = c;
        c = b;
        b = a;
        a = (MODE & 8) ? madd(t1, S0 + mj) : t1 + S0 + mj;
    }
    s[0] += a; s[1] += b; s[2] += c; s[3] += d;
    s[4] += e; s[5] += f; s[6] += g; s[7] += h;
}

template <int MODE>
__global__ void __launch_bounds__(128) thr_kernel(uint32_t* sink, uint32_t iters) {
    uint32_t s[8];
    sha256_init(s);
    s[0] ^= blockIdx.x * blockDim.x + threadIdx.x;
    for (uint32_t it = 0; it < iters; ++it) {
        uint32_t w[16];
#pragma unroll
        for (int k = 0; k < 8; ++k) { w[k] = s[k]; w[k + 8] = s[k] ^ it; }
        if (MODE < 0) sha256_compress(s, w);
        else sha256_compress_bal<MODE < 0 ? 0 : MODE>(s, w);
    }
    uint32_t x = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) x ^= s[k];
    if (x == 0x12345678u) sink[0] = x;
}

template <int MODE>
void thr(const char* name, uint32_t* sink) {
    const uint32_t iters = 200, grid = 148 * 8 * 4;
    thr_kernel<MODE><<<grid, 128>>>(sink, iters);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    thr_kernel<MODE><<<grid, 128>>>(sink, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("thr %-12s %.2f G compressions/s\n", name, double(grid) * 128 * iters / (ms * 1e-3) / 1e9);
}

template <int V>
__global__ void lat_kernel(uint32_t iters, unsigned long long* out, uint32_t* sink) {
    __shared__ uint32_t wk[64];
    if (threadIdx.x < 64) wk[threadIdx.x] = 0x9e3779b9u * (threadIdx.x + 1);
    for (int i = threadIdx.x + 32; i < 64; i += 32) wk[i] = 0x9e3779b9u * (i + 1);
    __syncthreads();
    uint32_t s[8];
    sha256_init(s);
    s[0] ^= threadIdx.x;
    const unsigned long long t0 = clock64();
    for (uint32_t it = 0; it < iters; ++it) {
        if constexpr (V == 0 || V == 1) {
            uint32_t w[16];
#pragma unroll
            for (int k = 0; k < 8; ++k) { w[k] = s[k]; w[k + 8] = s[k] ^ it; }
            if constexpr (V == 0) sha256_compress(s, w);
            else sha256_compress_c(s, w);
        } else if constexpr (V == 2) {
            sha256_rounds(s, [&](int i) { return wk[i]; });
        } else if constexpr (V == 3) {
            sha256_rounds_c(s, [&](int i) { return wk[i]; });
        } else {
            sha256_rounds_fast(s, [&](int i) { return wk[i]; });
        }
    }
    const unsigned long long t1 = clock64();
    uint32_t x = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) x ^= s[k];
    if (x == 0x12345678u) sink[0] = x;
    if (threadIdx.x == 0) out[0] = t1 - t0;
}

template <int V>
void run(const char* name, uint32_t iters, unsigned long long* d_out, uint32_t* sink) {
    lat_kernel<V><<<1, 32>>>(iters, d_out, sink);  // warm (I-cache)
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    lat_kernel<V><<<1, 32>>>(iters, d_out, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long cyc;
    cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
    printf("%-10s %8.1f cycles/compression  %7.3f us/compression (event)\n", name,
           double(cyc) / iters, 1e3 * ms / iters);
}

int main() {
    unsigned long long* d_out;
    uint32_t* sink;
    cudaMalloc(&d_out, 8);
    cudaMalloc(&sink, 4);
    const uint32_t it = 20000;
    run<0>("full", it, d_out, sink);
    run<1>("compact", it, d_out, sink);
    run<2>("rnd_smem", it, d_out, sink);
    run<3>("rndc_smem", it, d_out, sink);
    run<4>("rnd_fast", it, d_out, sink);
    thr<-1>("stock", sink);
    thr<0>("bal0", sink);
    thr<1>("bal_sched", sink);
    thr<2>("bal_hk", sink);
    thr<4>("bal_e", sink);
    thr<8>("bal_a", sink);
    thr<5>("bal_sched_e", sink);
    thr<6>("bal_hk_e", sink);
    thr<7>("bal_s_hk_e", sink);
    thr<15>("bal_all", sink);
    thr<12>("bal_e_a", sink);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
