// Probe (tools only): the FP64-domain lazy products (bn254.cuh W10 / redc10)
// against plain Montgomery products: redc10(mul_wide10(a, b)) == mul(a, b),
// Fq2 products / squares / a b - c d through curve.cuh's W10 units vs the
// same through mul(). Prints mismatch counts; bounded loops only.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "curve.cuh"

using namespace ace_gpu::bn;

__global__ void probe_kernel(const Fq* in, uint32_t n, uint32_t* bad) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const Fq a = in[4 * i], b = in[4 * i + 1], c = in[4 * i + 2], d = in[4 * i + 3];
    W10 w;
    mul_wide10(a, b, w);
    if (!(redc10<FqCfg>(w) == mul(a, b))) atomicAdd(&bad[0], 1u);
    const Fq2 x{a, b}, y{c, d};
    const Fq2 p = fmul(x, y);
    const Fq e0 = sub(mul(a, c), mul(b, d)), e1 = add(mul(a, d), mul(b, c));
    if (!(p.c0 == e0 && p.c1 == e1)) atomicAdd(&bad[1], 1u);
    const Fq2 q = fsqr(x);
    const Fq f0 = sub(mul(a, a), mul(b, b)), f1 = add(mul(a, b), mul(a, b));
    if (!(q.c0 == f0 && q.c1 == f1)) atomicAdd(&bad[2], 1u);
    const Fq2 r = fmul_sub(x, y, y, x);  // x y - y x = 0
    if (!(r.c0.is_zero() && r.c1.is_zero())) atomicAdd(&bad[3], 1u);
    const Fq2 t = fmul_sub(x, y, x, x);
    const Fq2 xx = fmul(x, x);
    if (!(t.c0 == sub(p.c0, xx.c0) && t.c1 == sub(p.c1, xx.c1))) atomicAdd(&bad[4], 1u);
}

int main() {
    const uint32_t n = 1 << 16;
    uint32_t* h = (uint32_t*)malloc(4ull * n * 32);
    uint64_t s = 0x9E3779B97F4A7C15ull;
    for (uint64_t i = 0; i < 4ull * n * 8; ++i) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        h[i] = (uint32_t)s;
    }
    for (uint64_t i = 0; i < 4ull * n; ++i) h[i * 8 + 7] &= 0x2fffffffu;  // < p
    // edge values: 0, 1, p - 1
    const uint32_t pm1[8] = {0xd87cfd46u, 0x3c208c16u, 0x6871ca8du, 0x97816a91u,
                             0x8181585du, 0xb85045b6u, 0xe131a029u, 0x30644e72u};
    for (int k = 0; k < 8; ++k) { h[k] = 0; h[8 + k] = pm1[k]; h[16 + k] = pm1[k]; h[24 + k] = k == 0; }
    Fq* d;
    uint32_t* bad;
    cudaMalloc(&d, 4ull * n * 32);
    cudaMalloc(&bad, 64);
    cudaMemset(bad, 0, 64);
    cudaMemcpy(d, h, 4ull * n * 32, cudaMemcpyHostToDevice);
    probe_kernel<<<(n + 127) / 128, 128>>>(d, n, bad);
    uint32_t hb[5];
    cudaError_t e = cudaMemcpy(hb, bad, 20, cudaMemcpyDeviceToHost);
    printf("%s mismatches: redc10 %u, fq2 mul %u, fq2 sqr %u, mul_sub zero %u, mul_sub %u (of %u)\n",
           cudaGetErrorString(e), hb[0], hb[1], hb[2], hb[3], hb[4], n);
    return 0;
}
