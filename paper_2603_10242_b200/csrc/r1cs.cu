// General R1CS kernels (r1cs.cuh): the prover's A z / B z / C z row
// evaluations (SpMV, one thread per row: R1CS rows hold a handful of
// entries) and the setup's column sums A^T L(tau) (one warp per column).
// Unit coefficients (the common case) skip the Montgomery product.
#include <cuda_runtime.h>

#include "bn254.cuh"
#include "r1cs.cuh"

namespace ace_gpu {
namespace bn {
namespace {

__device__ __forceinline__ Fr ld(const uint8_t* p) { return load<FrCfg>(p); }
__device__ __forceinline__ void st(uint8_t* p, const Fr& x) { store<FrCfg>(p, x); }

__device__ __forceinline__ Fr shfl_down(const Fr& a, int d) {
    Fr r;
#pragma unroll
    for (int i = 0; i < 8; ++i) r.v[i] = __shfl_down_sync(0xffffffffu, a.v[i], d);
    return r;
}

__global__ void spmv_kernel(const uint64_t* rowptr, const uint32_t* col, const uint8_t* val,
                            const uint8_t* zm, uint64_t rows, uint64_t pad, uint8_t* out) {
    const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j >= pad) return;
    Fr acc = Fr::zero();
    if (j < rows && rowptr[j + 1] - rowptr[j] > kR1csLongRow) return;  // long_rows_kernel
    if (j < rows) {
        const Fr one = Fr::one();
        for (uint64_t k = rowptr[j], e = rowptr[j + 1]; k < e; ++k) {
            const Fr v = ld(val + 32 * k), x = ld(zm + 32ull * col[k]);
            acc = add(acc, v == one ? x : mul(v, x));
        }
    }
    st(out + 32 * j, acc);
}

// one warp per long row: lanes stride over the entries, then a shuffle tree
__global__ void long_rows_kernel(const uint64_t* rowptr, const uint32_t* col, const uint8_t* val,
                                 const uint32_t* long_rows, uint64_t n_long, const uint8_t* zm,
                                 uint8_t* out) {
    const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= n_long) return;  // whole warps exit together
    const uint32_t j = long_rows[w];
    const Fr one = Fr::one();
    Fr acc = Fr::zero();
    for (uint64_t k = rowptr[j] + lane, e = rowptr[j + 1]; k < e; k += 32) {
        const Fr v = ld(val + 32 * k), x = ld(zm + 32ull * col[k]);
        acc = add(acc, v == one ? x : mul(v, x));
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) acc = add(acc, shfl_down(acc, d));
    if (lane == 0) st(out + 32ull * j, acc);
}

__global__ void colsum_kernel(const uint64_t* colptr, const uint32_t* crow, const uint8_t* cval,
                              const uint8_t* L, uint64_t vars, uint8_t* out) {
    const uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= vars) return;  // whole warps exit together
    const Fr one = Fr::one();
    Fr acc = Fr::zero();
    for (uint64_t k = colptr[i] + lane, e = colptr[i + 1]; k < e; k += 32) {
        const Fr v = ld(cval + 32 * k), l = ld(L + 32ull * crow[k]);
        acc = add(acc, v == one ? l : mul(v, l));
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) acc = add(acc, shfl_down(acc, d));
    if (lane == 0) st(out + 32 * i, acc);
}

__global__ void query_kernel(const uint8_t* c, const uint8_t* u, const uint8_t* v,
                             const uint8_t* w, uint64_t vars, uint64_t n_pub, uint8_t* su,
                             uint8_t* sv, uint8_t* sl, uint8_t* ic) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= vars) return;
    const Fr alpha = ld(c + 32), beta = ld(c + 64), gamma = ld(c + 96), dinv = ld(c + 32 * 8);
    const Fr ui = ld(u + 32 * i), vi = ld(v + 32 * i), wi = ld(w + 32 * i);
    st(su + 32 * i, from_mont(ui));
    st(sv + 32 * i, from_mont(vi));
    const Fr t = add(add(mul(beta, ui), mul(alpha, vi)), wi);
    if (i > n_pub) st(sl + 32 * (i - 1 - n_pub), from_mont(mul(t, dinv)));
    else st(ic + 32 * i, from_mont(mul(t, inv_fast(gamma))));
}

inline unsigned grid(uint64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

void r1cs_spmv(const R1csMat& M, const uint8_t* zm, uint64_t rows, uint64_t pad, uint8_t* out,
               cudaStream_t s) {
    if (pad) spmv_kernel<<<grid(pad, 128), 128, 0, s>>>(M.rowptr, M.col, M.val, zm, rows, pad, out);
    if (M.n_long)
        long_rows_kernel<<<grid(32 * M.n_long, 128), 128, 0, s>>>(M.rowptr, M.col, M.val,
                                                                 M.long_rows, M.n_long, zm, out);
}

void r1cs_colsum(const R1csMat& M, const uint8_t* L, uint64_t vars, uint8_t* out,
                 cudaStream_t s) {
    if (vars) colsum_kernel<<<grid(32 * vars, 256), 256, 0, s>>>(M.colptr, M.crow, M.cval, L, vars, out);
}

void r1cs_query_scalars(const uint8_t* consts, const uint8_t* u, const uint8_t* v,
                        const uint8_t* w, uint64_t vars, uint64_t n_pub, uint8_t* su, uint8_t* sv,
                        uint8_t* sl, uint8_t* ic, cudaStream_t s) {
    if (vars) query_kernel<<<grid(vars, 128), 128, 0, s>>>(consts, u, v, w, vars, n_pub, su, sv, sl, ic);
}

}  // namespace bn
}  // namespace ace_gpu
