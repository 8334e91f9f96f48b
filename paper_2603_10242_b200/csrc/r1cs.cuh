// General rank-1 constraint systems on the GPU (north-star "witness /
// constraint evaluation", r1cs.cu): CSR matrices A, B, C over Fr for the
// prover's row evaluations a = A z, b = B z, c = C z, and their CSC
// transposes for the Groth16 setup's query polynomials u = A^T L(tau),
// v = B^T L(tau), w = C^T L(tau).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace ace_gpu {
namespace bn {

// One sparse matrix, device-resident. Values are Fr in Montgomery form.
struct R1csMat {
    uint64_t nnz = 0;
    uint64_t* rowptr = nullptr;  // rows + 1
    uint32_t* col = nullptr;     // nnz
    uint8_t* val = nullptr;      // nnz x 32
    uint32_t* long_rows = nullptr;  // rows with more than kR1csLongRow entries (a warp each)
    uint64_t n_long = 0;
    uint64_t* colptr = nullptr;  // vars + 1 (CSC transpose, setup only)
    uint32_t* crow = nullptr;    // nnz
    uint8_t* cval = nullptr;     // nnz x 32
};

// Rows longer than this (the packing / 32-bit addition rows of a SHA-256
// circuit hold ~200 entries) are evaluated by a warp each.
constexpr uint64_t kR1csLongRow = 16;

// a[j] = sum_k val[k] zm[col[k]] over row j's entries (zm, out: Montgomery),
// rows [0, rows); rows < pad are written as zero up to pad.
void r1cs_spmv(const R1csMat& M, const uint8_t* zm, uint64_t rows, uint64_t pad, uint8_t* out,
               cudaStream_t s);
// out[i] = sum over column i's entries of val * L[row] (Montgomery), i < vars.
// One warp per column (a column such as ONE may hold a million entries).
void r1cs_colsum(const R1csMat& M, const uint8_t* L, uint64_t vars, uint8_t* out,
                 cudaStream_t s);
// Groth16 query scalars from u, v, w (Montgomery, vars entries), standard form
// out: su, sv (vars), sl (private vars i > n_pub: (beta u + alpha v + w)/delta)
// and ic (public vars i <= n_pub: (beta u + alpha v + w)/gamma).
void r1cs_query_scalars(const uint8_t* consts, const uint8_t* u, const uint8_t* v,
                        const uint8_t* w, uint64_t vars, uint64_t n_pub, uint8_t* su, uint8_t* sv,
                        uint8_t* sl, uint8_t* ic, cudaStream_t s);

}  // namespace bn
}  // namespace ace_gpu
