// Launchers of pairing.cu (host-visible).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace ace_gpu {
namespace bn {

size_t pairing_scratch_bytes(uint32_t n);
// prod_i e(P_i, Q_i) after the final exponentiation. Inputs in the oracle
// encodings (32-B LE standard form; G1 x|y, G2 x.c0|x.c1|y.c0|y.c1; all-zero
// = infinity). out384 (optional): 12 x 32-B Fq coefficients; is_one
// (optional): 1 iff the product is 1.
void launch_pairing_product(uint32_t n, const uint8_t* g1s, const uint8_t* g2s, uint8_t* scratch,
                            uint8_t* out384, int* is_one, cudaStream_t s);

// The product + final exponentiation half of launch_pairing_product, over n
// Miller-loop values already in scratch (raw Fq12 records).
void launch_pairing_finish(uint32_t n, uint8_t* scratch, uint8_t* out384, int* is_one,
                           cudaStream_t s);

// Fq12 unit op (codes of acegpu_bn_f12_op) on one element (or G1|G2 pair).
void launch_f12_op(int op, const uint8_t* in, uint8_t* out, cudaStream_t s);

}  // namespace bn
}  // namespace ace_gpu
