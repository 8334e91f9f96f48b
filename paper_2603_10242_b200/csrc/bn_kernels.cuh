// Launchers for bn_kernels.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace ace_gpu {
namespace bn {

// field: 0 = Fq, 1 = Fr; op: 0 mul, 1 add, 2 sub, 3 sqr, 4 inv (standard form I/O)
void launch_field_batch(int field, int op, const uint8_t* a, const uint8_t* b, uint64_t n,
                        uint8_t* out, cudaStream_t s);
// out[i] = scalars[i] * base; base and out affine Montgomery; scalars standard
void launch_scalar_muls(int group, const uint8_t* base, const uint8_t* scalars, uint64_t n,
                        uint8_t* out, cudaStream_t s);
// Fixed-base comb for the proving-key setup (every base is s_i * G for one
// generator G): tab[k][j] = (j 2^(8k)) G for k < 32, j < 256 (kCombEntries x
// 64 group bytes; once per generator), then out[i] = sum_k tab[k][byte_k(s_i)]:
// 32 mixed additions + one inversion per point instead of 256 doublings.
constexpr uint64_t kCombEntries = 32 * 256;
void launch_comb_table(int group, const uint8_t* base, uint8_t* scalar_scratch /* 256 KB */,
                       uint8_t* tab, cudaStream_t s);
void launch_comb_muls(int group, const uint8_t* tab, const uint8_t* scalars, uint64_t n,
                      uint8_t* out, cudaStream_t s);
void launch_imad_peak(uint32_t* sink, uint32_t iters, int blocks, int threads, cudaStream_t s);
void launch_mul_rate(int field, uint32_t* sink, uint32_t iters, int blocks, int threads,
                     cudaStream_t s);

}  // namespace bn
}  // namespace ace_gpu
