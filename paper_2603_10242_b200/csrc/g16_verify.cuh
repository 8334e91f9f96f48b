// Batched Groth16 verification (g16_verify.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "msm.cuh"

namespace ace_gpu {
namespace bn {

struct G16VerifyKey {
    uint32_t T = 0;                        // public inputs besides ONE
    const uint8_t* ic_table = nullptr;     // msm_prepare'd IC_0..IC_T (G1)
    const uint8_t* alpha1_mont = nullptr;  // alpha G1, affine Montgomery (64 B)
    const uint8_t* g2_std = nullptr;       // beta | gamma | delta G2, oracle encoding (3 x 128 B)
    const uint8_t* vk_digest = nullptr;    // SHA-256 of the acegpu_g16_vk export (32 B)
};

size_t g16_verify_scratch_bytes(uint32_t n, uint32_t T);
// proofs: n x 256 B EIP-197 (A | B | C, big-endian coordinates, B as
// x.c1 x.c0 y.c1 y.c0); pubs: n x T x 32 B little-endian public inputs
// (reduced mod r here). *d_ok (device) = 1 iff every proof verifies.
// seed_out (device, optional): the 32-B Fiat-Shamir seed of the weights.
int g16_verify_batch(const G16VerifyKey& vk, const uint8_t* proofs, const uint8_t* pubs,
                     uint32_t n, uint8_t* scratch, MsmScratch& msm, int* d_ok, cudaStream_t s,
                     uint8_t* seed_out = nullptr);
// SHA-256 of a device buffer (one thread; the verifying key's digest at setup)
void g16_vk_digest(const uint8_t* vk_bytes, uint32_t len, uint8_t* out, cudaStream_t s);
void combine_ok(int* ok, const int* bad, cudaStream_t s);

}  // namespace bn
}  // namespace ace_gpu
