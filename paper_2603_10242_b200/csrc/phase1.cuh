// Phase 1a kernels (phase1.cu): light admission check and block assembly.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace ace_gpu {

// attest_check_light per tx (codes: 0 Accept, 1 PayloadBinding, 2
// UnknownIdentity, 3 StaleDomain); tx_hashes (n x 32, optional) receives
// SHA-256(payload). reg: n_reg sorted 32-B id commitments.
void launch_light_check(const uint8_t* payloads, const uint64_t* offs, const uint8_t* atts,
                        uint32_t n, const uint8_t* reg, uint64_t n_reg, uint64_t cur,
                        uint64_t window, uint8_t* codes, uint8_t* tx_hashes, cudaStream_t s);

// Scratch bytes for launch_compact over n transactions.
size_t compact_scratch_bytes(uint32_t n);

// Order-preserving compaction of the txs with codes[i] == 0 (codes null: all):
// payloads / offsets / attestations / payload hashes to the out arrays, plus
// the attestation-record hashes (attest Merkle leaves). *d_count / *d_total
// point at the device-resident accepted count and payload byte total.
cudaError_t launch_compact(const uint8_t* payloads, const uint64_t* offs, const uint8_t* atts,
                           uint32_t n, const uint8_t* codes, const uint8_t* tx_hashes,
                           uint8_t* scratch, uint8_t* out_pay, uint64_t* out_offs,
                           uint8_t* out_atts, uint8_t* out_txh, uint8_t* out_ath,
                           uint32_t** d_count, uint64_t** d_total, cudaStream_t s);

// Header = template with tx_count, tx_merkle_root, attest_merkle_root set
// (wire.cpp:74-96 layout); also writes out_offs[count] = total.
void launch_header(const uint8_t* tmpl, const uint32_t* d_count, const uint64_t* d_total,
                   uint64_t* out_offs, const uint8_t* tx_root, const uint8_t* att_root,
                   uint8_t* out, cudaStream_t s);

}  // namespace ace_gpu
