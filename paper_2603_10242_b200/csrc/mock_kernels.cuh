// Launchers for the mock-Prove kernels (mock_kernels.cu). Internal to
// libacegpu; the public surface is include/acegpu.h.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace ace_gpu {

// Internal proof-node record: 320 B, 16-B aligned.
//   [0,256) proof bytes | [256,288) public_inputs_digest | [288] kind (0 Tx, 1 Agg)
constexpr int kNodeBytes = 320;

struct LeafArgs {
    const uint8_t* payloads;   // concatenated payload bytes (4-B aligned base)
    const uint64_t* offs;      // n+1 offsets into payloads
    const uint8_t* atts;       // n x 104 attestation records (8-B aligned)
    uint32_t n;
    uint8_t* codes;            // n verdicts, or nullptr to skip attestation
    uint8_t* nodes;            // n x 320 leaf proof records, or nullptr (attest-only)
    uint8_t* merkle;           // n x 32 merkle leaf hashes H(0x00|id_com), or nullptr
    const uint8_t* header;     // 256-B header; nullptr = no block hash
    uint8_t* block_hash;       // 32 B out when header != nullptr
    // With codes, the leaf kernel writes the payload verdict (0 / 1); the
    // credential verdict (2) follows in launch_credentials.
};

void launch_leaves(const LeafArgs& a, cudaStream_t s);
// Credential check of verify_attestation_full for every tx with codes[i] == 0
// (sets 2 on mismatch). keytab (launch_keytab for domain keydom) may be null.
// rev_index[i] >= n_revs sets *err (if given) and code 2 without reading.
void launch_credentials(const uint8_t* atts, uint32_t n, const uint8_t* revs,
                        const uint32_t* rev_index, const uint32_t* keytab, const uint8_t* keydom,
                        uint8_t* codes, uint32_t n_revs, int* err, cudaStream_t s);
// Attest-key cache: per REV u, the HMAC ipad/opad midstates of
// derive_attest_key(REV_u, D0), D0 = the 8-B domain at dom8 (16 words per REV).
void launch_keytab(const uint8_t* revs, uint32_t n_revs, const uint8_t* dom8, uint32_t* keytab,
                   cudaStream_t s);

// One tree level for the proof tree (pairs (2i,2i+1), odd node promoted,
// prover.cpp:112-124) and/or the Merkle tree (odd node duplicated,
// wire.cpp:240; `lift` self-pairs a lone node, used for aligned chunk roots).
void launch_level(const uint8_t* nodes_in, uint32_t n_nodes, uint8_t* nodes_out,
                  const uint8_t* merkle_in, uint32_t n_merkle, uint8_t* merkle_out, bool lift,
                  cudaStream_t s);

// Merkle leaf level over plain 32-B leaves (wire.cpp:229-238).
void launch_merkle_leaves(const uint8_t* leaves, uint32_t n, uint8_t* out, cudaStream_t s);

// Finalise: root node + merkle root + block hash -> 289-B proof and 328-B FC.
// prove_empty proves the empty block instead of using root_node
// (prover.cpp:134-139); merkle_root == nullptr means no leaves (0^32).
void launch_finalize(const uint8_t* root_node, const uint8_t* merkle_root, const uint8_t* header,
                     const uint8_t* block_hash, bool prove_empty, uint8_t* out_proof289,
                     uint8_t* out_fc328, cudaStream_t s);

// Pack / unpack 289-B external proofs <-> 320-B node records.
void launch_pack_nodes(const uint8_t* nodes, uint32_t n, uint8_t* out289, cudaStream_t s);
void launch_unpack_nodes(const uint8_t* in289, uint32_t n, uint8_t* nodes, cudaStream_t s);

// Batched primitives behind the single-call API.
void launch_sha256_varlen(const uint8_t* data, const uint64_t* offs, uint32_t n, uint8_t* out,
                          cudaStream_t s);
void launch_sha256_strided(const uint8_t* base, uint64_t stride, uint32_t len, uint32_t n,
                           uint8_t* out, cudaStream_t s);
void launch_prove_public_inputs(const uint8_t* pubs160, uint32_t n, uint8_t* nodes,
                                cudaStream_t s);
void launch_verify_mock(const uint8_t* nodes, uint32_t n, uint8_t* ok, cudaStream_t s);
void launch_aggregate_pairs(const uint8_t* a_nodes, const uint8_t* b_nodes, uint32_t n,
                            uint8_t* out_nodes, cudaStream_t s);

// Attestation / witness batch kernels.
void launch_attest_generate(const uint8_t* payloads, const uint64_t* offs, uint32_t n,
                            const uint8_t* revs, const uint32_t* rev_index, const uint8_t* doms8,
                            const uint8_t* id_coms, uint8_t* out104, cudaStream_t s);
void launch_derive_attest_keys(const uint8_t* revs, const uint8_t* doms8, uint32_t n,
                               uint8_t* out32, cudaStream_t s);
void launch_witness_check(const uint8_t* witnesses, const uint32_t* wlens, const uint8_t* atts,
                          uint32_t n, uint8_t* ok, cudaStream_t s);
void launch_build_witness(const uint8_t* keys, const uint8_t* tx_hashes, uint32_t n,
                          uint8_t* out256, cudaStream_t s);
void launch_witness_xor(const uint8_t* master, const uint8_t* tx_hashes, const uint64_t* masks,
                        const uint8_t* in, uint32_t len, uint32_t n, uint8_t* out,
                        cudaStream_t s);

// Throughput probe: `iters` dependent compressions per thread (roofline peak).
void launch_sha256_peak(uint32_t* sink, uint32_t iters, int blocks, int threads, cudaStream_t s);

}  // namespace ace_gpu
