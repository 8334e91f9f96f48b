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
    const uint8_t* revs;       // REV table (32 B each) — attestation only
    const uint32_t* rev_index; // n entries — attestation only
    uint8_t* codes;            // n verdicts, or nullptr to skip attestation
    uint8_t* nodes;            // n x 320 leaf proof records, or nullptr (attest-only)
    uint8_t* merkle;           // n x 32 merkle leaf hashes H(0x00|id_com), or nullptr
    const uint8_t* header;     // 256-B header; nullptr = no block hash
    uint8_t* block_hash;       // 32 B out when header != nullptr
    // Optional attest-key cache: per REV u, the HMAC ipad/opad midstates of
    // derive_attest_key(REV_u, D0) where D0 = the domain of tx 0. A tx whose
    // domain equals D0 uses them (2 compressions for the credential instead
    // of 12); any other domain takes the full path. Exact either way.
// launch_keytab builds it from the domain at `dom8` (8 device bytes).
    const uint32_t* keytab;    // n_revs x 16 words, or nullptr
    const uint8_t* keydom;     // the 8-B domain D0 the keytab was built for
};

void launch_leaves(const LeafArgs& a, cudaStream_t s);
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
