/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the Prove path.
 *
 * A plain-C restatement of the reference's mock Prove phase (ACE Runtime,
 * /root/reference/proj), used by tests/ and bench.py's cpu_baseline leg as the
 * checker. It is never linked into or called by the product library
 * (paper_2603_10242_b200/lib/libacegpu.so). Every function cites the reference
 * file:line it restates. Parity is pinned against the reference itself
 * (oracle/_ref/libaceref.so, built from the reference sources by
 * oracle/Makefile) and against the RFC/FIPS known answers the reference's own
 * tests hold (tests/test_oracle.py).
 *
 * Flat layouts shared with the product C-ABI (include/acegpu.h):
 *   payloads      concatenated bytes; tx i = payloads[offs[i] .. offs[i+1])
 *   attestation   104 B = obj_hash(32) | id_com(32) | domain(8) | credential(32)
 *                 (crypto.cpp:56-65)
 *   header        256 B BlockHeader encoding (wire.cpp:74-98)
 *   proof         289 B = bytes(256) | public_inputs_digest(32) | kind(1)
 *                 kind 0 = Tx, 1 = Aggregate (prover.hpp:33-43)
 *   fc            328 B = block_hash | slot_be64 | proof(256) | commitment
 *                 (wire.cpp:125-133)
 */
#ifndef ACE_ORACLE_H
#define ACE_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    uint32_t h[8];
    uint64_t total;
    uint8_t buf[64];
    size_t n;
} or_sha_ctx;

void or_sha_init(or_sha_ctx* c);
void or_sha_update(or_sha_ctx* c, const uint8_t* d, size_t len);
void or_sha_final(or_sha_ctx* c, uint8_t out[32]);
void or_sha256(const uint8_t* m, uint64_t len, uint8_t out[32]);
void or_hmac_sha256(const uint8_t* key, uint64_t klen, const uint8_t* msg, uint64_t mlen,
                    uint8_t out[32]);
int or_hkdf_sha256(const uint8_t* ikm, uint64_t ikm_len, const uint8_t* salt, uint64_t salt_len,
                   const uint8_t* info, uint64_t info_len, uint8_t* out, uint64_t out_len);

void or_rev_from_seed(uint64_t seed, uint8_t out[32]);
void or_domain_encode(uint16_t chain, uint64_t slot, uint8_t out[8]);
void or_id_commitment(const uint8_t rev[32], const uint8_t salt[32], uint16_t chain, uint64_t slot,
                      uint8_t out[32]);
void or_derive_attest_key(const uint8_t rev[32], const uint8_t dom8[8], uint8_t out[32]);
void or_generate_attestation(const uint8_t rev[32], const uint8_t* payload, uint64_t len,
                             const uint8_t dom8[8], const uint8_t id_com[32], uint8_t out104[104]);
int or_verify_attestation_full(const uint8_t att[104], const uint8_t* payload, uint64_t len,
                               const uint8_t rev[32]);
void or_verify_attestations_batch(const uint8_t* payloads, const uint64_t* offs,
                                  const uint8_t* atts, uint32_t n, const uint8_t* revs,
                                  const uint32_t* rev_index, uint8_t* codes, int threads);

void or_make_transfer_payload(const uint8_t from[32], const uint8_t to[32], uint64_t amount,
                              uint64_t nonce, const uint8_t recent[32], uint8_t out154[154]);
void or_block_hash(const uint8_t header[256], uint8_t out[32]);
void or_merkle_root(const uint8_t* leaves, uint64_t n, uint8_t out[32]);

/* Phase 1a. attest_check_light (pipeline.cpp:20-42):
 * 0 AcceptPendingProof, 1 PayloadBinding, 2 UnknownIdentity, 3 StaleDomain.
 * registry = n_reg sorted 32-B id commitments (std::set<Hash32> order). */
int or_attest_check_light(const uint8_t* payload, uint64_t len, const uint8_t att[104],
                          const uint8_t* registry, uint64_t n_reg, uint64_t current_slot,
                          uint64_t window_slots);
/* tx_merkle_root / attest_merkle_root (wire.cpp:257-273). */
void or_block_roots(const uint8_t* payloads, const uint64_t* offs, const uint8_t* atts,
                    uint64_t n, uint8_t tx_root[32], uint8_t att_root[32]);
void or_expand256(int kind, const uint8_t digest[32], uint8_t out[256]);
void or_prove_public_inputs(const uint8_t pub160[160], uint8_t out289[289]);
void or_prove_tx(const uint8_t* payload, uint64_t len, const uint8_t att[104], uint8_t out289[289]);
int or_verify_mock(const uint8_t p289[289]);
void or_aggregate_pair(const uint8_t a289[289], const uint8_t b289[289], uint8_t out289[289]);
int or_aggregate_tree(const uint8_t* proofs289, uint64_t n, uint8_t out289[289], uint64_t* levels,
                      uint64_t* pairs);
int or_prove_block(const uint8_t* payloads, const uint64_t* offs, const uint8_t* atts, uint32_t n,
                   const uint8_t header[256], uint8_t out289[289], uint64_t* levels,
                   uint64_t* pairs, int threads);
void or_build_fc(const uint8_t* atts, uint32_t n, const uint8_t header[256],
                 const uint8_t proof289[289], uint8_t out328[328]);
int or_verify_fc(const uint8_t fc[328], const uint8_t* payloads, const uint64_t* offs,
                 const uint8_t* atts, uint32_t n, const uint8_t header[256], int threads);

void or_build_witness(const uint8_t key[32], const uint8_t tx_hash[32], uint8_t out256[256]);
int or_witness_matches_tx(const uint8_t* witness, uint64_t wlen, const uint8_t att[104]);
unsigned or_scheme_threshold(unsigned n_validators);
uint64_t or_scheme_share_mask(unsigned n_validators, unsigned validator);
void or_scheme_share_value(const uint8_t master[32], const uint8_t tx_hash[32], unsigned index,
                           uint8_t out[32]);
void or_keystream(const uint8_t key[32], uint64_t len, uint8_t* out);
void or_scheme_encapsulate(unsigned n_validators, const uint8_t master[32],
                           const uint8_t tx_hash[32], const uint8_t* witness, uint64_t len,
                           uint8_t* out_ct);
void or_scheme_decrypt(unsigned n_validators, const uint8_t master[32], const uint8_t tx_hash[32],
                       const uint8_t* ct, uint64_t len, const unsigned* contributors,
                       unsigned n_contrib, uint8_t* out);

#ifdef __cplusplus
}
#endif
#endif
