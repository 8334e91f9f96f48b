// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" face over the UNMODIFIED reference library (proj/src/*.cpp built
// by oracle/Makefile into oracle/_ref/libace_core.a). Tests use it as the
// pinned checker; bench.py --impl reference times the reference's own CPU
// Prove path through it. Flat buffers in, flat buffers out:
//   payloads      concatenated payload bytes, payload i = payloads[offs[i]:offs[i+1]]
//   attestations  n x 104 B, Attestation::encode layout (crypto.cpp:56-65)
//   header        256 B, BlockHeader::encode layout (wire.cpp:74-98)
#include <chrono>
#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <stdexcept>
#include <thread>
#include <vector>

#include "ace/bench.hpp"
#include "ace/crypto.hpp"
#include "ace/hkdf.hpp"
#include "ace/pipeline.hpp"
#include "ace/prover.hpp"
#include "ace/sha256.hpp"
#include "ace/thread_pool.hpp"
#include "ace/wire.hpp"

using namespace ace;

namespace {

wire::Block make_block(const uint8_t* payloads, const uint64_t* offs, const uint8_t* atts,
                       uint32_t n, const uint8_t* header) {
    wire::Block b;
    auto h = wire::BlockHeader::decode({header, 256});
    if (!h) throw std::runtime_error("bad header");
    b.header = *h;
    b.transactions.resize(n);
    for (uint32_t i = 0; i < n; ++i) {
        auto& tx = b.transactions[i];
        tx.payload.assign(payloads + offs[i], payloads + offs[i + 1]);
        auto a = crypto::Attestation::decode({atts + 104ull * i, 104});
        if (!a) throw std::runtime_error("bad attestation");
        tx.attestation = *a;
    }
    return b;
}

void put_proof(const prover::MockProof& p, uint8_t* out289) {
    std::memcpy(out289, p.bytes.data(), 256);
    std::memcpy(out289 + 256, p.public_inputs_digest.data(), 32);
    out289[288] = static_cast<uint8_t>(p.kind);
}

prover::MockProof get_proof(const uint8_t* in289) {
    prover::MockProof p;
    std::memcpy(p.bytes.data(), in289, 256);
    std::memcpy(p.public_inputs_digest.data(), in289 + 256, 32);
    p.kind = static_cast<prover::ProofKind>(in289[288]);
    return p;
}

crypto::Rev rev_of(const uint8_t* r) { return *crypto::Rev::from_bytes({r, 32}); }

}  // namespace

extern "C" {

unsigned ref_threads() { return ThreadPool::global().size(); }

void ref_sha256(const uint8_t* msg, uint64_t len, uint8_t* out) {
    Hash32 h = sha256::digest({msg, static_cast<size_t>(len)});
    std::memcpy(out, h.data(), 32);
}

void ref_hash_batch_strided(const uint8_t* base, uint64_t stride, uint64_t len, uint64_t count,
                            uint8_t* out) {
    sha256::hash_batch_strided(base, stride, len, count, out);
}

void ref_hmac_sha256(const uint8_t* key, uint64_t klen, const uint8_t* msg, uint64_t mlen,
                     uint8_t* out) {
    Hash32 h = crypto::hmac_sha256({key, static_cast<size_t>(klen)},
                                   {msg, static_cast<size_t>(mlen)});
    std::memcpy(out, h.data(), 32);
}

int ref_hkdf_sha256(const uint8_t* ikm, uint64_t ikm_len, const uint8_t* salt, uint64_t salt_len,
                    const uint8_t* info, uint64_t info_len, uint8_t* out, uint64_t out_len) {
    try {
        Bytes okm = crypto::hkdf_sha256({ikm, static_cast<size_t>(ikm_len)},
                                        {salt, static_cast<size_t>(salt_len)},
                                        {info, static_cast<size_t>(info_len)}, out_len);
        std::memcpy(out, okm.data(), okm.size());
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

void ref_rev_from_seed(uint64_t seed, uint8_t* out32) {
    auto r = crypto::Rev::from_seed(seed);
    std::memcpy(out32, r.bytes().data(), 32);
}

void ref_id_commitment(const uint8_t* rev, const uint8_t* salt32, uint16_t chain, uint64_t slot,
                       uint8_t* out32) {
    Hash32 s;
    std::memcpy(s.data(), salt32, 32);
    auto c = crypto::id_commitment(rev_of(rev), s, crypto::Domain{chain, slot});
    std::memcpy(out32, c.bytes.data(), 32);
}

void ref_derive_attest_key(const uint8_t* rev, uint16_t chain, uint64_t slot, uint8_t* out32) {
    auto k = crypto::derive_attest_key(rev_of(rev), crypto::Domain{chain, slot});
    std::memcpy(out32, k.bytes.data(), 32);
}

void ref_generate_attestation(const uint8_t* rev, const uint8_t* payload, uint64_t len,
                              uint16_t chain, uint64_t slot, const uint8_t* id_com32,
                              uint8_t* out104) {
    crypto::IdCommitment idc;
    std::memcpy(idc.bytes.data(), id_com32, 32);
    auto a = crypto::generate_attestation(rev_of(rev), {payload, static_cast<size_t>(len)},
                                          crypto::Domain{chain, slot}, idc);
    auto enc = a.encode();
    std::memcpy(out104, enc.data(), 104);
}

int ref_verify_attestation_full(const uint8_t* att104, const uint8_t* payload, uint64_t len,
                                const uint8_t* rev) {
    auto a = crypto::Attestation::decode({att104, 104});
    return static_cast<int>(crypto::verify_attestation_full(*a, {payload, static_cast<size_t>(len)},
                                                            rev_of(rev)));
}

// Batched full verification, parallel over the reference's own ThreadPool.
// revs: table of 32-B REVs, rev_index[i] selects tx i's REV.
void ref_verify_attestations_batch(const uint8_t* payloads, const uint64_t* offs,
                                   const uint8_t* atts, uint32_t n, const uint8_t* revs,
                                   const uint32_t* rev_index, uint8_t* codes) {
    std::vector<crypto::Attestation> dec(n);
    for (uint32_t i = 0; i < n; ++i) dec[i] = *crypto::Attestation::decode({atts + 104ull * i, 104});
    ThreadPool::global().parallel_for(n, [&](size_t i) {
        auto r = rev_of(revs + 32ull * rev_index[i]);
        codes[i] = static_cast<uint8_t>(crypto::verify_attestation_full(
            dec[i], {payloads + offs[i], static_cast<size_t>(offs[i + 1] - offs[i])}, r));
    });
}

void ref_make_transfer_payload(const uint8_t* from32, const uint8_t* to32, uint64_t amount,
                               uint64_t nonce, const uint8_t* recent32, uint8_t* out154) {
    wire::AccountId a, b;
    Hash32 r;
    std::memcpy(a.data(), from32, 32);
    std::memcpy(b.data(), to32, 32);
    std::memcpy(r.data(), recent32, 32);
    Bytes p = wire::make_transfer_payload(a, b, amount, nonce, r);
    std::memcpy(out154, p.data(), p.size());
}

void ref_block_hash(const uint8_t* header256, uint8_t* out32) {
    auto h = wire::BlockHeader::decode({header256, 256});
    Hash32 d = wire::block_hash(*h);
    std::memcpy(out32, d.data(), 32);
}

void ref_merkle_root(const uint8_t* leaves, uint64_t n, uint8_t* out32) {
    std::vector<Hash32> v(n);
    if (n) std::memcpy(v.data(), leaves, 32 * n);
    Hash32 r = wire::merkle_root(v);
    std::memcpy(out32, r.data(), 32);
}

void ref_tx_merkle_root(const uint8_t* payloads, const uint64_t* offs, const uint8_t* atts,
                        uint32_t n, uint8_t* tx_root, uint8_t* att_root) {
    uint8_t zero[256] = {0};
    auto b = make_block(payloads, offs, atts, n, zero);
    Hash32 t = wire::tx_merkle_root(b.transactions);
    Hash32 a = wire::attest_merkle_root(b.transactions);
    std::memcpy(tx_root, t.data(), 32);
    std::memcpy(att_root, a.data(), 32);
}

// pipeline::attest_check_light over a block, with the reference's own
// IdentityRegistry; counters summed as process_slot does (pipeline.cpp:110-122).
void ref_attest_check_light_batch(const uint8_t* payloads, const uint64_t* offs,
                                  const uint8_t* atts, uint32_t n, const uint8_t* ids,
                                  uint64_t n_ids, uint64_t current_slot, uint64_t window,
                                  uint8_t* codes, uint64_t* counters3) {
    uint8_t zero[256] = {0};
    auto b = make_block(payloads, offs, atts, n, zero);
    pipeline::IdentityRegistry reg;
    for (uint64_t i = 0; i < n_ids; ++i) {
        Hash32 h;
        std::memcpy(h.data(), ids + 32 * i, 32);
        reg.add(h);
    }
    pipeline::PipelineConfig cfg;
    cfg.domain_window_slots = window;
    pipeline::LightCheckCounters c;
    for (uint32_t i = 0; i < n; ++i)
        codes[i] = static_cast<uint8_t>(
            pipeline::attest_check_light(b.transactions[i], reg, current_slot, cfg, &c));
    counters3[0] = c.sha256_ops;
    counters3[1] = c.registry_probes;
    counters3[2] = c.window_checks;
}

void ref_prove_tx(const uint8_t* payload, uint64_t len, const uint8_t* att104, uint8_t* out289) {
    wire::Transaction tx;
    tx.payload.assign(payload, payload + len);
    tx.attestation = *crypto::Attestation::decode({att104, 104});
    put_proof(prover::prove_tx(tx), out289);
}

void ref_prove_public_inputs(const uint8_t* five_words160, uint8_t* out289) {
    prover::PublicInputs pub;
    std::memcpy(pub.id_com.data(), five_words160, 32);
    std::memcpy(pub.tx_hash.data(), five_words160 + 32, 32);
    std::memcpy(pub.domain.data(), five_words160 + 64, 32);
    std::memcpy(pub.target.data(), five_words160 + 96, 32);
    std::memcpy(pub.rp_com.data(), five_words160 + 128, 32);
    put_proof(prover::prove_public_inputs(pub), out289);
}

int ref_verify_mock(const uint8_t* in289) { return prover::verify_mock(get_proof(in289)) ? 1 : 0; }

void ref_aggregate_pair(const uint8_t* a289, const uint8_t* b289, uint8_t* out289) {
    put_proof(prover::aggregate_pair(get_proof(a289), get_proof(b289)), out289);
}

int ref_aggregate_tree(const uint8_t* proofs289, uint64_t n, uint8_t* out289, uint64_t* levels,
                       uint64_t* pairs) {
    std::vector<prover::MockProof> v(n);
    for (uint64_t i = 0; i < n; ++i) v[i] = get_proof(proofs289 + 289 * i);
    try {
        prover::AggregationStats st;
        put_proof(prover::aggregate_tree(v, &st), out289);
        *levels = st.levels;
        *pairs = st.pair_ops;
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

int ref_prove_block(const uint8_t* payloads, const uint64_t* offs, const uint8_t* atts, uint32_t n,
                    const uint8_t* header, uint8_t* out289, uint64_t* levels, uint64_t* pairs) {
    try {
        auto b = make_block(payloads, offs, atts, n, header);
        prover::AggregationStats st;
        put_proof(prover::prove_block(b, &st), out289);
        *levels = st.levels;
        *pairs = st.pair_ops;
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

int ref_build_fc(const uint8_t* payloads, const uint64_t* offs, const uint8_t* atts, uint32_t n,
                 const uint8_t* header, const uint8_t* proof289, uint8_t* out328) {
    try {
        auto b = make_block(payloads, offs, atts, n, header);
        auto fc = prover::build_finality_certificate(b, get_proof(proof289));
        auto enc = fc.encode();
        std::memcpy(out328, enc.data(), 328);
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// prove_block + build_finality_certificate: the ProverService::run body (prover.cpp:350-351).
int ref_prove_and_certify(const uint8_t* payloads, const uint64_t* offs, const uint8_t* atts,
                          uint32_t n, const uint8_t* header, uint8_t* out328) {
    try {
        auto b = make_block(payloads, offs, atts, n, header);
        auto fc = prover::build_finality_certificate(b, prover::prove_block(b));
        auto enc = fc.encode();
        std::memcpy(out328, enc.data(), 328);
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

int ref_verify_fc(const uint8_t* fc328, const uint8_t* payloads, const uint64_t* offs,
                  const uint8_t* atts, uint32_t n, const uint8_t* header) {
    auto b = make_block(payloads, offs, atts, n, header);
    auto fc = wire::FinalityCertificate::decode({fc328, 328});
    return static_cast<int>(prover::verify_finality_certificate(*fc, b, nullptr));
}

void ref_build_witness(const uint8_t* key32, const uint8_t* tx_hash32, uint8_t* out256) {
    Hash32 k, t;
    std::memcpy(k.data(), key32, 32);
    std::memcpy(t.data(), tx_hash32, 32);
    Bytes w = prover::build_witness(k, t);
    std::memcpy(out256, w.data(), 256);
}

int ref_witness_matches_tx(const uint8_t* witness, uint64_t wlen, const uint8_t* payload,
                           uint64_t plen, const uint8_t* att104) {
    wire::Transaction tx;
    tx.payload.assign(payload, payload + plen);
    tx.attestation = *crypto::Attestation::decode({att104, 104});
    return prover::witness_matches_tx({witness, static_cast<size_t>(wlen)}, tx) ? 1 : 0;
}

void ref_witness_matches_batch(const uint8_t* witnesses, const uint8_t* payloads,
                               const uint64_t* offs, const uint8_t* atts, uint32_t n,
                               uint8_t* ok) {
    uint8_t zero[256] = {0};
    auto b = make_block(payloads, offs, atts, n, zero);
    ThreadPool::global().parallel_for(n, [&](size_t i) {
        ok[i] = prover::witness_matches_tx({witnesses + 256 * i, 256}, b.transactions[i]) ? 1 : 0;
    });
}

unsigned ref_scheme_threshold(unsigned n_validators) {
    Hash32 m{};
    return prover::WitnessScheme(n_validators, m).threshold();
}

// share_indices(validator) as a bitmask (n <= 64).
uint64_t ref_scheme_share_mask(unsigned n_validators, unsigned validator) {
    Hash32 m{};
    uint64_t mask = 0;
    for (unsigned j : prover::WitnessScheme(n_validators, m).share_indices(validator)) mask |= 1ull << j;
    return mask;
}

void ref_scheme_share_value(unsigned n_validators, const uint8_t* master32,
                            const uint8_t* tx_hash32, unsigned index, uint8_t* out32) {
    Hash32 m, t;
    std::memcpy(m.data(), master32, 32);
    std::memcpy(t.data(), tx_hash32, 32);
    Hash32 v = prover::WitnessScheme(n_validators, m).share_value(t, index);
    std::memcpy(out32, v.data(), 32);
}

void ref_scheme_encapsulate(unsigned n_validators, const uint8_t* master32,
                            const uint8_t* tx_hash32, const uint8_t* witness, uint64_t wlen,
                            uint8_t* out_ct) {
    Hash32 m, t;
    std::memcpy(m.data(), master32, 32);
    std::memcpy(t.data(), tx_hash32, 32);
    auto b = prover::WitnessScheme(n_validators, m).encapsulate(t, {witness, static_cast<size_t>(wlen)});
    std::memcpy(out_ct, b.ciphertext.data(), b.ciphertext.size());
}

void ref_scheme_decrypt(unsigned n_validators, const uint8_t* master32, const uint8_t* tx_hash32,
                        const uint8_t* ct, uint64_t len, const unsigned* contributors,
                        unsigned n_contrib, uint8_t* out) {
    Hash32 m;
    std::memcpy(m.data(), master32, 32);
    prover::WitnessScheme s(n_validators, m);
    prover::WitnessBundle b;
    std::memcpy(b.tx_hash.data(), tx_hash32, 32);
    b.ciphertext.assign(ct, ct + len);
    b.share_threshold = s.threshold();
    Bytes p = s.decrypt(b, {contributors, n_contrib});
    std::memcpy(out, p.data(), p.size());
}

// Full backup_prove over a block where every validator in [0, n_holders) holds
// every tx's shares except those listed as withheld (missing bundle).
// Returns 0 with out328 = FC, or the number of missing tx hashes (written to
// missing_out as 32-B hashes).
int ref_backup_prove(const uint8_t* payloads, const uint64_t* offs, const uint8_t* atts,
                     uint32_t n, const uint8_t* header, unsigned n_validators,
                     const uint8_t* master32, const uint8_t* ciphertexts /* n x 256 */,
                     const uint8_t* has_bundle /* n */, unsigned n_holders, uint8_t* out328,
                     uint8_t* missing_out) {
    auto b = make_block(payloads, offs, atts, n, header);
    Hash32 m;
    std::memcpy(m.data(), master32, 32);
    prover::WitnessScheme s(n_validators, m);
    std::map<Hash32, prover::WitnessBundle> bundles;
    std::map<unsigned, std::set<Hash32>> holders;
    for (uint32_t i = 0; i < n; ++i) {
        Hash32 h = sha256::digest(b.transactions[i].payload);
        if (has_bundle[i]) {
            prover::WitnessBundle wb;
            wb.tx_hash = h;
            wb.ciphertext.assign(ciphertexts + 256ull * i, ciphertexts + 256ull * (i + 1));
            wb.share_threshold = s.threshold();
            bundles[h] = wb;
        }
        for (unsigned v = 0; v < n_holders; ++v) holders[v].insert(h);
    }
    auto r = prover::backup_prove(b, bundles, holders, s);
    if (auto* fc = std::get_if<wire::FinalityCertificate>(&r)) {
        auto enc = fc->encode();
        std::memcpy(out328, enc.data(), 328);
        return 0;
    }
    const auto& miss = std::get<prover::BackupUnavailable>(r).missing_tx_hashes;
    for (size_t i = 0; i < miss.size(); ++i) std::memcpy(missing_out + 32 * i, miss[i].data(), 32);
    return static_cast<int>(miss.size());
}

uint64_t ref_work_tx_proofs() { return prover::work_counters().tx_proofs.load(); }
uint64_t ref_work_aggregations() { return prover::work_counters().aggregations.load(); }

// The reference's Phase-2 CPU path for one block as the bench times it:
// verify_attestation_full over every tx (crypto.cpp:141-154), then prove_block
// (prover.cpp:129-142) + build_finality_certificate (:144-156). Returns wall
// microseconds; codes/out328 receive the results.
double ref_attest_prove_certify(const uint8_t* payloads, const uint64_t* offs, const uint8_t* atts,
                                uint32_t n, const uint8_t* header, const uint8_t* revs,
                                const uint32_t* rev_index, uint8_t* codes, uint8_t* out328) {
    auto b = make_block(payloads, offs, atts, n, header);  // input marshalling, untimed
    auto t0 = std::chrono::steady_clock::now();
    ThreadPool::global().parallel_for(n, [&](size_t i) {
        auto r = rev_of(revs + 32ull * rev_index[i]);
        codes[i] = static_cast<uint8_t>(crypto::verify_attestation_full(
            b.transactions[i].attestation, b.transactions[i].payload, r));
    });
    auto fc = prover::build_finality_certificate(b, prover::prove_block(b));
    auto enc = fc.encode();
    std::memcpy(out328, enc.data(), 328);
    auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double, std::micro>(t1 - t0).count();
}

}  // extern "C"
