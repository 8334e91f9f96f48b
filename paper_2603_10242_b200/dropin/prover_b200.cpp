// Drop-in replacement for the reference's proj/src/prover.cpp.
//
// Implements every symbol of proj/include/ace/prover.hpp (compiled against
// that header, unchanged) on top of the B200 C ABI in include/acegpu.h: all
// hashing — leaf proofs, aggregation tree, finality certificate, witnesses,
// threshold-share keystreams — runs as sm_100a kernels in libacegpu.so.
// A maintainer swaps prover.cpp for this file in proj/src/CMakeLists.txt and
// links libacegpu. Semantics follow the reference line by
// line (cited); there is no CPU fallback: without an sm_100 device every
// entry point throws std::runtime_error.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "acegpu.h"
#include "ace/prover.hpp"

namespace ace::prover {

namespace {

acegpu_ctx* ctx() {
    static std::once_flag once;
    static acegpu_ctx* c = nullptr;
    static std::string err;
    std::call_once(once, [] {
        int dev = 0;
        if (const char* e = std::getenv("ACEGPU_DEVICE")) dev = std::atoi(e);
        if (acegpu_create(dev, &c) != ACEGPU_OK) err = acegpu_last_error();
    });
    if (!c) throw std::runtime_error("ace::prover (B200 drop-in): " + err);
    return c;
}

void check(int rc) {
    if (rc == ACEGPU_OK) return;
    if (rc == ACEGPU_EINVAL) throw std::invalid_argument(acegpu_last_error());
    throw std::runtime_error(std::string("acegpu: ") + acegpu_last_error());
}

// Flat C-ABI view of a block (acegpu.h layouts).
struct Flat {
    Bytes payloads;
    std::vector<uint64_t> offs;
    Bytes atts;
    std::array<uint8_t, 256> header{};
    uint64_t n = 0;
};

Flat flatten(const wire::Block& b) {
    Flat f;
    f.n = b.transactions.size();
    f.offs.resize(f.n + 1, 0);
    size_t total = 0;
    for (const auto& tx : b.transactions) total += tx.payload.size();
    f.payloads.reserve(total + 16);
    f.atts.resize(104 * f.n + 8);
    for (size_t i = 0; i < f.n; ++i) {
        const auto& tx = b.transactions[i];
        f.payloads.insert(f.payloads.end(), tx.payload.begin(), tx.payload.end());
        f.offs[i + 1] = f.payloads.size();
        auto a = tx.attestation.encode();
        std::memcpy(f.atts.data() + 104 * i, a.data(), 104);
    }
    f.payloads.resize(f.payloads.size() + 16);
    f.header = b.header.encode();
    return f;
}

void to_289(const MockProof& p, uint8_t* out) {
    std::memcpy(out, p.bytes.data(), 256);
    std::memcpy(out + 256, p.public_inputs_digest.data(), 32);
    out[288] = static_cast<uint8_t>(p.kind);
}

MockProof from_289(const uint8_t* in) {
    MockProof p;
    std::memcpy(p.bytes.data(), in, 256);
    std::memcpy(p.public_inputs_digest.data(), in + 256, 32);
    p.kind = static_cast<ProofKind>(in[288]);
    return p;
}

Hash32 gpu_sha256(std::span<const uint8_t> data) {
    Bytes buf(data.begin(), data.end());
    buf.resize(data.size() + 16);
    uint64_t offs[2] = {0, data.size()};
    Hash32 h;
    check(acegpu_sha256_varlen(ctx(), buf.data(), offs, 1, h.data()));
    return h;
}

std::vector<Hash32> gpu_sha256_many(const std::vector<Bytes>& msgs) {
    std::vector<Hash32> out(msgs.size());
    if (msgs.empty()) return out;
    Bytes buf;
    std::vector<uint64_t> offs(msgs.size() + 1, 0);
    for (size_t i = 0; i < msgs.size(); ++i) {
        buf.insert(buf.end(), msgs[i].begin(), msgs[i].end());
        offs[i + 1] = buf.size();
    }
    buf.resize(buf.size() + 16);
    check(acegpu_sha256_varlen(ctx(), buf.data(), offs.data(), msgs.size(),
                               reinterpret_cast<uint8_t*>(out.data())));
    return out;
}

wire::FinalityCertificate decode_fc(const uint8_t* fc328) {
    return *wire::FinalityCertificate::decode({fc328, 328});
}

}  // namespace

WorkCounters& work_counters() {
    static WorkCounters counters;
    return counters;
}

// prover.cpp:65-72
PublicInputs PublicInputs::for_tx(const wire::Transaction& tx) {
    PublicInputs pub;
    pub.id_com = tx.attestation.id_com;
    pub.tx_hash = gpu_sha256(tx.payload);
    auto dom = tx.attestation.domain.encode();
    std::memcpy(pub.domain.data(), dom.data(), dom.size());
    return pub;
}

// prover.cpp:74-76
Hash32 PublicInputs::digest() const {
    uint8_t m[160];
    std::memcpy(m, id_com.data(), 32);
    std::memcpy(m + 32, tx_hash.data(), 32);
    std::memcpy(m + 64, domain.data(), 32);
    std::memcpy(m + 96, target.data(), 32);
    std::memcpy(m + 128, rp_com.data(), 32);
    return gpu_sha256({m, 160});
}

// prover.cpp:78-85
MockProof prove_public_inputs(const PublicInputs& pub) {
    uint8_t m[160], out[289];
    std::memcpy(m, pub.id_com.data(), 32);
    std::memcpy(m + 32, pub.tx_hash.data(), 32);
    std::memcpy(m + 64, pub.domain.data(), 32);
    std::memcpy(m + 96, pub.target.data(), 32);
    std::memcpy(m + 128, pub.rp_com.data(), 32);
    check(acegpu_prove_public_inputs(ctx(), m, 1, out));
    work_counters().tx_proofs.fetch_add(1, std::memory_order_relaxed);
    return from_289(out);
}

// prover.cpp:87-89
MockProof prove_tx(const wire::Transaction& tx) {
    Bytes p(tx.payload);
    p.resize(p.size() + 16);
    uint64_t offs[2] = {0, tx.payload.size()};
    auto a = tx.attestation.encode();
    uint8_t out[289];
    check(acegpu_prove_txs(ctx(), p.data(), offs, a.data(), 1, out));
    work_counters().tx_proofs.fetch_add(1, std::memory_order_relaxed);
    return from_289(out);
}

// prover.cpp:91-95
bool verify_mock(const MockProof& proof) {
    uint8_t in[289], ok = 0;
    to_289(proof, in);
    check(acegpu_verify_mock(ctx(), in, 1, &ok));
    return ok != 0;
}

// prover.cpp:97-104
MockProof aggregate_pair(const MockProof& a, const MockProof& b) {
    uint8_t ia[289], ib[289], out[289];
    to_289(a, ia);
    to_289(b, ib);
    check(acegpu_aggregate_pairs(ctx(), ia, ib, 1, out));
    work_counters().aggregations.fetch_add(1, std::memory_order_relaxed);
    return from_289(out);
}

// prover.cpp:106-127 (throws std::invalid_argument on an empty list)
MockProof aggregate_tree(std::span<const MockProof> proofs, AggregationStats* stats) {
    if (proofs.empty()) throw std::invalid_argument("aggregate_tree: empty proof list");
    Bytes in(289 * proofs.size());
    for (size_t i = 0; i < proofs.size(); ++i) to_289(proofs[i], in.data() + 289 * i);
    uint8_t out[289];
    uint64_t levels = 0, pairs = 0;
    check(acegpu_aggregate_tree(ctx(), in.data(), proofs.size(), out, &levels, &pairs));
    work_counters().aggregations.fetch_add(pairs, std::memory_order_relaxed);
    if (stats) *stats = {static_cast<size_t>(levels), static_cast<size_t>(pairs)};
    return from_289(out);
}

// prover.cpp:129-142 (the empty block proves PublicInputs{tx_hash = block_hash})
MockProof prove_block(const wire::Block& block, AggregationStats* stats) {
    Flat f = flatten(block);
    uint8_t out[289];
    uint64_t levels = 0, pairs = 0;
    check(acegpu_prove_block(ctx(), f.payloads.data(), f.offs.data(), f.atts.data(), f.n,
                             f.header.data(), out, &levels, &pairs));
    work_counters().tx_proofs.fetch_add(f.n ? f.n : 1, std::memory_order_relaxed);
    work_counters().aggregations.fetch_add(pairs, std::memory_order_relaxed);
    if (stats) *stats = {static_cast<size_t>(levels), static_cast<size_t>(pairs)};
    return from_289(out);
}

// prover.cpp:144-156
wire::FinalityCertificate build_finality_certificate(const wire::Block& block,
                                                     const MockProof& aggregate) {
    Flat f = flatten(block);
    uint8_t proof[289], fc[328];
    to_289(aggregate, proof);
    check(acegpu_build_fc(ctx(), f.atts.data(), f.n, f.header.data(), proof, fc));
    return decode_fc(fc);
}

// prover.cpp:158-169: slot, block hash, then the full recompute.
FcCheck verify_finality_certificate(const wire::FinalityCertificate& fc, const wire::Block& block,
                                    std::uint64_t* cost_units) {
    if (cost_units) *cost_units += kFcVerifyCostUnits;
    if (fc.slot_number != block.header.slot_number) return FcCheck::SlotMismatch;
    Flat f = flatten(block);
    uint8_t expect[328];
    uint64_t pairs = 0;
    check(acegpu_attest_prove_certify(ctx(), f.payloads.data(), f.offs.data(), f.atts.data(), f.n,
                                      f.header.data(), nullptr, 0, nullptr, nullptr, nullptr,
                                      expect, nullptr, &pairs));
    work_counters().tx_proofs.fetch_add(f.n ? f.n : 1, std::memory_order_relaxed);
    work_counters().aggregations.fetch_add(pairs, std::memory_order_relaxed);
    wire::FinalityCertificate e = decode_fc(expect);
    if (fc.block_hash != e.block_hash) return FcCheck::HashMismatch;
    if (e.proof != fc.proof) return FcCheck::ProofMismatch;
    if (e.public_inputs_commitment != fc.public_inputs_commitment) return FcCheck::ProofMismatch;
    return FcCheck::Valid;
}

const char* to_string(FcCheck c) {
    static const char* const kNames[] = {"Valid", "SlotMismatch", "HashMismatch",
                                         "ProofMismatch"};
    const auto i = static_cast<unsigned>(c);
    return i < 4 ? kNames[i] : "?";
}

// prover.cpp:181-188
Bytes build_witness(const Hash32& attest_key, const Hash32& tx_hash) {
    Bytes w(kWitnessBytes);
    check(acegpu_build_witness(ctx(), attest_key.data(), tx_hash.data(), 1, w.data()));
    return w;
}

// prover.cpp:190-197
bool witness_matches_tx(std::span<const std::uint8_t> witness, const wire::Transaction& tx) {
    if (witness.size() != kWitnessBytes) return false;
    auto a = tx.attestation.encode();
    uint8_t ok = 0;
    uint32_t len = static_cast<uint32_t>(witness.size());
    check(acegpu_witness_check(ctx(), witness.data(), &len, a.data(), 1, &ok));
    return ok != 0;
}

// prover.cpp:199-204
WitnessScheme::WitnessScheme(unsigned n_validators, const Hash32& master_seed)
    : n_(n_validators), t_((2 * n_validators + 2) / 3), master_(master_seed) {
    if (n_validators == 0) {
        throw std::invalid_argument("WitnessScheme: need at least one validator");
    }
}

// prover.cpp:206-216: share j lives on validators j .. j+(n-t) mod n.
std::vector<unsigned> WitnessScheme::share_indices(unsigned validator) const {
    // validator v holds share j iff v is one of j, j+1, ..., j+(n-t) (mod n),
    // i.e. j in {v-(n-t), ..., v} (mod n), restricted to j < t.
    std::vector<unsigned> held;
    const unsigned reach = n_ - t_;
    for (unsigned back = 0; back <= reach; ++back) {
        const unsigned j = (validator % n_ + n_ - back) % n_;
        if (j < t_) held.push_back(j);
    }
    std::sort(held.begin(), held.end());
    return held;
}

namespace {
Bytes share_msg(const Hash32& master, const Hash32& tx_hash, unsigned index) {
    static const char tag[] = "witness-share-v1";  // prover.cpp:17
    Bytes m(tag, tag + 16);
    m.insert(m.end(), master.begin(), master.end());
    m.insert(m.end(), tx_hash.begin(), tx_hash.end());
    uint8_t be[4];
    put_u32be(be, index);
    m.insert(m.end(), be, be + 4);
    return m;
}

// XOR keystream with the key = XOR of the selected share values. Share sets
// up to 64 wide go through the fused GPU kernel; wider sets hash the shares
// and the keystream blocks in GPU batches.
Bytes xor_stream(const Hash32& master, const Hash32& tx_hash, const std::vector<unsigned>& shares,
                 std::span<const uint8_t> in) {
    Bytes out(in.size());
    if (in.empty()) return out;
    bool narrow = true;
    uint64_t mask = 0;
    for (unsigned j : shares) {
        if (j >= 64) narrow = false;
        else mask |= 1ull << j;
    }
    if (narrow) {
        check(acegpu_witness_xor(ctx(), master.data(), tx_hash.data(), &mask, in.data(), in.size(),
                                 1, out.data()));
        return out;
    }
    std::vector<Bytes> msgs;
    for (unsigned j : shares) msgs.push_back(share_msg(master, tx_hash, j));
    Hash32 key{};
    for (const auto& s : gpu_sha256_many(msgs))
        for (int i = 0; i < 32; ++i) key[i] ^= s[i];
    static const char stream_tag[] = "witness-stream-v1";  // prover.cpp:18
    std::vector<Bytes> blocks;
    for (uint32_t c = 0; 32ull * c < in.size(); ++c) {
        Bytes m(stream_tag, stream_tag + 17);
        m.insert(m.end(), key.begin(), key.end());
        uint8_t be[4];
        put_u32be(be, c);
        m.insert(m.end(), be, be + 4);
        blocks.push_back(std::move(m));
    }
    auto ks = gpu_sha256_many(blocks);
    for (size_t i = 0; i < in.size(); ++i) out[i] = in[i] ^ ks[i / 32][i % 32];
    return out;
}
}  // namespace

// prover.cpp:221-226
Hash32 WitnessScheme::share_value(const Hash32& tx_hash, unsigned index) const {
    return gpu_sha256(share_msg(master_, tx_hash, index));
}

// prover.cpp:228-235 (key = XOR of all t shares)
Hash32 WitnessScheme::tx_key(const Hash32& tx_hash) const {
    Hash32 key{};
    for (unsigned j = 0; j < t_; ++j) {
        Hash32 s = share_value(tx_hash, j);
        for (int i = 0; i < 32; ++i) key[i] ^= s[i];
    }
    return key;
}

// prover.cpp:237-243
WitnessBundle WitnessScheme::encapsulate(const Hash32& tx_hash,
                                         std::span<const std::uint8_t> witness) const {
    WitnessBundle b;
    b.tx_hash = tx_hash;
    b.share_threshold = t_;
    std::vector<unsigned> all(t_);
    for (unsigned j = 0; j < t_; ++j) all[j] = j;
    b.ciphertext = xor_stream(master_, tx_hash, all, witness);
    return b;
}

// prover.cpp:245-264: XOR of the share values the contributors cover.
Bytes WitnessScheme::decrypt(const WitnessBundle& bundle,
                             std::span<const unsigned> contributors) const {
    std::set<unsigned> covered;
    for (unsigned v : contributors)
        for (unsigned j : share_indices(v % n_)) covered.insert(j);
    return xor_stream(master_, bundle.tx_hash, {covered.begin(), covered.end()},
                      bundle.ciphertext);
}

// prover.cpp:266-299
BackupResult backup_prove(const wire::Block& block,
                          const std::map<Hash32, WitnessBundle>& bundles,
                          const std::map<unsigned, std::set<Hash32>>& holders,
                          const WitnessScheme& scheme) {
    // Batched where the public API allows it: every payload hash in one
    // launch and every witness check in one HMAC launch (decryption goes
    // through WitnessScheme::decrypt, whose master seed is private).
    // Verdicts per tx are exactly the reference's sequential ones.
    const size_t n = block.transactions.size();
    std::vector<Bytes> payloads;
    payloads.reserve(n);
    for (const auto& tx : block.transactions) payloads.push_back(tx.payload);
    const std::vector<Hash32> hashes = gpu_sha256_many(payloads);

    std::vector<char> bad(n, 0);
    std::vector<Bytes> plain(n);
    for (size_t i = 0; i < n; ++i) {
        auto it = bundles.find(hashes[i]);
        std::vector<unsigned> contributors;
        for (const auto& kv : holders)
            if (kv.second.count(hashes[i])) contributors.push_back(kv.first);
        if (it == bundles.end() || contributors.size() < scheme.threshold()) {
            bad[i] = 1;
            continue;
        }
        plain[i] = scheme.decrypt(it->second, contributors);  // GPU keystream (master is private)
    }
    std::vector<size_t> cand;
    for (size_t i = 0; i < n; ++i)
        if (!bad[i]) cand.push_back(i);
    if (!cand.empty()) {
        Bytes w(kWitnessBytes * cand.size()), atts(104 * cand.size() + 8);
        std::vector<uint32_t> lens(cand.size());
        std::vector<uint8_t> ok(cand.size());
        for (size_t k = 0; k < cand.size(); ++k) {
            const Bytes& p = plain[cand[k]];
            lens[k] = static_cast<uint32_t>(p.size());
            std::memcpy(w.data() + kWitnessBytes * k, p.data(), std::min(p.size(), kWitnessBytes));
            auto a = block.transactions[cand[k]].attestation.encode();
            std::memcpy(atts.data() + 104 * k, a.data(), 104);
        }
        check(acegpu_witness_check(ctx(), w.data(), lens.data(), atts.data(), cand.size(),
                                   ok.data()));
        for (size_t k = 0; k < cand.size(); ++k)
            if (!ok[k]) bad[cand[k]] = 1;
    }
    BackupUnavailable missing;
    for (size_t i = 0; i < n; ++i)
        if (bad[i]) missing.missing_tx_hashes.push_back(hashes[i]);
    if (!missing.missing_tx_hashes.empty()) return missing;
    return build_finality_certificate(block, prove_block(block));
}

// ProverService (prover.hpp:141-172): FIFO hand-off to one worker thread that
// owns the GPU pipeline; shutdown drains what is already queued
// (prover.cpp:339-359 semantics).
ProverService::ProverService() : worker_([this] { run(); }) {}

ProverService::~ProverService() {
    std::unique_lock lk(mu_);
    stop_ = true;
    lk.unlock();
    cv_in_.notify_all();
    if (worker_.joinable()) worker_.join();
}

void ProverService::enqueue(wire::Block block) {
    std::unique_lock lk(mu_);
    in_.emplace_back(std::move(block));
    lk.unlock();
    enqueued_++;
    cv_in_.notify_one();
}

std::optional<ProverService::Result> ProverService::try_pop_result() {
    std::optional<Result> r;
    std::lock_guard lk(mu_);
    if (!out_.empty()) {
        r.emplace(std::move(out_.front()));
        out_.pop_front();
    }
    return r;
}

ProverService::Result ProverService::wait_result() {
    std::unique_lock lk(mu_);
    while (out_.empty()) cv_out_.wait(lk);
    Result r{std::move(out_.front())};
    out_.pop_front();
    return r;
}

void ProverService::run() {
    std::unique_lock lk(mu_);
    while (true) {
        while (!stop_ && in_.empty()) cv_in_.wait(lk);
        if (in_.empty()) break;  // stopped and drained
        Result r{std::move(in_.front()), {}};
        in_.pop_front();
        lk.unlock();
        r.fc = build_finality_certificate(r.block, prove_block(r.block));
        lk.lock();
        out_.emplace_back(std::move(r));
        proved_++;
        cv_out_.notify_all();
    }
}

}  // namespace ace::prover
