/* TEST INFRASTRUCTURE ONLY — CPU oracle for the mock Prove path.
 * See ace_oracle.h for the contract. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg load this file's library, always as the checker.
 * References are to /root/reference/proj. */
#define _POSIX_C_SOURCE 200809L
#include "ace_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- SHA-256 --
 * FIPS 180-4; restates the scalar engine of src/sha256.cpp:104-141 and the
 * streaming Hasher of src/sha256.cpp:215-257. */
static const uint32_t K256[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

#define ROR(x, n) (((x) >> (n)) | ((x) << (32 - (n))))

static void sha_compress(uint32_t s[8], const uint8_t* p) {
    uint32_t w[64];
    for (int i = 0; i < 16; ++i)
        w[i] = ((uint32_t)p[4 * i] << 24) | ((uint32_t)p[4 * i + 1] << 16) |
               ((uint32_t)p[4 * i + 2] << 8) | p[4 * i + 3];
    for (int i = 16; i < 64; ++i) {
        uint32_t s0 = ROR(w[i - 15], 7) ^ ROR(w[i - 15], 18) ^ (w[i - 15] >> 3);
        uint32_t s1 = ROR(w[i - 2], 17) ^ ROR(w[i - 2], 19) ^ (w[i - 2] >> 10);
        w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = s[0], b = s[1], c = s[2], d = s[3], e = s[4], f = s[5], g = s[6], h = s[7];
    for (int i = 0; i < 64; ++i) {
        uint32_t t1 = h + (ROR(e, 6) ^ ROR(e, 11) ^ ROR(e, 25)) + ((e & f) ^ (~e & g)) + K256[i] + w[i];
        uint32_t t2 = (ROR(a, 2) ^ ROR(a, 13) ^ ROR(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
        h = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    s[0] += a; s[1] += b; s[2] += c; s[3] += d; s[4] += e; s[5] += f; s[6] += g; s[7] += h;
}

void or_sha_init(or_sha_ctx* c) {
    static const uint32_t iv[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                                   0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    memcpy(c->h, iv, sizeof iv);
    c->total = 0;
    c->n = 0;
}

void or_sha_update(or_sha_ctx* c, const uint8_t* d, size_t len) {
    c->total += len;
    while (len) {
        size_t take = 64 - c->n;
        if (take > len) take = len;
        memcpy(c->buf + c->n, d, take);
        c->n += take;
        d += take;
        len -= take;
        if (c->n == 64) {
            sha_compress(c->h, c->buf);
            c->n = 0;
        }
    }
}

void or_sha_final(or_sha_ctx* c, uint8_t out[32]) {
    uint64_t bits = c->total * 8;
    uint8_t pad = 0x80;
    uint8_t zero = 0;
    or_sha_update(c, &pad, 1);
    while (c->n != 56) or_sha_update(c, &zero, 1);
    uint8_t lb[8];
    for (int i = 0; i < 8; ++i) lb[i] = (uint8_t)(bits >> (56 - 8 * i));
    or_sha_update(c, lb, 8);
    for (int i = 0; i < 8; ++i) {
        out[4 * i] = (uint8_t)(c->h[i] >> 24);
        out[4 * i + 1] = (uint8_t)(c->h[i] >> 16);
        out[4 * i + 2] = (uint8_t)(c->h[i] >> 8);
        out[4 * i + 3] = (uint8_t)c->h[i];
    }
}

void or_sha256(const uint8_t* m, uint64_t len, uint8_t out[32]) {
    or_sha_ctx c;
    or_sha_init(&c);
    or_sha_update(&c, m, len);
    or_sha_final(&c, out);
}

static void put_u32be(uint8_t* p, uint32_t v) {
    p[0] = (uint8_t)(v >> 24); p[1] = (uint8_t)(v >> 16); p[2] = (uint8_t)(v >> 8); p[3] = (uint8_t)v;
}
static void put_u64be(uint8_t* p, uint64_t v) {
    for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(v >> (56 - 8 * i));
}

/* ------------------------------------------------------------ HMAC / HKDF --
 * HmacCtx: keys > 64 B are hashed, else zero-padded; ipad 0x36 / opad 0x5c
 * (src/hkdf.cpp:12-39). */
typedef struct {
    or_sha_ctx inner;
    uint8_t opad[64];
} hmac_ctx;

static void hmac_init(hmac_ctx* h, const uint8_t* key, uint64_t klen) {
    uint8_t kb[64] = {0}, ipad[64];
    if (klen > 64) or_sha256(key, klen, kb);
    else if (klen) memcpy(kb, key, klen);
    for (int i = 0; i < 64; ++i) {
        ipad[i] = kb[i] ^ 0x36;
        h->opad[i] = kb[i] ^ 0x5c;
    }
    or_sha_init(&h->inner);
    or_sha_update(&h->inner, ipad, 64);
}

static void hmac_final(hmac_ctx* h, uint8_t out[32]) {
    uint8_t ih[32];
    or_sha_final(&h->inner, ih);
    or_sha_ctx o;
    or_sha_init(&o);
    or_sha_update(&o, h->opad, 64);
    or_sha_update(&o, ih, 32);
    or_sha_final(&o, out);
}

void or_hmac_sha256(const uint8_t* key, uint64_t klen, const uint8_t* msg, uint64_t mlen,
                    uint8_t out[32]) {
    hmac_ctx h;
    hmac_init(&h, key, klen);
    or_sha_update(&h.inner, msg, mlen);
    hmac_final(&h, out);
}

/* hkdf_extract (empty salt => 32 zero bytes, hkdf.cpp:56-62), hkdf_expand
 * (L <= 8160, T(i) = HMAC(prk, T(i-1) | info | i), hkdf.cpp:64-82). */
int or_hkdf_sha256(const uint8_t* ikm, uint64_t ikm_len, const uint8_t* salt, uint64_t salt_len,
                   const uint8_t* info, uint64_t info_len, uint8_t* out, uint64_t out_len) {
    static const uint8_t zero_salt[32] = {0};
    if (out_len > 255 * 32) return -1;
    uint8_t prk[32];
    if (salt_len == 0) or_hmac_sha256(zero_salt, 32, ikm, ikm_len, prk);
    else or_hmac_sha256(salt, salt_len, ikm, ikm_len, prk);
    uint8_t t[32];
    size_t tlen = 0, done = 0;
    uint8_t ctr = 1;
    while (done < out_len) {
        hmac_ctx h;
        hmac_init(&h, prk, 32);
        or_sha_update(&h.inner, t, tlen);
        or_sha_update(&h.inner, info, info_len);
        or_sha_update(&h.inner, &ctr, 1);
        hmac_final(&h, t);
        ++ctr;
        tlen = 32;
        size_t take = out_len - done < 32 ? out_len - done : 32;
        memcpy(out + done, t, take);
        done += take;
    }
    return 0;
}

/* ---------------------------------------------------------------- crypto --*/
/* Rev::from_seed: SHA-256("rev-seed" | seed_be64) (crypto.cpp:28-33). */
void or_rev_from_seed(uint64_t seed, uint8_t out[32]) {
    uint8_t buf[16] = {'r', 'e', 'v', '-', 's', 'e', 'e', 'd'};
    put_u64be(buf + 8, seed);
    or_sha256(buf, 16, out);
}

/* Domain::encode: chain_id u16be | slot as 48-bit be (crypto.cpp:35-43). */
void or_domain_encode(uint16_t chain, uint64_t slot, uint8_t out[8]) {
    out[0] = (uint8_t)(chain >> 8);
    out[1] = (uint8_t)chain;
    for (int i = 0; i < 6; ++i) out[2 + i] = (uint8_t)(slot >> (40 - 8 * i));
}

/* id_commitment = SHA-256(REV | salt | domain) (crypto.cpp:115-122). */
void or_id_commitment(const uint8_t rev[32], const uint8_t salt[32], uint16_t chain, uint64_t slot,
                      uint8_t out[32]) {
    uint8_t m[72];
    memcpy(m, rev, 32);
    memcpy(m + 32, salt, 32);
    or_domain_encode(chain, slot, m + 64);
    or_sha256(m, 72, out);
}

/* derive_attest_key = HKDF(ikm=REV, salt=domain(8), info="ACEGF-V1-MEMPOOL-ATTEST", 32)
 * (crypto.cpp:78-89,124-127; info string crypto.hpp:19). */
static const char kInfoAttest[] = "ACEGF-V1-MEMPOOL-ATTEST";
void or_derive_attest_key(const uint8_t rev[32], const uint8_t dom8[8], uint8_t out[32]) {
    or_hkdf_sha256(rev, 32, dom8, 8, (const uint8_t*)kInfoAttest, sizeof(kInfoAttest) - 1, out, 32);
}

static void credential(const uint8_t key[32], const uint8_t obj_hash[32], const uint8_t dom8[8],
                       uint8_t out[32]) {
    uint8_t m[40];
    memcpy(m, obj_hash, 32);
    memcpy(m + 32, dom8, 8);
    or_hmac_sha256(key, 32, m, 40, out);
}

/* generate_attestation (crypto.cpp:129-139): obj_hash = SHA(payload);
 * credential = HMAC(attest_key, obj_hash | domain); encoded per :56-65. */
void or_generate_attestation(const uint8_t rev[32], const uint8_t* payload, uint64_t len,
                             const uint8_t dom8[8], const uint8_t id_com[32], uint8_t out[104]) {
    uint8_t key[32];
    or_sha256(payload, len, out);
    memcpy(out + 32, id_com, 32);
    memcpy(out + 64, dom8, 8);
    or_derive_attest_key(rev, dom8, key);
    credential(key, out, dom8, out + 72);
}

static int ct_eq32(const uint8_t* a, const uint8_t* b) {
    uint8_t d = 0;
    for (int i = 0; i < 32; ++i) d |= a[i] ^ b[i];
    return d == 0;
}

/* verify_attestation_full (crypto.cpp:141-154): payload check first
 * (1 = PayloadMismatch), then credential (2 = CredentialMismatch), else 0 = Accept. */
int or_verify_attestation_full(const uint8_t att[104], const uint8_t* payload, uint64_t len,
                               const uint8_t rev[32]) {
    uint8_t h[32], key[32], cred[32];
    or_sha256(payload, len, h);
    if (!ct_eq32(h, att)) return 1;
    or_derive_attest_key(rev, att + 64, key);
    credential(key, att, att + 64, cred);
    if (!ct_eq32(cred, att + 72)) return 2;
    return 0;
}

/* --------------------------------------------------------- tiny thread pool */
typedef struct {
    void (*fn)(void*, uint64_t);
    void* arg;
    uint64_t begin, end;
} par_job;

static void* par_worker(void* p) {
    par_job* j = (par_job*)p;
    for (uint64_t i = j->begin; i < j->end; ++i) j->fn(j->arg, i);
    return NULL;
}

static void parallel_for(uint64_t n, int threads, void (*fn)(void*, uint64_t), void* arg) {
    if (threads <= 1 || n < 64) {
        for (uint64_t i = 0; i < n; ++i) fn(arg, i);
        return;
    }
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    par_job jobs[256];
    for (int t = 0; t < threads; ++t) {
        jobs[t].fn = fn;
        jobs[t].arg = arg;
        jobs[t].begin = n * (uint64_t)t / (uint64_t)threads;
        jobs[t].end = n * (uint64_t)(t + 1) / (uint64_t)threads;
        pthread_create(&tid[t], NULL, par_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
}

typedef struct {
    const uint8_t *payloads, *atts, *revs;
    const uint64_t* offs;
    const uint32_t* rev_index;
    uint8_t* codes;
} att_batch;

static void att_one(void* a, uint64_t i) {
    att_batch* b = (att_batch*)a;
    b->codes[i] = (uint8_t)or_verify_attestation_full(b->atts + 104 * i, b->payloads + b->offs[i],
                                                      b->offs[i + 1] - b->offs[i],
                                                      b->revs + 32ull * b->rev_index[i]);
}

void or_verify_attestations_batch(const uint8_t* payloads, const uint64_t* offs,
                                  const uint8_t* atts, uint32_t n, const uint8_t* revs,
                                  const uint32_t* rev_index, uint8_t* codes, int threads) {
    att_batch b = {payloads, atts, revs, offs, rev_index, codes};
    parallel_for(n, threads, att_one, &b);
}

/* ------------------------------------------------------------------ wire --*/
/* make_transfer_payload (wire.cpp:59-72) via TxPayload::encode (:7-22):
 * version 1 | nonce | 2 accounts (writable) | program 0 | recent | instr(11). */
void or_make_transfer_payload(const uint8_t from[32], const uint8_t to[32], uint64_t amount,
                              uint64_t nonce, const uint8_t recent[32], uint8_t out[154]) {
    uint8_t* p = out;
    p[0] = 0; p[1] = 1; p += 2;
    put_u64be(p, nonce); p += 8;
    *p++ = 2;
    memcpy(p, from, 32); p += 32; *p++ = 1;
    memcpy(p, to, 32); p += 32; *p++ = 1;
    memset(p, 0, 32); p += 32;
    memcpy(p, recent, 32); p += 32;
    p[0] = 0; p[1] = 11; p += 2;
    p[0] = 1; p[1] = 0; p[2] = 1;
    put_u64be(p + 3, amount);
}

/* block_hash = SHA-256(256-B header encoding) (wire.cpp:214-221). */
void or_block_hash(const uint8_t header[256], uint8_t out[32]) { or_sha256(header, 256, out); }

/* merkle_root (wire.cpp:223-255): leaf H(0x00|h), inner H(0x01|l|r), an odd
 * level duplicates its last node, empty => 32 zero bytes. */
void or_merkle_root(const uint8_t* leaves, uint64_t n, uint8_t out[32]) {
    if (n == 0) {
        memset(out, 0, 32);
        return;
    }
    uint8_t* lvl = (uint8_t*)malloc(32 * (n + 1));
    uint8_t m[65];
    for (uint64_t i = 0; i < n; ++i) {
        m[0] = 0x00;
        memcpy(m + 1, leaves + 32 * i, 32);
        or_sha256(m, 33, lvl + 32 * i);
    }
    while (n > 1) {
        if (n & 1) {
            memcpy(lvl + 32 * n, lvl + 32 * (n - 1), 32);
            ++n;
        }
        for (uint64_t i = 0; i < n / 2; ++i) {
            m[0] = 0x01;
            memcpy(m + 1, lvl + 64 * i, 64);
            or_sha256(m, 65, lvl + 32 * i);
        }
        n /= 2;
    }
    memcpy(out, lvl, 32);
    free(lvl);
}

/* ------------------------------------------------------------- phase 1a --*/
/* pipeline.cpp:20-42: payload binding first, then the registry probe
 * (std::set<Hash32>::count == binary search over the sorted ids), then the
 * domain window |slot - current| <= w, written without underflow. */
int or_attest_check_light(const uint8_t* payload, uint64_t len, const uint8_t att[104],
                          const uint8_t* registry, uint64_t n_reg, uint64_t current_slot,
                          uint64_t window_slots) {
    uint8_t h[32];
    or_sha256(payload, len, h);
    if (memcmp(h, att, 32) != 0) return 1;
    uint64_t lo = 0, hi = n_reg;
    int found = 0;
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        int c = memcmp(registry + 32 * mid, att + 32, 32);
        if (c == 0) {
            found = 1;
            break;
        }
        if (c < 0) lo = mid + 1;
        else hi = mid;
    }
    if (!found) return 2;
    uint64_t slot = 0;
    for (int i = 0; i < 6; ++i) slot = (slot << 8) | att[66 + i];  /* Domain: u16 chain | u48 slot */
    int fresh = slot <= current_slot + window_slots && current_slot <= slot + window_slots;
    return fresh ? 0 : 3;
}

void or_block_roots(const uint8_t* payloads, const uint64_t* offs, const uint8_t* atts,
                    uint64_t n, uint8_t tx_root[32], uint8_t att_root[32]) {
    uint8_t* lv = (uint8_t*)calloc(n ? n : 1, 32);
    for (uint64_t i = 0; i < n; ++i) or_sha256(payloads + offs[i], offs[i + 1] - offs[i], lv + 32 * i);
    or_merkle_root(lv, n, tx_root);
    for (uint64_t i = 0; i < n; ++i) or_sha256(atts + 104 * i, 104, lv + 32 * i);
    or_merkle_root(lv, n, att_root);
    free(lv);
}

/* ---------------------------------------------------------------- prover --*/
static const char kTagTx[] = "zk-tx-proof-v1";       /* prover.cpp:14 */
static const char kTagAgg[] = "zk-agg-proof-v1";     /* prover.cpp:15 */
static const char kTagPad[] = "witness-pad-v1";      /* prover.cpp:16 */
static const char kTagShare[] = "witness-share-v1";  /* prover.cpp:17 */
static const char kTagStream[] = "witness-stream-v1";/* prover.cpp:18 */

/* expand256 (prover.cpp:24-35): seed = SHA(tag | digest);
 * out[32c..32c+32) = SHA(seed | c_be32), c = 0..7. kind 0 = Tx tag, 1 = Agg tag. */
void or_expand256(int kind, const uint8_t digest[32], uint8_t out[256]) {
    const char* tag = kind ? kTagAgg : kTagTx;
    size_t tl = strlen(tag);
    uint8_t m[64], seed[32];
    memcpy(m, tag, tl);
    memcpy(m + tl, digest, 32);
    or_sha256(m, tl + 32, seed);
    for (uint32_t c = 0; c < 8; ++c) {
        memcpy(m, seed, 32);
        put_u32be(m + 32, c);
        or_sha256(m, 36, out + 32 * c);
    }
}

/* prove_public_inputs (prover.cpp:78-85): digest = SHA(id_com|tx_hash|domain|target|rp_com)
 * (:74-76), bytes = expand256(tx tag). */
void or_prove_public_inputs(const uint8_t pub160[160], uint8_t out[289]) {
    or_sha256(pub160, 160, out + 256);
    or_expand256(0, out + 256, out);
    out[288] = 0;
}

/* PublicInputs::for_tx (prover.cpp:65-72): id_com from the attestation,
 * tx_hash = SHA(payload), domain's 8 encoded bytes zero-padded to 32. */
static void public_inputs_for_tx(const uint8_t* payload, uint64_t len, const uint8_t att[104],
                                 uint8_t pub[160]) {
    memset(pub, 0, 160);
    memcpy(pub, att + 32, 32);
    or_sha256(payload, len, pub + 32);
    memcpy(pub + 64, att + 64, 8);
}

void or_prove_tx(const uint8_t* payload, uint64_t len, const uint8_t att[104], uint8_t out[289]) {
    uint8_t pub[160];
    public_inputs_for_tx(payload, len, att, pub);
    or_prove_public_inputs(pub, out);
}

/* verify_mock (prover.cpp:91-95). */
int or_verify_mock(const uint8_t p[289]) {
    uint8_t e[256];
    or_expand256(p[288] == 0 ? 0 : 1, p + 256, e);
    return memcmp(e, p, 256) == 0;
}

/* aggregate_pair (prover.cpp:97-104): digest = SHA(a.bytes | b.bytes). */
void or_aggregate_pair(const uint8_t a[289], const uint8_t b[289], uint8_t out[289]) {
    or_sha_ctx c;
    or_sha_init(&c);
    or_sha_update(&c, a, 256);
    or_sha_update(&c, b, 256);
    or_sha_final(&c, out + 256);
    or_expand256(1, out + 256, out);
    out[288] = 1;
}

/* aggregate_tree (prover.cpp:106-127): pairs (2i, 2i+1), odd last node
 * promoted unchanged, -1 on empty (std::invalid_argument). */
int or_aggregate_tree(const uint8_t* proofs, uint64_t n, uint8_t out[289], uint64_t* levels,
                      uint64_t* pairs) {
    if (n == 0) return -1;
    uint8_t* lvl = (uint8_t*)malloc(289 * n);
    memcpy(lvl, proofs, 289 * n);
    uint64_t lv = 0, po = 0;
    while (n > 1) {
        ++lv;
        uint64_t p = n / 2;
        for (uint64_t i = 0; i < p; ++i) {
            uint8_t tmp[289];
            or_aggregate_pair(lvl + 289 * (2 * i), lvl + 289 * (2 * i + 1), tmp);
            memcpy(lvl + 289 * i, tmp, 289);
        }
        if (n & 1) memmove(lvl + 289 * p, lvl + 289 * (n - 1), 289);
        po += p;
        n = p + (n & 1);
    }
    memcpy(out, lvl, 289);
    free(lvl);
    if (levels) *levels = lv;
    if (pairs) *pairs = po;
    return 0;
}

typedef struct {
    const uint8_t *payloads, *atts;
    const uint64_t* offs;
    uint8_t* proofs;
} leaf_batch;

static void leaf_one(void* a, uint64_t i) {
    leaf_batch* b = (leaf_batch*)a;
    or_prove_tx(b->payloads + b->offs[i], b->offs[i + 1] - b->offs[i], b->atts + 104 * i,
                b->proofs + 289 * i);
}

/* prove_block (prover.cpp:129-142); the empty block proves
 * PublicInputs{tx_hash = block_hash} with stats {0, 0}. */
int or_prove_block(const uint8_t* payloads, const uint64_t* offs, const uint8_t* atts, uint32_t n,
                   const uint8_t header[256], uint8_t out[289], uint64_t* levels,
                   uint64_t* pairs, int threads) {
    if (n == 0) {
        uint8_t pub[160] = {0};
        or_block_hash(header, pub + 32);
        or_prove_public_inputs(pub, out);
        if (levels) *levels = 0;
        if (pairs) *pairs = 0;
        return 0;
    }
    uint8_t* proofs = (uint8_t*)malloc(289ull * n);
    leaf_batch b = {payloads, atts, offs, proofs};
    parallel_for(n, threads, leaf_one, &b);
    int rc = or_aggregate_tree(proofs, n, out, levels, pairs);
    free(proofs);
    return rc;
}

/* build_finality_certificate (prover.cpp:144-156) encoded per wire.cpp:125-133:
 * block_hash | slot_be64 (header bytes 0..8) | proof bytes | merkle_root(id_coms). */
void or_build_fc(const uint8_t* atts, uint32_t n, const uint8_t header[256],
                 const uint8_t proof[289], uint8_t out[328]) {
    or_block_hash(header, out);
    memcpy(out + 32, header, 8);
    memcpy(out + 40, proof, 256);
    uint8_t* ids = (uint8_t*)malloc(32ull * (n ? n : 1));
    for (uint32_t i = 0; i < n; ++i) memcpy(ids + 32ull * i, atts + 104ull * i + 32, 32);
    or_merkle_root(ids, n, out + 296);
    free(ids);
}

/* verify_finality_certificate (prover.cpp:158-169): 0 Valid, 1 SlotMismatch,
 * 2 HashMismatch, 3 ProofMismatch (full recompute). */
int or_verify_fc(const uint8_t fc[328], const uint8_t* payloads, const uint64_t* offs,
                 const uint8_t* atts, uint32_t n, const uint8_t header[256], int threads) {
    if (memcmp(fc + 32, header, 8) != 0) return 1;
    uint8_t bh[32];
    or_block_hash(header, bh);
    if (memcmp(fc, bh, 32) != 0) return 2;
    uint8_t root[289], exp[328];
    or_prove_block(payloads, offs, atts, n, header, root, NULL, NULL, threads);
    or_build_fc(atts, n, header, root, exp);
    if (memcmp(exp + 40, fc + 40, 256) != 0) return 3;
    if (memcmp(exp + 296, fc + 296, 32) != 0) return 3;
    return 0;
}

/* ------------------------------------------------------------- witnesses --*/
/* keystream (prover.cpp:41-56): block c = SHA("witness-stream-v1" | key | c_be32). */
void or_keystream(const uint8_t key[32], uint64_t len, uint8_t* out) {
    size_t tl = strlen(kTagStream);
    uint8_t m[64], blk[32];
    memcpy(m, kTagStream, tl);
    memcpy(m + tl, key, 32);
    for (uint32_t c = 0; (uint64_t)c * 32 < len; ++c) {
        put_u32be(m + tl + 32, c);
        or_sha256(m, tl + 36, blk);
        uint64_t take = len - 32ull * c < 32 ? len - 32ull * c : 32;
        memcpy(out + 32ull * c, blk, take);
    }
}

/* build_witness (prover.cpp:181-188): key | keystream(SHA("witness-pad-v1"|key|tx_hash))[224]. */
void or_build_witness(const uint8_t key[32], const uint8_t tx_hash[32], uint8_t out[256]) {
    size_t tl = strlen(kTagPad);
    uint8_t m[128], seed[32];
    memcpy(out, key, 32);
    memcpy(m, kTagPad, tl);
    memcpy(m + tl, key, 32);
    memcpy(m + tl + 32, tx_hash, 32);
    or_sha256(m, tl + 64, seed);
    or_keystream(seed, 224, out + 32);
}

/* witness_matches_tx (prover.cpp:190-197): size 256 and
 * HMAC(w[0:32], obj_hash | domain) == credential. */
int or_witness_matches_tx(const uint8_t* w, uint64_t wlen, const uint8_t att[104]) {
    if (wlen != 256) return 0;
    uint8_t c[32];
    credential(w, att, att + 64, c);
    return ct_eq32(c, att + 72);
}

/* WitnessScheme (prover.cpp:199-264): t = (2n+2)/3; share j on validators
 * j .. j+(n-t) mod n; share value SHA("witness-share-v1"|master|tx_hash|j_be32). */
unsigned or_scheme_threshold(unsigned n) { return (2 * n + 2) / 3; }

uint64_t or_scheme_share_mask(unsigned n, unsigned v) {
    unsigned t = or_scheme_threshold(n);
    uint64_t mask = 0;
    for (unsigned j = 0; j < t; ++j) {
        unsigned delta = (v + n - j) % n;
        if (delta <= n - t) mask |= 1ull << j;
    }
    return mask;
}

void or_scheme_share_value(const uint8_t master[32], const uint8_t tx_hash[32], unsigned index,
                           uint8_t out[32]) {
    size_t tl = strlen(kTagShare);
    uint8_t m[128];
    memcpy(m, kTagShare, tl);
    memcpy(m + tl, master, 32);
    memcpy(m + tl + 32, tx_hash, 32);
    put_u32be(m + tl + 64, index);
    or_sha256(m, tl + 68, out);
}

static void xor_key(const uint8_t master[32], const uint8_t tx_hash[32], uint64_t mask,
                    uint8_t key[32]) {
    memset(key, 0, 32);
    for (unsigned j = 0; j < 64; ++j) {
        if (!(mask >> j & 1)) continue;
        uint8_t s[32];
        or_scheme_share_value(master, tx_hash, j, s);
        for (int i = 0; i < 32; ++i) key[i] ^= s[i];
    }
}

void or_scheme_encapsulate(unsigned n, const uint8_t master[32], const uint8_t tx_hash[32],
                           const uint8_t* w, uint64_t len, uint8_t* ct) {
    unsigned t = or_scheme_threshold(n);
    uint64_t mask = t >= 64 ? ~0ull : ((1ull << t) - 1);
    uint8_t key[32];
    xor_key(master, tx_hash, mask, key);
    uint8_t* ks = (uint8_t*)malloc(len + 32);
    or_keystream(key, len, ks);
    for (uint64_t i = 0; i < len; ++i) ct[i] = w[i] ^ ks[i];
    free(ks);
}

/* decrypt (prover.cpp:245-264): XOR of the share values the contributors cover. */
void or_scheme_decrypt(unsigned n, const uint8_t master[32], const uint8_t tx_hash[32],
                       const uint8_t* ct, uint64_t len, const unsigned* contributors,
                       unsigned n_contrib, uint8_t* out) {
    uint64_t covered = 0;
    for (unsigned i = 0; i < n_contrib; ++i) covered |= or_scheme_share_mask(n, contributors[i] % n);
    uint8_t key[32];
    xor_key(master, tx_hash, covered, key);
    uint8_t* ks = (uint8_t*)malloc(len + 32);
    or_keystream(key, len, ks);
    for (uint64_t i = 0; i < len; ++i) out[i] = ct[i] ^ ks[i];
    free(ks);
}
