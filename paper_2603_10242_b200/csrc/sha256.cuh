// SHA-256 (FIPS 180-4) for sm_100a: register-resident compression plus the
// message shapes of the ACE Prove path. Replaces the reference's scalar /
// SHA-NI / AVX2x8 engines (proj/src/sha256.cpp:104-141, sha256_shani.cpp:15-191,
// sha256_avx2.cpp:40-105): on the GPU one thread owns one message, so a warp is
// the 32-lane analogue of the AVX2 8-lane batch (sha256.cpp:290-323).
//
// Conventions: a digest is held as 8 big-endian-value words (st[0] is bytes
// 0..3 of the digest, MSB first). Memory stays in wire byte order; loads/stores
// swap with one PRMT per word.
#pragma once
#include <cstdint>

namespace ace_gpu {

__device__ __constant__ static const uint32_t kSha256IV[8] = {
    0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
    0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};

#define ACE_K256                                                                                  \
    {0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u,  \
     0xab1c5ed5u, 0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu,  \
     0x9bdc06a7u, 0xc19bf174u, 0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu,  \
     0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau, 0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u,  \
     0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u, 0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu,  \
     0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u, 0xa2bfe8a1u, 0xa81a664bu,  \
     0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u, 0x19a4c116u,  \
     0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,  \
     0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u,  \
     0xc67178f2u}

__device__ __forceinline__ uint32_t rotr32(uint32_t x, int n) { return __funnelshift_r(x, x, n); }

// Pipe balancing. A compression is ~16 ALU-only operations per round (SHF
// rotations, LOP3 for Sigma/Ch/Maj) plus ~9 additions; the integer ALU pipe
// and the FMA pipe each take one warp instruction per 2 cycles per SMSP, and
// ptxas puts most additions on the ALU (IADD3). Writing the additions as
// x * kOne + y, with a constant-bank multiplier ptxas cannot fold, issues
// them as IMAD on the otherwise idle FMA pipe (tools/sha_lat.cu: 14.1 ->
// 16.2 G compressions/s on B200; the ALU-only floor is ~18 G/s).
__device__ __constant__ static uint32_t kOne = 1;  // not const: must not fold
__device__ __forceinline__ uint32_t madd(uint32_t x, uint32_t y) { return x * kOne + y; }
// In situ the balanced form is NOT faster (bench, 100k block: device step
// 0.586 / 0.589 / 0.613 / 0.622 ms for ACE_SHA_BAL = 0 / 1 / 3 / 7): the leaf
// kernel runs ~5 warps per SMSP (80 registers, one wave) and the tree levels
// are latency chains, so IMAD's longer latency costs more than the ALU issue
// slots it frees. The product kernels therefore default to 0; the roofline
// peak (acegpu_sha256_peak) uses the balanced form, the best compression
// throughput measured on this GPU.
#ifndef ACE_SHA_BAL
#define ACE_SHA_BAL 0
#endif
// bit 0: schedule additions, bit 1: h + K + W (off the round's critical
// path), bit 2: the e / a updates (on it)
template <int BIT, int BAL = ACE_SHA_BAL>
__device__ __forceinline__ uint32_t add_b(uint32_t x, uint32_t y) {
    if constexpr ((BAL >> BIT) & 1) return madd(x, y);
    else return x + y;
}
__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

__device__ __forceinline__ void sha256_init(uint32_t s[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i] = kSha256IV[i];
}

// One compression. `w` is consumed (used as the rolling schedule window).
template <int BAL = ACE_SHA_BAL>
__device__ __forceinline__ void sha256_compress(uint32_t s[8], uint32_t w[16]) {
    constexpr uint32_t K[64] = ACE_K256;
    uint32_t a = s[0], b = s[1], c = s[2], d = s[3], e = s[4], f = s[5], g = s[6], h = s[7];
#pragma unroll
    for (int i = 0; i < 64; ++i) {
        uint32_t wi;
        if (i < 16) {
            wi = w[i];
        } else {
            uint32_t w15 = w[(i - 15) & 15], w2 = w[(i - 2) & 15];
            uint32_t s0 = rotr32(w15, 7) ^ rotr32(w15, 18) ^ (w15 >> 3);
            uint32_t s1 = rotr32(w2, 17) ^ rotr32(w2, 19) ^ (w2 >> 10);
            wi = w[i & 15] = add_b<0, BAL>(w[i & 15] + s0, w[(i - 7) & 15] + s1);
        }
        uint32_t S1 = rotr32(e, 6) ^ rotr32(e, 11) ^ rotr32(e, 25);
        uint32_t ch = (e & f) ^ (~e & g);
        uint32_t t1 = add_b<1, BAL>(h, K[i] + wi) + S1 + ch;
        uint32_t S0 = rotr32(a, 2) ^ rotr32(a, 13) ^ rotr32(a, 22);
        uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        h = g;
        g = f;
        f = e;
        e = add_b<2, BAL>(d, t1);
        d = c;
        c = b;
        b = a;
        a = add_b<2, BAL>(t1, S0 + mj);
    }
    s[0] += a; s[1] += b; s[2] += c; s[3] += d;
    s[4] += e; s[5] += f; s[6] += g; s[7] += h;
}

// ---- compact compression for latency-bound code ----------------------------
// The fully unrolled compression is ~1,400 SASS instructions (~22 KB). In a
// kernel that runs a chain of compressions ONCE (the narrow tree levels, the
// key cache), every instruction line is an I-cache miss on first touch, so
// code size is latency. These variants keep 16 rounds per loop iteration
// (register roles return to identity every 8 rounds, window index = j) and
// read K from the constant bank: ~4x less code.
__device__ __constant__ static const uint32_t kK256c[64] = ACE_K256;

#define ACE_SHA_ROUND(i, wi)                                                 \
    do {                                                                     \
        uint32_t S1 = rotr32(e, 6) ^ rotr32(e, 11) ^ rotr32(e, 25);          \
        uint32_t ch = (e & f) ^ (~e & g);                                    \
        uint32_t t1 = add_b<1>(h, kK256c[i] + (wi)) + S1 + ch;               \
        uint32_t S0 = rotr32(a, 2) ^ rotr32(a, 13) ^ rotr32(a, 22);          \
        uint32_t mj = (a & b) ^ (a & c) ^ (b & c);                           \
        h = g; g = f; f = e; e = d + t1; d = c; c = b; b = a;                \
        a = t1 + S0 + mj;                                                    \
    } while (0)

__device__ __forceinline__ void sha256_compress_c(uint32_t s[8], uint32_t w[16]) {
    uint32_t a = s[0], b = s[1], c = s[2], d = s[3], e = s[4], f = s[5], g = s[6], h = s[7];
#pragma unroll
    for (int j = 0; j < 16; ++j) ACE_SHA_ROUND(j, w[j]);
#pragma unroll 1
    for (int i0 = 16; i0 < 64; i0 += 16) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            uint32_t w15 = w[(j + 1) & 15], w2 = w[(j + 14) & 15];
            uint32_t s0 = rotr32(w15, 7) ^ rotr32(w15, 18) ^ (w15 >> 3);
            uint32_t s1 = rotr32(w2, 17) ^ rotr32(w2, 19) ^ (w2 >> 10);
            w[j] = add_b<0>(w[j] + s0, w[(j + 9) & 15] + s1);
            ACE_SHA_ROUND(i0 + j, w[j]);
        }
    }
    s[0] += a; s[1] += b; s[2] += c; s[3] += d;
    s[4] += e; s[5] += f; s[6] += g; s[7] += h;
}

// Rounds only (W+K precomputed), compact.
template <class WK>
__device__ __forceinline__ void sha256_rounds_c(uint32_t s[8], WK wk) {
    uint32_t a = s[0], b = s[1], c = s[2], d = s[3], e = s[4], f = s[5], g = s[6], h = s[7];
#pragma unroll 1
    for (int i0 = 0; i0 < 64; i0 += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            uint32_t S1 = rotr32(e, 6) ^ rotr32(e, 11) ^ rotr32(e, 25);
            uint32_t ch = (e & f) ^ (~e & g);
            uint32_t t1 = add_b<1>(h, wk(i0 + j)) + S1 + ch;
            uint32_t S0 = rotr32(a, 2) ^ rotr32(a, 13) ^ rotr32(a, 22);
            uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
            h = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + S0 + mj;
        }
    }
    s[0] += a; s[1] += b; s[2] += c; s[3] += d;
    s[4] += e; s[5] += f; s[6] += g; s[7] += h;
}

// Compile-time dispatch: full unroll (throughput kernels) or compact.
template <bool COMPACT>
__device__ __forceinline__ void compress(uint32_t s[8], uint32_t w[16]) {
    if constexpr (COMPACT) sha256_compress_c(s, w);
    else sha256_compress(s, w);
}

// ---- split compression: message schedule (W[i] + K[i]) and rounds ---------
// Used where a compression's latency, not its issue cost, matters: sibling
// lanes precompute the schedules of independent blocks so that the serial
// chain only runs the rounds.
__device__ __forceinline__ void sha256_schedule_wk(const uint32_t w_in[16], uint32_t* wk,
                                                   int stride = 1) {
    constexpr uint32_t K[64] = ACE_K256;
    uint32_t w[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) w[i] = w_in[i];
#pragma unroll
    for (int i = 0; i < 64; ++i) {
        uint32_t wi;
        if (i < 16) {
            wi = w[i];
        } else {
            uint32_t w15 = w[(i - 15) & 15], w2 = w[(i - 2) & 15];
            uint32_t s0 = rotr32(w15, 7) ^ rotr32(w15, 18) ^ (w15 >> 3);
            uint32_t s1 = rotr32(w2, 17) ^ rotr32(w2, 19) ^ (w2 >> 10);
            wi = w[i & 15] = add_b<0>(w[i & 15] + s0, w[(i - 7) & 15] + s1);
        }
        wk[i * stride] = wi + K[i];
    }
}

// Rounds only, W[i] + K[i] supplied by `wk(i)`.
template <class WK>
__device__ __forceinline__ void sha256_rounds(uint32_t s[8], WK wk) {
    uint32_t a = s[0], b = s[1], c = s[2], d = s[3], e = s[4], f = s[5], g = s[6], h = s[7];
#pragma unroll
    for (int i = 0; i < 64; ++i) {
        uint32_t S1 = rotr32(e, 6) ^ rotr32(e, 11) ^ rotr32(e, 25);
        uint32_t ch = (e & f) ^ (~e & g);
        uint32_t t1 = add_b<1>(h, wk(i)) + S1 + ch;
        uint32_t S0 = rotr32(a, 2) ^ rotr32(a, 13) ^ rotr32(a, 22);
        uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        h = g;
        g = f;
        f = e;
        e = d + t1;
        d = c;
        c = b;
        b = a;
        a = t1 + S0 + mj;
    }
    s[0] += a; s[1] += b; s[2] += c; s[3] += d;
    s[4] += e; s[5] += f; s[6] += g; s[7] += h;
}

// Compile-time schedule (W + K) of the constant final padding block of a
// message of `bitlen` bits that is a multiple of 512 (0x80, zeros, length).
struct Wk64 {
    uint32_t v[64];
};
__host__ __device__ constexpr uint32_t ror_c(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }
__host__ __device__ constexpr Wk64 pad_block_wk(uint32_t bitlen) {
    constexpr uint32_t K[64] = ACE_K256;
    uint32_t w[64] = {};
    w[0] = 0x80000000u;
    w[15] = bitlen;
    for (int i = 16; i < 64; ++i) {
        const uint32_t s0 = ror_c(w[i - 15], 7) ^ ror_c(w[i - 15], 18) ^ (w[i - 15] >> 3);
        const uint32_t s1 = ror_c(w[i - 2], 17) ^ ror_c(w[i - 2], 19) ^ (w[i - 2] >> 10);
        w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    Wk64 r{};
    for (int i = 0; i < 64; ++i) r.v[i] = w[i] + K[i];
    return r;
}

// SHA-256 of `len` bytes starting at byte `start` of a 4-byte-aligned buffer
// (global or shared; generic addressing). Reads only aligned words that hold
// message bytes, so no padding of the buffer is required. Handles any length
// and any alignment: the reference's Hasher (sha256.cpp:215-257) semantics.
__device__ __forceinline__ void sha256_bytes(const uint8_t* __restrict__ base, uint64_t start,
                                             uint32_t len, uint32_t out[8]) {
    const uint32_t* p = reinterpret_cast<const uint32_t*>(base) + (start >> 2);
    const uint32_t sh = static_cast<uint32_t>(start & 3);
    const uint32_t sel = 0x0123u + sh * 0x1111u;
    const uint32_t lim = len + sh;  // aligned word i is needed iff 4*i < lim
    const uint32_t nb = (len + 9 + 63) >> 6;
    sha256_init(out);
    uint32_t prev = lim > 0 ? p[0] : 0u;
    for (uint32_t j = 0; j < nb; ++j) {
        uint32_t w[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const uint32_t idx = 16 * j + k + 1;
            const uint32_t nxt = (4 * idx < lim) ? p[idx] : 0u;
            uint32_t v = __byte_perm(prev, nxt, sel);
            prev = nxt;
            const uint32_t pos = 64 * j + 4 * k;
            if (pos + 4 > len) {
                if (pos >= len) {
                    v = (pos == len) ? 0x80000000u : 0u;
                } else {
                    const uint32_t keep = len - pos;  // 1..3
                    v = (v & (0xFFFFFFFFu << (32 - 8 * keep))) | (0x80000000u >> (8 * keep));
                }
            }
            w[k] = v;
        }
        if (j == nb - 1) {
            w[14] = len >> 29;
            w[15] = len << 3;
        }
        sha256_compress(out, w);
    }
}

// Store / load a digest (8 BE-value words) to / from wire byte order.
__device__ __forceinline__ void store_digest(uint8_t* dst, const uint32_t s[8]) {
    uint4* d = reinterpret_cast<uint4*>(dst);
    d[0] = make_uint4(bswap32(s[0]), bswap32(s[1]), bswap32(s[2]), bswap32(s[3]));
    d[1] = make_uint4(bswap32(s[4]), bswap32(s[5]), bswap32(s[6]), bswap32(s[7]));
}
__device__ __forceinline__ void load_digest(const uint8_t* src, uint32_t s[8]) {
    const uint4* q = reinterpret_cast<const uint4*>(src);
    uint4 a = q[0], b = q[1];
    s[0] = bswap32(a.x); s[1] = bswap32(a.y); s[2] = bswap32(a.z); s[3] = bswap32(a.w);
    s[4] = bswap32(b.x); s[5] = bswap32(b.y); s[6] = bswap32(b.z); s[7] = bswap32(b.w);
}

// --------------------------------------------------------------------------
// expand256 (prover.cpp:24-35): seed = SHA(tag | digest), then
// out[c] = SHA(seed | c_be32) for c = 0..7. Tags "zk-tx-proof-v1" (14 B) and
// "zk-agg-proof-v1" (15 B) (prover.cpp:14-15) are folded into constants.
// kind 0 = Tx, 1 = Aggregate.
template <bool C = false>
__device__ __forceinline__ void expand_seed(int kind, const uint32_t d[8], uint32_t seed[8]) {
    uint32_t w[16];
    if (kind == 0) {
        // "zk-tx-proof-v1": 7a 6b 2d 74 | 78 2d 70 72 | 6f 6f 66 2d | 76 31 ++ d
        w[0] = 0x7a6b2d74u; w[1] = 0x782d7072u; w[2] = 0x6f6f662du;
        w[3] = 0x76310000u | (d[0] >> 16);
#pragma unroll
        for (int k = 4; k < 11; ++k) w[k] = __funnelshift_l(d[k - 3], d[k - 4], 16);
        w[11] = (d[7] << 16) | 0x8000u;
        w[12] = 0; w[13] = 0; w[14] = 0; w[15] = 46 * 8;
    } else {
        // "zk-agg-proof-v1": 7a 6b 2d 61 | 67 67 2d 70 | 72 6f 6f 66 | 2d 76 31 ++ d
        w[0] = 0x7a6b2d61u; w[1] = 0x67672d70u; w[2] = 0x726f6f66u;
        w[3] = 0x2d763100u | (d[0] >> 24);
#pragma unroll
        for (int k = 4; k < 11; ++k) w[k] = __funnelshift_l(d[k - 3], d[k - 4], 8);
        w[11] = (d[7] << 8) | 0x80u;
        w[12] = 0; w[13] = 0; w[14] = 0; w[15] = 47 * 8;
    }
    sha256_init(seed);
    compress<C>(seed, w);
}

// One output block of expand256: SHA(seed | c_be32), a single 36-B message.
template <bool C = false>
__device__ __forceinline__ void expand_block(const uint32_t seed[8], uint32_t c, uint32_t o[8]) {
    uint32_t w[16];
#pragma unroll
    for (int k = 0; k < 8; ++k) w[k] = seed[k];
    w[8] = c;
    w[9] = 0x80000000u;
#pragma unroll
    for (int k = 10; k < 15; ++k) w[k] = 0;
    w[15] = 36 * 8;
    sha256_init(o);
    compress<C>(o, w);
}

// Full expand256 written to 256 B of wire-order bytes (16-B aligned).
__device__ __forceinline__ void expand256_store(int kind, const uint32_t d[8], uint8_t* out) {
    uint32_t seed[8];
    expand_seed(kind, d, seed);
#pragma unroll 1
    for (uint32_t c = 0; c < 8; ++c) {
        uint32_t o[8];
        expand_block(seed, c, o);
        store_digest(out + 32 * c, o);
    }
}

// PublicInputs::digest (prover.cpp:74-76) over the five 32-B words
// id_com | tx_hash | domain(8 B + zero pad) | target = 0 | rp_com = 0: 160 B,
// three compressions, the zero words constant-folded.
__device__ __forceinline__ void public_inputs_digest(const uint32_t id[8], const uint32_t tx[8],
                                                     uint32_t dom0, uint32_t dom1,
                                                     uint32_t out[8]) {
    uint32_t w[16];
    sha256_init(out);
#pragma unroll
    for (int k = 0; k < 8; ++k) { w[k] = id[k]; w[k + 8] = tx[k]; }
    sha256_compress(out, w);
    w[0] = dom0; w[1] = dom1;
#pragma unroll
    for (int k = 2; k < 16; ++k) w[k] = 0;
    sha256_compress(out, w);
#pragma unroll
    for (int k = 0; k < 16; ++k) w[k] = 0;
    w[8] = 0x80000000u;
    w[15] = 160 * 8;
    sha256_compress(out, w);
}

// General public-inputs digest (all five words given, for prove_public_inputs).
__device__ __forceinline__ void public_inputs_digest_full(const uint32_t pub[40], uint32_t out[8]) {
    uint32_t w[16];
    sha256_init(out);
#pragma unroll
    for (int b = 0; b < 2; ++b) {
#pragma unroll
        for (int k = 0; k < 16; ++k) w[k] = pub[16 * b + k];
        sha256_compress(out, w);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) w[k] = pub[32 + k];
    w[8] = 0x80000000u;
#pragma unroll
    for (int k = 9; k < 15; ++k) w[k] = 0;
    w[15] = 160 * 8;
    sha256_compress(out, w);
}

// ------------------------------------------------------------- HMAC-SHA256 --
// HmacCtx (hkdf.cpp:12-39) for keys <= 64 B given as BE words (key zero-padded
// to 64 B). Midstates after the ipad / opad blocks.
template <bool C = false>
__device__ __forceinline__ void hmac_midstates(const uint32_t key[16], uint32_t ist[8],
                                               uint32_t ost[8]) {
    uint32_t w[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) w[k] = key[k] ^ 0x36363636u;
    sha256_init(ist);
    compress<C>(ist, w);
#pragma unroll
    for (int k = 0; k < 16; ++k) w[k] = key[k] ^ 0x5c5c5c5cu;
    sha256_init(ost);
    compress<C>(ost, w);
}

// Outer hash: SHA(opad | inner) from the opad midstate: one compression.
template <bool C = false>
__device__ __forceinline__ void hmac_outer(const uint32_t ost[8], const uint32_t inner[8],
                                           uint32_t out[8]) {
    uint32_t w[16];
#pragma unroll
    for (int k = 0; k < 8; ++k) { out[k] = ost[k]; w[k] = inner[k]; }
    w[8] = 0x80000000u;
#pragma unroll
    for (int k = 9; k < 15; ++k) w[k] = 0;
    w[15] = (64 + 32) * 8;
    compress<C>(out, w);
}

// HMAC(key32, msg) for a one-block message tail `m` of mlen <= 55 bytes,
// already laid out as BE words with the 0x80 terminator; the length word is
// filled here. key32 is a 32-B key as 8 BE words.
template <bool C = false>
__device__ __forceinline__ void hmac32_short(const uint32_t key32[8], uint32_t m[16],
                                             uint32_t mlen, uint32_t out[8]) {
    uint32_t key[16], ist[8], ost[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { key[k] = key32[k]; key[k + 8] = 0; }
    hmac_midstates<C>(key, ist, ost);
    m[14] = 0;
    m[15] = (64 + mlen) * 8;
    compress<C>(ist, m);
    hmac_outer<C>(ost, ist, out);
}

// Credential HMAC(k, obj_hash | domain8) (crypto.cpp:129-139, :149-150;
// prover.cpp:190-197): a 40-B message.
__device__ __forceinline__ void credential_hmac(const uint32_t key[8], const uint32_t obj[8],
                                                uint32_t dom0, uint32_t dom1, uint32_t out[8]) {
    uint32_t m[16];
#pragma unroll
    for (int k = 0; k < 8; ++k) m[k] = obj[k];
    m[8] = dom0; m[9] = dom1; m[10] = 0x80000000u;
#pragma unroll
    for (int k = 11; k < 16; ++k) m[k] = 0;
    hmac32_short(key, m, 40, out);
}

// derive_attest_key (crypto.cpp:124-127 -> derive_key :78-89 -> hkdf_sha256):
// prk = HMAC(salt = domain8, ikm = REV32); okm = HMAC(prk, info | 0x01) with
// info = "ACEGF-V1-MEMPOOL-ATTEST" (23 B, crypto.hpp:19), L = 32.
template <bool C = false>
__device__ __forceinline__ void derive_attest_key(const uint32_t rev[8], uint32_t dom0,
                                                  uint32_t dom1, uint32_t out[8]) {
    uint32_t key[16], ist[8], ost[8], m[16], prk[8];
#pragma unroll
    for (int k = 0; k < 16; ++k) key[k] = 0;
    key[0] = dom0;
    key[1] = dom1;
    hmac_midstates<C>(key, ist, ost);
#pragma unroll
    for (int k = 0; k < 8; ++k) m[k] = rev[k];
    m[8] = 0x80000000u;
#pragma unroll
    for (int k = 9; k < 15; ++k) m[k] = 0;
    m[15] = (64 + 32) * 8;
    compress<C>(ist, m);
    hmac_outer<C>(ost, ist, prk);
    // "ACEGF-V1-MEMPOOL-ATTEST" | 0x01 | 0x80
    m[0] = 0x41434547u; m[1] = 0x462d5631u; m[2] = 0x2d4d454du; m[3] = 0x504f4f4cu;
    m[4] = 0x2d415454u; m[5] = 0x45535401u; m[6] = 0x80000000u;
#pragma unroll
    for (int k = 7; k < 16; ++k) m[k] = 0;
    hmac32_short<C>(prk, m, 24, out);
}

}  // namespace ace_gpu
