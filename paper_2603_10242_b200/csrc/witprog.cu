// GPU witness generation for bit-level circuits (the ZK-ACE credential
// relation, zkace_circuit.py): the host compiles the circuit once into a
// straight-line "witness program" — one op per value slot, in the order the
// circuit builder created them — and every transaction runs it on the
// device: slot values are -1 / 0 / 1 (bits, and the Ch products that can be
// -1), 32-bit additions keep their full sum. The private variables of the
// assignment are slots (var_slot); the public inputs are the attestation's
// obj_hash / domain / credential packed as big-endian integers.
//
// Program encoding (4 x u32 per op): w0 = opcode << 24 | dst (slot, or the
// addition's ordinal for ADD), then up to three operands:
//   KEY  i          key bit i (MSB first within each byte)
//   MSG  i          message bit i of obj_hash || domain
//   AND  a b        a & b          XOR  a b      a ^ b
//   CHP  e f g      e (f - g)      CH   e f g    e ? f : g
//   MAJP a b c      a (b ^ c)      MAJ  a b c    majority
//   ADD  off cnt K  sum[dst] = sum_k slot[addtab[off + k]] 2^(k mod 32) + K
//   SUMBIT add k    bit k of sum[add]
#include <cuda_runtime.h>

#include <cstdint>

#include "bn254.cuh"
#include "witprog.cuh"

namespace ace_gpu {
namespace bn {
namespace {

enum : uint32_t { kKey = 1, kMsg, kAnd, kXor, kChp, kCh, kMajp, kMaj, kAdd, kSumbit };

// One thread per transaction walks the whole program in lockstep with its
// warp; slot s of transaction t lives at slots[s T + t] (interleaved), so a
// warp's slot reads and writes are one coalesced 32-B access each.
struct Slots {
    int8_t* p;
    uint32_t T;
    __device__ __forceinline__ int8_t& operator[](uint32_t s) const { return p[(uint64_t)s * T]; }
};
__global__ void witprog_kernel(const uint4* __restrict__ ops, uint64_t n_ops,
                               const uint32_t* __restrict__ addtab, uint32_t n_slots,
                               uint32_t n_adds, const uint8_t* keys, uint64_t key_stride,
                               const uint8_t* atts, uint32_t T, int8_t* slots, int64_t* sums) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    const Slots sl{slots + t, T};
    int64_t* su = sums + (uint64_t)t * n_adds;
    const uint8_t* key = keys + key_stride * t;
    const uint8_t* att = atts + 104ull * t;
    sl[0] = 0;
    sl[1] = 1;
    for (uint64_t i = 0; i < n_ops; ++i) {
        const uint4 op = ops[i];
        const uint32_t code = op.x >> 24, dst = op.x & 0xFFFFFFu;
        int v = 0;
        switch (code) {
            case kKey: v = (key[op.y >> 3] >> (7 - (op.y & 7))) & 1; break;
            case kMsg: {
                const uint32_t byte = op.y >> 3;  // obj_hash (att 0..31) || domain (att 64..71)
                v = (att[byte < 32 ? byte : 32 + byte] >> (7 - (op.y & 7))) & 1;
                break;
            }
            case kAnd: v = sl[op.y] & sl[op.z]; break;
            case kXor: v = sl[op.y] ^ sl[op.z]; break;
            case kChp: v = sl[op.y] * (sl[op.z] - sl[op.w]); break;
            case kCh: v = sl[op.y] ? sl[op.z] : sl[op.w]; break;
            case kMajp: v = sl[op.y] * (sl[op.z] ^ sl[op.w]); break;
            case kMaj: {
                const int a = sl[op.y], b = sl[op.z], c = sl[op.w];
                v = (a & b) ^ (a & c) ^ (b & c);
                break;
            }
            case kAdd: {
                int64_t s = op.w;
                for (uint32_t k = 0; k < op.z; ++k)
                    s += (int64_t)sl[addtab[op.y + k]] << (k & 31);
                su[dst] = s;
                continue;
            }
            case kSumbit: v = (int)((su[op.y] >> op.z) & 1); break;
            default: break;
        }
        sl[dst] = (int8_t)v;
    }
}

// Per chunk c of Tc transactions (assignment size 1 + 5 Tc + Tc P, chunks
// back to back): z_c[1 + 5 Tc + l P + i] = slot[var_slot[i]] of its
// transaction l (-1 -> r - 1); 32-B little-endian standard form.
__global__ void witprog_expand_kernel(const int8_t* slots, const uint32_t* var_slot, uint32_t P,
                                      uint32_t T, uint32_t Tc, uint8_t* z) {
    const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j >= (uint64_t)T * P) return;
    const uint64_t t = j / P, i = j - t * P;
    const uint64_t c = t / Tc, l = t - c * Tc, zc = 1 + 5ull * Tc + (uint64_t)Tc * P;
    const int v = slots[(uint64_t)var_slot[i] * T + t];
    uint32_t w[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) w[k] = v < 0 ? mod_limb<FrCfg>(k) - (k == 0 ? 1u : 0u) : 0u;
    if (v > 0) w[0] = 1;
    uint4* o = reinterpret_cast<uint4*>(z + 32ull * (c * zc + 1 + 5ull * Tc + l * P + i));
    o[0] = make_uint4(w[0], w[1], w[2], w[3]);
    o[1] = make_uint4(w[4], w[5], w[6], w[7]);
}

// Per chunk: z_c[0] = ONE and the five public inputs of each transaction:
// obj_hash[0:16], obj_hash[16:32], domain[0:8], credential[0:16],
// credential[16:32] as big-endian integers.
__global__ void witprog_pub_kernel(const uint8_t* atts, uint32_t T, uint32_t Tc, uint32_t P,
                                   uint8_t* z) {
    const uint32_t nch = (T + Tc - 1) / Tc;
    const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j >= (uint64_t)nch * (1 + 5 * Tc)) return;
    const uint64_t c = j / (1 + 5 * Tc), q = j - c * (1 + 5 * Tc);
    const uint64_t zc = 1 + 5ull * Tc + (uint64_t)Tc * P;
    uint8_t* o = z + 32ull * (c * zc + q);
    for (int k = 0; k < 32; ++k) o[k] = 0;
    if (q == 0) {
        o[0] = 1;  // ONE
        return;
    }
    const uint64_t t = c * Tc + (q - 1) / 5, f = (q - 1) % 5;
    if (t >= T) return;
    const uint8_t* a = atts + 104ull * t;
    const uint8_t* src = f == 0 ? a : f == 1 ? a + 16 : f == 2 ? a + 64 : f == 3 ? a + 72 : a + 88;
    const int len = f == 2 ? 8 : 16;
    for (int k = 0; k < len; ++k) o[k] = src[len - 1 - k];  // big-endian -> little-endian
}

inline unsigned grid(uint64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

void witprog_run(const WitProg& p, const uint8_t* keys, uint64_t key_stride, const uint8_t* atts,
                 uint32_t T, uint32_t Tc, int8_t* slots, int64_t* sums, uint8_t* z,
                 cudaStream_t s) {
    if (!T) return;
    witprog_kernel<<<grid(T, 64), 64, 0, s>>>(p.ops, p.n_ops, p.addtab, p.n_slots, p.n_adds, keys,
                                              key_stride, atts, T, slots, sums);
    const uint64_t nch = (T + Tc - 1) / Tc;
    witprog_pub_kernel<<<grid(nch * (1 + 5ull * Tc), 128), 128, 0, s>>>(atts, T, Tc, p.n_vars, z);
    witprog_expand_kernel<<<grid((uint64_t)T * p.n_vars, 256), 256, 0, s>>>(
        slots, p.var_slot, p.n_vars, T, Tc, z);
}

}  // namespace bn
}  // namespace ace_gpu
