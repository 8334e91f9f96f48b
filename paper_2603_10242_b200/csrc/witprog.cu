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
// addition's ordinal for ADD), then up to three operands (the host compiles
// slots to physical slots by liveness, acegpu_witprog_create):
//   KEY  i          key bit i (MSB first within each byte)
//   MSG  i          message bit i of obj_hash || domain
//   AND  a b        a & b          XOR  a b      a ^ b
//   CHP  e f g      e (f - g)      CH   e f g    e ? f : g
//   MAJP a b c      a (b ^ c)      MAJ  a b c    majority
//   ADD  off cnt K  sum[dst] = sum_k slot[addtab[off + k]] 2^(k mod 32) + K
//   SUMBIT add k    bit k of sum[add] (always the latest ADD)
#include <cuda_runtime.h>

#include <cstdint>

#include "bn254.cuh"
#include "witprog.cuh"

namespace ace_gpu {
namespace bn {
namespace {

enum : uint32_t { kKey = 1, kMsg, kAnd, kXor, kChp, kCh, kMajp, kMaj, kAdd, kSumbit };

// One warp per 32 transactions, one lane per transaction: the warp stages
// 32 ops (+ their emit targets) at a time in shared memory and runs them in
// lockstep; slot values live in shared memory as [physical slot][lane] bytes
// (a warp's access to one slot is 32 consecutive bytes, conflict-free); the
// key bits and the message bytes are staged per lane; the one live 32-bit
// sum stays in a register. A value that is a private variable is written to
// the assignment when it is produced (32-B standard form, -1 -> r - 1).
__device__ __forceinline__ void put_fr_small(uint8_t* o, int v) {
    uint32_t w[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) w[k] = v < 0 ? mod_limb<FrCfg>(k) - (k == 0 ? 1u : 0u) : 0u;
    if (v > 0) w[0] = 1;
    uint4* q = reinterpret_cast<uint4*>(o);
    q[0] = make_uint4(w[0], w[1], w[2], w[3]);
    q[1] = make_uint4(w[4], w[5], w[6], w[7]);
}

__global__ void __launch_bounds__(kWitprogTxs) witprog_kernel(
    const uint4* __restrict__ ops, const uint32_t* __restrict__ emit, uint64_t n_ops,
    const uint32_t* __restrict__ addtab, uint32_t n_phys, const uint8_t* keys,
    uint64_t key_stride, const uint8_t* atts, uint32_t T, uint32_t Tc, uint32_t P, uint8_t* z) {
    constexpr int W = kWitprogTxs;
    extern __shared__ __align__(16) uint8_t sm[];
    uint4* opbuf = reinterpret_cast<uint4*>(sm);                 // W ops
    uint32_t* embuf = reinterpret_cast<uint32_t*>(sm + 16 * W);  // W emit targets
    uint8_t* keys_s = sm + 20 * W;                               // W x 32 key bytes
    uint8_t* msg_s = keys_s + 32 * W;                            // W x 40 message bytes
    int8_t* slots = reinterpret_cast<int8_t*>(msg_s + 40 * W);   // n_phys x W
    const int lane = threadIdx.x;
    const uint32_t t = blockIdx.x * W + lane;
    const bool act = t < T;
    if (act) {
        const uint8_t* key = keys + key_stride * t;
        const uint8_t* att = atts + 104ull * t;
        for (int k = 0; k < 32; ++k) keys_s[32 * lane + k] = key[k];
        for (int k = 0; k < 40; ++k) msg_s[40 * lane + k] = att[k < 32 ? k : 32 + k];  // obj_hash | domain
    }
    slots[lane] = 0;
    slots[W + lane] = 1;
    uint8_t* zt = nullptr;
    if (act) {
        const uint64_t c = t / Tc, l = t - c * Tc, zc = 1 + 5ull * Tc + (uint64_t)Tc * P;
        zt = z + 32ull * (c * zc + 1 + 5ull * Tc + l * P);
    }
    __syncwarp();
    auto S = [&](uint32_t p) -> int { return slots[p * W + lane]; };
    int64_t sum = 0;
    for (uint64_t base = 0; base < n_ops; base += W) {
        const uint32_t cnt = n_ops - base < (uint64_t)W ? uint32_t(n_ops - base) : uint32_t(W);
        if (lane < cnt) {
            opbuf[lane] = ops[base + lane];
            embuf[lane] = emit[base + lane];
        }
        __syncwarp();
        for (uint32_t j = 0; j < cnt; ++j) {
            const uint4 op = opbuf[j];
            const uint32_t code = op.x >> 24, dst = op.x & 0xFFFFFFu;
            int v = 0;
            switch (code) {
                case kKey: v = (keys_s[32 * lane + (op.y >> 3)] >> (7 - (op.y & 7))) & 1; break;
                case kMsg: v = (msg_s[40 * lane + (op.y >> 3)] >> (7 - (op.y & 7))) & 1; break;
                case kAnd: v = S(op.y) & S(op.z); break;
                case kXor: v = S(op.y) ^ S(op.z); break;
                case kChp: v = S(op.y) * (S(op.z) - S(op.w)); break;
                case kCh: v = S(op.y) ? S(op.z) : S(op.w); break;
                case kMajp: v = S(op.y) * (S(op.z) ^ S(op.w)); break;
                case kMaj: {
                    const int a = S(op.y), b = S(op.z), c = S(op.w);
                    v = (a & b) ^ (a & c) ^ (b & c);
                    break;
                }
                case kAdd: {
                    int64_t s = op.w;
#pragma unroll 8
                    for (uint32_t k = 0; k < op.z; ++k)
                        s += (int64_t)S(__ldg(&addtab[op.y + k])) << (k & 31);
                    sum = s;
                    continue;
                }
                case kSumbit: v = (int)((sum >> op.z) & 1); break;
                default: break;
            }
            slots[dst * W + lane] = (int8_t)v;
            const uint32_t e = embuf[j];
            if (e != 0xFFFFFFFFu && act) put_fr_small(zt + 32ull * e, v);
        }
        __syncwarp();
    }
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
                 uint32_t T, uint32_t Tc, uint8_t* z, cudaStream_t s) {
    if (!T) return;
    const size_t smem = (20 + 32 + 40) * kWitprogTxs + (size_t)p.n_phys * kWitprogTxs;
    cudaFuncSetAttribute(witprog_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    witprog_kernel<<<grid(T, kWitprogTxs), kWitprogTxs, smem, s>>>(
        p.ops, p.emit, p.n_ops, p.addtab, p.n_phys, keys, key_stride, atts, T, Tc, p.n_vars, z);
    const uint64_t nch = (T + Tc - 1) / Tc;
    witprog_pub_kernel<<<grid(nch * (1 + 5ull * Tc), 128), 128, 0, s>>>(atts, T, Tc, p.n_vars, z);
}

}  // namespace bn
}  // namespace ace_gpu
