// GPU witness programs for bit-level circuits (witprog.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace ace_gpu {
namespace bn {

// A liveness-compiled program (acegpu_witprog_create compiles the builder's
// slot program): operands and destinations are PHYSICAL slots (0 = the
// constant 0, 1 = the constant 1; a slot is reused once its value is dead),
// emit[i] = the private variable op i produces (0xFFFFFFFF: none), and every
// SUMBIT reads the latest ADD's sum (one live sum).
struct WitProg {
    const uint4* ops = nullptr;        // n_ops x (opcode << 24 | dst, a, b, c)
    const uint32_t* emit = nullptr;    // n_ops
    uint64_t n_ops = 0;
    const uint32_t* addtab = nullptr;  // physical operand slots of the ADD ops
    uint32_t n_phys = 0, n_vars = 0;
};

constexpr int kWitprogTxs = 32;       // transactions per CTA (one warp, one lane each)
constexpr uint32_t kWitprogMaxPhys = 6000;  // shared-memory slots x 32 lanes <= ~190 KB

// The assignments of ceil(T / Tc) chunks of Tc transactions, back to back,
// each ONE | 5 Tc public inputs | Tc x n_vars private values (32-B LE
// standard form; a short last chunk's missing transactions are left as is).
// keys: T attest keys (32 B each, key_stride apart); atts: T x 104 B.
void witprog_run(const WitProg& p, const uint8_t* keys, uint64_t key_stride, const uint8_t* atts,
                 uint32_t T, uint32_t Tc, uint8_t* z, cudaStream_t s);

}  // namespace bn
}  // namespace ace_gpu
