// GPU witness programs for bit-level circuits (witprog.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace ace_gpu {
namespace bn {

struct WitProg {
    const uint4* ops = nullptr;        // n_ops x (opcode << 24 | dst, a, b, c)
    uint64_t n_ops = 0;
    const uint32_t* addtab = nullptr;  // operand slots of the ADD ops
    const uint32_t* var_slot = nullptr;  // slot of each private variable (n_vars)
    uint32_t n_slots = 0, n_adds = 0, n_vars = 0;
};

// The assignments of ceil(T / Tc) chunks of Tc transactions, back to back,
// each ONE | 5 Tc public inputs | Tc x n_vars private values (32-B LE
// standard form; a short last chunk's missing transactions are left as is).
// keys: T attest keys (32 B each, key_stride apart); atts: T x 104 B.
// Scratch: slots T x n_slots bytes, sums T x n_adds int64.
void witprog_run(const WitProg& p, const uint8_t* keys, uint64_t key_stride, const uint8_t* atts,
                 uint32_t T, uint32_t Tc, int8_t* slots, int64_t* sums, uint8_t* z,
                 cudaStream_t s);

}  // namespace bn
}  // namespace ace_gpu
