// Pippenger MSM over BN254 G1 / G2 (msm.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace ace_gpu {
namespace bn {

constexpr int kMsmC = 16;                      // window bits
constexpr int kMsmWindows = 16;                // ceil(254 / 16), signed digits need no 17th
constexpr int kMsmBuckets = 1 << (kMsmC - 1);  // |digit| in 1..2^15
constexpr int kMsmSeg = 64;                    // max entries per chunk (one accumulating thread)

// Device scratch for one MSM size (grow-only, reused).
struct MsmScratch {
    uint32_t* hist = nullptr;      // kMsmBuckets + 1
    uint32_t* offs = nullptr;      // kMsmBuckets + 1
    uint32_t* coffs = nullptr;     // kMsmBuckets + 1 chunk offsets
    uint32_t* cursor = nullptr;    // kMsmBuckets
    uint32_t* sorted = nullptr;    // W * n entries
    uint8_t* partials = nullptr;   // 2 per segment, XYZZ records
    uint8_t* buckets = nullptr;    // kMsmBuckets XYZZ
    uint8_t* segsum = nullptr;     // reduction partials
    size_t cap_entries = 0;
    void release();
};

// group = 1 (G1, 64-B affine / 128-B XYZZ) or 2 (G2, 128-B affine / 256-B XYZZ).
// Bases: affine, Montgomery form, infinity = all-zero record.
// prepare: table[w*n + i] = 2^(16 w) * base[i] for w < 16 (affine, Montgomery).
int msm_prepare(int group, const uint8_t* bases, uint64_t n, uint8_t* table, cudaStream_t s);
// scalars: n x 32-B canonical little-endian (standard form). out: affine,
// Montgomery form (64 / 128 B).
int msm_run(int group, const uint8_t* table, uint64_t n, const uint8_t* scalars,
            MsmScratch& sc, uint8_t* out_affine, cudaStream_t s);

// Point format conversions (standard <-> Montgomery coordinates), in place.
void launch_points_convert(int group, uint8_t* pts, uint64_t n, int to_mont, cudaStream_t s);
void launch_fq_convert(uint8_t* elems, uint64_t n, int to_mont, cudaStream_t s);

}  // namespace bn
}  // namespace ace_gpu
