// Pippenger MSM over BN254 G1 / G2 (msm.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace ace_gpu {
namespace bn {

#ifndef ACEGPU_MSM_C
#define ACEGPU_MSM_C 17  // 15 windows x 17 = 255 bits exactly; c = 16/18/20 measured
#endif
constexpr int kMsmC = ACEGPU_MSM_C;                   // window bits
constexpr int kMsmWindows = (255 + kMsmC - 1) / kMsmC;  // 254-bit scalars + the signed-digit carry
constexpr int kMsmBuckets = 1 << (kMsmC - 1);         // |digit| in 1..2^(c-1)
#ifndef ACEGPU_MSM_SEG
#define ACEGPU_MSM_SEG 64
#endif
constexpr int kMsmSeg = ACEGPU_MSM_SEG;               // sorted entries per accumulating thread
constexpr int kMsmKernels = 9;  // kernel launches per msm_run (2 of them in the CUB scan)
static_assert(kMsmC >= 12 && kMsmC <= 24, "window bits");

// Device scratch for one MSM size (grow-only, reused).
struct MsmScratch {
    uint32_t* hist = nullptr;      // kMsmBuckets + 1
    uint32_t* offs = nullptr;      // kMsmBuckets + 1
    uint32_t* cursor = nullptr;    // kMsmBuckets
    uint32_t* sorted = nullptr;    // W * n entries
    uint8_t* partials = nullptr;   // 2 per accumulation segment, XYZZ records
    uint8_t* buckets = nullptr;    // kMsmBuckets XYZZ
    uint8_t* segsum = nullptr;     // reduction partials (one per CTA)
    uint32_t* heavy = nullptr;     // [count, bucket ids] of buckets spanning many segments
    uint8_t* heavy_part = nullptr; // per-slice sums of the heavy buckets (XYZZ records)
    void* scan_tmp = nullptr;      // CUB scan temporary storage
    uint8_t* aff_pts[2] = {nullptr, nullptr};     // batch-affine levels (G1): points
    uint32_t* aff_offs[2] = {nullptr, nullptr};   // and bucket offsets, ping-pong
    uint32_t* aff_cnt = nullptr;
    uint64_t aff_cap = 0;
    uint32_t* keys = nullptr;      // large variable-base sorts: window-major digit keys
    uint64_t keys_cap = 0;
    uint8_t* win = nullptr;        // variable base: window sums per sub-range (affine)
    uint64_t win_cap = 0;
    uint64_t cap_buckets = 0;      // buckets the hist / offs / buckets arrays hold
    size_t scan_bytes = 0;
    size_t cap_entries = 0;
    uint64_t cap_segs = 0;         // accumulation segments the partials hold
    void release();
};

// group = 1 (G1, 64-B affine / 128-B XYZZ) or 2 (G2, 128-B affine / 256-B XYZZ).
// Bases: affine, Montgomery form, infinity = all-zero record.
// prepare: table[w*n + i] = 2^(c w) * base[i] for w < kMsmWindows (affine, Montgomery).
int msm_prepare(int group, const uint8_t* bases, uint64_t n, uint8_t* table, cudaStream_t s);
// scalars: n x 32-B canonical little-endian (standard form). out: affine,
// Montgomery form (64 / 128 B).
int msm_run(int group, const uint8_t* table, uint64_t n, const uint8_t* scalars,
            MsmScratch& sc, uint8_t* out_affine, cudaStream_t s);

// Variable-base form for bases too many to hold window tables of (a whole
// block's proving key: 2^28 H bases): table = the n bases themselves (affine,
// Montgomery), c = kMsmVbC-bit windows, one bucket set per window, sub-ranges
// of <= sub points (0 = kMsmVbSubMax) whose window sums are combined by
// Horner's rule at the end.
// Same result as msm_run on msm_prepare'd tables of the same bases.
#ifndef ACEGPU_MSM_VB_C
#define ACEGPU_MSM_VB_C 20  // 13 windows; the per-window 2^19-bucket reductions amortise over 2^26 points
#endif
constexpr int kMsmVbC = ACEGPU_MSM_VB_C;
constexpr uint64_t kMsmVbSubMax = 80ull << 20;  // 80 Mi points: W x sub bucket entries < 2^32
int msm_run_vb(int group, const uint8_t* bases, uint64_t n, const uint8_t* scalars,
               MsmScratch& sc, uint8_t* out, cudaStream_t s, uint64_t sub = 0);

// Fixed base in two phases, so tables over the same scalars can accumulate
// on different streams: msm_sort (digits into bucket order in sc), then
// msm_accumulate per table with its own scratch `acc` reading srt's sorted
// entries (srt must not be re-sorted until those accumulations are done).
struct MsmSorted {
    uint64_t n = 0, nseg = 0;
    uint32_t segsz = 0;
};
int msm_sort(uint64_t n, const uint8_t* scalars, MsmScratch& sc, MsmSorted& info,
             cudaStream_t s);
int msm_accumulate(int group, const uint8_t* table, const MsmScratch& srt, const MsmSorted& info,
                   MsmScratch& acc, uint8_t* out, cudaStream_t s);
// k tables (group 1 or 2 each) over the SAME scalars: one digit sort, then
// each table's accumulation and reduction (Groth16's A, B1, B2 share z).
int msm_run_multi(int k, const int* groups, const uint8_t* const* tables, uint64_t n,
                  const uint8_t* scalars, MsmScratch& sc, uint8_t* const* outs, cudaStream_t s);
int msm_run_vb_multi(int k, const int* groups, const uint8_t* const* bases, uint64_t n,
                     const uint8_t* scalars, MsmScratch& sc, uint8_t* const* outs, cudaStream_t s,
                     uint64_t sub = 0);

// Point format conversions (standard <-> Montgomery coordinates), in place.
void launch_points_convert(int group, uint8_t* pts, uint64_t n, int to_mont, cudaStream_t s);
void launch_fq_convert(uint8_t* elems, uint64_t n, int to_mont, cudaStream_t s);

}  // namespace bn
}  // namespace ace_gpu
