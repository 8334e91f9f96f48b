// Phase 1a on the GPU: the leader's structural
// admission check and block assembly, feeding the prover without taking the
// transactions back to the host.
//
//   attest_check_light (pipeline.cpp:20-42): payload binding
//     SHA-256(payload) == obj_hash, then the identity registry probe
//     (std::set<Hash32>::count, here a binary search over the sorted 32-B
//     commitments resident in HBM), then the domain window
//     |domain.slot - current_slot| <= window (PipelineConfig, pipeline.hpp:16-21).
//   block build (pipeline.cpp:132-145): order-preserving compaction of the
//     accepted transactions, header.tx_count, tx_merkle_root and
//     attest_merkle_root (wire.cpp:257-273).
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>

#include "mock_kernels.cuh"
#include "phase1.cuh"
#include "sha256.cuh"

namespace ace_gpu {
namespace {

constexpr int kT = 128;

__device__ __forceinline__ void load_be8_any(const uint8_t* p, uint32_t w[8]) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
        w[k] = (uint32_t(p[4 * k]) << 24) | (uint32_t(p[4 * k + 1]) << 16) |
               (uint32_t(p[4 * k + 2]) << 8) | uint32_t(p[4 * k + 3]);
}

// -1 / 0 / 1 lexicographic comparison of two 32-B strings held as BE words.
__device__ __forceinline__ int cmp8(const uint32_t a[8], const uint32_t b[8]) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (a[k] != b[k]) return a[k] < b[k] ? -1 : 1;
    return 0;
}

__global__ void __launch_bounds__(kT) light_check_kernel(
    const uint8_t* __restrict__ payloads, const uint64_t* __restrict__ offs,
    const uint8_t* __restrict__ atts, uint32_t n, const uint8_t* __restrict__ reg, uint64_t n_reg,
    uint64_t cur, uint64_t window, uint8_t* __restrict__ codes, uint8_t* __restrict__ tx_hashes) {
    const uint32_t i = blockIdx.x * kT + threadIdx.x;
    if (i >= n) return;
    const uint64_t o = offs[i];
    uint32_t h[8], obj[8];
    sha256_bytes(payloads, o, static_cast<uint32_t>(offs[i + 1] - o), h);
    if (tx_hashes) store_digest(tx_hashes + 32ull * i, h);
    const uint8_t* att = atts + 104ull * i;
    load_be8_any(att, obj);
    uint8_t code = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (h[k] != obj[k]) code = 1;  // PayloadBinding
    if (!code) {
        uint32_t id[8];
        load_be8_any(att + 32, id);
        uint64_t lo = 0, hi = n_reg;
        bool found = false;
        while (lo < hi) {
            const uint64_t mid = lo + (hi - lo) / 2;
            uint32_t r[8];
            load_be8_any(reg + 32 * mid, r);
            const int c = cmp8(r, id);
            if (c == 0) {
                found = true;
                break;
            }
            if (c < 0) lo = mid + 1;
            else hi = mid;
        }
        if (!found) {
            code = 2;  // UnknownIdentity
        } else {
            uint64_t slot = 0;
#pragma unroll
            for (int k = 0; k < 6; ++k) slot = (slot << 8) | att[66 + k];  // Domain: u16 | u48 BE
            const bool fresh = slot <= cur + window && cur <= slot + window;
            code = fresh ? 0 : 3;  // AcceptPendingProof / StaleDomain
        }
    }
    codes[i] = code;
}

__global__ void accept_flags_kernel(const uint64_t* offs, const uint8_t* codes, uint32_t n,
                                    uint32_t* flag, uint64_t* len) {
    const uint32_t i = blockIdx.x * kT + threadIdx.x;
    if (i > n) return;
    const bool ok = i < n && (!codes || codes[i] == 0);
    flag[i] = ok ? 1u : 0u;  // element n: 0, so the exclusive scan's last entry is the total
    len[i] = ok ? offs[i + 1] - offs[i] : 0;
}

// One warp per transaction: copy the accepted payload (byte-granular, the
// offsets are arbitrary) and the 104-B attestation to their compacted slots,
// and hash the attestation record (attest_merkle_root leaf).
__global__ void __launch_bounds__(kT) scatter_kernel(
    const uint8_t* __restrict__ payloads, const uint64_t* __restrict__ offs,
    const uint8_t* __restrict__ atts, uint32_t n, const uint32_t* __restrict__ fscan,
    const uint64_t* __restrict__ lscan, const uint8_t* __restrict__ tx_hashes,
    uint8_t* __restrict__ out_pay, uint64_t* __restrict__ out_offs, uint8_t* __restrict__ out_atts,
    uint8_t* __restrict__ out_txh, uint8_t* __restrict__ out_ath) {
    const uint32_t warp = (blockIdx.x * kT + threadIdx.x) / 32, lane = threadIdx.x & 31;
    if (warp >= n) return;
    const uint32_t i = warp;
    if (fscan[i + 1] == fscan[i]) return;  // rejected
    const uint32_t j = fscan[i];
    const uint64_t o = offs[i], len = offs[i + 1] - o, d = lscan[i];
    for (uint64_t k = lane; k < len; k += 32) out_pay[d + k] = payloads[o + k];
    for (uint32_t k = lane; k < 104; k += 32) out_atts[104ull * j + k] = atts[104ull * i + k];
    if (lane < 8) {
        reinterpret_cast<uint32_t*>(out_txh + 32ull * j)[lane] =
            reinterpret_cast<const uint32_t*>(tx_hashes + 32ull * i)[lane];
    }
    if (lane == 0) {
        out_offs[j] = d;
        uint32_t h[8];
        sha256_bytes(atts, 104ull * i, 104, h);
        store_digest(out_ath + 32ull * j, h);
    }
}

__global__ void header_kernel(const uint8_t* tmpl, const uint32_t* count, const uint64_t* total,
                              uint64_t* out_offs, const uint8_t* tx_root, const uint8_t* att_root,
                              uint8_t* out) {
    const uint32_t k = threadIdx.x;
    if (k >= 256) return;
    const uint32_t cnt = *count;
    if (k == 0) out_offs[cnt] = *total;  // offsets[n_accepted] = payload bytes
    uint8_t v = tmpl[k];
    if (k >= 72 && k < 104) v = cnt ? tx_root[k - 72] : 0;        // tx_merkle_root
    if (k >= 104 && k < 136) v = cnt ? att_root[k - 104] : 0;     // attest_merkle_root
    if (k >= 208 && k < 212) v = static_cast<uint8_t>(cnt >> (8 * (211 - k)));  // tx_count u32be
    out[k] = v;
}

inline uint32_t grid(uint64_t n, int t = kT) { return static_cast<uint32_t>((n + t - 1) / t); }

}  // namespace

void launch_light_check(const uint8_t* payloads, const uint64_t* offs, const uint8_t* atts,
                        uint32_t n, const uint8_t* reg, uint64_t n_reg, uint64_t cur,
                        uint64_t window, uint8_t* codes, uint8_t* tx_hashes, cudaStream_t s) {
    if (n)
        light_check_kernel<<<grid(n), kT, 0, s>>>(payloads, offs, atts, n, reg, n_reg, cur, window,
                                                  codes, tx_hashes);
}

size_t compact_scratch_bytes(uint32_t n) {
    size_t a = 0, b = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, a, static_cast<uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr), n + 1);
    cub::DeviceScan::ExclusiveSum(nullptr, b, static_cast<uint64_t*>(nullptr),
                                  static_cast<uint64_t*>(nullptr), n + 1);
    const size_t arrays = (4 + 4 + 8 + 8) * size_t(n + 1);
    return arrays + (a > b ? a : b) + 256;
}

cudaError_t launch_compact(const uint8_t* payloads, const uint64_t* offs, const uint8_t* atts,
                           uint32_t n, const uint8_t* codes, const uint8_t* tx_hashes,
                           uint8_t* scratch, uint8_t* out_pay, uint64_t* out_offs,
                           uint8_t* out_atts, uint8_t* out_txh, uint8_t* out_ath,
                           uint32_t** d_count, uint64_t** d_total, cudaStream_t s) {
    uint32_t* flag = reinterpret_cast<uint32_t*>(scratch);
    uint32_t* fscan = flag + (n + 1);
    uint64_t* len = reinterpret_cast<uint64_t*>(fscan + (n + 1));  // 8(n+1) B in: aligned
    uint64_t* lscan = len + (n + 1);
    uint8_t* tmp = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(lscan + (n + 1)) + 255) & ~uintptr_t(255));
    size_t a = 0, b = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, a, flag, fscan, n + 1, s);
    cub::DeviceScan::ExclusiveSum(nullptr, b, len, lscan, n + 1, s);
    accept_flags_kernel<<<grid(n + 1), kT, 0, s>>>(offs, codes, n, flag, len);
    cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, a, flag, fscan, n + 1, s);
    if (e != cudaSuccess) return e;
    e = cub::DeviceScan::ExclusiveSum(tmp, b, len, lscan, n + 1, s);
    if (e != cudaSuccess) return e;
    if (n)
        scatter_kernel<<<grid(32ull * n), kT, 0, s>>>(payloads, offs, atts, n, fscan, lscan,
                                                      tx_hashes, out_pay, out_offs, out_atts,
                                                      out_txh, out_ath);
    *d_count = fscan + n;
    *d_total = lscan + n;
    return cudaGetLastError();
}

void launch_header(const uint8_t* tmpl, const uint32_t* d_count, const uint64_t* d_total,
                   uint64_t* out_offs, const uint8_t* tx_root, const uint8_t* att_root,
                   uint8_t* out, cudaStream_t s) {
    header_kernel<<<1, 256, 0, s>>>(tmpl, d_count, d_total, out_offs, tx_root, att_root, out);
}

}  // namespace ace_gpu
