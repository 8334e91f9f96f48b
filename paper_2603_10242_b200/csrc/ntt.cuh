// Fr NTT launchers (ntt.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "bn254.cuh"

namespace ace_gpu {
namespace bn {

constexpr int kNttSingleMax = 12;  // n <= 2^12: one CTA per transform
constexpr int kNttTwoPassMax = 22; // two passes (sub-DFTs <= 2^11 in 64 KB of smem, R = 1)
constexpr int kNttMaxLog = 28;     // three passes above 2^22 (a 100k-tx block's 2^28 domain)
constexpr int kNttR = 1;  // columns / rows per CTA: 1 -> 64 KB smem, 3 CTAs/SM (2^22 fwd 1.74 -> 1.60 ms vs R = 2)

// Device tables for one size (Montgomery form).
struct NttTables {
    int L = -1, L1 = 0, L2 = 0;
    Fr* consts = nullptr;  // w, w^-1, g, g^-1, n^-1
    Fr *w_a = nullptr, *wi_a = nullptr, *w_c = nullptr, *wi_c = nullptr;
    Fr *tw_lo = nullptr, *tw_hi = nullptr, *twi_lo = nullptr, *twi_hi = nullptr;
    Fr *tw_full = nullptr, *twi_full = nullptr;  // w^e, w^-e for e < n (one product per twiddle)
    Fr *g_full = nullptr, *gi_post_full = nullptr;  // g^i, n^-1 g^-i for i < n (coset)
    Fr *g_lo = nullptr, *g_hi = nullptr, *gi_post_lo = nullptr, *gi_post_hi = nullptr;
    // three-pass sizes (L > kNttTwoPassMax): n = nC * p * q; sub-DFT roots of
    // the q- and p-point passes (the nC-point pass uses w_c)
    int LC = 0, LP = 0, LQ = 0;
    Fr *w_q = nullptr, *wi_q = nullptr, *w_p = nullptr, *wi_p = nullptr;
    void release();
};

int ntt_tables(NttTables& t, int L, cudaStream_t s);
// in/out may alias; scratch (n x 32 B) is needed when L > kNttSingleMax.
// Data in Montgomery form. batch > 1 only for L <= kNttSingleMax.
int ntt_run(const NttTables& t, const uint8_t* in, uint8_t* out, uint8_t* scratch, int inverse,
            int coset, int batch, cudaStream_t s);
void launch_fr_convert(uint8_t* data, uint64_t n, int to_mont, cudaStream_t s);

}  // namespace bn
}  // namespace ace_gpu
