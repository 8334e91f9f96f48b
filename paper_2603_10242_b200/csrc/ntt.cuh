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
    Fr *tw_full = nullptr, *twi_full = nullptr;  // w^e, w^-e for e < n (one product per twiddle);
                                                 // three-pass: w^(nC e), e < p q (pass B1)
    Fr *g_full = nullptr, *gi_post_full = nullptr;  // g^i, n^-1 g^-i for i < n (coset)
    Fr *g_lo = nullptr, *g_hi = nullptr, *gi_post_lo = nullptr, *gi_post_hi = nullptr;
    // three-pass sizes (L > kNttTwoPassMax): n = nC * p * q; sub-DFT roots of
    // the q- and p-point passes (the nC-point pass uses w_c)
    int LC = 0, LP = 0, LQ = 0;
    Fr *w_q = nullptr, *wi_q = nullptr, *w_p = nullptr, *wi_p = nullptr;
    void release();
};

// Mixed radix N = 3 * 2^k (k <= kNtt3MaxLog): a 3-point DFT over three
// 2^k-point NTTs (four-step with n1 = 3): de-interleave (x[i1 + 3 i2] ->
// Y_i1[i2], coset scale fused), the sub-NTTs (the 2^k tables), then per k2
// the twiddles w_N^(i1 k2) and the 3-point DFT into natural order (inverse
// and coset scales fused). Groth16 domains of 3 * 2^b points cut the padding
// of m just above a power of two (a paper-size chunk: 1.57 M vs 2.10 M).
constexpr int kNtt3MaxLog = 26;
struct Ntt3Tables {
    int k = -1, S = 0;       // N = 3 * 2^k; split tables at S bits
    Fr* consts = nullptr;    // w_N, w_N^-1, w3, w3^-1, 3^-1, g, g^-1
    Fr *wn_lo = nullptr, *wn_hi = nullptr, *wni_lo = nullptr, *wni_hi = nullptr;  // w_N^(+-e), e < 2^k
    Fr *g_lo = nullptr, *g_hi = nullptr, *gi_lo = nullptr, *gi_hi = nullptr;      // g^(+-i), i < N
    void release();
};
int ntt3_tables(Ntt3Tables& t, int k, cudaStream_t s);
// in/out may alias; ybuf: N x 32 B, scratch: 3 x 2^k x 32 B (the sub-NTTs').
// Data in Montgomery form; the 2^k tables tM must be built (ntt_tables).
int ntt3_run(const Ntt3Tables& t, const NttTables& tM, const uint8_t* in, uint8_t* out,
             uint8_t* ybuf, uint8_t* scratch, int inverse, int coset, cudaStream_t s);

int ntt_tables(NttTables& t, int L, cudaStream_t s);
// in/out may alias; scratch (batch x n x 32 B) is needed when L > kNttSingleMax.
// Data in Montgomery form. batch > 1 (contiguous transforms) for L <= kNttTwoPassMax.
int ntt_run(const NttTables& t, const uint8_t* in, uint8_t* out, uint8_t* scratch, int inverse,
            int coset, int batch, cudaStream_t s);
void launch_fr_convert(uint8_t* data, uint64_t n, int to_mont, cudaStream_t s);

}  // namespace bn
}  // namespace ace_gpu
