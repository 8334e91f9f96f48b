/* TEST INFRASTRUCTURE ONLY — CPU oracle for the BN254 / Groth16 additions.
 *
 * PARITY UNPINNED BY THE REFERENCE: the reference has no BN254, NTT, MSM or
 * Groth16 code ("Out of scope: real Groth16 proving ... BN254
 * pairings"). This is a from-scratch restatement of the
 * published algorithms (Montgomery multiplication, radix-2 Cooley-Tukey NTT,
 * Jacobian short-Weierstrass arithmetic for y^2 = x^3 + 3 over Fq and
 * y^2 = x^3 + 3/(9+u) over Fq2 = Fq[u]/(u^2+1), double-and-add / bucket MSM,
 * Groth16 [Groth 2016]) with BN254 constants checked in SURVEY Appendix C. It
 * is pinned by self-consistency known answers instead (tests/test_bn254_oracle.py):
 * curve equations, r*G = O, NTT vs O(n^2) DFT, iNTT(NTT(x)) = x, Fermat
 * inverses, known-discrete-log MSM, Groth16 with a known trapdoor.
 *
 * Encodings: field elements are 32-B little-endian canonical integers
 * (standard form, not Montgomery). G1 affine = x | y (64 B); G2 affine =
 * x.c0 | x.c1 | y.c0 | y.c1 (128 B); the point at infinity is all zeros.
 */
#ifndef BN254_ORACLE_H
#define BN254_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* field: 0 = Fq (base field p), 1 = Fr (scalar field r) */
void bn_mul(int field, const uint8_t* a, const uint8_t* b, uint8_t* out);
void bn_add(int field, const uint8_t* a, const uint8_t* b, uint8_t* out);
void bn_sub(int field, const uint8_t* a, const uint8_t* b, uint8_t* out);
void bn_inv(int field, const uint8_t* a, uint8_t* out);
void bn_pow(int field, const uint8_t* a, const uint8_t* e, uint8_t* out);
/* Batched elementwise ops over n elements (for GPU parity tests). op: 0 mul, 1 add, 2 sub, 3 sqr */
void bn_batch(int field, int op, const uint8_t* a, const uint8_t* b, uint64_t n, uint8_t* out);
/* Reduce arbitrary 32-B little-endian integers mod the field. */
void bn_reduce(int field, const uint8_t* a, uint64_t n, uint8_t* out);

/* Fr NTT, natural order in and out, in place over 2^logn elements.
 * omega = 5^((r-1)/2^logn); inverse scales by 1/n; coset multiplies input
 * a_i by g^i (g = 5) before the forward transform / output by g^-i after the
 * inverse one. threads: worker count. */
void bn_ntt(uint8_t* data, uint32_t logn, int inverse, int coset, int threads);
void bn_dft_naive(const uint8_t* in, uint32_t logn, int inverse, uint8_t* out);

/* G1 / G2 affine ops (group = 1 or 2). */
int bn_on_curve(int group, const uint8_t* p);
void bn_generator(int group, uint8_t* out);
void bn_point_add(int group, const uint8_t* a, const uint8_t* b, uint8_t* out);
void bn_point_double(int group, const uint8_t* a, uint8_t* out);
void bn_point_neg(int group, const uint8_t* a, uint8_t* out);
void bn_scalar_mul(int group, const uint8_t* p, const uint8_t* scalar, uint8_t* out);
/* Many independent scalar multiples out[i] = s[i] * base (fixed base), threads. */
void bn_fixed_base_muls(int group, const uint8_t* base, const uint8_t* scalars, uint64_t n,
                        uint8_t* out, int threads);
/* MSM sum_i s[i] * P[i] by straightforward bucket method (window 8), threads. */
void bn_msm(int group, const uint8_t* points, const uint8_t* scalars, uint64_t n, uint8_t* out,
            int threads);

#ifdef __cplusplus
}
#endif
#endif
