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
/* Groth16 domain rule: the smallest N >= m among 2^a and 3 * 2^b; *logk =
 * log2 of its power-of-two factor, *three = 1 for 3 * 2^b. */
uint64_t bn_g16_domain(uint64_t m, uint32_t* logk, int* three);
/* naive DFT of size 2^logk or 3 * 2^logk (coset shift 5, inverse scaled by 1/n) */
void bn_dft_naive_n(const uint8_t* in, uint32_t logk, int three, int inverse, int coset,
                    uint8_t* out);

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

/* ---- Groth16 over the synthetic ZK-ACE stand-in circuit (known trapdoor) ----
 * Shape: T txs, K >= 2 constraints per tx. Variables: 0 = ONE, 1..T = pub_t
 * (public), then per tx t: w_t, x_{t,0}, ..., x_{t,K-1} (private).
 * Rows: tx t, base R = t*K: row R: (w_t + pub_t) * 1 = x_{t,0};
 * row R+k (k = 1..K-1): (x_{t,k-1} + c_k) * (x_{t,k-1} + c_k) = x_{t,k};
 * rows T*K + i (i = 0..T): z_i * 0 = 0 for the public variables (ONE, pub).
 * c_k = LE(SHA-256("ace-g16-chain-v1" | k_be32)) mod r.
 * Given the trapdoor (tau, alpha, beta, gamma, delta) and r, s, returns the
 * discrete logs of the proof (A, B, C) in Fr and whether the Groth16
 * verification identity A*B = alpha*beta + sum_pub z_i(beta u_i + alpha v_i
 * + w_i) + C*delta holds (1) — the pairing check, in exponents. */
void bn_g16_chain_const(uint32_t k, uint8_t out32[32]);
int bn_g16_expected(uint32_t T, uint32_t K, const uint8_t* w, const uint8_t* pub,
                    const uint8_t* trapdoor5, const uint8_t* rs2, uint8_t* out_abc3,
                    int threads);

/* ---- optimal ate pairing (tower Fq2/Fq6/Fq12 over xi = 9+u) ----
 * Fq12 encoding: 12 x 32-B LE standard form, order c0.c0.c0, c0.c0.c1,
 * c0.c1.c0, ..., c1.c2.c1 (Fq12 = Fq6 + Fq6 w, Fq6 = Fq2 + Fq2 v + Fq2 v^2).
 * bn_pairing: prod_i e(P_i, Q_i) after the final exponentiation;
 * bn_pairing_check: 1 iff that product is 1. */
void bn_pairing(uint64_t n, const uint8_t* g1s, const uint8_t* g2s, uint8_t* out384);
int bn_pairing_check(uint64_t n, const uint8_t* g1s, const uint8_t* g2s);
void bn_f12_pow(const uint8_t* a384, const uint8_t* e32, uint8_t* out384);
/* Verifying key: alpha G1 (64) | beta G2 (128) | gamma G2 (128) | delta G2 (128)
 * | IC_0..IC_T (64 each) = 448 + 64 (T + 1) bytes. */
/* Fq12 unit ops for parity tests: 0 final exp, 1 easy part, 2 hard part,
 * 3/4/5 Frobenius p/p^2/p^3, 6 ^x, 7 inverse, 8 square, 9 Miller loop of
 * the (G1 | G2) pair in `in` (its value is only defined up to subfield
 * factors: compare after op 1). */
void bn_f12_op(int op, const uint8_t* in, uint8_t* out384);
int bn_g16_vk(uint32_t T, uint32_t K, const uint8_t* trapdoor5, uint8_t* out);
int bn_g16_verify(uint32_t T, const uint8_t* vk, const uint8_t* abc, const uint8_t* pubs);

#ifdef __cplusplus
}
#endif
#endif
