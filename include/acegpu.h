/* acegpu.h — the C ABI of the B200-native ACE Prove phase (libacegpu.so).
 *
 * Drop-in boundary. The reference has no FFI: its Prove phase is the C++
 * header proj/include/ace/prover.hpp (+ crypto.hpp:84-121, hkdf.hpp:9-18,
 * wire.hpp:85-116, sha256.hpp:50-58), statically linked. This ABI is what a
 * replacement prover.cpp binds (paper_2603_10242_b200/dropin/prover_b200.cpp,
 * see INTEGRATION.md), and what the Python mirror binds via ctypes. Plain
 * pointers and sizes; no C++ or torch types; status codes instead of
 * exceptions (the C++ shim maps ACEGPU_EINVAL -> std::invalid_argument).
 *
 * Flat layouts (identical in oracle/ace_oracle.h):
 *   payloads      concatenated payload bytes; tx i = payloads[offs[i], offs[i+1])
 *   offs          n+1 uint64 offsets (offs[0] normally 0)
 *   atts          n x 104 B Attestation::encode (crypto.cpp:56-65):
 *                 obj_hash(32) | id_com(32) | domain(8) | credential(32)
 *   header        256 B BlockHeader::encode (wire.cpp:74-98); slot = bytes 0..8 BE
 *   proof         289 B MockProof = bytes(256) | public_inputs_digest(32) | kind(1),
 *                 kind 0 = ProofKind::Tx, 1 = ProofKind::Aggregate (prover.hpp:33-43)
 *   fc            328 B FinalityCertificate::encode (wire.cpp:125-133)
 *   revs          table of 32-B REVs; rev_index[i] selects tx i's REV
 *   codes         AttestationCheck: 0 Accept, 1 PayloadMismatch, 2 CredentialMismatch
 *                 (crypto.hpp:84-88)
 *
 * Host-pointer functions ("*" without _dev) copy inputs host->device, run
 * and copy results back; they are synchronous and thread-safe per context
 * (calls on one context serialise, like ThreadPool::job_mu_ in
 * thread_pool.hpp:40-49). `_dev` functions take DEVICE pointers and a
 * cudaStream_t (as void*, used as given: NULL = CUDA's legacy default
 * stream), enqueue only, and never synchronise; the context workspace they
 * use is stream-ordered, so drive one context from one stream. Device byte
 * buffers must be 16-B aligned (cudaMalloc).
 */
#ifndef ACEGPU_H
#define ACEGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ACEGPU_OK 0
#define ACEGPU_EINVAL (-1) /* std::invalid_argument in the reference */
#define ACEGPU_ECUDA (-2)  /* CUDA error; acegpu_last_error() has the text */
#define ACEGPU_ENODEV (-3) /* no usable sm_100 device */

typedef struct acegpu_ctx acegpu_ctx;

/* Message of the last failing call on this thread. */
const char* acegpu_last_error(void);
/* Build identity, e.g. "acegpu sm_100a <git describe>". */
const char* acegpu_version(void);

/* One context per device (one process per GPU; torch.distributed plumbing). */
int acegpu_create(int device, acegpu_ctx** out);
void acegpu_destroy(acegpu_ctx* ctx);
/* Kernel launches issued by this context so far (telemetry / bench). */
uint64_t acegpu_launch_count(const acegpu_ctx* ctx);
/* Per-phase CUDA-event timing of the block pipeline (on the launching
 * stream): ms3 = {leaves(+attestation), tree levels, finalize} of the most
 * recent attest_prove_certify call. */
int acegpu_set_phase_timing(acegpu_ctx* ctx, int enable);
/* Host-input calls on blocks of >= 16,384 txs copy 16,384-tx segments on a
 * copy stream overlapped with the leaf kernels of earlier segments (on four
 * streams). Default on (100k block e2e 1.23 vs 1.31 ms); results identical. */
int acegpu_set_segmented(acegpu_ctx* ctx, int enable);
int acegpu_phase_times(acegpu_ctx* ctx, float* ms3);
/* Pinned host memory for fast host<->device copies. */
void* acegpu_host_alloc(size_t bytes);
void acegpu_host_free(void* p);

/* ---- SHA-256 (replaces sha256::digest / hash_batch_strided, sha256.hpp:42-58) */
int acegpu_sha256_varlen(acegpu_ctx* ctx, const uint8_t* data, const uint64_t* offs, uint64_t n,
                         uint8_t* out32);
int acegpu_sha256_strided(acegpu_ctx* ctx, const uint8_t* base, uint64_t stride, uint64_t msg_len,
                          uint64_t n, uint8_t* out32);

/* ---- mock prover (prover.hpp:52-79) --------------------------------------- */
/* prove_public_inputs (prover.cpp:78-85), batched: pubs = n x 160 B (5 words). */
int acegpu_prove_public_inputs(acegpu_ctx* ctx, const uint8_t* pubs160, uint64_t n,
                               uint8_t* out289);
/* prove_tx (prover.cpp:87-89), batched over a flat tx list. */
int acegpu_prove_txs(acegpu_ctx* ctx, const uint8_t* payloads, const uint64_t* offs,
                     const uint8_t* atts, uint64_t n, uint8_t* out289);
/* verify_mock (prover.cpp:91-95), batched: ok[i] in {0,1}. */
int acegpu_verify_mock(acegpu_ctx* ctx, const uint8_t* proofs289, uint64_t n, uint8_t* ok);
/* aggregate_pair (prover.cpp:97-104), batched: out[i] = pair(a[i], b[i]). */
int acegpu_aggregate_pairs(acegpu_ctx* ctx, const uint8_t* a289, const uint8_t* b289, uint64_t n,
                           uint8_t* out289);
/* aggregate_tree (prover.cpp:106-127). n == 0 -> ACEGPU_EINVAL. */
int acegpu_aggregate_tree(acegpu_ctx* ctx, const uint8_t* proofs289, uint64_t n, uint8_t* out289,
                          uint64_t* levels, uint64_t* pair_ops);
/* prove_block (prover.cpp:129-142). */
int acegpu_prove_block(acegpu_ctx* ctx, const uint8_t* payloads, const uint64_t* offs,
                       const uint8_t* atts, uint64_t n, const uint8_t* header256, uint8_t* out289,
                       uint64_t* levels, uint64_t* pair_ops);
/* build_finality_certificate (prover.cpp:144-156). */
int acegpu_build_fc(acegpu_ctx* ctx, const uint8_t* atts, uint64_t n, const uint8_t* header256,
                    const uint8_t* proof289, uint8_t* out_fc328);
/* verify_finality_certificate (prover.cpp:158-169): *out_check = FcCheck
 * (0 Valid, 1 SlotMismatch, 2 HashMismatch, 3 ProofMismatch). */
int acegpu_verify_fc(acegpu_ctx* ctx, const uint8_t* fc328, const uint8_t* payloads,
                     const uint64_t* offs, const uint8_t* atts, uint64_t n,
                     const uint8_t* header256, int* out_check);
/* merkle_root (wire.cpp:223-255); block_hash (wire.cpp:214-221). */
int acegpu_merkle_root(acegpu_ctx* ctx, const uint8_t* leaves32, uint64_t n, uint8_t* out32);
int acegpu_block_hash(acegpu_ctx* ctx, const uint8_t* header256, uint8_t* out32);

/* The Phase-2 step (ProverService::run body, prover.cpp:350-351) with the
 * batched full attestation check fused in (crypto.cpp:141-154): per tx
 * verdict into codes (NULL = skip attestation), the block's root proof and
 * its finality certificate. Either output may be NULL. With codes, the REV
 * table (n_revs x 32 B) and the per-tx rev_index are required; an index
 * >= n_revs is detected on the device and the call returns ACEGPU_EINVAL
 * after the run (outputs undefined). */
int acegpu_attest_prove_certify(acegpu_ctx* ctx, const uint8_t* payloads, const uint64_t* offs,
                                const uint8_t* atts, uint64_t n, const uint8_t* header256,
                                const uint8_t* revs, uint64_t n_revs, const uint32_t* rev_index,
                                uint8_t* codes, uint8_t* out289, uint8_t* out_fc328,
                                uint64_t* levels, uint64_t* pair_ops);
/* As acegpu_attest_prove_certify, enqueued on `stream` without waiting: the
 * H2D copies, the pipeline and the D2H of codes / proof / FC are
 * stream-ordered; the caller synchronises (event / stream) before reading
 * the outputs. Host buffers should be pinned (acegpu_host_alloc) for the
 * copies to be asynchronous, and must stay untouched until completion.
 * Successive async calls on one context must use the same stream (the
 * context's device workspace is reused in stream order). This is the
 * sustained-stream entry point (one call per block, ~20 launches). */
int acegpu_attest_prove_certify_async(acegpu_ctx* ctx, void* stream, const uint8_t* payloads,
                                      const uint64_t* offs, const uint8_t* atts, uint64_t n,
                                      const uint8_t* header, const uint8_t* revs,
                                      uint64_t n_revs, const uint32_t* rev_index, uint8_t* codes,
                                      uint8_t* out289, uint8_t* out328);
/* As acegpu_attest_prove_certify_async, replayed as a CUDA graph: the first
 * block of a shape (n, payload bytes, REV count, stream, outputs) runs with
 * plain launches and the same call is captured; later blocks of that shape
 * re-point the graph's copy nodes at their host buffers and launch it (one
 * graph launch instead of ~20 kernel launches + copies + events). `stream`
 * must not be NULL. Same buffer rules as the async call. */
int acegpu_attest_prove_certify_graph(acegpu_ctx* ctx, void* stream, const uint8_t* payloads,
                                      const uint64_t* offs, const uint8_t* atts, uint64_t n,
                                      const uint8_t* header, const uint8_t* revs,
                                      uint64_t n_revs, const uint32_t* rev_index, uint8_t* codes,
                                      uint8_t* out289, uint8_t* out328);
int acegpu_attest_prove_certify_dev(acegpu_ctx* ctx, void* stream, const uint8_t* d_payloads,
                                    const uint64_t* d_offs, const uint8_t* d_atts, uint64_t n,
                                    const uint8_t* d_header256, const uint8_t* d_revs,
                                    uint64_t n_revs, const uint32_t* d_rev_index,
                                    uint8_t* d_codes, uint8_t* d_out289, uint8_t* d_out_fc328);

/* ---- multi-GPU sharding (power-of-two aligned chunks) -------- */
/* Reduce one rank's shard (txs [start, start+n) of an n_total-tx block, start
 * a multiple of 2^log2_chunk) to its chunk roots: ceil(n / 2^log2_chunk)
 * proofs (289 B) and Merkle nodes (32 B) of level log2_chunk of the global
 * trees. The last block chunk's Merkle node is lifted by self-pairing when
 * n_total > 2^log2_chunk, so that chunk roots combine exactly like the global
 * tree (prover.cpp:112-124 promotes, wire.cpp:240 duplicates). */
int acegpu_shard_roots_dev(acegpu_ctx* ctx, void* stream, const uint8_t* d_payloads,
                           const uint64_t* d_offs, const uint8_t* d_atts, uint64_t n,
                           uint64_t n_total, uint32_t log2_chunk, const uint8_t* d_revs,
                           uint64_t n_revs, const uint32_t* d_rev_index, uint8_t* d_codes,
                           uint8_t* d_roots289, uint8_t* d_merkle32);
/* Combine the ordered chunk roots of all ranks into the block proof + FC. */
int acegpu_combine_roots_dev(acegpu_ctx* ctx, void* stream, const uint8_t* d_roots289,
                             const uint8_t* d_merkle32, uint64_t n_chunks, uint64_t n_total,
                             const uint8_t* d_header256, uint8_t* d_out289, uint8_t* d_out_fc328);

/* ---- attestation (crypto.hpp:113-118) ------------------------------------ */
int acegpu_attest_verify(acegpu_ctx* ctx, const uint8_t* payloads, const uint64_t* offs,
                         const uint8_t* atts, uint64_t n, const uint8_t* revs, uint64_t n_revs,
                         const uint32_t* rev_index, uint8_t* codes);
/* generate_attestation (crypto.cpp:129-139), batched: doms8 = n x 8-B Domain
 * encodings, id_coms = n x 32. */
int acegpu_attest_generate(acegpu_ctx* ctx, const uint8_t* payloads, const uint64_t* offs,
                           uint64_t n, const uint8_t* revs, uint64_t n_revs,
                           const uint32_t* rev_index, const uint8_t* doms8,
                           const uint8_t* id_coms, uint8_t* out104);
int acegpu_attest_generate_dev(acegpu_ctx* ctx, void* stream, const uint8_t* d_payloads,
                               const uint64_t* d_offs, uint64_t n, const uint8_t* d_revs,
                               const uint32_t* d_rev_index, const uint8_t* d_doms8,
                               const uint8_t* d_id_coms, uint8_t* d_out104);
/* derive_attest_key (crypto.cpp:124-127), batched over (REV, domain) pairs. */
int acegpu_derive_attest_keys(acegpu_ctx* ctx, const uint8_t* revs32, const uint8_t* doms8,
                              uint64_t n, uint8_t* out32);

/* ---- witnesses (prover.hpp:81-137) ---------------------------------------- */
/* witness_matches_tx (prover.cpp:190-197): witnesses n x 256 B; wlens may be
 * NULL (all 256) — a length other than 256 fails like the reference. */
int acegpu_witness_check(acegpu_ctx* ctx, const uint8_t* witnesses, const uint32_t* wlens,
                         const uint8_t* atts, uint64_t n, uint8_t* ok);
/* build_witness (prover.cpp:181-188), batched. */
int acegpu_build_witness(acegpu_ctx* ctx, const uint8_t* keys32, const uint8_t* tx_hashes32,
                         uint64_t n, uint8_t* out256);
/* WitnessScheme encapsulate / decrypt (prover.cpp:229-264): out = in XOR
 * keystream(XOR of share values selected by share_masks[i]); len bytes each. */
int acegpu_witness_xor(acegpu_ctx* ctx, const uint8_t* master32, const uint8_t* tx_hashes32,
                       const uint64_t* share_masks, const uint8_t* in, uint64_t len, uint64_t n,
                       uint8_t* out);

/* ---- measurement ----------------------------------------------------------- */
/* SHA-256 compressions/s of a register-resident chain over the whole GPU (the
 * integer-ALU roofline of the mock path). */
int acegpu_sha256_peak(acegpu_ctx* ctx, double* compressions_per_s);
/* Wall time of `iters` chained compressions per thread on a blocks x threads
 * grid (blocks = 1, threads = 32 gives the single-warp compression latency). */
int acegpu_sha256_probe(acegpu_ctx* ctx, int blocks, int threads, uint32_t iters,
                        double* seconds);

/* ---- BN254 (north-star additions; the reference has none) ----
 * Field elements: 32-B little-endian canonical integers at the host
 * boundary (standard form); Montgomery form (R = 2^256) on device for the
 * `_dev` calls. G1 affine = x|y (64 B), G2 affine = x.c0|x.c1|y.c0|y.c1
 * (128 B), infinity = all zeros. Parity: oracle/bn254_oracle.c (unpinned by
 * the reference). */
/* field: 0 = Fq, 1 = Fr. op: 0 mul, 1 add, 2 sub, 3 sqr, 4 inv (inv(0) = 0). */
int acegpu_bn_field_batch(acegpu_ctx* ctx, int field, int op, const uint8_t* a, const uint8_t* b,
                          uint64_t n, uint8_t* out);
/* In-place standard <-> Montgomery conversion of n device elements. */
int acegpu_bn_convert_dev(acegpu_ctx* ctx, void* stream, int field, uint8_t* d_data, uint64_t n,
                          int to_mont);
/* Fr NTT over 2^logn elements (logn <= 28), natural order in and out:
 * omega = 5^((r-1)/2^logn); inverse scales by n^-1; coset multiplies the
 * input by g^i (g = 5) before the forward transform / the output by g^-i
 * after the inverse. Host version: standard form in place. */
int acegpu_bn_ntt(acegpu_ctx* ctx, uint8_t* data, uint32_t logn, int inverse, int coset);
/* Mixed radix: N = 3 * 2^logk points (logk <= 26), same conventions (a
 * 3-point DFT over three 2^logk NTTs; Groth16 domains of 3 * 2^b points). */
int acegpu_bn_ntt3(acegpu_ctx* ctx, uint8_t* data, uint32_t logk, int inverse, int coset);
int acegpu_bn_ntt3_dev(acegpu_ctx* ctx, void* stream, const uint8_t* d_in, uint8_t* d_out,
                       uint32_t logk, int inverse, int coset);
/* Device version: Montgomery form; d_in may equal d_out. */
int acegpu_bn_ntt_dev(acegpu_ctx* ctx, void* stream, const uint8_t* d_in, uint8_t* d_out,
                      uint32_t logn, int inverse, int coset);
/* out[i] = scalars[i] * base (group 1 or 2), affine, standard form. */
int acegpu_bn_scalar_muls(acegpu_ctx* ctx, int group, const uint8_t* base, const uint8_t* scalars,
                          uint64_t n, uint8_t* out);
/* Fixed-base Pippenger MSM: prepare once per base set (proving key), run per
 * scalar vector. Scalars: n x 32-B canonical Fr, standard form. */
typedef struct acegpu_msm_bases acegpu_msm_bases;
int acegpu_bn_msm_prepare(acegpu_ctx* ctx, int group, const uint8_t* points, uint64_t n,
                          int points_on_device, acegpu_msm_bases** out);
void acegpu_bn_msm_free(acegpu_msm_bases* bases);
int acegpu_bn_msm_run(acegpu_ctx* ctx, const acegpu_msm_bases* bases, const uint8_t* scalars,
                      uint8_t* out_affine);
/* Variable-base form (no window tables: n x 64 B / 128 B of bases instead of
 * windows x that — a whole block's proving key): c = 20-bit windows, one
 * bucket set per window, balanced sub-ranges of <= `sub` points (0 = 80 Mi, the maximum),
 * Horner-combined window sums. Same results as the fixed-base form; run with
 * acegpu_bn_msm_run(_dev). n up to 2^31. */
int acegpu_bn_msm_prepare_vb(acegpu_ctx* ctx, int group, const uint8_t* points, uint64_t n,
                             int points_on_device, uint64_t sub, acegpu_msm_bases** out);
/* The compiled window width c and window count ceil(255 / c) (each scalar
 * contributes up to that many bucket entries). */
int acegpu_bn_msm_params(acegpu_ctx* ctx, int* window_bits, int* windows);
/* Device version: d_scalars standard form, d_out affine Montgomery form. */
int acegpu_bn_msm_run_dev(acegpu_ctx* ctx, void* stream, const acegpu_msm_bases* bases,
                          const uint8_t* d_scalars, uint8_t* d_out);
/* ---- Groth16 per-chunk prover (north star; synthetic ZK-ACE stand-in
 * circuit documented in oracle/bn254_oracle.h: T txs x K constraints per
 * chunk, paper size T = 1024, K = 1400 -> 1,434,625 constraints, domain 2^21).
 * setup: CRS from a trapdoor tau|alpha|beta|gamma|delta (5 x 32-B standard
 * Fr), proving-key MSM tables resident on the device. prove: per-tx private
 * witness w (n x 32-B LE, reduced mod r; the attest key, prover.cpp:181-188)
 * and public input pub (LE(public_inputs_digest) mod r, prover.cpp:74-76);
 * rs = r | s (standard form) or NULL to derive them deterministically from
 * the witnesses and the public inputs (binding v2, groth16.cu):
 *   D(x) = SHA-256(tag16 | SHA-256(x_0..x_31) | SHA-256(x_32..x_63) | ... | T_be32)
 *   (32-input blocks of the T 32-B inputs, the last block short; tag16 =
 *   "ace-g16-pubs-v2:" / "ace-g16-wits-v2:"),
 *   r = LE(SHA-256("ace-g16-r-v2" | D(w) | D(pub))) mod r, s likewise with
 *   "ace-g16-s-v2" (RFC 6979 style: secret, yet reproducible by a backup
 *   prover holding the witnesses).
 * Output: the 256-B proof A(64) | B(128) | C(64) big-endian (EIP-197, G2 as
 * c1|c0), the raw affine points little-endian (A x,y | B x.c0,x.c1,y.c0,y.c1 |
 * C x,y) and the chunk digest SHA-256("ace-g16-chunk-v2" | D(pub)), which
 * commits to every public input of the chunk. */
typedef struct acegpu_g16 acegpu_g16;
int acegpu_g16_setup(acegpu_ctx* ctx, uint32_t txs_per_chunk, uint32_t constraints_per_tx,
                     const uint8_t* trapdoor5, acegpu_g16** out);
void acegpu_g16_free(acegpu_g16* g);
/* shape: log_domain = log2 of the domain's power-of-two factor; domain: N,
 * the smallest of 2^a and 3 * 2^b that holds the constraints (mixed-radix
 * NTTs for 3 * 2^b; env ACEGPU_G16_RADIX3=0 keeps powers of two). */
int acegpu_g16_shape(const acegpu_g16* g, uint64_t* variables, uint64_t* constraints,
                     uint32_t* log_domain);
int acegpu_g16_domain(const acegpu_g16* g, uint64_t* N);
int acegpu_g16_prove_chunk(acegpu_ctx* ctx, acegpu_g16* g, const uint8_t* w, const uint8_t* pub,
                           const uint8_t* rs, uint8_t* proof256, uint8_t* raw256,
                           uint8_t* digest32);
int acegpu_g16_prove_chunk_dev(acegpu_ctx* ctx, void* stream, acegpu_g16* g, const uint8_t* d_w,
                               const uint8_t* d_pub, const uint8_t* d_rs, uint8_t* d_proof256,
                               uint8_t* d_raw256, uint8_t* d_digest32);

/* ---- general rank-1 constraint systems (north-star witness / constraint
 * evaluation; r1cs.cu). m rows <A_j, z> * <B_j, z> = <C_j, z> over `vars`
 * variables, z_0 = ONE, z_1..z_{n_pub} the public inputs. Each matrix k
 * (0 = A, 1 = B, 2 = C) in CSR: rowptr[k] (m + 1 u64, rowptr[k][0] = 0),
 * cols[k] (u32 < vars), vals[k] (32-B little-endian integers, reduced mod r
 * on load). The library appends one z_i * 0 = 0 row per public variable
 * i = 0..n_pub (Groth16 needs the public u_i independent): rows = m + n_pub + 1.
 * eval: a, b, c = A z, B z, C z over all rows (standard form; any of them
 * may be NULL) — the satisfiability check is a_j b_j = c_j. */
typedef struct acegpu_r1cs acegpu_r1cs;
int acegpu_r1cs_create(acegpu_ctx* ctx, uint64_t m, uint64_t vars, uint64_t n_pub,
                       const uint64_t* const rowptr[3], const uint32_t* const cols[3],
                       const uint8_t* const vals[3], acegpu_r1cs** out);
void acegpu_r1cs_free(acegpu_r1cs* r);
int acegpu_r1cs_shape(const acegpu_r1cs* r, uint64_t* rows, uint64_t* vars, uint64_t* n_pub);
int acegpu_r1cs_eval(acegpu_ctx* ctx, const acegpu_r1cs* r, const uint8_t* z, uint8_t* a,
                     uint8_t* b, uint8_t* c);
/* GPU witness generation for bit-level circuits (witprog.cu): a straight-
 * line program compiled once by the host circuit builder (zkace_circuit.py:
 * 4 x u32 per op, opcode << 24 | dst then operands; ADD operand lists in
 * addtab; var_slot = the slot of each private variable in order) and run by
 * every transaction on the device. run / run_dev write the full assignment
 * z = ONE | 5T public inputs (obj_hash, domain, credential packed big-endian
 * from the 104-B attestations) | T x n_vars private values (32-B LE). */
typedef struct acegpu_witprog acegpu_witprog;
int acegpu_witprog_create(acegpu_ctx* ctx, const uint32_t* ops4, uint64_t n_ops,
                          const uint32_t* addtab, uint64_t n_addtab, uint32_t n_adds,
                          const uint32_t* var_slot, uint32_t n_vars, uint32_t n_slots,
                          acegpu_witprog** out);
void acegpu_witprog_free(acegpu_witprog* w);
int acegpu_witprog_run(acegpu_ctx* ctx, const acegpu_witprog* w, const uint8_t* keys,
                       const uint8_t* atts, uint32_t T, uint8_t* z);
/* run_dev: T transactions in chunks of Tc (0 = one chunk), the chunks'
 * assignments (each 1 + 5 Tc + Tc n_vars elements) back to back in d_z. */
int acegpu_witprog_run_dev(acegpu_ctx* ctx, void* stream, const acegpu_witprog* w,
                           const uint8_t* d_keys, uint64_t key_stride, const uint8_t* d_atts,
                           uint32_t T, uint32_t Tc, uint8_t* d_z);
/* Groth16 keys for a general R1CS (r must outlive the key): the query
 * polynomials are the column sums A^T L(tau), B^T L(tau), C^T L(tau) of the
 * Lagrange basis; the verifying key has n_pub + 1 IC points. prove_z takes the
 * full assignment z (vars x 32-B standard form); rs = NULL derives r, s as
 * r = LE(SHA-256("ace-g16-r-v2" | D(z_{n_pub+1..}) | D(z_1..z_{n_pub}))) mod r
 * (D as above, extended to any count by levels of 1-KB blocks until at most
 * 32 digests remain); digest = SHA-256("ace-g16-chunk-v2" | D(public inputs)). */
int acegpu_g16_setup_r1cs(acegpu_ctx* ctx, const acegpu_r1cs* r, const uint8_t* trapdoor5,
                          acegpu_g16** out);
int acegpu_g16_prove_z(acegpu_ctx* ctx, acegpu_g16* g, const uint8_t* z, const uint8_t* rs,
                       uint8_t* proof256, uint8_t* raw256, uint8_t* digest32);
int acegpu_g16_prove_z_dev(acegpu_ctx* ctx, void* stream, acegpu_g16* g, const uint8_t* d_z,
                           const uint8_t* d_rs, uint8_t* d_proof256, uint8_t* d_raw256,
                           uint8_t* d_digest32);

/* Verifying key in the oracle layout (32-B LE standard-form coordinates):
 * alpha G1 (64) | beta G2 (128) | gamma G2 (128) | delta G2 (128) |
 * IC_0..IC_T G1 (64 each) = 448 + 64 (T + 1) bytes (oracle: bn_g16_vk). */
int acegpu_g16_vk(acegpu_ctx* ctx, const acegpu_g16* g, uint8_t* out);
/* Batched pairing verification of n chunk proofs:
 * proofs256 = n x 256-B EIP-197 proofs (acegpu_g16_prove_chunk's proof256),
 * pubs = n x T x 32-B little-endian public inputs (the raw public-input
 * digests; reduced mod r). *ok = 1 iff every proof satisfies
 * e(A,B) = e(alpha,beta) e(sum z_j IC_j, gamma) e(C,delta) with its points on
 * the curves and B in the order-r subgroup (one random-linear-combination
 * check: n + 3 Miller loops, one final exponentiation, one MSM over IC).
 * The 128-bit weights rho_i = LE(SHA-256("ace-g16-batch-v2" | seed | i_be32))[0:16]
 * come from seed = SHA-256("ace-g16-seed-v2:" | SHA-256(acegpu_g16_vk export) |
 * SHA-256(proof_0) | D(pub_0) | ... | SHA-256(proof_{n-1}) | D(pub_{n-1})): they
 * commit to the key, every proof and every public input, so no input can be
 * adjusted after the weights are known. _seed also returns the seed (32 B). */
int acegpu_g16_verify_batch(acegpu_ctx* ctx, acegpu_g16* g, const uint8_t* proofs256,
                            const uint8_t* pubs, uint64_t n, int* ok);
int acegpu_g16_verify_batch_seed(acegpu_ctx* ctx, acegpu_g16* g, const uint8_t* proofs256,
                                 const uint8_t* pubs, uint64_t n, int* ok, uint8_t* seed32);

/* verify_finality_certificate in Groth16 mode (prover.cpp:158-169 with real
 * proofs): *result = 0 Valid, 1 SlotMismatch, 2
 * HashMismatch, 3 ProofMismatch, checked in the reference's order. Instead
 * of re-proving, the chunk proofs (n_chunks x 256 B, chunk k covering txs
 * [kT, kT+T), as acegpu_g16_shard_roots_dev emits them) are checked with one
 * batched pairing verification against the public inputs recomputed from the
 * block, and the FC is recomputed from them with the reference's tree rule.
 * cost_units (optional) += 1 as the reference does. */
int acegpu_g16_verify_fc(acegpu_ctx* ctx, acegpu_g16* g, const uint8_t* fc328,
                         const uint8_t* payloads, const uint64_t* offs, const uint8_t* atts,
                         uint64_t n, const uint8_t* header256, const uint8_t* chunk_proofs256,
                         uint64_t* cost_units, int* result);

/* Groth16-mode shard (north-star block path): like acegpu_shard_roots_dev,
 * but each aligned chunk of T txs (T = txs_per_chunk, a power of two) is one
 * Groth16 proof over the chunk's witnesses (d_witness256: n x 256-B
 * build_witness records, prover.cpp:181-188; w = LE(first 32 B) mod r) and
 * public-input digests; the last chunk of the block is zero-padded. Chunk
 * roots (289 B: proof | chunk digest | kind Tx) combine with
 * acegpu_combine_roots_dev under the reference's tree rule. */
int acegpu_g16_shard_roots_dev(acegpu_ctx* ctx, void* stream, acegpu_g16* g,
                               const uint8_t* d_payloads, const uint64_t* d_offs,
                               const uint8_t* d_atts, uint64_t n, uint64_t n_total,
                               const uint8_t* d_revs, uint64_t n_revs,
                               const uint32_t* d_rev_index, uint8_t* d_codes,
                               const uint8_t* d_witness256, uint8_t* d_roots289,
                               uint8_t* d_merkle32);

/* ---- one proof per block across ranks (DIZK-style split of the MSMs) ----
 * setup_slice: the key of rank `rank` of `world` — the same CRS as
 * acegpu_g16_setup (same trapdoor), but only the rank's slice of every base
 * array (A, B1, B2, L, H) is stored (variable-base form); the verifying key is
 * whole. Slice r of an array of t bases is [t P_r / S, t (P_r + shares[r]) / S)
 * with P_r = shares[0] + .. + shares[r-1], S = the sum (shares NULL = equal),
 * so ranks that also transform H vectors can take fewer bases. Each rank: block_inputs_dev (verdicts, Merkle root, w, pub for a
 * block of n <= T txs; every rank holds the whole block), prove_partial_dev
 * (its partial A | B1 | B2 | L | H, 384 B — the witness and the H
 * polynomial are computed on every rank), an all-gather of the 384-B
 * records, finish_dev (sum in rank order, s A + r B1, C, proof, root leaf),
 * then acegpu_combine_roots_dev with one root. world = 1 with a plain key
 * gives the same bytes as acegpu_g16_prove_block. Replaces prover.cpp:129-142
 * in one-proof mode. */
int acegpu_g16_setup_slice(acegpu_ctx* ctx, uint32_t T, uint32_t K, const uint8_t* trapdoor5,
                           uint32_t rank, uint32_t world, const uint32_t* shares,
                           acegpu_g16** out);
int acegpu_g16_block_inputs_dev(acegpu_ctx* ctx, void* stream, acegpu_g16* g,
                                const uint8_t* d_payloads, const uint64_t* d_offs,
                                const uint8_t* d_atts, uint64_t n, const uint8_t* d_revs,
                                uint64_t n_revs, const uint32_t* d_rev_index, uint8_t* d_codes,
                                const uint8_t* d_witness256, uint8_t* d_w, uint8_t* d_pub,
                                uint8_t* d_merkle32);
int acegpu_g16_prove_partial_dev(acegpu_ctx* ctx, void* stream, acegpu_g16* g,
                                 const uint8_t* d_w, const uint8_t* d_pub, uint8_t* d_part384);
/* Owner split of the H polynomial (>= 2 ranks; the witness's NTTs are 6 of
 * 2^28 points at 100k txs, too much to repeat on every rank): phase1_dev =
 * witness, r, s, the A / B1 / B2 / L slice MSMs (left running) and the coset
 * evaluations of the owned vectors (mask a = 1, b = 2, c = 4; vector k is
 * owned by rank k mod world) into d_own (N x 32 B each, a, b, c order); the
 * caller scatters slice r of every vector (the H array's share bounds, as
 * setup_slice) to rank r; phase2_dev = (a b - c) / Z and [h] over the rank's slice
 * (d_slices = a | b | c slices, overwritten) -> the 384-B partial record. */
int acegpu_g16_prove_phase1_dev(acegpu_ctx* ctx, void* stream, acegpu_g16* g, const uint8_t* d_w,
                                const uint8_t* d_pub, int owned, uint8_t* d_own);
int acegpu_g16_prove_phase2_dev(acegpu_ctx* ctx, void* stream, acegpu_g16* g, uint8_t* d_slices,
                                uint8_t* d_part384);
int acegpu_g16_finish_dev(acegpu_ctx* ctx, void* stream, acegpu_g16* g, const uint8_t* d_parts,
                          uint32_t world, uint8_t* d_proof256, uint8_t* d_raw256,
                          uint8_t* d_digest32, uint8_t* d_root289);
/* The north-star block path through ONE host-buffer call (the Groth16-mode
 * prove_block + build_finality_certificate, prover.cpp:129-156): the block's
 * H2D, batched attestation verdicts (revs / rev_index as
 * acegpu_attest_prove_certify; n_revs = 0 skips them), one Groth16 proof per
 * aligned chunk of T txs over the n x 256-B build_witness records
 * (prover.cpp:181-188), the reference's tree rule over the chunk proofs
 * (prover.cpp:106-127) and the FC; D2H of codes (n), the root proof (289 B:
 * bytes | digest | kind), the FC (328 B) and, if chunk_proofs256 is not NULL,
 * the ceil(n / T) chunk proofs (256 B each, acegpu_g16_verify_fc's input). */
int acegpu_g16_prove_block(acegpu_ctx* ctx, acegpu_g16* g, const uint8_t* payloads,
                           const uint64_t* offs, const uint8_t* atts, uint64_t n,
                           const uint8_t* header256, const uint8_t* revs, uint64_t n_revs,
                           const uint32_t* rev_index, const uint8_t* witness256, uint8_t* codes,
                           uint8_t* proof289, uint8_t* fc328, uint8_t* chunk_proofs256);

/* Optimal ate pairing product prod_i e(P_i, Q_i) (final exponentiation
 * included) over host buffers in the oracle encodings: G1 = x|y, G2 =
 * x.c0|x.c1|y.c0|y.c1, 32-B little-endian standard form, all-zero = infinity.
 * out384 (optional): Fq12 as 12 x 32 B (c0.c0.c0, c0.c0.c1, ..., c1.c2.c1);
 * is_one (optional): 1 iff the product is the identity (a pairing check). */
int acegpu_bn_pairing(acegpu_ctx* ctx, uint64_t n, const uint8_t* g1s, const uint8_t* g2s,
                      uint8_t* out384, int* is_one);

/* Fq12 unit operation for parity tests (one element, 384 B in/out in the
 * encoding above): 0 final exponentiation, 1 easy part ^((p^6-1)(p^2+1)),
 * 2 hard part ^((p^4-p^2+1)/r), 3/4/5 Frobenius p/p^2/p^3, 6 ^x (BN
 * parameter), 7 inverse, 8 square, 9 Miller loop of the G1|G2 pair in the
 * first 192 input bytes (defined up to subfield factors), 10 ^e with e the
 * u64 (LE) at in384[384..392) (the input buffer is then 392 bytes),
 * 11 square of an element of the cyclotomic subgroup (Granger-Scott). */
int acegpu_bn_f12_op(acegpu_ctx* ctx, int op, const uint8_t* in384, uint8_t* out384);

/* ---- Phase 1a on the GPU --------------------------------
 * attest_check_light (pipeline.cpp:20-42; LightCheck, pipeline.hpp:32-37):
 * codes[i] = 0 AcceptPendingProof, 1 PayloadBinding, 2 UnknownIdentity,
 * 3 StaleDomain. The IdentityRegistry (pipeline.hpp:22-30, a std::set<Hash32>)
 * is passed as n_registry 32-B commitments sorted ascending (bytewise), which
 * is the set's iteration order; window = PipelineConfig::domain_window_slots.
 * counters3 (host, optional): LightCheckCounters {sha256_ops, registry_probes,
 * window_checks} summed over the batch (pipeline.hpp:41-52). */
int acegpu_light_check(acegpu_ctx* ctx, const uint8_t* payloads, const uint64_t* offs,
                       const uint8_t* atts, uint64_t n, const uint8_t* registry32,
                       uint64_t n_registry, uint64_t current_slot, uint64_t window_slots,
                       uint8_t* codes, uint64_t* counters3);
int acegpu_light_check_dev(acegpu_ctx* ctx, void* stream, const uint8_t* d_payloads,
                           const uint64_t* d_offs, const uint8_t* d_atts, uint64_t n,
                           const uint8_t* d_registry32, uint64_t n_registry,
                           uint64_t current_slot, uint64_t window_slots, uint8_t* d_codes,
                           uint8_t* d_tx_hashes /* n x 32 SHA-256(payload), or NULL */);
/* Block build (process_slot, pipeline.cpp:132-145): order-preserving
 * compaction of the txs with d_codes[i] == 0 (all txs when d_codes is NULL)
 * into the out arrays (out_offs: n_accepted + 1 entries, rebased to 0), and the
 * 256-B header = header_tmpl with tx_count, tx_merkle_root, attest_merkle_root
 * set (wire.cpp:74-96, 257-273). The result is device-resident, ready for
 * acegpu_attest_prove_certify_dev. *n_accepted is written to HOST memory (the
 * call synchronises `stream` once to read it). */
int acegpu_build_block_dev(acegpu_ctx* ctx, void* stream, const uint8_t* d_payloads,
                           const uint64_t* d_offs, const uint8_t* d_atts, uint64_t n,
                           const uint8_t* d_codes, const uint8_t* d_header_tmpl,
                           uint8_t* d_out_payloads, uint64_t* d_out_offs, uint8_t* d_out_atts,
                           uint8_t* d_out_header, uint64_t* n_accepted);

/* Integer-pipe microbenchmarks (roofline denominators for MSM / NTT). */
int acegpu_imad_peak(acegpu_ctx* ctx, double* imad_per_s);
int acegpu_bn_mul_rate(acegpu_ctx* ctx, int field, double* muls_per_s);

#ifdef __cplusplus
}
#endif
#endif
