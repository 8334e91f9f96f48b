// Launchers for groth16.cu (synthetic ZK-ACE stand-in circuit, see
// oracle/bn254_oracle.h for the constraint system).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace ace_gpu {
namespace bn {

struct G16Dims {
    uint32_t T, K;  // txs per chunk, constraints per tx
    uint64_t V;     // variables 1 + T + T*(K+1)
    uint64_t m;     // constraints T*K + T + 1
};

// Setup (CRS from a trapdoor; all Fr in Montgomery form unless noted).
void g16_chain_consts(uint32_t K, uint8_t* out, cudaStream_t s);
// c[0..4] = tau, alpha, beta, gamma, delta in standard form -> converted;
// fills c[5..11] (see groth16.cu) for the domain N = 2^logn, or 3 * 2^logn
// when three (omega = 5^((r-1)/N)).
void g16_setup_consts(uint8_t* c, uint32_t logn, int three, cudaStream_t s);
void g16_lagrange(const uint8_t* c, uint64_t m, uint8_t* L, cudaStream_t s);
// su, sv: V scalars; sl: V - T - 1 scalars (standard form); part: 256*64 B scratch
void g16_query_scalars(const G16Dims& d, const uint8_t* L, const uint8_t* c, const uint8_t* cc,
                       uint8_t* part, uint8_t* su, uint8_t* sv, uint8_t* sl, cudaStream_t s);
void g16_h_scalars(const uint8_t* c, uint64_t n, uint8_t* out, cudaStream_t s);
// Verifying key: IC_j scalars (beta u_j + alpha v_j) / gamma, j = 0..T (standard form).
void g16_ic_scalars(uint32_t T, const uint8_t* c, const uint8_t* su, const uint8_t* sv,
                    uint8_t* out, cudaStream_t s);

// Prover.
void g16_witness(const G16Dims& d, const uint8_t* w, const uint8_t* pub, const uint8_t* cc,
                 uint8_t* z, uint8_t* ea, uint8_t* eb, uint8_t* ec, cudaStream_t s);
void g16_pointwise(uint8_t* ea, const uint8_t* eb, const uint8_t* ec, const uint8_t* c,
                   uint64_t n, cudaStream_t s);
// Binding v2 (groth16.cu): D(x) digests of T-input chunks, chunk digests
// SHA-256("ace-g16-chunk-v2" | D(pub)), and r, s from D(w) | D(pub).
size_t g16_digest_scratch_bytes(uint32_t T, uint32_t chunks);
void g16_input_digests(const uint8_t* x, uint32_t T, uint32_t chunks, int wits, uint8_t* scratch,
                       uint8_t* out, cudaStream_t s);
// scratch: g16_digest_scratch_bytes(T, chunks); D(pub_k) left at scratch + stride * chunks
void g16_chunk_digests(const uint8_t* pub, uint32_t T, uint32_t chunks, uint8_t* scratch,
                       uint8_t* digests, cudaStream_t s);
// D(x) for any count (levels of 1-KB blocks until <= 32 digests; == the
// chunk rule for count <= 1024); r, s and the chunk digest of a general
// R1CS assignment (w = its private part, n_w values)
size_t g16_long_digest_scratch_bytes(uint64_t count);
void g16_long_digest(const uint8_t* x, uint64_t count, int wits, uint8_t* scratch, uint8_t* out,
                     cudaStream_t s);
void g16_derive_rs_long(const uint8_t* w, uint64_t n_w, const uint8_t* pub, uint32_t T,
                        uint8_t* scratch, uint8_t* rs, uint8_t* digest, cudaStream_t s);
// scratch: g16_digest_scratch_bytes(T, 1) + 32
void g16_derive_rs(const uint8_t* w, const uint8_t* pub, uint32_t T, uint8_t* scratch,
                   uint8_t* rs, uint8_t* digest, cudaStream_t s);
void g16_extras(uint8_t* za, uint8_t* zb, uint8_t* zl, uint64_t V, uint64_t Vp, const uint8_t* rs,
                cudaStream_t s);
void g16_scale(const uint8_t* pts, const uint8_t* rs, uint8_t* out, cudaStream_t s);
void g16_assemble(const uint8_t* pts, const uint8_t* scaled, uint8_t* proof, uint8_t* raw,
                  cudaStream_t s);
// Split keys: pts (A | B1 | B2 | L | H, 384 B) = the sum of `world` partial records.
void g16_sum_parts(const uint8_t* parts, uint32_t world, uint8_t* pts, cudaStream_t s);
// Block glue.
void g16_gather32(const uint8_t* src, uint64_t stride, uint64_t n, uint64_t n_pad, uint8_t* dst,
                  cudaStream_t s);
void g16_chunk_node(const uint8_t* proof256, const uint8_t* digest32, uint8_t* node,
                    cudaStream_t s);

}  // namespace bn
}  // namespace ace_gpu
