// Batched Groth16 verification of chunk proofs on the GPU.
//
// For n proofs (A_i, B_i, C_i) with public inputs z_i = (1, pub_i) the
// verifier checks, with 128-bit weights rho_i derived Fiat-Shamir style from
// the whole statement (rho_i = LE(SHA-256("ace-g16-batch-v2" | seed | i))[0:16],
// seed = SHA-256("ace-g16-seed-v2:" | SHA-256(VK) | SHA-256(proof_0) | D(pub_0) |
// ... | SHA-256(proof_{n-1}) | D(pub_{n-1})), VK = the acegpu_g16_vk export and
// D(pub_i) the input digest of proof i's T public inputs, groth16.cu), so no
// public input can be changed after the weights are known:
//
//   prod_i e(rho_i A_i, B_i) * e(-(sum rho_i) alpha, beta)
//       * e(-sum_j (sum_i rho_i z_ij) IC_j, gamma) * e(-sum_i rho_i C_i, delta) == 1
//
// i.e. n + 3 Miller loops and ONE final exponentiation, plus one MSM over the
// T + 1 IC points with combined scalars. Every proof point is checked to be
// on its curve and B_i to be in the order-r subgroup of the twist
// (psi(B) = [6x^2] B).
#include <cuda_runtime.h>

#include "g16_kernels.cuh"
#include "g16_verify.cuh"
#include "pairing.cuh"
#include "pairing_kernels.cuh"
#include "sha256.cuh"

namespace ace_gpu {
namespace bn {
namespace {

__device__ __forceinline__ Fq ld_be(const uint8_t* p) {
    Fq x;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint8_t* q = p + 28 - 4 * k;
        x.v[k] = (uint32_t(q[0]) << 24) | (uint32_t(q[1]) << 16) | (uint32_t(q[2]) << 8) | q[3];
    }
    return to_mont(x);
}
__device__ __forceinline__ void st_std(uint8_t* p, const Fq& x) { store<FqCfg>(p, from_mont(x)); }
__device__ __forceinline__ void st_std2(uint8_t* p, const Fq2& x) {
    st_std(p, x.c0);
    st_std(p + 32, x.c1);
}

// LE 32 B mod r (any 256-bit value < 6r), Montgomery form.
__device__ __forceinline__ Fr fr_from_le(const uint8_t* p) {
    uint32_t x[8], m[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        x[i] = uint32_t(p[4 * i]) | (uint32_t(p[4 * i + 1]) << 8) | (uint32_t(p[4 * i + 2]) << 16) |
               (uint32_t(p[4 * i + 3]) << 24);
        m[i] = mod_limb<FrCfg>(i);
    }
    while (detail::limbs_geq(x, m)) detail::limbs_sub(x, m);
    Fr r;
#pragma unroll
    for (int i = 0; i < 8; ++i) r.v[i] = x[i];
    return to_mont(r);
}

template <class F>
__device__ __forceinline__ bool on_curve(const F& x, const F& y, const F& b) {
    return feq(fsqr(y), fadd(fmul(fsqr(x), x), b));
}
__device__ __forceinline__ Fq g1_b() {
    Fq b = Fq::zero();
    b.v[0] = 3;
    return to_mont(b);
}
__device__ __forceinline__ Fq2 g2_b() {  // 3 / (9 + u)
    Fq2 xi;
    xi.c0 = Fq::zero();
    xi.c1 = Fq::zero();
    xi.c0.v[0] = 9;
    xi.c1.v[0] = 1;
    xi = {to_mont(xi.c0), to_mont(xi.c1)};
    const Fq2 inv = f2_inv(xi);
    return {fq_mul_call(g1_b(), inv.c0), fq_mul_call(g1_b(), inv.c1)};
}

template <class F>
__device__ XYZZ<F> mul_bits(const F& x, const F& y, const uint32_t* k, int bits) {
    XYZZ<F> acc = XYZZ<F>::inf();
    for (int b = bits - 1; b >= 0; --b) {
        acc = xyzz_dbl(acc);
        if ((k[b >> 5] >> (b & 31)) & 1) acc = xyzz_madd(acc, x, y);
    }
    return acc;
}

template <class F>
__device__ void to_affine(const XYZZ<F>& p, F& x, F& y);
template <>
__device__ void to_affine<Fq>(const XYZZ<Fq>& p, Fq& x, Fq& y) {
    const Fq t = inv_fast(fmul(p.ZZ, p.ZZZ));  // 1 / (ZZ ZZZ)
    x = fmul(p.X, fmul(t, p.ZZZ));
    y = fmul(p.Y, fmul(t, p.ZZ));
}

// msg = "ace-g16-seed-v2:" | vk_digest | (SHA-256(proof_i) | D(pub_i))_i
__global__ void proof_hash_kernel(const uint8_t* proofs, const uint8_t* pd, uint32_t n,
                                  const uint8_t* vk_digest, uint8_t* msg) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) {
        const char tag[] = "ace-g16-seed-v2:";
        for (int k = 0; k < 16; ++k) msg[k] = tag[k];
        for (int k = 0; k < 32; ++k) msg[16 + k] = vk_digest[k];
    }
    if (i >= n) return;
    uint32_t d[8];
    sha256_bytes(proofs, 256ull * i, 256, d);
    uint8_t* o = msg + 48 + 64ull * i;
    store_digest(o, d);
    for (int k = 0; k < 32; ++k) o[32 + k] = pd[32ull * i + k];
}

__global__ void seed_kernel(const uint8_t* msg, uint32_t n, uint8_t* seed) {
    if (threadIdx.x || blockIdx.x) return;
    uint32_t d[8];
    sha256_bytes(msg, 0, 48 + 64 * n, d);
    store_digest(seed, d);
}

__global__ void hash_kernel(const uint8_t* x, uint32_t len, uint8_t* out) {
    if (threadIdx.x || blockIdx.x) return;
    uint32_t d[8];
    sha256_bytes(x, 0, len, d);
    store_digest(out, d);
}

__global__ void rho_kernel(const uint8_t* seed, uint32_t n, uint8_t* rho) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    __align__(16) uint8_t m[52];
    const char tag[] = "ace-g16-batch-v2";
    for (int k = 0; k < 16; ++k) m[k] = tag[k];
    for (int k = 0; k < 32; ++k) m[16 + k] = seed[k];
    m[48] = i >> 24; m[49] = i >> 16; m[50] = i >> 8; m[51] = i;
    uint32_t d[8];
    sha256_bytes(m, 0, 52, d);
    uint8_t* o = rho + 32ull * i;
    uint32_t nz = 0;
    for (int k = 0; k < 4; ++k) {  // first 16 digest bytes as a little-endian integer
        const uint32_t w = d[k];
        o[4 * k] = w >> 24; o[4 * k + 1] = w >> 16; o[4 * k + 2] = w >> 8; o[4 * k + 3] = w;
        nz |= w;
    }
    for (int k = 16; k < 32; ++k) o[k] = 0;
    if (!nz) o[0] = 1;  // never a zero weight
}

// s_0 = sum_i rho_i, s_{1+t} = sum_i rho_i pub_{i,t} (standard form).
__global__ void combine_kernel(const uint8_t* pubs, const uint8_t* rho, uint32_t n, uint32_t T,
                               uint8_t* out) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j > T) return;
    Fr acc = Fr::zero();
    for (uint32_t i = 0; i < n; ++i) {
        const Fr r = fr_from_le(rho + 32ull * i);
        acc = add(acc, j ? mul(r, fr_from_le(pubs + 32ull * (uint64_t(i) * T + j - 1))) : r);
    }
    store<FrCfg>(out + 32ull * j, from_mont(acc));
}

__device__ void put_neg_g1(uint8_t* o, const XYZZ<Fq>& p) {
    if (p.is_inf()) {
        for (int b = 0; b < 64; ++b) o[b] = 0;
        return;
    }
    Fq x, y;
    to_affine(p, x, y);
    st_std(o, x);
    st_std(o + 32, neg(y));
}

// Two threads per proof: thread 2i validates proof i and writes rho_i A_i
// (pair i) and B_i; thread 2i+1 computes rho_i C_i (XYZZ, Montgomery).
// Thread 2n computes s0 * alpha (pair n, negated), s0 = sum_i rho_i, so the
// three serial scalar multiplications run side by side.
__global__ void points_kernel(const uint8_t* proofs, const uint8_t* rho, uint32_t n,
                              uint8_t* g1s, uint8_t* g2s, XYZZ<Fq>* cacc, int* bad,
                              const uint8_t* s0_std, const uint8_t* vk_mont) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t i = t >> 1;
    if (t == 2 * n) {
        const Fq alx = load<FqCfg>(vk_mont), aly = load<FqCfg>(vk_mont + 32);
        const uint4* sq = reinterpret_cast<const uint4*>(s0_std);
        const uint4 lo = sq[0], hi = sq[1];
        const uint32_t s0[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
        put_neg_g1(g1s + 64ull * n, mul_bits(alx, aly, s0, 256));
        return;
    }
    if (i >= n) return;
    const uint8_t* p = proofs + 256ull * i;
    uint32_t k[4];
    for (int w = 0; w < 4; ++w) {
        const uint8_t* q = rho + 32ull * i + 4 * w;
        k[w] = uint32_t(q[0]) | (uint32_t(q[1]) << 8) | (uint32_t(q[2]) << 16) | (uint32_t(q[3]) << 24);
    }
    if (t & 1) {
        const Fq cx = ld_be(p + 192), cy = ld_be(p + 224);
        cacc[i] = mul_bits(cx, cy, k, 128);
        return;
    }
    const Fq ax = ld_be(p), ay = ld_be(p + 32), cx = ld_be(p + 192), cy = ld_be(p + 224);
    const Fq2 bx = {ld_be(p + 96), ld_be(p + 64)}, by = {ld_be(p + 160), ld_be(p + 128)};
    const bool ok = on_curve(ax, ay, g1_b()) && on_curve(cx, cy, g1_b()) && on_curve(bx, by, g2_b());
    if (!ok) atomicExch(bad, 1);  // the subgroup test of B runs beside the Miller loops
    const XYZZ<Fq> ra = mul_bits(ax, ay, k, 128);
    uint8_t* o1 = g1s + 64ull * i;
    if (ra.is_inf()) {
        for (int b = 0; b < 64; ++b) o1[b] = 0;
    } else {
        Fq x, y;
        to_affine(ra, x, y);
        st_std(o1, x);
        st_std(o1 + 32, y);
    }
    uint8_t* o2 = g2s + 128ull * i;
    st_std2(o2, bx);
    st_std2(o2 + 64, by);
}

// Blocks [0, mb): one Miller loop per pair (raw Fq12 to scratch, as
// launch_pairing_product). Blocks [mb, ...): the order-r subgroup test of
// proof i's B: psi(B) == [6x^2] B (El Housni-Guillevic-Piellard 2022 for
// BN254; psi = the untwist-Frobenius-twist map, the Miller loop's frob_twist)
// -- a 127-bit scalar instead of r's 254 bits, run concurrently with the
// Miller loops instead of before them.
// Blocks [0, mb): 32 pairs per 128-thread CTA, Miller loops split over four
// warps (miller_loop_4w). Blocks >= mb: the psi(B) = [6x^2]B subgroup checks.
__global__ void __launch_bounds__(128) miller_check_kernel(uint32_t n_pairs, const uint8_t* g1s,
                                                          const uint8_t* g2s, uint8_t* scratch,
                                                          uint32_t mb, const uint8_t* proofs,
                                                          uint32_t n, int* bad) {
    if (blockIdx.x < mb) {
        __shared__ MillerSmem sm;
        const uint32_t i = blockIdx.x * 32 + (threadIdx.x & 31);
        bool active = i < n_pairs;
        Fq xp = Fq::zero(), yp = Fq::zero();
        Fq2 xq = {xp, xp}, yq = {xp, xp};
        if (active) {
            const uint8_t* p = g1s + 64ull * i;
            const uint8_t* q = g2s + 128ull * i;
            bool inf = true;
            for (int b = 0; b < 64 && inf; ++b) inf = p[b] == 0;
            bool qinf = true;
            for (int b = 0; b < 128 && qinf; ++b) qinf = q[b] == 0;
            active = !(inf || qinf);
            xp = to_mont(load<FqCfg>(p));
            yp = to_mont(load<FqCfg>(p + 32));
            xq = {to_mont(load<FqCfg>(q)), to_mont(load<FqCfg>(q + 32))};
            yq = {to_mont(load<FqCfg>(q + 64)), to_mont(load<FqCfg>(q + 96))};
        }
        const Fq12 f = miller_loop_4w(xp, yp, xq, yq, active, sm);
        if (threadIdx.x < 32 && i < n_pairs)  // degenerate pairs: f = 1
            *reinterpret_cast<Fq12*>(scratch + sizeof(Fq12) * i) = active ? f : f12_one();
        return;
    }
    const uint32_t i = (blockIdx.x - mb) * 128 + threadIdx.x;
    if (i >= n) return;
    const uint8_t* pr = proofs + 256ull * i;
    const Fq2 bx = {ld_be(pr + 96), ld_be(pr + 64)}, by = {ld_be(pr + 160), ld_be(pr + 128)};
    if (!on_curve(bx, by, g2_b())) return;  // flagged by points_kernel
    const uint32_t k6x2[4] = {0xe87cfd46u, 0xf83e9682u, 0xeeb859fbu, 0x6f4d8248u};
    const XYZZ<Fq2> m = mul_bits(bx, by, k6x2, 127);
    Fq2 px = bx, py = by;
    frob_twist(px, py);
    if (m.is_inf() || !feq(fmul(px, m.ZZ), m.X) || !feq(fmul(py, m.ZZZ), m.Y)) atomicExch(bad, 1);
}


// Pairs n, n+1, n+2: (-(s_0) alpha, beta), (-L, gamma), (-sum rho_i C_i, delta).
__global__ void finish_kernel(const XYZZ<Fq>* cacc, uint32_t n, const uint8_t* s0_std,
                              const uint8_t* vk_mont, const uint8_t* L_mont,
                              const uint8_t* vk_g2_std, uint8_t* g1s, uint8_t* g2s) {
    if (threadIdx.x || blockIdx.x) return;
    XYZZ<Fq> cs = XYZZ<Fq>::inf();
    for (uint32_t i = 0; i < n; ++i) cs = xyzz_add(cs, cacc[i]);
    (void)s0_std;
    (void)vk_mont;  // s0 * alpha (pair n) is written by points_kernel
    const Fq lx = load<FqCfg>(L_mont), ly = load<FqCfg>(L_mont + 32);
    uint8_t* ol = g1s + 64ull * (n + 1);
    if (lx.is_zero() && ly.is_zero()) {
        for (int b = 0; b < 64; ++b) ol[b] = 0;
    } else {
        st_std(ol, lx);
        st_std(ol + 32, neg(ly));
    }
    put_neg_g1(g1s + 64ull * (n + 2), cs);
    for (int b = 0; b < 3 * 128; ++b) g2s[128ull * n + b] = vk_g2_std[b];  // beta | gamma | delta
}

inline unsigned grid(uint64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

size_t g16_verify_scratch_bytes(uint32_t n, uint32_t T) {
    const size_t a = (48 + 64ull * n) + 32ull * n + 32 + 32ull * (T + 1) + 64 + 64ull * (n + 3) +
                     128ull * (n + 3) + sizeof(XYZZ<Fq>) * (n ? n : 1) + 16 * 8 +
                     g16_digest_scratch_bytes(T, n) + 32ull * n;
    return a + pairing_scratch_bytes(n + 3) + 256 + 128 * 4;
}

void g16_vk_digest(const uint8_t* vk_bytes, uint32_t len, uint8_t* out, cudaStream_t s) {
    hash_kernel<<<1, 32, 0, s>>>(vk_bytes, len, out);
}

int g16_verify_batch(const G16VerifyKey& vk, const uint8_t* proofs, const uint8_t* pubs,
                     uint32_t n, uint8_t* scratch, MsmScratch& msm, int* d_ok, cudaStream_t s,
                     uint8_t* seed_out) {
    const uint32_t T = vk.T;
    auto take = [&scratch](size_t bytes) {
        uint8_t* p = scratch;
        scratch += (bytes + 127) & ~size_t(127);
        return p;
    };
    uint8_t* hashes = take(48 + 64ull * n);
    uint8_t* rho = take(32ull * n);
    uint8_t* seed = take(32);
    uint8_t* dsc = take(g16_digest_scratch_bytes(T, n));
    uint8_t* pd = take(32ull * n);
    uint8_t* sc = take(32ull * (T + 1));
    uint8_t* L = take(64);
    uint8_t* g1s = take(64ull * (n + 3));
    uint8_t* g2s = take(128ull * (n + 3));
    auto* cacc = reinterpret_cast<XYZZ<Fq>*>(take(sizeof(XYZZ<Fq>) * (n ? n : 1)));
    int* bad = reinterpret_cast<int*>(take(16));
    uint8_t* pscratch = take(pairing_scratch_bytes(n + 3));
    cudaMemsetAsync(bad, 0, sizeof(int), s);
    g16_input_digests(pubs, T, n, 0, dsc, pd, s);
    proof_hash_kernel<<<grid(n, 64), 64, 0, s>>>(proofs, pd, n, vk.vk_digest, hashes);
    seed_kernel<<<1, 32, 0, s>>>(hashes, n, seed);
    if (seed_out) cudaMemcpyAsync(seed_out, seed, 32, cudaMemcpyDeviceToDevice, s);
    rho_kernel<<<grid(n, 64), 64, 0, s>>>(seed, n, rho);
    combine_kernel<<<grid(T + 1, 64), 64, 0, s>>>(pubs, rho, n, T, sc);
    if (msm_run(1, vk.ic_table, T + 1, sc, msm, L, s)) return -1;
    points_kernel<<<grid(2ull * n + 1, 32), 32, 0, s>>>(proofs, rho, n, g1s, g2s, cacc, bad, sc,
                                                        vk.alpha1_mont);
    finish_kernel<<<1, 32, 0, s>>>(cacc, n, sc, vk.alpha1_mont, L, vk.g2_std, g1s, g2s);
    const uint32_t mb = (n + 3 + 31) / 32;
    miller_check_kernel<<<mb + (n + 127) / 128, 128, 0, s>>>(n + 3, g1s, g2s, pscratch, mb,
                                                            proofs, n, bad);
    launch_pairing_finish(n + 3, pscratch, nullptr, d_ok, s);
    // d_ok &= !bad
    combine_ok(d_ok, bad, s);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

namespace {
__global__ void combine_ok_kernel(int* ok, const int* bad) {
    if (threadIdx.x || blockIdx.x) return;
    if (*bad) *ok = 0;
}
}  // namespace

void combine_ok(int* ok, const int* bad, cudaStream_t s) { combine_ok_kernel<<<1, 32, 0, s>>>(ok, bad); }

}  // namespace bn
}  // namespace ace_gpu
