// BN254 pairing products on the GPU (pairing.cuh): one thread per Miller
// loop, a CTA tree for the Fq12 product, one final exponentiation.
#include <cuda_runtime.h>

#include "pairing.cuh"
#include "pairing_kernels.cuh"

namespace ace_gpu {
namespace bn {
namespace {

__device__ __forceinline__ Fq ldq(const uint8_t* p) { return to_mont(load<FqCfg>(p)); }
__device__ __forceinline__ void stq(uint8_t* p, const Fq& x) { store<FqCfg>(p, from_mont(x)); }

__device__ __forceinline__ bool all_zero(const uint8_t* p, int n) {
    for (int i = 0; i < n; ++i)
        if (p[i]) return false;
    return true;
}

__device__ void store_f12(uint8_t* out, const Fq12& f) {
    const Fq2* c[6] = {&f.c0.c0, &f.c0.c1, &f.c0.c2, &f.c1.c0, &f.c1.c1, &f.c1.c2};
    for (int i = 0; i < 6; ++i) {
        stq(out + 64 * i, c[i]->c0);
        stq(out + 64 * i + 32, c[i]->c1);
    }
}

// Raw Montgomery limbs in the scratch buffer (no conversion).
__device__ __forceinline__ void put_raw(uint8_t* p, const Fq12& f) {
    *reinterpret_cast<Fq12*>(p) = f;
}
__device__ __forceinline__ Fq12 get_raw(const uint8_t* p) {
    return *reinterpret_cast<const Fq12*>(p);
}

// One Miller loop per pair (oracle encodings: G1 x|y, G2 x.c0|x.c1|y.c0|y.c1,
// 32-B LE standard form; all-zero = infinity, whose pairing is 1).
__global__ void miller_kernel(uint32_t n, const uint8_t* g1s, const uint8_t* g2s,
                              uint8_t* scratch) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint8_t* p = g1s + 64ull * i;
    const uint8_t* q = g2s + 128ull * i;
    Fq12 f;
    if (all_zero(p, 64) || all_zero(q, 128)) {
        f = f12_one();
    } else {
        const Fq2 xq = {ldq(q), ldq(q + 32)}, yq = {ldq(q + 64), ldq(q + 96)};
        f = miller_loop(ldq(p), ldq(p + 32), xq, yq);
    }
    put_raw(scratch + sizeof(Fq12) * i, f);
}

// Product of the n Miller values (one CTA, tree over shared indices in the
// scratch buffer), final exponentiation, standard-form output.
__global__ void product_final_kernel(uint32_t n, uint8_t* scratch, uint8_t* out384,
                                     int* is_one) {
    for (uint32_t stride = 1; stride < n; stride <<= 1) {
        for (uint32_t i = threadIdx.x * 2 * stride; i + stride < n; i += blockDim.x * 2 * stride) {
            const Fq12 a = get_raw(scratch + sizeof(Fq12) * i);
            const Fq12 b = get_raw(scratch + sizeof(Fq12) * (i + stride));
            put_raw(scratch + sizeof(Fq12) * i, f12_mul(a, b));
        }
        __syncthreads();
    }
    // the final exponentiation on warp 0, lane-parallel products
    if (threadIdx.x >= 32) return;
    __shared__ WarpProducts ws;
    const Fq12 f = final_exp_warp(n ? get_raw(scratch) : f12_one(), ws);
    if (threadIdx.x) return;
    if (out384) store_f12(out384, f);
    if (is_one) *is_one = f12_is_one(f) ? 1 : 0;
}

__device__ Fq12 load_f12(const uint8_t* in) {
    Fq12 f;
    Fq2* c[6] = {&f.c0.c0, &f.c0.c1, &f.c0.c2, &f.c1.c0, &f.c1.c1, &f.c1.c2};
    for (int i = 0; i < 6; ++i) {
        c[i]->c0 = ldq(in + 64 * i);
        c[i]->c1 = ldq(in + 64 * i + 32);
    }
    return f;
}

// Unit operations (parity tests against bn_f12_op of the oracle).
__global__ void f12_op_kernel(int op, const uint8_t* in, uint8_t* out) {
    if (threadIdx.x || blockIdx.x) return;
    Fq12 r;
    if (op == 9) {
        const Fq2 xq = {ldq(in + 64), ldq(in + 96)}, yq = {ldq(in + 128), ldq(in + 160)};
        r = miller_loop(ldq(in), ldq(in + 32), xq, yq);
    } else {
        const Fq12 a = load_f12(in);
        switch (op) {
            case 0: r = final_exp(a); break;
            case 1: {
                const Fq12 t = f12_mul(f12_conj(a), f12_inv(a));
                r = f12_mul(t, f12_frob(t, 2));
                break;
            }
            case 2: r = final_exp_hard(a); break;
            case 3: r = f12_frob(a, 1); break;
            case 4: r = f12_frob(a, 2); break;
            case 5: r = f12_frob(a, 3); break;
            case 6: r = f12_pow_x(a); break;
            case 7: r = f12_inv(a); break;
            case 10: {  // a^e, e = u64 LE at in[384..392)
                uint64_t e = 0;
                for (int k = 7; k >= 0; --k) e = (e << 8) | in[384 + k];
                r = f12_one();
                for (int i = 63; i >= 0; --i) {
                    r = f12_sqr(r);
                    if ((e >> i) & 1) r = f12_mul(r, a);
                }
                break;
            }
            case 11: r = f12_cyc_sqr(a); break;  // input in the cyclotomic subgroup
            default: r = f12_sqr(a); break;
        }
    }
    store_f12(out, r);
}

}  // namespace

void launch_f12_op(int op, const uint8_t* in, uint8_t* out, cudaStream_t s) {
    f12_op_kernel<<<1, 32, 0, s>>>(op, in, out);
}

size_t pairing_scratch_bytes(uint32_t n) { return sizeof(Fq12) * (n ? n : 1); }

void launch_pairing_finish(uint32_t n, uint8_t* scratch, uint8_t* out384, int* is_one,
                           cudaStream_t s) {
    product_final_kernel<<<1, 128, 0, s>>>(n, scratch, out384, is_one);
}

void launch_pairing_product(uint32_t n, const uint8_t* g1s, const uint8_t* g2s, uint8_t* scratch,
                            uint8_t* out384, int* is_one, cudaStream_t s) {
    if (n) miller_kernel<<<(n + 63) / 64, 64, 0, s>>>(n, g1s, g2s, scratch);
    product_final_kernel<<<1, 128, 0, s>>>(n, scratch, out384, is_one);
}

}  // namespace bn
}  // namespace ace_gpu
