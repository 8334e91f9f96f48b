// The C ABI of include/acegpu.h: contexts, device workspaces, host<->device
// marshalling and the pipelines that chain the mock-Prove kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <array>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/acegpu.h"
#include "bn_kernels.cuh"
#include "g16_kernels.cuh"
#include "mock_kernels.cuh"
#include "phase1.cuh"
#include "pairing_kernels.cuh"
#include "g16_verify.cuh"
#include "msm.cuh"
#include "ntt.cuh"
#include "r1cs.cuh"
#include "witprog.cuh"

#ifndef ACEGPU_GIT
#define ACEGPU_GIT "dev"
#endif

using namespace ace_gpu;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CK(expr)                                                                        \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess)                                                          \
            return fail(ACEGPU_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

#define CKL()                                                                           \
    do {                                                                                \
        cudaError_t _e = cudaGetLastError();                                            \
        if (_e != cudaSuccess)                                                          \
            return fail(ACEGPU_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(_e)); \
    } while (0)

#define RET(expr)                   \
    do {                            \
        int _r = (expr);            \
        if (_r != ACEGPU_OK) return _r; \
    } while (0)

enum Slot {
    kPayloads, kOffs, kAtts, kHeader, kRevs, kRevIdx, kCodes, kNodesA, kNodesB, kMerkA, kMerkB,
    kBlockHash, kOut, kIn2, kMisc, kBnA, kBnB, kBnOut, kBnScratch, kSegRoots, kSegMerk,
    kKeytab, kKeydom, kP1Scratch, kP1Hash, kP1Reg, kErr, kG16Wit, kG16Roots, kNumSlots
};

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
};

uint32_t ceil_log2(uint64_t n) {
    uint32_t l = 0;
    while ((1ull << l) < n) ++l;
    return l;
}

}  // namespace

struct BlockGraph;
void free_block_graph(BlockGraph* g);

struct acegpu_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::mutex mu;
    std::atomic<uint64_t> launches{0};
    DevBuf bufs[kNumSlots];
    // Optional per-phase CUDA events (leaves | levels | finalize) recorded on
    // the launching stream by the block pipeline.
    bool timing = false;
    bool ev_recorded = false;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    // BN254: NTT twiddle tables per log-size, MSM scratch.
    ace_gpu::bn::NttTables ntt[ace_gpu::bn::kNttMaxLog + 1];
    ace_gpu::bn::Ntt3Tables ntt3[ace_gpu::bn::kNtt3MaxLog + 1];  // N = 3 * 2^k
    ace_gpu::bn::MsmScratch msm;
    // Segmented block pipeline: sub-contexts (own stream + workspace).
    cudaStream_t copy_stream = nullptr;  // overlapped host-input pipeline
    std::vector<cudaEvent_t> seg_events;
    cudaStream_t leaf_streams[8] = {};
    cudaEvent_t leaf_events[8] = {};
    bool force_single = false;  // acegpu_set_segmented(ctx, 0) forces the single-pass pipeline
    // attest-key cache of the call in flight (launch_keytab / launch_credentials)
    const uint32_t* cur_keytab = nullptr;
    const uint8_t* cur_keydom = nullptr;
    uint32_t cur_n_revs = 0;  // REV table size of the call in flight (index guard)
    int* cur_err = nullptr;   // device flag: an out-of-range rev_index was seen
    // CUDA-graph replay of the host-buffer pipeline (acegpu_attest_prove_certify_graph)
    struct BlockGraph* graph = nullptr;
    // Side stream of the attestation credential check (keytab + credential
    // kernels), overlapping the leaf kernel and the tree levels.
    cudaStream_t cred_stream = nullptr;
    cudaEvent_t cred_in = nullptr, cred_out = nullptr;
};

// A prepared MSM: fixed base (proving-key bases with their window shifts)
// or variable base (the bases alone; vb_sub = sub-range size, 0 = default).
struct acegpu_msm_bases {
    int device = 0;
    int group = 1;
    uint64_t n = 0;
    uint8_t* table = nullptr;  // kMsmWindows * n (vb: n) affine points, Montgomery form
    int vb = 0;
    uint64_t vb_sub = 0;
    uint64_t lo = 0;  // a split key's slice: bases [lo, lo + n) of the full array
};

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// Grow-only device workspace. Growth synchronises the device (the old buffer
// may still be read by in-flight work on any stream).
int ensure(acegpu_ctx* c, Slot s, size_t bytes, void** out) {
    DevBuf& b = c->bufs[s];
    if (bytes == 0) bytes = 16;
    if (b.cap < bytes) {
        if (b.p) {
            CK(cudaDeviceSynchronize());
            CK(cudaFree(b.p));
            b.p = nullptr;
            b.cap = 0;
        }
        size_t cap = std::max(bytes + 64, b.cap * 3 / 2);
        CK(cudaMalloc(&b.p, cap));
        b.cap = cap;
    }
    *out = b.p;
    return ACEGPU_OK;
}

template <class T>
int ws(acegpu_ctx* c, Slot s, size_t bytes, T** out) {
    void* p = nullptr;
    RET(ensure(c, s, bytes, &p));
    *out = static_cast<T*>(p);
    return ACEGPU_OK;
}

int h2d(acegpu_ctx* c, Slot s, const void* src, size_t bytes, cudaStream_t st, void** out) {
    RET(ensure(c, s, bytes, out));
    if (bytes) CK(cudaMemcpyAsync(*out, src, bytes, cudaMemcpyHostToDevice, st));
    return ACEGPU_OK;
}

template <class T>
int h2d_t(acegpu_ctx* c, Slot s, const T* src, size_t bytes, cudaStream_t st, T** out) {
    void* p = nullptr;
    RET(h2d(c, s, src, bytes, st, &p));
    *out = static_cast<T*>(p);
    return ACEGPU_OK;
}

// `_dev` calls run on the caller's stream exactly as given: NULL is CUDA's
// legacy default stream (what torch.cuda.current_stream() reports as 0).
cudaStream_t pick(acegpu_ctx*, void* stream) { return static_cast<cudaStream_t>(stream); }

struct TreeResult {
    uint8_t* nodes = nullptr;   // level nodes (320 B each)
    uint8_t* merkle = nullptr;  // level merkle nodes (32 B each)
    uint8_t* bh = nullptr;      // block hash (when a header was given)
    uint32_t count = 0;
};

int side_stream(acegpu_ctx* c) {
    if (!c->cred_stream) {
        CK(cudaStreamCreateWithFlags(&c->cred_stream, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->cred_in, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->cred_out, cudaEventDisableTiming));
    }
    return ACEGPU_OK;
}

// Leaves (+attestation verdicts, merkle leaves, header hash) and up to
// `max_levels` fused proof/merkle levels. With lift, a lone merkle node keeps
// self-pairing until max_levels (aligned-chunk roots).
int run_tree(acegpu_ctx* c, cudaStream_t s, const uint8_t* payloads, const uint64_t* offs,
             const uint8_t* atts, uint32_t n, const uint8_t* header, const uint8_t* revs,
             const uint32_t* rev_index, uint8_t* codes, bool prove, uint32_t max_levels,
             bool lift, TreeResult* r) {
    uint8_t *na = nullptr, *nb = nullptr, *ma = nullptr, *mb = nullptr, *bh = nullptr;
    const size_t half = n / 2 + 1;
    if (prove) {
        RET(ws(c, kNodesA, size_t(kNodeBytes) * n, &na));
        RET(ws(c, kNodesB, size_t(kNodeBytes) * half, &nb));
    }
    RET(ws(c, kMerkA, 32ull * n, &ma));
    RET(ws(c, kMerkB, 32ull * half, &mb));
    RET(ws(c, kBlockHash, 32, &bh));
    LeafArgs a{};
    a.payloads = payloads;
    a.offs = offs;
    a.atts = atts;
    a.n = n;
    a.codes = codes;
    a.nodes = prove ? na : nullptr;
    a.merkle = ma;
    a.header = header;
    a.block_hash = bh;
    if (c->timing) CK(cudaEventRecord(c->ev[0], s));
    if (n || header) {
        launch_leaves(a, s);
        CKL();
        c->launches++;
    }
    if (c->timing) CK(cudaEventRecord(c->ev[1], s));
    const bool cred = codes && n;
    if (cred) {
        // credential verdicts on the side stream, concurrent with the levels
        RET(side_stream(c));
        CK(cudaEventRecord(c->cred_in, s));
        CK(cudaStreamWaitEvent(c->cred_stream, c->cred_in, 0));
        launch_credentials(atts, n, revs, rev_index, c->cur_keytab, c->cur_keydom, codes,
                           c->cur_n_revs, c->cur_err, c->cred_stream);
        CKL();
        c->launches++;
        CK(cudaEventRecord(c->cred_out, c->cred_stream));
    }
    uint32_t cur = n, lv = 0;
    uint8_t *nin = na, *nout = nb, *min_ = ma, *mout = mb;
    while (lv < max_levels && (cur > 1 || (lift && cur == 1))) {
        launch_level(prove ? nin : nullptr, cur, nout, min_, cur, mout, lift, s);
        CKL();
        c->launches++;
        cur = (cur + 1) / 2;
        std::swap(nin, nout);
        std::swap(min_, mout);
        ++lv;
    }
    if (cred) CK(cudaStreamWaitEvent(s, c->cred_out, 0));
    if (c->timing) CK(cudaEventRecord(c->ev[2], s));
    r->nodes = nin;
    r->merkle = min_;
    r->bh = bh;
    r->count = cur;
    return ACEGPU_OK;
}

int check_n(uint64_t n) {
    if (n > 0xFFFFFFFFull / kNodeBytes) return fail(ACEGPU_EINVAL, "batch too large");
    return ACEGPU_OK;
}

// Whole-block pipeline on device buffers: -> proof289 + fc328 (either may be null).
int block_pipeline(acegpu_ctx* c, cudaStream_t s, const uint8_t* payloads, const uint64_t* offs,
                   const uint8_t* atts, uint32_t n, const uint8_t* header, const uint8_t* revs,
                   const uint32_t* rev_index, uint8_t* codes, uint8_t* out289, uint8_t* out328) {
    TreeResult t;
    RET(run_tree(c, s, payloads, offs, atts, n, header, revs, rev_index, codes, true, 64, false,
                 &t));
    launch_finalize(t.nodes, n ? t.merkle : nullptr, header, t.bh, n == 0, out289, out328, s);
    CKL();
    c->launches++;
    if (c->timing) {
        CK(cudaEventRecord(c->ev[3], s));
        c->ev_recorded = true;
    }
    return ACEGPU_OK;
}

// Attest-key cache for one call: keytab for every REV under the domain at
// d_dom8 (tx 0's), consumed by the credential kernel through ctx->cur_keytab.
struct KeytabScope {
    acegpu_ctx* c;
    explicit KeytabScope(acegpu_ctx* ctx) : c(ctx) {}
    ~KeytabScope() {
        c->cur_keytab = nullptr;
        c->cur_keydom = nullptr;
        c->cur_n_revs = 0;
        c->cur_err = nullptr;
    }
    int build(cudaStream_t s, const uint8_t* d_revs, uint64_t n_revs, const uint8_t* d_dom8) {
        c->cur_n_revs = uint32_t(std::min<uint64_t>(n_revs, 0xFFFFFFFFull));
        if (!d_revs || !n_revs || n_revs > 0xFFFFFFFFull) return ACEGPU_OK;
        uint32_t* kt;
        RET(ws(c, kKeytab, 64 * n_revs, &kt));
        // on the credential side stream: off the leaf kernel's critical path
        RET(side_stream(c));
        CK(cudaEventRecord(c->cred_in, s));
        CK(cudaStreamWaitEvent(c->cred_stream, c->cred_in, 0));
        launch_keytab(d_revs, uint32_t(n_revs), d_dom8, kt, c->cred_stream);
        CKL();
        c->launches++;
        c->cur_keytab = kt;
        c->cur_keydom = d_dom8;
        return ACEGPU_OK;
    }
};

struct HostBlock;
int overlapped_pipeline(acegpu_ctx* c, cudaStream_t s, const uint8_t* payloads,
                        const uint64_t* offs, const uint8_t* atts, uint64_t n,
                        const uint8_t* header, const uint8_t* revs, const uint32_t* rev_index,
                        uint8_t* codes, uint8_t* out289, uint8_t* out328, const HostBlock& host,
                        const uint32_t* host_rix);

// Large blocks take the segmented pipeline, except under phase timing (whose
// leaves | levels | finalize split needs the single-pass pipeline).
inline bool use_segments(const acegpu_ctx* c, uint64_t n) {
    return !c->timing && !c->force_single && n >= (2ull << 13);
}

struct HostBlock {
    const uint8_t* payloads;
    const uint64_t* offs;
    const uint8_t* atts;
    uint64_t n;
};

// Upload a flat block; returns device pointers (payload offsets are kept as given).
int upload_block(acegpu_ctx* c, cudaStream_t s, const HostBlock& h, uint8_t** dp, uint64_t** doff,
                 uint8_t** da) {
    if (h.n == 0) {  // empty block: inputs may be NULL
        RET(ws(c, kPayloads, 16, dp));
        RET(ws(c, kOffs, 16, doff));
        RET(ws(c, kAtts, 16, da));
        return ACEGPU_OK;
    }
    const uint64_t pbytes = h.offs[h.n];
    RET(h2d_t(c, kPayloads, h.payloads, pbytes, s, dp));
    RET(h2d_t(c, kOffs, h.offs, 8 * (h.n + 1), s, doff));
    RET(h2d_t(c, kAtts, h.atts, 104 * h.n, s, da));
    return ACEGPU_OK;
}

}  // namespace

// =========================================================================
extern "C" {

const char* acegpu_last_error(void) { return g_err.c_str(); }

const char* acegpu_version(void) { return "acegpu sm_100a " ACEGPU_GIT; }

int acegpu_create(int device, acegpu_ctx** out) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return fail(ACEGPU_ENODEV, "no CUDA device");
    }
    if (device < 0 || device >= count) return fail(ACEGPU_ENODEV, "bad device index");
    cudaDeviceProp prop{};
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
        return fail(ACEGPU_ENODEV, std::string("libacegpu is built for sm_100a; device is ") +
                                       prop.name);
    }
    DeviceGuard g(device);
    auto* c = new acegpu_ctx();
    c->device = device;
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return fail(ACEGPU_ECUDA, cudaGetErrorString(e));
    }
    *out = c;
    return ACEGPU_OK;
}

void acegpu_destroy(acegpu_ctx* c) {
    if (!c) return;
    DeviceGuard g(c->device);
    cudaStreamSynchronize(c->stream);
    free_block_graph(c->graph);
    c->graph = nullptr;
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    for (auto& t : c->ntt) t.release();
    for (auto& t : c->ntt3) t.release();
    c->msm.release();
    for (auto& e : c->seg_events) cudaEventDestroy(e);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);

    if (c->cred_stream) {
        cudaStreamSynchronize(c->cred_stream);
        cudaStreamDestroy(c->cred_stream);
        cudaEventDestroy(c->cred_in);
        cudaEventDestroy(c->cred_out);
    }
    for (int k = 0; k < 8; ++k) {
        if (c->leaf_streams[k]) cudaStreamDestroy(c->leaf_streams[k]);
        if (c->leaf_events[k]) cudaEventDestroy(c->leaf_events[k]);
    }
    for (auto& b : c->bufs)
        if (b.p) cudaFree(b.p);
    cudaStreamDestroy(c->stream);
    delete c;
}

uint64_t acegpu_launch_count(const acegpu_ctx* c) { return c ? c->launches.load() : 0; }

int acegpu_set_segmented(acegpu_ctx* c, int enable) {
    std::lock_guard<std::mutex> lk(c->mu);
    c->force_single = !enable;
    return ACEGPU_OK;
}

int acegpu_set_phase_timing(acegpu_ctx* c, int enable) {
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    if (enable && !c->ev[0]) {
        for (auto& e : c->ev) CK(cudaEventCreate(&e));
    }
    c->timing = enable != 0;
    c->ev_recorded = false;
    return ACEGPU_OK;
}

int acegpu_phase_times(acegpu_ctx* c, float* ms3) {
    std::lock_guard<std::mutex> lk(c->mu);
    if (!c->timing || !c->ev_recorded) return fail(ACEGPU_EINVAL, "no timed block pipeline yet");
    DeviceGuard g(c->device);
    CK(cudaEventSynchronize(c->ev[3]));
    for (int i = 0; i < 3; ++i) CK(cudaEventElapsedTime(&ms3[i], c->ev[i], c->ev[i + 1]));
    return ACEGPU_OK;
}

void* acegpu_host_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes ? bytes : 1) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}

void acegpu_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

// ---------------------------------------------------------------- SHA-256
int acegpu_sha256_varlen(acegpu_ctx* c, const uint8_t* data, const uint64_t* offs, uint64_t n,
                         uint8_t* out) {
    RET(check_n(n));
    if (n == 0) return ACEGPU_OK;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    uint8_t* dd;
    uint64_t* doff;
    uint8_t* dout;
    RET(h2d_t(c, kPayloads, data, offs[n], s, &dd));
    RET(h2d_t(c, kOffs, offs, 8 * (n + 1), s, &doff));
    RET(ws(c, kOut, 32 * n, &dout));
    launch_sha256_varlen(dd, doff, uint32_t(n), dout, s);
    CKL();
    c->launches++;
    CK(cudaMemcpyAsync(out, dout, 32 * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ACEGPU_OK;
}

int acegpu_sha256_strided(acegpu_ctx* c, const uint8_t* base, uint64_t stride, uint64_t len,
                          uint64_t n, uint8_t* out) {
    RET(check_n(n));
    if (n == 0) return ACEGPU_OK;
    if (len > 0xFFFFFFFFull) return fail(ACEGPU_EINVAL, "message too long");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    uint8_t *dd, *dout;
    RET(h2d_t(c, kPayloads, base, stride * (n - 1) + len, s, &dd));
    RET(ws(c, kOut, 32 * n, &dout));
    launch_sha256_strided(dd, stride, uint32_t(len), uint32_t(n), dout, s);
    CKL();
    c->launches++;
    CK(cudaMemcpyAsync(out, dout, 32 * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ACEGPU_OK;
}

// ------------------------------------------------------------ mock prover
int acegpu_prove_public_inputs(acegpu_ctx* c, const uint8_t* pubs, uint64_t n, uint8_t* out289) {
    RET(check_n(n));
    if (n == 0) return ACEGPU_OK;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    uint8_t *dp, *nodes, *dout;
    RET(h2d_t(c, kIn2, pubs, 160 * n, s, &dp));
    RET(ws(c, kNodesA, size_t(kNodeBytes) * n, &nodes));
    RET(ws(c, kOut, 289 * n, &dout));
    launch_prove_public_inputs(dp, uint32_t(n), nodes, s);
    launch_pack_nodes(nodes, uint32_t(n), dout, s);
    CKL();
    c->launches += 2;
    CK(cudaMemcpyAsync(out289, dout, 289 * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ACEGPU_OK;
}

int acegpu_prove_txs(acegpu_ctx* c, const uint8_t* payloads, const uint64_t* offs,
                     const uint8_t* atts, uint64_t n, uint8_t* out289) {
    RET(check_n(n));
    if (n == 0) return ACEGPU_OK;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    uint8_t *dp, *da, *nodes, *dout;
    uint64_t* doff;
    RET(upload_block(c, s, {payloads, offs, atts, n}, &dp, &doff, &da));
    RET(ws(c, kNodesA, size_t(kNodeBytes) * n, &nodes));
    RET(ws(c, kOut, 289 * n, &dout));
    LeafArgs a{};
    a.payloads = dp;
    a.offs = doff;
    a.atts = da;
    a.n = uint32_t(n);
    a.nodes = nodes;
    launch_leaves(a, s);
    launch_pack_nodes(nodes, uint32_t(n), dout, s);
    CKL();
    c->launches += 2;
    CK(cudaMemcpyAsync(out289, dout, 289 * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ACEGPU_OK;
}

int acegpu_verify_mock(acegpu_ctx* c, const uint8_t* proofs, uint64_t n, uint8_t* ok) {
    RET(check_n(n));
    if (n == 0) return ACEGPU_OK;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    uint8_t *dp, *nodes, *dok;
    RET(h2d_t(c, kIn2, proofs, 289 * n, s, &dp));
    RET(ws(c, kNodesA, size_t(kNodeBytes) * n, &nodes));
    RET(ws(c, kOut, n, &dok));
    launch_unpack_nodes(dp, uint32_t(n), nodes, s);
    launch_verify_mock(nodes, uint32_t(n), dok, s);
    CKL();
    c->launches += 2;
    CK(cudaMemcpyAsync(ok, dok, n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ACEGPU_OK;
}

int acegpu_aggregate_pairs(acegpu_ctx* c, const uint8_t* a289, const uint8_t* b289, uint64_t n,
                           uint8_t* out289) {
    RET(check_n(n));
    if (n == 0) return ACEGPU_OK;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    uint8_t *da, *db, *na, *nb, *dout;
    RET(h2d_t(c, kIn2, a289, 289 * n, s, &da));
    RET(h2d_t(c, kMisc, b289, 289 * n, s, &db));
    RET(ws(c, kNodesA, size_t(kNodeBytes) * 2 * n, &na));
    RET(ws(c, kNodesB, size_t(kNodeBytes) * n, &nb));
    RET(ws(c, kOut, 289 * n, &dout));
    launch_unpack_nodes(da, uint32_t(n), na, s);
    launch_unpack_nodes(db, uint32_t(n), na + size_t(kNodeBytes) * n, s);
    launch_aggregate_pairs(na, na + size_t(kNodeBytes) * n, uint32_t(n), nb, s);
    launch_pack_nodes(nb, uint32_t(n), dout, s);
    CKL();
    c->launches += 4;
    CK(cudaMemcpyAsync(out289, dout, 289 * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ACEGPU_OK;
}

int acegpu_aggregate_tree(acegpu_ctx* c, const uint8_t* proofs, uint64_t n, uint8_t* out289,
                          uint64_t* levels, uint64_t* pair_ops) {
    if (n == 0) return fail(ACEGPU_EINVAL, "aggregate_tree: empty proof list");
    RET(check_n(n));
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    uint8_t *dp, *na, *nb, *dout;
    RET(h2d_t(c, kIn2, proofs, 289 * n, s, &dp));
    RET(ws(c, kNodesA, size_t(kNodeBytes) * n, &na));
    RET(ws(c, kNodesB, size_t(kNodeBytes) * (n / 2 + 1), &nb));
    RET(ws(c, kOut, 289, &dout));
    launch_unpack_nodes(dp, uint32_t(n), na, s);
    CKL();
    c->launches++;
    uint32_t cur = uint32_t(n);
    while (cur > 1) {
        launch_level(na, cur, nb, nullptr, 0, nullptr, false, s);
        CKL();
        c->launches++;
        cur = (cur + 1) / 2;
        std::swap(na, nb);
    }
    launch_pack_nodes(na, 1, dout, s);
    CKL();
    c->launches++;
    CK(cudaMemcpyAsync(out289, dout, 289, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (levels) *levels = ceil_log2(n);
    if (pair_ops) *pair_ops = n - 1;
    return ACEGPU_OK;
}

}  // extern "C"

namespace {
// Host-buffer attest+prove+certify on stream s; sync = wait for completion.
int apc_host(acegpu_ctx* c, cudaStream_t s, bool sync, const uint8_t* payloads,
             const uint64_t* offs, const uint8_t* atts, uint64_t n, const uint8_t* header,
             const uint8_t* revs, uint64_t n_revs, const uint32_t* rev_index, uint8_t* codes,
             uint8_t* out289, uint8_t* out328) {
    RET(check_n(n));
    if (codes && n && (!revs || !rev_index || n_revs == 0))
        return fail(ACEGPU_EINVAL, "attestation needs a REV table and index");
    if (n_revs > 0xFFFFFFFFull) return fail(ACEGPU_EINVAL, "REV table too large");
    // rev_index bounds are checked on the device (credential_kernel), not in an
    // O(n) host loop ahead of the copies (measured ~45 us of the 100k e2e)
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    uint8_t *dp, *da, *dh, *dout, *dr = nullptr, *dc = nullptr;
    uint64_t* doff;
    uint32_t* dri = nullptr;
    int* derr = nullptr;
    RET(h2d_t(c, kHeader, header, 256, s, &dh));
    RET(ws(c, kOut, 289 + 328 + 16, &dout));
    KeytabScope kts(c);
    if (codes && n) {
        RET(ws(c, kErr, 16, &derr));
        CK(cudaMemsetAsync(derr, 0, sizeof(int), s));
    }
    uint8_t* dkeydom = nullptr;
    if (codes && n) {
        RET(h2d_t(c, kRevs, revs, 32 * n_revs, s, &dr));
        RET(h2d_t(c, kKeydom, atts + 64, 8, s, &dkeydom));  // tx 0's domain
        RET(kts.build(s, dr, n_revs, dkeydom));
        c->cur_err = derr;
    }
    if (use_segments(c, n)) {
        // REV table first; offset/payload/attestation slices are copied per
        // segment on the copy streams, overlapping the compute of earlier ones
        const HostBlock hb{payloads, offs, atts, n};
        RET(ws(c, kPayloads, offs[n] + 16, &dp));
        RET(ws(c, kAtts, 104 * n + 16, &da));
        RET(ws(c, kOffs, 8 * (n + 1), &doff));  // copied per segment
        if (codes) {
            RET(ws(c, kRevIdx, 4 * n, &dri));
            RET(ws(c, kCodes, n, &dc));
        }
        RET(overlapped_pipeline(c, s, dp, doff, da, n, dh, dr, dri, dc, dout, dout + 304, hb,
                                codes ? rev_index : nullptr));
    } else {
        RET(upload_block(c, s, {payloads, offs, atts, n}, &dp, &doff, &da));
        if (codes && n) {
            RET(h2d_t(c, kRevIdx, rev_index, 4 * n, s, &dri));
            RET(ws(c, kCodes, n, &dc));
        }
        RET(block_pipeline(c, s, dp, doff, da, uint32_t(n), dh, dr, dri, dc, dout, dout + 304));
    }
    if (dc) CK(cudaMemcpyAsync(codes, dc, n, cudaMemcpyDeviceToHost, s));
    if (out289) CK(cudaMemcpyAsync(out289, dout, 289, cudaMemcpyDeviceToHost, s));
    if (out328) CK(cudaMemcpyAsync(out328, dout + 304, 328, cudaMemcpyDeviceToHost, s));
    int herr = 0;
    if (derr && sync) CK(cudaMemcpyAsync(&herr, derr, sizeof(int), cudaMemcpyDeviceToHost, s));
    if (sync) CK(cudaStreamSynchronize(s));
    if (herr) return fail(ACEGPU_EINVAL, "rev_index out of range");
    return ACEGPU_OK;
}
}  // namespace

extern "C" {

int acegpu_attest_prove_certify(acegpu_ctx* c, const uint8_t* payloads, const uint64_t* offs,
                                const uint8_t* atts, uint64_t n, const uint8_t* header,
                                const uint8_t* revs, uint64_t n_revs, const uint32_t* rev_index,
                                uint8_t* codes, uint8_t* out289, uint8_t* out328,
                                uint64_t* levels, uint64_t* pair_ops) {
    RET(apc_host(c, c->stream, true, payloads, offs, atts, n, header, revs, n_revs, rev_index,
                 codes, out289, out328));
    if (levels) *levels = n ? ceil_log2(n) : 0;
    if (pair_ops) *pair_ops = n ? n - 1 : 0;
    return ACEGPU_OK;
}

int acegpu_attest_prove_certify_async(acegpu_ctx* c, void* stream, const uint8_t* payloads,
                                      const uint64_t* offs, const uint8_t* atts, uint64_t n,
                                      const uint8_t* header, const uint8_t* revs,
                                      uint64_t n_revs, const uint32_t* rev_index,
                                      uint8_t* codes, uint8_t* out289, uint8_t* out328) {
    return apc_host(c, pick(c, stream), false, payloads, offs, atts, n, header, revs, n_revs,
                    rev_index, codes, out289, out328);
}

}  // extern "C"

// One captured host-buffer pipeline (apc_host) for a block shape, replayed
// with its memcpy nodes re-pointed at the next block's host buffers.
struct BlockGraph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaStream_t stream = nullptr;
    std::vector<uint64_t> key;
    // host ranges of the captured call: 0 payloads 1 offs 2 atts 3 header
    // 4 revs 5 rev_index (H2D sources), 6 codes 7 out289 8 out328 (D2H targets)
    const uint8_t* base[9] = {};
    uint64_t len[9] = {};
    struct Node {
        cudaGraphNode_t node;
        int role;
        uint64_t off, bytes;
        void* dev;
        bool h2d;
    };
    std::vector<Node> nodes;
    uint64_t kernels = 0;
    ~BlockGraph() {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
    }
};

void free_block_graph(BlockGraph* g) {
    if (!g) return;
    if (g->stream) cudaStreamSynchronize(g->stream);
    delete g;
}

namespace {
struct ApcArgs {
    const uint8_t* payloads;
    const uint64_t* offs;
    const uint8_t* atts;
    uint64_t n;
    const uint8_t* header;
    const uint8_t* revs;
    uint64_t n_revs;
    const uint32_t* rev_index;
    uint8_t* codes;
    uint8_t* out289;
    uint8_t* out328;
    void ranges(const uint8_t** b, uint64_t* l) const {
        const uint8_t* p[9] = {payloads, reinterpret_cast<const uint8_t*>(offs), atts, header, revs,
                               reinterpret_cast<const uint8_t*>(rev_index), codes, out289, out328};
        const uint64_t pb = n ? offs[n] : 0;
        const uint64_t q[9] = {pb, 8 * (n + 1), 104 * n, 256, 32 * n_revs, 4 * n, n, 289, 328};
        for (int k = 0; k < 9; ++k) {
            b[k] = p[k];
            l[k] = p[k] ? q[k] : 0;
        }
    }
};

std::vector<uint64_t> graph_key(const ApcArgs& a, cudaStream_t s) {
    std::vector<uint64_t> k = {a.n, a.n ? a.offs[a.n] : 0, a.n_revs, uint64_t(uintptr_t(s)),
                               uint64_t(a.codes != nullptr), uint64_t(a.out289 != nullptr),
                               uint64_t(a.out328 != nullptr)};
    // segment boundaries of the host pipeline (payload offsets baked into copies)
    for (uint64_t i = 0; i <= a.n; i += 1 << 13) k.push_back(a.offs[i]);
    if (a.n) k.push_back(a.offs[a.n]);
    return k;
}

int capture_block_graph(acegpu_ctx* c, cudaStream_t s, const ApcArgs& a, BlockGraph* g) {
    const uint64_t launches0 = c->launches.load();
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    const int rc = apc_host(c, s, false, a.payloads, a.offs, a.atts, a.n, a.header, a.revs,
                            a.n_revs, a.rev_index, a.codes, a.out289, a.out328);
    cudaGraph_t graph = nullptr;
    const cudaError_t e = cudaStreamEndCapture(s, &graph);
    g->kernels = c->launches.load() - launches0;
    c->launches = launches0;  // nothing ran: replays count them
    if (rc != ACEGPU_OK || e != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        return rc != ACEGPU_OK ? rc : fail(ACEGPU_ECUDA, cudaGetErrorString(e));
    }
    g->graph = graph;
    CK(cudaGraphInstantiate(&g->exec, graph, 0));
    a.ranges(g->base, g->len);
    size_t nn = 0;
    CK(cudaGraphGetNodes(graph, nullptr, &nn));
    std::vector<cudaGraphNode_t> all(nn);
    CK(cudaGraphGetNodes(graph, all.data(), &nn));
    for (cudaGraphNode_t nd : all) {
        cudaGraphNodeType t;
        CK(cudaGraphNodeGetType(nd, &t));
        if (t != cudaGraphNodeTypeMemcpy) continue;
        cudaMemcpy3DParms p{};
        CK(cudaGraphMemcpyNodeGetParams(nd, &p));
        const bool h2d = p.kind == cudaMemcpyHostToDevice;
        const uint8_t* host = static_cast<const uint8_t*>(h2d ? p.srcPtr.ptr : p.dstPtr.ptr);
        void* dev = h2d ? p.dstPtr.ptr : p.srcPtr.ptr;
        if (p.kind != cudaMemcpyHostToDevice && p.kind != cudaMemcpyDeviceToHost) continue;
        int role = -1;
        for (int k = 0; k < 9; ++k)
            if (g->base[k] && host >= g->base[k] && host < g->base[k] + std::max<uint64_t>(g->len[k], 1))
                role = k;
        if (role < 0) return fail(ACEGPU_ECUDA, "graph: unmapped host copy");
        g->nodes.push_back({nd, role, uint64_t(host - g->base[role]), uint64_t(p.extent.width),
                            dev, h2d});
    }
    g->stream = s;
    return ACEGPU_OK;
}
}  // namespace

extern "C" {

int acegpu_attest_prove_certify_graph(acegpu_ctx* c, void* stream, const uint8_t* payloads,
                                      const uint64_t* offs, const uint8_t* atts, uint64_t n,
                                      const uint8_t* header, const uint8_t* revs,
                                      uint64_t n_revs, const uint32_t* rev_index,
                                      uint8_t* codes, uint8_t* out289, uint8_t* out328) {
    cudaStream_t s = pick(c, stream);
    if (!s) return fail(ACEGPU_EINVAL, "graph replay needs an explicit stream");
    const ApcArgs a{payloads, offs, atts, n, header, revs, n_revs, rev_index, codes, out289, out328};
    const std::vector<uint64_t> key = graph_key(a, s);
    if (!c->graph || c->graph->key != key) {
        // this block with plain launches (sizes the workspace), then capture
        // the same call for the following blocks of this shape
        RET(apc_host(c, s, false, payloads, offs, atts, n, header, revs, n_revs, rev_index,
                     codes, out289, out328));
        free_block_graph(c->graph);  // waits for its replays in flight
        c->graph = nullptr;
        auto* g = new BlockGraph();
        DeviceGuard dg(c->device);
        const int rc = capture_block_graph(c, s, a, g);  // apc_host takes c->mu itself
        if (rc != ACEGPU_OK) {
            delete g;
            return rc;
        }
        g->key = key;
        c->graph = g;
        return ACEGPU_OK;
    }
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    BlockGraph* g = c->graph;
    const uint8_t* b[9];
    uint64_t l[9];
    a.ranges(b, l);
    for (const auto& nd : g->nodes) {
        uint8_t* host = const_cast<uint8_t*>(b[nd.role]) + nd.off;
        if (nd.h2d)
            CK(cudaGraphExecMemcpyNodeSetParams1D(g->exec, nd.node, nd.dev, host, nd.bytes,
                                                  cudaMemcpyHostToDevice));
        else
            CK(cudaGraphExecMemcpyNodeSetParams1D(g->exec, nd.node, host, nd.dev, nd.bytes,
                                                  cudaMemcpyDeviceToHost));
    }
    CK(cudaGraphLaunch(g->exec, s));
    c->launches += g->kernels;
    return ACEGPU_OK;
}

int acegpu_attest_prove_certify_dev(acegpu_ctx* c, void* stream, const uint8_t* payloads,
                                    const uint64_t* offs, const uint8_t* atts, uint64_t n,
                                    const uint8_t* header, const uint8_t* revs, uint64_t n_revs,
                                    const uint32_t* rev_index, uint8_t* codes, uint8_t* out289,
                                    uint8_t* out328) {
    RET(check_n(n));
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = pick(c, stream);
    KeytabScope kts(c);
    if (codes && n) RET(kts.build(s, revs, n_revs, atts + 64));
    return block_pipeline(c, s, payloads, offs, atts, uint32_t(n), header, revs, rev_index,
                          n ? codes : nullptr, out289, out328);
}

int acegpu_prove_block(acegpu_ctx* c, const uint8_t* payloads, const uint64_t* offs,
                       const uint8_t* atts, uint64_t n, const uint8_t* header, uint8_t* out289,
                       uint64_t* levels, uint64_t* pair_ops) {
    return acegpu_attest_prove_certify(c, payloads, offs, atts, n, header, nullptr, 0, nullptr,
                                       nullptr, out289, nullptr, levels, pair_ops);
}

int acegpu_build_fc(acegpu_ctx* c, const uint8_t* atts, uint64_t n, const uint8_t* header,
                    const uint8_t* proof289, uint8_t* out328) {
    RET(check_n(n));
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    uint8_t *da, *dh, *dproof, *node, *dout;
    RET(h2d_t(c, kAtts, atts, 104 * n, s, &da));
    RET(h2d_t(c, kHeader, header, 256, s, &dh));
    RET(h2d_t(c, kIn2, proof289, 289, s, &dproof));
    RET(ws(c, kMisc, kNodeBytes, &node));
    RET(ws(c, kOut, 328, &dout));
    launch_unpack_nodes(dproof, 1, node, s);
    CKL();
    c->launches++;
    TreeResult t;
    RET(run_tree(c, s, nullptr, nullptr, da, uint32_t(n), dh, nullptr, nullptr, nullptr, false,
                 64, false, &t));
    launch_finalize(node, n ? t.merkle : nullptr, dh, t.bh, false, nullptr, dout, s);
    CKL();
    c->launches++;
    CK(cudaMemcpyAsync(out328, dout, 328, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ACEGPU_OK;
}

int acegpu_verify_fc(acegpu_ctx* c, const uint8_t* fc, const uint8_t* payloads,
                     const uint64_t* offs, const uint8_t* atts, uint64_t n,
                     const uint8_t* header, int* out_check) {
    // prover.cpp:158-169: slot, then block hash, then the full recompute.
    if (std::memcmp(fc + 32, header, 8) != 0) {
        *out_check = 1;
        return ACEGPU_OK;
    }
    uint8_t expect[328];
    RET(acegpu_attest_prove_certify(c, payloads, offs, atts, n, header, nullptr, 0, nullptr,
                                    nullptr, nullptr, expect, nullptr, nullptr));
    if (std::memcmp(expect, fc, 32) != 0) *out_check = 2;
    else if (std::memcmp(expect + 40, fc + 40, 256) != 0) *out_check = 3;
    else if (std::memcmp(expect + 296, fc + 296, 32) != 0) *out_check = 3;
    else *out_check = 0;
    return ACEGPU_OK;
}

int acegpu_bn_pairing(acegpu_ctx* c, uint64_t n, const uint8_t* g1s, const uint8_t* g2s,
                      uint8_t* out384, int* is_one) {
    if (n > (1u << 20)) return fail(ACEGPU_EINVAL, "too many pairs");
    if (n && (!g1s || !g2s)) return fail(ACEGPU_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    uint8_t *d1 = nullptr, *d2 = nullptr, *scratch, *out;
    if (n) {
        RET(h2d_t(c, kBnA, g1s, 64 * n, s, &d1));
        RET(h2d_t(c, kBnB, g2s, 128 * n, s, &d2));
    }
    RET(ws(c, kBnScratch, bn::pairing_scratch_bytes(uint32_t(n)), &scratch));
    RET(ws(c, kBnOut, 384 + 16, &out));
    bn::launch_pairing_product(uint32_t(n), d1, d2, scratch, out,
                               reinterpret_cast<int*>(out + 384), s);
    CKL();
    c->launches += n ? 2 : 1;
    if (out384) CK(cudaMemcpyAsync(out384, out, 384, cudaMemcpyDeviceToHost, s));
    if (is_one) CK(cudaMemcpyAsync(is_one, out + 384, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ACEGPU_OK;
}

int acegpu_bn_f12_op(acegpu_ctx* c, int op, const uint8_t* in384, uint8_t* out384) {
    if (op < 0 || op > 11 || !in384 || !out384) return fail(ACEGPU_EINVAL, "bad f12 op");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    uint8_t *din, *dout;
    RET(h2d_t(c, kBnA, in384, op >= 10 ? 392 : 384, s, &din));
    RET(ws(c, kBnOut, 384, &dout));
    bn::launch_f12_op(op, din, dout, s);
    CKL();
    c->launches++;
    CK(cudaMemcpyAsync(out384, dout, 384, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ACEGPU_OK;
}

// ---- Phase 1a ----------------------------------------------------------
int acegpu_light_check_dev(acegpu_ctx* c, void* stream, const uint8_t* payloads,
                           const uint64_t* offs, const uint8_t* atts, uint64_t n,
                           const uint8_t* registry, uint64_t n_registry, uint64_t current_slot,
                           uint64_t window_slots, uint8_t* codes, uint8_t* tx_hashes) {
    RET(check_n(n));
    if (n == 0) return ACEGPU_OK;
    if (!codes || (n_registry && !registry)) return fail(ACEGPU_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    launch_light_check(payloads, offs, atts, uint32_t(n), registry, n_registry, current_slot,
                       window_slots, codes, tx_hashes, pick(c, stream));
    CKL();
    c->launches++;
    return ACEGPU_OK;
}

int acegpu_light_check(acegpu_ctx* c, const uint8_t* payloads, const uint64_t* offs,
                       const uint8_t* atts, uint64_t n, const uint8_t* registry,
                       uint64_t n_registry, uint64_t current_slot, uint64_t window_slots,
                       uint8_t* codes, uint64_t* counters3) {
    RET(check_n(n));
    if (counters3) counters3[0] = counters3[1] = counters3[2] = 0;
    if (n == 0) return ACEGPU_OK;
    if (!codes || (n_registry && !registry)) return fail(ACEGPU_EINVAL, "null argument");
    {
        std::lock_guard<std::mutex> lk(c->mu);
        DeviceGuard g(c->device);
        cudaStream_t s = c->stream;
        uint8_t *dp, *da, *dr = nullptr, *dc;
        uint64_t* doff;
        RET(upload_block(c, s, {payloads, offs, atts, n}, &dp, &doff, &da));
        if (n_registry) RET(h2d_t(c, kP1Reg, registry, 32 * n_registry, s, &dr));
        RET(ws(c, kCodes, n, &dc));
        launch_light_check(dp, doff, da, uint32_t(n), dr, n_registry, current_slot, window_slots,
                           dc, nullptr, s);
        CKL();
        c->launches++;
        CK(cudaMemcpyAsync(codes, dc, n, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    if (counters3) {  // every tx hashes its payload; later stages run only if reached
        counters3[0] = n;
        for (uint64_t i = 0; i < n; ++i) {
            counters3[1] += codes[i] != 1;
            counters3[2] += codes[i] == 0 || codes[i] == 3;
        }
    }
    return ACEGPU_OK;
}

int acegpu_build_block_dev(acegpu_ctx* c, void* stream, const uint8_t* payloads,
                           const uint64_t* offs, const uint8_t* atts, uint64_t n,
                           const uint8_t* codes, const uint8_t* header_tmpl,
                           uint8_t* out_payloads, uint64_t* out_offs, uint8_t* out_atts,
                           uint8_t* out_header, uint64_t* n_accepted) {
    RET(check_n(n));
    if (!header_tmpl || !out_header || !out_offs || !n_accepted)
        return fail(ACEGPU_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = pick(c, stream);
    uint8_t *scratch, *hash, *ma, *mb;
    RET(ws(c, kP1Scratch, compact_scratch_bytes(uint32_t(n)), &scratch));
    RET(ws(c, kP1Hash, 96ull * n + 64, &hash));
    uint8_t *txh = hash, *ctxh = hash + 32ull * n, *cath = hash + 64ull * n,
            *roots = hash + 96ull * n;
    if (n) {
        launch_sha256_varlen(payloads, offs, uint32_t(n), txh, s);  // tx Merkle leaves
        CKL();
        c->launches++;
    }
    uint32_t *d_count;
    uint64_t* d_total;
    CK(launch_compact(payloads, offs, atts, uint32_t(n), codes, txh, scratch, out_payloads,
                      out_offs, out_atts, ctxh, cath, &d_count, &d_total, s));
    c->launches += n ? 4 : 3;
    uint32_t cnt = 0;
    CK(cudaMemcpyAsync(&cnt, d_count, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    // tx_merkle_root and attest_merkle_root over the accepted txs (wire.cpp:223-273)
    if (cnt) {
        RET(ws(c, kMerkA, 32ull * cnt, &ma));
        RET(ws(c, kMerkB, 32ull * (cnt / 2 + 1), &mb));
        for (int r = 0; r < 2; ++r) {
            uint8_t *a = ma, *b = mb;
            launch_merkle_leaves(r ? cath : ctxh, cnt, a, s);
            CKL();
            c->launches++;
            for (uint32_t cur = cnt; cur > 1; cur = (cur + 1) / 2) {
                launch_level(nullptr, 0, nullptr, a, cur, b, false, s);
                CKL();
                c->launches++;
                std::swap(a, b);
            }
            CK(cudaMemcpyAsync(roots + 32 * r, a, 32, cudaMemcpyDeviceToDevice, s));
        }
    }
    launch_header(header_tmpl, d_count, d_total, out_offs, roots, roots + 32, out_header, s);
    CKL();
    c->launches++;
    *n_accepted = cnt;
    return ACEGPU_OK;
}

int acegpu_merkle_root(acegpu_ctx* c, const uint8_t* leaves, uint64_t n, uint8_t* out32) {
    RET(check_n(n));
    if (n == 0) {
        std::memset(out32, 0, 32);
        return ACEGPU_OK;
    }
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    uint8_t *dl, *ma, *mb;
    RET(h2d_t(c, kIn2, leaves, 32 * n, s, &dl));
    RET(ws(c, kMerkA, 32 * n, &ma));
    RET(ws(c, kMerkB, 32 * (n / 2 + 1), &mb));
    launch_merkle_leaves(dl, uint32_t(n), ma, s);
    CKL();
    c->launches++;
    uint32_t cur = uint32_t(n);
    while (cur > 1) {
        launch_level(nullptr, 0, nullptr, ma, cur, mb, false, s);
        CKL();
        c->launches++;
        cur = (cur + 1) / 2;
        std::swap(ma, mb);
    }
    CK(cudaMemcpyAsync(out32, ma, 32, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ACEGPU_OK;
}

int acegpu_block_hash(acegpu_ctx* c, const uint8_t* header, uint8_t* out32) {
    return acegpu_sha256_strided(c, header, 256, 256, 1, out32);
}

// ------------------------------------------------------------- sharding
}  // extern "C"

namespace {
int shard_impl(acegpu_ctx* c, cudaStream_t s, const uint8_t* payloads, const uint64_t* offs,
               const uint8_t* atts, uint64_t n, uint64_t n_total, uint32_t log2_chunk,
               const uint8_t* revs, const uint32_t* rev_index, uint8_t* codes, uint8_t* roots289,
               uint8_t* merkle32);
int combine_impl(acegpu_ctx* c, cudaStream_t s, const uint8_t* roots289, const uint8_t* merkle32,
                 uint64_t n_chunks, uint64_t n_total, const uint8_t* header, uint8_t* out289,
                 uint8_t* out328);
}  // namespace

extern "C" {

int acegpu_shard_roots_dev(acegpu_ctx* c, void* stream, const uint8_t* payloads,
                           const uint64_t* offs, const uint8_t* atts, uint64_t n, uint64_t n_total,
                           uint32_t log2_chunk, const uint8_t* revs, uint64_t n_revs,
                           const uint32_t* rev_index, uint8_t* codes, uint8_t* roots289,
                           uint8_t* merkle32) {
    RET(check_n(n));
    if (n == 0 || log2_chunk > 31) return fail(ACEGPU_EINVAL, "empty shard or chunk too large");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = pick(c, stream);
    KeytabScope kts(c);
    if (codes) RET(kts.build(s, revs, n_revs, atts + 64));
    return shard_impl(c, s, payloads, offs, atts, n, n_total, log2_chunk, revs, rev_index, codes,
                      roots289, merkle32);
}

int acegpu_combine_roots_dev(acegpu_ctx* c, void* stream, const uint8_t* roots289,
                             const uint8_t* merkle32, uint64_t n_chunks, uint64_t n_total,
                             const uint8_t* header, uint8_t* out289, uint8_t* out328) {
    RET(check_n(n_chunks));
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    return combine_impl(c, pick(c, stream), roots289, merkle32, n_chunks, n_total, header, out289,
                        out328);
}

}  // extern "C"

namespace {
int shard_impl(acegpu_ctx* c, cudaStream_t s, const uint8_t* payloads, const uint64_t* offs,
               const uint8_t* atts, uint64_t n, uint64_t n_total, uint32_t log2_chunk,
               const uint8_t* revs, const uint32_t* rev_index, uint8_t* codes, uint8_t* roots289,
               uint8_t* merkle32) {
    const bool lift = n_total > (1ull << log2_chunk);
    TreeResult t;
    RET(run_tree(c, s, payloads, offs, atts, uint32_t(n), nullptr, revs, rev_index, codes, true,
                 log2_chunk, lift, &t));
    const uint64_t chunks = (n + (1ull << log2_chunk) - 1) >> log2_chunk;
    if (t.count != chunks) return fail(ACEGPU_EINVAL, "internal: chunk count mismatch");
    launch_pack_nodes(t.nodes, t.count, roots289, s);
    CKL();
    c->launches++;
    CK(cudaMemcpyAsync(merkle32, t.merkle, 32ull * t.count, cudaMemcpyDeviceToDevice, s));
    return ACEGPU_OK;
}

int combine_impl(acegpu_ctx* c, cudaStream_t s, const uint8_t* roots289, const uint8_t* merkle32,
                 uint64_t n_chunks, uint64_t n_total, const uint8_t* header, uint8_t* out289,
                 uint8_t* out328) {
    uint8_t *na, *nb, *ma, *mb, *bh;
    RET(ws(c, kBlockHash, 32, &bh));
    launch_sha256_strided(header, 256, 256, 1, bh, s);
    CKL();
    c->launches++;
    if (n_total == 0 || n_chunks == 0) {
        launch_finalize(nullptr, nullptr, header, bh, true, out289, out328, s);
        CKL();
        c->launches++;
        return ACEGPU_OK;
    }
    RET(ws(c, kNodesA, size_t(kNodeBytes) * n_chunks, &na));
    RET(ws(c, kNodesB, size_t(kNodeBytes) * (n_chunks / 2 + 1), &nb));
    RET(ws(c, kMerkA, 32 * n_chunks, &ma));
    RET(ws(c, kMerkB, 32 * (n_chunks / 2 + 1), &mb));
    launch_unpack_nodes(roots289, uint32_t(n_chunks), na, s);
    CKL();
    c->launches++;
    CK(cudaMemcpyAsync(ma, merkle32, 32 * n_chunks, cudaMemcpyDeviceToDevice, s));
    uint32_t cur = uint32_t(n_chunks);
    while (cur > 1) {
        launch_level(na, cur, nb, ma, cur, mb, false, s);
        CKL();
        c->launches++;
        cur = (cur + 1) / 2;
        std::swap(na, nb);
        std::swap(ma, mb);
    }
    launch_finalize(na, ma, header, bh, false, out289, out328, s);
    CKL();
    c->launches++;
    return ACEGPU_OK;
}

// Host-input block pipeline with the H2D copy overlapped: the payload,
// attestation and REV-index slices of 2^kSegLog-tx segments are copied on a
// copy stream while the leaf kernel of earlier segments runs on the compute
// stream; the tree levels and the FC then follow as in block_pipeline.
#ifndef ACEGPU_SEG_LOG
#define ACEGPU_SEG_LOG 14  // 100k e2e (tools/e2e_probe.py): 2^13 1.20 ms, 2^14 1.08, 2^15 1.12
#endif
constexpr uint32_t kSegLog = ACEGPU_SEG_LOG;
constexpr int kLeafStreams = 8;

int ensure_copy(acegpu_ctx* c, size_t nev) {
    if (!c->copy_stream) {
        CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));

        for (int k = 0; k < kLeafStreams; ++k) {
            CK(cudaStreamCreateWithFlags(&c->leaf_streams[k], cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&c->leaf_events[k], cudaEventDisableTiming));
        }
    }
    while (c->seg_events.size() < nev) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->seg_events.push_back(e);
    }
    return ACEGPU_OK;
}

int overlapped_pipeline(acegpu_ctx* c, cudaStream_t s, const uint8_t* payloads,
                        const uint64_t* offs, const uint8_t* atts, uint64_t n,
                        const uint8_t* header, const uint8_t* revs, const uint32_t* rev_index,
                        uint8_t* codes, uint8_t* out289, uint8_t* out328, const HostBlock& host,
                        const uint32_t* host_rix) {
    const uint64_t seg = 1ull << kSegLog, S = (n + seg - 1) / seg;
    RET(ensure_copy(c, S + 1));
    // Level-major node arrays: level L >= 1 occupies [off[L], off[L] + ceil(n / 2^L))
    // of nb / mb, so the subtrees of different segments (aligned 2^kSegLog
    // ranges) write disjoint slices of every level and can run concurrently.
    uint64_t off[66], tot = 0;
    off[0] = 0;
    for (uint32_t L = 1; L < 66; ++L) {
        off[L] = tot;
        tot += (n + (1ull << std::min(L, 63u)) - 1) >> std::min(L, 63u);
    }
    // levels run per segment on the segment's stream (the rest on s)
    static const uint32_t sub = [] {
        const char* e = getenv("ACEGPU_SEG_LEVELS");
        return e ? std::min<uint32_t>(uint32_t(atoi(e)), kSegLog) : kSegLog;
    }();
    uint8_t *na, *nb, *ma, *mb, *bh;
    RET(ws(c, kNodesA, size_t(kNodeBytes) * n, &na));
    RET(ws(c, kNodesB, size_t(kNodeBytes) * (tot + 2), &nb));
    RET(ws(c, kMerkA, 32ull * n, &ma));
    RET(ws(c, kMerkB, 32ull * (tot + 2), &mb));
    RET(ws(c, kBlockHash, 32, &bh));
    auto nodes_at = [&](uint32_t L, uint64_t i) {
        return L ? nb + size_t(kNodeBytes) * (off[L] + i) : na + size_t(kNodeBytes) * i;
    };
    auto merk_at = [&](uint32_t L, uint64_t i) { return L ? mb + 32 * (off[L] + i) : ma + 32 * i; };
    // the copy stream starts after what is already enqueued on s (offsets, REVs, header)
    // ACEGPU_TRACE=1: per-segment timeline on stderr (debug; adds a sync)
    static const bool trace = getenv("ACEGPU_TRACE") != nullptr;
    std::vector<cudaEvent_t> tev;
    auto mark = [&](cudaStream_t st) {
        if (!trace) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        tev.push_back(e);
    };
    mark(s);
    CK(cudaEventRecord(c->seg_events[S], s));
    CK(cudaStreamWaitEvent(c->copy_stream, c->seg_events[S], 0));
    const bool lift = n > seg;  // short last segment: Merkle self-pairing up to level kSegLog
    const bool cred = codes != nullptr;
    if (cred) RET(side_stream(c));
    for (uint64_t j = 0; j < S; ++j) {
        const uint64_t a = j * seg, cnt = std::min(seg, n - a);
        const uint64_t b0 = host.offs[a], b1 = host.offs[a + cnt];
        // (one copy stream: a second one split by field measured no faster,
        // ~43 GB/s either way on this PCIe 5 x16 host)
        if (j == 0) {
            // offsets and REV indices of the whole block first (1.2 MB in two
            // copies; per-segment slices measured ~15 us slower end to end)
            CK(cudaMemcpyAsync(const_cast<uint64_t*>(offs), host.offs, 8 * (n + 1),
                               cudaMemcpyHostToDevice, c->copy_stream));
            if (host_rix)
                CK(cudaMemcpyAsync(const_cast<uint32_t*>(rev_index), host_rix, 4 * n,
                                   cudaMemcpyHostToDevice, c->copy_stream));
        }
        CK(cudaMemcpyAsync(const_cast<uint8_t*>(payloads) + b0, host.payloads + b0, b1 - b0,
                           cudaMemcpyHostToDevice, c->copy_stream));
        CK(cudaMemcpyAsync(const_cast<uint8_t*>(atts) + 104 * a, host.atts + 104 * a, 104 * cnt,
                           cudaMemcpyHostToDevice, c->copy_stream));
        CK(cudaEventRecord(c->seg_events[j], c->copy_stream));
        // Each segment's leaves AND its subtree (levels 1..kSegLog) on its own
        // stream: they overlap the copies of later segments and each other
        // (a segment's narrow levels alone would leave the GPU idle).
        cudaStream_t ls = c->leaf_streams[j % kLeafStreams];
        CK(cudaStreamWaitEvent(ls, c->seg_events[j], 0));
        mark(ls);
        LeafArgs la{};
        la.payloads = payloads;
        la.offs = offs + a;
        la.atts = atts + 104 * a;
        la.n = uint32_t(cnt);
        la.codes = codes ? codes + a : nullptr;
        la.nodes = na + size_t(kNodeBytes) * a;
        la.merkle = ma + 32 * a;
        la.header = j == 0 ? header : nullptr;
        la.block_hash = bh;
        launch_leaves(la, ls);
        CKL();
        c->launches++;
        mark(ls);
        if (cred) {
            CK(cudaEventRecord(c->leaf_events[j % kLeafStreams], ls));
            CK(cudaStreamWaitEvent(c->cred_stream, c->leaf_events[j % kLeafStreams], 0));
            launch_credentials(atts + 104 * a, uint32_t(cnt), revs, rev_index + a,
                               c->cur_keytab, c->cur_keydom, codes + a, c->cur_n_revs,
                               c->cur_err, c->cred_stream);
            CKL();
            c->launches++;
        }
        uint64_t cur = cnt;
        for (uint32_t L = 0; L < sub && (cur > 1 || (lift && cur == 1)); ++L) {
            launch_level(nodes_at(L, a >> L), uint32_t(cur), nodes_at(L + 1, a >> (L + 1)),
                         merk_at(L, a >> L), uint32_t(cur), merk_at(L + 1, a >> (L + 1)), lift, ls);
            CKL();
            c->launches++;
            cur = (cur + 1) / 2;
        }
        mark(ls);
    }
    for (int k = 0; k < int(std::min<uint64_t>(S, kLeafStreams)); ++k) {  // the streams used
        CK(cudaEventRecord(c->leaf_events[k], c->leaf_streams[k]));
        CK(cudaStreamWaitEvent(s, c->leaf_events[k], 0));
    }
    if (cred) {
        CK(cudaEventRecord(c->cred_out, c->cred_stream));
        CK(cudaStreamWaitEvent(s, c->cred_out, 0));
    }
    // the rest of the tree from level `sub` (the concatenated segment slices
    // are the global level array), reference rules
    uint32_t L = sub;
    uint64_t cur = (n + (1ull << sub) - 1) >> sub;
    while (cur > 1) {
        launch_level(nodes_at(L, 0), uint32_t(cur), nodes_at(L + 1, 0), merk_at(L, 0),
                     uint32_t(cur), merk_at(L + 1, 0), false, s);
        CKL();
        c->launches++;
        cur = (cur + 1) / 2;
        ++L;
    }
    mark(s);
    const uint8_t *root = nodes_at(L, 0), *mroot = merk_at(L, 0);
    launch_finalize(root, mroot, header, bh, false, out289, out328, s);
    CKL();
    c->launches++;
    if (trace) {
        mark(s);
        cudaStreamSynchronize(s);
        std::string line = "acegpu trace (us):";
        for (size_t k = 1; k < tev.size(); ++k) {
            float ms = 0;
            cudaEventElapsedTime(&ms, tev[0], tev[k]);
            char buf[32];
            snprintf(buf, sizeof buf, " %.0f", 1e3 * ms);
            line += buf;
            if (k < tev.size() - 2 && k % 3 == 0) line += " |";
        }
        fprintf(stderr, "%s\n", line.c_str());
        for (auto e : tev) cudaEventDestroy(e);
    }
    return ACEGPU_OK;
}

}  // namespace

extern "C" {

// ------------------------------------------------------------ attestation
int acegpu_attest_verify(acegpu_ctx* c, const uint8_t* payloads, const uint64_t* offs,
                         const uint8_t* atts, uint64_t n, const uint8_t* revs, uint64_t n_revs,
                         const uint32_t* rev_index, uint8_t* codes) {
    RET(check_n(n));
    if (n == 0) return ACEGPU_OK;
    if (!revs || !rev_index || n_revs == 0) return fail(ACEGPU_EINVAL, "REV table required");
    for (uint64_t i = 0; i < n; ++i)
        if (rev_index[i] >= n_revs) return fail(ACEGPU_EINVAL, "rev_index out of range");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    uint8_t *dp, *da, *dr, *dc;
    uint64_t* doff;
    uint32_t* dri;
    RET(upload_block(c, s, {payloads, offs, atts, n}, &dp, &doff, &da));
    RET(h2d_t(c, kRevs, revs, 32 * n_revs, s, &dr));
    RET(h2d_t(c, kRevIdx, rev_index, 4 * n, s, &dri));
    RET(ws(c, kCodes, n, &dc));
    LeafArgs a{};
    a.payloads = dp;
    a.offs = doff;
    a.atts = da;
    a.n = uint32_t(n);
    a.codes = dc;
    launch_leaves(a, s);  // payload verdicts
    CKL();
    uint32_t* kt;
    RET(ws(c, kKeytab, 64 * n_revs, &kt));
    launch_keytab(dr, uint32_t(n_revs), da + 64, kt, s);  // tx 0's domain
    CKL();
    launch_credentials(da, uint32_t(n), dr, dri, kt, da + 64, dc, uint32_t(n_revs), nullptr, s);
    CKL();
    c->launches += 3;
    CK(cudaMemcpyAsync(codes, dc, n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ACEGPU_OK;
}

int acegpu_attest_generate_dev(acegpu_ctx* c, void* stream, const uint8_t* payloads,
                               const uint64_t* offs, uint64_t n, const uint8_t* revs,
                               const uint32_t* rev_index, const uint8_t* doms8,
                               const uint8_t* id_coms, uint8_t* out104) {
    RET(check_n(n));
    if (n == 0) return ACEGPU_OK;
    DeviceGuard g(c->device);
    launch_attest_generate(payloads, offs, uint32_t(n), revs, rev_index, doms8, id_coms, out104,
                           pick(c, stream));
    CKL();
    c->launches++;
    return ACEGPU_OK;
}

int acegpu_attest_generate(acegpu_ctx* c, const uint8_t* payloads, const uint64_t* offs,
                           uint64_t n, const uint8_t* revs, uint64_t n_revs,
                           const uint32_t* rev_index, const uint8_t* doms8,
                           const uint8_t* id_coms, uint8_t* out104) {
    RET(check_n(n));
    if (n == 0) return ACEGPU_OK;
    for (uint64_t i = 0; i < n; ++i)
        if (rev_index[i] >= n_revs) return fail(ACEGPU_EINVAL, "rev_index out of range");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    uint8_t *dp, *dr, *dd, *di, *dout;
    uint64_t* doff;
    uint32_t* dri;
    RET(h2d_t(c, kPayloads, payloads, offs[n], s, &dp));
    RET(h2d_t(c, kOffs, offs, 8 * (n + 1), s, &doff));
    RET(h2d_t(c, kRevs, revs, 32 * n_revs, s, &dr));
    RET(h2d_t(c, kRevIdx, rev_index, 4 * n, s, &dri));
    RET(h2d_t(c, kIn2, doms8, 8 * n, s, &dd));
    RET(h2d_t(c, kMisc, id_coms, 32 * n, s, &di));
    RET(ws(c, kOut, 104 * n, &dout));
    launch_attest_generate(dp, doff, uint32_t(n), dr, dri, dd, di, dout, s);
    CKL();
    c->launches++;
    CK(cudaMemcpyAsync(out104, dout, 104 * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ACEGPU_OK;
}

int acegpu_derive_attest_keys(acegpu_ctx* c, const uint8_t* revs, const uint8_t* doms8,
                              uint64_t n, uint8_t* out32) {
    RET(check_n(n));
    if (n == 0) return ACEGPU_OK;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    uint8_t *dr, *dd, *dout;
    RET(h2d_t(c, kRevs, revs, 32 * n, s, &dr));
    RET(h2d_t(c, kIn2, doms8, 8 * n, s, &dd));
    RET(ws(c, kOut, 32 * n, &dout));
    launch_derive_attest_keys(dr, dd, uint32_t(n), dout, s);
    CKL();
    c->launches++;
    CK(cudaMemcpyAsync(out32, dout, 32 * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ACEGPU_OK;
}

// --------------------------------------------------------------- witnesses
int acegpu_witness_check(acegpu_ctx* c, const uint8_t* w, const uint32_t* wlens,
                         const uint8_t* atts, uint64_t n, uint8_t* ok) {
    RET(check_n(n));
    if (n == 0) return ACEGPU_OK;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    uint8_t *dw, *da, *dok;
    uint32_t* dl = nullptr;
    RET(h2d_t(c, kIn2, w, 256 * n, s, &dw));
    RET(h2d_t(c, kAtts, atts, 104 * n, s, &da));
    if (wlens) RET(h2d_t(c, kRevIdx, wlens, 4 * n, s, &dl));
    RET(ws(c, kOut, n, &dok));
    launch_witness_check(dw, dl, da, uint32_t(n), dok, s);
    CKL();
    c->launches++;
    CK(cudaMemcpyAsync(ok, dok, n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ACEGPU_OK;
}

int acegpu_build_witness(acegpu_ctx* c, const uint8_t* keys, const uint8_t* txh, uint64_t n,
                         uint8_t* out) {
    RET(check_n(n));
    if (n == 0) return ACEGPU_OK;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    uint8_t *dk, *dt, *dout;
    RET(h2d_t(c, kIn2, keys, 32 * n, s, &dk));
    RET(h2d_t(c, kMisc, txh, 32 * n, s, &dt));
    RET(ws(c, kOut, 256 * n, &dout));
    launch_build_witness(dk, dt, uint32_t(n), dout, s);
    CKL();
    c->launches++;
    CK(cudaMemcpyAsync(out, dout, 256 * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ACEGPU_OK;
}

int acegpu_witness_xor(acegpu_ctx* c, const uint8_t* master, const uint8_t* txh,
                       const uint64_t* masks, const uint8_t* in, uint64_t len, uint64_t n,
                       uint8_t* out) {
    RET(check_n(n));
    if (n == 0 || len == 0) return ACEGPU_OK;
    if (len > (1u << 20)) return fail(ACEGPU_EINVAL, "witness too long");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    uint8_t *dm, *dt, *din, *dout;
    uint64_t* dmask;
    RET(h2d_t(c, kHeader, master, 32, s, &dm));
    RET(h2d_t(c, kMisc, txh, 32 * n, s, &dt));
    RET(h2d_t(c, kOffs, masks, 8 * n, s, &dmask));
    RET(h2d_t(c, kIn2, in, len * n, s, &din));
    RET(ws(c, kOut, len * n, &dout));
    launch_witness_xor(dm, dt, dmask, din, uint32_t(len), uint32_t(n), dout, s);
    CKL();
    c->launches++;
    CK(cudaMemcpyAsync(out, dout, len * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ACEGPU_OK;
}

// ------------------------------------------------------------- measurement
int acegpu_sha256_peak(acegpu_ctx* c, double* cps) {
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    uint32_t* sink;
    RET(ws(c, kMisc, 16, &sink));
    const int threads = 128, blocks = sms * 8;
    const uint32_t iters = 1024;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    launch_sha256_peak(sink, 64, blocks, threads, s);  // warm-up
    CK(cudaEventRecord(e0, s));
    launch_sha256_peak(sink, iters, blocks, threads, s);
    CK(cudaEventRecord(e1, s));
    CKL();
    c->launches += 2;
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *cps = double(blocks) * threads * iters / (ms * 1e-3);
    return ACEGPU_OK;
}

}  // extern "C"

extern "C" int acegpu_sha256_probe(acegpu_ctx* c, int blocks, int threads, uint32_t iters,
                                   double* seconds) {
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    uint32_t* sink;
    RET(ws(c, kMisc, 16, &sink));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    launch_sha256_peak(sink, 16, blocks, threads, s);  // warm-up
    CK(cudaEventRecord(e0, s));
    launch_sha256_peak(sink, iters, blocks, threads, s);
    CK(cudaEventRecord(e1, s));
    CKL();
    c->launches += 2;
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *seconds = ms * 1e-3;
    return ACEGPU_OK;
}

// ===================================================================== BN254
// North-star additions. No reference counterpart.
namespace {

int bn_time(acegpu_ctx* c, cudaStream_t s, void (*launch)(void*), void* arg, float* ms) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    launch(arg);  // warm-up
    CK(cudaEventRecord(e0, s));
    launch(arg);
    CK(cudaEventRecord(e1, s));
    CKL();
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    (void)c;
    return ACEGPU_OK;
}

}  // namespace

extern "C" int acegpu_bn_field_batch(acegpu_ctx* c, int field, int op, const uint8_t* a,
                                     const uint8_t* b, uint64_t n, uint8_t* out) {
    if (field < 0 || field > 1 || op < 0 || op > 4) return fail(ACEGPU_EINVAL, "bad field/op");
    if (n == 0) return ACEGPU_OK;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    uint8_t *da, *db = nullptr, *dout;
    RET(h2d_t(c, kBnA, a, 32 * n, s, &da));
    if (b && op <= 2) RET(h2d_t(c, kBnB, b, 32 * n, s, &db));
    RET(ws(c, kBnOut, 32 * n, &dout));
    bn::launch_field_batch(field, op, da, db, n, dout, s);
    CKL();
    c->launches++;
    CK(cudaMemcpyAsync(out, dout, 32 * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ACEGPU_OK;
}

extern "C" int acegpu_bn_convert_dev(acegpu_ctx* c, void* stream, int field, uint8_t* d_data,
                                     uint64_t n, int to_mont) {
    DeviceGuard g(c->device);
    cudaStream_t s = pick(c, stream);
    if (field == 1) bn::launch_fr_convert(d_data, n, to_mont, s);
    else bn::launch_fq_convert(d_data, n, to_mont, s);
    CKL();
    c->launches++;
    return ACEGPU_OK;
}

extern "C" int acegpu_bn_ntt_dev(acegpu_ctx* c, void* stream, const uint8_t* d_in, uint8_t* d_out,
                                 uint32_t logn, int inverse, int coset) {
    if (logn > (uint32_t)bn::kNttMaxLog) return fail(ACEGPU_EINVAL, "NTT size above 2^28");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = pick(c, stream);
    if (bn::ntt_tables(c->ntt[logn], (int)logn, s)) return fail(ACEGPU_ECUDA, "NTT tables");
    uint8_t* scratch = nullptr;
    if ((int)logn > bn::kNttSingleMax) RET(ws(c, kBnScratch, 32ull << logn, &scratch));
    if (bn::ntt_run(c->ntt[logn], d_in, d_out, scratch, inverse, coset, 1, s))
        return fail(ACEGPU_ECUDA, std::string("NTT launch: ") + cudaGetErrorString(cudaGetLastError()));
    c->launches += (int)logn > bn::kNttTwoPassMax ? 3 : (int)logn > bn::kNttSingleMax ? 2 : 1;
    return ACEGPU_OK;
}

// Mixed radix N = 3 * 2^logk (device, Montgomery form).
extern "C" int acegpu_bn_ntt3_dev(acegpu_ctx* c, void* stream, const uint8_t* d_in,
                                  uint8_t* d_out, uint32_t logk, int inverse, int coset) {
    if (logk > (uint32_t)bn::kNtt3MaxLog) return fail(ACEGPU_EINVAL, "NTT size above 3 x 2^26");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = pick(c, stream);
    if (bn::ntt_tables(c->ntt[logk], (int)logk, s) || bn::ntt3_tables(c->ntt3[logk], (int)logk, s))
        return fail(ACEGPU_ECUDA, "NTT tables");
    const uint64_t M = 1ull << logk;
    uint8_t* scratch;
    RET(ws(c, kBnScratch, 32 * (3 * M + 3 * M), &scratch));
    if (bn::ntt3_run(c->ntt3[logk], c->ntt[logk], d_in, d_out, scratch, scratch + 96 * M, inverse,
                     coset, s))
        return fail(ACEGPU_ECUDA, std::string("NTT3 launch: ") + cudaGetErrorString(cudaGetLastError()));
    c->launches += 5;
    return ACEGPU_OK;
}

extern "C" int acegpu_bn_ntt3(acegpu_ctx* c, uint8_t* data, uint32_t logk, int inverse,
                              int coset) {
    if (logk > (uint32_t)bn::kNtt3MaxLog) return fail(ACEGPU_EINVAL, "NTT size above 3 x 2^26");
    const uint64_t n = 3ull << logk;
    uint8_t* d;
    {
        std::lock_guard<std::mutex> lk(c->mu);
        DeviceGuard g(c->device);
        RET(h2d_t(c, kBnA, data, 32 * n, c->stream, &d));
        bn::launch_fr_convert(d, n, 1, c->stream);
        CKL();
    }
    RET(acegpu_bn_ntt3_dev(c, c->stream, d, d, logk, inverse, coset));
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    bn::launch_fr_convert(d, n, 0, c->stream);
    CKL();
    CK(cudaMemcpyAsync(data, d, 32 * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return ACEGPU_OK;
}

extern "C" int acegpu_bn_ntt(acegpu_ctx* c, uint8_t* data, uint32_t logn, int inverse,
                             int coset) {
    if (logn > (uint32_t)bn::kNttMaxLog) return fail(ACEGPU_EINVAL, "NTT size above 2^28");
    const uint64_t n = 1ull << logn;
    uint8_t* d;
    {
        std::lock_guard<std::mutex> lk(c->mu);
        DeviceGuard g(c->device);
        RET(h2d_t(c, kBnA, data, 32 * n, c->stream, &d));
        bn::launch_fr_convert(d, n, 1, c->stream);
        CKL();
    }
    RET(acegpu_bn_ntt_dev(c, c->stream, d, d, logn, inverse, coset));
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    bn::launch_fr_convert(d, n, 0, c->stream);
    CKL();
    c->launches += 2;
    CK(cudaMemcpyAsync(data, d, 32 * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return ACEGPU_OK;
}

extern "C" int acegpu_bn_scalar_muls(acegpu_ctx* c, int group, const uint8_t* base,
                                     const uint8_t* scalars, uint64_t n, uint8_t* out) {
    if (group != 1 && group != 2) return fail(ACEGPU_EINVAL, "group must be 1 or 2");
    if (n == 0) return ACEGPU_OK;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    const uint64_t pb = 64ull * group;
    uint8_t *dbase, *dsc, *dout;
    RET(h2d_t(c, kBnA, base, pb, s, &dbase));
    RET(h2d_t(c, kBnB, scalars, 32 * n, s, &dsc));
    RET(ws(c, kBnOut, pb * n, &dout));
    bn::launch_points_convert(group, dbase, 1, 1, s);
    bn::launch_scalar_muls(group, dbase, dsc, n, dout, s);
    bn::launch_points_convert(group, dout, n, 0, s);
    CKL();
    c->launches += 3;
    CK(cudaMemcpyAsync(out, dout, pb * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ACEGPU_OK;
}

extern "C" int acegpu_bn_msm_params(acegpu_ctx* c, int* window_bits, int* windows) {
    if (!window_bits || !windows) return fail(ACEGPU_EINVAL, "null output");
    (void)c;
    *window_bits = bn::kMsmC;
    *windows = bn::kMsmWindows;
    return ACEGPU_OK;
}

namespace {
int msm_prepare_impl(acegpu_ctx* c, int group, const uint8_t* points, uint64_t n, int on_device,
                     int vb, uint64_t sub, acegpu_msm_bases** out) {
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    const uint64_t pb = 64ull * group;
    // owned until success: every error path frees the table and the staging copy
    std::unique_ptr<acegpu_msm_bases, void (*)(acegpu_msm_bases*)> b(new acegpu_msm_bases(),
                                                                      acegpu_bn_msm_free);
    b->device = c->device;
    b->group = group;
    b->n = n;
    b->vb = vb;
    b->vb_sub = sub;
    const auto kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (vb) {
        // variable base: the bases themselves, converted in place
        cudaError_t e = cudaMalloc(&b->table, pb * n);
        if (e != cudaSuccess)
            return fail(ACEGPU_ECUDA, std::string("msm_prepare alloc: ") + cudaGetErrorString(e));
        CK(cudaMemcpyAsync(b->table, points, pb * n, kind, s));
        bn::launch_points_convert(group, b->table, n, 1, s);
        CKL();
        CK(cudaStreamSynchronize(s));
        c->launches += 1;
        *out = b.release();
        return ACEGPU_OK;
    }
    std::unique_ptr<uint8_t, cudaError_t (*)(void*)> tmp(nullptr, cudaFree);
    cudaError_t e = cudaMalloc(&b->table, pb * n * bn::kMsmWindows);
    uint8_t* t = nullptr;
    if (e == cudaSuccess) e = cudaMalloc(&t, pb * n);
    tmp.reset(t);
    if (e != cudaSuccess)
        return fail(ACEGPU_ECUDA, std::string("msm_prepare alloc: ") + cudaGetErrorString(e));
    CK(cudaMemcpyAsync(t, points, pb * n, kind, s));
    bn::launch_points_convert(group, t, n, 1, s);
    if (bn::msm_prepare(group, t, n, b->table, s)) return fail(ACEGPU_ECUDA, "msm_prepare launch");
    CK(cudaStreamSynchronize(s));
    c->launches += 2;
    *out = b.release();
    return ACEGPU_OK;
}
}  // namespace

extern "C" int acegpu_bn_msm_prepare(acegpu_ctx* c, int group, const uint8_t* points,
                                     uint64_t n, int on_device, acegpu_msm_bases** out) {
    if (group != 1 && group != 2) return fail(ACEGPU_EINVAL, "group must be 1 or 2");
    if (n == 0 || n > (1ull << 27)) return fail(ACEGPU_EINVAL, "MSM size must be 1..2^27");
    if (!points || !out) return fail(ACEGPU_EINVAL, "null argument");
    return msm_prepare_impl(c, group, points, n, on_device, 0, 0, out);
}

extern "C" int acegpu_bn_msm_prepare_vb(acegpu_ctx* c, int group, const uint8_t* points,
                                        uint64_t n, int on_device, uint64_t sub,
                                        acegpu_msm_bases** out) {
    if (group != 1 && group != 2) return fail(ACEGPU_EINVAL, "group must be 1 or 2");
    if (n == 0 || n > (1ull << 31)) return fail(ACEGPU_EINVAL, "MSM size must be 1..2^31");
    if (sub > bn::kMsmVbSubMax) return fail(ACEGPU_EINVAL, "MSM sub-range above 80 Mi points");
    if (!points || !out) return fail(ACEGPU_EINVAL, "null argument");
    return msm_prepare_impl(c, group, points, n, on_device, 1, sub, out);
}

extern "C" void acegpu_bn_msm_free(acegpu_msm_bases* b) {
    if (!b) return;
    DeviceGuard g(b->device);
    if (b->table) cudaFree(b->table);
    delete b;
}

extern "C" int acegpu_bn_msm_run_dev(acegpu_ctx* c, void* stream, const acegpu_msm_bases* b,
                                     const uint8_t* d_scalars, uint8_t* d_out) {
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = pick(c, stream);
    if (b->vb ? bn::msm_run_vb(b->group, b->table, b->n, d_scalars, c->msm, d_out, s, b->vb_sub)
              : bn::msm_run(b->group, b->table, b->n, d_scalars, c->msm, d_out, s))
        return fail(ACEGPU_ECUDA, std::string("msm_run: ") + cudaGetErrorString(cudaGetLastError()));
    c->launches += bn::kMsmKernels;
    return ACEGPU_OK;
}

extern "C" int acegpu_bn_msm_run(acegpu_ctx* c, const acegpu_msm_bases* b,
                                 const uint8_t* scalars, uint8_t* out) {
    uint8_t *dsc, *dout;
    const uint64_t pb = 64ull * b->group;
    {
        std::lock_guard<std::mutex> lk(c->mu);
        DeviceGuard g(c->device);
        RET(h2d_t(c, kBnB, scalars, 32 * b->n, c->stream, &dsc));
        RET(ws(c, kBnOut, pb, &dout));
    }
    RET(acegpu_bn_msm_run_dev(c, c->stream, b, dsc, dout));
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    bn::launch_points_convert(b->group, dout, 1, 0, c->stream);
    CKL();
    c->launches++;
    CK(cudaMemcpyAsync(out, dout, pb, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return ACEGPU_OK;
}

namespace {
struct PeakArg {
    uint32_t* sink;
    int blocks, threads, field;
    uint32_t iters;
    cudaStream_t s;
};
void imad_launch(void* p) {
    auto* a = static_cast<PeakArg*>(p);
    bn::launch_imad_peak(a->sink, a->iters, a->blocks, a->threads, a->s);
}
void mulrate_launch(void* p) {
    auto* a = static_cast<PeakArg*>(p);
    bn::launch_mul_rate(a->field, a->sink, a->iters, a->blocks, a->threads, a->s);
}
}  // namespace

extern "C" int acegpu_imad_peak(acegpu_ctx* c, double* imad_per_s) {
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    uint32_t* sink;
    RET(ws(c, kMisc, 16, &sink));
    PeakArg a{sink, sms * 8, 256, 0, 4096, c->stream};
    float ms = 0;
    RET(bn_time(c, c->stream, imad_launch, &a, &ms));
    c->launches += 2;
    *imad_per_s = double(a.blocks) * a.threads * a.iters * 16 * 8 / (ms * 1e-3);
    return ACEGPU_OK;
}

extern "C" int acegpu_bn_mul_rate(acegpu_ctx* c, int field, double* muls_per_s) {
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    uint32_t* sink;
    RET(ws(c, kMisc, 16, &sink));
    PeakArg a{sink, sms * 4, 256, field, 2048, c->stream};
    float ms = 0;
    RET(bn_time(c, c->stream, mulrate_launch, &a, &ms));
    c->launches += 2;
    *muls_per_s = double(a.blocks) * a.threads * a.iters * 4 / (ms * 1e-3);
    return ACEGPU_OK;
}

// ==================================================================== Groth16
// A general constraint system (r1cs.cu): the caller's rows, then one
// z_i * 0 = 0 row per public variable i = 0..n_pub (ONE and the public
// inputs), which makes the public u_i linearly independent (as Groth16 needs).
struct acegpu_r1cs {
    int device = 0;
    uint64_t m_user = 0, rows = 0, vars = 0, n_pub = 0;
    bn::R1csMat mat[3];
    ~acegpu_r1cs() {
        DeviceGuard g(device);
        for (auto& M : mat)
            for (void* p : {(void*)M.rowptr, (void*)M.col, (void*)M.val, (void*)M.colptr,
                            (void*)M.crow, (void*)M.cval, (void*)M.long_rows})
                if (p) cudaFree(p);
    }
};

struct acegpu_g16 {
    int device = 0;
    bn::G16Dims d{};
    uint32_t logn = 0;
    uint64_t N = 0, Vp = 0;  // Vp: private variables
    acegpu_msm_bases *qa = nullptr, *qb1 = nullptr, *qb2 = nullptr, *ql = nullptr, *qh = nullptr;
    // verifying key: IC MSM table; alpha1 (Montgomery affine); beta2 | gamma2 |
    // delta2 in the oracle encoding; IC_0..IC_T Montgomery affine (export)
    acegpu_msm_bases* qic = nullptr;
    uint8_t *vk_alpha1 = nullptr, *vk_g2_std = nullptr, *vk_ic = nullptr;
    uint8_t* vk_digest = nullptr;  // SHA-256 of the acegpu_g16_vk export (verifier seed)
    uint8_t *consts = nullptr, *cc = nullptr;
    // per-proof buffers of the current slot (pointers into slot[cur])
    uint8_t *z = nullptr, *zb = nullptr, *zl = nullptr, *ea = nullptr, *eb = nullptr, *ec = nullptr;
    uint8_t *pts = nullptr, *scaled = nullptr, *rs = nullptr, *digest = nullptr;
    // two buffer slots: chunk k+1's witness chain (stream s_w) runs while
    // chunk k's NTTs / MSMs still read the other slot; `done` = the slot's
    // proof assembled (its buffers free again)
    struct Slot {
        uint8_t *z, *zb, *zl, *ea, *eb, *ec, *pts, *scaled, *rs, *digest, *dsc;
        cudaEvent_t done;
    } slot[2] = {};
    int cur = 1;
    cudaStream_t s_w = nullptr;
    cudaEvent_t ev_in = nullptr;
    cudaStream_t side = nullptr;
    cudaEvent_t ev_ab = nullptr, ev_scaled = nullptr;
    // concurrent MSM streams: B2 + L on s_bl, NTTs + H on s_h, each with its
    // own MSM scratch, so one MSM's latency-bound sort/reduction phases
    // overlap another's throughput-bound bucket accumulation
    cudaStream_t s_bl = nullptr, s_h = nullptr;
    cudaStream_t s_ab = nullptr;  // A, B1, then s*A, r*B1 on `side` overlapping the others
    cudaStream_t s_n = nullptr;   // the H-polynomial NTTs (then ev_n -> the H MSM on s_h)
    cudaEvent_t ev_n = nullptr;
    cudaEvent_t ev_z = nullptr, ev_bl = nullptr, ev_h = nullptr;
    // fixed-base keys: A / B1 / B2 share one digit sort (msm_ab's), B2
    // accumulates on s_bl: ev_sorted = sorted, ev_b2 = B2 done with them
    cudaEvent_t ev_sorted = nullptr, ev_b2 = nullptr;
    bn::MsmScratch msm_bl, msm_h, msm_ab;  // one per MSM stream (no cross-stream scratch)
    const acegpu_r1cs* r1cs = nullptr;  // general circuit (setup_r1cs), else the synthetic chain
    uint8_t* zsc = nullptr;             // general path: r, s digest scratch
    // variable-base key (domain above 2^22, e.g. one proof for a whole block):
    // bases without window tables, one buffer slot (proofs serialise)
    bool vb = false;
    // split key (acegpu_g16_setup_slice): this rank's slice of every base array
    uint32_t rank = 0, world = 1;
    // domain N = 2^logn, or 3 * 2^logn (mixed radix) when three
    bool three = false;
    // split-proof protocol state: 1 = phase 1 done, 2 = partial record ready
    int split_state = 0;
};

namespace {

// The verifying key's export encoding (acegpu_g16_vk) into device memory d
// (448 + 64 (T + 1) bytes): alpha1 | beta2 | gamma2 | delta2 | IC_0..IC_T.
int vk_export_dev(acegpu_ctx* c, const acegpu_g16* g, uint8_t* d, cudaStream_t s) {
    const uint64_t T = g->d.T;
    CK(cudaMemcpyAsync(d, g->vk_alpha1, 64, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(d + 64, g->vk_g2_std, 384, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(d + 448, g->vk_ic, 64 * (T + 1), cudaMemcpyDeviceToDevice, s));
    bn::launch_points_convert(1, d, 1, 0, s);
    bn::launch_points_convert(1, d + 448, T + 1, 0, s);
    CKL();
    c->launches += 2;
    return ACEGPU_OK;
}

int bases_from_device(int device, int group, const uint8_t* d_pts_mont, uint64_t n,
                      cudaStream_t s, acegpu_msm_bases** out) {
    auto* b = new acegpu_msm_bases();
    b->device = device;
    b->group = group;
    b->n = n;
    cudaError_t e = cudaMalloc(&b->table, 64ull * group * n * bn::kMsmWindows);
    if (e != cudaSuccess) {
        delete b;
        return fail(ACEGPU_ECUDA, std::string("g16 table alloc: ") + cudaGetErrorString(e));
    }
    if (bn::msm_prepare(group, d_pts_mont, n, b->table, s)) {
        acegpu_bn_msm_free(b);
        return fail(ACEGPU_ECUDA, "g16 msm_prepare");
    }
    *out = b;
    return ACEGPU_OK;
}

const char* kG2Gen[4] = {
    "10857046999023057135944570762232829481370756359578518086990519993285655852781",
    "11559732032986387107991004021392285783925812861821192530917403151452391805634",
    "8495653923123431417604973247489272438418190587263600148770280649306958101930",
    "4082367875863433681332203403145435568316851327593401208105741076214120093531"};

void dec_to_le32(const char* s, uint8_t* out) {
    uint32_t v[8] = {0};
    for (; *s; ++s) {
        uint64_t c = uint64_t(*s - '0');
        for (int i = 0; i < 8; ++i) {
            uint64_t x = uint64_t(v[i]) * 10 + c;
            v[i] = uint32_t(x);
            c = x >> 32;
        }
    }
    std::memcpy(out, v, 32);
}

}  // namespace

extern "C" void acegpu_g16_free(acegpu_g16* g) {
    if (!g) return;
    DeviceGuard guard(g->device);
    cudaDeviceSynchronize();
    for (acegpu_msm_bases* b : {g->qa, g->qb1, g->qb2, g->ql, g->qh, g->qic})
        acegpu_bn_msm_free(b);
    for (uint8_t* p : {g->consts, g->cc, g->vk_alpha1, g->vk_g2_std, g->vk_ic, g->vk_digest,
                       g->zsc})
        if (p) cudaFree(p);
    for (int k = 0; k < 2; ++k) {
        auto& sl = g->slot[k];
        if (sl.done) cudaEventDestroy(sl.done);
        if (k == 1 && sl.z && sl.z == g->slot[0].z) continue;  // vb: slot 1 aliases slot 0
        for (uint8_t* p : {sl.z, sl.zb, sl.zl, sl.ea, sl.eb, sl.ec, sl.pts, sl.scaled, sl.rs,
                           sl.digest, sl.dsc})
            if (p) cudaFree(p);
    }
    if (g->s_w) cudaStreamDestroy(g->s_w);
    if (g->ev_in) cudaEventDestroy(g->ev_in);
    if (g->side) cudaStreamDestroy(g->side);
    if (g->ev_ab) cudaEventDestroy(g->ev_ab);
    if (g->ev_scaled) cudaEventDestroy(g->ev_scaled);
    for (cudaStream_t t : {g->s_bl, g->s_h, g->s_ab, g->s_n})
        if (t) cudaStreamDestroy(t);
    if (g->ev_n) cudaEventDestroy(g->ev_n);
    for (cudaEvent_t e : {g->ev_z, g->ev_bl, g->ev_h, g->ev_sorted, g->ev_b2})
        if (e) cudaEventDestroy(e);
    g->msm_bl.release();
    g->msm_h.release();
    g->msm_ab.release();
    delete g;
}

extern "C" int acegpu_g16_domain(const acegpu_g16* g, uint64_t* N) {
    if (!g || !N) return fail(ACEGPU_EINVAL, "null argument");
    *N = g->N;
    return ACEGPU_OK;
}

extern "C" int acegpu_g16_shape(const acegpu_g16* g, uint64_t* V, uint64_t* m, uint32_t* logn) {
    if (V) *V = g->d.V;
    if (m) *m = g->d.m;
    if (logn) *logn = g->logn;
    return ACEGPU_OK;
}

namespace {
// Proving + verifying key: the synthetic chain circuit (r == nullptr: T txs
// x K constraints) or a general R1CS r (T = its public inputs, K = 0).
int g16_setup_impl(acegpu_ctx* c, uint32_t T, uint32_t K, const acegpu_r1cs* r,
                   const uint8_t* trapdoor5, acegpu_g16** out, uint32_t rank = 0,
                   uint32_t world = 1, const uint32_t* shares = nullptr) {
    cudaStream_t s = c->stream;
    auto* g = new acegpu_g16();
    std::unique_ptr<acegpu_g16, void (*)(acegpu_g16*)> own(g, acegpu_g16_free);
    g->device = c->device;
    g->r1cs = r;
    g->d.T = T;
    g->d.K = K;
    g->d.V = r ? r->vars : 1 + uint64_t(T) + uint64_t(T) * (K + 1);
    g->d.m = r ? r->rows : uint64_t(T) * K + T + 1;
    // the smallest domain >= m among 2^a and 3 * 2^b (oracle: bn_g16_domain);
    // ACEGPU_G16_RADIX3=0 keeps powers of two
    while ((1ull << g->logn) < g->d.m) ++g->logn;
    {
        const char* e = std::getenv("ACEGPU_G16_RADIX3");
        uint32_t b = 0;
        while ((3ull << b) < g->d.m) ++b;
        if (!(e && e[0] == '0') && (3ull << b) < (1ull << g->logn) &&
            b <= uint32_t(bn::kNtt3MaxLog)) {
            g->three = true;
            g->logn = b;
        }
    }
    if (g->logn > uint32_t(bn::kNttMaxLog)) return fail(ACEGPU_EINVAL, "g16: domain above 2^28");
    g->N = (g->three ? 3ull : 1ull) << g->logn;
    {
        const char* e = std::getenv("ACEGPU_G16_VB");  // 1: force variable-base (tests)
        g->vb = g->N > (1ull << bn::kNttTwoPassMax) || (e && e[0] == '1') || world > 1;
    }
    g->rank = rank;
    g->world = world;
    g->Vp = g->d.V - 1 - T;
    const uint64_t V = g->d.V, N = g->N, m = g->d.m;
    auto dm = [&](uint8_t** p, size_t bytes) { return cudaMalloc(p, bytes ? bytes : 16); };
    if (dm(&g->consts, 32 * 16) || dm(&g->cc, 32ull * K))
        return fail(ACEGPU_ECUDA, "g16 alloc");
    if (r && dm(&g->zsc, bn::g16_long_digest_scratch_bytes(std::max<uint64_t>(g->d.V, T)) + 64))
        return fail(ACEGPU_ECUDA, "g16 alloc");
    for (int k = 0; k < 2; ++k) {
        auto& sl = g->slot[k];
        CK(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
        if (k == 1 && g->vb) {  // one slot: proofs serialise on slot 0
            cudaEvent_t ev = sl.done;
            sl = g->slot[0];
            sl.done = ev;
            break;
        }
        if (dm(&sl.z, 32 * (V + 3)) || dm(&sl.zb, 32 * (V + 2)) || dm(&sl.zl, 32 * (g->Vp + 1)) ||
            dm(&sl.ea, 32 * N) || dm(&sl.eb, 32 * N) || dm(&sl.ec, 32 * N) || dm(&sl.pts, 512) ||
            dm(&sl.scaled, 256) || dm(&sl.rs, 64) || dm(&sl.digest, 32) ||
            dm(&sl.dsc, bn::g16_digest_scratch_bytes(T, 1) + 32))
            return fail(ACEGPU_ECUDA, "g16 alloc");
    }
    CK(cudaStreamCreateWithFlags(&g->s_w, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&g->ev_in, cudaEventDisableTiming));
    CK(cudaStreamCreateWithFlags(&g->side, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&g->ev_ab, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&g->ev_scaled, cudaEventDisableTiming));
    {
        // stream priorities (ACEGPU_G16_PRIO: which of ab / h / bl run at the
        // highest priority; "none" = all equal). Measured (chunk, ms) with
        // the coset-Lagrange H (6 NTTs): ab 49.35, ab+bl 49.56, bl 50.1,
        // none 51.6; with 7 NTTs bl had led (49.75 vs ab 50.3): the stream
        // balance shifts with the H stream's length.
        int least = 0, greatest = 0;
        CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        const char* e = std::getenv("ACEGPU_G16_PRIO");
        const std::string pr = e ? e : "ab";
        auto prio = [&](const char* k) { return pr.find(k) != std::string::npos ? greatest : least; };
        // "n": the H-polynomial NTTs on their own top-priority stream (the H
        // MSM then waits for them on s_h) with the others one level below
        const bool n_top = pr.find('n') != std::string::npos && greatest < least;
        auto lvl = [&](const char* k) { return n_top && prio(k) == greatest ? greatest + 1 : prio(k); };
        CK(cudaStreamCreateWithPriority(&g->s_bl, cudaStreamNonBlocking, lvl("bl")));
        CK(cudaStreamCreateWithPriority(&g->s_h, cudaStreamNonBlocking, lvl("h")));
        CK(cudaStreamCreateWithPriority(&g->s_ab, cudaStreamNonBlocking, lvl("ab")));
        CK(cudaStreamCreateWithPriority(&g->s_n, cudaStreamNonBlocking, n_top ? greatest : lvl("h")));
        CK(cudaEventCreateWithFlags(&g->ev_n, cudaEventDisableTiming));
    }
    for (cudaEvent_t* e : {&g->ev_z, &g->ev_bl, &g->ev_h, &g->ev_sorted, &g->ev_b2})
        CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    // constants
    CK(cudaMemcpyAsync(g->consts, trapdoor5, 160, cudaMemcpyHostToDevice, s));
    bn::g16_setup_consts(g->consts, g->logn, g->three ? 1 : 0, s);
    if (K) bn::g16_chain_consts(K, g->cc, s);
    // query scalars
    uint8_t *L = nullptr, *su = nullptr, *sv = nullptr, *sl = nullptr, *part = nullptr,
            *hs = nullptr, *gens = nullptr, *ext = nullptr, *pts = nullptr, *icsc = nullptr,
            *tab1 = nullptr, *tab2 = nullptr, *ex2 = nullptr, *inf = nullptr;
    // setup temporaries: freed on every exit (after the stream drains)
    struct Temps {
        std::array<uint8_t**, 14> ps;
        cudaStream_t s;
        ~Temps() {
            cudaStreamSynchronize(s);
            for (uint8_t** p : ps)
                if (*p) cudaFree(*p);
        }
    } temps{{&L, &su, &sv, &sl, &part, &hs, &gens, &ext, &pts, &icsc, &tab1, &tab2, &ex2, &inf}, s};
    // pts: the bases before their window tables (fixed base), the u, v, w
    // column sums (general R1CS) and the verifying-key export
    uint64_t pts_bytes = 448 + 64 * (uint64_t(T) + 1);
    if (r) pts_bytes = std::max<uint64_t>(pts_bytes, 96 * V);
    pts_bytes = std::max<uint64_t>(pts_bytes, 32 * bn::kCombEntries);
    if (!g->vb) pts_bytes = std::max<uint64_t>(pts_bytes, 128 * (std::max(V, N) + 2));
    if (dm(&L, 32 * m) || dm(&su, 32 * V) || dm(&sv, 32 * V) || dm(&sl, 32 * g->Vp) ||
        dm(&part, 256 * 64) || dm(&hs, 32 * N) || dm(&gens, 256) || dm(&ext, 512) ||
        dm(&pts, pts_bytes) || dm(&icsc, 32ull * (T + 1)) ||
        dm(&tab1, 64 * bn::kCombEntries) || dm(&tab2, 128 * bn::kCombEntries))
        return fail(ACEGPU_ECUDA, "g16 setup alloc");
    bn::g16_lagrange(g->consts, m, L, s);
    if (r) {
        // u, v, w = A^T L(tau), B^T L(tau), C^T L(tau) (pts as scratch: 3 V x 32 B)
        uint8_t* uvw = pts;
        for (int k = 0; k < 3; ++k) bn::r1cs_colsum(r->mat[k], L, V, uvw + 32 * V * k, s);
        bn::r1cs_query_scalars(g->consts, uvw, uvw + 32 * V, uvw + 64 * V, V, T, su, sv, sl,
                               icsc, s);
    } else {
        bn::g16_query_scalars(g->d, L, g->consts, g->cc, part, su, sv, sl, s);
        bn::g16_ic_scalars(T, g->consts, su, sv, icsc, s);
    }
    bn::g16_h_scalars(g->consts, N, hs, s);  // coset-Lagrange H bases (groth16.cu)
    // generators (Montgomery affine) and the extra bases alpha1 beta1 delta1 | beta2 delta2
    uint8_t hgen[192] = {0};
    hgen[0] = 1;
    hgen[32] = 2;
    for (int i = 0; i < 4; ++i) dec_to_le32(kG2Gen[i], hgen + 64 + 32 * i);
    uint8_t hsc[96];
    std::memcpy(hsc, trapdoor5 + 32, 32);      // alpha
    std::memcpy(hsc + 32, trapdoor5 + 64, 32); // beta
    std::memcpy(hsc + 64, trapdoor5 + 128, 32);// delta
    CK(cudaMemcpyAsync(gens, hgen, 192, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(ext + 256, hsc, 96, cudaMemcpyHostToDevice, s));  // scalars at ext+256
    bn::launch_points_convert(1, gens, 1, 1, s);
    bn::launch_points_convert(2, gens + 64, 1, 1, s);
    uint8_t* ex1 = ext;  // 3 G1 points: alpha1, beta1, delta1 (192 B) -> then G2 below
    bn::launch_scalar_muls(1, gens, ext + 256, 3, ex1, s);
    if (dm(&ex2, 256)) return fail(ACEGPU_ECUDA, "g16 setup alloc");
    bn::launch_scalar_muls(2, gens + 64, ext + 256 + 32, 2, ex2, s);  // beta2, delta2
    CKL();
    // bases = scalars x generator by the fixed-base comb (pts as the comb's
    // scalar scratch first), then the extra points appended
    bn::launch_comb_table(1, gens, pts, tab1, s);
    bn::launch_comb_table(2, gens + 64, pts, tab2, s);
    CKL();
    auto bases = [&](int group, const uint8_t* scal, uint64_t cnt,
                     std::initializer_list<const uint8_t*> extra, acegpu_msm_bases** out) -> int {
        const uint64_t pb = 64ull * group, total = cnt + extra.size();
        // a split key holds the slice [lo, hi) of the array (the extras last):
        // rank r's share of the bases is shares[r] / sum(shares) (equal if null)
        uint64_t pre = rank, sum = world;
        if (shares) {
            pre = sum = 0;
            for (uint32_t j = 0; j < world; ++j) {
                if (j < rank) pre += shares[j];
                sum += shares[j];
            }
        }
        const uint64_t lo = total * pre / sum,
                       hi = total * (pre + (shares ? shares[rank] : 1)) / sum;
        uint8_t* dst = pts;
        std::unique_ptr<acegpu_msm_bases, void (*)(acegpu_msm_bases*)> b(nullptr,
                                                                          acegpu_bn_msm_free);
        if (g->vb) {  // the bases are the MSM table
            b.reset(new acegpu_msm_bases());
            b->device = c->device;
            b->group = group;
            b->n = hi - lo;
            b->lo = lo;
            b->vb = 1;
            const cudaError_t e = cudaMalloc(&b->table, pb * std::max<uint64_t>(hi - lo, 1));
            if (e != cudaSuccess)
                return fail(ACEGPU_ECUDA, std::string("g16 bases alloc: ") + cudaGetErrorString(e));
            dst = b->table;
        }
        if (lo < std::min(hi, cnt))
            bn::launch_comb_muls(group, group == 1 ? tab1 : tab2, scal + 32 * lo,
                                 std::min(hi, cnt) - lo, dst, s);
        uint64_t k = cnt;
        for (const uint8_t* x : extra) {
            if (k >= lo && k < hi)
                CK(cudaMemcpyAsync(dst + pb * (k - lo), x, pb, cudaMemcpyDeviceToDevice, s));
            ++k;
        }
        CKL();
        if (g->vb) {
            *out = b.release();
            return ACEGPU_OK;
        }
        return bases_from_device(c->device, group, pts, total, s, out);
    };
    // A, B1, B2 take the same scalars z | 1 | r | s (one digit sort per proof):
    // A: [u]1 | alpha1 | delta1 | O, B: [v] | beta | O | delta (O = infinity)
    if (dm(&inf, 128)) return fail(ACEGPU_ECUDA, "g16 setup alloc");
    CK(cudaMemsetAsync(inf, 0, 128, s));
    RET(bases(1, su, V, {ex1, ex1 + 128, inf}, &g->qa));
    RET(bases(1, sv, V, {ex1 + 64, inf, ex1 + 128}, &g->qb1));
    RET(bases(2, sv, V, {ex2, inf, ex2 + 128}, &g->qb2));
    RET(bases(1, sl, g->Vp, {ex1 + 128}, &g->ql));         // L: [l]1 (private) | delta1
    // H: [L^g_j(tau) Z(tau)/delta]1, j < N (coset-Lagrange basis, N points)
    RET(bases(1, hs, N, {}, &g->qh));
    // verifying key (the Groth16 verifier, g16_verify.cu)
    if (dm(&g->vk_alpha1, 64) || dm(&g->vk_g2_std, 384) || dm(&g->vk_ic, 64ull * (T + 1)))
        return fail(ACEGPU_ECUDA, "g16 vk alloc");
    bn::launch_comb_muls(1, tab1, icsc, T + 1, g->vk_ic, s);
    RET(bases_from_device(c->device, 1, g->vk_ic, T + 1, s, &g->qic));
    CK(cudaMemcpyAsync(g->vk_alpha1, ex1, 64, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(ext + 256, trapdoor5 + 96, 32, cudaMemcpyHostToDevice, s));  // gamma
    CK(cudaMemcpyAsync(g->vk_g2_std, ex2, 128, cudaMemcpyDeviceToDevice, s));        // beta2
    bn::launch_scalar_muls(2, gens + 64, ext + 256, 1, g->vk_g2_std + 128, s);       // gamma2
    CK(cudaMemcpyAsync(g->vk_g2_std + 256, ex2 + 128, 128, cudaMemcpyDeviceToDevice, s));
    bn::launch_points_convert(2, g->vk_g2_std, 3, 0, s);
    CKL();
    // the verifier's Fiat-Shamir seed commits to the verifying key
    if (dm(&g->vk_digest, 32)) return fail(ACEGPU_ECUDA, "g16 vk alloc");
    RET(vk_export_dev(c, g, pts, s));  // pts: free scratch by now
    bn::g16_vk_digest(pts, uint32_t(448 + 64 * (T + 1)), g->vk_digest, s);
    CKL();
    CK(cudaStreamSynchronize(s));
    if (bn::ntt_tables(c->ntt[g->logn], int(g->logn), s) ||
        (g->three && bn::ntt3_tables(c->ntt3[g->logn], int(g->logn), s)))
        return fail(ACEGPU_ECUDA, "g16 NTT tables");
    CK(cudaStreamSynchronize(s));
    c->launches += 20;
    *out = own.release();
    return ACEGPU_OK;
}
}  // namespace

extern "C" int acegpu_g16_setup(acegpu_ctx* c, uint32_t T, uint32_t K, const uint8_t* trapdoor5,
                                acegpu_g16** out) {
    if (T < 1 || K < 2) return fail(ACEGPU_EINVAL, "g16: need T >= 1 and K >= 2");
    if (!trapdoor5 || !out) return fail(ACEGPU_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard guard(c->device);
    return g16_setup_impl(c, T, K, nullptr, trapdoor5, out);
}

extern "C" int acegpu_g16_setup_r1cs(acegpu_ctx* c, const acegpu_r1cs* r, const uint8_t* trapdoor5,
                                     acegpu_g16** out) {
    if (!r || !trapdoor5 || !out) return fail(ACEGPU_EINVAL, "null argument");
    if (r->device != c->device) return fail(ACEGPU_EINVAL, "r1cs on another device");
    if (r->n_pub < 1 || r->n_pub > 0xFFFFFFFFull) return fail(ACEGPU_EINVAL, "g16: need >= 1 public input");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard guard(c->device);
    return g16_setup_impl(c, uint32_t(r->n_pub), 0, r, trapdoor5, out);
}

extern "C" int acegpu_g16_setup_slice(acegpu_ctx* c, uint32_t T, uint32_t K,
                                      const uint8_t* trapdoor5, uint32_t rank, uint32_t world,
                                      const uint32_t* shares, acegpu_g16** out) {
    if (T < 1 || K < 2) return fail(ACEGPU_EINVAL, "g16: need T >= 1 and K >= 2");
    if (!trapdoor5 || !out) return fail(ACEGPU_EINVAL, "null argument");
    if (world < 1 || rank >= world) return fail(ACEGPU_EINVAL, "g16: need rank < world");
    if (shares) {
        uint64_t sum = 0;
        for (uint32_t j = 0; j < world; ++j) sum += shares[j];
        if (sum == 0 || sum > (1u << 20)) return fail(ACEGPU_EINVAL, "g16: shares sum in 1..2^20");
    }
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard guard(c->device);
    return g16_setup_impl(c, T, K, nullptr, trapdoor5, out, rank, world, shares);
}

// ---- witness programs (GPU witness generation for bit circuits) ---------------
struct acegpu_witprog {
    int device = 0;
    bn::WitProg p;
    uint4* ops = nullptr;
    uint32_t *addtab = nullptr, *emit = nullptr;
    ~acegpu_witprog() {
        DeviceGuard g(device);
        for (void* q : {(void*)ops, (void*)addtab, (void*)emit})
            if (q) cudaFree(q);
    }
};

extern "C" void acegpu_witprog_free(acegpu_witprog* w) { delete w; }

namespace {
// The builder's slot program -> physical slots by liveness: a slot's
// physical slot is released after its last read (operands are read before
// the destination is written, so an op may reuse its operands' slots); a
// slot never read is released right after it is written. Private variables
// are emitted by the op producing their slot. Errors: operands read before
// they are produced, a SUMBIT of an addition other than the latest.
enum : uint32_t { kWpKey = 1, kWpMsg, kWpAnd, kWpXor, kWpChp, kWpCh, kWpMajp, kWpMaj, kWpAdd,
                  kWpSumbit };
int witprog_compile(const uint32_t* ops4, uint64_t n_ops, const uint32_t* addtab,
                    uint64_t n_addtab, uint32_t n_adds, const uint32_t* var_slot, uint32_t n_vars,
                    uint32_t n_slots, std::vector<uint32_t>& ops, std::vector<uint32_t>& tab,
                    std::vector<uint32_t>& emit, uint32_t& n_phys) {
    constexpr uint32_t kNone = 0xFFFFFFFFu;
    auto nread = [](uint32_t code) { return code == kWpAnd || code == kWpXor ? 2 : code >= kWpChp && code <= kWpMaj ? 3 : 0; };
    std::vector<int64_t> last(n_slots, -1);
    std::vector<uint8_t> made(n_slots, 0);
    made[0] = made[1] = 1;
    int64_t latest_add = -1;
    for (uint64_t i = 0; i < n_ops; ++i) {
        const uint32_t* o = ops4 + 4 * i;
        const uint32_t code = o[0] >> 24, dst = o[0] & 0xFFFFFFu;
        if (code < kWpKey || code > kWpSumbit) return fail(ACEGPU_EINVAL, "witprog: bad opcode");
        auto use = [&](uint32_t sl) -> int {
            if (sl >= n_slots || !made[sl]) return fail(ACEGPU_EINVAL, "witprog: operand read before written");
            last[sl] = int64_t(i);
            return ACEGPU_OK;
        };
        for (int k = 0; k < nread(code); ++k) RET(use(o[1 + k]));
        if (code == kWpAdd) {
            if (uint64_t(o[1]) + o[2] > n_addtab) return fail(ACEGPU_EINVAL, "witprog: addtab range");
            for (uint32_t k = 0; k < o[2]; ++k) RET(use(addtab[o[1] + k]));
            if (dst >= n_adds) return fail(ACEGPU_EINVAL, "witprog: destination out of range");
            latest_add = dst;
            continue;
        }
        if (code == kWpSumbit && int64_t(o[1]) != latest_add)
            return fail(ACEGPU_EINVAL, "witprog: SUMBIT of an addition other than the latest");
        // key bits < 256, message bits (obj_hash | domain) < 320, sum bits < 64
        if ((code == kWpKey && o[1] >= 256) || (code == kWpMsg && o[1] >= 320) ||
            (code == kWpSumbit && o[2] >= 64))
            return fail(ACEGPU_EINVAL, "witprog: input bit out of range");
        if (dst < 2 || dst >= n_slots) return fail(ACEGPU_EINVAL, "witprog: destination out of range");
        made[dst] = 1;
    }
    std::vector<uint32_t> var_of(n_slots, kNone);
    for (uint32_t v = 0; v < n_vars; ++v) {
        if (var_slot[v] < 2 || var_slot[v] >= n_slots || var_of[var_slot[v]] != kNone)
            return fail(ACEGPU_EINVAL, "witprog: var slot out of range or shared");
        var_of[var_slot[v]] = v;
    }
    std::vector<uint32_t> phys(n_slots, kNone), freel;
    phys[0] = 0;
    phys[1] = 1;
    n_phys = 2;
    ops.assign(4 * n_ops, 0);
    tab.assign(addtab, addtab + n_addtab);
    emit.assign(n_ops, kNone);
    uint64_t emitted = 0;
    for (uint64_t i = 0; i < n_ops; ++i) {
        const uint32_t* o = ops4 + 4 * i;
        uint32_t* q = &ops[4 * i];
        const uint32_t code = o[0] >> 24, dst = o[0] & 0xFFFFFFu;
        std::copy(o, o + 4, q);
        std::vector<uint32_t> reads;
        for (int k = 0; k < nread(code); ++k) {
            q[1 + k] = phys[o[1 + k]];
            reads.push_back(o[1 + k]);
        }
        if (code == kWpAdd) {
            for (uint32_t k = 0; k < o[2]; ++k) {
                tab[o[1] + k] = phys[addtab[o[1] + k]];
                reads.push_back(addtab[o[1] + k]);
            }
        }
        for (uint32_t sl : reads)  // release operands at their last read (once)
            if (sl >= 2 && last[sl] == int64_t(i) && phys[sl] != kNone) {
                freel.push_back(phys[sl]);
                phys[sl] = kNone;
            }
        if (code == kWpAdd) continue;
        uint32_t p;
        if (!freel.empty()) {
            p = freel.back();
            freel.pop_back();
        } else {
            p = n_phys++;
        }
        q[0] = code << 24 | p;
        emit[i] = var_of[dst];
        if (var_of[dst] != kNone) ++emitted;
        if (last[dst] < 0) freel.push_back(p);  // never read: only its emit
        else phys[dst] = p;
    }
    if (emitted != n_vars) return fail(ACEGPU_EINVAL, "witprog: a private variable is never produced");
    if (n_phys > bn::kWitprogMaxPhys) return fail(ACEGPU_EINVAL, "witprog: too many live slots");
    return ACEGPU_OK;
}
}  // namespace

extern "C" int acegpu_witprog_create(acegpu_ctx* c, const uint32_t* ops4, uint64_t n_ops,
                                     const uint32_t* addtab, uint64_t n_addtab, uint32_t n_adds,
                                     const uint32_t* var_slot, uint32_t n_vars, uint32_t n_slots,
                                     acegpu_witprog** out) {
    if (!ops4 || !var_slot || !out || !n_ops || n_slots < 2) return fail(ACEGPU_EINVAL, "null argument");
    if (n_slots >= (1u << 24)) return fail(ACEGPU_EINVAL, "witprog: too many slots");
    std::vector<uint32_t> ops, tab, emit;
    uint32_t n_phys = 0;
    RET(witprog_compile(ops4, n_ops, addtab, n_addtab, n_adds, var_slot, n_vars, n_slots, ops, tab,
                        emit, n_phys));
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard guard(c->device);
    cudaStream_t s = c->stream;
    std::unique_ptr<acegpu_witprog> w(new acegpu_witprog());
    w->device = c->device;
    if (cudaMalloc(&w->ops, 16 * n_ops) || cudaMalloc(&w->emit, 4 * n_ops) ||
        cudaMalloc(&w->addtab, 4 * (tab.empty() ? 1 : tab.size())))
        return fail(ACEGPU_ECUDA, "witprog alloc");
    CK(cudaMemcpyAsync(w->ops, ops.data(), 16 * n_ops, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(w->emit, emit.data(), 4 * n_ops, cudaMemcpyHostToDevice, s));
    if (!tab.empty())
        CK(cudaMemcpyAsync(w->addtab, tab.data(), 4 * tab.size(), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    w->p = {w->ops, w->emit, n_ops, w->addtab, n_phys, n_vars};
    *out = w.release();
    return ACEGPU_OK;
}

// z (device) for T transactions in chunks of Tc (0: one chunk of T), each
// chunk's assignment (1 + 5 Tc + Tc n_vars) x 32 B, back to back: attest
// keys (32 B each, key_stride apart: 256 for build_witness records) and their
// 104-B attestations, all on the device.
extern "C" int acegpu_witprog_run_dev(acegpu_ctx* c, void* stream, const acegpu_witprog* w,
                                      const uint8_t* d_keys, uint64_t key_stride,
                                      const uint8_t* d_atts, uint32_t T, uint32_t Tc,
                                      uint8_t* d_z) {
    if (!w || !d_keys || !d_atts || !d_z) return fail(ACEGPU_EINVAL, "null argument");
    if (Tc == 0) Tc = T;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard guard(c->device);
    bn::witprog_run(w->p, d_keys, key_stride, d_atts, T, Tc, d_z, pick(c, stream));
    CKL();
    c->launches += 2;
    return ACEGPU_OK;
}

// host-buffer form: keys T x 32 B, atts T x 104 B -> z
extern "C" int acegpu_witprog_run(acegpu_ctx* c, const acegpu_witprog* w, const uint8_t* keys,
                                  const uint8_t* atts, uint32_t T, uint8_t* z) {
    if (!w || !keys || !atts || !z) return fail(ACEGPU_EINVAL, "null argument");
    uint8_t *dk, *da, *dz;
    const uint64_t zb = 32ull * (1 + 5ull * T + (uint64_t)T * w->p.n_vars);
    {
        std::lock_guard<std::mutex> lk(c->mu);
        DeviceGuard guard(c->device);
        RET(h2d_t(c, kBnA, keys, 32ull * T, c->stream, &dk));
        RET(h2d_t(c, kBnB, atts, 104ull * T, c->stream, &da));
        RET(ws(c, kBnOut, zb, &dz));
    }
    RET(acegpu_witprog_run_dev(c, c->stream, w, dk, 32, da, T, T, dz));
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard guard(c->device);
    CK(cudaMemcpyAsync(z, dz, zb, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return ACEGPU_OK;
}

// ---- general R1CS ------------------------------------------------------------
extern "C" void acegpu_r1cs_free(acegpu_r1cs* r) { delete r; }

extern "C" int acegpu_r1cs_create(acegpu_ctx* c, uint64_t m, uint64_t vars, uint64_t n_pub,
                                  const uint64_t* const rowptr[3], const uint32_t* const cols[3],
                                  const uint8_t* const vals[3], acegpu_r1cs** out) {
    if (!out || !rowptr || !cols || !vals) return fail(ACEGPU_EINVAL, "null argument");
    if (m == 0 || vars < 2 || n_pub + 1 >= vars || vars > 0xFFFFFFFFull)
        return fail(ACEGPU_EINVAL, "r1cs: need m >= 1 and 1 + n_pub < vars < 2^32");
    const uint64_t rows = m + n_pub + 1;
    // host-side validation + the public rows + the CSC transposes
    struct Host {
        std::vector<uint64_t> rp, cp;
        std::vector<uint32_t> col, crow, longr;
        std::vector<uint8_t> val, cval;
    } h[3];
    for (int k = 0; k < 3; ++k) {
        if (!rowptr[k] || rowptr[k][0] != 0) return fail(ACEGPU_EINVAL, "r1cs: rowptr[0] != 0");
        for (uint64_t j = 0; j < m; ++j)
            if (rowptr[k][j + 1] < rowptr[k][j]) return fail(ACEGPU_EINVAL, "r1cs: rowptr not monotone");
        const uint64_t nnz_u = rowptr[k][m];
        if (nnz_u && (!cols[k] || !vals[k])) return fail(ACEGPU_EINVAL, "r1cs: null cols / vals");
        for (uint64_t e = 0; e < nnz_u; ++e)
            if (cols[k][e] >= vars) return fail(ACEGPU_EINVAL, "r1cs: column out of range");
        Host& H = h[k];
        const uint64_t nnz = nnz_u + (k == 0 ? n_pub + 1 : 0);  // A gets z_i * 0 = 0 rows
        H.rp.assign(rowptr[k], rowptr[k] + m + 1);
        H.col.assign(cols[k], cols[k] + nnz_u);
        H.val.assign(vals[k], vals[k] + 32 * nnz_u);
        for (uint64_t i = 0; i <= n_pub; ++i) {
            if (k == 0) {
                H.col.push_back(uint32_t(i));
                uint8_t one[32] = {1};
                H.val.insert(H.val.end(), one, one + 32);
            }
            H.rp.push_back(H.col.size());
        }
        for (uint64_t j = 0; j < rows; ++j)
            if (H.rp[j + 1] - H.rp[j] > bn::kR1csLongRow) H.longr.push_back(uint32_t(j));
        // CSC (counting sort by column, stable in row order)
        H.cp.assign(vars + 1, 0);
        for (uint64_t e = 0; e < nnz; ++e) ++H.cp[H.col[e] + 1];
        for (uint64_t i = 0; i < vars; ++i) H.cp[i + 1] += H.cp[i];
        std::vector<uint64_t> cur(H.cp.begin(), H.cp.end() - 1);
        H.crow.resize(nnz);
        H.cval.resize(32 * nnz);
        for (uint64_t j = 0; j < rows; ++j)
            for (uint64_t e = H.rp[j]; e < H.rp[j + 1]; ++e) {
                const uint64_t d = cur[H.col[e]]++;
                H.crow[d] = uint32_t(j);
                std::memcpy(&H.cval[32 * d], &H.val[32 * e], 32);
            }
    }
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard guard(c->device);
    cudaStream_t s = c->stream;
    std::unique_ptr<acegpu_r1cs> r(new acegpu_r1cs());
    r->device = c->device;
    r->m_user = m;
    r->rows = rows;
    r->vars = vars;
    r->n_pub = n_pub;
    auto up = [&](auto** dst, const auto& v) -> int {
        const size_t bytes = v.size() * sizeof(v[0]);
        if (cudaMalloc(reinterpret_cast<void**>(dst), bytes ? bytes : 16) != cudaSuccess)
            return fail(ACEGPU_ECUDA, "r1cs alloc");
        if (bytes) CK(cudaMemcpyAsync(*dst, v.data(), bytes, cudaMemcpyHostToDevice, s));
        return ACEGPU_OK;
    };
    for (int k = 0; k < 3; ++k) {
        bn::R1csMat& M = r->mat[k];
        M.nnz = h[k].col.size();
        RET(up(&M.rowptr, h[k].rp));
        RET(up(&M.col, h[k].col));
        RET(up(&M.val, h[k].val));
        RET(up(&M.colptr, h[k].cp));
        RET(up(&M.crow, h[k].crow));
        RET(up(&M.cval, h[k].cval));
        M.n_long = h[k].longr.size();
        RET(up(&M.long_rows, h[k].longr));
        // values: 32-B LE integers -> Montgomery (to_mont reduces any value < 2^256)
        bn::launch_fr_convert(M.val, M.nnz, 1, s);
        bn::launch_fr_convert(M.cval, M.nnz, 1, s);
        CKL();
    }
    CK(cudaStreamSynchronize(s));
    c->launches += 12;
    *out = r.release();
    return ACEGPU_OK;
}

extern "C" int acegpu_r1cs_shape(const acegpu_r1cs* r, uint64_t* rows, uint64_t* vars,
                                 uint64_t* n_pub) {
    if (!r) return fail(ACEGPU_EINVAL, "null argument");
    if (rows) *rows = r->rows;
    if (vars) *vars = r->vars;
    if (n_pub) *n_pub = r->n_pub;
    return ACEGPU_OK;
}

// a = A z, b = B z, c = C z (rows entries, incl. the public rows), host buffers.
extern "C" int acegpu_r1cs_eval(acegpu_ctx* c, const acegpu_r1cs* r, const uint8_t* z,
                                uint8_t* a, uint8_t* b, uint8_t* cc) {
    if (!r || !z) return fail(ACEGPU_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard guard(c->device);
    cudaStream_t s = c->stream;
    uint8_t *dz, *out;
    RET(h2d_t(c, kBnA, z, 32 * r->vars, s, &dz));
    RET(ws(c, kBnOut, 96 * r->rows, &out));
    bn::launch_fr_convert(dz, r->vars, 1, s);
    for (int k = 0; k < 3; ++k) {
        bn::r1cs_spmv(r->mat[k], dz, r->rows, r->rows, out + 32 * r->rows * k, s);
        bn::launch_fr_convert(out + 32 * r->rows * k, r->rows, 0, s);
    }
    CKL();
    c->launches += 8;
    uint8_t* dst[3] = {a, b, cc};
    for (int k = 0; k < 3; ++k)
        if (dst[k]) CK(cudaMemcpyAsync(dst[k], out + 32 * r->rows * k, 32 * r->rows,
                                       cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ACEGPU_OK;
}

namespace {
int g16_prove_locked(acegpu_ctx* c, cudaStream_t s, acegpu_g16* g, const uint8_t* d_w,
                     const uint8_t* d_pub, const uint8_t* d_rs, uint8_t* d_proof256,
                     uint8_t* d_raw256, uint8_t* d_digest32, cudaEvent_t inputs_ready = nullptr,
                     const uint8_t* d_z = nullptr, uint8_t* d_part384 = nullptr,
                     int owned = -1, uint8_t* d_own = nullptr);
}

// General R1CS: prove from the full assignment z (vars x 32-B standard form,
// z[0] = 1, z[1..n_pub] the public inputs).
extern "C" int acegpu_g16_prove_z_dev(acegpu_ctx* c, void* stream, acegpu_g16* g,
                                      const uint8_t* d_z, const uint8_t* d_rs,
                                      uint8_t* d_proof256, uint8_t* d_raw256,
                                      uint8_t* d_digest32) {
    if (!g || !d_z) return fail(ACEGPU_EINVAL, "null argument");
    if (!g->r1cs) return fail(ACEGPU_EINVAL, "g16: key not built from an R1CS (acegpu_g16_setup_r1cs)");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard guard(c->device);
    return g16_prove_locked(c, pick(c, stream), g, nullptr, nullptr, d_rs, d_proof256, d_raw256,
                            d_digest32, nullptr, d_z);
}

extern "C" int acegpu_g16_prove_z(acegpu_ctx* c, acegpu_g16* g, const uint8_t* z,
                                  const uint8_t* rs, uint8_t* proof256, uint8_t* raw256,
                                  uint8_t* digest32) {
    if (!g || !z) return fail(ACEGPU_EINVAL, "null argument");
    uint8_t *dz, *drs = nullptr, *dout;
    {
        std::lock_guard<std::mutex> lk(c->mu);
        DeviceGuard guard(c->device);
        RET(h2d_t(c, kBnB, z, 32 * g->d.V, c->stream, &dz));
        if (rs) RET(h2d_t(c, kIn2, rs, 64, c->stream, &drs));
        RET(ws(c, kBnOut, 512 + 32, &dout));
    }
    RET(acegpu_g16_prove_z_dev(c, c->stream, g, dz, drs, dout, dout + 256, dout + 512));
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard guard(c->device);
    if (proof256) CK(cudaMemcpyAsync(proof256, dout, 256, cudaMemcpyDeviceToHost, c->stream));
    if (raw256) CK(cudaMemcpyAsync(raw256, dout + 256, 256, cudaMemcpyDeviceToHost, c->stream));
    if (digest32) CK(cudaMemcpyAsync(digest32, dout + 512, 32, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return ACEGPU_OK;
}

extern "C" int acegpu_g16_prove_chunk_dev(acegpu_ctx* c, void* stream, acegpu_g16* g,
                                          const uint8_t* d_w, const uint8_t* d_pub,
                                          const uint8_t* d_rs, uint8_t* d_proof256,
                                          uint8_t* d_raw256, uint8_t* d_digest32) {
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard guard(c->device);
    return g16_prove_locked(c, pick(c, stream), g, d_w, d_pub, d_rs, d_proof256, d_raw256,
                            d_digest32);
}

namespace {
// ACEGPU_G16_TRACE=1: per-stream stage completion times of one chunk proof
// (events, printed to stderr after a synchronize) — a timeline without nsys.
struct G16Trace {
    bool on = std::getenv("ACEGPU_G16_TRACE") != nullptr;
    cudaEvent_t ev[16] = {};
    const char* name[16] = {};
    int n = 0;
    void mark(const char* what, cudaStream_t st) {
        if (!on || n >= 16) return;
        if (!ev[n]) cudaEventCreate(&ev[n]);
        name[n] = what;
        cudaEventRecord(ev[n++], st);
    }
    void dump() {
        if (!on || !n) return;
        cudaEventSynchronize(ev[n - 1]);
        cudaDeviceSynchronize();
        for (int i = 1; i < n; ++i) {
            float ms = 0;
            cudaEventElapsedTime(&ms, ev[0], ev[i]);
            std::fprintf(stderr, "[g16] %-10s %8.3f ms\n", name[i], ms);
        }
        n = 0;
    }
};
G16Trace g_g16_trace;
int g16_prove_locked(acegpu_ctx* c, cudaStream_t s, acegpu_g16* g, const uint8_t* d_w,
                     const uint8_t* d_pub, const uint8_t* d_rs, uint8_t* d_proof256,
                     uint8_t* d_raw256, uint8_t* d_digest32, cudaEvent_t inputs_ready,
                     const uint8_t* d_z, uint8_t* d_part384, int owned, uint8_t* d_own) {
    const bool phase1 = owned >= 0;  // owner split, phase 1 (acegpu_g16_prove_phase1_dev)
    if (g->world > 1 && !d_part384 && !phase1)
        return fail(ACEGPU_EINVAL, "g16: a split key proves partials (acegpu_g16_prove_partial_dev)");
    if (!g->r1cs != !d_z)
        return fail(ACEGPU_EINVAL, g->r1cs ? "g16: an R1CS key proves full assignments "
                                             "(acegpu_g16_prove_z)"
                                           : "g16: full assignments need an R1CS key");
    const uint64_t V = g->d.V, N = g->N, m = g->d.m;
    uint8_t* scratch;
    RET(ws(c, kBnScratch, (g->three ? 64 : 32) * N, &scratch));  // mixed radix: + the 3 sub-vectors
    // next buffer slot; its previous proof must be assembled before reuse
    g->cur = g->vb ? 0 : g->cur ^ 1;
    acegpu_g16::Slot& sl = g->slot[g->cur];
    g->z = sl.z, g->zb = sl.zb, g->zl = sl.zl, g->ea = sl.ea, g->eb = sl.eb, g->ec = sl.ec;
    g->pts = sl.pts, g->scaled = sl.scaled, g->rs = sl.rs, g->digest = sl.digest;
    cudaStream_t sw = g->s_w;
    if (!inputs_ready) {  // inputs produced on s up to now
        CK(cudaEventRecord(g->ev_in, s));
        inputs_ready = g->ev_in;
    }
    CK(cudaStreamWaitEvent(sw, inputs_ready, 0));
    CK(cudaStreamWaitEvent(sw, sl.done, 0));
    G16Trace& tr = g_g16_trace;
    tr.mark("start", sw);
    // phase 1 of the owner split needs only the owned row vectors (the
    // others arrive as slices): skip writing the rest
    const int rows_needed = phase1 ? owned : 7;
    uint8_t* e3w[3] = {(rows_needed & 1) ? g->ea : nullptr, (rows_needed & 2) ? g->eb : nullptr,
                       (rows_needed & 4) ? g->ec : nullptr};
    for (uint8_t* e : e3w)
        if (e && N > m) CK(cudaMemsetAsync(e + 32 * m, 0, 32 * (N - m), sw));
    if (g->r1cs) {
        // general R1CS: the caller's full assignment z (standard form); the
        // row evaluations a, b, c = A z, B z, C z by SpMV (zb holds z in
        // Montgomery form meanwhile), zero-padded to the domain
        const acegpu_r1cs* r = g->r1cs;
        CK(cudaMemcpyAsync(g->zb, d_z, 32 * V, cudaMemcpyDeviceToDevice, sw));
        bn::launch_fr_convert(g->zb, V, 1, sw);
        uint8_t* e3[3] = {g->ea, g->eb, g->ec};
        for (int k = 0; k < 3; ++k) bn::r1cs_spmv(r->mat[k], g->zb, r->rows, N, e3[k], sw);
        // z canonical for the MSM scalars and the digests
        bn::launch_fr_convert(g->zb, V, 0, sw);
        CK(cudaMemcpyAsync(g->z, g->zb, 32 * V, cudaMemcpyDeviceToDevice, sw));
        bn::g16_derive_rs_long(g->z + 32 * (1 + g->d.T), V - 1 - g->d.T, g->z + 32, g->d.T,
                               g->zsc, g->rs, g->digest, sw);
    } else {
        bn::g16_witness(g->d, d_w, d_pub, g->cc, g->z, e3w[0], e3w[1], e3w[2], sw);
        bn::g16_derive_rs(d_w, d_pub, g->d.T, sl.dsc, g->rs, g->digest, sw);
    }
    if (d_rs) CK(cudaMemcpyAsync(g->rs, d_rs, 64, cudaMemcpyDeviceToDevice, sw));
    // scalar vectors with their extras
    {
        // L's scalars: the private part of z (a split key needs its slice only)
        uint64_t lo = 0, cnt = g->Vp;
        if (g->ql->vb && g->world > 1) {
            lo = std::min<uint64_t>(g->ql->lo, g->Vp);
            cnt = std::min<uint64_t>(g->ql->lo + g->ql->n, g->Vp) - lo;
        }
        if (cnt)
            CK(cudaMemcpyAsync(g->zl + 32 * lo, g->z + 32 * (1 + g->d.T + lo), 32 * cnt,
                               cudaMemcpyDeviceToDevice, sw));
    }
    bn::g16_extras(g->z, g->zb, g->zl, V, g->Vp, g->rs, sw);
    CKL();
    CK(cudaEventRecord(g->ev_z, sw));
    tr.mark("witness", sw);
    // s_h: H(g w^j) = (a b - c) / Z on the coset, then [h] over those evaluations
    const bn::NttTables& t = c->ntt[g->logn];
    const bn::Ntt3Tables& t3 = c->ntt3[g->logn];
    if (t.L != int(g->logn) || (g->three && t3.k != int(g->logn)))
        return fail(ACEGPU_EINVAL, "g16: NTT tables missing");
    cudaStream_t sh = g->s_h, sn = g->s_n;
    auto ntt = [&](uint8_t* e, int inverse, int coset) {
        return g->three ? bn::ntt3_run(t3, t, e, e, scratch, scratch + 32 * N, inverse, coset, sn)
                        : bn::ntt_run(t, e, e, scratch, inverse, coset, 1, sn);
    };
    CK(cudaStreamWaitEvent(sn, g->ev_z, 0));
    if (phase1) {
        // phase 1 of the owner split: only the owned vectors' coset
        // evaluations (a = bit 0, b = 1, c = 2), copied out for the exchange;
        // the pointwise step and [h] follow in phase 2 on each rank's slice
        int k = 0, idx = 0;
        for (uint8_t* e : {g->ea, g->eb, g->ec}) {
            if ((owned >> k++) & 1) {
                if (ntt(e, 1, 0) || ntt(e, 0, 1)) return fail(ACEGPU_ECUDA, "g16 ntt");
                CK(cudaMemcpyAsync(d_own + 32 * N * idx++, e, 32 * N, cudaMemcpyDeviceToDevice, sn));
            }
        }
        CKL();
        CK(cudaEventRecord(g->ev_n, sn));
    }
    for (uint8_t* e : {g->ea, g->eb, g->ec}) {
        if (phase1) break;
        if (ntt(e, 1, 0)) return fail(ACEGPU_ECUDA, "g16 intt");
        if (ntt(e, 0, 1)) return fail(ACEGPU_ECUDA, "g16 coset ntt");
    }
    if (!phase1) bn::g16_pointwise(g->ea, g->eb, g->ec, g->consts, N, sn);
    // H(g w^j) are the MSM scalars as they stand (Lagrange-coset H bases): no
    // coset iNTT back to coefficients
    if (!phase1) {
        bn::launch_fr_convert(g->ea, N, 0, sn);  // -> standard form scalars
        CK(cudaEventRecord(g->ev_n, sn));
    }
    tr.mark("ntt", sn);
    CKL();
    CK(cudaStreamWaitEvent(sh, g->ev_n, 0));
    // (n: the full array's length; a split key's bases cover [lo, lo + b->n))
    auto msm = [](const acegpu_msm_bases* b, uint64_t n, const uint8_t* sc, bn::MsmScratch& scr,
                  uint8_t* out, cudaStream_t st) {
        if (b->vb && b->n == 0) return int(cudaMemsetAsync(out, 0, 64 * b->group, st) != cudaSuccess);
        return b->vb ? bn::msm_run_vb(b->group, b->table, b->n, sc + 32 * b->lo, scr, out, st,
                                      b->vb_sub)
                     : bn::msm_run(b->group, b->table, n, sc, scr, out, st);
    };
    if (!phase1 && msm(g->qh, N, g->ea, g->msm_h, g->pts + 320, sh))
        return fail(ACEGPU_ECUDA, "g16 msm H");
    CK(cudaEventRecord(g->ev_h, sh));
    tr.mark("msm_h", sh);
    const int groups[3] = {1, 1, 2};
    const uint8_t* tabs[3] = {g->qa->table, g->qb1->table, g->qb2->table};
    uint8_t* outs[3] = {g->pts, g->pts + 64, g->pts + 128};
    const acegpu_msm_bases* qa = g->qa;
    if (!qa->vb) {
        // fixed base: s_ab sorts z | 1 | r | s once (after the previous
        // proof's B2 has finished reading msm_ab's sorted entries) and
        // accumulates A, B1; s_bl accumulates B2 from the same sort, then L
        bn::MsmSorted info;
        CK(cudaStreamWaitEvent(g->s_ab, g->ev_z, 0));
        CK(cudaStreamWaitEvent(g->s_ab, g->ev_b2, 0));
        if (bn::msm_sort(V + 3, g->z, g->msm_ab, info, g->s_ab))
            return fail(ACEGPU_ECUDA, "g16 msm sort");
        CK(cudaEventRecord(g->ev_sorted, g->s_ab));
        CK(cudaStreamWaitEvent(g->s_bl, g->ev_sorted, 0));
        if (bn::msm_accumulate(2, tabs[2], g->msm_ab, info, g->msm_bl, outs[2], g->s_bl))
            return fail(ACEGPU_ECUDA, "g16 msm B2");
        CK(cudaEventRecord(g->ev_b2, g->s_bl));
        tr.mark("msm_b2", g->s_bl);
        if (msm(g->ql, g->Vp + 1, g->zl, g->msm_bl, g->pts + 256, g->s_bl))
            return fail(ACEGPU_ECUDA, "g16 msm L");
        CK(cudaEventRecord(g->ev_bl, g->s_bl));
        tr.mark("msm_l", g->s_bl);
        for (int i = 0; i < 2; ++i)
            if (bn::msm_accumulate(1, tabs[i], g->msm_ab, info, g->msm_ab, outs[i], g->s_ab))
                return fail(ACEGPU_ECUDA, "g16 msm A/B1");
    } else {
        // variable base (block-size keys): s_bl: [l]; s_ab: A, B1, B2 over
        // the same scalars, each sub-range sorted once
        CK(cudaStreamWaitEvent(g->s_bl, g->ev_z, 0));
        if (msm(g->ql, g->Vp + 1, g->zl, g->msm_bl, g->pts + 256, g->s_bl))
            return fail(ACEGPU_ECUDA, "g16 msm L");
        CK(cudaEventRecord(g->ev_bl, g->s_bl));
        tr.mark("msm_l", g->s_bl);
        CK(cudaStreamWaitEvent(g->s_ab, g->ev_z, 0));
        int rc = 0;
        if (qa->n == 0)
            rc = cudaMemsetAsync(g->pts, 0, 256, g->s_ab) != cudaSuccess;
        else
            rc = bn::msm_run_vb_multi(3, groups, tabs, qa->n, g->z + 32 * qa->lo, g->msm_ab, outs,
                                      g->s_ab, qa->vb_sub);
        if (rc) return fail(ACEGPU_ECUDA, "g16 msm A/B1/B2");
    }
    CK(cudaEventRecord(g->ev_ab, g->s_ab));
    tr.mark("msm_b1", g->s_ab);
    if (phase1) {  // phase 1 done: the owned evaluations are ready on s
        g->split_state = 1;
        CK(cudaStreamWaitEvent(s, g->ev_n, 0));
        c->launches += 12 + 4 * bn::kMsmKernels;
        return ACEGPU_OK;
    }
    if (d_part384) {
        // this rank's partial points A | B1 | B2 | L | H; the sum over ranks,
        // s A, r B1 and the assembly follow in acegpu_g16_finish_dev
        for (cudaEvent_t e : {g->ev_ab, g->ev_bl, g->ev_h}) CK(cudaStreamWaitEvent(s, e, 0));
        CK(cudaMemcpyAsync(d_part384, g->pts, 384, cudaMemcpyDeviceToDevice, s));
        CK(cudaEventRecord(sl.done, s));
        g->split_state = 2;
        tr.dump();
        c->launches += 15 + 5 * bn::kMsmKernels;
        return ACEGPU_OK;
    }
    CK(cudaStreamWaitEvent(g->side, g->ev_ab, 0));
    bn::g16_scale(g->pts, g->rs, g->scaled, g->side);
    CK(cudaEventRecord(g->ev_scaled, g->side));
    tr.mark("scale", g->side);
    for (cudaEvent_t e : {g->ev_scaled, g->ev_bl, g->ev_h}) CK(cudaStreamWaitEvent(s, e, 0));
    // outputs on s (the caller's order): the slot's digest was written on s_w
    // before ev_z, which every wait above follows
    if (d_digest32) CK(cudaMemcpyAsync(d_digest32, g->digest, 32, cudaMemcpyDeviceToDevice, s));
    bn::g16_assemble(g->pts, g->scaled, d_proof256, d_raw256, s);
    CKL();
    CK(cudaEventRecord(sl.done, s));
    tr.mark("assemble", s);
    tr.dump();
    c->launches += 15 + 5 * bn::kMsmKernels + 6;
    return ACEGPU_OK;
}
}  // namespace

// Groth16-mode shard: attestation verdicts + per-tx public-input digests
// (the leaf kernel), the id_com Merkle tree up to the chunk level (lifted
// like the mock shard), and one Groth16 proof per chunk of T txs (the last
// chunk of the block zero-padded). Chunk roots = chunk proofs as mock-tree
// leaves (proof | chunk digest | kind Tx), so acegpu_combine_roots_dev
// aggregates them with the reference's tree rule (prover.cpp:106-127).
namespace {
int g16_verify_locked(acegpu_ctx* c, cudaStream_t s, acegpu_g16* g, const uint8_t* d_proofs,
                      const uint8_t* d_pubs, uint64_t n, int* d_ok, uint8_t* d_seed = nullptr);
// Per-chunk inputs of a (shard of a) block in Groth16 mode: leaves (verdicts,
// public-input digests, Merkle leaves), Merkle levels up to the chunk level
// (the block's short last chunk lifted), the chunk Merkle roots, and the
// zero-padded public inputs pub (chunks x T x 32 B raw digests).
int g16_chunk_inputs(acegpu_ctx* c, cudaStream_t s, acegpu_g16* g, const uint8_t* d_payloads,
                     const uint64_t* d_offs, const uint8_t* d_atts, uint64_t n, uint64_t n_total,
                     const uint8_t* d_revs, const uint32_t* d_rev_index, uint8_t* d_codes,
                     uint8_t* d_merkle32, uint8_t** pub_out, TreeResult* t) {
    const uint32_t T = g->d.T;
    // chunk roots must be Merkle-tree nodes: T a power of two, unless one
    // chunk holds the whole block (a block-size key: one proof per block)
    if ((T & (T - 1)) && n_total > T)
        return fail(ACEGPU_EINVAL, "g16: txs per chunk must be a power of two (or >= the block)");
    if (n == 0) return fail(ACEGPU_EINVAL, "g16: empty block or shard");
    RET(check_n(n));
    uint32_t log2_chunk = 0;
    while ((1u << log2_chunk) < T) ++log2_chunk;
    RET(run_tree(c, s, d_payloads, d_offs, d_atts, uint32_t(n), nullptr, d_revs, d_rev_index,
                 d_codes, true, 0, false, t));
    const bool lift = n_total > T;
    uint8_t* min_ = t->merkle;  // kMerkA after zero levels
    uint8_t* mout = static_cast<uint8_t*>(c->bufs[kMerkB].p);
    uint32_t cur = uint32_t(n), lv = 0;
    while (lv < log2_chunk && (cur > 1 || (lift && cur == 1))) {
        launch_level(nullptr, 0, nullptr, min_, cur, mout, lift, s);
        CKL();
        c->launches++;
        cur = (cur + 1) / 2;
        std::swap(min_, mout);
        ++lv;
    }
    const uint64_t chunks = (n + T - 1) / T;
    if (cur != chunks) return fail(ACEGPU_EINVAL, "g16: chunk count mismatch");
    CK(cudaMemcpyAsync(d_merkle32, min_, 32 * chunks, cudaMemcpyDeviceToDevice, s));
    uint8_t* pub;
    RET(ws(c, kBnA, 32 * chunks * T, &pub));
    bn::g16_gather32(t->nodes + 256, kNodeBytes, n, chunks * T, pub, s);
    CKL();
    *pub_out = pub;
    return ACEGPU_OK;
}
}  // namespace

namespace {
int g16_shard_roots_locked(acegpu_ctx* c, cudaStream_t s, acegpu_g16* g,
                           const uint8_t* d_payloads, const uint64_t* d_offs,
                           const uint8_t* d_atts, uint64_t n, uint64_t n_total,
                           const uint8_t* d_revs, uint64_t n_revs, const uint32_t* d_rev_index,
                           uint8_t* d_codes, const uint8_t* d_witness256, uint8_t* d_roots289,
                           uint8_t* d_merkle32) {
    KeytabScope kts(c);  // attest keys for the credential verdicts (as the mock shard)
    if (d_codes && n) RET(kts.build(s, d_revs, n_revs, d_atts + 64));
    const uint32_t T = g->d.T;
    TreeResult t;
    uint8_t *pub, *w, *proof, *node;
    RET(g16_chunk_inputs(c, s, g, d_payloads, d_offs, d_atts, n, n_total, d_revs, d_rev_index,
                         d_codes, d_merkle32, &pub, &t));
    const uint64_t chunks = (n + T - 1) / T;
    // w = LE(witness[0:32]), zero padded
    RET(ws(c, kBnB, 32 * chunks * T, &w));
    RET(ws(c, kIn2, 256 + 32 + 320, &proof));
    node = proof + 288;
    bn::g16_gather32(d_witness256, 256, n, chunks * T, w, s);
    CKL();
    // every chunk's inputs are ready now: chunk k+1's witness chain may start
    // while chunk k's MSMs run (two buffer slots)
    cudaEvent_t ready = g->ev_in;
    CK(cudaEventRecord(ready, s));
    for (uint64_t k = 0; k < chunks; ++k) {
        RET(g16_prove_locked(c, s, g, w + 32 * T * k, pub + 32 * T * k, nullptr, proof, nullptr,
                             proof + 256, ready));
        bn::g16_chunk_node(proof, proof + 256, node, s);
        launch_pack_nodes(node, 1, d_roots289 + 289 * k, s);
        CKL();
        c->launches += 2;
    }
    return ACEGPU_OK;
}
}  // namespace

extern "C" int acegpu_g16_shard_roots_dev(acegpu_ctx* c, void* stream, acegpu_g16* g,
                                          const uint8_t* d_payloads, const uint64_t* d_offs,
                                          const uint8_t* d_atts, uint64_t n, uint64_t n_total,
                                          const uint8_t* d_revs, uint64_t n_revs,
                                          const uint32_t* d_rev_index, uint8_t* d_codes,
                                          const uint8_t* d_witness256, uint8_t* d_roots289,
                                          uint8_t* d_merkle32) {
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard guard(c->device);
    return g16_shard_roots_locked(c, pick(c, stream), g, d_payloads, d_offs, d_atts, n, n_total,
                                  d_revs, n_revs, d_rev_index, d_codes, d_witness256, d_roots289,
                                  d_merkle32);
}

// ---- one proof per block across ranks (split keys) ----------------------------
// The block's inputs for a block-size key (n <= T): verdicts, the id_com
// Merkle root, the zero-padded witnesses w and public inputs pub (T x 32 B).
extern "C" int acegpu_g16_block_inputs_dev(acegpu_ctx* c, void* stream, acegpu_g16* g,
                                           const uint8_t* d_payloads, const uint64_t* d_offs,
                                           const uint8_t* d_atts, uint64_t n,
                                           const uint8_t* d_revs, uint64_t n_revs,
                                           const uint32_t* d_rev_index, uint8_t* d_codes,
                                           const uint8_t* d_witness256, uint8_t* d_w,
                                           uint8_t* d_pub, uint8_t* d_merkle32) {
    if (!g || !d_witness256 || !d_w || !d_pub || !d_merkle32) return fail(ACEGPU_EINVAL, "null argument");
    if (n == 0 || n > g->d.T) return fail(ACEGPU_EINVAL, "g16 block inputs: need 1 <= n <= T");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard guard(c->device);
    cudaStream_t s = pick(c, stream);
    KeytabScope kts(c);
    if (d_codes) RET(kts.build(s, d_revs, n_revs, d_atts + 64));
    TreeResult t;
    uint8_t* pub;
    RET(g16_chunk_inputs(c, s, g, d_payloads, d_offs, d_atts, n, n, d_revs, d_rev_index, d_codes,
                         d_merkle32, &pub, &t));
    CK(cudaMemcpyAsync(d_pub, pub, 32ull * g->d.T, cudaMemcpyDeviceToDevice, s));
    bn::g16_gather32(d_witness256, 256, n, g->d.T, d_w, s);
    CKL();
    c->launches++;
    return ACEGPU_OK;
}

// This rank's partial proof points (A | B1 | B2 | L | H, 384 B, affine
// Montgomery) over its slice of the bases; every rank computes the same
// witness, r, s and H polynomial.
extern "C" int acegpu_g16_prove_partial_dev(acegpu_ctx* c, void* stream, acegpu_g16* g,
                                            const uint8_t* d_w, const uint8_t* d_pub,
                                            uint8_t* d_part384) {
    if (!g || !d_w || !d_pub || !d_part384) return fail(ACEGPU_EINVAL, "null argument");
    if (g->r1cs) return fail(ACEGPU_EINVAL, "g16 partial: synthetic-circuit keys only");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard guard(c->device);
    return g16_prove_locked(c, pick(c, stream), g, d_w, d_pub, nullptr, nullptr, nullptr, nullptr,
                            nullptr, nullptr, d_part384);
}

// Owner split of the H polynomial (one proof per block across >= 2 ranks):
// phase 1 = the witness, r, s, the A / B1 / B2 / L MSMs of this rank's slices
// (left running) and the coset evaluations of the OWNED vectors (mask: a = 1,
// b = 2, c = 4; vector k owned by rank k mod world) into d_own (one N x 32-B
// Montgomery vector each, in a, b, c order); after the caller's exchange,
// phase 2 takes this rank's slice [N rank / world, N (rank + 1) / world) of
// a, b, c — the same share-weighted bounds as the key's H slice — (d_slices:
// a | b | c, S x 32 B each, overwritten), the pointwise
// (a b - c) / Z, [h] over the slice, and writes the partial record.
extern "C" int acegpu_g16_prove_phase1_dev(acegpu_ctx* c, void* stream, acegpu_g16* g,
                                           const uint8_t* d_w, const uint8_t* d_pub, int owned,
                                           uint8_t* d_own) {
    if (!g || !d_w || !d_pub || (owned && !d_own)) return fail(ACEGPU_EINVAL, "null argument");
    if (g->r1cs) return fail(ACEGPU_EINVAL, "g16 partial: synthetic-circuit keys only");
    if (owned < 0 || owned > 7) return fail(ACEGPU_EINVAL, "g16 phase 1: owned mask in 0..7");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard guard(c->device);
    return g16_prove_locked(c, pick(c, stream), g, d_w, d_pub, nullptr, nullptr, nullptr, nullptr,
                            nullptr, nullptr, nullptr, owned, d_own);
}

extern "C" int acegpu_g16_prove_phase2_dev(acegpu_ctx* c, void* stream, acegpu_g16* g,
                                           uint8_t* d_slices, uint8_t* d_part384) {
    if (!g || !d_slices || !d_part384) return fail(ACEGPU_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard guard(c->device);
    cudaStream_t s = pick(c, stream);
    acegpu_g16::Slot& sl = g->slot[g->cur];
    const acegpu_msm_bases* qh = g->qh;
    if (!qh->vb) return fail(ACEGPU_EINVAL, "g16 phase 2: variable-base keys only");
    if (g->split_state != 1) return fail(ACEGPU_EINVAL, "g16 phase 2 before phase 1");
    const uint64_t S = qh->n;
    cudaStream_t sh = g->s_h;
    CK(cudaEventRecord(g->ev_in, s));  // the exchanged slices are ready on s
    CK(cudaStreamWaitEvent(sh, g->ev_in, 0));
    if (S) {
        bn::g16_pointwise(d_slices, d_slices + 32 * S, d_slices + 64 * S, g->consts, S, sh);
        bn::launch_fr_convert(d_slices, S, 0, sh);
        if (bn::msm_run_vb(1, qh->table, S, d_slices, g->msm_h, sl.pts + 320, sh, qh->vb_sub))
            return fail(ACEGPU_ECUDA, "g16 msm H");
    } else {
        CK(cudaMemsetAsync(sl.pts + 320, 0, 64, sh));
    }
    CKL();
    CK(cudaEventRecord(g->ev_h, sh));
    for (cudaEvent_t e : {g->ev_ab, g->ev_bl, g->ev_h}) CK(cudaStreamWaitEvent(s, e, 0));
    CK(cudaMemcpyAsync(d_part384, sl.pts, 384, cudaMemcpyDeviceToDevice, s));
    CK(cudaEventRecord(sl.done, s));
    g->split_state = 2;
    c->launches += 2 + bn::kMsmKernels;
    return ACEGPU_OK;
}

// Sum the `world` partial records (in rank order), then s A, r B1, C and the
// proof (EIP-197 256 B), raw points, chunk digest and/or the chunk root
// (289-B tree leaf: proof | digest | kind Tx) — for the proof whose partial
// this key computed last.
extern "C" int acegpu_g16_finish_dev(acegpu_ctx* c, void* stream, acegpu_g16* g,
                                     const uint8_t* d_parts, uint32_t world, uint8_t* d_proof256,
                                     uint8_t* d_raw256, uint8_t* d_digest32, uint8_t* d_root289) {
    if (!g || !d_parts || world == 0) return fail(ACEGPU_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard guard(c->device);
    cudaStream_t s = pick(c, stream);
    if (g->split_state != 2) return fail(ACEGPU_EINVAL, "g16 finish before this key's partial");
    g->split_state = 0;
    acegpu_g16::Slot& sl = g->slot[g->cur];
    CK(cudaStreamWaitEvent(s, sl.done, 0));
    uint8_t* proof;
    RET(ws(c, kIn2, 256 + 32 + 320, &proof));
    bn::g16_sum_parts(d_parts, world, sl.pts, s);
    bn::g16_scale(sl.pts, sl.rs, sl.scaled, s);
    bn::g16_assemble(sl.pts, sl.scaled, proof, d_raw256, s);
    CKL();
    if (d_proof256) CK(cudaMemcpyAsync(d_proof256, proof, 256, cudaMemcpyDeviceToDevice, s));
    if (d_digest32) CK(cudaMemcpyAsync(d_digest32, sl.digest, 32, cudaMemcpyDeviceToDevice, s));
    if (d_root289) {
        uint8_t* node = proof + 288;
        bn::g16_chunk_node(proof, sl.digest, node, s);
        launch_pack_nodes(node, 1, d_root289, s);
        CKL();
    }
    CK(cudaEventRecord(sl.done, s));
    c->launches += 5;
    return ACEGPU_OK;
}

extern "C" int acegpu_g16_prove_block(acegpu_ctx* c, acegpu_g16* g, const uint8_t* payloads,
                                      const uint64_t* offs, const uint8_t* atts, uint64_t n,
                                      const uint8_t* header256, const uint8_t* revs,
                                      uint64_t n_revs, const uint32_t* rev_index,
                                      const uint8_t* witness256, uint8_t* codes,
                                      uint8_t* proof289, uint8_t* fc328,
                                      uint8_t* chunk_proofs256) {
    if (!g || !header256 || !witness256) return fail(ACEGPU_EINVAL, "null argument");
    if (n == 0) return fail(ACEGPU_EINVAL, "g16 prove_block: empty block");
    if (n_revs && (!revs || !rev_index)) return fail(ACEGPU_EINVAL, "revs without rev_index");
    RET(check_n(n));
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard guard(c->device);
    cudaStream_t s = c->stream;
    const uint64_t T = g->d.T, chunks = (n + T - 1) / T;
    uint8_t *dp, *da, *dh, *dw, *dcodes = nullptr, *drevs = nullptr, *roots;
    uint64_t* doff;
    uint32_t* drix = nullptr;
    RET(upload_block(c, s, {payloads, offs, atts, n}, &dp, &doff, &da));
    RET(h2d_t(c, kHeader, header256, 256, s, &dh));
    RET(h2d_t(c, kG16Wit, witness256, 256 * n, s, &dw));
    if (n_revs) {
        RET(h2d_t(c, kRevs, revs, 32 * n_revs, s, &drevs));
        RET(h2d_t(c, kRevIdx, rev_index, 4 * n, s, &drix));
        RET(ws(c, kCodes, n, &dcodes));
    }
    auto al = [](uint64_t b) { return (b + 255) & ~uint64_t(255); };
    RET(ws(c, kG16Roots, al(289 * chunks) + al(32 * chunks) + 640, &roots));
    uint8_t* merk = roots + al(289 * chunks);
    uint8_t* out = merk + al(32 * chunks);
    RET(g16_shard_roots_locked(c, s, g, dp, doff, da, n, n, drevs, n_revs, drix, dcodes, dw,
                               roots, merk));
    RET(combine_impl(c, s, roots, merk, chunks, n, dh, out, out + 304));
    if (codes && dcodes) CK(cudaMemcpyAsync(codes, dcodes, n, cudaMemcpyDeviceToHost, s));
    if (proof289) CK(cudaMemcpyAsync(proof289, out, 289, cudaMemcpyDeviceToHost, s));
    if (fc328) CK(cudaMemcpyAsync(fc328, out + 304, 328, cudaMemcpyDeviceToHost, s));
    if (chunk_proofs256)
        CK(cudaMemcpy2DAsync(chunk_proofs256, 256, roots, 289, 256, chunks, cudaMemcpyDeviceToHost,
                             s));
    CK(cudaStreamSynchronize(s));
    return ACEGPU_OK;
}

extern "C" int acegpu_g16_verify_fc(acegpu_ctx* c, acegpu_g16* g, const uint8_t* fc328,
                                    const uint8_t* payloads, const uint64_t* offs,
                                    const uint8_t* atts, uint64_t n, const uint8_t* header,
                                    const uint8_t* chunk_proofs256, uint64_t* cost_units,
                                    int* result) {
    if (!g || !fc328 || !header || !result || (n && (!payloads || !offs || !atts)))
        return fail(ACEGPU_EINVAL, "null argument");
    if (cost_units) *cost_units += 1;  // K_FC_VERIFY_COST_UNITS (prover.hpp:77)
    // slot first (prover.cpp:160-162): FC bytes 32..40 vs header bytes 0..8
    if (std::memcmp(fc328 + 32, header, 8) != 0) {
        *result = 1;
        return ACEGPU_OK;
    }
    if (n == 0) return fail(ACEGPU_EINVAL, "g16 verify_fc: empty block");
    if (!chunk_proofs256) return fail(ACEGPU_EINVAL, "g16 verify_fc: chunk proofs required");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard guard(c->device);
    cudaStream_t s = c->stream;
    const uint32_t T = g->d.T;
    const uint64_t chunks = (n + T - 1) / T;
    uint8_t *dp, *da, *dh, *dproofs, *roots, *merk, *pub, *digest, *node, *out, *dok;
    uint64_t* doff;
    RET(upload_block(c, s, {payloads, offs, atts, n}, &dp, &doff, &da));
    RET(h2d_t(c, kHeader, header, 256, s, &dh));
    RET(h2d_t(c, kSegRoots, chunk_proofs256, 256 * chunks, s, &dproofs));
    auto al = [](uint64_t b) { return (b + 255) & ~uint64_t(255); };  // 16-B vector stores
    const uint64_t dsc_bytes = bn::g16_digest_scratch_bytes(T, uint32_t(chunks));
    RET(ws(c, kSegMerk, al(32 * chunks) + al(289 * chunks) + al(32 * chunks) + al(320) + al(640) +
                            al(16) + dsc_bytes, &merk));
    roots = merk + al(32 * chunks);
    digest = roots + al(289 * chunks);
    node = digest + al(32 * chunks);
    out = node + al(320);
    dok = out + al(640);
    uint8_t* dsc = dok + al(16);
    TreeResult t;
    RET(g16_chunk_inputs(c, s, g, dp, doff, da, n, n, nullptr, nullptr, nullptr, merk, &pub, &t));
    // chunk roots: proof | chunk digest | kind Tx, as the prover built them
    bn::g16_chunk_digests(pub, T, uint32_t(chunks), dsc, digest, s);
    for (uint64_t k = 0; k < chunks; ++k) {
        bn::g16_chunk_node(dproofs + 256 * k, digest + 32 * k, node, s);
        launch_pack_nodes(node, 1, roots + 289 * k, s);
        CKL();
        c->launches += 3;
    }
    RET(combine_impl(c, s, roots, merk, chunks, n, dh, out, out + 304));
    RET(g16_verify_locked(c, s, g, dproofs, pub, chunks, reinterpret_cast<int*>(dok)));
    uint8_t fc[328];
    int ok = 0;
    CK(cudaMemcpyAsync(fc, out + 304, 328, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&ok, dok, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (std::memcmp(fc, fc328, 32) != 0) *result = 2;                       // HashMismatch
    else if (!ok || std::memcmp(fc + 40, fc328 + 40, 288) != 0) *result = 3;  // ProofMismatch
    else *result = 0;                                                        // Valid
    return ACEGPU_OK;
}

extern "C" int acegpu_g16_vk(acegpu_ctx* c, const acegpu_g16* g, uint8_t* out) {
    if (!g || !out) return fail(ACEGPU_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard guard(c->device);
    cudaStream_t s = c->stream;
    const uint64_t bytes = 448 + 64 * (uint64_t(g->d.T) + 1);
    uint8_t* d;
    RET(ws(c, kBnOut, bytes, &d));
    RET(vk_export_dev(c, g, d, s));
    CK(cudaMemcpyAsync(out, d, bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ACEGPU_OK;
}

namespace {
int g16_verify_locked(acegpu_ctx* c, cudaStream_t s, acegpu_g16* g, const uint8_t* d_proofs,
                      const uint8_t* d_pubs, uint64_t n, int* d_ok, uint8_t* d_seed) {
    if (n == 0 || n > (1u << 20)) return fail(ACEGPU_EINVAL, "g16 verify: bad proof count");
    uint8_t* scratch;
    RET(ws(c, kP1Scratch, bn::g16_verify_scratch_bytes(uint32_t(n), g->d.T), &scratch));
    bn::G16VerifyKey vk;
    vk.T = g->d.T;
    vk.ic_table = g->qic->table;
    vk.alpha1_mont = g->vk_alpha1;
    vk.g2_std = g->vk_g2_std;
    vk.vk_digest = g->vk_digest;
    if (bn::g16_verify_batch(vk, d_proofs, d_pubs, uint32_t(n), scratch, c->msm, d_ok, s, d_seed))
        return fail(ACEGPU_ECUDA, "g16 verify launch");
    CKL();
    c->launches += 3 + bn::kMsmKernels;
    return ACEGPU_OK;
}
}  // namespace

extern "C" int acegpu_g16_verify_batch_seed(acegpu_ctx* c, acegpu_g16* g,
                                            const uint8_t* proofs256, const uint8_t* pubs,
                                            uint64_t n, int* ok, uint8_t* seed32) {
    if (!g || !proofs256 || !pubs || !ok) return fail(ACEGPU_EINVAL, "null argument");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard guard(c->device);
    cudaStream_t s = c->stream;
    uint8_t *dp, *dq, *dok;
    RET(h2d_t(c, kBnA, proofs256, 256 * n, s, &dp));
    RET(h2d_t(c, kBnB, pubs, 32ull * g->d.T * n, s, &dq));
    RET(ws(c, kBnOut, 64, &dok));
    RET(g16_verify_locked(c, s, g, dp, dq, n, reinterpret_cast<int*>(dok), dok + 32));
    CK(cudaMemcpyAsync(ok, dok, sizeof(int), cudaMemcpyDeviceToHost, s));
    if (seed32) CK(cudaMemcpyAsync(seed32, dok + 32, 32, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ACEGPU_OK;
}

extern "C" int acegpu_g16_verify_batch(acegpu_ctx* c, acegpu_g16* g, const uint8_t* proofs256,
                                       const uint8_t* pubs, uint64_t n, int* ok) {
    return acegpu_g16_verify_batch_seed(c, g, proofs256, pubs, n, ok, nullptr);
}

extern "C" int acegpu_g16_prove_chunk(acegpu_ctx* c, acegpu_g16* g, const uint8_t* w,
                                      const uint8_t* pub, const uint8_t* rs, uint8_t* proof256,
                                      uint8_t* raw256, uint8_t* digest32) {
    uint8_t *dw, *dp, *drs = nullptr, *dout;
    const uint64_t T = g->d.T;
    {
        std::lock_guard<std::mutex> lk(c->mu);
        DeviceGuard guard(c->device);
        RET(h2d_t(c, kBnA, w, 32 * T, c->stream, &dw));
        RET(h2d_t(c, kBnB, pub, 32 * T, c->stream, &dp));
        if (rs) RET(h2d_t(c, kIn2, rs, 64, c->stream, &drs));
        RET(ws(c, kBnOut, 512 + 32, &dout));
    }
    RET(acegpu_g16_prove_chunk_dev(c, c->stream, g, dw, dp, drs, dout, dout + 256, dout + 512));
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard guard(c->device);
    if (proof256) CK(cudaMemcpyAsync(proof256, dout, 256, cudaMemcpyDeviceToHost, c->stream));
    if (raw256) CK(cudaMemcpyAsync(raw256, dout + 256, 256, cudaMemcpyDeviceToHost, c->stream));
    if (digest32) CK(cudaMemcpyAsync(digest32, dout + 512, 32, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return ACEGPU_OK;
}
