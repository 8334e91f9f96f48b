"""BN254 field / NTT / curve / MSM kernels vs the from-scratch CPU oracle
(oracle/bn254_oracle.c — parity unpinned by the reference, which has no BN254
code; the oracle itself is pinned by tests/test_bn254_oracle.py)."""
import ctypes as C
import random

import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu

P = 0x30644E72E131A029B85045B68181585D97816A916871CA8D3C208C16D87CFD47
R = 0x30644E72E131A029B85045B68181585D2833E84879B9709143E1F593F0000001


@pytest.fixture(scope="module")
def ctx():
    from paper_2603_10242_b200 import _native as N
    return N.context(0)


def le(x):
    return x.to_bytes(32, "little")


def arr(vals):
    return np.frombuffer(b"".join(le(v) for v in vals), np.uint8).copy()


def ints(a):
    b = a.tobytes()
    return [int.from_bytes(b[32 * i:32 * i + 32], "little") for i in range(len(b) // 32)]


def edge(m):
    return [0, 1, 2, m - 1, m - 2, (m - 1) // 2, (m + 1) // 2, 1 << 253, (1 << 254) % m,
            0xFFFFFFFF, 1 << 32, (1 << 128) - 1]


@pytest.mark.parametrize("field,m", [(0, P), (1, R)])
def test_field_ops_match_python_and_oracle(ctx, field, m):
    rng = random.Random(field + 10)
    a = edge(m) + [rng.randrange(m) for _ in range(4000)]
    b = list(reversed(edge(m))) + [rng.randrange(m) for _ in range(4000)]
    A, B = arr(a), arr(b)
    n = len(a)
    for op, f in [(0, lambda x, y: x * y % m), (1, lambda x, y: (x + y) % m),
                  (2, lambda x, y: (x - y) % m), (3, lambda x, y: x * x % m),
                  (4, lambda x, y: pow(x, m - 2, m))]:
        out = np.zeros(32 * n, np.uint8)
        ctx.call("acegpu_bn_field_batch", field, op, A, B, n, out)
        got = ints(out)
        assert got == [f(x, y) for x, y in zip(a, b)], f"op {op}"
    # oracle agreement (the oracle is the checker of record)
    out = np.zeros(32 * n, np.uint8)
    ctx.call("acegpu_bn_field_batch", field, 0, A, B, n, out)
    ref = O.buf(32 * n)
    O.oracle().bn_batch(C.c_int(field), C.c_int(0), O.ptr(A), O.ptr(B), C.c_uint64(n), ref)
    assert out.tobytes() == bytes(ref)


def oracle_ntt(vals, logn, inverse, coset):
    buf = (C.c_uint8 * (32 << logn)).from_buffer_copy(b"".join(le(v) for v in vals))
    O.oracle().bn_ntt(buf, C.c_uint32(logn), C.c_int(inverse), C.c_int(coset), C.c_int(8))
    return ints(np.frombuffer(bytes(buf), np.uint8))


@pytest.mark.parametrize("logn", [0, 1, 2, 3, 5, 8, 11, 12, 13, 14, 16, 17])
def test_ntt_matches_oracle(ctx, logn):
    rng = random.Random(logn)
    vals = [rng.randrange(R) for _ in range(1 << logn)]
    for inverse in (0, 1):
        for coset in (0, 1):
            data = arr(vals)
            ctx.call("acegpu_bn_ntt", data, logn, inverse, coset)
            assert ints(data) == oracle_ntt(vals, logn, inverse, coset), (inverse, coset)


def test_ntt_small_vs_naive_dft(ctx):
    for logn in range(0, 8):
        vals = [random.randrange(R) for _ in range(1 << logn)]
        data = arr(vals)
        ctx.call("acegpu_bn_ntt", data, logn, 0, 0)
        ref = O.buf(32 << logn)
        O.oracle().bn_dft_naive(O.ptr(arr(vals)), C.c_uint32(logn), C.c_int(0), ref)
        assert data.tobytes() == bytes(ref)


@pytest.mark.parametrize("logn", [20, 22, 23, 24])
def test_ntt_large_roundtrip_and_oracle(ctx, logn):
    """2^22 (BASELINE configs[1]) and 2^20 (two passes), 2^23 and 2^24 (the
    three-pass transform of block-size domains): forward, inverse and
    coset-forward transforms each bit-exact vs the oracle's radix-2 NTT
    (multi-threaded, ~1 s at 2^22), plus iNTT(NTT(x)) = x and the coset round
    trip."""
    import os
    thr = C.c_int(os.cpu_count() or 8)
    rng = np.random.default_rng(logn)
    n = 1 << logn
    raw = rng.integers(0, 2**63, size=(n, 4), dtype=np.uint64)
    raw[:, 3] &= (1 << 61) - 1  # < 2^253 < r: canonical
    orig = raw.view(np.uint8).reshape(-1).copy()

    def oracle(x, inverse, coset):
        y = x.copy()
        O.oracle().bn_ntt((C.c_uint8 * (32 * n)).from_buffer(y), C.c_uint32(logn),
                          C.c_int(inverse), C.c_int(coset), thr)
        return y
    data = orig.copy()
    ctx.call("acegpu_bn_ntt", data, logn, 0, 0)
    fwd = data.copy()
    assert not np.array_equal(fwd, orig)
    assert np.array_equal(fwd, oracle(orig, 0, 0)), "forward"
    inv = orig.copy()
    ctx.call("acegpu_bn_ntt", inv, logn, 1, 0)
    assert np.array_equal(inv, oracle(orig, 1, 0)), "inverse"
    cos = orig.copy()
    ctx.call("acegpu_bn_ntt", cos, logn, 0, 1)
    assert np.array_equal(cos, oracle(orig, 0, 1)), "coset forward"
    ctx.call("acegpu_bn_ntt", data, logn, 1, 0)
    assert np.array_equal(data, orig)
    ctx.call("acegpu_bn_ntt", cos, logn, 1, 1)
    assert np.array_equal(cos, orig)


@pytest.mark.parametrize("logn", [25, 26, 27, 28])
def test_ntt_block_domains_sparse_evaluations_and_roundtrip(ctx, logn):
    """Block-size domains up to 2^28 (a whole 100k-tx block: 8.6 GB per
    vector, device resident; each size has its own three-pass split): a
    sparse input's forward and coset-forward transforms checked at sampled
    outputs against X[k] = sum_i x_i (g^c w^k)^i evaluated here, and
    iNTT(NTT(x)) = x on dense random data."""
    import torch
    n = 1 << logn
    dev = torch.device("cuda:0")
    rng = random.Random(logn)
    w = pow(5, (R - 1) >> logn, R)
    pos = sorted(rng.sample(range(n), 64))
    val = [rng.randrange(R) for _ in pos]
    ks = [0, 1, 2, n - 1, n // 2, n // 3] + [rng.randrange(n) for _ in range(10)]
    buf = torch.zeros(n, 32, dtype=torch.uint8, device=dev)
    src = torch.from_numpy(np.frombuffer(b"".join(le(v) for v in val), np.uint8).reshape(-1, 32).copy())
    try:
        for coset in (0, 1):
            buf.zero_()
            buf[torch.tensor(pos, device=dev)] = src.to(dev)
            p = buf.data_ptr()
            ctx.call("acegpu_bn_convert_dev", None, 1, p, n, 1)
            ctx.call("acegpu_bn_ntt_dev", None, p, p, logn, 0, coset)
            ctx.call("acegpu_bn_convert_dev", None, 1, p, n, 0)
            got = ints(buf[torch.tensor(ks, device=dev)].cpu().numpy().reshape(-1))
            for k, gk in zip(ks, got):
                z = pow(w, k, R) * (5 if coset else 1) % R
                assert gk == sum(v * pow(z, i, R) for i, v in zip(pos, val)) % R, (coset, k)
        # dense round trip (values < 2^253: canonical)
        g = torch.Generator(device=dev).manual_seed(7)
        x = torch.randint(0, 256, (n, 32), dtype=torch.uint8, device=dev, generator=g)
        x[:, 31] &= 0x1F
        orig = x.clone()
        p = x.data_ptr()
        ctx.call("acegpu_bn_convert_dev", None, 1, p, n, 1)
        ctx.call("acegpu_bn_ntt_dev", None, p, p, logn, 0, 1)
        ctx.call("acegpu_bn_ntt_dev", None, p, p, logn, 1, 1)
        ctx.call("acegpu_bn_convert_dev", None, 1, p, n, 0)
        assert torch.equal(x, orig)
        del x, orig
    finally:
        del buf
        torch.cuda.empty_cache()


def g_gen(group):
    g = O.buf(64 * group)
    O.oracle().bn_generator(C.c_int(group), g)
    return bytes(g)


@pytest.mark.parametrize("group", [1, 2])
def test_scalar_muls_match_oracle(ctx, group):
    rng = random.Random(group)
    ks = [0, 1, 2, 3, R - 1, R - 2] + [rng.randrange(R) for _ in range(200)]
    G = np.frombuffer(g_gen(group), np.uint8).copy()
    out = np.zeros(64 * group * len(ks), np.uint8)
    ctx.call("acegpu_bn_scalar_muls", group, G, arr(ks), len(ks), out)
    for i, k in enumerate(ks):
        ref = O.buf(64 * group)
        O.oracle().bn_scalar_mul(C.c_int(group), O.ptr(bytes(G)), O.ptr(le(k)), ref)
        assert out[64 * group * i:64 * group * (i + 1)].tobytes() == bytes(ref), (i, k)


def msm_gpu(ctx, group, pts, scalars, n, vb_sub=None):
    """Fixed-base MSM, or the variable-base form (vb_sub = its sub-range
    size, 0 = default) when vb_sub is given."""
    from paper_2603_10242_b200 import _native as N
    h = C.c_void_p()
    if vb_sub is None:
        ctx.call("acegpu_bn_msm_prepare", group, pts, n, 0, C.byref(h))
    else:
        ctx.call("acegpu_bn_msm_prepare_vb", group, pts, n, 0, vb_sub, C.byref(h))
    try:
        out = np.zeros(64 * group, np.uint8)
        ctx.call("acegpu_bn_msm_run", h, scalars, out)
        return out.tobytes()
    finally:
        N.lib().acegpu_bn_msm_free(h)


@pytest.mark.parametrize("group,n", [(1, 1), (1, 2), (1, 700), (1, 5000), (2, 300)])
def test_msm_matches_oracle(ctx, group, n):
    rng = random.Random(1000 * group + n)
    ks = [rng.randrange(1, R) for _ in range(n)]
    G = np.frombuffer(g_gen(group), np.uint8).copy()
    pts = np.zeros(64 * group * n, np.uint8)
    ctx.call("acegpu_bn_scalar_muls", group, G, arr(ks), n, pts)
    sc = [rng.randrange(R) for _ in range(n)]
    special = [0, 1, R - 1, 2, R - 2, 1 << 253]
    for j, v in enumerate(special[:n]):
        sc[j] = v
    got = msm_gpu(ctx, group, pts, arr(sc), n)
    ref = O.buf(64 * group)
    O.oracle().bn_msm(C.c_int(group), O.ptr(pts.tobytes()), O.ptr(arr(sc).tobytes()),
                      C.c_uint64(n), ref, C.c_int(8))
    assert got == bytes(ref)
    # discrete-log cross-check: sum s_i k_i mod r times G
    e = sum(s * k for s, k in zip(sc, ks)) % R
    dl = O.buf(64 * group)
    O.oracle().bn_scalar_mul(C.c_int(group), O.ptr(bytes(G)), O.ptr(le(e)), dl)
    assert got == bytes(dl)


def test_msm_degenerate_scalars(ctx):
    """Skewed digit distributions: all-equal scalars (one huge bucket), all
    zero, repeated bases, an infinity base."""
    n = 20000
    G = np.frombuffer(g_gen(1), np.uint8).copy()
    ks = [(i % 7) + 1 for i in range(n)]
    pts = np.zeros(64 * n, np.uint8)
    ctx.call("acegpu_bn_scalar_muls", 1, G, arr(ks), n, pts)
    pts[64 * 5:64 * 6] = 0  # infinity base
    for sc, label in [([1] * n, "ones"), ([0] * n, "zeros"), ([R - 1] * n, "minus ones"),
                      ([(1 << 16) + 3] * n, "two windows"), ([(1 << 17) + 5] * n, "c=17 edge"),
                      ([i & 1 for i in range(n)], "0/1 witness")]:
        got = msm_gpu(ctx, 1, pts, arr(sc), n)
        e = sum(s * (k if i != 5 else 0) for i, (s, k) in enumerate(zip(sc, ks))) % R
        dl = O.buf(64)
        O.oracle().bn_scalar_mul(C.c_int(1), O.ptr(bytes(G)), O.ptr(le(e)), dl)
        assert got == bytes(dl), label


@pytest.mark.parametrize("group,n", [(2, 3000), (1, 1 << 18)])
def test_msm_heavy_buckets(ctx, group, n):
    """A 0/1-valued witness (one bucket holds every window-0 entry: it spans
    thousands of accumulation segments and goes through the heavy-bucket
    queue) on G2 and at 2^18 points on G1, checked by discrete logs."""
    G = np.frombuffer(g_gen(group), np.uint8).copy()
    ks = [(i * 2654435761) % (1 << 40) + 1 for i in range(n)]
    pts = np.zeros(64 * group * n, np.uint8)
    ctx.call("acegpu_bn_scalar_muls", group, G, arr(ks), n, pts)
    sc = [(i % 3) & 1 for i in range(n)]
    sc[-1] = R - 1
    got = msm_gpu(ctx, group, pts, arr(sc), n)
    e = sum(s * k for s, k in zip(sc, ks)) % R
    dl = O.buf(64 * group)
    O.oracle().bn_scalar_mul(C.c_int(group), O.ptr(bytes(G)), O.ptr(le(e)), dl)
    assert got == bytes(dl)


@pytest.mark.parametrize("c20", [False, True])
@pytest.mark.parametrize("group,n,sub", [(1, 1, 0), (1, 5000, 0), (1, 5000, 777), (2, 3000, 1000),
                                         (1, 20000, 4096)])
def test_msm_variable_base_matches_fixed_base_and_oracle(ctx, group, n, sub, c20, monkeypatch):
    """The variable-base MSM (a whole block's keys: no window tables, one
    bucket set per window, sub-ranges Horner-combined) equals the fixed-base
    MSM and the oracle on the same bases and scalars, including the 0/1
    witness shape (heavy buckets) and sub-ranges that do not divide n; both
    window sizes (c = 17 up to 2^25 points, c = 20 above: forced here)."""
    if c20:
        monkeypatch.setenv("ACEGPU_MSM_VB_SMALL", "0")
    rng = random.Random(7 * n + group + sub)
    ks = [rng.randrange(1, R) for _ in range(n)]
    G = np.frombuffer(g_gen(group), np.uint8).copy()
    pts = np.zeros(64 * group * n, np.uint8)
    ctx.call("acegpu_bn_scalar_muls", group, G, arr(ks), n, pts)
    for label, sc in [("random", [rng.randrange(R) for _ in range(n)]),
                      ("0/1", [(i % 3) & 1 for i in range(n)])]:
        sc[0] = R - 1
        vb = msm_gpu(ctx, group, pts, arr(sc), n, vb_sub=sub)
        assert vb == msm_gpu(ctx, group, pts, arr(sc), n), label
        ref = O.buf(64 * group)
        O.oracle().bn_msm(C.c_int(group), O.ptr(pts.tobytes()), O.ptr(arr(sc).tobytes()),
                          C.c_uint64(n), ref, C.c_int(8))
        assert vb == bytes(ref), label


def test_msm_2_20_discrete_log(ctx):
    """BASELINE configs[1]: G1 MSM of 2^20 points, checked exactly through
    known discrete logs (bases k_i * G)."""
    n = 1 << 20
    rng = np.random.default_rng(20)
    kraw = rng.integers(0, 2**63, size=(n, 4), dtype=np.uint64)
    kraw[:, 3] &= (1 << 61) - 1
    sraw = rng.integers(0, 2**63, size=(n, 4), dtype=np.uint64)
    sraw[:, 3] &= (1 << 61) - 1
    K = kraw.view(np.uint8).reshape(-1).copy()
    S = sraw.view(np.uint8).reshape(-1).copy()
    G = np.frombuffer(g_gen(1), np.uint8).copy()
    pts = np.zeros(64 * n, np.uint8)
    ctx.call("acegpu_bn_scalar_muls", 1, G, K, n, pts)
    for i in (0, 1, n // 2, n - 1):  # spot-check the generated bases
        ref = O.buf(64)
        O.oracle().bn_scalar_mul(C.c_int(1), O.ptr(bytes(G)), O.ptr(K[32 * i:32 * i + 32].tobytes()), ref)
        assert pts[64 * i:64 * i + 64].tobytes() == bytes(ref)
    got = msm_gpu(ctx, 1, pts, S, n)
    ki = [int.from_bytes(K[32 * i:32 * i + 32].tobytes(), "little") for i in range(n)]
    si = [int.from_bytes(S[32 * i:32 * i + 32].tobytes(), "little") for i in range(n)]
    e = sum(a * b for a, b in zip(si, ki)) % R
    dl = O.buf(64)
    O.oracle().bn_scalar_mul(C.c_int(1), O.ptr(bytes(G)), O.ptr(le(e)), dl)
    assert got == bytes(dl)


def test_integer_peaks_positive(ctx):
    v = C.c_double()
    ctx.call("acegpu_imad_peak", C.byref(v))
    assert v.value > 1e12
    for f in (0, 1):
        ctx.call("acegpu_bn_mul_rate", f, C.byref(v))
        assert v.value > 1e9


def test_eip196_vectors_on_gpu(ctx):
    """EIP-196 ecMul / ecAdd vectors (tests/golden/eip196_197.json) through the
    GPU: scalar multiplication (acegpu_bn_scalar_muls) and a 2-point MSM with
    unit scalars (the bucket additions)."""
    import eip_vectors as E
    from paper_2603_10242_b200 import bn254
    d = E.load()
    for v in d["ecmul"]:
        p, k, exp = E.ecmul(v)
        out = bn254.scalar_muls(1, np.frombuffer(p, np.uint8).copy(),
                                np.frombuffer(k, np.uint8).copy(), ctx)
        assert out.tobytes() == exp, v["name"]
    one = np.frombuffer((1).to_bytes(32, "little") * 2, np.uint8).copy()
    for v in d["ecadd"]:
        a, b, exp = E.ecadd(v)
        if a == b:  # the doubling vector: MSM of one point with scalar 2
            bases = bn254.MsmBases(1, np.frombuffer(a, np.uint8).copy(), 1, ctx=ctx)
            got = bases.run(np.frombuffer((2).to_bytes(32, "little"), np.uint8).copy())
        else:
            bases = bn254.MsmBases(1, np.frombuffer(a + b, np.uint8).copy(), 2, ctx=ctx)
            got = bases.run(one)
        bases.close()
        assert got.tobytes() == exp, v["name"]


@pytest.mark.parametrize("logk", [0, 1, 2, 5, 8, 10, 12, 13])
def test_ntt3_matches_naive_dft(ctx, logk):
    """Mixed-radix NTT of 3 * 2^k points (Groth16 domains just above a power
    of two) vs the oracle's O(n^2) DFT (bn_dft_naive_n), forward / inverse /
    coset both ways, plus the round trips."""
    n = 3 << logk
    rng = random.Random(100 + logk)
    vals = [rng.randrange(R) for _ in range(n)]
    modes = [(i, c) for i in (0, 1) for c in (0, 1)] if logk <= 10 else [(0, 1), (1, 1)]
    for inverse, coset in modes:
        if True:
            data = arr(vals)
            ctx.call("acegpu_bn_ntt3", data, logk, inverse, coset)
            ref = O.buf(32 * n)
            O.oracle().bn_dft_naive_n(O.ptr(arr(vals).tobytes()), C.c_uint32(logk), C.c_int(1),
                                      C.c_int(inverse), C.c_int(coset), ref)
            assert data.tobytes() == bytes(ref), (inverse, coset)
    for coset in (0, 1):
        data = arr(vals)
        ctx.call("acegpu_bn_ntt3", data, logk, 0, coset)
        ctx.call("acegpu_bn_ntt3", data, logk, 1, coset)
        assert ints(data) == vals


@pytest.mark.parametrize("logk", [19, 26])
def test_ntt3_large_sparse_evaluations_and_roundtrip(ctx, logk):
    """3 * 2^19 (a paper-size chunk's domain) and 3 * 2^26 (a 100k block's):
    sampled outputs of sparse inputs vs sums evaluated here, and the coset
    round trip on dense device data."""
    import torch
    n = 3 << logk
    dev = torch.device("cuda:0")
    rng = random.Random(logk)
    w = pow(5, (R - 1) // n, R)
    pos = sorted(rng.sample(range(n), 48))
    val = [rng.randrange(R) for _ in pos]
    ks = [0, 1, 2, n - 1, n // 3, 2 * n // 3 + 5] + [rng.randrange(n) for _ in range(8)]
    buf = torch.zeros(n, 32, dtype=torch.uint8, device=dev)
    src = torch.from_numpy(np.frombuffer(b"".join(le(v) for v in val), np.uint8).reshape(-1, 32).copy())
    try:
        for coset in (0, 1):
            buf.zero_()
            buf[torch.tensor(pos, device=dev)] = src.to(dev)
            p = buf.data_ptr()
            ctx.call("acegpu_bn_convert_dev", None, 1, p, n, 1)
            ctx.call("acegpu_bn_ntt3_dev", None, p, p, logk, 0, coset)
            ctx.call("acegpu_bn_convert_dev", None, 1, p, n, 0)
            got = ints(buf[torch.tensor(ks, device=dev)].cpu().numpy().reshape(-1))
            for k, gk in zip(ks, got):
                z = pow(w, k, R) * (5 if coset else 1) % R
                assert gk == sum(v * pow(z, i, R) for i, v in zip(pos, val)) % R, (coset, k)
        g = torch.Generator(device=dev).manual_seed(9)
        x = torch.randint(0, 256, (n, 32), dtype=torch.uint8, device=dev, generator=g)
        x[:, 31] &= 0x1F
        orig = x.clone()
        p = x.data_ptr()
        ctx.call("acegpu_bn_convert_dev", None, 1, p, n, 1)
        ctx.call("acegpu_bn_ntt3_dev", None, p, p, logk, 0, 1)
        ctx.call("acegpu_bn_ntt3_dev", None, p, p, logk, 1, 1)
        ctx.call("acegpu_bn_convert_dev", None, 1, p, n, 0)
        assert torch.equal(x, orig)
        del x, orig
    finally:
        del buf
        torch.cuda.empty_cache()


def test_msm_variable_base_windowed_sort_large(ctx):
    """From 2^22 points the variable-base digit sort runs in window passes
    (window-major keys, L2-sized scatter ranges) and the windows are c = 20
    (8 x 20 + 5 x 19 bits): at 2^22 + 5 points (bases tiled from 2^16
    generated points, random scalars, the first few edge values) the result
    equals the fixed-base MSM over the same bases."""
    import torch
    n0, n = 1 << 16, (1 << 22) + 5
    rng = np.random.default_rng(22)
    k = rng.integers(0, 2**63, size=(n0, 4), dtype=np.uint64)
    k[:, 3] &= (1 << 61) - 1
    G = np.frombuffer(g_gen(1), np.uint8).copy()
    base = np.zeros(64 * n0, np.uint8)
    ctx.call("acegpu_bn_scalar_muls", 1, G, k.view(np.uint8).reshape(-1), n0, base)
    pts = torch.from_numpy(base).cuda().repeat((n + n0 - 1) // n0)[:64 * n].contiguous()
    sc = torch.randint(0, 256, (n, 32), dtype=torch.uint8, device="cuda")
    sc[:, 31] &= 0x1F
    edge = torch.from_numpy(arr([0, 1, R - 1, 2, R - 2])).cuda().view(5, 32)
    sc[:5] = edge
    outs = []
    try:
        for vb in (1, 0):
            h = C.c_void_p()
            if vb:
                ctx.call("acegpu_bn_msm_prepare_vb", 1, pts.data_ptr(), n, 1, 0, C.byref(h))
            else:
                ctx.call("acegpu_bn_msm_prepare", 1, pts.data_ptr(), n, 1, C.byref(h))
            out = torch.empty(64, dtype=torch.uint8, device="cuda")
            ctx.call("acegpu_bn_msm_run_dev", None, h, sc.data_ptr(), out.data_ptr())
            torch.cuda.synchronize()
            outs.append(out.cpu().numpy().tobytes())
            from paper_2603_10242_b200 import _native as N
            N.lib().acegpu_bn_msm_free(h)
        assert outs[0] == outs[1] and any(outs[0])
    finally:
        del pts, sc
        torch.cuda.empty_cache()
