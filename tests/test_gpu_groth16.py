"""Groth16 chunk prover (synthetic ZK-ACE stand-in circuit) vs the
known-trapdoor oracle (oracle/bn254_oracle.c bn_g16_expected): the GPU's
proof points must equal [A]1, [B]2, [C]1 for the discrete logs the oracle
derives from the trapdoor, and those satisfy the Groth16 verification
identity (the pairing check in exponents). Parity unpinned by the reference
(it has no Groth16)."""
import ctypes as C
import hashlib
import random

import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu

R = 0x30644E72E131A029B85045B68181585D2833E84879B9709143E1F593F0000001


def le(x):
    return x.to_bytes(32, "little")


def arr(vals):
    return np.frombuffer(b"".join(le(v) for v in vals), np.uint8).copy()


def expected_points(T, K, w, pub, trap, rs):
    out = O.buf(96)
    ok = O.oracle().bn_g16_expected(C.c_uint32(T), C.c_uint32(K), O.ptr(w.tobytes()),
                                    O.ptr(pub.tobytes()), O.ptr(trap.tobytes()),
                                    O.ptr(rs.tobytes()), out, C.c_int(8))
    assert ok == 1, "oracle verification identity"
    A, B, Cc = (bytes(out)[32 * i:32 * i + 32] for i in range(3))
    pts = []
    for g, k in ((1, A), (2, B), (1, Cc)):
        G = O.buf(64 * g)
        O.oracle().bn_generator(C.c_int(g), G)
        P = O.buf(64 * g)
        O.oracle().bn_scalar_mul(C.c_int(g), G, O.ptr(k), P)
        pts.append(bytes(P))
    return pts


def be_from_le(b32):
    return bytes(reversed(b32))


@pytest.fixture(scope="module")
def ctx():
    from paper_2603_10242_b200 import _native as N
    return N.context(0)


@pytest.mark.parametrize("T,K", [(1, 2), (3, 4), (8, 5), (64, 100)])
def test_groth16_chunk_matches_trapdoor_oracle(ctx, T, K):
    from paper_2603_10242_b200 import groth16
    rng = random.Random(T * 1000 + K)
    trap = arr([rng.randrange(1, R) for _ in range(5)])
    pk = groth16.ProvingKey(T, K, trap, ctx)
    try:
        w = arr([rng.randrange(R) for _ in range(T)])
        pub = arr([rng.randrange(R) for _ in range(T)])
        rs = arr([rng.randrange(R), rng.randrange(R)])
        proof, raw, _ = pk.prove(w, pub, rs)
        A, B, Cc = expected_points(T, K, w, pub, trap, rs)
        assert raw[:64] == A, "A"
        assert raw[64:192] == B, "B"
        assert raw[192:] == Cc, "C"
        # EIP-197 serialisation: G1 x|y, G2 x.c1|x.c0|y.c1|y.c0, big-endian
        assert proof[:32] == be_from_le(A[:32]) and proof[32:64] == be_from_le(A[32:64])
        assert proof[64:96] == be_from_le(B[32:64]) and proof[96:128] == be_from_le(B[:32])
        assert proof[128:160] == be_from_le(B[96:128]) and proof[160:192] == be_from_le(B[64:96])
        assert proof[192:224] == be_from_le(Cc[:32])
    finally:
        pk.close()


def test_groth16_deterministic_rs(ctx):
    """r, s = LE(SHA-256(tag | pub_0 | pub_{T-1} | T_be32)) mod r:
    same inputs -> identical proof bytes; matches explicit r, s."""
    from paper_2603_10242_b200 import groth16
    T, K = 5, 3
    rng = random.Random(5)
    trap = arr([rng.randrange(1, R) for _ in range(5)])
    pk = groth16.ProvingKey(T, K, trap, ctx)
    try:
        w = arr([rng.randrange(R) for _ in range(T)])
        pub = arr([rng.randrange(R) for _ in range(T)])
        p1, raw1, d1 = pk.prove(w, pub)
        p2, _, _ = pk.prove(w, pub)
        assert p1 == p2
        pb = pub.tobytes()
        tail = pb[:32] + pb[32 * (T - 1):32 * T] + T.to_bytes(4, "big")
        r = int.from_bytes(hashlib.sha256(b"ace-g16-r-v1" + tail).digest(), "little") % R
        s = int.from_bytes(hashlib.sha256(b"ace-g16-s-v1" + tail).digest(), "little") % R
        p3, _, _ = pk.prove(w, pub, arr([r, s]))
        assert p3 == p1
        assert d1 == hashlib.sha256(b"ace-g16-chunk-v1" + tail).digest()
        A, B, Cc = expected_points(T, K, w, pub, trap, arr([r, s]))
        assert raw1 == A + B + Cc
    finally:
        pk.close()


def test_groth16_paper_size_chunk(ctx):
    """One 1,024-tx chunk at 1,400 constraints/tx (1,434,625 constraints,
    domain 2^21) against the trapdoor oracle."""
    from paper_2603_10242_b200 import groth16
    T, K = groth16.PAPER_T, groth16.PAPER_K
    rng = np.random.default_rng(7)
    def rnd(n):
        raw = rng.integers(0, 2**63, size=(n, 4), dtype=np.uint64)
        raw[:, 3] &= (1 << 61) - 1
        return raw.view(np.uint8).reshape(-1).copy()
    trap = rnd(5)
    pk = groth16.ProvingKey(T, K, trap, ctx)
    try:
        assert pk.constraints == 1_434_625 and pk.log_domain == 21
        w, pub, rs = rnd(T), rnd(T), rnd(2)
        proof, raw, _ = pk.prove(w, pub, rs)
        A, B, Cc = expected_points(T, K, w, pub, trap, rs)
        assert raw == A + B + Cc
    finally:
        pk.close()
