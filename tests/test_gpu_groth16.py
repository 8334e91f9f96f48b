"""Groth16 chunk prover (synthetic ZK-ACE stand-in circuit) vs the
known-trapdoor oracle (oracle/bn254_oracle.c bn_g16_expected): the GPU's
proof points must equal [A]1, [B]2, [C]1 for the discrete logs the oracle
derives from the trapdoor, and those satisfy the Groth16 verification
identity (the pairing check in exponents). Parity unpinned by the reference
(it has no Groth16)."""
import ctypes as C
import random

import numpy as np
import pytest

import g16_spec as SP
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


@pytest.mark.parametrize("T,K", [(1, 2), (3, 4), (8, 5), (64, 100), (5, 3), (11, 15), (100, 14)])
def test_groth16_chunk_matches_trapdoor_oracle(ctx, T, K):
    """(5, 3), (11, 15), (100, 14): m = 21, 177, 1,501 -> mixed-radix domains
    of 24, 192, 1,536 points (3 x 2^b below the next power of two)."""
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
    """r, s = LE(SHA-256(tag | D(w) | D(pub))) mod r (binding v2):
    same inputs -> identical proof bytes; matches explicit r, s (tests/g16_spec.py)."""
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
        r, s = SP.derive_rs(w.tobytes(), pub.tobytes(), T)
        p3, _, _ = pk.prove(w, pub, arr([r, s]))
        assert p3 == p1
        assert d1 == SP.chunk_digest(pub.tobytes(), T)
        A, B, Cc = expected_points(T, K, w, pub, trap, arr([r, s]))
        assert raw1 == A + B + Cc
    finally:
        pk.close()


@pytest.mark.parametrize("T", [5, 33, 64, 1100, 2100])
def test_groth16_binding_covers_every_input(ctx, T):
    """Binding v2: flipping one MIDDLE public input changes r, s,
    the chunk digest and the verifier's weight seed; flipping a middle
    witness changes r and s but not the chunk digest. The GPU's values equal
    the Python statement of the rules (tests/g16_spec.py)."""
    from paper_2603_10242_b200 import groth16
    K = 3
    rng = random.Random(T)
    trap = arr([rng.randrange(1, R) for _ in range(5)])
    pk = groth16.ProvingKey(T, K, trap, ctx)
    try:
        vk = pk.verifying_key()
        w = arr([rng.randrange(R) for _ in range(T)])
        pub = arr([rng.randrange(R) for _ in range(T)])
        p0, raw0, d0 = pk.prove(w, pub)
        r0, s0 = SP.derive_rs(w.tobytes(), pub.tobytes(), T)
        assert raw0 == b"".join(expected_points(T, K, w, pub, trap, arr([r0, s0])))
        assert d0 == SP.chunk_digest(pub.tobytes(), T)
        ok, seed0 = pk.verify_batch([p0], [pub.tobytes()], return_seed=True)
        assert ok and seed0 == SP.batch_seed(vk, [p0], [pub.tobytes()], T)
        mid = T // 2
        pub1 = pub.copy()
        pub1[32 * mid + 5] ^= 1
        p1, raw1, d1 = pk.prove(w, pub1)
        r1, s1 = SP.derive_rs(w.tobytes(), pub1.tobytes(), T)
        assert (r1, s1) != (r0, s0) and r1 != r0 and s1 != s0
        assert raw1 == b"".join(expected_points(T, K, w, pub1, trap, arr([r1, s1])))
        assert d1 != d0 and d1 == SP.chunk_digest(pub1.tobytes(), T)
        ok1, seed1 = pk.verify_batch([p0], [pub1.tobytes()], return_seed=True)
        assert not ok1 and seed1 != seed0
        assert seed1 == SP.batch_seed(vk, [p0], [pub1.tobytes()], T)
        w2 = w.copy()
        w2[32 * mid + 1] ^= 2
        _, raw2, d2 = pk.prove(w2, pub)
        r2, s2 = SP.derive_rs(w2.tobytes(), pub.tobytes(), T)
        assert r2 != r0 and s2 != s0 and d2 == d0
        assert raw2 == b"".join(expected_points(T, K, w2, pub, trap, arr([r2, s2])))
    finally:
        pk.close()


def test_batch_verifier_rejects_compensated_inputs(ctx):
    """with weights that did not commit to the public
    inputs, pub_0[j] += d and pub_1[j] -= (rho_0 / rho_1) d would leave
    sum_i rho_i z_ij unchanged and pass. The weights now hash every public
    input, so the compensated pair (built from the honest weights) fails."""
    from paper_2603_10242_b200 import groth16
    T, K = 8, 3
    rng = random.Random(99)
    trap = arr([rng.randrange(1, R) for _ in range(5)])
    pk = groth16.ProvingKey(T, K, trap, ctx)
    try:
        vk = pk.verifying_key()
        proofs, pubs = [], []
        for _ in range(2):
            w = arr([rng.randrange(R) for _ in range(T)])
            pub = arr([rng.randrange(R) for _ in range(T)])
            proofs.append(pk.prove(w, pub)[0])
            pubs.append(pub.tobytes())
        ok, seed = pk.verify_batch(proofs, pubs, return_seed=True)
        assert ok and seed == SP.batch_seed(vk, proofs, pubs, T)
        rho0, rho1 = SP.batch_rho(seed, 0), SP.batch_rho(seed, 1)
        j, d = 3, 12345
        q0 = int.from_bytes(pubs[0][32 * j:32 * j + 32], "little") % R
        q1 = int.from_bytes(pubs[1][32 * j:32 * j + 32], "little") % R
        n0 = (q0 + d) % R
        n1 = (q1 - rho0 * pow(rho1, -1, R) * d) % R
        assert (rho0 * n0 + rho1 * n1) % R == (rho0 * q0 + rho1 * q1) % R  # the old attack
        e0 = bytearray(pubs[0]); e0[32 * j:32 * j + 32] = le(n0)
        e1 = bytearray(pubs[1]); e1[32 * j:32 * j + 32] = le(n1)
        ok2, seed2 = pk.verify_batch(proofs, [bytes(e0), bytes(e1)], return_seed=True)
        assert seed2 != seed and not ok2
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
        assert pk.constraints == 1_434_625 and pk.domain == 3 << 19  # 1.57 M (2^21 = 2.10 M)
        w, pub, rs = rnd(T), rnd(T), rnd(2)
        proof, raw, _ = pk.prove(w, pub, rs)
        A, B, Cc = expected_points(T, K, w, pub, trap, rs)
        assert raw == A + B + Cc
    finally:
        pk.close()


@pytest.mark.parametrize("n,world", [(1, 1), (11, 1), (11, 2), (16, 3), (37, 4)])
def test_groth16_block_shards(ctx, n, world):
    """Groth16 mode end to end: attestation + per-tx public-input digests ->
    one Groth16 proof per aligned 4-tx chunk (last chunk zero-padded) ->
    reference tree rule over chunk proofs -> FC; ranks emulated in sequence.
    Each chunk proof is checked against the trapdoor oracle; the root and FC
    against the oracle's aggregate_tree / merkle_root."""
    from paper_2603_10242_b200 import groth16, shard, wire
    T, K = 4, 3
    rng = random.Random(n * 10 + world)
    trap = arr([rng.randrange(1, R) for _ in range(5)])
    pk = groth16.ProvingKey(T, K, trap, ctx)
    try:
        fb = O.multi_user_block(n, 3)
        # witnesses: build_witness(attest_key, tx_hash) (prover.cpp:181-188)
        wit = b""
        for i in range(n):
            att = fb.att(i)
            u = int(fb.rev_index[i])
            key = O.derive_attest_key(fb.revs[32 * u:32 * u + 32].tobytes(), att[64:72])
            out = O.buf(256)
            O.oracle().or_build_witness(O.ptr(key), O.ptr(att[:32]), out)
            wit += bytes(out)
        witnesses = np.frombuffer(wit, np.uint8).copy()
        wfb = wire.FlatBlock(fb.payloads, fb.offs, fb.atts, np.frombuffer(fb.header, np.uint8).copy())
        proof, fc = shard.prove_sharded_single_process(wfb, world, 2, ctx, pk=pk, witnesses=witnesses)
        # expected: per-chunk proofs from the chunk prover on the same inputs
        digests = []
        for i in range(n):
            p = O.buf(289)
            O.oracle().or_prove_tx(O.ptr(fb.payload(i)), C.c_uint64(len(fb.payload(i))),
                                   O.ptr(fb.att(i)), p)
            digests.append(bytes(p)[256:288])
        nodes = b""
        for c0 in range(0, n, T):
            pubs = digests[c0:c0 + T] + [bytes(32)] * (T - len(digests[c0:c0 + T]))
            ws = [wit[256 * i:256 * i + 32] for i in range(c0, min(n, c0 + T))]
            ws += [bytes(32)] * (T - len(ws))
            pa = np.frombuffer(b"".join(pubs), np.uint8).copy()
            wa = np.frombuffer(b"".join(ws), np.uint8).copy()
            pr, raw, dg = pk.prove(wa, pa)
            # the chunk proof verifies (trapdoor oracle), with the derived r, s
            r, s = SP.derive_rs(b"".join(ws), b"".join(pubs), T)
            wred = arr([int.from_bytes(x, "little") % R for x in ws])
            pred = arr([int.from_bytes(x, "little") % R for x in pubs])
            assert raw == b"".join(expected_points(T, K, wred, pred, trap, arr([r, s])))
            nodes += pr + dg + b"\0"
        out = O.buf(289)
        lv, pp = C.c_uint64(), C.c_uint64()
        O.oracle().or_aggregate_tree(O.ptr(nodes), C.c_uint64(len(nodes) // 289), out,
                                     C.byref(lv), C.byref(pp))
        assert proof == bytes(out)
        assert fc == O.oracle_build_fc(fb, bytes(out))
    finally:
        pk.close()


# ------------------------------------------------------------- verifier
def _vk_oracle(T, K, trap):
    vk = O.buf(448 + 64 * (T + 1))
    O.oracle().bn_g16_vk(C.c_uint32(T), C.c_uint32(K), O.ptr(trap.tobytes()), vk)
    return bytes(vk)


@pytest.mark.parametrize("T,K", [(1, 2), (4, 3), (64, 20), (5, 3), (100, 14)])
def test_verifying_key_matches_oracle(ctx, T, K):
    from paper_2603_10242_b200 import _native as N, groth16
    rng = random.Random(T + 7 * K)
    trap = arr([rng.randrange(1, R) for _ in range(5)])
    pk = groth16.ProvingKey(T, K, trap, ctx)
    try:
        out = np.zeros(448 + 64 * (T + 1), np.uint8)
        ctx.call("acegpu_g16_vk", pk.h, N.addr(out))
        assert out.tobytes() == _vk_oracle(T, K, trap)
    finally:
        pk.close()


def test_gpu_proofs_verify_under_oracle_pairing(ctx):
    """The GPU prover's proofs pass the oracle's pairing verifier (bn_g16_verify,
    a full e(A,B) = e(alpha,beta) e(L,gamma) e(C,delta) check)."""
    from paper_2603_10242_b200 import groth16
    T, K = 4, 3
    rng = random.Random(5)
    trap = arr([rng.randrange(1, R) for _ in range(5)])
    pk = groth16.ProvingKey(T, K, trap, ctx)
    try:
        vk = _vk_oracle(T, K, trap)
        for _ in range(2):
            w = arr([rng.randrange(R) for _ in range(T)])
            pub = arr([rng.randrange(R) for _ in range(T)])
            _, raw, _ = pk.prove(w, pub)
            assert O.oracle().bn_g16_verify(C.c_uint32(T), O.ptr(vk), O.ptr(raw),
                                            O.ptr(pub.tobytes())) == 1
            bad = bytearray(pub.tobytes())
            bad[3] ^= 4
            assert O.oracle().bn_g16_verify(C.c_uint32(T), O.ptr(vk), O.ptr(raw),
                                            O.ptr(bytes(bad))) == 0
    finally:
        pk.close()


def _gpu_verify(ctx, pk, proofs, pubs):
    from paper_2603_10242_b200 import _native as N
    ok = C.c_int(-1)
    p = np.frombuffer(b"".join(proofs), np.uint8).copy()
    q = np.frombuffer(b"".join(pubs), np.uint8).copy()
    ctx.call("acegpu_g16_verify_batch", pk.h, N.addr(p), N.addr(q), len(proofs), C.byref(ok))
    return ok.value


def test_gpu_batch_verifier(ctx):
    """acegpu_g16_verify_batch accepts honest proofs and rejects a changed
    public input, swapped proofs, an off-curve point and a B on the twist
    outside the order-r subgroup."""
    from paper_2603_10242_b200 import groth16
    T, K = 8, 3
    rng = random.Random(17)
    trap = arr([rng.randrange(1, R) for _ in range(5)])
    pk = groth16.ProvingKey(T, K, trap, ctx)
    try:
        proofs, pubs = [], []
        for _ in range(5):
            w = arr([rng.randrange(R) for _ in range(T)])
            pub = arr([rng.randrange(R) for _ in range(T)])
            proof, _, _ = pk.prove(w, pub)
            proofs.append(bytes(proof))
            pubs.append(pub.tobytes())
        assert _gpu_verify(ctx, pk, proofs, pubs) == 1
        assert _gpu_verify(ctx, pk, proofs[:1], pubs[:1]) == 1
        bad = bytearray(pubs[2])
        bad[40] ^= 1
        assert _gpu_verify(ctx, pk, proofs, pubs[:2] + [bytes(bad)] + pubs[3:]) == 0
        assert _gpu_verify(ctx, pk, [proofs[1], proofs[0]] + proofs[2:], pubs) == 0
        off = bytearray(proofs[3])
        off[63] ^= 1  # A.y changed: off the curve
        assert _gpu_verify(ctx, pk, proofs[:3] + [bytes(off)] + proofs[4:], pubs) == 0
        nb = bytearray(proofs[4])
        nb[64:192] = _twist_point_outside_g2(rng)
        assert _gpu_verify(ctx, pk, proofs[:4] + [bytes(nb)], pubs) == 0
        # raw digests >= r are reduced like the prover's
        assert _gpu_verify(ctx, pk, proofs, pubs) == 1
    finally:
        pk.close()


PQ = 0x30644E72E131A029B85045B68181585D97816A916871CA8D3C208C16D87CFD47


def _f2mul(a, b):
    return ((a[0] * b[0] - a[1] * b[1]) % PQ, (a[0] * b[1] + a[1] * b[0]) % PQ)


def _f2pow(a, e):
    r = (1, 0)
    while e:
        if e & 1:
            r = _f2mul(r, a)
        a = _f2mul(a, a)
        e >>= 1
    return r


def _f2sqrt(a):
    """Square root in Fq2 for p = 3 mod 4 (or None)."""
    a1 = _f2pow(a, (PQ - 3) // 4)
    alpha = _f2mul(_f2mul(a1, a1), a)
    x0 = _f2mul(a1, a)
    if alpha == (PQ - 1, 0):
        x = _f2mul((0, 1), x0)
    else:
        x = _f2mul(_f2pow(((1 + alpha[0]) % PQ, alpha[1]), (PQ - 1) // 2), x0)
    return x if _f2mul(x, x) == a else None


def _twist_point_outside_g2(rng):
    """A point of y^2 = x^3 + 3/(9+u) over Fq2 that is not in the order-r
    subgroup (the twist's cofactor is 2p - r), EIP-197-encoded (128 B)."""
    binv = _f2pow((9, 1), PQ * PQ - 2)
    b = ((3 * binv[0]) % PQ, (3 * binv[1]) % PQ)
    while True:
        x = (rng.randrange(PQ), rng.randrange(PQ))
        rhs = _f2mul(_f2mul(x, x), x)
        rhs = ((rhs[0] + b[0]) % PQ, (rhs[1] + b[1]) % PQ)
        y = _f2sqrt(rhs)
        if y is not None:
            break
    be = lambda v: v.to_bytes(32, "big")  # noqa: E731
    return be(x[1]) + be(x[0]) + be(y[1]) + be(y[0])


def _witnesses(fb, n):
    wit = b""
    for i in range(n):
        att = fb.att(i)
        u = int(fb.rev_index[i])
        key = O.derive_attest_key(fb.revs[32 * u:32 * u + 32].tobytes(), att[64:72])
        out = O.buf(256)
        O.oracle().or_build_witness(O.ptr(key), O.ptr(att[:32]), out)
        wit += bytes(out)
    return np.frombuffer(wit, np.uint8).copy()


@pytest.mark.parametrize("n", [4, 11, 37])
def test_groth16_verify_finality_certificate(ctx, n):
    """verify_finality_certificate in Groth16 mode: the
    prover's FC + chunk proofs verify by pairings; slot, header, payload and
    proof tampering give SlotMismatch / HashMismatch / ProofMismatch."""
    from paper_2603_10242_b200 import groth16, prover, shard, wire
    T, K = 4, 3
    rng = random.Random(n)
    trap = arr([rng.randrange(1, R) for _ in range(5)])
    pk = groth16.ProvingKey(T, K, trap, ctx)
    try:
        fb = O.multi_user_block(n, 3)
        wfb = wire.FlatBlock(fb.payloads, fb.offs, fb.atts,
                             np.frombuffer(fb.header, np.uint8).copy())
        _, fc, roots = shard.prove_sharded_single_process(
            wfb, 2, 2, ctx, pk=pk, witnesses=_witnesses(fb, n), return_roots=True)
        chunks = (n + T - 1) // T
        proofs = b"".join(roots[289 * k:289 * k + 256] for k in range(chunks))
        cu = prover.CostUnits()
        V = prover.FcCheck
        assert pk.verify_finality_certificate(fc, wfb, proofs, cu) == V.Valid
        assert cu.value == 1
        bad_slot = bytearray(fc)
        bad_slot[39] ^= 1
        assert pk.verify_finality_certificate(bytes(bad_slot), wfb, proofs) == V.SlotMismatch
        hdr = bytearray(fb.header)
        hdr[100] ^= 1  # a root byte: same slot, different block hash
        wfb2 = wire.FlatBlock(fb.payloads, fb.offs, fb.atts, np.frombuffer(bytes(hdr), np.uint8).copy())
        assert pk.verify_finality_certificate(fc, wfb2, proofs) == V.HashMismatch
        pay = fb.payloads.copy()
        pay[int(fb.offs[n - 1]) + 20] ^= 1  # last tx's payload -> its public input
        wfb3 = wire.FlatBlock(pay, fb.offs, fb.atts, np.frombuffer(fb.header, np.uint8).copy())
        assert pk.verify_finality_certificate(fc, wfb3, proofs) == V.ProofMismatch
        pr = bytearray(proofs)
        pr[0:256], pr[-256:] = pr[-256:], pr[0:256]
        if chunks > 1:
            assert pk.verify_finality_certificate(fc, wfb, bytes(pr)) == V.ProofMismatch
    finally:
        pk.close()


@pytest.mark.parametrize("n", [1, 11, 37])
def test_groth16_prove_block_host_call(ctx, n):
    """acegpu_g16_prove_block (one host-buffer call: H2D, verdicts, chunk
    proofs, tree, FC, D2H) == the device-resident shard path, and its chunk
    proofs verify the FC (verify_finality_certificate in Groth16 mode)."""
    from paper_2603_10242_b200 import groth16, prover, shard, wire
    T, K = 4, 3
    rng = random.Random(3 * n)
    trap = arr([rng.randrange(1, R) for _ in range(5)])
    pk = groth16.ProvingKey(T, K, trap, ctx)
    try:
        fb = O.multi_user_block(n, 3)
        wfb = wire.FlatBlock(fb.payloads, fb.offs, fb.atts, np.frombuffer(fb.header, np.uint8).copy())
        wit = _witnesses(fb, n)
        proof, fc, roots = shard.prove_sharded_single_process(wfb, 1, 2, ctx, pk=pk, witnesses=wit,
                                                              return_roots=True)
        codes, p2, fc2, cps = pk.prove_block(wfb, wit, np.frombuffer(fb.revs, np.uint8).copy(),
                                             np.asarray(fb.rev_index, np.uint32))
        assert p2 == proof and fc2 == fc
        assert (codes == 0).all()
        chunks = (n + T - 1) // T
        assert cps == b"".join(roots[289 * k:289 * k + 256] for k in range(chunks))
        assert pk.verify_finality_certificate(fc2, wfb, cps) == prover.FcCheck.Valid
        c3, p3, fc3, _ = pk.prove_block(wfb, wit)  # no REVs: verdicts skipped, proof unchanged
        assert p3 == proof and fc3 == fc
    finally:
        pk.close()


def test_groth16_mode_attestation_verdicts(ctx):
    """Groth16 mode runs the same batched HKDF/HMAC attestation check as the
    hash-proof path: per-tx verdicts are identical to the mock shard's (and
    all-accept on an honest block), including forged credentials."""
    import torch
    from paper_2603_10242_b200 import groth16, shard, wire
    T, K, n = 4, 3, 23
    pk = groth16.ProvingKey(T, K, arr([3, 5, 7, 11, 13]), ctx)
    try:
        fb = O.multi_user_block(n, 3)
        atts = fb.atts.copy()
        atts[104 * 5 + 100] ^= 1   # tx 5: credential bytes corrupted
        atts[104 * 17 + 90] ^= 4   # tx 17
        for forged in (False, True):
            a = atts if forged else fb.atts
            wfb = wire.FlatBlock(fb.payloads, fb.offs, a, np.frombuffer(fb.header, np.uint8).copy())
            revs = np.frombuffer(fb.revs, np.uint8).copy()
            rix = np.asarray(fb.rev_index, np.uint32)
            db = shard.DeviceBlock.upload(wfb, 0, n, revs, rix, device=0)
            db.witnesses = torch.zeros(256 * n, dtype=torch.uint8, device="cuda")
            got = {}
            for name, be in (("g16", shard.G16Backend(pk, ctx)), ("mock", shard.GpuBackend(ctx))):
                codes = torch.full((n,), 0xEE, dtype=torch.uint8, device="cuda")
                be.shard_roots(db, n, 2, codes=codes)
                torch.cuda.synchronize()
                got[name] = codes.cpu().numpy().copy()
            assert (got["g16"] == got["mock"]).all()
            bad = np.nonzero(got["g16"])[0].tolist()
            assert bad == ([5, 17] if forged else [])
    finally:
        pk.close()


@pytest.mark.parametrize("T,K", [(3, 4), (64, 100)])
def test_variable_base_key_proves_identical_proofs(ctx, T, K, monkeypatch):
    """A variable-base key (ACEGPU_G16_VB=1: the bases without window tables,
    one buffer slot — what a block-size key uses above 2^22) gives the same
    proof bytes as the fixed-base key, equal to the trapdoor oracle's."""
    from paper_2603_10242_b200 import groth16
    rng = random.Random(T + 7 * K)
    trap = arr([rng.randrange(1, R) for _ in range(5)])
    w = arr([rng.randrange(R) for _ in range(T)])
    pub = arr([rng.randrange(R) for _ in range(T)])
    rs = arr([rng.randrange(R), rng.randrange(R)])
    out = []
    for vb in ("0", "1"):
        monkeypatch.setenv("ACEGPU_G16_VB", vb)
        pk = groth16.ProvingKey(T, K, trap, ctx)
        try:
            out.append(pk.prove(w, pub, rs)[:2])
            out.append(pk.prove(w, pub)[:2])
        finally:
            pk.close()
    assert out[0] == out[2] and out[1] == out[3]
    assert out[0][1] == b"".join(expected_points(T, K, w, pub, trap, rs))


@pytest.mark.parametrize("n", [1, 37, 50])
def test_single_proof_per_block(ctx, n, monkeypatch):
    """One Groth16 proof for the whole block (the paper's FC: a single 256-B
    proof checked by pairings): a key whose T covers the block (T = 50, not
    a power of two) proves blocks of n <= T txs as one chunk; the FC carries
    that proof, verify_finality_certificate accepts it with the one proof
    and rejects tampering; the variable-base key gives the same FC."""
    from paper_2603_10242_b200 import groth16, prover, wire
    T, K = 50, 6
    rng = random.Random(50 + n)
    trap = arr([rng.randrange(1, R) for _ in range(5)])
    fb = O.multi_user_block(n, 3)
    wfb = wire.FlatBlock(fb.payloads, fb.offs, fb.atts, np.frombuffer(fb.header, np.uint8).copy())
    wit = _witnesses(fb, n)
    fcs = []
    for vb in ("0", "1"):
        monkeypatch.setenv("ACEGPU_G16_VB", vb)
        pk = groth16.ProvingKey(T, K, trap, ctx)
        try:
            codes, proof, fc, cps = pk.prove_block(wfb, wit)
            assert len(cps) == 256 and proof[:256] == cps
            V = prover.FcCheck
            assert pk.verify_finality_certificate(fc, wfb, cps) == V.Valid
            bad = bytearray(cps)
            bad[5] ^= 1
            assert pk.verify_finality_certificate(fc, wfb, bytes(bad)) == V.ProofMismatch
            pay = fb.payloads.copy()
            pay[int(fb.offs[n - 1]) + 20] ^= 1
            wfb3 = wire.FlatBlock(pay, fb.offs, fb.atts, np.frombuffer(fb.header, np.uint8).copy())
            assert pk.verify_finality_certificate(fc, wfb3, cps) == V.ProofMismatch
            fcs.append(fc)
        finally:
            pk.close()
    assert fcs[0] == fcs[1]
    if n > 32:  # a non-power-of-two key still rejects blocks above T
        pk = groth16.ProvingKey(32 + 1, K, trap, ctx)
        try:
            with pytest.raises(ValueError):
                pk.prove_block(wire.FlatBlock(fb.payloads, fb.offs, fb.atts,
                                              np.frombuffer(fb.header, np.uint8).copy()), wit)
        finally:
            pk.close()


@pytest.mark.parametrize("world", [1, 2, 3])
def test_one_proof_split_keys_match_whole_key(ctx, world):
    """One proof per block across ranks (DIZK-style MSM split), the ranks
    emulated one after another: each split key holds its slice of the bases
    (same trapdoor), each rank's partial points summed in rank order give the
    whole key's proof and FC; world = 1 through the same partial/finish calls
    with a whole key gives prove_block's bytes. A split key refuses the
    whole-proof entry points."""
    import torch
    from paper_2603_10242_b200 import groth16, prover, shard, wire
    T, K, n = 45, 5, 37
    rng = random.Random(world)
    trap = arr([rng.randrange(1, R) for _ in range(5)])
    fb = O.multi_user_block(n, 3)
    wfb = wire.FlatBlock(fb.payloads, fb.offs, fb.atts, np.frombuffer(fb.header, np.uint8).copy())
    wit = _witnesses(fb, n)
    whole = groth16.ProvingKey(T, K, trap, ctx)
    try:
        _, p_ref, fc_ref, cps = whole.prove_block(wfb, wit)
        revs = np.frombuffer(fb.revs, np.uint8).copy()
        rix = np.asarray(fb.rev_index, np.uint32)
        db = shard.DeviceBlock.upload(wfb, 0, n, revs, rix, device=0)
        db.witnesses = torch.from_numpy(wit).cuda()
        if world == 1:
            p, f = shard.prove_one_proof(db, n, 0, 1, whole)
            assert p.cpu().numpy().tobytes() == p_ref and f.cpu().numpy().tobytes() == fc_ref
            return
        keys = [groth16.ProvingKey(T, K, trap, ctx, rank=r, world=world) for r in range(world)]
        try:
            parts, merks = [], []
            for k in keys:
                codes = torch.full((n,), 0xEE, dtype=torch.uint8, device="cuda:0")
                part, merk = shard.one_proof_partial(db, k, codes)
                assert int((codes != 0).sum().item()) == 0
                parts.append(part)
                merks.append(merk)
            allp = torch.cat(parts)
            for k, merk in zip(keys, merks):
                p, f = shard.one_proof_finish(allp, world, merk, n, db.header, k)
                assert p.cpu().numpy().tobytes() == p_ref and f.cpu().numpy().tobytes() == fc_ref
            assert whole.verify_finality_certificate(fc_ref, wfb, cps) == prover.FcCheck.Valid
            with pytest.raises(ValueError):
                keys[0].prove_block(wfb, wit)
        finally:
            for k in keys:
                k.close()
    finally:
        whole.close()


@pytest.mark.parametrize("world,shares", [(2, None), (3, None), (5, None), (3, [1, 5, 2]),
                                          (4, "balanced")])
def test_one_proof_owner_split_matches_whole_key(ctx, world, shares):
    """The owner split of the H polynomial (phase 1: each rank transforms the
    vectors it owns, k mod world; the slices exchanged; phase 2: (a b - c)/Z
    and [h] on the rank's slice), ranks emulated one after another with the
    exchange done here: the summed partials give the whole key's proof and
    FC (world = 5: ranks 3, 4 own no vector; weighted shares: uneven slices
    of every base array and of H)."""
    import torch
    from paper_2603_10242_b200 import groth16, shard, wire
    T, K, n = 45, 5, 37
    rng = random.Random(10 + world)
    trap = arr([rng.randrange(1, R) for _ in range(5)])
    fb = O.multi_user_block(n, 3)
    wfb = wire.FlatBlock(fb.payloads, fb.offs, fb.atts, np.frombuffer(fb.header, np.uint8).copy())
    wit = _witnesses(fb, n)
    whole = groth16.ProvingKey(T, K, trap, ctx)
    try:
        _, p_ref, fc_ref, _ = whole.prove_block(wfb, wit)
    finally:
        whole.close()
    db = shard.DeviceBlock.upload(wfb, 0, n, np.frombuffer(fb.revs, np.uint8).copy(),
                                  np.asarray(fb.rev_index, np.uint32), device=0)
    db.witnesses = torch.from_numpy(wit).cuda()
    if shares == "balanced":
        shares = shard.balanced_shares(world)
    keys = [groth16.ProvingKey(T, K, trap, ctx, rank=r, world=world, shares=shares)
            for r in range(world)]
    try:
        N = keys[0].domain
        owns, merks = [], []
        for r, k in enumerate(keys):
            own, merk = shard.one_proof_phase1(db, k, r, world)
            owns.append(own)
            merks.append(merk)
        vec = {}
        for r in range(world):
            idx = 0
            for v in range(3):
                if v % world == r:
                    vec[v] = owns[r][32 * N * idx:32 * N * (idx + 1)]
                    idx += 1
        parts = []
        for r, k in enumerate(keys):
            lo, hi = shard.slice_bounds(N, r, world, shares)
            sl = torch.cat([vec[v][32 * lo:32 * hi] for v in range(3)]).contiguous()
            parts.append(shard.one_proof_phase2(sl, k))
        allp = torch.cat(parts)
        for k, merk in zip(keys, merks):
            p, f = shard.one_proof_finish(allp, world, merk, n, db.header, k)
            assert p.cpu().numpy().tobytes() == p_ref and f.cpu().numpy().tobytes() == fc_ref
    finally:
        for k in keys:
            k.close()


def test_one_proof_entry_points_reject_bad_arguments(ctx):
    """The split-key / one-proof entry points fail loudly (EINVAL ->
    ValueError): rank >= world, empty shares, a block larger than the key,
    an owned mask beyond a|b|c, a whole-proof call on a split key."""
    import torch
    from paper_2603_10242_b200 import _native as N, groth16, shard, wire
    trap = arr([3, 5, 7, 11, 13])
    h = C.c_void_p()
    with pytest.raises(ValueError):
        ctx.call("acegpu_g16_setup_slice", 8, 3, trap, 2, 2, None, C.byref(h))
    with pytest.raises(ValueError):
        ctx.call("acegpu_g16_setup_slice", 8, 3, trap, 0, 2, np.zeros(2, np.uint32), C.byref(h))
    pk = groth16.ProvingKey(8, 3, trap, ctx, rank=0, world=2)
    try:
        fb = O.multi_user_block(11, 2)  # 11 txs > T = 8
        wfb = wire.FlatBlock(fb.payloads, fb.offs, fb.atts, np.frombuffer(fb.header, np.uint8).copy())
        db = shard.DeviceBlock.upload(wfb, 0, 11, device=0)
        db.witnesses = torch.zeros(11 * 256, dtype=torch.uint8, device="cuda:0")
        with pytest.raises(ValueError):
            shard.one_proof_partial(db, pk)
        w = torch.zeros(8 * 32, dtype=torch.uint8, device="cuda:0")
        own = torch.zeros(3 * 32 * pk.domain, dtype=torch.uint8, device="cuda:0")
        with pytest.raises(ValueError):
            ctx.call("acegpu_g16_prove_phase1_dev", None, pk.h, w.data_ptr(), w.data_ptr(), 9,
                     own.data_ptr())
        with pytest.raises(ValueError):  # a split key has no whole-proof path
            pk.prove(arr([1] * 8), arr([2] * 8))
        parts = torch.zeros(2 * 384, dtype=torch.uint8, device="cuda:0")
        with pytest.raises(ValueError):  # finish before this key's partial
            ctx.call("acegpu_g16_finish_dev", None, pk.h, parts.data_ptr(), 2, None, None, None,
                     None)
        with pytest.raises(ValueError):  # phase 2 before phase 1
            ctx.call("acegpu_g16_prove_phase2_dev", None, pk.h, own.data_ptr(),
                     parts.data_ptr())
    finally:
        pk.close()


def test_variable_base_key_block_equals_fixed_key_block(ctx, monkeypatch):
    """A multi-chunk Groth16 block through a variable-base key (one buffer
    slot: the chunks serialise) gives the same chunk proofs and FC as the
    fixed-base key (two slots, chunk k+1's witness under chunk k's MSMs)."""
    from paper_2603_10242_b200 import groth16, wire
    T, K, n = 4, 3, 23
    trap = arr([5, 7, 11, 13, 17])
    fb = O.multi_user_block(n, 3)
    wfb = wire.FlatBlock(fb.payloads, fb.offs, fb.atts, np.frombuffer(fb.header, np.uint8).copy())
    wit = _witnesses(fb, n)
    out = []
    for vb in ("0", "1"):
        monkeypatch.setenv("ACEGPU_G16_VB", vb)
        pk = groth16.ProvingKey(T, K, trap, ctx)
        try:
            out.append(pk.prove_block(wfb, wit)[1:])
        finally:
            pk.close()
    assert out[0] == out[1]


def test_one_proof_for_the_100k_block_verifies(ctx):
    """BASELINE configs[3] in one-proof mode at full size: the canonical 100k
    block (the reference's acceptance generator) proven as ONE Groth16 proof
    (140.1 M constraints, 3 x 2^26 domain, ~100 GB of key and vectors in
    HBM), the FC carrying it; verify_finality_certificate accepts it with the
    one 256-B proof and rejects a flipped proof byte."""
    import bench
    from paper_2603_10242_b200 import groth16, prover, wire
    n = 100_000
    fb, revs, rix = bench.canonical_block_host(n, ctx)
    wit = bench.make_witnesses(fb, revs, rix, ctx)
    wfb = wire.FlatBlock(fb.payloads, fb.offs, fb.atts, np.frombuffer(bytes(fb.header), np.uint8).copy())
    pk = groth16.ProvingKey(n, groth16.PAPER_K, ctx=ctx)
    try:
        assert pk.constraints == 140_100_001 and pk.domain == 3 << 26
        codes, proof, fc, cps = pk.prove_block(wfb, wit, revs, rix)
        assert (codes == 0).all() and len(cps) == 256 and proof[:256] == cps
        assert pk.verify_finality_certificate(fc, wfb, cps) == prover.FcCheck.Valid
        bad = bytearray(cps)
        bad[200] ^= 1
        assert pk.verify_finality_certificate(fc, wfb, bytes(bad)) == prover.FcCheck.ProofMismatch
    finally:
        pk.close()
