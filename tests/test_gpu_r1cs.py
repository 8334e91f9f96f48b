"""General R1CS path (north-star witness / constraint evaluation, csrc/r1cs.cu):
CSR SpMV row evaluations vs Python big integers; the stand-in circuit run
through the general path gives the bespoke prover's verifying key and proof
bytes; a non-synthetic circuit proves, verifies (GPU batch verifier and the
oracle's pairing verifier) and binds its public inputs."""
import ctypes as C
import random

import numpy as np
import pytest

import g16_spec as SP
import oracle_lib as O

pytestmark = pytest.mark.gpu

R = 0x30644E72E131A029B85045B68181585D2833E84879B9709143E1F593F0000001


def le(x):
    return (x % R).to_bytes(32, "little")


def arr(vals):
    return np.frombuffer(b"".join(le(v) for v in vals), np.uint8).copy()


def ints(a):
    b = a.tobytes()
    return [int.from_bytes(b[i:i + 32], "little") for i in range(0, len(b), 32)]


@pytest.fixture(scope="module")
def ctx():
    from paper_2603_10242_b200 import _native as N
    return N.context(0)


def test_r1cs_eval_matches_python(ctx):
    from paper_2603_10242_b200 import r1cs
    rng = random.Random(1)
    m, V, npub = 200, 60, 4
    mats = []
    for _ in range(3):
        rows = []
        for _ in range(m):
            rows.append({rng.randrange(V): rng.choice([1, 2, R - 1, rng.randrange(R), 2**256 - 1])
                         for _ in range(rng.randrange(0, 5))})
        mats.append(rows)
    z = [1] + [rng.randrange(R) for _ in range(V - 1)]
    r = r1cs.R1CS(m, V, npub, *[r1cs.Csr.from_rows(x) for x in mats], ctx=ctx)
    try:
        a, b, c = r.eval(arr(z))
        for k, (got, rows) in enumerate(zip((a, b, c), mats)):
            exp = [sum(v * z[i] for i, v in row.items()) % R for row in rows]
            # appended public rows: A_{m+i} = z_i, B = C = 0
            exp += [z[i] if k == 0 else 0 for i in range(npub + 1)]
            assert ints(got) == exp
    finally:
        r.close()


def test_r1cs_rejects_malformed(ctx):
    from paper_2603_10242_b200 import r1cs
    good = r1cs.Csr.from_rows([{0: 1}, {1: 1}])
    bad_col = r1cs.Csr.from_rows([{0: 1}, {7: 1}])
    with pytest.raises(ValueError):
        r1cs.R1CS(2, 5, 1, good, good, bad_col, ctx=ctx)
    with pytest.raises(ValueError):
        r1cs.R1CS(2, 5, 4, good, good, good, ctx=ctx)  # n_pub + 1 >= vars


@pytest.mark.parametrize("T,K", [(4, 3), (64, 20)])
def test_synthetic_circuit_through_the_general_path(ctx, T, K):
    """The stand-in circuit as CSR matrices: same verifying key, same proof
    bytes and digest as the bespoke chunk prover."""
    from paper_2603_10242_b200 import groth16, r1cs
    rng = random.Random(T * 7 + K)
    trap = arr([rng.randrange(1, R) for _ in range(5)])
    m, V, npub, A, B, Cm = r1cs.synthetic_chunk(T, K, ctx)
    rc = r1cs.R1CS(m, V, npub, A, B, Cm, ctx=ctx)
    pk1 = groth16.ProvingKey(T, K, trap, ctx)
    pk2 = groth16.ProvingKey.from_r1cs(rc, trap, ctx)
    try:
        assert (pk2.variables, pk2.constraints, pk2.log_domain) == \
               (pk1.variables, pk1.constraints, pk1.log_domain)
        assert pk2.verifying_key() == pk1.verifying_key()
        w = arr([rng.randrange(R) for _ in range(T)])
        pub = arr([rng.randrange(R) for _ in range(T)])
        z = r1cs.synthetic_assignment(T, K, w, pub, r1cs.chain_constants(K, ctx))
        a, b, c = rc.eval(z)
        assert all(x * y % R == v for x, y, v in zip(ints(a), ints(b), ints(c)))  # satisfied
        rs = arr(SP.derive_rs(w.tobytes(), pub.tobytes(), T))
        p1, raw1, d1 = pk1.prove(w, pub, rs)
        p2, raw2, d2 = pk2.prove_z(z, rs)
        assert p2 == p1 and raw2 == raw1 and d2 == d1
        # derived r, s of the general path: D(private assignment) | D(public inputs)
        p3, raw3, d3 = pk2.prove_z(z)
        zb = z.tobytes()
        wd = SP.input_digest(zb[32 * (1 + T):], V - 1 - T, True)
        pd = SP.input_digest(zb[32:32 * (1 + T)], T)
        r_ = int.from_bytes(SP.sha(b"ace-g16-r-v2" + wd + pd), "little") % R
        s_ = int.from_bytes(SP.sha(b"ace-g16-s-v2" + wd + pd), "little") % R
        assert pk2.prove_z(z, arr([r_, s_]))[0] == p3 and d3 == d1
        with pytest.raises(ValueError):
            pk1.prove_z(z)  # a synthetic key takes (w, pub), not an assignment
    finally:
        pk1.close()
        pk2.close()
        rc.close()


def _cubic_circuit(n_inst, rng):
    """n_inst instances of x^3 + a x + 5 = y (y public), 3 rows each:
    s1 = x * x, s2 = s1 * x, (s2 + a x + 5) * 1 = y. Not the stand-in chain."""
    npub = n_inst
    V = 1 + npub + 3 * n_inst  # ONE, y_i, then x_i, s1_i, s2_i
    A, B, Cm, z = [], [], [], [1] + [0] * (V - 1)
    for i in range(n_inst):
        y, x, s1, s2 = 1 + i, 1 + npub + 3 * i, 2 + npub + 3 * i, 3 + npub + 3 * i
        a = rng.randrange(R)
        xv = rng.randrange(R)
        z[x], z[s1] = xv, xv * xv % R
        z[s2] = z[s1] * xv % R
        z[y] = (z[s2] + a * xv + 5) % R
        A += [{x: 1}, {s1: 1}, {s2: 1, x: a, 0: 5}]
        B += [{x: 1}, {x: 1}, {0: 1}]
        Cm += [{s1: 1}, {s2: 1}, {y: 1}]
    return 3 * n_inst, V, npub, A, B, Cm, z


def test_general_circuit_proves_and_verifies(ctx):
    from paper_2603_10242_b200 import groth16, r1cs
    rng = random.Random(42)
    m, V, npub, A, B, Cm, z = _cubic_circuit(6, rng)
    rc = r1cs.R1CS(m, V, npub, *[r1cs.Csr.from_rows(x) for x in (A, B, Cm)], ctx=ctx)
    trap = arr([rng.randrange(1, R) for _ in range(5)])
    pk = groth16.ProvingKey.from_r1cs(rc, trap, ctx)
    try:
        za = arr(z)
        proof, raw, dig = pk.prove_z(za)
        pubs = za.tobytes()[32:32 * (1 + npub)]
        assert dig == SP.chunk_digest(pubs, npub)
        assert pk.verify_batch([proof], [pubs])
        vk = pk.verifying_key()
        assert O.oracle().bn_g16_verify(C.c_uint32(npub), O.ptr(vk), O.ptr(raw), O.ptr(pubs)) == 1
        bad = bytearray(pubs)
        bad[0] ^= 1
        assert not pk.verify_batch([proof], [bytes(bad)])
        assert O.oracle().bn_g16_verify(C.c_uint32(npub), O.ptr(vk), O.ptr(raw), O.ptr(bytes(bad))) == 0
        # an unsatisfying assignment does not verify
        z2 = list(z)
        z2[1 + npub] = (z2[1 + npub] + 1) % R
        p2, _, _ = pk.prove_z(arr(z2))
        assert not pk.verify_batch([p2], [pubs])
    finally:
        pk.close()
        rc.close()


def test_paper_size_chunk_through_the_general_path(ctx):
    """1,024 txs x 1,400 constraints (1,434,625 rows, domain 2^21) as CSR:
    proof bytes equal the bespoke prover's."""
    from paper_2603_10242_b200 import bn254, groth16, r1cs
    T, K = groth16.PAPER_T, groth16.PAPER_K
    m, V, npub, A, B, Cm = r1cs.synthetic_chunk(T, K, ctx)
    rc = r1cs.R1CS(m, V, npub, A, B, Cm, ctx=ctx)
    w, pub = bn254.random_scalars(T, 5), bn254.random_scalars(T, 6)
    z = r1cs.synthetic_assignment(T, K, w, pub, r1cs.chain_constants(K, ctx))
    trap = groth16.deterministic_trapdoor(ctx=ctx)
    rs = arr(SP.derive_rs(w.tobytes(), pub.tobytes(), T))
    pk1 = groth16.ProvingKey(T, K, trap, ctx)
    try:
        p1 = pk1.prove(w, pub, rs)
    finally:
        pk1.close()
    pk2 = groth16.ProvingKey.from_r1cs(rc, trap, ctx)
    try:
        assert pk2.prove_z(z, rs) == p1
    finally:
        pk2.close()
        rc.close()


def test_zkace_hmac_circuit_proves_on_gpu(ctx):
    """The ZK-ACE credential relation (zkace_circuit.py: HMAC-SHA256(attest key,
    obj_hash || domain) == credential, ~103k constraints per tx) for 2 txs of a
    multi-user block: satisfied on the GPU (A z o B z == C z), proven and
    verified by the GPU batch verifier and the oracle's pairing check; a
    forged credential makes the system unsatisfiable and its proof fails."""
    from paper_2603_10242_b200 import groth16, r1cs, zkace_circuit as Z
    fb = O.multi_user_block(2, 2)
    keys, atts = [], []
    for i in range(2):
        att = fb.att(i)
        u = int(fb.rev_index[i])
        keys.append(bytes(O.derive_attest_key(fb.revs[32 * u:32 * u + 32].tobytes(), att[64:72])))
        atts.append(bytes(att))
    m, V, npub, A, B, Cm, z = Z.chunk(keys, atts)
    rc = r1cs.R1CS(m, V, npub, A, B, Cm, ctx=ctx)
    rng = random.Random(9)
    pk = groth16.ProvingKey.from_r1cs(rc, arr([rng.randrange(1, R) for _ in range(5)]), ctx)
    try:
        a, b, c = rc.eval(z)
        assert all(x * y % R == v for x, y, v in zip(ints(a), ints(b), ints(c)))
        proof, raw, _ = pk.prove_z(z)
        pubs = z.tobytes()[32:32 * (1 + npub)]
        assert pk.verify_batch([proof], [pubs])
        vk = pk.verifying_key()
        assert O.oracle().bn_g16_verify(C.c_uint32(npub), O.ptr(vk), O.ptr(raw), O.ptr(pubs)) == 1
        bad = list(atts)
        bad[1] = bad[1][:80] + bytes([bad[1][80] ^ 4]) + bad[1][81:]
        _, _, _, _, _, _, zf = Z.chunk(keys, bad)
        a, b, c = rc.eval(zf)
        assert any(x * y % R != v for x, y, v in zip(ints(a), ints(b), ints(c)))
        pf, _, _ = pk.prove_z(zf)
        assert not pk.verify_batch([pf], [zf.tobytes()[32:32 * (1 + npub)]])
    finally:
        pk.close()
        rc.close()


def test_zkace_gpu_witness_program(ctx):
    """GPU witness generation (csrc/witprog.cu): the circuit compiled to a
    straight-line program and run per tx on the device gives exactly the
    host builder's assignment — honest and forged transactions — and the
    chunk proves and verifies from the GPU-made assignment."""
    from paper_2603_10242_b200 import groth16, r1cs, zkace_circuit as Z
    fb = O.multi_user_block(3, 2)
    keys, atts = [], []
    for i in range(3):
        att = fb.att(i)
        u = int(fb.rev_index[i])
        keys.append(bytes(O.derive_attest_key(fb.revs[32 * u:32 * u + 32].tobytes(), att[64:72])))
        atts.append(bytes(att))
    atts[2] = atts[2][:90] + bytes([atts[2][90] ^ 1]) + atts[2][91:]  # tx 2 forged
    prog = Z.WitnessProgram(ctx)
    try:
        _, _, _, _, _, _, z_host = Z.chunk(keys, atts)
        z_gpu = prog.run(keys, atts)
        assert z_gpu.tobytes() == z_host.tobytes()
        m, V, npub, A, B, Cm = Z.chunk_r1cs(2)
        rc = r1cs.R1CS(m, V, npub, A, B, Cm, ctx=ctx)
        pk = groth16.ProvingKey.from_r1cs(rc, arr([3, 5, 7, 11, 13]), ctx)
        try:
            z2 = prog.run(keys[:2], atts[:2])
            proof, _, _ = pk.prove_z(z2)
            assert pk.verify_batch([proof], [z2.tobytes()[32:32 * (1 + npub)]])
        finally:
            pk.close()
            rc.close()
    finally:
        prog.close()


@pytest.mark.parametrize("n", [16, 37])
def test_zkace_block_prover(ctx, n):
    """The block path over the REAL credential relation (zkace.py): 16-tx
    chunks, GPU witness generation, one Groth16 proof per chunk, the
    reference's tree over the chunk proofs and the FC. The FC equals the
    oracle's tree / FC over nodes (chunk proof | chunk digest | Tx) built from
    the chunk proofs; the chunk proofs verify against the public inputs
    recomputed from the block; a forged credential fails verification."""
    from paper_2603_10242_b200 import shard, wire, zkace
    fb = O.multi_user_block(n, 3)
    wit = b""
    for i in range(n):
        att = fb.att(i)
        u = int(fb.rev_index[i])
        key = O.derive_attest_key(fb.revs[32 * u:32 * u + 32].tobytes(), att[64:72])
        out = O.buf(256)
        O.oracle().or_build_witness(O.ptr(key), O.ptr(att[:32]), out)
        wit += bytes(out)
    zp = zkace.ZkAceProver(16, arr([3, 5, 7, 11, 13]), ctx)
    try:
        for forged in (False, True):
            atts = fb.atts.copy()
            if forged:
                atts[104 * (n - 1) + 80] ^= 2
            wfb = wire.FlatBlock(fb.payloads, fb.offs, atts, np.frombuffer(fb.header, np.uint8).copy())
            db = shard.DeviceBlock.upload(wfb, 0, n, np.frombuffer(fb.revs, np.uint8).copy(),
                                          np.asarray(fb.rev_index, np.uint32), device=0)
            import torch
            db.witnesses = torch.from_numpy(np.frombuffer(wit, np.uint8).copy()).cuda()
            codes = torch.full((n,), 0xEE, dtype=torch.uint8, device="cuda")
            proof, fc, cps = zp.prove_block(db, n, codes=codes, return_chunk_proofs=True)
            proofs = [bytes(x) for x in cps.cpu().numpy()]
            pubs = zp.public_inputs(atts, n)
            ok = zp.verify_chunk_proofs(proofs, atts, n)
            assert ok == (not forged)
            assert int((codes.cpu().numpy() != 0).sum()) == (1 if forged else 0)
            nodes = b"".join(p + SP.chunk_digest(q, 16 * 5) + b"\0" for p, q in zip(proofs, pubs))
            outp = O.buf(289)
            lv, pr = C.c_uint64(), C.c_uint64()
            O.oracle().or_aggregate_tree(O.ptr(nodes), C.c_uint64(len(proofs)), outp,
                                         C.byref(lv), C.byref(pr))
            assert proof.cpu().numpy().tobytes() == bytes(outp)
            ofb = O.FlatBlock(fb.payloads, fb.offs, atts, fb.header, fb.revs, fb.rev_index)
            assert fc.cpu().numpy().tobytes() == O.oracle_build_fc(ofb, bytes(outp))
    finally:
        zp.close()
