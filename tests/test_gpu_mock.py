"""Parity of the CUDA mock-Prove path against the oracle, the reference
(oracle/_ref, when present) and the reference-derived goldens.

Mirrors the reference's own hot-path tests: test_prover.cpp, test_crypto.cpp
(attestation rows), test_sha256.cpp, test_wire.cpp (Merkle / FC), acceptance
criteria 1 and 8. Everything here calls through the C ABI (libacegpu.so).
"""
import ctypes as C
import random

import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    from paper_2603_10242_b200 import _native as N, crypto, prover, wire
    ctx = N.context(0)
    return type("P", (), {"N": N, "ctx": ctx, "prover": prover, "wire": wire, "crypto": crypto})


def gpu_block(P, fb: O.FlatBlock, codes=True):
    """Run the fused attest+prove+certify C-ABI call on an oracle FlatBlock."""
    N = P.N
    proof = np.zeros(289, np.uint8)
    fc = np.zeros(328, np.uint8)
    cd = np.zeros(max(fb.n, 1), np.uint8)
    lv, pr = C.c_uint64(), C.c_uint64()
    hdr = np.frombuffer(fb.header, np.uint8).copy()
    P.ctx.call("acegpu_attest_prove_certify", N.addr(fb.payloads), N.addr(fb.offs),
               N.addr(fb.atts), fb.n, N.addr(hdr), N.addr(fb.revs) if codes else None,
               len(fb.revs) // 32 if codes else 0, N.addr(fb.rev_index) if codes else None,
               N.addr(cd) if codes else None, N.addr(proof), N.addr(fc), C.byref(lv),
               C.byref(pr))
    return proof.tobytes(), fc.tobytes(), cd[:fb.n], lv.value, pr.value


def to_wire_flat(P, fb: O.FlatBlock):
    return P.wire.FlatBlock(fb.payloads, fb.offs, fb.atts, np.frombuffer(fb.header, np.uint8).copy())


# ------------------------------------------------------------------ SHA-256
def test_sha256_varlen_matches_oracle(P):
    rng = random.Random(5)
    msgs = [bytes(rng.getrandbits(8) for _ in range(rng.randrange(0, 700))) for _ in range(300)]
    msgs += [b"", b"abc", bytes(range(65)), b"\0" * 55, b"\0" * 56, b"\0" * 63, b"\0" * 64]
    got = P.wire.sha256_many(msgs, P.ctx)
    assert got == [O.sha256(m) for m in msgs]


@pytest.mark.parametrize("length", [1, 32, 33, 36, 64, 65, 154, 244])
@pytest.mark.parametrize("count", [1, 7, 8, 9, 16, 33])
def test_sha256_strided_matches_oracle(P, length, count):
    """test_sha256.cpp:75-97 (the AVX2 batch kernel's cross-check)."""
    rng = np.random.default_rng(length * 100 + count)
    data = rng.integers(0, 256, length * count + 16, dtype=np.uint8)
    out = np.zeros(32 * count, np.uint8)
    P.ctx.call("acegpu_sha256_strided", P.N.addr(data), length, length, count, P.N.addr(out))
    for i in range(count):
        assert out[32 * i:32 * i + 32].tobytes() == O.sha256(data[i * length:(i + 1) * length].tobytes())


def test_sha256_peak_positive(P):
    v = C.c_double()
    P.ctx.call("acegpu_sha256_peak", C.byref(v))
    assert v.value > 1e9


# ---------------------------------------------------------- whole blocks
@pytest.mark.parametrize("n", [0, 1, 2, 3, 5, 7, 100, 1024, 1025, 4097, 16384, 100000])
def test_canonical_block_matches_reference_goldens(P, kats, n):
    k = kats["canonical_blocks"][str(n)]
    fb = O.canonical_block(n)
    proof, fc, codes, lv, pr = gpu_block(P, fb)
    assert fc.hex() == k["fc"]
    assert proof[256:288].hex() == k["root_digest"] and proof[288] == k["root_kind"]
    assert O.sha256(proof[:256]).hex() == k["root_proof_sha"]
    assert (lv, pr) == (k["levels"], k["pairs"])
    assert int((codes == 0).sum()) == k["accept"]


@pytest.mark.parametrize("n", [64, 1024])
def test_forged_attestation_codes(P, kats, n):
    fb = O.forge(O.canonical_block(n))
    _, _, codes, _, _ = gpu_block(P, fb)
    assert bytes(codes).hex() == kats["forged"][str(n)]["codes"]
    assert (codes == O.oracle_attest_codes(fb)).all()


def test_multi_user_block(P, kats):
    fb = O.multi_user_block(1000, 16)
    _, fc, codes, _, _ = gpu_block(P, fb)
    assert fc.hex() == kats["multi_user_1000"]["fc"]
    assert (codes == 0).all()


def test_prover_test_blocks(P, kats):
    for n, fc_hex in kats["prover_test_blocks"].items():
        _, fc, _, _, _ = gpu_block(P, O.prover_test_block(int(n)), codes=False)
        assert fc.hex() == fc_hex


def test_random_blocks_vs_oracle_and_reference(P):
    """Random payload lengths (0..3000 B: staged and unstaged payload paths),
    random headers, domains, ids, REVs and forged credentials."""
    rng = random.Random(77)
    for trial in range(25):
        n = rng.choice([1, 2, 3, 31, 127, 128, 129, 300, 1000])
        big = trial % 3 == 0
        payloads, atts, revs = [], [], []
        for i in range(n):
            rev = bytes(rng.getrandbits(8) for _ in range(32))
            ln = rng.randrange(0, 3000 if big else 300)
            p = bytes(rng.getrandbits(8) for _ in range(ln))
            dom = O.domain_encode(rng.randrange(65536), rng.randrange(1 << 48))
            a = O.generate_attestation(rev, p, dom, bytes(rng.getrandbits(8) for _ in range(32)))
            if rng.random() < 0.25:
                a = a[:72] + bytes(32)
            if rng.random() < 0.1:
                a = bytes(32) + a[32:]
            payloads.append(p)
            atts.append(a)
            revs.append(rev)
        hdr = bytes(rng.getrandbits(8) for _ in range(212)) + b"\0" * 44
        fb = O.flat_from_lists(payloads, atts, hdr, revs, list(range(n)))
        proof, fc, codes, lv, pr = gpu_block(P, fb)
        oproof, olv, opr = O.oracle_prove_block(fb)
        assert proof == oproof and (lv, pr) == (olv, opr)
        assert fc == O.oracle_build_fc(fb, oproof)
        assert (codes == O.oracle_attest_codes(fb)).all()
        if O.ref_available() and trial < 8:
            assert fc == O.ref_prove_and_certify(fb)
            assert (codes == O.ref_attest_codes(fb)).all()


# ------------------------------------------------------ prover.hpp surface
def test_mock_proofs_deterministic_and_verifiable(P):
    """test_prover.cpp:45-62."""
    pr = P.prover
    blk = to_wire_flat(P, O.prover_test_block(1)).to_block()
    tx = blk.transactions[0]
    p1, p2 = pr.prove_tx(tx, P.ctx), pr.prove_tx(tx, P.ctx)
    assert p1 == p2 and pr.verify_mock(p1, P.ctx)
    ob = O.buf(289)
    O.oracle().or_prove_tx(O.ptr(tx.payload), C.c_uint64(len(tx.payload)),
                           O.ptr(tx.attestation.encode()), ob)
    assert p1.to_bytes() == bytes(ob)
    bad = pr.MockProof(bytearray(p1.bytes), p1.public_inputs_digest, p1.kind)
    bad.bytes[5] ^= 1
    bad.bytes = bytes(bad.bytes)
    assert not pr.verify_mock(bad, P.ctx)
    agg = pr.aggregate_pair(p1, p2, P.ctx)
    assert agg.kind == pr.ProofKind.Aggregate and pr.verify_mock(agg, P.ctx)
    tx2 = P.wire.Transaction(tx.payload, P.wire.Attestation(
        tx.attestation.obj_hash, tx.attestation.id_com,
        P.wire.Domain(tx.attestation.domain.chain_id, tx.attestation.domain.slot + 1),
        tx.attestation.credential))
    assert pr.prove_tx(tx2, P.ctx).bytes != p1.bytes


def test_aggregate_tree_structure(P):
    """test_prover.cpp:64-104 and acceptance criterion 8 (levels for 1..4096)."""
    pr = P.prover
    blk = to_wire_flat(P, O.prover_test_block(5)).to_block()
    proofs = [pr.prove_tx(t, P.ctx) for t in blk.transactions]
    st = pr.AggregationStats()
    assert pr.aggregate_tree(proofs[:1], st, P.ctx) == proofs[0] and st.levels == 0
    pr.aggregate_tree(proofs[:4], st, P.ctx)
    assert st.levels == 2
    base = pr.aggregate_tree(proofs, st, P.ctx)
    assert st.levels == 3
    with pytest.raises(ValueError):
        pr.aggregate_tree([], None, P.ctx)
    sw = [proofs[0], proofs[2], proofs[1], proofs[3], proofs[4]]
    assert pr.aggregate_tree(sw, None, P.ctx).bytes != base.bytes
    out = O.buf(289)
    lv, pp = C.c_uint64(), C.c_uint64()
    arr = b"".join(p.to_bytes() for p in proofs)
    O.oracle().or_aggregate_tree(O.ptr(arr), C.c_uint64(5), out, C.byref(lv), C.byref(pp))
    assert base.to_bytes() == bytes(out)
    for n in (1, 2, 3, 4, 5, 7, 8, 9, 64, 100, 1024, 4095, 4096):
        pr.aggregate_tree([proofs[0]] * n, st, P.ctx)
        assert st.levels == (n - 1).bit_length() and st.pair_ops == n - 1


def test_finality_certificate_checks(P):
    """test_prover.cpp:106-148."""
    pr, wire = P.prover, P.wire
    fb = O.prover_test_block(7)
    block = to_wire_flat(P, fb).to_block()
    root = pr.prove_block(block, None, P.ctx)
    fc = pr.build_finality_certificate(block, root, P.ctx)
    assert len(fc.encode()) == 328
    assert fc.block_hash == wire.block_hash(block, P.ctx) == O.sha256(fb.header)
    cost = pr.CostUnits()
    assert pr.verify_finality_certificate(fc, block, cost, P.ctx) == pr.FcCheck.Valid
    assert cost.value == 1
    other = to_wire_flat(P, O.prover_test_block(7, slot=10)).to_block()
    assert pr.verify_finality_certificate(fc, other, None, P.ctx) == pr.FcCheck.SlotMismatch
    other = to_wire_flat(P, fb).to_block()
    other.header.parent_hash = b"\x01" + other.header.parent_hash[1:]
    assert pr.verify_finality_certificate(fc, other, None, P.ctx) == pr.FcCheck.HashMismatch
    bad = wire.FinalityCertificate.decode(fc.encode())
    bad.proof = bad.proof[:100] + bytes([bad.proof[100] ^ 1]) + bad.proof[101:]
    assert pr.verify_finality_certificate(bad, block, None, P.ctx) == pr.FcCheck.ProofMismatch
    other = to_wire_flat(P, fb).to_block()
    a = other.transactions[3].attestation
    other.transactions[3].attestation = wire.Attestation(a.obj_hash, bytes([a.id_com[0] ^ 1]) + a.id_com[1:],
                                                         a.domain, a.credential)
    exp = pr.build_finality_certificate(other, pr.prove_block(other, None, P.ctx), P.ctx)
    assert exp.public_inputs_commitment != fc.public_inputs_commitment
    assert fc.encode() == O.oracle_build_fc(fb, root.to_bytes())


def test_aggregation_soundness_1000_mutations(P):
    """test_prover.cpp:150-174: any mutation changes the root."""
    rng = random.Random(99)
    fb = O.prover_test_block(16)
    base, _, _, _, _ = gpu_block(P, fb, codes=False)
    for _ in range(1000):
        m = fb.copy()
        tx = rng.randrange(16)
        kind = rng.randrange(3)
        if kind == 0:
            m.payloads[int(m.offs[tx]) + rng.randrange(154)] ^= 1 + rng.randrange(255)
        elif kind == 1:
            m.atts[104 * tx + 32 + rng.randrange(32)] ^= 1 + rng.randrange(255)
        else:
            other = rng.randrange(16)
            if other == tx:
                other = (tx + 1) % 16
            a, b = sorted((tx, other))
            pa, pb = m.payload(a), m.payload(b)
            aa, ab = m.att(a), m.att(b)
            pls = [m.payload(i) for i in range(16)]
            ats = [m.att(i) for i in range(16)]
            pls[a], pls[b], ats[a], ats[b] = pb, pa, ab, aa
            m = O.flat_from_lists(pls, ats, m.header)
        proof, _, _, _, _ = gpu_block(P, m, codes=False)
        assert proof[:256] != base[:256]


def test_merkle_root_cases(P):
    """test_wire.cpp:79-105."""
    rng = random.Random(4242)
    for n in list(range(0, 40)) + [101, 257, 1000]:
        leaves = [bytes(rng.getrandbits(8) for _ in range(32)) for _ in range(n)]
        assert P.wire.merkle_root(leaves, P.ctx) == O.merkle_root(leaves)
    a, b, c = (bytes([i]) * 32 for i in (1, 2, 3))
    assert P.wire.merkle_root([a, b, c], P.ctx) == P.wire.merkle_root([a, b, c, c], P.ctx)


def test_empty_block_and_wire_goldens(P, kats):
    """Reference golden wire files (test_wire.cpp:265-319) by hash."""
    import hashlib
    wire = P.wire
    g = kats["reference_golden_files"]
    b = wire.Block()
    b.header.slot_number = 7
    b.header.parent_hash = b"\x11" * 32
    b.header.state_root = b"\x22" * 32
    b.header.poh_hash = b"\x33" * 32
    b.header.leader_id_com = b"\x44" * 32
    b.header.timestamp_ms = 2800
    for i in range(3):
        p = wire.make_transfer_payload(b"\x01" * 32, b"\x02" * 32, 100 + i, i, b"\0" * 32)
        att = wire.Attestation(wire.sha256(p, P.ctx), bytes([0x50 + i]) * 32, wire.Domain(1, 7),
                               bytes([0x60 + i]) * 32)
        b.transactions.append(wire.Transaction(p, att, b"treasury:0" if i == 2 else b""))
    b.header.tx_count = 3
    b.header.tx_merkle_root = wire.tx_merkle_root(b.transactions, P.ctx)
    b.header.attest_merkle_root = wire.attest_merkle_root(b.transactions, P.ctx)
    empty = wire.Block(wire.BlockHeader(**{**b.header.__dict__}), [])
    empty.header.tx_count = 0
    empty.header.tx_merkle_root = wire.tx_merkle_root([], P.ctx)
    empty.header.attest_merkle_root = wire.attest_merkle_root([], P.ctx)
    fc = wire.FinalityCertificate(wire.block_hash(b, P.ctx), 7, bytes(range(256)), b"\x77" * 32)

    def hx(raw):
        return hashlib.sha256(raw.hex().encode()).hexdigest()
    if g:
        assert hx(wire.encode_block(empty)) == g["empty_block.hex"]["sha256_of_hex_text"]
        assert hx(wire.encode_block(b)) == g["block_3tx.hex"]["sha256_of_hex_text"]
        assert hx(fc.encode()) == g["fc_328.hex"]["sha256_of_hex_text"]
        assert hx(b.transactions[0].attestation.encode()) == g["attestation_104.hex"]["sha256_of_hex_text"]
    assert wire.decode_block(wire.encode_block(b)) == b


# ------------------------------------------------------------ attestation
def test_attestation_api(P, kats):
    """test_crypto.cpp:162-214 + fixture KATs, on the GPU."""
    cr, wire = P.crypto, P.wire
    f = kats["fixture"]
    rev = cr.Rev.from_seed(20240801)
    assert rev.bytes().hex() == f["rev"]
    dom = wire.Domain(1, 40)
    idc = cr.id_commitment(rev, b"\0" * 32, dom)
    assert idc.bytes.hex() == f["id_com"]
    assert cr.derive_attest_key(rev, dom, P.ctx).hex() == f["attest_key"]
    assert cr.hkdf_sha256(rev.bytes(), dom.encode(), cr.INFO_MEMPOOL_ATTEST, 32, P.ctx).hex() == f["attest_key"]
    for v in kats["hmac"]:
        assert cr.hmac_sha256(bytes.fromhex(v["key"]), bytes.fromhex(v["msg"]), P.ctx).hex() == v["mac"]
    for v in kats["hkdf"]:
        assert cr.hkdf_sha256(bytes.fromhex(v["ikm"]), bytes.fromhex(v["salt"]),
                              bytes.fromhex(v["info"]), v["L"], P.ctx).hex() == v["okm"]
    with pytest.raises(ValueError):
        cr.hkdf_expand(b"k" * 32, b"i", 8161)
    pay = bytes.fromhex(f["payload0"])
    att = cr.generate_attestation(rev, pay, dom, idc, P.ctx)
    assert att.encode().hex() == f["attestation0"]
    assert cr.verify_attestation_full(att, pay, rev, P.ctx) == cr.AttestationCheck.Accept
    rng = random.Random(123)
    for _ in range(64):
        m = bytearray(pay)
        m[rng.randrange(len(m))] ^= 1 + rng.randrange(255)
        assert cr.verify_attestation_full(att, bytes(m), rev, P.ctx) == cr.AttestationCheck.PayloadMismatch
    moved = wire.Attestation(att.obj_hash, att.id_com, wire.Domain(1, 41), att.credential)
    assert cr.verify_attestation_full(moved, pay, rev, P.ctx) == cr.AttestationCheck.CredentialMismatch


def test_random_credentials_never_verify(P):
    """test_crypto.cpp:200-214 and acceptance criterion 6 (10^4 forgeries), batched."""
    rng = np.random.default_rng(77)
    n = 10000
    fb = O.canonical_block(1)
    pay, att = fb.payload(0), fb.att(0)
    atts = np.tile(np.frombuffer(att, np.uint8), n)
    atts.reshape(n, 104)[:, 72:] = rng.integers(0, 256, (n, 32), dtype=np.uint8)
    fbn = O.flat_from_lists([pay] * n, [atts[104 * i:104 * i + 104].tobytes() for i in range(n)],
                            fb.header, [O.rev_from_seed(20240801)], [0] * n)
    codes = P.crypto.verify_attestations(to_wire_flat(P, fbn), fbn.revs, fbn.rev_index, P.ctx)
    assert (codes == 2).all()


def test_generate_attestations_batch(P):
    fb = O.multi_user_block(2000, 16)
    doms = np.frombuffer(b"".join(fb.att(i)[64:72] for i in range(fb.n)), np.uint8).copy()
    ids = np.frombuffer(b"".join(fb.att(i)[32:64] for i in range(fb.n)), np.uint8).copy()
    out = P.crypto.generate_attestations(fb.payloads, fb.offs, fb.revs, fb.rev_index, doms, ids,
                                         P.ctx)
    assert out[:104 * fb.n].tobytes() == fb.atts[:104 * fb.n].tobytes()


# --------------------------------------------------------------- witnesses
def test_witness_scheme_and_backup(P, kats):
    """test_prover.cpp:176-263 on the GPU."""
    pr, cr = P.prover, P.crypto
    w = kats["witness"]
    key = bytes.fromhex(kats["fixture"]["attest_key"])
    th = bytes.fromhex(w["tx_hash"])
    wit = pr.build_witness(key, th, P.ctx)
    assert wit.hex() == w["witness"]
    scheme = pr.WitnessScheme(4, bytes.fromhex(w["master"]))
    assert scheme.threshold() == 3
    for n, masks in w["share_masks"].items():
        s = pr.WitnessScheme(int(n), b"\0" * 32)
        assert [sum(1 << j for j in s.share_indices(v)) for v in range(int(n))] == masks
    assert [scheme.share_value(th, j).hex() for j in range(3)] == w["shares_n4"]
    b = scheme.encapsulate(th, wit, P.ctx)
    assert b.ciphertext.hex() == w["ciphertext_n4"] and b.share_threshold == 3
    for skip in range(4):
        assert scheme.decrypt(b, [v for v in range(4) if v != skip], P.ctx) == wit
    garbage = scheme.decrypt(b, [0, 1], P.ctx)
    assert garbage != wit
    fbt = O.canonical_block(1)
    tx = to_wire_flat(P, fbt).to_block().transactions[0]
    assert pr.witness_matches_tx(wit, tx, P.ctx)
    assert not pr.witness_matches_tx(garbage, tx, P.ctx)
    assert not pr.witness_matches_tx(wit[:255], tx, P.ctx)
    with pytest.raises(ValueError):
        pr.WitnessScheme(0, b"\0" * 32)

    # backup_prove == builder FC (test_prover.cpp:201-263)
    fb = O.prover_test_block(9)
    block = to_wire_flat(P, fb).to_block()
    rev = cr.Rev.from_seed(7777)
    scheme = pr.WitnessScheme(4, b"\x77" * 32)
    bundles, holders = {}, {v: set() for v in range(4)}
    for t in block.transactions:
        h = P.wire.sha256(t.payload, P.ctx)
        k = cr.derive_attest_key(rev, t.attestation.domain, P.ctx)
        bundles[h] = scheme.encapsulate(h, pr.build_witness(k, h, P.ctx), P.ctx)
        for v in range(4):
            holders[v].add(h)
    builder = pr.build_finality_certificate(block, pr.prove_block(block, None, P.ctx), P.ctx)
    r = pr.backup_prove(block, bundles, holders, scheme, P.ctx)
    assert isinstance(r, P.wire.FinalityCertificate) and r == builder
    r = pr.backup_prove(block, bundles, {0: holders[0], 1: holders[1]}, scheme, P.ctx)
    assert isinstance(r, pr.BackupUnavailable) and len(r.missing_tx_hashes) == 9
    victim = P.wire.sha256(block.transactions[4].payload, P.ctx)
    partial = {k: v for k, v in bundles.items() if k != victim}
    r = pr.backup_prove(block, partial, holders, scheme, P.ctx)
    assert isinstance(r, pr.BackupUnavailable) and r.missing_tx_hashes == [victim]


def test_prover_service_and_counters(P):
    """test_prover.cpp:265-278."""
    pr = P.prover
    block = to_wire_flat(P, O.prover_test_block(12)).to_block()
    before = pr.work_counters().tx_proofs
    with pr.ProverService(P.ctx) as svc:
        svc.enqueue(block)
        res = svc.wait_result()
        assert res.fc.slot_number == block.header.slot_number
        assert pr.verify_finality_certificate(res.fc, block, None, P.ctx) == pr.FcCheck.Valid
        assert svc.blocks_enqueued() == 1 and svc.blocks_proved() == 1
    assert pr.work_counters().tx_proofs >= before + 12


# --------------------------------------------------------------- sharding
@pytest.mark.parametrize("n,k", [(1, 2), (5, 1), (7, 2), (100, 3), (1000, 4), (1025, 10),
                                 (4097, 10), (6250, 8), (100000, 10)])
def test_shards_combine_to_global(P, kats, n, k):
    """aligned 2^k chunks proven shard-by-shard combine to the
    single-GPU root and FC bit-exactly (ranks emulated one after another), and
    both equal the FC the reference itself printed for this block (kats)."""
    from paper_2603_10242_b200 import shard
    fb = O.canonical_block(n)
    world = 4
    proof, fc = shard.prove_sharded_single_process(to_wire_flat(P, fb), world, k, P.ctx)
    gproof, gfc, _, _, _ = gpu_block(P, fb, codes=False)
    assert proof == gproof and fc == gfc
    g = kats["canonical_blocks"][str(n)]
    assert fc.hex() == g["fc"] and proof[256:288].hex() == g["root_digest"]


def test_segmented_pipeline_equals_single_pass(P):
    """The overlapped host-input pipeline (per-segment H2D + leaf kernels)
    must give the single-pass pipeline's verdicts, proof and FC (and the oracle's)."""
    fb = O.forge(O.multi_user_block(40000, 5), every=5, phase=3)
    seg = gpu_block(P, fb)
    P.ctx.call("acegpu_set_segmented", 0)
    try:
        single = gpu_block(P, fb)
    finally:
        P.ctx.call("acegpu_set_segmented", 1)
    assert seg[0] == single[0] and seg[1] == single[1] and (seg[2] == single[2]).all()
    assert (seg[2] == O.oracle_attest_codes(fb)).all()
    oproof, _, _ = O.oracle_prove_block(fb)
    assert seg[0] == oproof and seg[1] == O.oracle_build_fc(fb, oproof)


def test_pipelined_prover_stream():
    """Sustained-stream prover (stream.py): consecutive blocks over pipelined
    lanes give the oracle's verdicts, proof and FC, in submission order."""
    from paper_2603_10242_b200.stream import PipelinedProver
    blocks = [O.forge(O.multi_user_block(n, 4), every=7, phase=2) for n in (1, 700, 1024, 3000, 333)]
    pp = PipelinedProver(lanes=2, max_tx=4096, max_revs=8)
    try:
        tickets = [pp.submit(fb, fb.revs, fb.rev_index) for fb in blocks]
        res = pp.drain()
    finally:
        pp.close()
    assert [r.ticket for r in res] == tickets
    for fb, r in zip(blocks, res):
        assert (r.codes == O.oracle_attest_codes(fb)).all()
        oproof, _, _ = O.oracle_prove_block(fb)
        assert r.proof289 == oproof
        assert r.fc328 == O.oracle_build_fc(fb, oproof)
        assert r.latency_ms > 0


def test_rev_index_out_of_range_is_einval_after_the_run(P):
    """An out-of-range REV index is caught on the device (no O(n) host scan
    ahead of the copies): the host API still raises (EINVAL), for both the
    single-pass and the segmented pipeline, and the context stays usable."""
    for n in (1000, 20000):
        fb = O.multi_user_block(n, 3)
        bad = fb.rev_index.copy()
        bad[n // 2] = 7  # 3 REVs
        fb2 = O.FlatBlock(fb.payloads, fb.offs, fb.atts, fb.header, fb.revs, bad)
        with pytest.raises(ValueError):
            gpu_block(P, fb2)
        proof, fc, codes, _, _ = gpu_block(P, fb)
        assert (codes == 0).all()
        oproof, _, _ = O.oracle_prove_block(fb)
        assert proof == oproof


@pytest.mark.parametrize("graphs", [False, True])
def test_pipelined_prover_graph_replay(graphs):
    """Consecutive same-shape blocks through the CUDA-graph replay path (and
    the plain async path): each block's verdicts / proof / FC equal the
    oracle's, i.e. the replayed copy nodes really read the new block."""
    from paper_2603_10242_b200.stream import PipelinedProver
    base = O.multi_user_block(1500, 4)
    blocks = [O.forge(base, every=e, phase=p) for e, p in ((3, 0), (5, 1), (7, 2), (4, 3), (9, 4),
                                                          (6, 5), (11, 0))]
    pp = PipelinedProver(lanes=2, max_tx=2048, max_revs=8, graphs=graphs)
    try:
        tickets = [pp.submit(fb, fb.revs, fb.rev_index) for fb in blocks]
        res = pp.drain()
    finally:
        pp.close()
    assert [r.ticket for r in res] == tickets
    for fb, r in zip(blocks, res):
        assert (r.codes == O.oracle_attest_codes(fb)).all()
        oproof, _, _ = O.oracle_prove_block(fb)
        assert r.proof289 == oproof
        assert r.fc328 == O.oracle_build_fc(fb, oproof)


def test_graph_replay_segmented_pipeline():
    """Graph capture / replay of the segmented host pipeline (n >= 16,384:
    copy stream, per-segment leaf + subtree streams, side stream)."""
    from paper_2603_10242_b200.stream import PipelinedProver
    base = O.multi_user_block(20000, 3)
    blocks = [O.forge(base, every=e, phase=p) for e, p in ((3, 0), (5, 1), (7, 2))]
    pp = PipelinedProver(lanes=1, max_tx=20000, max_revs=4, graphs=True)
    try:
        for fb in blocks:
            pp.submit(fb, fb.revs, fb.rev_index)
        res = pp.drain()
    finally:
        pp.close()
    for fb, r in zip(blocks, res):
        assert (r.codes == O.oracle_attest_codes(fb)).all()
        oproof, _, _ = O.oracle_prove_block(fb)
        assert r.fc328 == O.oracle_build_fc(fb, oproof)
