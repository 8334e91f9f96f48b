"""Phase 1a on the GPU: attest_check_light and the block
build (compaction + header Merkle roots) against the C oracle and the
reference's own pipeline::attest_check_light / wire::tx_merkle_root
(oracle/_ref, when present), then the built block proved on the device.
Mirrors test_pipeline.cpp's light-check cases."""
import ctypes as C

import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M():
    from paper_2603_10242_b200 import _native as N, pipeline, wire
    return type("M", (), {"N": N, "ctx": N.context(0), "pl": pipeline, "wire": wire})


def registry(M, ids):
    r = M.pl.IdentityRegistry()
    for i in ids:
        r.add(i)
    return r


def wire_flat(M, fb):
    return M.wire.FlatBlock(fb.payloads, fb.offs, fb.atts,
                            np.frombuffer(fb.header, np.uint8).copy())


@pytest.mark.parametrize("n,seed", [(1, 1), (2, 2), (255, 3), (4097, 4)])
@pytest.mark.parametrize("window", [0, 2])
def test_light_check_matches_oracle_and_reference(M, n, seed, window):
    fb, reg, cur = O.phase1_block(n, seed=seed)
    cfg = M.pl.PipelineConfig(domain_window_slots=window)
    cnt = M.pl.LightCheckCounters()
    got = M.pl.attest_check_light_batch(wire_flat(M, fb), registry(M, reg), cur, cfg, cnt,
                                        M.ctx)
    want = O.oracle_light_check(fb, reg, cur, window)
    assert (got == want).all()
    if O.ref_available():
        rc, rcnt = O.ref_light_check(fb, reg, cur, window)
        assert (got == rc).all()
        assert [cnt.sha256_ops, cnt.registry_probes, cnt.window_checks] == rcnt


def test_light_check_single_tx_api(M):
    """test_pipeline.cpp:58-82 through the single-transaction call."""
    rev = O.rev_from_seed(4242)
    dom = O.domain_encode(1, 50)
    idc = O.id_commitment(rev, b"\0" * 32, 1, 50)
    p = O.transfer_payload(b"\x01" * 32, b"\x02" * 32, 5, 0, b"\0" * 32)
    att = M.wire.Attestation.decode(O.generate_attestation(rev, p, dom, idc))
    tx = M.wire.Transaction(p, att)
    reg = registry(M, [idc])
    L = M.pl.LightCheck
    assert M.pl.attest_check_light(tx, reg, 50, ctx=M.ctx) == L.AcceptPendingProof
    bad = M.wire.Transaction(p[:10] + bytes([p[10] ^ 1]) + p[11:], att)
    assert M.pl.attest_check_light(bad, reg, 50, ctx=M.ctx) == L.PayloadBinding
    assert M.pl.attest_check_light(tx, registry(M, []), 50, ctx=M.ctx) == L.UnknownIdentity
    for cur, want in ((52, L.AcceptPendingProof), (53, L.StaleDomain),
                      (48, L.AcceptPendingProof), (47, L.StaleDomain)):
        assert M.pl.attest_check_light(tx, reg, cur, ctx=M.ctx) == want


@pytest.mark.parametrize("n,seed", [(0, 0), (1, 5), (3, 6), (1000, 7), (20000, 8)])
def test_build_block_then_prove(M, n, seed):
    """Light check -> compaction -> header roots -> attest/prove/FC, all on
    the device; equals the oracle's selection, roots, proof and FC."""
    import torch
    fb, reg, cur = O.phase1_block(n, seed=seed)
    hdr = M.wire.BlockHeader(slot_number=cur, parent_hash=b"\x07" * 32, state_root=b"\x09" * 32,
                             timestamp_ms=cur * 400)
    built = M.pl.build_block_device(wire_flat(M, fb), registry(M, reg), hdr, ctx=M.ctx)
    codes = O.oracle_light_check(fb, reg, cur, 2)
    keep = codes == 0
    assert built.n == int(keep.sum())
    assert (built.codes.cpu().numpy() == codes).all()
    tx_root, att_root = O.oracle_block_roots(O.select(fb, keep, b"\0" * 256))
    want_hdr = O.encode_header(slot=cur, parent=b"\x07" * 32, state=b"\x09" * 32,
                               tx_root=tx_root, att_root=att_root, ts=cur * 400,
                               tx_count=built.n)
    got_hdr = built.header.cpu().numpy().tobytes()
    assert got_hdr == want_hdr
    sel = O.select(fb, keep, want_hdr)
    offs = built.offs.cpu().numpy().view(np.uint64)
    assert (offs == sel.offs).all()
    k = built.n
    assert built.payloads.cpu().numpy()[:int(offs[-1])].tobytes() == sel.payloads[:int(offs[-1])].tobytes()
    assert built.atts.cpu().numpy()[:104 * k].tobytes() == sel.atts[:104 * k].tobytes()
    if O.ref_available() and k:
        assert O.ref_block_roots(sel) == (tx_root, att_root)
    # feed the prover straight from device memory
    out = torch.empty(640, dtype=torch.uint8, device=built.header.device)
    M.ctx.call("acegpu_attest_prove_certify_dev", torch.cuda.current_stream().cuda_stream,
               built.payloads.data_ptr(), built.offs.data_ptr(), built.atts.data_ptr(), k,
               built.header.data_ptr(), None, 0, None, None, out.data_ptr(),
               out.data_ptr() + 304)
    o = out.cpu().numpy()
    oproof, _, _ = O.oracle_prove_block(sel)
    assert o[:289].tobytes() == oproof
    assert o[304:632].tobytes() == O.oracle_build_fc(sel, oproof)


def test_tx_merkle_roots(M):
    for n in (1, 2, 5, 1024, 1025):
        fb, _, _ = O.phase1_block(n, seed=n)
        assert M.pl.tx_merkle_roots(wire_flat(M, fb), ctx=M.ctx) == O.oracle_block_roots(fb)


def test_light_check_rejects_null_codes(M):
    fb, reg, cur = O.phase1_block(4, seed=1)
    with pytest.raises(ValueError):
        M.ctx.call("acegpu_light_check", M.N.addr(fb.payloads), M.N.addr(fb.offs),
                   M.N.addr(fb.atts), fb.n, None, 0, cur, 2, None, None)
    _ = C


def test_phase1_does_no_proof_work(M):
    """test_pipeline.cpp:169-190: Phase 1 (light check + block build) leaves
    the prover's work counters unchanged."""
    from paper_2603_10242_b200 import prover
    fb, reg, cur = O.phase1_block(500, seed=9)
    wc = prover.work_counters()
    before = (wc.tx_proofs, wc.aggregations)
    M.pl.attest_check_light_batch(wire_flat(M, fb), registry(M, reg), cur, ctx=M.ctx)
    M.pl.build_block_device(wire_flat(M, fb), registry(M, reg),
                            M.wire.BlockHeader(slot_number=cur), ctx=M.ctx)
    assert (wc.tx_proofs, wc.aggregations) == before
