"""CPU-only checks of the host side: the C-ABI library loads and exports every
symbol include/acegpu.h declares (no compute calls — there is no GPU here),
the product fails loudly without a GPU, wire codecs, and the multi-rank
sharding plumbing over gloo (world size 2) with the oracle standing in for the
per-rank GPU work."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle_lib as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "acegpu.h")).read()
    return sorted(set(re.findall(r"\b(acegpu_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_2603_10242_b200 import _native as N
    lib = N.lib()
    syms = declared_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(N._SIGS), "ctypes signatures must cover the header exactly"
    assert lib.acegpu_version().startswith(b"acegpu sm_100a")


def test_library_is_sm100a_only():
    import subprocess
    so = os.path.join(ROOT, "paper_2603_10242_b200", "lib", "libacegpu.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2603_10242_b200 import _native as N
    with pytest.raises(N.AceGpuError):
        N.Context(0)


def test_wire_codecs_match_oracle(kats):
    from paper_2603_10242_b200 import wire
    p = wire.make_transfer_payload(b"\x01" * 32, b"\x02" * 32, 10, 0, b"\0" * 32)
    assert p.hex() == kats["fixture"]["payload0"]
    assert len(p) == wire.CANONICAL_TRANSFER_PAYLOAD_SIZE
    att = wire.Attestation.decode(bytes.fromhex(kats["fixture"]["attestation0"]))
    assert att.domain == wire.Domain(1, 40) and att.encode().hex() == kats["fixture"]["attestation0"]
    fb = O.canonical_block(3)
    hdr = wire.BlockHeader.decode(fb.header)
    assert hdr.encode() == fb.header and hdr.slot_number == 40 and hdr.tx_count == 3
    fc = wire.FinalityCertificate.decode(bytes.fromhex(kats["canonical_blocks"]["3"]["fc"]))
    assert fc.encode().hex() == kats["canonical_blocks"]["3"]["fc"] and fc.slot_number == 40
    assert wire.FinalityCertificate.decode(b"\0" * 327) is None
    blk = wire.FlatBlock(fb.payloads, fb.offs, fb.atts, np.frombuffer(fb.header, np.uint8)).to_block()
    raw = wire.encode_block(blk)
    assert wire.decode_block(raw) == blk
    assert wire.decode_block(raw[:-1]) is None


def test_partition_balanced_and_aligned():
    from paper_2603_10242_b200.shard import partition
    for n in (1, 5, 1023, 1024, 1025, 100000, 12800, 16384):
        for w in (1, 2, 4, 8):
            parts = partition(n, w, 10)
            assert sum(c for _, c in parts) == n
            pos = 0
            for s, c in parts:
                assert s == pos and s % 1024 == 0 or c == 0
                pos += c
    # 100k on 8 GPUs: 98 chunks -> 12 or 13 per rank (not 6x16384 + 1696)
    chunks = [-(-c // 1024) for _, c in partition(100000, 8, 10)]
    assert sorted(set(chunks)) == [12, 13]


# ------------------------------------------------- gloo multi-rank plumbing
class OracleBackend:
    """Test stand-in for GpuBackend: per-rank chunk roots by the CPU oracle."""

    def __init__(self, fb_global, start):
        self.fb, self.start = fb_global, start

    def shard_roots(self, db, n_total, k, codes=None):
        import torch
        C_ = 1 << k
        roots, merk = b"", b""
        for c0 in range(0, db.n, C_):
            lo, hi = self.start + c0, self.start + min(c0 + C_, db.n)
            proofs = b""
            for i in range(lo, hi):
                p = O.buf(289)
                O.oracle().or_prove_tx(O.ptr(self.fb.payload(i)),
                                       C.c_uint64(len(self.fb.payload(i))), O.ptr(self.fb.att(i)), p)
                proofs += bytes(p)
            out = O.buf(289)
            lv, pr = C.c_uint64(), C.c_uint64()
            O.oracle().or_aggregate_tree(O.ptr(proofs), C.c_uint64(hi - lo), out, C.byref(lv),
                                         C.byref(pr))
            roots += bytes(out)
            m = O.merkle_root([self.fb.att(i)[32:64] for i in range(lo, hi)])
            if n_total > C_:
                for _ in range((hi - lo - 1).bit_length(), k):
                    m = O.sha256(b"\x01" + m + m)  # lift the short last chunk
            merk += m
        t = lambda b: torch.frombuffer(bytearray(b or b"\0"), dtype=torch.uint8)[:len(b)]
        return t(roots), t(merk)

    def combine(self, roots, merk, chunks, n_total, header):
        import torch
        r = roots.numpy().tobytes()
        lv, pr = C.c_uint64(), C.c_uint64()
        out = O.buf(289)
        O.oracle().or_aggregate_tree(O.ptr(r), C.c_uint64(chunks), out, C.byref(lv), C.byref(pr))
        level = [merk.numpy().tobytes()[32 * i:32 * i + 32] for i in range(chunks)]
        while len(level) > 1:
            if len(level) % 2:
                level.append(level[-1])
            level = [O.sha256(b"\x01" + level[2 * i] + level[2 * i + 1]) for i in range(len(level) // 2)]
        hdr = header.numpy().tobytes()
        fc = O.sha256(hdr) + hdr[:8] + bytes(out)[:256] + level[0]
        return torch.frombuffer(bytearray(bytes(out)), dtype=torch.uint8), \
            torch.frombuffer(bytearray(fc), dtype=torch.uint8)


def _worker(rank, world, port, n, k, q):
    import torch.distributed as dist
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_10242_b200 import shard
        fb = O.canonical_block(n)
        s, c = shard.partition(n, world, k)[rank]
        db = shard.DeviceBlock(None, None, None, torch.frombuffer(bytearray(fb.header), dtype=torch.uint8), c)
        proof, fc = shard.prove_sharded(db, n, rank, world, k, backend=OracleBackend(fb, s))
        q.put((rank, proof.numpy().tobytes(), fc.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,k", [(5, 1), (1025, 4), (3000, 8)])
def test_sharded_gloo_world2_matches_global(n, k):
    import multiprocessing as mp
    import random
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randrange(20000, 40000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, k, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    fb = O.canonical_block(n)
    root, _, _ = O.oracle_prove_block(fb)
    fc = O.oracle_build_fc(fb, root)
    for _, proof, got_fc in res:
        assert proof == root and got_fc == fc


def test_identity_registry_is_the_sorted_set():
    """IdentityRegistry (pipeline.hpp:22-30): set semantics, and the device
    layout is the std::set<Hash32> iteration order (bytewise ascending)."""
    import random

    from paper_2603_10242_b200 import pipeline
    rng = random.Random(4)
    ids = [bytes(rng.getrandbits(8) for _ in range(32)) for _ in range(200)]
    reg = pipeline.IdentityRegistry()
    for i in ids + ids[:50]:
        reg.add(i)
    assert reg.size() == len(set(ids))
    arr = reg.array().reshape(-1, 32)
    got = [bytes(r) for r in arr]
    assert got == sorted(set(ids))
    assert all(reg.contains(i) for i in ids)
    assert not reg.contains(b"\xff" * 32)
    assert pipeline.IdentityRegistry().array().shape == (32,)  # empty: one dummy row, size 0


def test_light_check_counters_accumulate():
    from paper_2603_10242_b200 import pipeline
    c = pipeline.LightCheckCounters()
    c += pipeline.LightCheckCounters(3, 2, 1)
    c += pipeline.LightCheckCounters(1, 1, 1)
    assert (c.sha256_ops, c.registry_probes, c.window_checks) == (4, 3, 2)
    assert pipeline.to_string(pipeline.LightCheck.StaleDomain) == "StaleDomain"


def _exchange_worker(rank, world, port, N, shares, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_10242_b200 import shard
        # vector k (32-B elements, byte pattern (k, index)) lives on its owner
        vecs = []
        for k in range(3):
            v = torch.zeros(N, 32, dtype=torch.uint8)
            v[:, 0] = k + 1
            v[:, 1] = torch.arange(N) % 251
            v[:, 2] = torch.arange(N) // 251
            vecs.append(v.reshape(-1))
        own = [vecs[k] for k in range(3) if k % world == rank]
        own = torch.cat(own) if own else torch.zeros(32, dtype=torch.uint8)
        out = shard.exchange_slices(own, rank, world, N, shares=shares)
        q.put((rank, out.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shares", [(2, None), (2, [3, 5]), (3, [1, 4, 2])])
def test_one_proof_slice_exchange_gloo(world, shares):
    """The one-proof-per-block exchange (shard.exchange_slices): every owner
    of an H vector (k mod world) sends each rank its share-bounded slice —
    scatter for equal shares, point-to-point sends for weighted ones — and
    every rank ends with the a | b | c slices of its own range."""
    import multiprocessing as mp
    import random

    import numpy as np
    from paper_2603_10242_b200 import shard
    N = 1000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randrange(20000, 40000)
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, N, shares, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        lo, hi = shard.slice_bounds(N, r, world, shares)
        got = np.frombuffer(res[r], np.uint8).reshape(3, hi - lo, 32)
        for k in range(3):
            idx = np.arange(lo, hi)
            assert (got[k, :, 0] == k + 1).all()
            assert (got[k, :, 1] == idx % 251).all() and (got[k, :, 2] == idx // 251).all()


def test_one_proof_shares_and_slices_partition_the_arrays():
    """Split one-proof keys (acegpu_g16_setup_slice): the share-weighted slices
    of an array cover it exactly once, in rank order, for the measured
    tables and the formula alike; vector k of the H polynomial is owned by
    rank k mod world (every vector exactly once)."""
    from paper_2603_10242_b200 import shard
    for world in (1, 2, 3, 4, 5, 8):
        shares = shard.balanced_shares(world) if world > 1 else None
        if shares is not None:
            assert len(shares) == world and min(shares) >= 1
        for N in (1, 7, 24, 3 << 19, 140_100_004, 3 << 26):
            prev = 0
            for r in range(world):
                lo, hi = shard.slice_bounds(N, r, world, shares)
                assert lo == prev and hi >= lo
                prev = hi
            assert prev == N
        owners = [shard.owned_mask(r, world) for r in range(world)]
        assert sum(bin(m).count("1") for m in owners) == 3
        assert owners[0] & 1 and (owners[1 % world] >> 1) & 1 and (owners[2 % world] >> 2) & 1
    assert shard.balanced_shares(8, ntt_frac=0.1) != shard.balanced_shares(8, ntt_frac=0.0)
