"""ctypes bindings to the CHECKERS under oracle/ (test infrastructure only).

* ``Oracle``  -> oracle/liboracle.so, our plain-C restatement (always present
  once built; ``make -C oracle oracle``).
* ``Ref``     -> oracle/_ref/libaceref.so, the unmodified reference sources
  (/root/reference/proj/src) behind our extern "C" shim. Built here by
  ``make -C oracle ref``; the prebuilt .so travels to the GPU box.

Also the deterministic fixture builders the reference tests use
(acceptance.cpp:35-60 ``canonical_block``; test_prover.cpp:17-41 ``make_block``),
computed with the oracle, so that every test feeds identical inputs to the
oracle, the reference and the CUDA path.
"""
from __future__ import annotations

import ctypes as C
import os
import struct
from dataclasses import dataclass, field

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libaceref.so")

u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)


def buf(n: int) -> C.Array:
    return (C.c_uint8 * max(n, 1))()


def ptr(b) -> u8p:
    if isinstance(b, np.ndarray):
        return b.ctypes.data_as(u8p)
    if isinstance(b, (bytes, bytearray)):
        return C.cast(C.c_char_p(bytes(b)), u8p)
    return C.cast(b, u8p)


def np_ptr(a: np.ndarray, t):
    return a.ctypes.data_as(C.POINTER(t))


_oracle = None
_ref = None


def oracle() -> C.CDLL:
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"{ORACLE_SO} missing: run `make -C oracle oracle`")
        _oracle = C.CDLL(ORACLE_SO)
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        _ref = C.CDLL(REF_SO)
        _ref.ref_attest_prove_certify.restype = C.c_double
        _ref.ref_work_tx_proofs.restype = C.c_uint64
        _ref.ref_work_aggregations.restype = C.c_uint64
        _ref.ref_scheme_share_mask.restype = C.c_uint64
    return _ref


# ------------------------------------------------------------------ helpers
def sha256(data: bytes) -> bytes:
    out = buf(32)
    oracle().or_sha256(ptr(data), C.c_uint64(len(data)), out)
    return bytes(out)


def rev_from_seed(seed: int) -> bytes:
    out = buf(32)
    oracle().or_rev_from_seed(C.c_uint64(seed), out)
    return bytes(out)


def domain_encode(chain: int, slot: int) -> bytes:
    return struct.pack(">H", chain) + slot.to_bytes(6, "big")


def id_commitment(rev: bytes, salt: bytes, chain: int, slot: int) -> bytes:
    out = buf(32)
    oracle().or_id_commitment(ptr(rev), ptr(salt), C.c_uint16(chain), C.c_uint64(slot), out)
    return bytes(out)


def derive_attest_key(rev: bytes, dom8: bytes) -> bytes:
    out = buf(32)
    oracle().or_derive_attest_key(ptr(rev), ptr(dom8), out)
    return bytes(out)


def transfer_payload(frm: bytes, to: bytes, amount: int, nonce: int, recent: bytes) -> bytes:
    out = buf(154)
    oracle().or_make_transfer_payload(ptr(frm), ptr(to), C.c_uint64(amount), C.c_uint64(nonce),
                                      ptr(recent), out)
    return bytes(out)


def generate_attestation(rev: bytes, payload: bytes, dom8: bytes, id_com: bytes) -> bytes:
    out = buf(104)
    oracle().or_generate_attestation(ptr(rev), ptr(payload), C.c_uint64(len(payload)), ptr(dom8),
                                     ptr(id_com), out)
    return bytes(out)


def encode_header(slot=0, parent=b"\0" * 32, state=b"\0" * 32, tx_root=b"\0" * 32,
                  att_root=b"\0" * 32, poh=b"\0" * 32, leader=b"\0" * 32, ts=0,
                  tx_count=0) -> bytes:
    """BlockHeader::encode (wire.cpp:74-98)."""
    h = (struct.pack(">Q", slot) + parent + state + tx_root + att_root + poh + leader
         + struct.pack(">QI", ts, tx_count))
    assert len(h) == 212
    return h + b"\0" * 44


def merkle_root(leaves: list[bytes]) -> bytes:
    out = buf(32)
    arr = b"".join(leaves)
    oracle().or_merkle_root(ptr(arr), C.c_uint64(len(leaves)), out)
    return bytes(out)


@dataclass
class FlatBlock:
    """A block in the flat layout shared by oracle, reference shim and C-ABI."""
    payloads: np.ndarray          # uint8, concatenated
    offs: np.ndarray              # uint64, n+1
    atts: np.ndarray              # uint8, n*104
    header: bytes                 # 256
    revs: np.ndarray = field(default_factory=lambda: np.zeros(32, np.uint8))
    rev_index: np.ndarray = field(default_factory=lambda: np.zeros(1, np.uint32))

    @property
    def n(self) -> int:
        return len(self.offs) - 1

    def payload(self, i: int) -> bytes:
        return self.payloads[self.offs[i]:self.offs[i + 1]].tobytes()

    def att(self, i: int) -> bytes:
        return self.atts[104 * i:104 * (i + 1)].tobytes()

    def copy(self) -> "FlatBlock":
        return FlatBlock(self.payloads.copy(), self.offs.copy(), self.atts.copy(), self.header,
                         self.revs.copy(), self.rev_index.copy())


def flat_from_lists(payloads: list[bytes], atts: list[bytes], header: bytes,
                    revs: list[bytes] | None = None, rev_index=None) -> FlatBlock:
    offs = np.zeros(len(payloads) + 1, np.uint64)
    if payloads:
        offs[1:] = np.cumsum([len(p) for p in payloads])
    pl = np.frombuffer(b"".join(payloads) or b"\0", np.uint8).copy()
    at = np.frombuffer(b"".join(atts) or b"\0", np.uint8).copy()
    fb = FlatBlock(pl, offs, at, header)
    if revs is not None:
        fb.revs = np.frombuffer(b"".join(revs), np.uint8).copy()
        fb.rev_index = np.asarray(rev_index if rev_index is not None else [0] * len(payloads),
                                  np.uint32)
    if len(fb.rev_index) < max(1, fb.n):
        fb.rev_index = np.zeros(max(1, fb.n), np.uint32)
    return fb


def _header_for(payloads, atts, slot, ts=0):
    tx_root = merkle_root([sha256(p) for p in payloads])
    att_root = merkle_root([sha256(a) for a in atts])
    return encode_header(slot=slot, tx_root=tx_root, att_root=att_root, ts=ts,
                         tx_count=len(payloads))


def canonical_block(n: int) -> FlatBlock:
    """acceptance.cpp:35-60: REV seed 20240801, Domain{1,40}, id_com salt 0^32,
    tx i = transfer(0x01^32 -> 0x02^32, amount 10, nonce i)."""
    rev = rev_from_seed(20240801)
    dom = domain_encode(1, 40)
    idc = id_commitment(rev, b"\0" * 32, 1, 40)
    a, b = b"\x01" * 32, b"\x02" * 32
    payloads, atts = [], []
    for i in range(n):
        p = transfer_payload(a, b, 10, i, b"\0" * 32)
        payloads.append(p)
        atts.append(generate_attestation(rev, p, dom, idc))
    return flat_from_lists(payloads, atts, _header_for(payloads, atts, 40), [rev], [0] * n)


def multi_user_block(n: int, users: int = 16, slot: int = 40) -> FlatBlock:
    """user u's REV = Rev::from_seed(0xFACE000+u)
    (seed formula after sim.cpp:345-350); tx i attested by user i mod users."""
    revs = [rev_from_seed(0xFACE000 + u) for u in range(users)]
    dom = domain_encode(1, slot)
    idcs = [id_commitment(r, b"\0" * 32, 1, slot) for r in revs]
    keys = [derive_attest_key(r, dom) for r in revs]
    a, b = b"\x01" * 32, b"\x02" * 32
    payloads, atts = [], []
    for i in range(n):
        u = i % users
        p = transfer_payload(a, b, 10, i, b"\0" * 32)
        payloads.append(p)
        obj = sha256(p)
        cred = hmac(keys[u], obj + dom)
        atts.append(obj + idcs[u] + dom + cred)
    return flat_from_lists(payloads, atts, _header_for(payloads, atts, slot), revs,
                           [i % users for i in range(n)])


def prover_test_block(n: int, slot: int = 9) -> FlatBlock:
    """test_prover.cpp:17-41 make_block: REV seed 7777, Domain{1,slot},
    amount 10+nonce, timestamp slot*400."""
    rev = rev_from_seed(7777)
    dom = domain_encode(1, slot)
    idc = id_commitment(rev, b"\0" * 32, 1, slot)
    a, b = b"\x01" * 32, b"\x02" * 32
    payloads, atts = [], []
    for i in range(n):
        p = transfer_payload(a, b, 10 + i, i, b"\0" * 32)
        payloads.append(p)
        atts.append(generate_attestation(rev, p, dom, idc))
    return flat_from_lists(payloads, atts, _header_for(payloads, atts, slot, ts=slot * 400),
                           [rev], [0] * n)


def hmac(key: bytes, msg: bytes) -> bytes:
    out = buf(32)
    oracle().or_hmac_sha256(ptr(key), C.c_uint64(len(key)), ptr(msg), C.c_uint64(len(msg)), out)
    return bytes(out)


# ---------------------------------------------------------- block-level calls
def _blk_args(fb: FlatBlock):
    return (np_ptr(fb.payloads, C.c_uint8), np_ptr(fb.offs, C.c_uint64),
            np_ptr(fb.atts, C.c_uint8), C.c_uint32(fb.n))


def oracle_prove_block(fb: FlatBlock, threads: int = 8):
    out = buf(289)
    lv, pr = C.c_uint64(), C.c_uint64()
    rc = oracle().or_prove_block(*_blk_args(fb), ptr(fb.header), out, C.byref(lv), C.byref(pr),
                                 C.c_int(threads))
    assert rc == 0
    return bytes(out), lv.value, pr.value


def oracle_build_fc(fb: FlatBlock, proof289: bytes) -> bytes:
    out = buf(328)
    oracle().or_build_fc(np_ptr(fb.atts, C.c_uint8), C.c_uint32(fb.n), ptr(fb.header),
                         ptr(proof289), out)
    return bytes(out)


def oracle_verify_fc(fc: bytes, fb: FlatBlock, threads: int = 8) -> int:
    return oracle().or_verify_fc(ptr(fc), *_blk_args(fb), ptr(fb.header), C.c_int(threads))


def oracle_attest_codes(fb: FlatBlock, threads: int = 8) -> np.ndarray:
    codes = np.zeros(max(fb.n, 1), np.uint8)
    oracle().or_verify_attestations_batch(*_blk_args(fb), np_ptr(fb.revs, C.c_uint8),
                                          np_ptr(fb.rev_index, C.c_uint32),
                                          np_ptr(codes, C.c_uint8), C.c_int(threads))
    return codes[:fb.n]


def ref_prove_block(fb: FlatBlock):
    out = buf(289)
    lv, pr = C.c_uint64(), C.c_uint64()
    rc = ref().ref_prove_block(*_blk_args(fb), ptr(fb.header), out, C.byref(lv), C.byref(pr))
    assert rc == 0
    return bytes(out), lv.value, pr.value


def ref_prove_and_certify(fb: FlatBlock) -> bytes:
    out = buf(328)
    assert ref().ref_prove_and_certify(*_blk_args(fb), ptr(fb.header), out) == 0
    return bytes(out)


def ref_attest_codes(fb: FlatBlock) -> np.ndarray:
    codes = np.zeros(max(fb.n, 1), np.uint8)
    ref().ref_verify_attestations_batch(*_blk_args(fb), np_ptr(fb.revs, C.c_uint8),
                                        np_ptr(fb.rev_index, C.c_uint32),
                                        np_ptr(codes, C.c_uint8))
    return codes[:fb.n]


def forge(fb: FlatBlock, every: int = 8, phase: int = 7) -> FlatBlock:
    """Forged variant: tx i ≡ phase mod every is forged,
    cycling four forgery types after sim.cpp:392-407 — random credential,
    domain replay (slot+1), payload mutation, foreign REV credential."""
    out = fb.copy()
    k = 0
    for i in range(fb.n):
        if i % every != phase:
            continue
        a = bytearray(out.att(i))
        kind = k % 4
        k += 1
        if kind == 0:
            a[72:104] = sha256(b"forged-cred" + i.to_bytes(8, "big"))
        elif kind == 1:
            slot = int.from_bytes(a[66:72], "big") + 1
            a[66:72] = slot.to_bytes(6, "big")
        elif kind == 2:
            j = int(out.offs[i]) + (i * 37) % int(out.offs[i + 1] - out.offs[i])
            out.payloads[j] ^= 0x5A
        else:
            other = rev_from_seed(0xBAD000 + i)
            key = derive_attest_key(other, bytes(a[64:72]))
            a[72:104] = hmac(key, bytes(a[0:32]) + bytes(a[64:72]))
        out.atts[104 * i:104 * (i + 1)] = np.frombuffer(bytes(a), np.uint8)
    return out


# ------------------------------------------------------------- phase 1a
def phase1_block(n: int, seed: int = 5, cur: int = 100, users: int = 6):
    """Candidate txs for the light check (pipeline.cpp:20-42): honest txs of
    `users` registered identities with domain slots in cur-4..cur+4, some
    mutated payloads (PayloadBinding), some unregistered identities
    (UnknownIdentity). Returns (FlatBlock, sorted registry ids (+ decoys), cur)."""
    import random
    rng = random.Random(seed)
    revs = [rev_from_seed(0xB10C00 + u) for u in range(users + 2)]
    a, b = b"\x01" * 32, b"\x02" * 32
    payloads, atts = [], []
    for i in range(n):
        u = rng.randrange(users + 2)  # users, users+1: never registered
        slot = cur + rng.randint(-4, 4)
        dom = domain_encode(1, slot)
        idc = id_commitment(revs[u], b"\0" * 32, 1, slot)
        p = transfer_payload(a, b, 1 + i, i, b"\0" * 32)
        att = generate_attestation(revs[u], p, dom, idc)
        if rng.random() < 0.15:
            p = bytearray(p)
            p[rng.randrange(len(p))] ^= 1 << rng.randrange(8)
            p = bytes(p)
        payloads.append(p)
        atts.append(att)
    reg = set()
    for u in range(users):
        for slot in range(cur - 4, cur + 5):
            reg.add(id_commitment(revs[u], b"\0" * 32, 1, slot))
    for k in range(50):  # decoys
        reg.add(sha256(b"decoy" + k.to_bytes(4, "big")))
    fb = flat_from_lists(payloads, atts, encode_header(slot=cur), revs[:users], [0] * n)
    return fb, sorted(reg), cur


def oracle_light_check(fb: FlatBlock, reg: list[bytes], cur: int, window: int = 2) -> np.ndarray:
    r = b"".join(reg) or b"\0" * 32
    out = np.zeros(max(fb.n, 1), np.uint8)
    for i in range(fb.n):
        p = fb.payload(i)
        out[i] = oracle().or_attest_check_light(
            ptr(p), C.c_uint64(len(p)), ptr(fb.atts[104 * i:104 * i + 104].tobytes()), ptr(r),
            C.c_uint64(len(reg)), C.c_uint64(cur), C.c_uint64(window))
    return out[:fb.n]


def ref_light_check(fb: FlatBlock, reg: list[bytes], cur: int, window: int = 2):
    r = b"".join(reg) or b"\0" * 32
    codes = np.zeros(max(fb.n, 1), np.uint8)
    cnt = np.zeros(3, np.uint64)
    ref().ref_attest_check_light_batch(*_blk_args(fb), ptr(r), C.c_uint64(len(reg)),
                                       C.c_uint64(cur), C.c_uint64(window),
                                       np_ptr(codes, C.c_uint8), np_ptr(cnt, C.c_uint64))
    return codes[:fb.n], [int(x) for x in cnt]


def oracle_block_roots(fb: FlatBlock) -> tuple[bytes, bytes]:
    t, a = buf(32), buf(32)
    oracle().or_block_roots(np_ptr(fb.payloads, C.c_uint8), np_ptr(fb.offs, C.c_uint64),
                            np_ptr(fb.atts, C.c_uint8), C.c_uint64(fb.n), t, a)
    return bytes(t), bytes(a)


def ref_block_roots(fb: FlatBlock) -> tuple[bytes, bytes]:
    t, a = buf(32), buf(32)
    ref().ref_tx_merkle_root(*_blk_args(fb), t, a)
    return bytes(t), bytes(a)


def select(fb: FlatBlock, keep: np.ndarray, header: bytes) -> FlatBlock:
    """The sub-block of the txs with keep[i] (order preserved)."""
    idx = [i for i in range(fb.n) if keep[i]]
    return flat_from_lists([fb.payload(i) for i in idx],
                           [fb.atts[104 * i:104 * i + 104].tobytes() for i in idx], header)
