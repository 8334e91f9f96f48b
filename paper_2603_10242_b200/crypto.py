"""Attestation crypto of the Prove path (reference proj/include/ace/crypto.hpp,
hkdf.hpp; proj/src/crypto.cpp, hkdf.cpp), every hash on the GPU.

The batched entry points (``verify_attestations``, ``generate_attestations``,
``derive_attest_keys``) are the B200-native form; the single-item functions
keep the reference's names and semantics on top of them.
"""
from __future__ import annotations

import enum
import struct
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .wire import Attestation, Domain, FlatBlock, sha256, sha256_many

INFO_MEMPOOL_ATTEST = b"ACEGF-V1-MEMPOOL-ATTEST"  # crypto.hpp:19


class AttestationCheck(enum.IntEnum):
    Accept = 0
    PayloadMismatch = 1
    CredentialMismatch = 2


def to_string(c: AttestationCheck) -> str:
    return AttestationCheck(c).name


class Rev:
    """Root entropy value, 32 B (crypto.hpp:27-40)."""

    def __init__(self, b: bytes):
        assert len(b) == 32
        self._b = bytes(b)

    @staticmethod
    def from_bytes(b: bytes) -> "Rev | None":
        return Rev(b) if len(b) == 32 else None

    @staticmethod
    def from_seed(seed: int) -> "Rev":
        """SHA-256("rev-seed" | seed_be64) (crypto.cpp:28-33)."""
        return Rev(sha256(b"rev-seed" + struct.pack(">Q", seed)))

    def bytes(self) -> bytes:
        return self._b

    def __eq__(self, o):
        return isinstance(o, Rev) and o._b == self._b

    def __hash__(self):
        return hash(self._b)


@dataclass
class IdCommitment:
    bytes: bytes
    salt: bytes
    domain: Domain


def id_commitment(rev: Rev, salt: bytes, domain: Domain) -> IdCommitment:
    """SHA-256(REV | salt | domain) (crypto.cpp:115-122)."""
    return IdCommitment(sha256(rev.bytes() + salt + domain.encode()), salt, domain)


# --------------------------------------------------------- HMAC / HKDF
def _hmac_many(pairs: list[tuple[bytes, bytes]], ctx=None) -> list[bytes]:
    """HmacCtx (hkdf.cpp:12-39) over a batch: keys > 64 B are hashed first."""
    long_keys = [k for k, _ in pairs if len(k) > 64]
    hashed = dict(zip(long_keys, sha256_many(long_keys, ctx))) if long_keys else {}
    kbs = [(hashed.get(k, k) if len(k) > 64 else k).ljust(64, b"\0") for k, _ in pairs]
    inner = sha256_many([bytes(x ^ 0x36 for x in kb) + m for kb, (_, m) in zip(kbs, pairs)], ctx)
    return sha256_many([bytes(x ^ 0x5C for x in kb) + ih for kb, ih in zip(kbs, inner)], ctx)


def hmac_sha256(key: bytes, msg: bytes, ctx=None) -> bytes:
    return _hmac_many([(key, msg)], ctx)[0]


def hkdf_extract(salt: bytes, ikm: bytes, ctx=None) -> bytes:
    """Empty salt is 32 zero bytes (hkdf.cpp:56-62)."""
    return hmac_sha256(salt if salt else b"\0" * 32, ikm, ctx)


def hkdf_expand(prk: bytes, info: bytes, out_len: int, ctx=None) -> bytes:
    if out_len > 255 * 32:
        raise ValueError("hkdf_expand: output length too large")  # hkdf.cpp:65-67
    okm, t, ctr = b"", b"", 1
    while len(okm) < out_len:
        t = hmac_sha256(prk, t + info + bytes([ctr]), ctx)
        ctr += 1
        okm += t
    return okm[:out_len]


def hkdf_sha256(ikm: bytes, salt: bytes, info: bytes, out_len: int, ctx=None) -> bytes:
    return hkdf_expand(hkdf_extract(salt, ikm, ctx), info, out_len, ctx)


def derive_key(rev: Rev, info: bytes, salt: bytes, ctx=None) -> bytes:
    """crypto.cpp:78-89: info must be non-empty."""
    if not info:
        raise ValueError("derive_key: info must be non-empty")
    return hkdf_sha256(rev.bytes(), salt, info, 32, ctx)


# ----------------------------------------------------- batched attestation
def derive_attest_keys(revs: list[bytes], domains: list[bytes], ctx=None) -> list[bytes]:
    """derive_attest_key (crypto.cpp:124-127) over (REV, 8-B domain) pairs."""
    if not revs:
        return []
    ctx = ctx or N.context()
    r = np.frombuffer(b"".join(revs), np.uint8).copy()
    d = np.frombuffer(b"".join(domains), np.uint8).copy()
    out = np.zeros(32 * len(revs), np.uint8)
    ctx.call("acegpu_derive_attest_keys", N.addr(r), N.addr(d), len(revs), N.addr(out))
    return [out[32 * i:32 * i + 32].tobytes() for i in range(len(revs))]


def derive_attest_key(rev: Rev, domain: Domain, ctx=None) -> bytes:
    return derive_attest_keys([rev.bytes()], [domain.encode()], ctx)[0]


def generate_attestations(payloads: np.ndarray, offs: np.ndarray, revs: np.ndarray,
                          rev_index: np.ndarray, doms8: np.ndarray, id_coms: np.ndarray,
                          ctx=None) -> np.ndarray:
    """generate_attestation (crypto.cpp:129-139), batched; returns n x 104 B."""
    n = len(offs) - 1
    ctx = ctx or N.context()
    out = np.zeros(104 * max(n, 1), np.uint8)
    if n:
        ctx.call("acegpu_attest_generate", N.addr(payloads), N.addr(offs), n, N.addr(revs),
                 len(revs) // 32, N.addr(rev_index), N.addr(doms8), N.addr(id_coms), N.addr(out))
    return out


def generate_attestation(rev: Rev, payload: bytes, domain: Domain, id_com: IdCommitment,
                         ctx=None) -> Attestation:
    pl = np.frombuffer(payload + b"\0" * 16, np.uint8).copy()
    offs = np.array([0, len(payload)], np.uint64)
    out = generate_attestations(pl, offs, np.frombuffer(rev.bytes(), np.uint8).copy(),
                                np.zeros(1, np.uint32),
                                np.frombuffer(domain.encode(), np.uint8).copy(),
                                np.frombuffer(id_com.bytes, np.uint8).copy(), ctx)
    return Attestation.decode(out[:104].tobytes())


def verify_attestations(fb: FlatBlock, revs: np.ndarray, rev_index: np.ndarray,
                        ctx=None) -> np.ndarray:
    """verify_attestation_full (crypto.cpp:141-154) over a whole block: one
    AttestationCheck code per tx."""
    ctx = ctx or N.context()
    codes = np.zeros(max(fb.n, 1), np.uint8)
    if fb.n:
        ctx.call("acegpu_attest_verify", N.addr(fb.payloads), N.addr(fb.offs), N.addr(fb.atts),
                 fb.n, N.addr(revs), len(revs) // 32, np.ascontiguousarray(rev_index, np.uint32),
                 N.addr(codes))
    return codes[:fb.n]


def verify_attestation_full(att: Attestation, payload: bytes, rev: Rev, ctx=None) -> AttestationCheck:
    fb = FlatBlock.from_lists([payload], [att.encode()], b"\0" * 256)
    codes = verify_attestations(fb, np.frombuffer(rev.bytes(), np.uint8).copy(),
                                np.zeros(1, np.uint32), ctx)
    return AttestationCheck(int(codes[0]))
