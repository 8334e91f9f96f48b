"""Python statement of the Groth16 binding rules (binding v2, include/acegpu.h
and csrc/groth16.cu / csrc/g16_verify.cu) — test-side checker only.

D(x)   = SHA-256(tag16 | SHA-256(x_0..x_31) | SHA-256(x_32..x_63) | ... | T_be32)
r, s   = LE(SHA-256("ace-g16-r-v2" / "ace-g16-s-v2" | D(w) | D(pub))) mod r
digest = SHA-256("ace-g16-chunk-v2" | D(pub))
seed   = SHA-256("ace-g16-seed-v2:" | SHA-256(vk) | (SHA-256(proof_i) | D(pub_i))_i)
rho_i  = LE(SHA-256("ace-g16-batch-v2" | seed | i_be32)[0:16])  (1 if zero)
"""
from __future__ import annotations

import hashlib

R = 21888242871839275222246405745257275088548364400416034343698204186575808495617


def sha(b: bytes) -> bytes:
    return hashlib.sha256(b).digest()


def input_digest(x: bytes, T: int, wits: bool = False) -> bytes:
    """D(x): 1-KB blocks (32 inputs) hashed, then (for more than 32 blocks)
    the digests again in 1-KB blocks until at most 32 remain; the top hashes
    tag16 | digests | T_be32."""
    assert len(x) == 32 * T
    tag = b"ace-g16-wits-v2:" if wits else b"ace-g16-pubs-v2:"
    level = [sha(x[1024 * b:1024 * b + 1024]) for b in range((T + 31) // 32)]
    while len(level) > 32:
        cat = b"".join(level)
        level = [sha(cat[1024 * b:1024 * b + 1024]) for b in range((len(level) + 31) // 32)]
    return sha(tag + b"".join(level) + T.to_bytes(4, "big"))


def derive_rs(w: bytes, pub: bytes, T: int) -> tuple[int, int]:
    wd, pd = input_digest(w, T, True), input_digest(pub, T)
    r = int.from_bytes(sha(b"ace-g16-r-v2" + wd + pd), "little") % R
    s = int.from_bytes(sha(b"ace-g16-s-v2" + wd + pd), "little") % R
    return r, s


def chunk_digest(pub: bytes, T: int) -> bytes:
    return sha(b"ace-g16-chunk-v2" + input_digest(pub, T))


def batch_seed(vk: bytes, proofs: list[bytes], pubs: list[bytes], T: int) -> bytes:
    m = b"ace-g16-seed-v2:" + sha(vk)
    for p, q in zip(proofs, pubs):
        m += sha(p) + input_digest(q, T)
    return sha(m)


def batch_rho(seed: bytes, i: int) -> int:
    v = int.from_bytes(sha(b"ace-g16-batch-v2" + seed + i.to_bytes(4, "big"))[:16], "little")
    return v or 1
