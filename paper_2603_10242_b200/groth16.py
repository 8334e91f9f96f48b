"""Groth16 per-chunk prover over BN254 (north star) — host API over libacegpu.

Synthetic ZK-ACE stand-in circuit (constraint system in
oracle/bn254_oracle.h): per tx a private witness w_t (the attest key,
prover.cpp:181-188) and public input pub_t (the tx's public-inputs digest,
prover.cpp:74-76), K constraints of a squaring chain. A proving key is built
once per (T, K) from a trapdoor and stays resident on the device.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .bn254 import R

PAPER_T, PAPER_K = 1024, 1400  # 1,024-tx chunks x ~1,400 constraints/tx


def deterministic_trapdoor(label: bytes = b"ace-g16-setup-v1", ctx=None) -> np.ndarray:
    """tau, alpha, beta, gamma, delta = LE(SHA-256(label | i)) mod r (hashed on
    the GPU) — a synthetic, reproducible ceremony stand-in, never for production."""
    from .wire import sha256_many
    digests = sha256_many([label + bytes([i]) for i in range(5)], ctx)
    vals = [(int.from_bytes(d, "little") % R).to_bytes(32, "little") for d in digests]
    return np.frombuffer(b"".join(vals), np.uint8).copy()


class ProvingKey:
    def __init__(self, T: int, K: int, trapdoor: np.ndarray | None = None, ctx=None,
                 rank: int = 0, world: int = 1, shares=None):
        """world > 1: rank `rank`'s split key for one proof per block across
        ranks (acegpu_g16_setup_slice): its slice of the bases (rank r gets
        shares[r] / sum(shares) of each array; None = equal), the whole
        verifying key; prove with shard.prove_one_proof."""
        self.ctx = ctx or N.context()
        self.T, self.K = T, K
        self.rank, self.world = rank, world
        self.shares = None if shares is None else np.ascontiguousarray(shares, np.uint32)
        self.trapdoor = deterministic_trapdoor(ctx=self.ctx) if trapdoor is None else trapdoor
        h = C.c_void_p()
        if world > 1:
            self.ctx.call("acegpu_g16_setup_slice", T, K, self.trapdoor, rank, world, self.shares,
                          C.byref(h))
        else:
            self.ctx.call("acegpu_g16_setup", T, K, self.trapdoor, C.byref(h))
        self.h = h
        V, m, L = C.c_uint64(), C.c_uint64(), C.c_uint32()
        N.lib().acegpu_g16_shape(self.h, C.byref(V), C.byref(m), C.byref(L))
        self.variables, self.constraints, self.log_domain = V.value, m.value, L.value
        D = C.c_uint64()
        N.lib().acegpu_g16_domain(self.h, C.byref(D))
        self.domain = D.value  # 2^log_domain, or 3 x 2^log_domain (mixed radix)

    @classmethod
    def from_r1cs(cls, r1cs, trapdoor: np.ndarray | None = None, ctx=None) -> "ProvingKey":
        """Keys for a general constraint system (r1cs.R1CS; it must outlive
        the key): prove with prove_z(z) on the full assignment."""
        self = cls.__new__(cls)
        self.ctx = ctx or r1cs.ctx
        self.T, self.K, self.r1cs = r1cs.n_pub, 0, r1cs
        self.rank, self.world, self.shares = 0, 1, None
        self.trapdoor = deterministic_trapdoor(ctx=self.ctx) if trapdoor is None else trapdoor
        h = C.c_void_p()
        self.ctx.call("acegpu_g16_setup_r1cs", r1cs.h, self.trapdoor, C.byref(h))
        self.h = h
        V, m, L = C.c_uint64(), C.c_uint64(), C.c_uint32()
        N.lib().acegpu_g16_shape(self.h, C.byref(V), C.byref(m), C.byref(L))
        self.variables, self.constraints, self.log_domain = V.value, m.value, L.value
        D = C.c_uint64()
        N.lib().acegpu_g16_domain(self.h, C.byref(D))
        self.domain = D.value  # 2^log_domain, or 3 x 2^log_domain (mixed radix)
        return self

    def prove_z(self, z: np.ndarray, rs: np.ndarray | None = None):
        """General R1CS key: the full assignment z (vars x 32-B) ->
        (proof256, raw affine points, public-inputs digest)."""
        proof = np.zeros(256, np.uint8)
        raw = np.zeros(256, np.uint8)
        dig = np.zeros(32, np.uint8)
        self.ctx.call("acegpu_g16_prove_z", self.h, np.ascontiguousarray(z, np.uint8), rs, proof,
                      raw, dig)
        return proof.tobytes(), raw.tobytes(), dig.tobytes()

    def prove(self, w: np.ndarray, pub: np.ndarray, rs: np.ndarray | None = None):
        """-> (proof256 bytes, raw affine points bytes, chunk digest bytes)."""
        proof = np.zeros(256, np.uint8)
        raw = np.zeros(256, np.uint8)
        dig = np.zeros(32, np.uint8)
        self.ctx.call("acegpu_g16_prove_chunk", self.h, w, pub, rs, proof, raw, dig)
        return proof.tobytes(), raw.tobytes(), dig.tobytes()

    def prove_dev(self, d_w, d_pub, d_proof, d_raw=None, d_digest=None, d_rs=None, stream=None):
        self.ctx.call("acegpu_g16_prove_chunk_dev", stream, self.h, d_w, d_pub, d_rs, d_proof,
                      d_raw, d_digest)

    def prove_block(self, block, witnesses: np.ndarray, revs=None, rev_index=None):
        """The Groth16-mode prove_block + FC through one host-buffer call
        (acegpu_g16_prove_block): -> (codes, proof289, fc328, chunk proofs
        (ceil(n/T) x 256 B)). witnesses: n x 256-B build_witness records."""
        from .prover import _flat
        fb = _flat(block)
        n = fb.n
        chunks = -(-n // self.T)
        codes = np.zeros(max(n, 1), np.uint8)
        proof = np.zeros(289, np.uint8)
        fc = np.zeros(328, np.uint8)
        cps = np.zeros(256 * max(chunks, 1), np.uint8)
        nrev = 0 if revs is None else len(revs) // 32
        rix = None if rev_index is None else np.ascontiguousarray(rev_index, np.uint32)
        self.ctx.call("acegpu_g16_prove_block", self.h, fb.payloads, fb.offs, fb.atts, n,
                      np.ascontiguousarray(fb.header, np.uint8), revs, nrev, rix,
                      np.ascontiguousarray(witnesses, np.uint8), codes, proof, fc, cps)
        return codes[:n], proof.tobytes(), fc.tobytes(), cps[:256 * chunks].tobytes()

    def verifying_key(self) -> bytes:
        """alpha G1 | beta G2 | gamma G2 | delta G2 | IC_0..IC_T (oracle encoding)."""
        out = np.zeros(448 + 64 * (self.T + 1), np.uint8)
        self.ctx.call("acegpu_g16_vk", self.h, out)
        return out.tobytes()

    def verify_batch(self, proofs: list[bytes], pubs: list[bytes], return_seed: bool = False):
        """Batched pairing verification of chunk proofs (EIP-197 256 B each)
        against their T x 32-B public inputs. return_seed: also return the
        32-B Fiat-Shamir seed of the batch weights (include/acegpu.h)."""
        if not proofs:
            return (True, None) if return_seed else True
        ok = C.c_int(0)
        p = np.frombuffer(b"".join(proofs), np.uint8).copy()
        q = np.frombuffer(b"".join(pubs), np.uint8).copy()
        seed = np.zeros(32, np.uint8)
        self.ctx.call("acegpu_g16_verify_batch_seed", self.h, p, q, len(proofs), C.byref(ok),
                      seed)
        return (ok.value == 1, seed.tobytes()) if return_seed else ok.value == 1

    def verify_finality_certificate(self, fc, block, chunk_proofs: bytes, cost_units=None):
        """verify_finality_certificate (prover.cpp:158-169) in Groth16 mode:
        slot, block hash, then the chunk proofs by one batched pairing check
        and the FC recomputed from them -> prover.FcCheck."""
        from .prover import FcCheck, _flat
        fb = _flat(block)
        fcb = np.frombuffer(fc.encode() if hasattr(fc, "encode") else bytes(fc), np.uint8).copy()
        cu = C.c_uint64(0)
        res = C.c_int(-1)
        cp = np.frombuffer(bytes(chunk_proofs) or b"\0", np.uint8).copy()
        hdr = np.ascontiguousarray(fb.header, np.uint8)
        self.ctx.call("acegpu_g16_verify_fc", self.h, fcb, fb.payloads, fb.offs, fb.atts, fb.n,
                      hdr, cp, C.byref(cu), C.byref(res))
        if cost_units is not None:
            cost_units.value += cu.value
        return FcCheck(res.value)

    def close(self):
        if self.h:
            N.lib().acegpu_g16_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
