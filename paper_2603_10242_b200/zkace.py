"""Block prover over the REAL ZK-ACE credential relation (zkace_circuit.py:
HMAC-SHA256(attest key, obj_hash || domain) == credential, ~103k constraints
per tx) instead of the paper-size stand-in circuit: every aligned chunk of T
txs (a power of two, so chunk roots are tree nodes, shard.py) is one Groth16
proof whose witness the GPU generates from the block's build_witness records
(prover.cpp:181-188; the attest key is its first 32 B) and attestations
(csrc/witprog.cu), whose constraints the GPU evaluates (csrc/r1cs.cu), and
whose public inputs are each tx's obj_hash / domain / credential. Chunk
proofs are leaves of the reference's aggregation tree (prover.cpp:106-127)
under the FC, as in the stand-in path. A short last chunk repeats its last
transaction (a satisfiable padding the verifier recomputes the same way).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .groth16 import ProvingKey
from .r1cs import R1CS
from .zkace_circuit import N_PUB_PER_TX, WitnessProgram, chunk_r1cs


class ZkAceProver:
    def __init__(self, T: int = 16, trapdoor: np.ndarray | None = None, ctx=None):
        assert T & (T - 1) == 0, "txs per chunk must be a power of two"
        self.ctx = ctx or N.context()
        self.T = T
        self.log2_chunk = T.bit_length() - 1
        m, V, npub, A, B, Cm = chunk_r1cs(T)
        self.r1cs = R1CS(m, V, npub, A, B, Cm, ctx=self.ctx)
        self.pk = ProvingKey.from_r1cs(self.r1cs, trapdoor, self.ctx)
        self.prog = WitnessProgram(self.ctx)
        self.n_pub = npub
        self.zbytes = 32 * V
        self.batch_chunks = 64  # witness batch: 64 x 16 txs, ~3.4 GB of assignments

    def _padded(self, n: int) -> np.ndarray:
        """Index of the tx each chunk slot proves (the last tx repeats)."""
        chunks = -(-n // self.T)
        idx = np.arange(chunks * self.T)
        return np.minimum(idx, n - 1)

    def prove_block(self, db, n_total: int, codes=None, return_chunk_proofs: bool = False):
        """db: a shard.DeviceBlock of the whole block with `witnesses` (n x 256 B)
        -> (root proof 289 B, FC 328 B[, chunk proofs]) as device tensors.
        Verdicts (and the id_com Merkle tree) come from the hash-proof shard
        path; the chunk roots are the Groth16 proofs."""
        import torch
        from . import shard
        n = db.n
        assert n == n_total and n > 0
        dev = db.atts.device
        T = self.T
        chunks = -(-n // T)
        # verdicts + Merkle nodes at the chunk level (the mock roots are discarded)
        _, merk = shard.GpuBackend(self.ctx).shard_roots(db, n, self.log2_chunk, codes)
        sel = torch.from_numpy(self._padded(n)).to(dev)
        keys = db.witnesses.view(n, 256)[sel, :32].contiguous()
        atts = db.atts[:104 * n].view(n, 104)[sel].contiguous()
        out = torch.empty(chunks * 544, dtype=torch.uint8, device=dev)
        sp = torch.cuda.current_stream().cuda_stream
        # the witness program runs for a batch of chunks at once (one thread
        # per tx, slots interleaved), then each chunk is proven from its slice
        for c0 in range(0, chunks, self.batch_chunks):
            nb = min(self.batch_chunks, chunks - c0)
            z = torch.empty(nb * self.zbytes, dtype=torch.uint8, device=dev)
            self.prog.run_dev(keys[T * c0:].data_ptr(), 32, atts[T * c0:].data_ptr(), nb * T,
                              z.data_ptr(), stream=sp, Tc=T)
            for k in range(nb):
                o = out.data_ptr() + 544 * (c0 + k)
                self.ctx.call("acegpu_g16_prove_z_dev", sp, self.pk.h,
                              z.data_ptr() + self.zbytes * k, None, o, o + 256, o + 512)
        o = out.view(chunks, 544)
        roots = torch.zeros(chunks, 289, dtype=torch.uint8, device=dev)
        roots[:, :256] = o[:, :256]
        roots[:, 256:288] = o[:, 512:544]  # kind byte 0 = ProofKind::Tx
        proof, fc = shard.GpuBackend(self.ctx).combine(roots.view(-1), merk, chunks, n, db.header)
        if return_chunk_proofs:
            return proof, fc, o[:, :256].contiguous()
        return proof, fc

    def public_inputs(self, atts_host: np.ndarray, n: int) -> list[bytes]:
        """Each chunk's public inputs (T x 5 x 32 B) recomputed from the
        attestations, with the same padding rule."""
        sel = self._padded(n)
        out = []
        for k in range(len(sel) // self.T):
            b = b""
            for i in sel[self.T * k:self.T * (k + 1)]:
                a = atts_host[104 * i:104 * i + 104].tobytes()
                for lo, ln in ((0, 16), (16, 16), (64, 8), (72, 16), (88, 16)):
                    b += int.from_bytes(a[lo:lo + ln], "big").to_bytes(32, "little")
            out.append(b)
        return out

    def verify_chunk_proofs(self, proofs: list[bytes], atts_host: np.ndarray, n: int) -> bool:
        """The batched pairing check of every chunk proof against the public
        inputs recomputed from the block."""
        return self.pk.verify_batch(proofs, self.public_inputs(atts_host, n))

    def close(self):
        for o in (self.prog, self.pk, self.r1cs):
            o.close()
