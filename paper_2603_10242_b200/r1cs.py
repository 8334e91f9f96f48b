"""General rank-1 constraint systems on the GPU (north-star "witness /
constraint evaluation") — host API over libacegpu (csrc/r1cs.cu).

A constraint system is three CSR matrices over Fr (A, B, C); the prover's
row evaluations A z, B z, C z and the Groth16 setup's column sums A^T L(tau)
run on the device. `synthetic_chunk` builds the stand-in circuit of
oracle/bn254_oracle.h as such a matrix triple (rows in the order
csrc/groth16.cu's witness kernel evaluates them), so the bespoke chunk prover
and the general one can be checked against each other bit for bit.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .bn254 import R

ONE_LE = (1).to_bytes(32, "little")


class Csr:
    """One sparse matrix: rowptr (m + 1 u64), cols (u32), vals (nnz x 32-B LE)."""

    def __init__(self, rowptr, cols, vals):
        self.rowptr = np.ascontiguousarray(rowptr, np.uint64)
        self.cols = np.ascontiguousarray(cols, np.uint32)
        self.vals = np.ascontiguousarray(vals, np.uint8).reshape(-1)
        assert len(self.vals) == 32 * len(self.cols) and int(self.rowptr[-1]) == len(self.cols)

    @staticmethod
    def from_rows(rows: list[dict[int, int]]) -> "Csr":
        """rows: one {column: coefficient} dict per constraint row (small cases)."""
        rp, cols, vals = [0], [], []
        for r in rows:
            for c, v in sorted(r.items()):
                cols.append(c)
                vals.append((v % R).to_bytes(32, "little"))
            rp.append(len(cols))
        return Csr(np.array(rp, np.uint64), np.array(cols, np.uint32),
                   np.frombuffer(b"".join(vals) or b"", np.uint8).copy())


class R1CS:
    """A constraint system resident on the device (acegpu_r1cs). The library
    appends one z_i * 0 = 0 row per public variable (rows = m + n_pub + 1)."""

    def __init__(self, m: int, vars: int, n_pub: int, A: Csr, B: Csr, Cm: Csr, ctx=None):
        self.ctx = ctx or N.context()
        self.m, self.vars, self.n_pub = m, vars, n_pub
        self.rows = m + n_pub + 1
        self._keep = (A, B, Cm)
        rp = (C.c_void_p * 3)(*[x.rowptr.ctypes.data for x in (A, B, Cm)])
        cl = (C.c_void_p * 3)(*[x.cols.ctypes.data if len(x.cols) else None for x in (A, B, Cm)])
        vl = (C.c_void_p * 3)(*[x.vals.ctypes.data if len(x.vals) else None for x in (A, B, Cm)])
        h = C.c_void_p()
        self.ctx.call("acegpu_r1cs_create", m, vars, n_pub, rp, cl, vl, C.byref(h))
        self.h = h

    def eval(self, z: np.ndarray) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """(A z, B z, C z) over all rows, 32-B LE standard form each."""
        out = [np.zeros(32 * self.rows, np.uint8) for _ in range(3)]
        self.ctx.call("acegpu_r1cs_eval", self.h, np.ascontiguousarray(z, np.uint8), *out)
        return tuple(out)

    def close(self):
        if self.h:
            N.lib().acegpu_r1cs_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def chain_constants(K: int, ctx=None) -> list[int]:
    """c_k = LE(SHA-256("ace-g16-chain-v1" | k_be32)) mod r (c_0 unused = 0),
    hashed on the GPU."""
    from .wire import sha256_many
    d = sha256_many([b"ace-g16-chain-v1" + k.to_bytes(4, "big") for k in range(K)], ctx)
    return [0] + [int.from_bytes(bytes(x), "little") % R for x in d[1:]]


def synthetic_chunk(T: int, K: int, ctx=None) -> tuple[int, int, int, Csr, Csr, Csr]:
    """The stand-in circuit (oracle/bn254_oracle.h) as CSR: -> (m, vars, n_pub,
    A, B, C). Variables: 0 ONE, 1..T pub_t, then per tx t: w_t, x_{t,0..K-1}.
    Rows t K: (w_t + pub_t) * ONE = x_{t,0}; t K + k: (x_{t,k-1} + c_k ONE)^2 = x_{t,k}."""
    cks = chain_constants(K, ctx)
    cbytes = np.frombuffer(b"".join(c.to_bytes(32, "little") for c in cks), np.uint8).reshape(K, 32)
    one = np.frombuffer(ONE_LE, np.uint8)
    m = T * K
    t = np.repeat(np.arange(T, dtype=np.int64), K)
    k = np.tile(np.arange(K, dtype=np.int64), T)
    vb = 1 + T + t * (K + 1)                  # w_t
    x_prev = vb + k                          # x_{t,k-1} for k >= 1 (== w_t + k)
    x_cur = vb + 1 + k                       # x_{t,k}
    first = k == 0
    # A: row k=0 -> {pub_t: 1, w_t: 1}; k>=1 -> {ONE: c_k, x_{k-1}: 1}; 2 entries per row
    a_c0 = np.where(first, 1 + t, 0)
    a_c1 = np.where(first, vb, x_prev)
    a_cols = np.stack([a_c0, a_c1], 1).reshape(-1).astype(np.uint32)
    a_v0 = np.where(first[:, None], one[None, :], cbytes[k])
    a_vals = np.stack([a_v0, np.broadcast_to(one, (m, 32))], 1).reshape(-1)
    A = Csr(np.arange(m + 1, dtype=np.uint64) * 2, a_cols, a_vals)
    # B: row k=0 -> {ONE: 1}; k>=1 -> same as A
    b_rp = np.concatenate([[0], np.cumsum(np.where(first, 1, 2))]).astype(np.uint64)
    sel = np.stack([~first, np.ones(m, bool)], 1).reshape(-1)
    b_cols = np.stack([a_c0, np.where(first, 0, a_c1)], 1).reshape(-1)[sel].astype(np.uint32)
    b_vals = np.stack([a_v0, np.broadcast_to(one, (m, 32))], 1).reshape(-1, 32)[sel].reshape(-1)
    B = Csr(b_rp, b_cols, b_vals)
    Cm = Csr(np.arange(m + 1, dtype=np.uint64), x_cur.astype(np.uint32),
             np.broadcast_to(one, (m, 32)).reshape(-1))
    return m, 1 + T + T * (K + 1), T, A, B, Cm


def synthetic_assignment(T: int, K: int, w: np.ndarray, pub: np.ndarray, cks: list[int]) -> np.ndarray:
    """The full assignment z of the stand-in circuit (standard form, LE)."""
    ws = [int.from_bytes(w[32 * i:32 * i + 32].tobytes(), "little") % R for i in range(T)]
    ps = [int.from_bytes(pub[32 * i:32 * i + 32].tobytes(), "little") % R for i in range(T)]
    z = [1] + ps
    for t in range(T):
        x = (ws[t] + ps[t]) % R
        z += [ws[t], x]
        for kk in range(1, K):
            y = (x + cks[kk]) % R
            x = y * y % R
            z.append(x)
    return np.frombuffer(b"".join(v.to_bytes(32, "little") for v in z), np.uint8).copy()
