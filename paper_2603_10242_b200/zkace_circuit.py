"""The ZK-ACE credential relation as a rank-1 constraint system: a proof of
knowledge of the attest key w with HMAC-SHA256(w, obj_hash || domain) ==
credential — the check the reference's prover runs in the clear
(witness_matches_tx, proj/src/prover.cpp:190-197; crypto.cpp:141-154) —
compiled to R1CS for the general Groth16 path (r1cs.py, csrc/r1cs.cu).

Circuit per transaction (SHA-256 in R1CS over bits, FIPS 180-4):
  private : the 256 key bits (boolean-constrained)
  public  : obj_hash (2 x 128-bit words), domain (64 bits), credential (2 x
            128-bit words) -> 5 field elements, each tied to its bits by one
            packing constraint
  HMAC    : inner = SHA-256((w || 0^32) ^ ipad || obj_hash || domain)  (2 compressions)
            outer = SHA-256((w || 0^32) ^ opad || inner)               (2 compressions)
            outer == credential (packed)
Gadgets: XOR a + b - 2ab (1 constraint; with a constant bit it is affine,
free), Ch = e (f - g) + g (1), Maj = a (b + c - 2bc) + bc (2), rotations and
shifts are wiring, a k-word addition mod 2^32 is one linear constraint plus
32 result and ceil(log2 k) carry bits (boolean-constrained).
About 27k constraints per compression, ~109k per transaction; the count is
reported by `constraints_per_tx()`. The host builds the circuit once per
transaction shape and evaluates the assignment (the witness generator); the
device does everything else (r1cs.cu SpMV, NTT, MSM).
"""
from __future__ import annotations

import numpy as np

from .bn254 import R

_K = [
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2]
_IV = [0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a, 0x510e527f, 0x9b05688c, 0x1f83d9ab,
       0x5be0cd19]

N_PUB_PER_TX = 5  # obj_hash (2), domain (1), credential (2)


class Bit:
    """A boolean value as a linear combination {var: coef} (var 0 = ONE) and,
    for the witness program, the slot that holds its value (slots 0 / 1 are
    the constants)."""
    __slots__ = ("lc", "v", "s")

    def __init__(self, lc: dict, v: int, s: int | None = None):
        self.lc, self.v = lc, v
        self.s = v if s is None else s  # constants live in slots 0 / 1


def _const(b: int) -> Bit:
    return Bit({0: 1} if b else {}, b)


class Builder:
    """Constraint rows + the assignment, built together (var 0 = ONE,
    1..n_pub the public inputs)."""

    def __init__(self, n_pub: int):
        self.vals = [1] + [0] * n_pub
        self.A: list[dict] = []
        self.B: list[dict] = []
        self.C: list[dict] = []
        # witness program (zkace_witness.py): ops computing every slot from
        # earlier ones, and the slot of each private variable in creation order
        self.prog: list[tuple] = []
        self.nslot = 2
        self.var_slot: list[int] = []

    def slot(self, op: tuple) -> int:
        s = self.nslot
        self.nslot += 1
        self.prog.append((op[0], s) + op[1:])
        return s

    def var(self, value: int, slot: int | None = None) -> int:
        self.vals.append(value % R)
        self.var_slot.append(slot)
        return len(self.vals) - 1

    def row(self, a: dict, b: dict, c: dict) -> None:
        self.A.append(a)
        self.B.append(b)
        self.C.append(c)

    # ---- bits
    def bit(self, v: int, src: tuple) -> Bit:
        """A new boolean variable whose value the witness program computes
        with `src` (("KEY", i) / ("MSG", i) / ("SUMBIT", add, k))."""
        s = self.slot(src)
        x = self.var(v, s)
        self.row({x: 1}, {x: 1}, {x: 1})  # x * x = x
        return Bit({x: 1}, v, s)

    @staticmethod
    def _is_const(lc: dict) -> bool:
        return all(k == 0 for k in lc)

    @staticmethod
    def lin(*terms) -> dict:  # terms: (coef, lc)
        out: dict = {}
        for c, lc in terms:
            for k, x in lc.items():
                y = (out.get(k, 0) + c * x) % R
                if y:
                    out[k] = y
                else:
                    out.pop(k, None)
        return out

    def prod(self, a: dict, av: int, b: dict, bv: int, op: tuple = ()) -> dict:
        """a * b: a constant factor scales the other (no constraint), else one
        multiplication row with a fresh variable (its value computed by the
        witness program op `op`)."""
        if self._is_const(a):
            return self.lin((av, b))
        if self._is_const(b):
            return self.lin((bv, a))
        t = self.var(av * bv, self.slot(op))
        self.row(a, b, {t: 1})
        return {t: 1}

    def _bit(self, lc: dict, v: int, op: tuple) -> Bit:
        """A result bit: a constant, or a slot the program computes."""
        if self._is_const(lc):
            return Bit(lc, v)
        return Bit(lc, v, self.slot(op))

    def xor(self, a: Bit, b: Bit) -> Bit:  # a + b - 2ab
        t = self.prod(a.lc, a.v, b.lc, b.v, ("AND", a.s, b.s))
        return self._bit(self.lin((1, a.lc), (1, b.lc), (-2, t)), a.v ^ b.v, ("XOR", a.s, b.s))

    def ch(self, e: Bit, f: Bit, g: Bit) -> Bit:  # e (f - g) + g
        t = self.prod(e.lc, e.v, self.lin((1, f.lc), (-1, g.lc)), f.v - g.v,
                      ("CHP", e.s, f.s, g.s))
        return self._bit(self.lin((1, t), (1, g.lc)), (e.v & f.v) ^ ((1 - e.v) & g.v),
                         ("CH", e.s, f.s, g.s))

    def maj(self, a: Bit, b: Bit, c: Bit) -> Bit:  # a (b + c - 2bc) + bc
        bc = self.prod(b.lc, b.v, c.lc, c.v, ("AND", b.s, c.s))
        inner = self.lin((1, b.lc), (1, c.lc), (-2, bc))
        t = self.prod(a.lc, a.v, inner, b.v ^ c.v, ("MAJP", a.s, b.s, c.s))
        return self._bit(self.lin((1, t), (1, bc)), (a.v & b.v) ^ (a.v & c.v) ^ (b.v & c.v),
                         ("MAJ", a.s, b.s, c.s))

    # ---- 32-bit words: lists of 32 Bits, LSB first
    def add(self, words: list, k: int = 0) -> list:
        s = sum(sum(b.v << i for i, b in enumerate(w)) for w in words) + k
        nc = max(1, (len(words) + (1 if k else 0) - 1).bit_length())
        # the sum itself: an "ADD" op over the words' bit slots (+ k)
        add = self.slot(("ADD", tuple(b.s for w in words for b in w), k))
        r = [self.bit((s >> i) & 1, ("SUMBIT", add, i)) for i in range(32)]
        cr = [self.bit((s >> (32 + j)) & 1, ("SUMBIT", add, 32 + j)) for j in range(nc)]
        terms = [(1 << i, b.lc) for w in words for i, b in enumerate(w)]
        terms += [(-(1 << i), b.lc) for i, b in enumerate(r)]
        terms += [(-(1 << (32 + j)), b.lc) for j, b in enumerate(cr)]
        terms.append((k, {0: 1}))
        self.row(self.lin(*terms), {0: 1}, {})  # linear: sum - result - carry 2^32 = 0
        return r


def _wconst(x: int) -> list:
    return [_const((x >> i) & 1) for i in range(32)]


def _rotr(w, n):
    return [w[(i + n) % 32] for i in range(32)]


def _shr(w, n):
    return [w[i + n] if i + n < 32 else _const(0) for i in range(32)]


def _xor3(B: Builder, x, y, z):
    return [B.xor(B.xor(a, b), c) for a, b, c in zip(x, y, z)]


def compress(B: Builder, H: list, W: list) -> list:
    """SHA-256 compression of one block (16 words) onto state H (8 words)."""
    W = list(W)
    for t in range(16, 64):
        s0 = _xor3(B, _rotr(W[t - 15], 7), _rotr(W[t - 15], 18), _shr(W[t - 15], 3))
        s1 = _xor3(B, _rotr(W[t - 2], 17), _rotr(W[t - 2], 19), _shr(W[t - 2], 10))
        W.append(B.add([s1, W[t - 7], s0, W[t - 16]]))
    a, b, c, d, e, f, g, h = H
    for t in range(64):
        S1 = _xor3(B, _rotr(e, 6), _rotr(e, 11), _rotr(e, 25))
        ch = [B.ch(x, y, z) for x, y, z in zip(e, f, g)]
        S0 = _xor3(B, _rotr(a, 2), _rotr(a, 13), _rotr(a, 22))
        mj = [B.maj(x, y, z) for x, y, z in zip(a, b, c)]
        e2 = B.add([d, h, S1, ch, W[t]], _K[t])
        a2 = B.add([h, S1, ch, W[t], S0, mj], _K[t])
        h, g, f, e, d, c, b, a = g, f, e, e2, c, b, a, a2
    return [B.add([x, y]) for x, y in zip(H, [a, b, c, d, e, f, g, h])]


def _bytes_to_words(bits_by_byte: list) -> list:
    """64 bytes (each a list of 8 Bits, MSB first) -> 16 big-endian words."""
    words = []
    for w in range(16):
        bb = bits_by_byte[4 * w:4 * w + 4]
        msb_first = [b for byte in bb for b in byte]
        words.append(list(reversed(msb_first)))
    return words


def _const_byte(x: int) -> list:
    return [_const((x >> (7 - i)) & 1) for i in range(8)]


def hmac_tx(B: Builder, key: bytes, obj_hash: bytes, domain: bytes, credential: bytes,
            pub_vars: list[int]) -> None:
    """HMAC-SHA256(key, obj_hash || domain) == credential for one tx; the five
    public variables pub_vars get their packed values."""
    kb = [[B.bit((byte >> (7 - i)) & 1, ("KEY", 8 * j + i)) for i in range(8)]
          for j, byte in enumerate(key)]  # private key bits
    msg = obj_hash + domain
    mb = [[B.bit((byte >> (7 - i)) & 1, ("MSG", 8 * j + i)) for i in range(8)]
          for j, byte in enumerate(msg)]
    # public packing: obj_hash halves, domain, credential halves (big-endian integers)
    def pack(byte_bits, pv):
        flat = [b for byte in byte_bits for b in byte]  # MSB first
        n = len(flat)
        v = sum(b.v << (n - 1 - i) for i, b in enumerate(flat))
        B.vals[pv] = v
        B.row(B.lin(*[(1 << (n - 1 - i), b.lc) for i, b in enumerate(flat)], (-1, {pv: 1})),
              {0: 1}, {})
    pack(mb[0:16], pub_vars[0])
    pack(mb[16:32], pub_vars[1])
    pack(mb[32:40], pub_vars[2])

    def keyblock(pad):
        out = []
        for i in range(64):
            src = kb[i] if i < 32 else _const_byte(0)
            out.append([B.xor(b, _const((pad >> (7 - j)) & 1)) for j, b in enumerate(src)])
        return out
    iv = [_wconst(x) for x in _IV]
    inner1 = compress(B, iv, _bytes_to_words(keyblock(0x36)))
    pad2 = mb + [_const_byte(0x80)] + [_const_byte(0)] * (64 - 40 - 1 - 8) + \
        [_const_byte(b) for b in (104 * 8).to_bytes(8, "big")]
    inner = compress(B, inner1, _bytes_to_words(pad2))
    outer1 = compress(B, iv, _bytes_to_words(keyblock(0x5C)))
    ib = []
    for w in inner:  # digest words -> bytes (big-endian), MSB first per byte
        msb = list(reversed(w))
        ib += [msb[8 * j:8 * j + 8] for j in range(4)]
    pad3 = ib + [_const_byte(0x80)] + [_const_byte(0)] * (64 - 32 - 1 - 8) + \
        [_const_byte(b) for b in (96 * 8).to_bytes(8, "big")]
    out = compress(B, outer1, _bytes_to_words(pad3))
    ob = []
    for w in out:
        msb = list(reversed(w))
        ob += [msb[8 * j:8 * j + 8] for j in range(4)]
    pack(ob[0:16], pub_vars[3])
    pack(ob[16:32], pub_vars[4])
    cred = sum(b.v << (255 - i) for i, b in enumerate(x for byte in ob for x in byte))
    if cred.to_bytes(32, "big") != credential:
        # the relation does not hold: the packed public credential is still the
        # attestation's, so the system is unsatisfiable (a forged credential)
        B.vals[pub_vars[3]] = int.from_bytes(credential[:16], "big")
        B.vals[pub_vars[4]] = int.from_bytes(credential[16:], "big")


def build_tx(key: bytes, att104: bytes) -> Builder:
    """One transaction's circuit + assignment from its attest key and its
    104-B attestation (obj_hash | id_com | domain | credential, crypto.hpp:70-82)."""
    B = Builder(N_PUB_PER_TX)
    hmac_tx(B, key, att104[0:32], att104[64:72], att104[72:104], list(range(1, 6)))
    return B


def constraints_per_tx() -> int:
    return len(build_tx(bytes(32), bytes(104)).A)


def _structure(b0: Builder, T: int):
    """CSR matrices of T copies of one tx's circuit, with variables ONE | 5T
    public inputs | T x (the tx's private variables)."""
    from .r1cs import Csr
    P = len(b0.vals) - 1 - N_PUB_PER_TX  # private variables per tx
    npub = N_PUB_PER_TX * T
    vars_ = 1 + npub + T * P
    mats = []
    for M in (b0.A, b0.B, b0.C):
        rp, cols, vals = [0], [], []
        for row in M:
            for c, v in sorted(row.items()):
                cols.append(c)
                vals.append(v)
            rp.append(len(cols))
        mats.append((np.array(rp, np.int64), np.array(cols, np.int64), vals))
    out = []
    m0 = len(b0.A)
    for rp, cols, vals in mats:
        nnz = len(cols)
        vb = np.frombuffer(b"".join(v.to_bytes(32, "little") for v in vals) or b"", np.uint8)
        allc, allv, allr = [], [], [np.zeros(1, np.int64)]
        for t in range(T):
            c = cols.copy()
            pub = (c >= 1) & (c <= N_PUB_PER_TX)
            prv = c > N_PUB_PER_TX
            c[pub] = 1 + N_PUB_PER_TX * t + (c[pub] - 1)
            c[prv] = 1 + npub + P * t + (c[prv] - 1 - N_PUB_PER_TX)
            allc.append(c)
            allv.append(vb)
            allr.append(rp[1:] + nnz * t)
        out.append(Csr(np.concatenate(allr).astype(np.uint64),
                       np.concatenate(allc).astype(np.uint32), np.concatenate(allv)))
    return m0 * T, vars_, npub, out[0], out[1], out[2], P


def chunk(keys: list[bytes], atts: list[bytes]):
    """T transactions -> (m, vars, n_pub, A, B, C as r1cs.Csr, z) with
    variables ONE | 5T public inputs | T x (the tx's private variables); z is
    evaluated here on the host (the checker for the GPU witness program)."""
    T = len(keys)
    builders = [build_tx(k, a) for k, a in zip(keys, atts)]
    m, vars_, npub, A, B, Cm, P = _structure(builders[0], T)
    z = [1] + [0] * npub + [0] * (T * P)
    for t, b in enumerate(builders):
        z[1 + N_PUB_PER_TX * t:1 + N_PUB_PER_TX * (t + 1)] = b.vals[1:1 + N_PUB_PER_TX]
        z[1 + npub + P * t:1 + npub + P * (t + 1)] = b.vals[1 + N_PUB_PER_TX:]
    za = np.frombuffer(b"".join(v.to_bytes(32, "little") for v in z), np.uint8).copy()
    return m, vars_, npub, A, B, Cm, za


def chunk_r1cs(T: int):
    """The constraint system of a T-tx chunk alone (-> m, vars, n_pub, A, B, C):
    the circuit's shape does not depend on the transactions."""
    return _structure(build_tx(bytes(32), bytes(104)), T)[:6]


_OPS = {"KEY": 1, "MSG": 2, "AND": 3, "XOR": 4, "CHP": 5, "CH": 6, "MAJP": 7, "MAJ": 8,
        "ADD": 9, "SUMBIT": 10}


class WitnessProgram:
    """The circuit compiled to a GPU witness program (csrc/witprog.cu): the
    builder's value ops in creation order, uploaded once; `run_dev` writes a
    chunk's full assignment z from its attest keys and attestations."""

    def __init__(self, ctx=None):
        import ctypes as C
        from . import _native as N
        self.ctx = ctx or N.context()
        b = build_tx(bytes(32), bytes(104))
        add_ord: dict[int, int] = {}
        ops = np.zeros((len(b.prog), 4), np.uint32)
        addtab: list[int] = []
        for i, op in enumerate(b.prog):
            code, dst = _OPS[op[0]], op[1]
            if op[0] == "ADD":
                add_ord[dst] = len(add_ord)
                ops[i] = (code << 24 | add_ord[dst], len(addtab), len(op[2]), op[3])
                addtab.extend(op[2])
            elif op[0] == "SUMBIT":
                ops[i] = (code << 24 | dst, add_ord[op[2]], op[3], 0)
            else:
                ops[i] = [code << 24 | dst] + list(op[2:]) + [0] * (3 - len(op[2:]))
        self.n_vars = len(b.var_slot)
        self.n_slots = b.nslot
        at = np.array(addtab or [0], np.uint32)
        vs = np.array(b.var_slot, np.uint32)
        h = C.c_void_p()
        self.ctx.call("acegpu_witprog_create", ops.reshape(-1), len(b.prog), at, len(addtab),
                      len(add_ord), vs, self.n_vars, self.n_slots, C.byref(h))
        self.h = h
        self.n_ops = len(b.prog)

    def run(self, keys: list[bytes], atts: list[bytes]) -> np.ndarray:
        T = len(keys)
        z = np.zeros(32 * (1 + N_PUB_PER_TX * T + T * self.n_vars), np.uint8)
        k = np.frombuffer(b"".join(keys), np.uint8).copy()
        a = np.frombuffer(b"".join(atts), np.uint8).copy()
        self.ctx.call("acegpu_witprog_run", self.h, k, a, T, z)
        return z

    def run_dev(self, d_keys, key_stride: int, d_atts, T: int, d_z, stream=None, Tc: int = 0):
        """T transactions in chunks of Tc (0: one chunk), assignments back to back."""
        self.ctx.call("acegpu_witprog_run_dev", stream, self.h, d_keys, key_stride, d_atts, T, Tc,
                      d_z)

    def close(self):
        from . import _native as N
        if self.h:
            N.lib().acegpu_witprog_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
