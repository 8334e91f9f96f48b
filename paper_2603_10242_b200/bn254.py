"""BN254 host API over libacegpu (north-star additions: Fr NTT, G1/G2 MSM).

Host-side values are 32-B little-endian canonical integers (numpy uint8
arrays). Device-resident `_dev` variants take torch CUDA tensors holding
Montgomery-form data. No CPU fallback.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N

P = 0x30644E72E131A029B85045B68181585D97816A916871CA8D3C208C16D87CFD47
R = 0x30644E72E131A029B85045B68181585D2833E84879B9709143E1F593F0000001
FQ, FR = 0, 1


def to_arr(vals) -> np.ndarray:
    return np.frombuffer(b"".join(int(v).to_bytes(32, "little") for v in vals), np.uint8).copy()


def from_arr(a: np.ndarray) -> list[int]:
    b = a.tobytes()
    return [int.from_bytes(b[i:i + 32], "little") for i in range(0, len(b), 32)]


def random_scalars(n: int, seed: int) -> np.ndarray:
    """n uniform canonical Fr elements (< 2^253 < r) as n x 32 B."""
    rng = np.random.default_rng(seed)
    raw = rng.integers(0, 2**63, size=(n, 4), dtype=np.uint64)
    raw[:, 3] &= (1 << 61) - 1
    return raw.view(np.uint8).reshape(-1).copy()


def field_batch(field: int, op: int, a: np.ndarray, b: np.ndarray | None = None, ctx=None):
    ctx = ctx or N.context()
    n = len(a) // 32
    out = np.zeros_like(a)
    ctx.call("acegpu_bn_field_batch", field, op, a, b if b is not None else a, n, out)
    return out


def ntt(data: np.ndarray, logn: int, inverse: bool = False, coset: bool = False, ctx=None):
    """In place on a host array (standard form)."""
    ctx = ctx or N.context()
    ctx.call("acegpu_bn_ntt", data, logn, int(inverse), int(coset))
    return data


def ntt_dev(d_in, d_out, logn: int, inverse=False, coset=False, stream=None, ctx=None):
    ctx = ctx or N.context()
    ctx.call("acegpu_bn_ntt_dev", stream, d_in, d_out, logn, int(inverse), int(coset))


def generator(group: int) -> np.ndarray:
    if group == 1:
        g = np.zeros(64, np.uint8)
        g[0], g[32] = 1, 2
        return g
    xs = [10857046999023057135944570762232829481370756359578518086990519993285655852781,
          11559732032986387107991004021392285783925812861821192530917403151452391805634,
          8495653923123431417604973247489272438418190587263600148770280649306958101930,
          4082367875863433681332203403145435568316851327593401208105741076214120093531]
    return to_arr(xs)


def scalar_muls(group: int, base: np.ndarray, scalars: np.ndarray, ctx=None) -> np.ndarray:
    ctx = ctx or N.context()
    n = len(scalars) // 32
    out = np.zeros(64 * group * n, np.uint8)
    ctx.call("acegpu_bn_scalar_muls", group, base, scalars, n, out)
    return out


class MsmBases:
    """Fixed bases prepared once (all 16 window shifts resident on device)."""

    def __init__(self, group: int, points, n: int, on_device: bool = False, ctx=None):
        self.ctx = ctx or N.context()
        self.group, self.n = group, n
        h = C.c_void_p()
        self.ctx.call("acegpu_bn_msm_prepare", group, points, n, int(on_device), C.byref(h))
        self.h = h

    def run(self, scalars: np.ndarray) -> np.ndarray:
        out = np.zeros(64 * self.group, np.uint8)
        self.ctx.call("acegpu_bn_msm_run", self.h, scalars, out)
        return out

    def run_dev(self, d_scalars, d_out, stream=None):
        self.ctx.call("acegpu_bn_msm_run_dev", stream, self.h, d_scalars, d_out)

    def close(self):
        if self.h:
            N.lib().acegpu_bn_msm_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def msm_params(ctx=None) -> tuple[int, int]:
    """(window bits c, windows per scalar) of the compiled Pippenger MSM."""
    ctx = ctx or N.context()
    c, w = C.c_int(), C.c_int()
    ctx.call("acegpu_bn_msm_params", C.byref(c), C.byref(w))
    return c.value, w.value


def imad_peak(ctx=None) -> float:
    ctx = ctx or N.context()
    v = C.c_double()
    ctx.call("acegpu_imad_peak", C.byref(v))
    return v.value


def mul_rate(field: int, ctx=None) -> float:
    ctx = ctx or N.context()
    v = C.c_double()
    ctx.call("acegpu_bn_mul_rate", field, C.byref(v))
    return v.value
