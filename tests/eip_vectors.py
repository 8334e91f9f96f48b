"""EIP-196 / EIP-197 precompile vectors (tests/golden/eip196_197.json) in the
oracle encodings: 32-B little-endian standard-form coordinates, G1 = x | y,
G2 = x.c0 | x.c1 | y.c0 | y.c1. Test-side helper only."""
import json
import os

_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "eip196_197.json")


def load() -> dict:
    with open(_PATH) as f:
        return json.load(f)


def words(hexs: str) -> list[bytes]:
    b = bytes.fromhex(hexs)
    return [b[i:i + 32] for i in range(0, len(b), 32)]


def g1(x_be: bytes, y_be: bytes) -> bytes:
    return x_be[::-1] + y_be[::-1]


def g2(xc1_be: bytes, xc0_be: bytes, yc1_be: bytes, yc0_be: bytes) -> bytes:
    return xc0_be[::-1] + xc1_be[::-1] + yc0_be[::-1] + yc1_be[::-1]


def ecadd(v: dict) -> tuple[bytes, bytes, bytes]:
    w, e = words(v["input"]), words(v["expected"])
    return g1(w[0], w[1]), g1(w[2], w[3]), g1(e[0], e[1])


def ecmul(v: dict) -> tuple[bytes, bytes, bytes]:
    """-> (point, scalar as 32-B LE, expected point)."""
    w, e = words(v["input"]), words(v["expected"])
    return g1(w[0], w[1]), w[2][::-1], g1(e[0], e[1])


def ecpairing(v: dict) -> tuple[int, bytes, bytes, int]:
    """-> (pairs, concatenated G1s, concatenated G2s, expected 0/1)."""
    w = words(v["input"])
    n = len(w) // 6
    a = b"".join(g1(w[6 * k], w[6 * k + 1]) for k in range(n))
    b = b"".join(g2(*w[6 * k + 2:6 * k + 6]) for k in range(n))
    return n, a, b, int.from_bytes(bytes.fromhex(v["expected"]), "big")
