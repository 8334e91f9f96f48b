"""GPU optimal ate pairing (pairing.cuh) against the CPU oracle's pairing
(oracle/bn254_oracle.c): Fq12 values after the final exponentiation must be
identical; bilinearity and pairing checks on the GPU itself."""
import ctypes as C
import random

import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu

R = 0x30644E72E131A029B85045B68181585D2833E84879B9709143E1F593F0000001


@pytest.fixture(scope="module")
def M():
    from paper_2603_10242_b200 import _native as N
    return type("M", (), {"N": N, "ctx": N.context(0)})


def le(x):
    return (x % R).to_bytes(32, "little")


def gens():
    g1, g2 = O.buf(64), O.buf(128)
    O.oracle().bn_generator(1, g1)
    O.oracle().bn_generator(2, g2)
    return bytes(g1), bytes(g2)


def smul(g, p, k):
    o = O.buf(64 * g)
    O.oracle().bn_scalar_mul(g, O.ptr(p), O.ptr(le(k)), o)
    return bytes(o)


def gpu_pair(M, ps, qs):
    out = np.zeros(384, np.uint8)
    one = C.c_int(-1)
    a = np.frombuffer(b"".join(ps) or b"\0" * 64, np.uint8).copy()
    b = np.frombuffer(b"".join(qs) or b"\0" * 128, np.uint8).copy()
    M.ctx.call("acegpu_bn_pairing", len(ps), M.N.addr(a), M.N.addr(b), M.N.addr(out), C.byref(one))
    return out.tobytes(), one.value


def cpu_pair(ps, qs):
    o = O.buf(384)
    O.oracle().bn_pairing(C.c_uint64(len(ps)), O.ptr(b"".join(ps) or b"\0" * 64),
                          O.ptr(b"".join(qs) or b"\0" * 128), o)
    return bytes(o)


def test_pairing_matches_oracle(M):
    g1, g2 = gens()
    rng = random.Random(3)
    ps = [smul(1, g1, rng.randrange(1, R)) for _ in range(3)] + [g1]
    qs = [smul(2, g2, rng.randrange(1, R)) for _ in range(3)] + [g2]
    for k in range(len(ps)):
        got, _ = gpu_pair(M, [ps[k]], [qs[k]])
        assert got == cpu_pair([ps[k]], [qs[k]])
    got, _ = gpu_pair(M, ps, qs)
    assert got == cpu_pair(ps, qs)


def test_pairing_bilinear_and_checks(M):
    g1, g2 = gens()
    a, b = 987654321987654321, 1234567
    eab, _ = gpu_pair(M, [smul(1, g1, a)], [smul(2, g2, b)])
    assert eab == gpu_pair(M, [smul(1, g1, a * b)], [g2])[0]
    assert eab == gpu_pair(M, [g1], [smul(2, g2, a * b)])[0]
    neg = smul(1, g1, R - 1)
    assert gpu_pair(M, [g1, neg], [g2, g2])[1] == 1
    assert gpu_pair(M, [g1, g1], [g2, g2])[1] == 0
    assert gpu_pair(M, [b"\0" * 64, g1, neg], [g2, g2, g2])[1] == 1  # infinity contributes 1
    assert gpu_pair(M, [], [])[1] == 1


def rand_f12(rng):
    P = 0x30644E72E131A029B85045B68181585D97816A916871CA8D3C208C16D87CFD47
    return b"".join(rng.randrange(P).to_bytes(32, "little") for _ in range(12))


def gpu_op(M, op, x):
    a = np.frombuffer(x, np.uint8).copy()
    if len(a) < 384:
        a = np.concatenate([a, np.zeros(384 - len(a), np.uint8)])
    out = np.zeros(384, np.uint8)
    M.ctx.call("acegpu_bn_f12_op", op, M.N.addr(a), M.N.addr(out))
    return out.tobytes()


def cpu_op(op, x):
    x = x + b"\0" * (384 - len(x))
    o = O.buf(384)
    O.oracle().bn_f12_op(op, O.ptr(x), o)
    return bytes(o)


@pytest.mark.parametrize("op", [8, 7, 3, 4, 5, 6])
def test_f12_unit_ops(M, op):
    """Square, inverse, Frobenius^1,2,3 (vs plain ^p powers) and ^x (on
    cyclotomic-subgroup elements, where the GPU uses Granger-Scott squarings)."""
    rng = random.Random(op)
    for _ in range(2):
        x = rand_f12(rng)
        if op == 6:
            x = cpu_op(1, x)
        assert gpu_op(M, op, x) == cpu_op(op, x)


def test_easy_hard_parts(M):
    rng = random.Random(11)
    x = rand_f12(rng)
    e = gpu_op(M, 1, x)
    assert e == cpu_op(1, x)
    assert gpu_op(M, 2, e) == cpu_op(2, e)


def test_miller_loop_up_to_subfield_factors(M):
    g1, g2 = gens()
    p, q = smul(1, g1, 5), smul(2, g2, 7)
    mg = gpu_op(M, 9, p + q)
    mc = cpu_op(9, p + q)
    assert gpu_op(M, 1, mg) == cpu_op(1, mc)


def test_cyclotomic_square(M):
    """Granger-Scott squaring on elements after the easy part (cyclotomic
    subgroup) equals the plain square."""
    rng = random.Random(21)
    for _ in range(3):
        c = gpu_op(M, 1, rand_f12(rng))
        assert gpu_op(M, 11, c) == cpu_op(8, c)


def test_pairing_g2_generator_multiples(M):
    g1, g2 = gens()
    ps = [smul(1, g1, k) for k in (2, 3, 11)]
    qs = [smul(2, g2, k) for k in (5, 7, 13)]
    assert gpu_pair(M, ps, qs)[0] == cpu_pair(ps, qs)


def test_eip197_vector_on_gpu(M):
    """The EIP-197 ecPairing vector (tests/golden/eip196_197.json, jeff1)
    checks to 1 on the GPU pairing, and a changed statement does not."""
    import eip_vectors as E
    for v in E.load()["ecpairing"]:
        n, a, b, exp = E.ecpairing(v)
        ps = [a[64 * k:64 * k + 64] for k in range(n)]
        qs = [b[128 * k:128 * k + 128] for k in range(n)]
        f, one = gpu_pair(M, ps, qs)
        assert one == exp and f == cpu_pair(ps, qs)
        d1 = O.buf(64)
        O.oracle().bn_point_double(1, O.ptr(ps[0]), d1)
        assert gpu_pair(M, [bytes(d1)] + ps[1:], qs)[1] == 0
