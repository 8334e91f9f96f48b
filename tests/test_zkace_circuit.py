"""The ZK-ACE credential circuit (paper_2603_10242_b200/zkace_circuit.py) on
the CPU: its assignment satisfies every row exactly when the attestation's
credential is HMAC-SHA256(attest key, obj_hash || domain) — the reference's
witness_matches_tx relation (proj/src/prover.cpp:190-197) — checked against
the reference-derived fixture (tests/golden/kats.json) and Python's hmac."""
import hashlib
import hmac
import json
import os
import random

from paper_2603_10242_b200 import zkace_circuit as Z
from paper_2603_10242_b200.bn254 import R


def _unsatisfied(B) -> int:
    z = B.vals

    def ev(lc):
        return sum(c * z[k] for k, c in lc.items()) % R
    return sum(1 for a, b, c in zip(B.A, B.B, B.C) if ev(a) * ev(b) % R != ev(c))


def test_circuit_accepts_the_reference_fixture_and_rejects_forgeries():
    kats = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "kats.json")))
    fx = kats["fixture"]
    key = bytes.fromhex(fx["attest_key"])
    att = bytes.fromhex(fx["attestation0"])
    # the fixture's credential is HMAC(key, obj_hash || domain) (crypto.cpp:129-139)
    assert hmac.new(key, att[0:32] + att[64:72], hashlib.sha256).digest() == att[72:104]
    B = Z.build_tx(key, att)
    assert _unsatisfied(B) == 0
    assert len(B.A) == Z.constraints_per_tx()
    assert 90_000 < len(B.A) < 120_000  # ~4 SHA-256 compressions
    # public inputs: obj_hash halves, domain, credential halves (big-endian packs)
    assert B.vals[1:6] == [int.from_bytes(att[0:16], "big"), int.from_bytes(att[16:32], "big"),
                           int.from_bytes(att[64:72], "big"), int.from_bytes(att[72:88], "big"),
                           int.from_bytes(att[88:104], "big")]
    rng = random.Random(1)
    for off in (72, 100, 0, 64):  # credential, obj_hash, domain bytes
        bad = bytearray(att)
        bad[off] ^= 1 << rng.randrange(8)
        assert _unsatisfied(Z.build_tx(key, bytes(bad))) > 0
    wrong_key = bytes([key[0] ^ 1]) + key[1:]
    assert _unsatisfied(Z.build_tx(wrong_key, att)) > 0
