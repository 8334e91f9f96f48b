"""Regenerates tests/golden/kats.json FROM THE REFERENCE ITSELF.

Run in the build container (needs oracle/_ref/libaceref.so, built from the
unmodified /root/reference/proj sources by ``make -C oracle ref``):

    python tests/golden/make_golden.py

Every value below is printed by the reference's own code (ref_* symbols of
oracle/ref_shim.cpp, which call straight into proj/src/*.cpp); the CPU oracle
and the CUDA path are then checked against this file. The reference's own
golden wire files (proj/tests/golden/*.hex) are not copied; their SHA-256 is
recorded so tests can check our encodings against them byte-for-byte.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_lib as O  # noqa: E402

REF_GOLDEN = "/root/reference/proj/tests/golden"


def h(b: bytes) -> str:
    return b.hex()


def main() -> None:
    R = O.ref()
    out: dict = {"source": "reference proj/src via oracle/_ref/libaceref.so"}

    # --- SHA-256 (test_sha256.cpp:31-47) and batch lengths
    sha = {}
    for name, msg in [("empty", b""), ("abc", b"abc"),
                      ("448", b"abcdbcdecdefdefgefghfghighijhijkijkljklmklmnlmnomnopnopq"),
                      ("seq65", bytes(range(65))), ("seq300", bytes(i % 251 for i in range(300)))]:
        o = O.buf(32)
        R.ref_sha256(O.ptr(msg), C.c_uint64(len(msg)), o)
        sha[name] = {"msg": msg.hex(), "digest": h(bytes(o))}
    out["sha256"] = sha

    # --- HMAC RFC 4231 / HKDF RFC 5869 TC1 (test_crypto.cpp:27-52)
    hm = []
    for key, msg in [(b"\x0b" * 20, b"Hi There"), (b"Jefe", b"what do ya want for nothing?"),
                     (b"\xaa" * 131, b"Test Using Larger Than Block-Size Key - Hash Key First")]:
        o = O.buf(32)
        R.ref_hmac_sha256(O.ptr(key), C.c_uint64(len(key)), O.ptr(msg), C.c_uint64(len(msg)), o)
        hm.append({"key": key.hex(), "msg": msg.hex(), "mac": h(bytes(o))})
    out["hmac"] = hm
    ikm, salt, info = b"\x0b" * 22, bytes(range(13)), bytes(range(0xF0, 0xFA))
    hk = []
    for L in (32, 42, 82):
        o = O.buf(L)
        R.ref_hkdf_sha256(O.ptr(ikm), C.c_uint64(22), O.ptr(salt), C.c_uint64(13), O.ptr(info),
                          C.c_uint64(10), o, C.c_uint64(L))
        hk.append({"ikm": ikm.hex(), "salt": salt.hex(), "info": info.hex(), "L": L,
                   "okm": h(bytes(o))})
    o = O.buf(32)
    R.ref_hkdf_sha256(O.ptr(ikm), C.c_uint64(22), None, C.c_uint64(0), O.ptr(info),
                      C.c_uint64(10), o, C.c_uint64(32))
    hk.append({"ikm": ikm.hex(), "salt": "", "info": info.hex(), "L": 32, "okm": h(bytes(o))})
    out["hkdf"] = hk

    # --- attestation fixture values (acceptance.cpp:35-60)
    rev = O.buf(32)
    R.ref_rev_from_seed(C.c_uint64(20240801), rev)
    rev = bytes(rev)
    idc = O.buf(32)
    R.ref_id_commitment(O.ptr(rev), O.ptr(b"\0" * 32), C.c_uint16(1), C.c_uint64(40), idc)
    key = O.buf(32)
    R.ref_derive_attest_key(O.ptr(rev), C.c_uint16(1), C.c_uint64(40), key)
    pay = O.buf(154)
    R.ref_make_transfer_payload(O.ptr(b"\x01" * 32), O.ptr(b"\x02" * 32), C.c_uint64(10),
                                C.c_uint64(0), O.ptr(b"\0" * 32), pay)
    att = O.buf(104)
    R.ref_generate_attestation(O.ptr(rev), pay, C.c_uint64(154), C.c_uint16(1), C.c_uint64(40),
                               idc, att)
    p0 = O.buf(289)
    R.ref_prove_tx(pay, C.c_uint64(154), att, p0)
    out["fixture"] = {"rev": h(rev), "id_com": h(bytes(idc)), "attest_key": h(bytes(key)),
                      "payload0": h(bytes(pay)), "attestation0": h(bytes(att)),
                      "proof0": h(bytes(p0))}

    # --- canonical blocks: root digest, SHA(root proof), SHA(FC)
    blocks = {}
    for n in (0, 1, 2, 3, 5, 7, 100, 1000, 1024, 1025, 4097, 6250, 16384, 100000):
        fb = O.canonical_block(n)
        root, lv, pr = O.ref_prove_block(fb)
        fc = O.ref_prove_and_certify(fb)
        codes = O.ref_attest_codes(fb)
        blocks[str(n)] = {"levels": lv, "pairs": pr, "root_digest": h(root[256:288]),
                          "root_kind": root[288], "root_proof_sha": h(O.sha256(root[:256])),
                          "fc": h(fc), "fc_sha": h(O.sha256(fc)),
                          "header_sha": h(O.sha256(fb.header)),
                          "accept": int((codes == 0).sum())}
    out["canonical_blocks"] = blocks

    # --- forged mix (config 1 variant): per-tx codes from verify_attestation_full
    forged = {}
    for n in (64, 1024):
        fb = O.forge(O.canonical_block(n))
        codes = O.ref_attest_codes(fb)
        forged[str(n)] = {"codes": bytes(codes).hex(),
                          "inputs_sha": h(O.sha256(fb.payloads.tobytes() + fb.atts.tobytes()))}
    out["forged"] = forged

    # --- multi-user block (config 3 shape at small n) and test_prover make_block
    mu = O.multi_user_block(1000, 16)
    out["multi_user_1000"] = {"fc": h(O.ref_prove_and_certify(mu)),
                              "accept": int((O.ref_attest_codes(mu) == 0).sum())}
    tp = {}
    for n in (7, 9, 12, 16):
        tp[str(n)] = h(O.ref_prove_and_certify(O.prover_test_block(n)))
    out["prover_test_blocks"] = tp

    # --- witness + threshold scheme (test_prover.cpp:176-263)
    th = O.sha256(pay)
    w = O.buf(256)
    R.ref_build_witness(key, O.ptr(th), w)
    master = b"\x5a" * 32
    ct = O.buf(256)
    R.ref_scheme_encapsulate(C.c_uint(4), O.ptr(master), O.ptr(th), w, C.c_uint64(256), ct)
    shares = []
    for j in range(3):
        s = O.buf(32)
        R.ref_scheme_share_value(C.c_uint(4), O.ptr(master), O.ptr(th), C.c_uint(j), s)
        shares.append(h(bytes(s)))
    masks = {str(n): [int(R.ref_scheme_share_mask(C.c_uint(n), C.c_uint(v))) for v in range(n)]
             for n in (1, 2, 3, 4, 7, 10, 21)}
    out["witness"] = {"tx_hash": h(th), "witness": h(bytes(w)), "master": h(master),
                      "ciphertext_n4": h(bytes(ct)), "shares_n4": shares, "share_masks": masks,
                      "thresholds": {str(n): int(R.ref_scheme_threshold(C.c_uint(n)))
                                     for n in (1, 2, 3, 4, 5, 7, 10, 21, 64)}}

    # --- the reference's own golden wire files, by hash
    gold = {}
    if os.path.isdir(REF_GOLDEN):
        for f in sorted(os.listdir(REF_GOLDEN)):
            if f.endswith(".hex"):
                raw = open(os.path.join(REF_GOLDEN, f)).read().strip()
                gold[f] = {"sha256_of_hex_text": hashlib.sha256(raw.encode()).hexdigest(),
                           "bytes": len(raw) // 2}
    out["reference_golden_files"] = gold

    with open(os.path.join(HERE, "kats.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", os.path.join(HERE, "kats.json"))


if __name__ == "__main__":
    main()
