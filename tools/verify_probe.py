"""16 chunk proofs of a T = 1,024-tx circuit (K = 4 constraints per tx to keep
setup short; verification cost depends on T and the proof count only), then
the batched pairing verifier twice — for ncu launch lists. Not a benchmark."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_10242_b200 import _native as N, bn254, groth16  # noqa: E402

ctx = N.context(0)
T, n = 1024, int(os.environ.get("VERIFY_N", 16))
pk = groth16.ProvingKey(T, 4, ctx=ctx)
proofs, pubs = [], []
for i in range(n):
    w, pub = bn254.random_scalars(T, 100 + i), bn254.random_scalars(T, 200 + i)
    proofs.append(pk.prove(w, pub)[0])
    pubs.append(pub.tobytes())
for _ in range(2):
    t0 = time.perf_counter()
    ok = pk.verify_batch(proofs, pubs)
    print("verify", ok, (time.perf_counter() - t0) * 1e3, "ms")
pk.close()
