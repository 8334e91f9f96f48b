"""One Groth16 proof for a whole block (the paper's FC): setup of a
block-size key (T = n txs x K = 1,400 constraints, domain 2^28 for 100k),
prove_block through the host C-ABI call, FC verification by pairings.
Prints setup / prove / verify times and device memory."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2603_10242_b200 import _native as N, groth16, prover, wire  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
K = 1400
ctx = N.context(0)
fb, revs, rix = bench.canonical_block_host(n, ctx)
wit = bench.make_witnesses(fb, revs, rix, ctx)
wfb = wire.FlatBlock(fb.payloads, fb.offs, fb.atts, np.frombuffer(bytes(fb.header), np.uint8).copy())


def mem():
    f, t = torch.cuda.mem_get_info(0)
    return f"{(t - f) / 1e9:.1f} GB used of {t / 1e9:.1f}"


print("before setup:", mem(), flush=True)
t0 = time.perf_counter()
pk = groth16.ProvingKey(n, K, ctx=ctx)
print(f"setup T={n} K={K}: {time.perf_counter() - t0:.1f} s; {mem()}", flush=True)
for i in range(reps):
    t0 = time.perf_counter()
    codes, proof, fc, cps = pk.prove_block(wfb, wit, revs, rix)
    print(f"prove_block {i}: {(time.perf_counter() - t0) * 1e3:.0f} ms; accepted "
          f"{int((codes == 0).sum())}; {mem()}", flush=True)
t0 = time.perf_counter()
v = pk.verify_finality_certificate(fc, wfb, cps)
print(f"verify_fc: {v} in {(time.perf_counter() - t0) * 1e3:.1f} ms; proofs {len(cps)} B", flush=True)
pk.close()
