"""Throughput probe (tools only): 16 paper-size chunk proofs back to back on
one proving key (the block path's pipelining) vs 8 + 8 on two independent
contexts / keys proving concurrently from two host threads. If the second
is much faster, the block path wants more chunks in flight."""
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_10242_b200 import _native as N, bn254, groth16  # noqa: E402

T, K = groth16.PAPER_T, groth16.PAPER_K
trap = groth16.deterministic_trapdoor(ctx=N.context(0))
ctxs = [N.Context(0), N.Context(0)]
pks = [groth16.ProvingKey(T, K, trap, c) for c in ctxs]
w = torch.from_numpy(bn254.random_scalars(T, 1)).cuda()
pub = torch.from_numpy(bn254.random_scalars(T, 2)).cuda()
outs = [torch.zeros(256, dtype=torch.uint8, device="cuda") for _ in range(2)]
streams = [torch.cuda.Stream() for _ in range(2)]


def run(i, n):
    for _ in range(n):
        pks[i].prove_dev(w.data_ptr(), pub.data_ptr(), outs[i].data_ptr(),
                         stream=streams[i].cuda_stream)


for _ in range(2):
    run(0, 2)
    run(1, 2)
torch.cuda.synchronize()
t0 = time.perf_counter()
run(0, 16)
torch.cuda.synchronize()
one = (time.perf_counter() - t0) * 1e3
t0 = time.perf_counter()
th = [threading.Thread(target=run, args=(i, 8)) for i in range(2)]
for t in th:
    t.start()
for t in th:
    t.join()
torch.cuda.synchronize()
two = (time.perf_counter() - t0) * 1e3
print(f"16 chunks one key: {one:.1f} ms ({one / 16:.2f} per chunk); two keys 8+8 concurrent: "
      f"{two:.1f} ms ({two / 16:.2f} per chunk); same proof: {bool((outs[0] == outs[1]).all())}")
