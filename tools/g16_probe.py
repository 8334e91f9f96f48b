"""One paper-size Groth16 chunk proof (after setup + one warm-up) — for ncu
launch lists of the Groth16 kernels. Not a benchmark (see bench.py)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_10242_b200 import _native as N, bn254, groth16  # noqa: E402

ctx = N.context(0)
T, K = int(os.environ.get("G16_T", groth16.PAPER_T)), int(os.environ.get("G16_K", groth16.PAPER_K))
pk = groth16.ProvingKey(T, K, ctx=ctx)
w = torch.from_numpy(bn254.random_scalars(T, 1)).cuda()
pub = torch.from_numpy(bn254.random_scalars(T, 2)).cuda()
out = torch.zeros(256, dtype=torch.uint8, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    pk.prove_dev(w.data_ptr(), pub.data_ptr(), out.data_ptr(), stream=sp)
torch.cuda.synchronize()
print("ok", out[:8].tolist())
