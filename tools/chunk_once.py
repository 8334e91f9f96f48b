"""A paper-size Groth16 chunk proved twice (device-resident inputs): for ncu
launch lists (take the second proof's launches)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_10242_b200 import _native as N, groth16  # noqa: E402

ctx = N.context(0)
pk = groth16.ProvingKey(groth16.PAPER_T, groth16.PAPER_K, ctx=ctx)
rng = np.random.default_rng(1)
w = torch.from_numpy(rng.integers(0, 256, 32 * pk.T, dtype=np.uint8)).cuda()
pub = torch.from_numpy(rng.integers(0, 256, 32 * pk.T, dtype=np.uint8)).cuda()
out = torch.empty(544, dtype=torch.uint8, device="cuda")
for _ in range(2):
    pk.prove_dev(w.data_ptr(), pub.data_ptr(), out.data_ptr())
    torch.cuda.synchronize()
print("ok")
