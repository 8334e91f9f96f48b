"""One G1 (or G2, MSM_GROUP=2) MSM of 2^MSM_LOG points, run twice after
setup — for ncu launch lists of the MSM kernels. Not a benchmark."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_10242_b200 import _native as N, bn254  # noqa: E402

ctx = N.context(0)
g, n = int(os.environ.get("MSM_GROUP", 1)), 1 << int(os.environ.get("MSM_LOG", 20))
pts = bn254.scalar_muls(g, bn254.generator(g), bn254.random_scalars(n, 1), ctx)
bases = bn254.MsmBases(g, pts, n, ctx=ctx)
sc = torch.from_numpy(bn254.random_scalars(n, 2)).cuda()
res = torch.zeros(64 * g, dtype=torch.uint8, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    bases.run_dev(sc.data_ptr(), res.data_ptr(), sp)
torch.cuda.synchronize()
print("ok", res[:8].tolist())
