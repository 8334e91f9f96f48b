"""One NTT 2^22 and one G1 MSM 2^20 (after one warm-up each) — for ncu launch
lists / captures of the BN254 kernels. Not a benchmark (see bench.py)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_10242_b200 import _native as N, bn254  # noqa: E402

ctx = N.context(0)
sp = torch.cuda.current_stream().cuda_stream
L = 22
x = torch.from_numpy(bn254.random_scalars(1 << L, 22)).cuda()
ctx.call("acegpu_bn_convert_dev", sp, 1, x.data_ptr(), 1 << L, 1)
y = torch.empty_like(x)
for _ in range(2):
    ctx.call("acegpu_bn_ntt_dev", sp, x.data_ptr(), y.data_ptr(), L, 0, 0)
n = 1 << int(os.environ.get("MSM_LOG", "20"))
pts = bn254.scalar_muls(1, bn254.generator(1), bn254.random_scalars(n, 1), ctx)
bases = bn254.MsmBases(1, pts, n, ctx=ctx)
sc = torch.from_numpy(bn254.random_scalars(n, 2)).cuda()
res = torch.zeros(64, dtype=torch.uint8, device="cuda")
for _ in range(2):
    bases.run_dev(sc.data_ptr(), res.data_ptr(), sp)
torch.cuda.synchronize()
print("ok", res[:8].tolist())
