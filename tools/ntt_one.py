"""One coset-forward Fr NTT of 2^L points (device resident) after a warm-up:
for ncu captures of the three-pass transform (L > 22)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_10242_b200 import _native as N  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 28
n = 1 << L
ctx = N.context(0)
x = torch.randint(0, 256, (n, 32), dtype=torch.uint8, device="cuda")
x[:, 31] &= 0x1F
p = x.data_ptr()
ctx.call("acegpu_bn_convert_dev", None, 1, p, n, 1)
for _ in range(2):
    ctx.call("acegpu_bn_ntt_dev", None, p, p, L, 0, 1)
torch.cuda.synchronize()
print("ok")
