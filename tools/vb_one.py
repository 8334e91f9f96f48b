"""One variable-base MSM (G1 2^26 or G2 2^24) after a warm-up: for ncu launch lists."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import vb_probe as P  # noqa: E402

group = int(sys.argv[1]) if len(sys.argv) > 1 else 1
logn = int(sys.argv[2]) if len(sys.argv) > 2 else 26
base = P.gen(group, 1 << 18)
n = 1 << logn
pts = base.repeat(n // (1 << 18))
sc = torch.randint(0, 256, (n, 32), dtype=torch.uint8, device="cuda")
sc[:, 31] &= 0x1F
h = C.c_void_p()
P.ctx.call("acegpu_bn_msm_prepare_vb", group, pts.data_ptr(), n, 1, 0, C.byref(h))
out = torch.empty(64 * group, dtype=torch.uint8, device="cuda")
for _ in range(2):
    P.ctx.call("acegpu_bn_msm_run_dev", None, h, sc.data_ptr(), out.data_ptr())
torch.cuda.synchronize()
print("ok")
