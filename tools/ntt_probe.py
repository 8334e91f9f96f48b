"""Median time of the Fr NTT (forward, inverse, coset forward) per size:
tools/ntt_probe.py [L ...] (default 20 21 22)."""
import statistics
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_2603_10242_b200 import _native as N, bn254  # noqa: E402

ctx = N.context(0)
sp = torch.cuda.current_stream().cuda_stream
for L in [int(a) for a in sys.argv[1:]] or (20, 21, 22):
    x = torch.from_numpy(bn254.random_scalars(1 << min(L, 22), L)).cuda().repeat(1 << max(0, L - 22), 1)
    ctx.call("acegpu_bn_convert_dev", sp, 1, x.data_ptr(), 1 << L, 1)
    y = torch.empty_like(x)
    for inv, coset in ((0, 0), (1, 0), (0, 1)):
        for _ in range(3):
            ctx.call("acegpu_bn_ntt_dev", sp, x.data_ptr(), y.data_ptr(), L, inv, coset)
        ts = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); ctx.call("acegpu_bn_ntt_dev", sp, x.data_ptr(), y.data_ptr(), L, inv, coset); b.record(); b.synchronize()
            ts.append(a.elapsed_time(b))
        print(L, inv, coset, round(statistics.median(ts), 4), flush=True)
