"""e2e (host pinned buffers -> FC) latency of the 100k-tx block with the
single-pass vs the overlapped host pipeline. Not a benchmark (see bench.py)."""
import ctypes as C
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_10242_b200 import _native as N  # noqa: E402

ctx = N.context(0)
fb, revs, rix = bench.canonical_block_host(100000, ctx)
lib = N.lib()


def pinned(a):
    p = lib.acegpu_host_alloc(max(a.nbytes, 1))
    arr = np.ctypeslib.as_array((C.c_uint8 * max(a.nbytes, 1)).from_address(p))
    arr[:a.nbytes] = a.view(np.uint8).reshape(-1)
    return arr


hp, ho, ha, hh, hr, hx = (pinned(x) for x in (fb.payloads, fb.offs, fb.atts, fb.header, revs,
                                              rix.astype(np.uint32)))
codes = pinned(np.zeros(100000, np.uint8))
out = pinned(np.zeros(640, np.uint8))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for seg in (0, 1, 0, 1):
    ctx.call("acegpu_set_segmented", seg)
    ts = []
    for i in range(25):
        flush.fill_(i)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.call("acegpu_attest_prove_certify", hp.ctypes.data, ho.ctypes.data, ha.ctypes.data,
                 100000, hh.ctypes.data, hr.ctypes.data, 1, hx.ctypes.data, codes.ctypes.data,
                 out.ctypes.data, out.ctypes.data + 304, None, None)
        ts.append((time.perf_counter() - t0) * 1e3)
    print("segmented" if seg else "single   ", f"median {statistics.median(ts[5:]):.3f} ms  "
          f"min {min(ts[5:]):.3f} ms  fc {out[304:312].tobytes().hex()}")
