"""Two device-resident steps of the 100k-tx hash-proof block (bench.py's
step: attestation + prove_block + FC) — for ncu captures of the leaf / level
kernels of one full step. Not a benchmark (see bench.py)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_10242_b200 import _native as N, shard  # noqa: E402

ctx = N.context(0)
n = int(os.environ.get("MOCK_N", "100000"))
fb, revs, rix = bench.canonical_block_host(n, ctx)
db = shard.DeviceBlock.upload(fb, 0, n, revs, rix, device=0)
codes = torch.zeros(n, dtype=torch.uint8, device="cuda")
out = torch.zeros(640, dtype=torch.uint8, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    ctx.call("acegpu_attest_prove_certify_dev", sp, db.payloads.data_ptr(), db.offs.data_ptr(),
             db.atts.data_ptr(), n, db.header.data_ptr(), db.revs.data_ptr(),
             db.revs.numel() // 32, db.rev_index.data_ptr(), codes.data_ptr(), out.data_ptr(),
             out.data_ptr() + 304)
torch.cuda.synchronize()
print("ok", out[:8].tolist())
