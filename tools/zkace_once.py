"""The real-circuit block prover on a 32-tx block (two 16-tx chunks), run
twice: for ncu launch lists of one chunk proof."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2603_10242_b200 import _native as N, shard, zkace  # noqa: E402

ctx = N.context(0)
n = 32
fb, revs, rix = bench.canonical_block_host(n, ctx)
wit = bench.make_witnesses(fb, revs, rix, ctx)
zp = zkace.ZkAceProver(16, ctx=ctx)
db = shard.DeviceBlock.upload(fb, 0, n, revs, rix, device=0)
db.witnesses = torch.from_numpy(wit).cuda()
codes = torch.zeros(n, dtype=torch.uint8, device="cuda")
for _ in range(2):
    zp.prove_block(db, n, codes=codes)
    torch.cuda.synchronize()
zp.close()
print("ok")
