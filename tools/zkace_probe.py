"""One ZK-ACE HMAC-circuit chunk proof (20 txs, ~2.07 M constraints) after a
warm-up — for ncu launch lists of the general-R1CS path. Not a benchmark."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_10242_b200 import _native as N, groth16, r1cs, zkace_circuit as Z  # noqa: E402

ctx = N.context(0)
fb, revs, rix = bench.canonical_block_host(64, ctx)
import numpy as np  # noqa: E402
T = int(os.environ.get("ZK_T", "20"))
keys_all = np.zeros(32 * T, np.uint8)
doms = fb.atts[:104 * T].reshape(T, 104)[:, 64:72].copy()
rv = revs.reshape(-1, 32)[rix[:T]].copy()
ctx.call("acegpu_derive_attest_keys", rv, doms, T, keys_all)
m, V, npub, A, B, Cm, z = Z.chunk([keys_all[32 * i:32 * i + 32].tobytes() for i in range(T)],
                                  [fb.atts[104 * i:104 * i + 104].tobytes() for i in range(T)])
rc = r1cs.R1CS(m, V, npub, A, B, Cm, ctx=ctx)
pk = groth16.ProvingKey.from_r1cs(rc, ctx=ctx)
dz = torch.from_numpy(z).cuda()
out = torch.zeros(544, dtype=torch.uint8, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    ctx.call("acegpu_g16_prove_z_dev", sp, pk.h, dz.data_ptr(), None, out.data_ptr(),
             out.data_ptr() + 256, out.data_ptr() + 512)
torch.cuda.synchronize()
print("ok", out[:8].tolist())
