"""The stand-in witness kernel at 100k txs (one-proof key) and the ZK-ACE
witness program at 1,024 txs, each run twice: for ncu --set full captures."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_10242_b200 import _native as N, zkace_circuit as Z  # noqa: E402

ctx = N.context(0)
prog = Z.WitnessProgram(ctx)
T = 1024
keys = torch.randint(0, 256, (T, 32), dtype=torch.uint8, device="cuda")
atts = torch.randint(0, 256, (T, 104), dtype=torch.uint8, device="cuda")
z = torch.empty((1 + 5 * T + T * prog.n_vars) * 32, dtype=torch.uint8, device="cuda")
for _ in range(2):
    prog.run_dev(keys.data_ptr(), 32, atts.data_ptr(), T, z.data_ptr())
torch.cuda.synchronize()
prog.close()
print("ok")
