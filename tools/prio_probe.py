"""Chunk prove time under each ACEGPU_G16_PRIO stream-priority setting (tools
only; one process per setting: the priorities are read at key setup)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, os, json
sys.path.insert(0, %r)
import bench
from paper_2603_10242_b200 import _native as N, bn254, groth16
ctx = N.context(0)
pk = groth16.ProvingKey(groth16.PAPER_T, groth16.PAPER_K, ctx=ctx)
r = bench.bench_groth16(ctx, 0, bn254.mul_rate(0, ctx), pk, reps=5)
print(json.dumps({"prio": os.environ.get("ACEGPU_G16_PRIO"), "chunk_ms": r["chunk_prove_ms"]}))
''' % ROOT
for p in sys.argv[1:] or ["ab", "n", "nab", "h", "bl", "none", "abh"]:
    out = subprocess.run([sys.executable, "-c", CODE], env=dict(os.environ, ACEGPU_G16_PRIO=p),
                         capture_output=True, text=True, timeout=300)
    print(out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:], flush=True)
