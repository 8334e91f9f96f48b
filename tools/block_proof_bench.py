import sys, json; sys.path.insert(0, ".")
import bench
from paper_2603_10242_b200 import _native as N
ctx = N.context(0)
fb, revs, rix = bench.canonical_block_host(100000, ctx)
r = bench.bench_groth16_single_block(ctx, 0, fb, revs, rix)
print(json.dumps({k: r[k] for k in ("setup_s_once", "device_mem_gb_after_setup", "latency_ms", "e2e_ms", "verify_fc", "verify_fc_ms")}))
