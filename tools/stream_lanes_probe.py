import sys, os, json
sys.path.insert(0, "/root/repo")
import bench
from paper_2603_10242_b200 import _native as N
ctx = N.context(0)
for lanes in (2, 4, 6, 8, 4):
    r = bench.bench_stream(ctx, 0, blocks=30, n=12800, lanes=lanes)
    print(lanes, round(r["sustained_tx_per_s"] / 1e6, 1), {k: round(v, 3) for k, v in r["block_latency_ms"].items()}, r["fc_matches_single_call"])
