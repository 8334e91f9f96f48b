"""The slowest ranks of ONE proof for the 100k block split over 2 / 4 / 8 GPUs,
measured alone on one GPU (bench.bench_one_proof_split)."""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2603_10242_b200 import _native as N  # noqa: E402

ctx = N.context(0)
fb, revs, rix = bench.canonical_block_host(100000, ctx)
print(json.dumps(bench.bench_one_proof_split(ctx, 0, fb, revs, rix, worlds=(2, 4, 8))))
