"""Live time of one paper-size Groth16 chunk proof (bench.bench_groth16's
chunk_prove_ms) and the 16,384-tx block: for A/B of library variants."""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2603_10242_b200 import _native as N, bn254, groth16  # noqa: E402

ctx = N.context(0)
fq_rate = bn254.mul_rate(0, ctx)
pk = groth16.ProvingKey(groth16.PAPER_T, groth16.PAPER_K, ctx=ctx)
ch = bench.bench_groth16(ctx, 0, fq_rate, pk)
fb, revs, rix = bench.canonical_block_host(16384, ctx)
blk = bench.run_groth16_block(ctx, 0, fb, revs, rix, 0, 1, steps=3, warmup=1, pk=pk)
print(json.dumps({"chunk_ms": ch["chunk_prove_ms"], "block16k_ms": blk["latency_ms"]}))
