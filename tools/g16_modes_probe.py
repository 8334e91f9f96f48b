"""Groth16 chunk alone, the 100k block in chunks, the one-proof block and
its 8-rank split (slowest rank), in one process: for A/B of prover changes
(ACEGPU_G16_RADIX3=0 keeps power-of-two domains)."""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2603_10242_b200 import _native as N, bn254, groth16  # noqa: E402

ctx = N.context(0)
fq_rate = bn254.mul_rate(0, ctx)
pk = groth16.ProvingKey(groth16.PAPER_T, groth16.PAPER_K, ctx=ctx)
ch = bench.bench_groth16(ctx, 0, fq_rate, pk)
fb, revs, rix = bench.canonical_block_host(100000, ctx)
blk = bench.run_groth16_block(ctx, 0, fb, revs, rix, 0, 1, steps=3, warmup=1, pk=pk)
pk.close()
one = bench.bench_groth16_single_block(ctx, 0, fb, revs, rix, e2e_steps=1)
split = bench.bench_one_proof_split(ctx, 0, fb, revs, rix, worlds=(8,))
print(json.dumps({"domain": pk.domain, "chunk_ms": ch["chunk_prove_ms"],
                  "block_100k_chunked_ms": blk["latency_ms"],
                  "per_chunk_pipelined_ms": blk["pipelined_ms_per_chunk_on_rank"],
                  "one_proof_ms": one["latency_ms"], "one_proof_domain": one["domain"],
                  "split8_slowest_ms": split["8"]["slowest_rank_ms"],
                  "split8": {k: split["8"][k]["ms"] for k in split["8"] if k.startswith("rank")}}))
