"""calibrate the reference simulator's CostModel
(proj/include/ace/sim.hpp:41-57) from measured B200 latencies, so
`simulate normal` reports hard-finality timing for this prover instead of the
paper's modelled 15 ms per 128-proof batch.

Writes profiles/sim_costmodel_b200.json with, per proof mode, the CostModel
fields (proof_batch_us for proof_parallelism = 128 txs, aggregation_us,
fc_verify_us, attest_check_us_per_tx) plus the raw measurements, and prints
the C++ initialiser a maintainer pastes into SimConfig::cost. Run on a B200:

    python tools/calibrate_sim.py
"""
from __future__ import annotations

import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> None:
    import torch

    import bench
    from paper_2603_10242_b200 import _native as N, groth16, pipeline, prover, shard, wire
    ctx = N.context(0)
    n = 100_000
    fb, revs, rix = bench.canonical_block_host(n, ctx)

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e6)
        return statistics.median(ts)

    # mock mode: the whole Phase-2 step (attestation + proofs + tree + FC) per block
    step_us = timed(lambda: prover.attest_prove_certify(fb, revs, rix, ctx=ctx))
    fc = prover.attest_prove_certify(fb, revs, rix, ctx=ctx).fc
    verify_us = timed(lambda: prover.verify_finality_certificate(fc, fb, ctx=ctx))
    reg = pipeline.IdentityRegistry()
    reg.add(fb.atts[32:64].tobytes())
    light_us = timed(lambda: pipeline.attest_check_light_batch(fb, reg, 40, ctx=ctx))
    mock = {
        "proof_parallelism": 128,
        "proof_batch_us": step_us * 128 / n,
        "aggregation_us": 0.0,  # the tree runs inside the step above
        "fc_verify_us": verify_us,
        "attest_check_us_per_tx": light_us / n,
        "measured": {"block_txs": n, "attest_prove_certify_us": step_us,
                     "verify_fc_us": verify_us, "light_check_batch_us": light_us},
    }

    # Groth16 mode: one paper-size chunk (1,024 txs) per proof batch of 1,024
    pk = groth16.ProvingKey(groth16.PAPER_T, groth16.PAPER_K, ctx=ctx)
    try:
        fb16, revs16, rix16 = bench.canonical_block_host(16384, ctx)
        r = bench.run_groth16_block(ctx, 0, fb16, revs16, rix16, 0, 1, steps=1, warmup=1, pk=pk)
        chunk = bench.bench_groth16(ctx, 0, 42.5e9, chunks=2, reps=2)
    finally:
        pk.close()
    g16 = {
        "proof_parallelism": 1024,
        "proof_batch_us": chunk["chunk_prove_ms"] * 1e3,
        "aggregation_us": max(0.0, r["latency_ms"] * 1e3 - 16 * chunk["chunk_prove_ms"] * 1e3),
        "fc_verify_us": r["verify_fc"]["ms"] * 1e3,
        "attest_check_us_per_tx": light_us / n,
        "measured": {"block_txs": 16384, "block_us": r["latency_ms"] * 1e3,
                     "chunk_us": chunk["chunk_prove_ms"] * 1e3},
    }
    out = {"gpu": torch.cuda.get_device_name(0), "mock": mock, "groth16": g16,
           "note": "CostModel fields of proj/include/ace/sim.hpp:41-57; times in microseconds"}
    path = os.path.join(ROOT, "profiles", "sim_costmodel_b200.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    for mode, m in (("mock", mock), ("groth16", g16)):
        print(f"// {mode}: SimConfig cfg; cfg.cost = {{...}} fields measured on {out['gpu']}")
        print(f"cfg.cost.proof_parallelism = {m['proof_parallelism']};")
        print(f"cfg.cost.proof_batch_us = {max(1, round(m['proof_batch_us']))};")
        print(f"cfg.cost.aggregation_us = {round(m['aggregation_us'])};")
        print(f"cfg.cost.fc_verify_us = {max(1, round(m['fc_verify_us']))};")
        print(f"cfg.cost.attest_check_us_per_tx = {max(0, round(m['attest_check_us_per_tx']))};")
    print("wrote", path)
    _ = (np, shard, wire)


if __name__ == "__main__":
    main()
