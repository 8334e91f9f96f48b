"""the reference's own simulator (`simulate normal`,
proj/src/sim.cpp, run unmodified through oracle/_ref/ace_sim_b200) with the
CostModel (proj/include/ace/sim.hpp:41-57) set from this B200 prover's
MEASURED costs, next to the paper's modelled prover.

Inputs: a committed bench line (profiles/r02_bench_line*.json, a 1-GPU run).
Cost models:
  paper          the reference defaults (15 ms per 128-proof batch, 45 ms
                 aggregation, 0.5 ms FC check)
  b200_mock      hash-proof mode: the whole block's attest+prove+FC in one
                 batch = the measured e2e block latency; FC check = measured
  b200_groth16   Groth16 chunk proofs on ONE B200: 1,024 txs per batch at the
                 measured pipelined per-chunk time; FC check = the measured
                 batched pairing verification of the chunk proofs
  b200_groth16_x8  the same per-GPU chunk time with 8 GPUs proving
                 concurrently (8 x 1,024 txs per batch): a PROJECTION from the
                 1-GPU measurement, not an 8-GPU measurement
at the simulator's default load (2,000 txs per 400 ms slot) and at the
32,000-TPS load of BASELINE configs[4] (12,800 txs per slot).

    python tools/sim_b200.py [profiles/r02_bench_line_a.json]
Writes profiles/r02_sim_normal.json.
"""
from __future__ import annotations

import glob
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SIM = os.path.join(ROOT, "oracle", "_ref", "ace_sim_b200")


def load_line(path: str) -> dict:
    with open(path) as f:
        lines = [ln for ln in f.read().splitlines() if ln.startswith("{")]
    return json.loads(lines[-1])


def run(overrides: dict) -> dict:
    args = [SIM, "normal"] + [f"{k}={int(round(v))}" for k, v in overrides.items()]
    out = subprocess.run(args, capture_output=True, text=True, timeout=600)
    summary = json.loads(out.stdout.strip().splitlines()[-1])
    summary["rc"] = out.returncode
    h = [x for x in summary["hard_after_publish_us"] if x]
    summary["hard_after_publish_ms_median"] = statistics.median(h) / 1e3 if h else None
    return summary


def main() -> None:
    path = sys.argv[1] if len(sys.argv) > 1 else sorted(
        glob.glob(os.path.join(ROOT, "profiles", "r02_bench_line*.json")))[-1]
    line = load_line(path)
    g16 = line["groth16_block_100000"]
    mock_e2e_ms = line["latency_ms"]["e2e"]
    mock_fc_ms = line["phase1a_and_verify"]["verify_fc_mock_ms"]
    chunk_ms = g16["pipelined_ms_per_chunk_on_rank"]
    g16_fc_ms = g16["verify_fc"]["ms"]
    models = {
        "paper": {},
        "b200_mock": {"proof_parallelism": line["config"]["n_tx"],
                      "proof_batch_us": mock_e2e_ms * 1e3, "aggregation_us": 0,
                      "fc_verify_us": mock_fc_ms * 1e3},
        "b200_groth16": {"proof_parallelism": 1024, "proof_batch_us": chunk_ms * 1e3,
                         "aggregation_us": 0, "fc_verify_us": g16_fc_ms * 1e3},
        "b200_groth16_x8": {"proof_parallelism": 8 * 1024, "proof_batch_us": chunk_ms * 1e3,
                            "aggregation_us": 0, "fc_verify_us": g16_fc_ms * 1e3},
    }
    res = {"source_bench_line": os.path.relpath(path, ROOT),
           "simulator": "reference proj/src/sim.cpp via oracle/_ref/ace_sim_b200 (unmodified)",
           "note": "aggregation_us = 0 for the B200 models: the tree over chunk proofs and the FC "
                   "are inside the measured block / chunk times. b200_groth16_x8 is a projection "
                   "from the 1-GPU per-chunk time.",
           "runs": {}}
    for load in (2000, 12800):
        for name, ov in models.items():
            r = run(dict(ov, txs_per_slot=load))
            res["runs"][f"{name}@{load}tx"] = {k: r[k] for k in (
                "hard", "blocks", "assertions_ok", "proving_us_per_block", "proof_batch_us",
                "proof_parallelism", "fc_verify_us", "hard_after_publish_ms_median",
                "hard_after_publish_us")}
    out = os.path.join(ROOT, "profiles", "r02_sim_normal.json")
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    for k, v in res["runs"].items():
        print(f"{k:28s} hard {v['hard']}/{v['blocks']}  proving/block {v['proving_us_per_block'] / 1e3:8.1f} ms"
              f"  hard after publish (median) {v['hard_after_publish_ms_median']} ms")


if __name__ == "__main__":
    main()
