"""A/B probe for BN254 arithmetic variants: G1 MSM 2^20, G2 MSM 2^18, one
paper-size Groth16 chunk, and a 16-proof batched verify, device-resident,
CUDA events. Run once per library build (swap lib/libacegpu.so between runs).
Not a benchmark line (see bench.py)."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_10242_b200 import _native as N, bn254  # noqa: E402


def timed(fn, k=5):
    s = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(k)]
    for a, b in evs:
        a.record(s)
        fn()
        b.record(s)
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in evs)


def msm_ms(ctx, group, n):
    sp = torch.cuda.current_stream().cuda_stream
    pts = bn254.scalar_muls(group, bn254.generator(group), bn254.random_scalars(n, 1), ctx)
    bases = bn254.MsmBases(group, pts, n, ctx=ctx)
    sc = torch.from_numpy(bn254.random_scalars(n, 2)).cuda()
    res = torch.zeros(64 * group, dtype=torch.uint8, device="cuda")
    ms = timed(lambda: bases.run_dev(sc.data_ptr(), res.data_ptr(), sp), k=3)
    out = res.cpu().numpy().tobytes().hex()[:32]
    bases.close()
    return ms, out


def ntt_ms(ctx, L=22):
    sp = torch.cuda.current_stream().cuda_stream
    n = 1 << L
    x = torch.from_numpy(bn254.random_scalars(n, 22)).cuda()
    ctx.call("acegpu_bn_convert_dev", sp, 1, x.data_ptr(), n, 1)
    y = torch.empty_like(x)
    f = timed(lambda: ctx.call("acegpu_bn_ntt_dev", sp, x.data_ptr(), y.data_ptr(), L, 0, 0))
    return f, y[:16].cpu().numpy().tobytes().hex()


def main():
    ctx = N.context(0)
    r = {"tag": os.environ.get("AB_TAG", "")}
    r["ntt_2^22_ms"], r["ntt_digest"] = ntt_ms(ctx)
    r["g1_2^20_ms"], r["g1_digest"] = msm_ms(ctx, 1, 1 << 20)
    r["g2_2^18_ms"], r["g2_digest"] = msm_ms(ctx, 2, 1 << 18)
    from paper_2603_10242_b200 import groth16
    pk = groth16.ProvingKey(groth16.PAPER_T, groth16.PAPER_K, ctx=ctx)
    g = bench.bench_groth16(ctx, 0, bn254.mul_rate(0, ctx), pk, reps=3)
    r["chunk_ms"] = g["chunk_prove_ms"]
    pk.close()
    print(json.dumps(r))


if __name__ == "__main__":
    main()
