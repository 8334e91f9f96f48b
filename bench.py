#!/usr/bin/env python3
"""Benchmark of the B200-native Prove phase (BASELINE.json metric: block proof
latency & proven tx/s for a 100k-tx block).

A step = the reference's Phase-2 work for one 100,000-tx block: batched full
attestation verification of every tx (crypto.cpp:141-154), prove_block
(prover.cpp:129-142) and build_finality_certificate (prover.cpp:144-156),
bit-exact with the reference (the step's FC is checked against the golden the
reference printed, tests/golden/kats.json). Workload: the acceptance fixture
canonical_block(100000) (acceptance.cpp:35-60), generated on the GPU.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

N>1 runs under torchrun: aligned 1,024-tx chunks sharded across ranks, one
NCCL all-gather of chunk roots (paper_2603_10242_b200/shard.py).
`--impl reference` times the reference's own CPU implementation
(oracle/_ref/libaceref.so, compiled from the unmodified reference sources) on
this host's cores.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_TX = 100_000
SLOT = 40


def bench_device() -> int:
    return int(os.environ.get("ACE_BENCH_DEVICE", os.environ.get("LOCAL_RANK", 0)))


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------- workload
def canonical_block_host(n: int, ctx, nonce_base: int = 0, slot: int | None = None):
    """canonical_block(n) of acceptance.cpp:35-60 built with GPU hashing:
    REV = Rev::from_seed(20240801), Domain{1,40}, id_com salt 0^32,
    tx i = transfer(0x01^32 -> 0x02^32, amount 10, nonce i). The sustained
    stream varies nonce_base (tx nonces) and the header slot per block."""
    from paper_2603_10242_b200 import _native as N, crypto, wire
    rev = crypto.Rev.from_seed(20240801)
    dom = wire.Domain(1, SLOT)
    idc = crypto.id_commitment(rev, b"\0" * 32, dom).bytes
    tmpl = np.frombuffer(wire.make_transfer_payload(b"\x01" * 32, b"\x02" * 32, 10, 0, b"\0" * 32),
                         np.uint8)
    L = len(tmpl)
    pay = np.tile(tmpl, n).reshape(n, L)
    nonces = (np.arange(n, dtype=np.uint64) + np.uint64(nonce_base)).astype(">u8")
    nonces = nonces.view(np.uint8).reshape(n, 8)
    pay[:, 2:10] = nonces
    payloads = np.zeros(n * L + 16, np.uint8)
    payloads[:n * L] = pay.reshape(-1)
    offs = (np.arange(n + 1, dtype=np.uint64) * L).astype(np.uint64)
    revs = np.frombuffer(rev.bytes(), np.uint8).copy()
    rev_index = np.zeros(n, np.uint32)
    doms = np.tile(np.frombuffer(dom.encode(), np.uint8), n)
    ids = np.tile(np.frombuffer(idc, np.uint8), n)
    atts = crypto.generate_attestations(payloads, offs, revs, rev_index, doms, ids, ctx)
    atts = np.concatenate([atts[:104 * n], np.zeros(8, np.uint8)])
    # header: slot 40, tx_count, tx / attest Merkle roots (wire.cpp:257-273)
    h_tx = np.zeros(32 * n, np.uint8)
    ctx.call("acegpu_sha256_varlen", N.addr(payloads), N.addr(offs), n, N.addr(h_tx))
    h_at = np.zeros(32 * n, np.uint8)
    ctx.call("acegpu_sha256_strided", N.addr(atts), 104, 104, n, N.addr(h_at))
    roots = []
    for h in (h_tx, h_at):
        out = np.zeros(32, np.uint8)
        ctx.call("acegpu_merkle_root", N.addr(h), n, N.addr(out))
        roots.append(out.tobytes())
    hdr = wire.BlockHeader(slot_number=SLOT if slot is None else slot, tx_merkle_root=roots[0],
                           attest_merkle_root=roots[1], tx_count=n).encode()
    return wire.FlatBlock(payloads, offs, atts, np.frombuffer(hdr, np.uint8).copy()), revs, rev_index


def multi_rev_block_host(n: int, users: int, ctx, slot: int = SLOT):
    """A block where tx i is attested by user i mod `users` (REV u =
    Rev::from_seed(0xACE0000 + u), crypto.cpp:28-33; id_com per user; same
    transfer payloads as canonical_block): with users = n every tx has its own
    REV, so every credential check derives its own attest key (HKDF + HMAC,
    15 compressions, crypto.cpp:141-154) — the expensive case of attestation."""
    from paper_2603_10242_b200 import crypto, wire
    revs_l = wire.sha256_many([b"rev-seed" + (0xACE0000 + u).to_bytes(8, "big")
                               for u in range(users)], ctx)
    dom = wire.Domain(1, slot)
    idcs = wire.sha256_many([r + b"\0" * 32 + dom.encode() for r in revs_l], ctx)
    tmpl = np.frombuffer(wire.make_transfer_payload(b"\x01" * 32, b"\x02" * 32, 10, 0, b"\0" * 32),
                         np.uint8)
    L = len(tmpl)
    pay = np.tile(tmpl, n).reshape(n, L)
    pay[:, 2:10] = np.arange(n, dtype=np.uint64).astype(">u8").view(np.uint8).reshape(n, 8)
    payloads = np.zeros(n * L + 16, np.uint8)
    payloads[:n * L] = pay.reshape(-1)
    offs = (np.arange(n + 1, dtype=np.uint64) * L).astype(np.uint64)
    revs = np.frombuffer(b"".join(revs_l), np.uint8).copy()
    rev_index = (np.arange(n) % users).astype(np.uint32)
    doms = np.tile(np.frombuffer(dom.encode(), np.uint8), n)
    ids = np.frombuffer(b"".join(idcs), np.uint8).reshape(users, 32)[rev_index].reshape(-1).copy()
    atts = crypto.generate_attestations(payloads, offs, revs, rev_index, doms, ids, ctx)
    atts = np.concatenate([atts[:104 * n], np.zeros(8, np.uint8)])
    from paper_2603_10242_b200 import _native as N
    h_tx = np.zeros(32 * n, np.uint8)
    ctx.call("acegpu_sha256_varlen", N.addr(payloads), N.addr(offs), n, N.addr(h_tx))
    h_at = np.zeros(32 * n, np.uint8)
    ctx.call("acegpu_sha256_strided", N.addr(atts), 104, 104, n, N.addr(h_at))
    roots = []
    for h in (h_tx, h_at):
        out = np.zeros(32, np.uint8)
        ctx.call("acegpu_merkle_root", N.addr(h), n, N.addr(out))
        roots.append(out.tobytes())
    hdr = wire.BlockHeader(slot_number=slot, tx_merkle_root=roots[0], attest_merkle_root=roots[1],
                           tx_count=n).encode()
    return wire.FlatBlock(payloads, offs, atts, np.frombuffer(hdr, np.uint8).copy()), revs, rev_index


def bench_many_revs(ctx, dev: int, n: int, with_ref: bool, reps: int = 10) -> dict:
    """The 100k-tx hash-proof step on a block with one REV per tx (every
    attestation derives its own key), device-resident, L2 flushed, CUDA events;
    the FC is compared with the reference's own CPU path on the same block."""
    import torch
    from paper_2603_10242_b200 import shard
    fb, revs, rix = multi_rev_block_host(n, n, ctx)
    db = shard.DeviceBlock.upload(fb, 0, n, revs, rix, device=dev)
    codes = torch.zeros(n, dtype=torch.uint8, device=f"cuda:{dev}")
    out = torch.zeros(640, dtype=torch.uint8, device=f"cuda:{dev}")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")
    s = torch.cuda.current_stream()

    def step():
        ctx.call("acegpu_attest_prove_certify_dev", s.cuda_stream, db.payloads.data_ptr(),
                 db.offs.data_ptr(), db.atts.data_ptr(), n, db.header.data_ptr(),
                 db.revs.data_ptr(), db.revs.numel() // 32, db.rev_index.data_ptr(),
                 codes.data_ptr(), out.data_ptr(), out.data_ptr() + 304)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ts = []
    for i in range(reps):
        flush.fill_(i & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        step()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.mean(ts)
    fc = out[304:632].cpu().numpy().tobytes()
    res = {"n_tx": n, "revs": n, "ms_per_step": ms, "tx_per_s": n / (ms * 1e-3), "reps": reps,
           "accepted": int((codes == 0).sum().item()),
           "compressions_per_tx_attestation": 15,
           "note": "every tx attested by its own REV: per-REV HKDF + HMAC on the GPU "
                   "(keytab + credential kernels)"}
    so = os.path.join(ROOT, "oracle", "_ref", "libaceref.so")
    if with_ref and os.path.exists(so):
        ref = C.CDLL(so)
        ref.ref_attest_prove_certify.restype = C.c_double
        rc = np.zeros(n, np.uint8)
        rfc = np.zeros(328, np.uint8)
        vp = lambda x: x.ctypes.data_as(C.c_void_p)  # noqa: E731
        us = ref.ref_attest_prove_certify(vp(fb.payloads), vp(fb.offs), vp(fb.atts), C.c_uint32(n),
                                          vp(np.ascontiguousarray(fb.header)), vp(revs), vp(rix),
                                          vp(rc), vp(rfc))
        res["reference_cpu_ms"] = us / 1e3
        res["fc_matches_reference"] = rfc.tobytes() == fc
        res["codes_match_reference"] = bool((rc == codes.cpu().numpy()).all())
    return res


def golden_fc(n: int) -> str | None:
    try:
        with open(os.path.join(ROOT, "tests", "golden", "kats.json")) as f:
            return json.load(f)["canonical_blocks"].get(str(n), {}).get("fc")
    except OSError:
        return None


# --------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------ reference
def run_reference(args, rank: int, world: int) -> None:
    """The reference's own CPU Prove path (oracle/_ref) on this host's cores."""
    if rank != 0:
        return
    so = os.path.join(ROOT, "oracle", "_ref", "libaceref.so")
    line = {"impl": "reference", "metric": METRIC, "unit": "tx/s", "higher_is_better": True}
    if not os.path.exists(so):
        line["unavailable"] = "oracle/_ref/libaceref.so not built (needs /root/reference at build time)"
        print(json.dumps(line), flush=True)
        return
    ref = C.CDLL(so)
    ref.ref_attest_prove_certify.restype = C.c_double
    ref.ref_threads.restype = C.c_uint
    threads = ref.ref_threads()
    # Inputs: the same canonical block, generated by the reference itself.
    n = args.n_tx
    from_ = b"\x01" * 32
    rev = (C.c_uint8 * 32)()
    ref.ref_rev_from_seed(C.c_uint64(20240801), rev)
    idc = (C.c_uint8 * 32)()
    ref.ref_id_commitment(rev, (C.c_uint8 * 32)(), C.c_uint16(1), C.c_uint64(SLOT), idc)
    pay = np.zeros(n * 154 + 16, np.uint8)
    atts = np.zeros(n * 104 + 8, np.uint8)
    p = (C.c_uint8 * 154)()
    a = (C.c_uint8 * 104)()
    zero = (C.c_uint8 * 32)()
    to = (C.c_uint8 * 32)(*([2] * 32))
    fr = (C.c_uint8 * 32)(*from_)
    for i in range(n):
        ref.ref_make_transfer_payload(fr, to, C.c_uint64(10), C.c_uint64(i), zero, p)
        pay[154 * i:154 * i + 154] = np.frombuffer(p, np.uint8)
        ref.ref_generate_attestation(rev, p, C.c_uint64(154), C.c_uint16(1), C.c_uint64(SLOT), idc, a)
        atts[104 * i:104 * i + 104] = np.frombuffer(a, np.uint8)
    offs = (np.arange(n + 1, dtype=np.uint64) * 154).astype(np.uint64)
    txr, atr = (C.c_uint8 * 32)(), (C.c_uint8 * 32)()
    vp = lambda x: x.ctypes.data_as(C.c_void_p)
    ref.ref_tx_merkle_root(vp(pay), vp(offs), vp(atts), C.c_uint32(n), txr, atr)
    import struct
    hdr = (struct.pack(">Q", SLOT) + b"\0" * 64 + bytes(txr) + bytes(atr) + b"\0" * 64
           + struct.pack(">QI", 0, n) + b"\0" * 44)
    hdr = np.frombuffer(hdr, np.uint8).copy()
    revs = np.frombuffer(bytes(rev), np.uint8).copy()
    rix = np.zeros(n, np.uint32)
    codes = np.zeros(n, np.uint8)
    fc = np.zeros(328, np.uint8)
    times = []
    for s in range(args.warmup + args.steps):
        us = ref.ref_attest_prove_certify(vp(pay), vp(offs), vp(atts), C.c_uint32(n), vp(hdr),
                                          vp(revs), vp(rix), vp(codes), vp(fc))
        if s >= args.warmup:
            times.append(us / 1e3)
    ms = statistics.mean(times)
    g = golden_fc(n)
    line.update({
        "value": n / (ms / 1e3), "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": workload_config(n, world),
        "cpu_baseline": {"value": n / (ms / 1e3), "unit": "tx/s", "cores": threads,
                         "kind": "reference",
                         "sample": f"{args.steps} timed x full {n}-tx block (after {args.warmup} warm-up)"},
        "e2e": {"value": n / (ms / 1e3), "unit": "tx/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "parity": {"fc_matches_golden": (fc.tobytes().hex() == g) if g else None,
                   "accepted": int((codes == 0).sum())},
    })
    print(json.dumps(line), flush=True)


METRIC = "proven tx/s (100k-tx block: attest + prove + FC; latency = ms_per_step)"


def workload_config(n: int, world: int) -> dict:
    return {"workload": f"canonical_block({n}) attest-then-prove + finality certificate "
                        f"(BASELINE configs[3], mock-proof mode bit-exact with the reference)",
            "n_tx": n, "chunk": 1024 if world > 1 else None,
            "parallelism": f"chunk-sharded x{world}" if world > 1 else "single GPU",
            "l2": "flushed (256 MiB write) before every timed step"}


# ------------------------------------------------------------------ ours
def run_ours(args, rank: int, world: int) -> None:
    import torch
    import torch.distributed as dist
    from paper_2603_10242_b200 import _native as N, shard

    dev = bench_device()
    torch.cuda.set_device(dev)
    ctx = N.context(dev)
    n = args.n_tx
    t0 = time.time()
    fb, revs, rev_index = canonical_block_host(n, ctx)
    log(f"[rank {rank}] block generated in {time.time() - t0:.2f}s")
    parts = shard.partition(n, world, shard.LOG2_CHUNK) if world > 1 else [(0, n)]
    start, count = parts[rank]
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    # ---- device-resident inputs (value leg)
    db = shard.DeviceBlock.upload(fb, start, count, revs, rev_index, device=dev)
    codes = torch.zeros(max(count, 1), dtype=torch.uint8, device=f"cuda:{dev}")
    out = torch.zeros(640, dtype=torch.uint8, device=f"cuda:{dev}")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")
    be = shard.GpuBackend(ctx)

    def step():
        if world == 1:
            ctx.call("acegpu_attest_prove_certify_dev", sptr, db.payloads.data_ptr(),
                     db.offs.data_ptr(), db.atts.data_ptr(), n, db.header.data_ptr(),
                     db.revs.data_ptr(), db.revs.numel() // 32, db.rev_index.data_ptr(),
                     codes.data_ptr(), out.data_ptr(), out.data_ptr() + 304)
            return out[:289], out[304:632]
        return shard.prove_sharded(db, n, rank, world, shard.LOG2_CHUNK, be, codes=codes)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    # ---- parity of the step's output with the reference-derived golden
    proof, fc = step()
    torch.cuda.synchronize()
    g = golden_fc(n)
    fc_hex = fc.cpu().numpy().tobytes().hex()
    acc_t = (codes[:count] == 0).sum().to(torch.int64).reshape(1)
    if world > 1:  # verdicts of the whole block
        import torch.distributed as dist
        dist.all_reduce(acc_t)
    acc = int(acc_t.item())
    parity = {"fc_matches_golden": (fc_hex == g) if g else None, "accepted": acc,
              "fc_sha256_prefix": None}

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    clocks = ClockSampler(dev)
    l0 = ctx.launches
    with clocks:
        barrier()
        for i in range(args.steps):
            flush.fill_(i & 0xFF)  # evict the 126 MB L2 (inputs are 26 MB)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        barrier()
        launches = ctx.launches - l0
        step_ms = [a.elapsed_time(b) for a, b in ev]
        ms = statistics.mean(step_ms)
        if world > 1:
            t = torch.tensor([ms], device=f"cuda:{dev}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())

        # ---- phase split + roofline of the dominant kernel (1 GPU pipeline)
        phase = None
        if world == 1:
            ctx.call("acegpu_set_phase_timing", 1)
            ph = []
            for i in range(max(5, args.steps // 2)):
                flush.fill_(i & 0xFF)
                step()
                v = (C.c_float * 3)()
                ctx.call("acegpu_phase_times", v)
                ph.append(list(v))
            ctx.call("acegpu_set_phase_timing", 0)
            phase = [statistics.mean(p[j] for p in ph) for j in range(3)]

        # ---- e2e: host pinned buffers through the public C-ABI call
        e2e_ms, h2d, d2h = run_e2e(args, ctx, fb, revs, rev_index, rank, world, start, count,
                                   be, dev)
    peak = C.c_double()
    ctx.call("acegpu_sha256_peak", C.byref(peak))
    peak_cps = peak.value
    lat = C.c_double()
    ctx.call("acegpu_sha256_probe", 1, 32, 512, C.byref(lat))
    lat_us = lat.value / 512 * 1e6  # one warp's chained compression latency
    bn = None
    g16 = {}
    g16_roof = None
    if not args.no_bn254:
        # north star: the Groth16 block path at every N (BASELINE configs[2], [3]),
        # one proving key (9 GB, resident) for all of it
        from paper_2603_10242_b200 import bn254, groth16
        msm_in = {}
        if world == 1:
            bn = bench_bn254(ctx, dev, keep=msm_in)
        fq_rate = bn["peaks"]["fq_mul_per_s"] if bn else bn254.mul_rate(0, ctx)
        t0 = time.perf_counter()
        pk = groth16.ProvingKey(groth16.PAPER_T, groth16.PAPER_K, ctx=ctx)
        setup_s = time.perf_counter() - t0
        chunk = bench_groth16(ctx, dev, fq_rate, pk)
        chunk["setup_s_once"] = setup_s
        if bn is not None:
            bn["groth16"] = chunk
        fb16, revs16, rix16 = canonical_block_host(16384, ctx)
        g16["16384"] = run_groth16_block(ctx, dev, fb16, revs16, rix16, rank, world, steps=3,
                                         warmup=1, pk=pk)
        g16["100000"] = run_groth16_block(ctx, dev, fb, revs, rev_index, rank, world, steps=3,
                                          warmup=1, pk=pk, e2e=True, verify=True)
        g16["100000"]["chunk_prove_ms_alone"] = chunk["chunk_prove_ms"]
        if world == 1:
            g16["rank_shares"] = bench_chunked_rank_shares(ctx, dev, fb, revs, rev_index, pk)
        wk = chunk["work"]
        ach = wk["fq_mul_equivalents"] / (chunk["chunk_prove_ms"] * 1e-3)
        g16_roof = {"bound": "fmaheavy issue pipe (IMAD / IMAD.HI / DFMA share it)",
                    "kernel": "Groth16 chunk (bucket accumulations dominate: G1 + G2)",
                    "achieved": ach / 1e9, "peak": fq_rate / 1e9, "unit": "G Fq-mul-equivalents/s",
                    "frac": ach / fq_rate, "work_per_chunk": wk,
                    "peak_source": "acegpu_bn_mul_rate: a chain of the library's own Fq product "
                                   "(FP64 split), same run",
                    "ncu": g16_ncu_summary()}
        if not args.no_stream:
            g16["stream"] = bench_groth16_stream(ctx, dev, pk, rank, world)
        pk.close()
        if world == 1:
            g16["zkace_hmac"] = bench_zkace_hmac_chunk(ctx, dev, fb, revs, rev_index)
            g16["zkace_block"] = bench_zkace_block(ctx, dev)
            g16["block_proof"] = bench_groth16_single_block(ctx, dev, fb, revs, rev_index)
            g16["block_proof_split"] = bench_one_proof_split(ctx, dev, fb, revs, rev_index)
        elif os.environ.get("ACE_BENCH_SHARED_GPU") != "1":
            # N GPUs: ONE proof for the block across the ranks, the real
            # exchange and gather included (max over ranks)
            try:
                g16["block_proof_dist"] = bench_one_proof_dist(ctx, dev, fb, revs, rev_index,
                                                               rank, world)
            except Exception as e:  # keep the line: record why
                g16["block_proof_dist"] = {"error": f"{type(e).__name__}: {e}"[:300]}
        if world == 1 and not args.no_cpu_baseline:
            bn["cpu_oracle"] = bn254_cpu_baseline(msm_in)

    stream = None
    if not args.no_stream:
        # config 5 on N GPUs: every rank proves its own consecutive blocks
        # (independent replicas, no collective on the data path)
        stream = bench_stream(ctx, dev)
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([stream["sustained_tx_per_s"], stream["block_latency_ms"]["p99"],
                              stream["block_latency_ms"]["max"]], dtype=torch.float64,
                             device=f"cuda:{dev}")
            tot = t[:1].clone()
            dist.all_reduce(tot)
            mx = t[1:].clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            stream["per_rank_sustained_tx_per_s"] = stream["sustained_tx_per_s"]
            stream["sustained_tx_per_s"] = float(tot.item())
            stream["block_latency_ms"]["p99"] = float(mx[0].item())
            stream["block_latency_ms"]["max"] = float(mx[1].item())
            stream["config"] += " per rank, %d ranks (aggregate = sum over ranks)" % world
    phase1a = None
    many_revs = None
    if world == 1 and not args.no_stream:
        many_revs = bench_many_revs(ctx, dev, n, with_ref=not args.no_cpu_baseline)
    if world == 1 and not args.no_stream:
        phase1a = bench_phase1a_and_verify(ctx, dev, fb, revs, rev_index,
                                           with_cpu=not args.no_cpu_baseline)

    if rank != 0:
        return
    # Work actually executed (SHA-256 compressions): leaf
    # kernel = 15 (leaf proof: payload 3 + public inputs 3 + seed 1 + expand 8;
    # the attestation's payload check reuses the payload hash) + 1 (Merkle
    # leaf) per tx. The credential HMAC (2 per tx from the cached attest-key
    # midstates: every tx of this block shares tx 0's domain, so the
    # 8-compression key derivation runs once per REV in keytab_kernel) runs in
    # credential_kernel on a side stream, overlapped with the tree levels.
    # tree = 18 per pair + 2 per Merkle pair.
    leaf_c = 16 * n
    tree_c = 18 * (n - 1) + 2 * (n - 1)
    roof = None
    if phase:
        leaf_ach = leaf_c / (phase[0] * 1e-3)
        tree_ach = tree_c / (phase[1] * 1e-3)
        # dominant kernel BY TIME: the tree levels (level_kernel, 17 launches)
        roof = {"bound": "int_alu (wide levels) / one 11-compression dependent chain per "
                         "narrow level (latency)",
                "kernel": "level_kernel (K2+K3 fused: proof tree + id_com Merkle), all levels",
                "achieved": tree_ach / 1e9, "peak": peak_cps / 1e9,
                "unit": "G SHA-256 compressions/s", "frac": tree_ach / peak_cps,
                "traffic": level_traffic_bytes(),
                "traffic_source": "ncu --set full dram__bytes_read.sum + dram__bytes_write.sum "
                                  "summed over one step's level_kernel launches, "
                                  "profiles/r01_ncu_full_levels.csv",
                "algorithmic_compressions_per_step": tree_c,
                "phase_ms": {"leaves": phase[0], "tree_levels": phase[1], "finalize": phase[2]},
                "single_warp_compression_latency_us": lat_us,
                "peak_source": "acegpu_sha256_peak register-resident microkernel, same run",
                "secondary": {
                    "kernel": "leaf_kernel (K1+K4 fused)", "achieved": leaf_ach / 1e9,
                    "frac": leaf_ach / peak_cps, "traffic": leaf_traffic_bytes(),
                    "traffic_source": "profiles/r01_ncu_full_leaf_credential_keytab.csv",
                    "algorithmic_bytes_per_launch":
                        int(fb.offs[n]) + 104 * n + 4 * n + 320 * n + 32 * n,
                    "hbm_gbs_achieved": (int(fb.offs[n]) + 104 * n + 352 * n) / (phase[0] * 1e-3) / 1e9}}
    cpu = cpu_baseline(args, n)
    cl = clocks.summary()
    line = {
        "metric": METRIC, "value": n / (ms / 1e3), "unit": "tx/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": workload_config(n, world),
        "latency_ms": {"device_resident": ms, "e2e": e2e_ms, "target_block_interval": 400.0},
        "roofline": roof, "cpu_baseline": cpu,
        "e2e": {"value": n / (e2e_ms / 1e3), "unit": "tx/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "clocks": cl, "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
        "parity": parity, "impl": "ours", "stream": stream, "phase1a_and_verify": phase1a,
        "attest_many_revs": many_revs,
        "groth16_block_100000": g16.get("100000"), "groth16_block_16384": g16.get("16384"),
        "zkace_hmac_chunk": g16.get("zkace_hmac"), "zkace_block_1024": g16.get("zkace_block"),
        "groth16_chunked_rank_shares": g16.get("rank_shares"),
        "groth16_one_proof_block_100000": g16.get("block_proof"),
        "groth16_one_proof_split_ranks": g16.get("block_proof_split"),
        "groth16_one_proof_block_dist": g16.get("block_proof_dist"),
        "groth16_stream": g16.get("stream"),
        "groth16_roofline": g16_roof, "bn254": bn,
    }
    if world > 1 and os.environ.get("ACE_BENCH_SHARED_GPU"):
        line["config"]["ranks_share_one_gpu"] = True
        line["config"]["note"] = ("functional multi-rank run (gloo, every rank on cuda:0): "
                                  "not a scaling measurement")
    print(json.dumps(line), flush=True)


def run_e2e(args, ctx, fb, revs, rev_index, rank, world, start, count, be, dev):
    """Same step through the public API with HOST buffers: pinned inputs
    copied host->device every step, codes + proof + FC copied back."""
    import torch
    import torch.distributed as dist
    from paper_2603_10242_b200 import _native as N, shard
    n = fb.n
    lib = N.lib()

    def pinned(a: np.ndarray) -> np.ndarray:
        p = lib.acegpu_host_alloc(max(a.nbytes, 1))
        arr = np.ctypeslib.as_array((C.c_uint8 * max(a.nbytes, 1)).from_address(p))
        arr[:a.nbytes] = a.view(np.uint8).reshape(-1)
        return arr
    b0, b1 = int(fb.offs[start]), int(fb.offs[start + count])
    h_pay = pinned(fb.payloads[b0:b1 + 16])
    h_offs = pinned((fb.offs[start:start + count + 1] - b0).astype(np.uint64))
    h_atts = pinned(fb.atts[104 * start:104 * (start + count)])
    h_hdr = pinned(fb.header)
    h_revs = pinned(revs)
    h_rix = pinned(rev_index[start:start + count].astype(np.uint32))
    h_codes = pinned(np.zeros(count, np.uint8))
    h_out = pinned(np.zeros(640, np.uint8))
    h2d = (b1 - b0) + 8 * (count + 1) + 104 * count + 256 + revs.nbytes + 4 * count
    d2h = count + 289 + 328
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")
    times = []
    u64 = lambda a: a.ctypes.data

    for s in range(args.warmup + args.steps):
        flush.fill_(s & 0xFF)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        if world == 1:
            ctx.call("acegpu_attest_prove_certify", u64(h_pay), u64(h_offs), u64(h_atts), n,
                     u64(h_hdr), u64(h_revs), len(revs) // 32, u64(h_rix), u64(h_codes),
                     u64(h_out), u64(h_out) + 304, None, None)
        else:
            # rank slice host->device, shard, all-gather, combine, FC back
            stream = torch.cuda.current_stream()
            d_pay = torch.from_numpy(h_pay).to(f"cuda:{dev}", non_blocking=True)
            d_offs = torch.from_numpy(h_offs.view(np.int64)[:count + 1]).to(f"cuda:{dev}", non_blocking=True)
            d_atts = torch.from_numpy(h_atts).to(f"cuda:{dev}", non_blocking=True)
            d_hdr = torch.from_numpy(h_hdr[:256]).to(f"cuda:{dev}", non_blocking=True)
            d_revs = torch.from_numpy(h_revs[:revs.nbytes]).to(f"cuda:{dev}", non_blocking=True)
            d_rix = torch.from_numpy(h_rix[:4 * count].view(np.int32)).to(f"cuda:{dev}", non_blocking=True)
            d_codes = torch.empty(max(count, 1), dtype=torch.uint8, device=f"cuda:{dev}")
            db = shard.DeviceBlock(d_pay, d_offs, d_atts, d_hdr, count, d_revs, d_rix)
            proof, fc = shard.prove_sharded(db, n, rank, world, shard.LOG2_CHUNK, be, codes=d_codes)
            h_codes[:count] = d_codes[:count].cpu().numpy()
            h_out[:289] = proof.cpu().numpy()
            h_out[304:632] = fc.cpu().numpy()
            stream.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        if s >= args.warmup:
            times.append(dt)
    ms = statistics.mean(times)
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms, h2d, d2h


def bench_bn254(ctx, dev: int, reps: int = 5, keep: dict | None = None) -> dict:
    """BASELINE configs[1]: Fr NTT/iNTT 2^22 and G1 MSM 2^20 (device-resident,
    CUDA events on the launching stream), with the integer-pipe roofline."""
    import torch
    from paper_2603_10242_b200 import bn254
    out: dict = {}
    imad = bn254.imad_peak(ctx)
    fq_rate, fr_rate = bn254.mul_rate(0, ctx), bn254.mul_rate(1, ctx)
    out["peaks"] = {"imad_per_s": imad, "fq_mul_per_s": fq_rate, "fr_mul_per_s": fr_rate,
                    "imad_per_fq_mul_implied": imad / fq_rate,
                    "source": "acegpu_imad_peak / acegpu_bn_mul_rate microkernels, same run"}
    s = torch.cuda.current_stream()
    sp = s.cuda_stream

    def timed(fn, k=reps):
        fn()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(k)]
        for a, b in evs:
            a.record(s)
            fn()
            b.record(s)
        torch.cuda.synchronize()
        return statistics.median(x.elapsed_time(y) for x, y in evs)

    # ---- NTT 2^22
    L = 22
    n = 1 << L
    x = torch.from_numpy(bn254.random_scalars(n, 22)).to(f"cuda:{dev}")
    ctx.call("acegpu_bn_convert_dev", sp, 1, x.data_ptr(), n, 1)
    y = torch.empty_like(x)
    f_ms = timed(lambda: ctx.call("acegpu_bn_ntt_dev", sp, x.data_ptr(), y.data_ptr(), L, 0, 0))
    i_ms = timed(lambda: ctx.call("acegpu_bn_ntt_dev", sp, y.data_ptr(), y.data_ptr(), L, 1, 0))
    c_ms = timed(lambda: ctx.call("acegpu_bn_ntt_dev", sp, x.data_ptr(), y.data_ptr(), L, 0, 1))
    # butterflies + one pass-A twiddle product per element (full-size tables);
    # the j = 0 butterflies skip their product but are counted, as usual
    muls = (n // 2) * L + n
    bytes_moved = 2 * 2 * n * 32  # two passes, read + write
    out["ntt_2^22"] = {
        "forward_ms": f_ms, "inverse_ms": i_ms, "coset_forward_ms": c_ms,
        "fr_muls": muls, "achieved_fr_mul_per_s": muls / (f_ms * 1e-3),
        "frac_of_fr_mul_peak": muls / (f_ms * 1e-3) / fr_rate,
        "hbm_gbs": bytes_moved / (f_ms * 1e-3) / 1e9,
        "bound": "imad (Fr CIOS multiplications)"}
    del x, y
    # ---- G1 MSM 2^20 (bases k_i*G generated on the GPU, prepared once)
    n = 1 << 20
    ks = bn254.random_scalars(n, 1)
    pts = bn254.scalar_muls(1, bn254.generator(1), ks, ctx)
    t0 = time.perf_counter()
    bases = bn254.MsmBases(1, pts, n, ctx=ctx)
    setup_ms = (time.perf_counter() - t0) * 1e3
    sc = torch.from_numpy(bn254.random_scalars(n, 2)).to(f"cuda:{dev}")
    res = torch.zeros(64, dtype=torch.uint8, device=f"cuda:{dev}")
    m_ms = timed(lambda: bases.run_dev(sc.data_ptr(), res.data_ptr(), sp), k=3)
    c_bits, windows = bn254.msm_params(ctx)
    if keep is not None:  # the same bases / scalars for the CPU oracle's cross-check
        keep["pts"], keep["scalars"] = pts, bn254.random_scalars(n, 2)
        keep["gpu_result"] = bases.run(keep["scalars"])
        keep["ntt_in"] = bn254.random_scalars(1 << L, 22)
        d = keep["ntt_in"].copy()
        ctx.call("acegpu_bn_ntt", d, L, 0, 0)
        keep["ntt_gpu"] = d
    entries = windows * n  # nonzero signed digits (uniform scalars)
    fq_muls = entries * 10  # mixed XYZZ add = 8M + 2S (Fq-mul equivalents)
    out["msm_g1_2^20"] = {
        "ms": m_ms, "setup_ms_once_per_base_set": setup_ms, "window_bits": c_bits,
        "fq_muls_accumulate": fq_muls,
        "achieved_fq_mul_per_s": fq_muls / (m_ms * 1e-3),
        "frac_of_fq_mul_peak": fq_muls / (m_ms * 1e-3) / fq_rate,
        # madd: 8 Montgomery products (264 IMAD) + Y = R(Q - X3) - Y1 PPP as two
        # 512-bit products and one reduction (2 x 128 + 136)
        "achieved_imad_per_s": entries * (8 * 264 + 392) / (m_ms * 1e-3),
        "frac_of_imad_peak": entries * (8 * 264 + 392) / (m_ms * 1e-3) / imad,
        "bound": "imad (Fq CIOS multiplications, 264 IMAD each; lazy-reduced Y)"}
    bases.close()
    return out


def bench_stream(ctx, dev: int, blocks: int = 30, n: int = 12800, lanes: int = 8) -> dict:
    """32,000 TPS x 0.4 s = 12,800-tx blocks, >= 30
    consecutive blocks through the pipelined prover (block n+1's H2D copy and
    attestation overlap block n's tree). Host inputs are pinned once before
    the timed region; each block's H2D copy, attestation, proof, FC and the
    verdict/FC D2H are inside it. Latency = device timeline of each block
    (H2D start -> results in host memory); sustained = blocks * n / wall."""
    import torch
    from paper_2603_10242_b200 import prover as P
    from paper_2603_10242_b200.stream import PipelinedProver, pin_block
    made = [canonical_block_host(n, ctx, nonce_base=k * n, slot=SLOT + k) for k in range(blocks)]
    pins = [pin_block(fb, rv, rx) for fb, rv, rx in made]
    pp = PipelinedProver(lanes=lanes, max_tx=n, max_payload=int(made[0][0].offs[n]) + 64,
                         max_revs=1, device=dev)
    try:
        for k in range(lanes):  # warm-up: one block per lane
            pp.submit(*made[k], pinned=pins[k])
        pp.drain()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tickets = [pp.submit(*made[k], pinned=pins[k]) for k in range(blocks)]
        res = pp.drain()
        wall = time.perf_counter() - t0
        assert [r.ticket for r in res] == tickets
        lat = sorted(r.latency_ms for r in res)
        ok = all(int(r.codes.max()) == 0 for r in res)
        # parity: the first and last blocks against the single-call host API
        chk = []
        for k in (0, blocks - 1):
            fb, rv, rx = made[k]
            ref = P.attest_prove_certify(fb, rv, rx, ctx=ctx)
            chk.append(ref.fc.encode() == res[k].fc328)
        return {"config": "sustained stream: %d consecutive %d-tx blocks (32,000 TPS x 0.4 s), "
                          "%d pipelined lanes, 1 GPU" % (blocks, n, lanes),
                "sustained_tx_per_s": blocks * n / wall, "wall_ms": wall * 1e3,
                "block_latency_ms": {"p50": lat[len(lat) // 2],
                                     "p99": lat[min(len(lat) - 1, int(0.99 * len(lat)))],
                                     "max": lat[-1]},
                "block_interval_ms": 400.0, "all_accepted": ok,
                "fc_matches_single_call": all(chk)}
    finally:
        pp.close()


def chunk_work(pk, ctx) -> dict:
    """Algorithmic work of one chunk proof (Fq-mul equivalents: 10 per G1
    mixed add, 30 per G2 mixed add (3 Fq muls per Fq2 product); Fr muls of
    the 6 NTTs)."""
    from paper_2603_10242_b200 import bn254
    T = pk.T
    V, Np = pk.variables, pk.domain
    Vp = V - 1 - T
    W = bn254.msm_params(ctx)[1]
    g1_adds = W * ((V + 2) * 2 + Vp + 1 + Np)  # A, B1, L, H (coset-Lagrange, N points)
    g2_adds = W * (V + 2)                       # B2
    fr_muls = 6 * ((Np // 2) * (Np - 1).bit_length() + Np)  # 3 iNTT + 3 coset NTT
    return {"g1_mixed_adds": g1_adds, "g2_mixed_adds": g2_adds, "ntt_fr_muls": fr_muls,
            "fq_mul_equivalents": g1_adds * 10 + g2_adds * 30 + fr_muls}


def bench_groth16(ctx, dev: int, fq_rate: float, pk, reps: int = 5) -> dict:
    """BASELINE configs[2] shape: one 1,024-tx chunk x 1,400 constraints
    (1,434,625 constraints, domain 2^21) of the synthetic ZK-ACE stand-in
    circuit, proven alone (device-resident inputs, CUDA events, median of
    `reps` after one warm-up)."""
    import torch
    from paper_2603_10242_b200 import bn254
    T = pk.T
    s = torch.cuda.current_stream()
    sp = s.cuda_stream
    w = torch.from_numpy(bn254.random_scalars(T, 31)).to(f"cuda:{dev}")
    pub = torch.from_numpy(bn254.random_scalars(T, 32)).to(f"cuda:{dev}")
    out = torch.zeros(256, dtype=torch.uint8, device=f"cuda:{dev}")

    def one():
        pk.prove_dev(w.data_ptr(), pub.data_ptr(), out.data_ptr(), stream=sp)
    one()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(reps)]
    for a, b in evs:
        a.record(s)
        one()
        b.record(s)
    torch.cuda.synchronize()
    chunk_ms = statistics.median(a.elapsed_time(b) for a, b in evs)
    wk = chunk_work(pk, ctx)
    return {"txs_per_chunk": T, "constraints_per_tx": pk.K, "constraints": pk.constraints,
            "domain": pk.domain, "chunk_prove_ms": chunk_ms, "reps": reps,
            "work": wk, "frac_of_fq_mul_peak": wk["fq_mul_equivalents"] / (chunk_ms * 1e-3) / fq_rate,
            "note": "synthetic stand-in circuit (oracle/bn254_oracle.h); proofs checked "
                    "bit-exact vs the known-trapdoor oracle in tests/test_gpu_groth16.py"}


def bench_groth16_stream(ctx, dev: int, pk, rank: int, world: int, blocks: int = 30,
                         n: int = 12800) -> dict:
    """SURVEY §8d config 5 in Groth16 mode: 32,000 TPS x 0.4 s = 12,800-tx
    blocks, `blocks` consecutive blocks proven back to back (attestation +
    13 chunk proofs + tree + FC per block), sharded over `world` ranks. Every
    block's H2D runs on a copy stream ahead of the prover (block n+1's inputs
    land while block n is proven); each block's verdicts and FC come back to
    pinned host memory. Service time = the device time between consecutive
    block completions (CUDA events); sustained = blocks x n / (first H2D ->
    last FC, device time, max over ranks)."""
    import torch
    import torch.distributed as dist
    from paper_2603_10242_b200 import shard
    be = shard.G16Backend(pk, ctx)
    d = f"cuda:{dev}"
    parts = shard.partition(n, world, shard.LOG2_CHUNK) if world > 1 else [(0, n)]
    start, count = parts[rank]
    host = []
    for k in range(blocks):
        fb, rv, rx = canonical_block_host(n, ctx, nonce_base=k * n, slot=SLOT + k)
        wit = make_witnesses(fb, rv, rx, ctx)
        b0, b1 = int(fb.offs[start]), int(fb.offs[start + count])
        host.append({
            "pay": pinned_copy(np.concatenate([fb.payloads[b0:b1], np.zeros(16, np.uint8)])),
            "offs": pinned_copy((fb.offs[start:start + count + 1] - b0).astype(np.uint64)).view(np.int64),
            "atts": pinned_copy(fb.atts[104 * start:104 * (start + count)]),
            "hdr": pinned_copy(np.ascontiguousarray(fb.header, np.uint8)),
            "revs": pinned_copy(rv), "rix": pinned_copy(rx[start:start + count].astype(np.uint32)).view(np.int32),
            "wit": pinned_copy(wit[256 * start:256 * (start + count)]),
            "codes": pinned_copy(np.zeros(count, np.uint8)), "fc": pinned_copy(np.zeros(328, np.uint8))})
    comp = torch.cuda.current_stream()
    cs = torch.cuda.Stream(device=d)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def run_all(nb=blocks):
        t_up, t_done, dbs = [], [], []
        for k in range(nb):  # all H2D copies queued on the copy stream
            h = host[k]
            with torch.cuda.stream(cs):
                e0 = ev()
                e0.record(cs)
                to = lambda a: torch.from_numpy(a).to(d, non_blocking=True)  # noqa: E731
                db = shard.DeviceBlock(to(h["pay"]), to(h["offs"]), to(h["atts"]), to(h["hdr"]),
                                       count, to(h["revs"]), to(h["rix"]))
                db.witnesses = to(h["wit"])
                e1 = ev()
                e1.record(cs)
            for t in (db.payloads, db.offs, db.atts, db.header, db.revs, db.rev_index, db.witnesses):
                t.record_stream(comp)
            t_up.append((e0, e1))
            dbs.append(db)
        for k in range(nb):
            comp.wait_event(t_up[k][1])
            codes = torch.empty(max(count, 1), dtype=torch.uint8, device=d)
            proof, fc = shard.prove_sharded(dbs[k], n, rank, world, shard.LOG2_CHUNK, be, codes=codes)
            torch.from_numpy(host[k]["codes"][:count]).copy_(codes[:count], non_blocking=True)
            torch.from_numpy(host[k]["fc"]).copy_(fc, non_blocking=True)
            e2 = ev()
            e2.record(comp)
            t_done.append(e2)
        torch.cuda.synchronize()
        return t_up, t_done
    run_all(2)  # warm-up (allocations, key tables, streams)
    if world > 1:
        dist.barrier()
    t_up, t_done = run_all()
    service = [t_up[0][0].elapsed_time(t_done[0])] + \
        [t_done[k - 1].elapsed_time(t_done[k]) for k in range(1, blocks)]
    total_ms = t_up[0][0].elapsed_time(t_done[-1])
    if world > 1:
        t = torch.tensor([total_ms], device=d)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    srt = sorted(service)
    acc = sum(int((h["codes"][:count] == 0).sum()) for h in host)
    return {"config": "%d consecutive %d-tx blocks (32,000 TPS x 0.4 s), Groth16 chunk proofs, "
                      "chunk-sharded x%d" % (blocks, n, world),
            "sustained_tx_per_s": blocks * n / (total_ms * 1e-3), "total_ms": total_ms,
            "service_ms": {"p50": srt[len(srt) // 2], "p99": srt[min(len(srt) - 1, int(0.99 * len(srt)))],
                           "max": srt[-1]},
            "block_interval_ms": 400.0,
            "keeps_up_with_32k_tps": blocks * n / (total_ms * 1e-3) >= 32000,
            "accepted_on_rank": acc, "timing": "CUDA events; H2D on a copy stream ahead of the prover"}


def bench_groth16_single_block(ctx, dev: int, fb, revs, rev_index, steps: int = 3,
                               e2e_steps: int = 2) -> dict:
    """ONE Groth16 proof for the whole 100k-tx block (the paper's FC: a single
    256-B proof checked by pairings): a block-size key (T = n txs x 1,400
    constraints = 140.1 M constraints, domain 2^28; variable-base bases, no
    window tables: ~62 GB of bases + ~39 GB of per-proof vectors in HBM).
    Device-resident step (attestation + the proof + tree + FC, CUDA events)
    and e2e through acegpu_g16_prove_block (host buffers in/out, wall clock),
    then verify_finality_certificate with that one proof."""
    import torch
    from paper_2603_10242_b200 import groth16, prover, shard, wire
    n = fb.n
    torch.cuda.empty_cache()
    wit = make_witnesses(fb, revs, rev_index, ctx)
    t0 = time.perf_counter()
    pk = groth16.ProvingKey(n, groth16.PAPER_K, ctx=ctx)
    setup_s = time.perf_counter() - t0
    try:
        free, total = torch.cuda.mem_get_info(dev)
        db = shard.DeviceBlock.upload(fb, 0, n, revs, rev_index, device=dev)
        db.witnesses = torch.from_numpy(wit).to(f"cuda:{dev}")
        codes = torch.zeros(n, dtype=torch.uint8, device=f"cuda:{dev}")
        be = shard.G16Backend(pk, ctx)
        lg = (n - 1).bit_length()
        s = torch.cuda.current_stream()

        def step():
            return shard.prove_sharded(db, n, 0, 1, lg, be, codes=codes, return_roots=True)
        step()
        torch.cuda.synchronize()
        ts = []
        with ClockSampler(dev) as clocks:
            for _ in range(steps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                proof, fc, roots = step()
                b.record(s)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
        fcb = fc.cpu().numpy().tobytes()
        ms = statistics.mean(ts)
        wfb = wire.FlatBlock(fb.payloads, fb.offs, fb.atts,
                             np.frombuffer(bytes(fb.header), np.uint8).copy())
        e2e = []
        for _ in range(e2e_steps):
            t0 = time.perf_counter()
            c2, p2, fc2, cps = pk.prove_block(wfb, wit, revs, rev_index)
            e2e.append((time.perf_counter() - t0) * 1e3)
        v = pk.verify_finality_certificate(fc2, wfb, cps)  # warm-up (buffers grow once)
        vts = []
        for _ in range(3):
            t0 = time.perf_counter()
            v = pk.verify_finality_certificate(fc2, wfb, cps)
            vts.append((time.perf_counter() - t0) * 1e3)
        vms = statistics.median(vts)
        return {"n_tx": n, "proofs_per_block": 1, "constraints": pk.constraints,
                "domain": pk.domain, "setup_s_once": setup_s,
                "device_mem_gb_after_setup": (total - free) / 1e9,
                "latency_ms": ms, "latency_ms_per_step": ts, "steps": steps,
                "proven_tx_per_s": n / (ms * 1e-3), "vs_400ms_interval": ms / 400.0,
                "e2e_ms": statistics.mean(e2e), "e2e_ms_per_step": e2e,
                "e2e_fc_equal": fc2 == fcb, "accepted": int((codes == 0).sum().item()),
                "fc_bytes": 328, "proof_bytes_beside_fc": len(cps),
                "verify_fc": v.name, "verify_fc_ms": vms,
                "verify_fc_timing": "host call incl. the block's H2D, median of 3 after a warm-up",
                "fc_sha256": hashlib_sha256(fcb),
                "clocks": clocks.summary(),
                "note": "one Groth16 proof for the whole block; 1 GPU (a DIZK-style split of "
                        "the MSMs / NTTs across GPUs is not built)"}
    finally:
        pk.close()
        torch.cuda.empty_cache()


def bench_chunked_rank_shares(ctx, dev: int, fb, revs, rev_index, pk, worlds=(2, 4, 8),
                              steps: int = 3) -> dict:
    """The chunked Groth16 block's busiest rank at 2 / 4 / 8 GPUs, measured
    alone on one GPU: the rank's contiguous whole chunks (shard.partition:
    49 / 25 / 13 of the 98) — attestation verdicts, leaves, Merkle lift and
    one Groth16 proof per chunk (acegpu_g16_shard_roots_dev), CUDA events.
    Not included: the all-gather of 289 + 32 B per chunk and the 7-level
    combine + FC over the 98 roots (both on every rank, ~0.3 ms)."""
    import torch
    from paper_2603_10242_b200 import shard
    n = fb.n
    wit = make_witnesses(fb, revs, rev_index, ctx)
    be = shard.G16Backend(pk, ctx)
    s = torch.cuda.current_stream()
    out = {}
    for world in worlds:
        parts = shard.partition(n, world, shard.LOG2_CHUNK)
        r = max(range(world), key=lambda k: parts[k][1])
        start, count = parts[r]
        db = shard.DeviceBlock.upload(fb, start, count, revs, rev_index, device=dev)
        db.witnesses = torch.from_numpy(wit[256 * start:256 * (start + count)].copy()).to(f"cuda:{dev}")
        codes = torch.zeros(count, dtype=torch.uint8, device=f"cuda:{dev}")
        be.shard_roots(db, n, shard.LOG2_CHUNK, codes)
        torch.cuda.synchronize()
        ts = []
        for _ in range(steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            be.shard_roots(db, n, shard.LOG2_CHUNK, codes)
            b.record(s)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        out[str(world)] = {"busiest_rank": r, "txs": count, "chunks": -(-count // pk.T),
                           "ms": statistics.mean(ts), "ms_per_step": ts,
                           "accepted": int((codes == 0).sum().item())}
    out["note"] = ("busiest rank of the chunked 100k block at N GPUs, measured alone on one "
                   "B200 (the gather + combine of 98 roots, ~0.3 ms, not included)")
    return out


def bench_one_proof_dist(ctx, dev: int, fb, revs, rev_index, rank: int, world: int,
                         steps: int = 3, warmup: int = 1) -> dict:
    """ONE proof for the 100k block across `world` GPUs (shard.prove_one_proof
    with balanced shares): every rank holds the whole block and its split
    key; the slice exchange and the all-gather of partial records are inside
    the timed region; CUDA events, max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2603_10242_b200 import groth16, shard
    n = fb.n
    torch.cuda.empty_cache()
    wit = make_witnesses(fb, revs, rev_index, ctx)
    shares = shard.balanced_shares(world)
    t0 = time.perf_counter()
    pk = groth16.ProvingKey(n, groth16.PAPER_K, ctx=ctx, rank=rank, world=world, shares=shares)
    setup_s = time.perf_counter() - t0
    try:
        db = shard.DeviceBlock.upload(fb, 0, n, revs, rev_index, device=dev)
        db.witnesses = torch.from_numpy(wit).to(f"cuda:{dev}")
        codes = torch.zeros(n, dtype=torch.uint8, device=f"cuda:{dev}")
        s = torch.cuda.current_stream()
        for _ in range(warmup):
            shard.prove_one_proof(db, n, rank, world, pk, codes=codes)
        ts = []
        for _ in range(steps):
            dist.barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            proof, fc = shard.prove_one_proof(db, n, rank, world, pk, codes=codes)
            b.record(s)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        t = torch.tensor([statistics.mean(ts)],
                         device="cpu" if dist.get_backend() == "gloo" else f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return {"n_tx": n, "world": world, "shares": shares, "latency_ms": float(t.item()),
                "rank_ms_per_step": ts, "setup_s": setup_s, "proofs_per_block": 1,
                "vs_400ms_interval": float(t.item()) / 400.0,
                "accepted": int((codes == 0).sum().item()),
                "fc_sha256": hashlib_sha256(fc.cpu().numpy().tobytes()),
                "timing": "CUDA events, exchange + all-gather inside, max over ranks"}
    finally:
        pk.close()
        torch.cuda.empty_cache()


def bench_one_proof_split(ctx, dev: int, fb, revs, rev_index, worlds=(4, 8),
                          steps: int = 2) -> dict:
    """ONE proof for the 100k block split across `world` ranks (split keys,
    shard.prove_one_proof): rank 0's share — the block's inputs, the witness,
    the MSMs over 1/world of the bases, the coset evaluations of the H
    vectors it owns (vector k on rank k mod world: 2 of the 6 2^28 NTTs at
    world >= 3), then (a b - c)/Z and [h] on its slice, the sum of all ranks'
    partial records, s A, r B1, C, the tree and the FC — timed with CUDA
    events on ONE GPU (the other ranks' same-size shares run on their own
    GPUs). Not included: the slice exchange (3 x 2^28 x 32 B / world received
    per rank) and the all-gather of world x 384 B. Stand-ins: the slices of
    vectors rank 0 does not own are its own buffers' bytes (same sizes; the
    proof itself is checked by tests/test_gpu_groth16.py)."""
    import torch
    from paper_2603_10242_b200 import groth16, shard
    n = fb.n
    wit = make_witnesses(fb, revs, rev_index, ctx)
    db = shard.DeviceBlock.upload(fb, 0, n, revs, rev_index, device=dev)
    db.witnesses = torch.from_numpy(wit).to(f"cuda:{dev}")
    codes = torch.zeros(n, dtype=torch.uint8, device=f"cuda:{dev}")
    s = torch.cuda.current_stream()
    out = {}
    for world in worlds:
        shares = shard.balanced_shares(world)
        res = {"shares": shares}
        # the slowest ranks: an owner of one H vector (rank 0) and a rank that
        # owns none (the largest MSM share, rank world - 1)
        for rank in sorted({0, world - 1}):
            torch.cuda.empty_cache()
            t0 = time.perf_counter()
            pk = groth16.ProvingKey(n, groth16.PAPER_K, ctx=ctx, rank=rank, world=world,
                                    shares=shares)
            setup_s = time.perf_counter() - t0
            N = pk.domain
            lo, hi = shard.slice_bounds(N, rank, world, shares)
            try:
                def step():
                    own, merk = shard.one_proof_phase1(db, pk, rank, world, codes)
                    src = own if own.numel() >= 32 * N else torch.zeros(32 * N, dtype=torch.uint8,
                                                                       device=own.device)
                    sl = torch.cat([src[32 * lo:32 * hi]] * 3)  # a | b | c slice stand-ins
                    del own, src
                    part = shard.one_proof_phase2(sl, pk)
                    parts = part.repeat(world)  # stand-in for the gathered records
                    return shard.one_proof_finish(parts, world, merk, n, db.header, pk)
                step()
                torch.cuda.synchronize()
                ts = []
                for _ in range(steps):
                    a, b = (torch.cuda.Event(enable_timing=True),
                            torch.cuda.Event(enable_timing=True))
                    a.record(s)
                    step()
                    b.record(s)
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(b))
                free, total = torch.cuda.mem_get_info(dev)
                res[f"rank{rank}"] = {"ms": statistics.mean(ts), "ms_per_step": ts,
                                      "owned_vectors": bin(shard.owned_mask(rank, world)).count("1"),
                                      "setup_s": setup_s, "device_mem_gb": (total - free) / 1e9,
                                      "exchange_bytes_in": 3 * 32 * (hi - lo)}
            finally:
                pk.close()
        res["slowest_rank_ms"] = max(v["ms"] for k, v in res.items() if k.startswith("rank"))
        out[str(world)] = res
    out["note"] = ("ONE proof for the 100k block split over `world` GPUs (balanced shares): "
                   "rank 0 (owns an H vector) and rank world-1 (largest base share) each "
                   "measured alone on one B200; not included: the slice exchange and the "
                   "all-gather of world x 384 B")
    return out


def bench_zkace_block(ctx, dev: int, n: int = 1024, steps: int = 3) -> dict:
    """The block path over the REAL credential relation (zkace.py): the
    canonical n-tx block in 16-tx chunks (power of two: chunk roots are tree
    nodes), witnesses generated on the GPU from the build_witness records,
    one Groth16 proof per chunk, tree + FC; CUDA events, device-resident;
    then the batched pairing check of the chunk proofs."""
    import torch
    from paper_2603_10242_b200 import shard, zkace
    fb, revs, rix = canonical_block_host(n, ctx)
    wit = make_witnesses(fb, revs, rix, ctx)
    zp = zkace.ZkAceProver(16, ctx=ctx)
    try:
        db = shard.DeviceBlock.upload(fb, 0, n, revs, rix, device=dev)
        db.witnesses = torch.from_numpy(wit).to(f"cuda:{dev}")
        codes = torch.zeros(n, dtype=torch.uint8, device=f"cuda:{dev}")
        s = torch.cuda.current_stream()
        zp.prove_block(db, n, codes=codes)
        torch.cuda.synchronize()
        ts = []
        for _ in range(steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            proof, fc, cps = zp.prove_block(db, n, codes=codes, return_chunk_proofs=True)
            b.record(s)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = statistics.mean(ts)
        # the witness program alone: the whole block's txs in one batch
        chunks = -(-n // 16)
        z = torch.empty(chunks * zp.zbytes, dtype=torch.uint8, device=f"cuda:{dev}")
        keys = db.witnesses.view(n, 256)[:, :32].contiguous()
        at = db.atts[:104 * n].contiguous()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        zp.prog.run_dev(keys.data_ptr(), 32, at.data_ptr(), n, z.data_ptr(), stream=s.cuda_stream,
                        Tc=16)
        b.record(s)
        torch.cuda.synchronize()
        del z
        proofs = [bytes(x) for x in cps.cpu().numpy()]
        t0 = time.perf_counter()
        ok = zp.verify_chunk_proofs(proofs, fb.atts, n)
        vms = (time.perf_counter() - t0) * 1e3
        return {"n_tx": n, "txs_per_chunk": 16, "chunks": chunks,
                "constraints_per_chunk": zp.pk.constraints, "latency_ms": ms, "steps": steps,
                "latency_ms_per_step": ts, "ms_per_chunk": ms / chunks,
                "proven_tx_per_s": n / (ms * 1e-3), "witness_program_ms_block": a.elapsed_time(b),
                "witness_program_ops_per_tx": zp.prog.n_ops, "accepted": int((codes == 0).sum().item()),
                "chunk_proofs_verify": bool(ok), "verify_ms": vms,
                "fc_sha256": hashlib_sha256(fc.cpu().numpy().tobytes()),
                "note": "the real credential relation (HMAC-SHA256 in R1CS, 103,279 constraints/tx); "
                        "a 100k-tx block is 6,250 such chunks (projection: ms_per_chunk x 6,250)"}
    finally:
        zp.close()


def bench_zkace_hmac_chunk(ctx, dev: int, fb, revs, rev_index, reps: int = 3) -> dict:
    """The ZK-ACE credential relation as a real circuit (zkace_circuit.py:
    HMAC-SHA256(attest key, obj_hash || domain) == credential, ~103k
    constraints per tx) through the general R1CS Groth16 path: as many txs of
    the 100k block as fit a 2^21 domain, the assignment generated on the GPU
    by the circuit's witness program (timed separately), proven on the device
    (CUDA events), verified by the batch verifier."""
    import torch
    from paper_2603_10242_b200 import groth16, r1cs, zkace_circuit as Z
    per_tx = Z.constraints_per_tx()
    T = ((1 << 21) - 1) // (per_tx + Z.N_PUB_PER_TX)
    n = T
    keys_all = np.zeros(32 * n, np.uint8)
    doms = fb.atts[:104 * n].reshape(n, 104)[:, 64:72].copy()
    rv = revs.reshape(-1, 32)[rev_index[:n]].copy()
    ctx.call("acegpu_derive_attest_keys", rv, doms, n, keys_all)
    m, V, npub, A, B, Cm = Z.chunk_r1cs(T)
    prog = Z.WitnessProgram(ctx)
    dk = torch.from_numpy(keys_all).to(f"cuda:{dev}")
    da = torch.from_numpy(fb.atts[:104 * n].copy()).to(f"cuda:{dev}")
    dz = torch.empty(32 * V, dtype=torch.uint8, device=f"cuda:{dev}")
    s = torch.cuda.current_stream()
    prog.run_dev(dk.data_ptr(), 32, da.data_ptr(), T, dz.data_ptr(), stream=s.cuda_stream)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    prog.run_dev(dk.data_ptr(), 32, da.data_ptr(), T, dz.data_ptr(), stream=s.cuda_stream)
    b.record(s)
    torch.cuda.synchronize()
    wgen_ms = a.elapsed_time(b)
    prog.close()
    z = dz.cpu().numpy()
    rc = r1cs.R1CS(m, V, npub, A, B, Cm, ctx=ctx)
    t0 = time.perf_counter()
    pk = groth16.ProvingKey.from_r1cs(rc, ctx=ctx)
    setup_s = time.perf_counter() - t0
    try:
        out = torch.zeros(256 + 256 + 32, dtype=torch.uint8, device=f"cuda:{dev}")

        def one():
            ctx.call("acegpu_g16_prove_z_dev", s.cuda_stream, pk.h, dz.data_ptr(), None,
                     out.data_ptr(), out.data_ptr() + 256, out.data_ptr() + 512)
        one()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(reps)]
        for a, b in evs:
            a.record(s)
            one()
            b.record(s)
        torch.cuda.synchronize()
        ms = statistics.median(a.elapsed_time(b) for a, b in evs)
        proof = out[:256].cpu().numpy().tobytes()
        ok = pk.verify_batch([proof], [z.tobytes()[32:32 * (1 + npub)]])
        return {"txs": T, "constraints_per_tx": per_tx, "constraints": pk.constraints,
                "variables": V, "domain": pk.domain, "public_inputs": npub,
                "prove_ms": ms, "reps": reps, "proven_tx_per_s": T / (ms * 1e-3),
                "verifies": bool(ok), "setup_s_once": setup_s,
                "gpu_witness_program_ms": wgen_ms,
                "100k_block_chunks": -(-100_000 // T),
                "note": "relation witness_matches_tx (prover.cpp:190-197) as R1CS: 4 SHA-256 "
                        "compressions per tx; the witness is mostly bits, so the MSM scalars "
                        "are mostly 0/1"}
    finally:
        pk.close()
        rc.close()


def make_witnesses(fb, revs, rev_index, ctx) -> np.ndarray:
    """Per-tx witnesses in the reference layout build_witness(attest_key,
    tx_hash) (prover.cpp:181-188), computed on the GPU."""
    from paper_2603_10242_b200 import _native as N
    n = fb.n
    doms = fb.atts[:104 * n].reshape(n, 104)[:, 64:72].copy()
    rv = revs.reshape(-1, 32)[rev_index[:n]].copy()
    keys = np.zeros(32 * n, np.uint8)
    ctx.call("acegpu_derive_attest_keys", rv, doms, n, keys)
    txh = fb.atts[:104 * n].reshape(n, 104)[:, 0:32].copy()  # obj_hash == SHA(payload)
    wit = np.zeros(256 * n, np.uint8)
    ctx.call("acegpu_build_witness", keys, txh, n, wit)
    return wit


def pinned_copy(a: np.ndarray) -> np.ndarray:
    """A page-locked host copy (acegpu_host_alloc) of a byte array."""
    from paper_2603_10242_b200 import _native as N
    nb = max(a.nbytes, 1)
    p = N.lib().acegpu_host_alloc(nb)
    arr = np.ctypeslib.as_array((C.c_uint8 * nb).from_address(p))
    arr[:a.nbytes] = np.ascontiguousarray(a).view(np.uint8).reshape(-1)
    return arr


def run_groth16_block(ctx, dev, fb, revs, rev_index, rank, world, steps, warmup, pk,
                      e2e: bool = False, verify: bool = False):
    """The north-star block path: attestation + one Groth16 proof per aligned
    1,024-tx chunk (synthetic stand-in circuit, 1,400 constraints/tx) + the
    reference's tree rule over chunk proofs + FC, sharded over `world` ranks
    (one all-gather of chunk roots). Device-resident inputs, CUDA events on
    the launching stream, max over ranks. e2e: the same block through the
    host-buffer C-ABI call acegpu_g16_prove_block (1 rank) / the rank's host
    slice copied in + prove_sharded (N ranks), pinned buffers, every copy
    inside the timed region."""
    import torch
    import torch.distributed as dist
    from paper_2603_10242_b200 import shard
    n = fb.n
    wit = make_witnesses(fb, revs, rev_index, ctx)
    parts = shard.partition(n, world, shard.LOG2_CHUNK) if world > 1 else [(0, n)]
    start, count = parts[rank]
    db = shard.DeviceBlock.upload(fb, start, count, revs, rev_index, device=dev)
    db.witnesses = torch.from_numpy(wit[256 * start:256 * (start + count)].copy()).to(f"cuda:{dev}")
    codes = torch.zeros(max(count, 1), dtype=torch.uint8, device=f"cuda:{dev}")
    be = shard.G16Backend(pk, ctx)
    s = torch.cuda.current_stream()

    def step():
        return shard.prove_sharded(db, n, rank, world, shard.LOG2_CHUNK, be, codes=codes)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def maxed(ms):
        if world > 1:
            t = torch.tensor([ms], device=f"cuda:{dev}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        return ms
    for _ in range(warmup):
        step()
    barrier()
    times = []
    with ClockSampler(dev) as clocks:
        for _ in range(steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier()
            a.record(s)
            proof, fc = step()
            b.record(s)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
    ms = maxed(statistics.mean(times))
    chunks_total = -(-n // pk.T)
    my_chunks = -(-count // pk.T)
    fcb = fc.cpu().numpy().tobytes()
    out = {"n_tx": n, "chunks": chunks_total, "chunks_on_busiest_rank": -(-chunks_total // world),
           "latency_ms": ms, "latency_ms_per_step": times, "steps": steps, "warmup": warmup,
           "proven_tx_per_s": n / (ms * 1e-3), "vs_400ms_interval": ms / 400.0,
           "pipelined_ms_per_chunk_on_rank": statistics.mean(times) / max(my_chunks, 1),
           "accepted": accepted_total(codes[:count], world),
           "fc_sha256": hashlib_sha256(fcb), "clocks": clocks.summary(),
           "timing": "CUDA events on the launching stream, device-resident inputs, max over ranks"}
    if e2e:
        out["e2e"] = groth16_block_e2e(ctx, dev, fb, revs, rev_index, wit, rank, world, start,
                                       count, pk, be, fcb, steps, warmup)
    if verify and world == 1:
        # verify_finality_certificate in Groth16 mode: the
        # host API (block H2D, public inputs recomputed, one batched pairing
        # check of all chunk proofs, FC recomputed) vs the reference's O(N)
        # re-prove
        _, fc2, roots = shard.prove_sharded(db, n, 0, 1, shard.LOG2_CHUNK, be, codes=codes,
                                            return_roots=True)
        r = roots.cpu().numpy().tobytes()
        proofs = b"".join(r[289 * k:289 * k + 256] for k in range(chunks_total))
        fcb2 = fc2.cpu().numpy().tobytes()
        pk.verify_finality_certificate(fcb2, fb, proofs)  # warm-up
        vt = []
        for _ in range(3):
            t0 = time.perf_counter()
            verdict = pk.verify_finality_certificate(fcb2, fb, proofs)
            vt.append((time.perf_counter() - t0) * 1e3)
        out["verify_fc"] = {"ms": statistics.median(vt), "verdict": verdict.name, "reps": 3,
                            "chunk_proofs": chunks_total, "chunk_proof_bytes": 256 * chunks_total,
                            "method": "batched pairing check of %d chunk proofs (%d Miller loops, "
                                      "1 final exponentiation) + FC recompute, host buffers, "
                                      "wall clock around the host call" % (chunks_total,
                                                                          chunks_total + 3)}
    return out


def groth16_block_e2e(ctx, dev, fb, revs, rev_index, wit, rank, world, start, count, pk, be,
                      fc_expect, steps, warmup):
    """e2e of the Groth16 block: pinned host inputs -> device -> codes, root
    proof and FC back in host memory, wall clock around each step (max over
    ranks). 1 rank: ONE C-ABI call (acegpu_g16_prove_block)."""
    import torch
    import torch.distributed as dist
    from paper_2603_10242_b200 import shard
    n = fb.n
    b0, b1 = int(fb.offs[start]), int(fb.offs[start + count])
    h_pay = pinned_copy(np.concatenate([fb.payloads[b0:b1], np.zeros(16, np.uint8)]))
    h_offs = pinned_copy((fb.offs[start:start + count + 1] - b0).astype(np.uint64))
    h_atts = pinned_copy(fb.atts[104 * start:104 * (start + count)])
    h_hdr = pinned_copy(np.ascontiguousarray(fb.header, np.uint8))
    h_revs = pinned_copy(revs)
    h_rix = pinned_copy(np.ascontiguousarray(rev_index[start:start + count], np.uint32))
    h_wit = pinned_copy(wit[256 * start:256 * (start + count)])
    h_codes = pinned_copy(np.zeros(count, np.uint8))
    h_out = pinned_copy(np.zeros(640, np.uint8))
    h2d = (b1 - b0) + 8 * (count + 1) + 104 * count + 256 + revs.nbytes + 4 * count + 256 * count
    d2h = count + 289 + 328
    a = lambda x: x.ctypes.data  # noqa: E731
    times = []
    for k in range(warmup + steps):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        if world == 1:
            ctx.call("acegpu_g16_prove_block", pk.h, a(h_pay), a(h_offs), a(h_atts), n, a(h_hdr),
                     a(h_revs), len(revs) // 32, a(h_rix), a(h_wit), a(h_codes), a(h_out),
                     a(h_out) + 304, None)
        else:
            d = f"cuda:{dev}"
            to = lambda x: torch.from_numpy(x).to(d, non_blocking=True)  # noqa: E731
            db = shard.DeviceBlock(to(h_pay), to(h_offs.view(np.int64)), to(h_atts), to(h_hdr),
                                   count, to(h_revs), to(h_rix.view(np.int32)))
            db.witnesses = to(h_wit)
            codes = torch.empty(max(count, 1), dtype=torch.uint8, device=d)
            proof, fc = shard.prove_sharded(db, n, rank, world, shard.LOG2_CHUNK, be, codes=codes)
            h_codes[:count] = codes[:count].cpu().numpy()
            h_out[:289] = proof.cpu().numpy()
            h_out[304:632] = fc.cpu().numpy()
        dt = (time.perf_counter() - t0) * 1e3
        if k >= warmup:
            times.append(dt)
    ms = statistics.mean(times)
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"latency_ms": ms, "proven_tx_per_s": n / (ms * 1e-3), "steps": steps,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "fc_matches_device_path": h_out[304:632].tobytes() == fc_expect,
            "accepted": int((h_codes[:count] == 0).sum()),
            "api": "acegpu_g16_prove_block (one host-buffer C-ABI call)" if world == 1 else
                   "rank slice H2D from pinned buffers + prove_sharded (all-gather) + D2H"}


def ncu_dram_bytes(name: str, kernel: str) -> tuple[float, int] | None:
    """(sum of dram__bytes_read.sum + dram__bytes_write.sum, launches) over the
    launches of `kernel` in the committed ncu capture profiles/<name>."""
    import csv
    path = os.path.join(ROOT, "profiles", name)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    try:
        rows = list(csv.reader(open(path)))
        hdr, units = rows[0], rows[1]
        tot, cnt = 0.0, 0
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            if kernel in d.get("Kernel Name", ""):
                for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    tot += float(d[k].replace(",", "")) * scale[units[hdr.index(k)]]
                cnt += 1
        return (tot, cnt) if cnt else None
    except (OSError, KeyError, ValueError, IndexError):
        return None


def leaf_traffic_bytes() -> float | None:
    """DRAM bytes per leaf_kernel launch from the committed ncu capture."""
    r = ncu_dram_bytes("r01_ncu_full_leaf_credential_keytab.csv", "leaf_kernel")
    return r[0] / r[1] if r else None


def level_traffic_bytes() -> float | None:
    """DRAM bytes of one step's level_kernel launches (all levels), from the
    committed ncu capture of a full step (profiles/r02_ncu_levels_step.csv)."""
    r = ncu_dram_bytes("r02_ncu_levels_step.csv", "level_kernel")
    return r[0] if r else None


def g16_ncu_summary() -> dict | None:
    """fmaheavy-pipe utilisation and DRAM bytes of the Groth16 chunk's bucket
    accumulation kernels from the committed ncu capture (one chunk)."""
    import csv
    path = os.path.join(ROOT, "profiles", "r02_ncu_g16_accumulate_final.csv")
    try:
        rows = list(csv.reader(open(path)))
    except OSError:
        return None
    hdr = rows[0]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        if "accumulate" not in d.get("Kernel Name", ""):
            continue
        pick = {k: d.get(k) for k in hdr if k in (
            "gpu__time_duration.sum", "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
            "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
            "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread")}
        pick["kernel"] = d["Kernel Name"][:80]
        out.append(pick)
    return {"source": "profiles/r02_ncu_g16_accumulate_final.csv", "launches": out} if out else None


def accepted_total(codes, world: int) -> int:
    """Accepted verdicts of the whole block (summed over ranks)."""
    import torch
    t = (codes == 0).sum().to(torch.int64).reshape(1)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t)
    return int(t.item())


def hashlib_sha256(b: bytes) -> str:
    import hashlib  # a label for the output FC only (not on any measured path)
    return hashlib.sha256(b).hexdigest()


def bn254_cpu_baseline(msm_in: dict) -> dict | None:
    """Framework CPU oracle (NOT the reference: it has no BN254 code) at the
    benched sizes, all host threads: Fr NTT 2^22 and G1 MSM 2^20 on the very
    inputs the GPU ran (outputs cross-checked), plus the Groth16 chunk's CPU
    cost from the measured component rates (bounded sample: one G2 MSM 2^16
    and one NTT 2^21 are timed; the chunk's 5 MSMs and 6 NTTs are summed)."""
    so = os.path.join(ROOT, "oracle", "liboracle.so")
    if not os.path.exists(so) or "pts" not in msm_in:
        return None
    L = C.CDLL(so)
    thr = os.cpu_count() or 1
    from paper_2603_10242_b200 import bn254, groth16
    vp = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    out = {"kind": "framework CPU oracle, not reference", "cores": thr,
           "oracle": "oracle/bn254_oracle.c (plain C, 4 x 64-bit Montgomery, radix-2 NTT, "
                     "window-8 bucket MSM)"}
    d = msm_in["ntt_in"].copy()
    t0 = time.perf_counter()
    L.bn_ntt(vp(d), C.c_uint32(22), 0, 0, thr)
    out["ntt_2^22_ms"] = (time.perf_counter() - t0) * 1e3
    out["ntt_2^22_matches_gpu"] = bool(np.array_equal(d, msm_in["ntt_gpu"]))
    n = len(msm_in["scalars"]) // 32
    res = np.zeros(64, np.uint8)
    t0 = time.perf_counter()
    L.bn_msm(1, vp(msm_in["pts"]), vp(msm_in["scalars"]), C.c_uint64(n), vp(res), thr)
    out["msm_g1_2^20_ms"] = (time.perf_counter() - t0) * 1e3
    out["msm_g1_2^20_matches_gpu"] = bool(np.array_equal(res, msm_in["gpu_result"]))
    # chunk components: G2 MSM 2^16 and NTT 2^21, scaled to the chunk's sizes
    n2 = 1 << 16
    p2 = bn254.scalar_muls(2, bn254.generator(2), bn254.random_scalars(n2, 41))
    s2 = bn254.random_scalars(n2, 42)
    r2 = np.zeros(128, np.uint8)
    t0 = time.perf_counter()
    L.bn_msm(2, vp(p2), vp(s2), C.c_uint64(n2), vp(r2), thr)
    g2_ms = (time.perf_counter() - t0) * 1e3
    d21 = bn254.random_scalars(1 << 21, 43)
    t0 = time.perf_counter()
    L.bn_ntt(vp(d21), C.c_uint32(21), 0, 0, thr)
    ntt21_ms = (time.perf_counter() - t0) * 1e3
    T, K = groth16.PAPER_T, groth16.PAPER_K
    V = 1 + T + T * (K + 1)
    Vp = V - 1 - T
    g1_pts = 2 * (V + 2) + (Vp + 1) + (1 << 21)
    chunk_ms = (out["msm_g1_2^20_ms"] * g1_pts / n + g2_ms * (V + 2) / n2 + 6 * ntt21_ms)
    out["groth16_chunk"] = {
        "ms_estimate": chunk_ms, "g1_msm_points": g1_pts, "g2_msm_points": V + 2,
        "ntt_2^21_count": 6, "g2_msm_2^16_ms": g2_ms, "ntt_2^21_ms": ntt21_ms,
        "sample": "timed: G1 MSM 2^20 (above), G2 MSM 2^16, NTT 2^21; the paper-size chunk's "
                  "CPU time = those rates x its MSM sizes + 6 NTTs (linear in points)"}
    return out


def cpu_baseline(args, n: int) -> dict | None:
    """The reference's CPU path (oracle/_ref) on this host, bounded sample."""
    so = os.path.join(ROOT, "oracle", "_ref", "libaceref.so")
    if args.no_cpu_baseline or not os.path.exists(so):
        return None
    r = subprocess.run([sys.executable, os.path.abspath(__file__), "--impl", "reference",
                        "--steps", "3", "--warmup", "1", "--n-tx", str(n)],
                       capture_output=True, text=True, timeout=900)
    for ln in r.stdout.splitlines():
        if ln.startswith("{"):
            d = json.loads(ln)
            if "cpu_baseline" in d:
                cb = d["cpu_baseline"]
                cb["ms_per_block"] = d["ms_per_step"]
                cb["fc_matches_golden"] = d.get("parity", {}).get("fc_matches_golden")
                cb["one_core"] = cpu_baseline_one_core(n)
                return cb
    return {"unavailable": (r.stderr or "")[-300:]}


def cpu_baseline_one_core(n: int) -> dict | None:
    """the same reference path pinned to ONE host core (taskset;
    its ThreadPool still starts hardware_concurrency() threads, time-sliced on
    that core), one timed block."""
    import shutil
    if not shutil.which("taskset"):
        return None
    try:
        r = subprocess.run(["taskset", "-c", "0", sys.executable, os.path.abspath(__file__),
                            "--impl", "reference", "--steps", "1", "--warmup", "0",
                            "--n-tx", str(n)], capture_output=True, text=True, timeout=600)
    except (OSError, subprocess.TimeoutExpired):
        return None
    for ln in r.stdout.splitlines():
        if ln.startswith("{"):
            d = json.loads(ln)
            if "ms_per_step" in d:
                return {"ms_per_block": d["ms_per_step"], "tx_per_s": d["value"], "cores": 1,
                        "sample": "1 timed block, taskset -c 0"}
    return None


def bench_phase1a_and_verify(ctx, dev, fb, revs, rev_index, with_cpu: bool) -> dict:
    """SURVEY 8f rows measured on the same 100k-tx block: Phase 1a on the GPU
    (light check against a 4,096-id registry + order-preserving block build
    with header roots, device-resident, L2 not flushed) and the mock
    verify_finality_certificate (host C ABI: O(N) recompute), each next to the
    reference's own CPU function on this host (oracle/_ref, when built)."""
    import ctypes as C
    import torch
    from paper_2603_10242_b200 import _native as N, crypto, pipeline, prover, wire
    n = fb.n
    # registry: the block's identity + 4,095 others (sorted, the std::set order)
    idc = fb.atts[32:64].tobytes()
    others = wire.sha256_many([b"id" + k.to_bytes(4, "big") for k in range(4095)], ctx)
    ids = sorted({idc} | {bytes(h) for h in others})
    reg = pipeline.IdentityRegistry()
    for i in ids:
        reg.add(i)
    d = torch.device("cuda", dev)
    pay = torch.from_numpy(np.concatenate([fb.payloads, np.zeros(16, np.uint8)])).to(d)
    offs = torch.from_numpy(np.ascontiguousarray(fb.offs, np.uint64).view(np.int64)).to(d)
    atts = torch.from_numpy(np.concatenate([fb.atts[:104 * n], np.zeros(8, np.uint8)])).to(d)
    rg = torch.from_numpy(reg.array()).to(d)
    codes = torch.empty(n, dtype=torch.uint8, device=d)
    hdr = wire.BlockHeader.decode(fb.header.tobytes())
    tmpl = torch.from_numpy(np.frombuffer(hdr.encode(), np.uint8).copy()).to(d)
    out = [torch.empty_like(pay), torch.zeros(n + 1, dtype=torch.int64, device=d),
           torch.empty_like(atts), torch.empty(256, dtype=torch.uint8, device=d)]
    sp = torch.cuda.current_stream().cuda_stream
    cnt = C.c_uint64()

    def light():
        ctx.call("acegpu_light_check_dev", sp, pay.data_ptr(), offs.data_ptr(), atts.data_ptr(),
                 n, rg.data_ptr(), reg.size(), int(hdr.slot_number), 2, codes.data_ptr(), None)

    def build():
        ctx.call("acegpu_build_block_dev", sp, pay.data_ptr(), offs.data_ptr(), atts.data_ptr(),
                 n, codes.data_ptr(), tmpl.data_ptr(), out[0].data_ptr(), out[1].data_ptr(),
                 out[2].data_ptr(), out[3].data_ptr(), C.byref(cnt))

    def timed(fn, reps=10):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(reps):
            a.record()
            fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)
    t_light = timed(light)
    t_build = timed(build)
    built_hdr = wire.BlockHeader.decode(out[3].cpu().numpy().tobytes())
    res = {"n_tx": n, "registry_ids": reg.size(),
           "light_check_ms": t_light, "light_check_tx_per_s": n / (t_light * 1e-3),
           "build_block_ms": t_build, "accepted": int(cnt.value),
           "header_roots_match_input": built_hdr.tx_merkle_root == hdr.tx_merkle_root
           and built_hdr.attest_merkle_root == hdr.attest_merkle_root}
    # mock verify_finality_certificate through the host C ABI (O(N) recompute)
    r = prover.attest_prove_certify(fb, ctx=ctx)
    fcb = r.fc
    t0 = time.perf_counter()
    v = prover.verify_finality_certificate(fcb, fb, ctx=ctx)
    res["verify_fc_mock_ms"] = (time.perf_counter() - t0) * 1e3
    res["verify_fc_mock_verdict"] = v.name
    so = os.path.join(ROOT, "oracle", "_ref", "libaceref.so")
    if with_cpu and os.path.exists(so):
        ref = C.CDLL(so)
        ref.ref_threads.restype = C.c_uint
        rc = np.zeros(n, np.uint8)
        c3 = np.zeros(3, np.uint64)
        regb = reg.array()
        t0 = time.perf_counter()
        ref.ref_attest_check_light_batch(
            fb.payloads.ctypes.data_as(C.c_void_p), fb.offs.ctypes.data_as(C.c_void_p),
            fb.atts.ctypes.data_as(C.c_void_p), C.c_uint32(n), regb.ctypes.data_as(C.c_void_p),
            C.c_uint64(reg.size()), C.c_uint64(hdr.slot_number), C.c_uint64(2),
            rc.ctypes.data_as(C.c_void_p), c3.ctypes.data_as(C.c_void_p))
        t_ref = (time.perf_counter() - t0) * 1e3
        res["cpu_reference"] = {
            "light_check_ms": t_ref, "cores": 1,
            "sample": "pipeline::attest_check_light over the same %d txs, one thread "
                      "(process_slot runs it under ThreadPool::parallel_for)" % n,
            "codes_match": bool((rc == codes.cpu().numpy()).all())}
    return res


def run_groth16_mode(args, rank: int, world: int) -> None:
    """`--mode groth16`: the 100k-tx block with Groth16 chunk proofs at N GPUs
    (BASELINE configs[3]); latency vs the 400 ms block interval."""
    import torch
    from paper_2603_10242_b200 import _native as N, groth16
    dev = bench_device()
    torch.cuda.set_device(dev)
    ctx = N.context(dev)
    fb, revs, rix = canonical_block_host(args.n_tx, ctx)
    steps, warmup = max(min(args.steps, 5), 3), 1
    pk = groth16.ProvingKey(groth16.PAPER_T, groth16.PAPER_K, ctx=ctx)
    with ClockSampler(dev) as clocks:
        r = run_groth16_block(ctx, dev, fb, revs, rix, rank, world, steps, warmup, pk,
                              e2e=True, verify=True)
    pk.close()
    if rank != 0:
        return
    print(json.dumps({
        "metric": f"proven tx/s ({args.n_tx}-tx block, Groth16 chunk proofs + tree + FC; "
                  "latency = ms_per_step)",
        "value": r["proven_tx_per_s"], "unit": "tx/s", "n_gpus": world, "steps": steps,
        "warmup": warmup, "ms_per_step": r["latency_ms"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32 (Fq/Fr Montgomery limbs)",
        "data": "synthetic", "config": {"workload": f"canonical_block({args.n_tx}), 1,024-tx chunks "
                                                    "x 1,400 constraints (synthetic stand-in circuit)",
                                        "parallelism": f"chunk-sharded x{world}"},
        "groth16": r, "clocks": clocks.summary(), "impl": "ours", "mode": "groth16"}), flush=True)


def spawn_ranks(n: int) -> int:
    """`--gpus N` without a launcher: re-exec this command under
    torch.distributed.run with N ranks (127.0.0.1). With fewer GPUs than ranks
    (a functional run), every rank uses cuda:0 over gloo and the line says so."""
    import socket
    env = dict(os.environ)
    try:
        import torch
        ngpu = torch.cuda.device_count()
    except Exception:
        ngpu = 0
    if ngpu < n:
        env.update({"ACE_BENCH_DEVICE": "0", "ACEGPU_DEVICE": "0", "ACE_DIST_BACKEND": "gloo",
                    "ACE_BENCH_SHARED_GPU": "1"})
        log(f"bench.py: {n} ranks on {ngpu} GPU(s): functional run, gloo, all ranks on cuda:0")
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)]
    return subprocess.call(cmd + sys.argv[1:], env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n-tx", type=int, default=N_TX)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-bn254", action="store_true", help="skip the NTT/MSM microbenchmarks")
    ap.add_argument("--no-stream", action="store_true",
                    help="skip the sustained 12,800-tx block stream (SURVEY 8d config 5)")
    ap.add_argument("--mode", default="mock", choices=["mock", "groth16"],
                    help="mock: the reference's hash-based proof (bit-exact, the headline); "
                         "groth16: the north-star chunk-Groth16 block path")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        sys.exit(spawn_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "ours" and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(bench_device())
        # ACE_DIST_BACKEND / ACE_BENCH_DEVICE: functional multi-rank runs on a
        # one-GPU box (gloo, every rank on cuda:0) -- never a measurement
        dist.init_process_group(os.environ.get("ACE_DIST_BACKEND", "nccl"))
    try:
        if args.mode == "groth16":
            run_groth16_mode(args, rank, world)
        else:
            run_ours(args, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
