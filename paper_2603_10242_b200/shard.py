"""Multi-GPU Prove: power-of-two-aligned transaction chunks sharded across
ranks (one process per GPU, torch.distributed over NCCL for the plumbing).

Why it is bit-exact: the reference pairs nodes (2i, 2i+1) and
promotes an odd last node (prover.cpp:112-124), so the root of every aligned
2^k-leaf chunk IS a level-k node of the global proof tree. The id_com Merkle
tree duplicates an odd last node (wire.cpp:240); the block's last chunk is
therefore lifted by self-pairing up to level k (acegpu_shard_roots_dev does
this when n_total > 2^k). The only exchange is one all-gather of the chunk
roots (289 B proof + 32 B Merkle node per chunk) before the top levels.

Device work goes through the C ABI (acegpu_shard_roots_dev /
acegpu_combine_roots_dev) on torch's current stream; torch supplies device
memory, streams and the collective.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N

LOG2_CHUNK = 10  # 1,024-tx chunks: the Groth16 chunk size of SURVEY §8d


def partition(n_total: int, world: int, log2_chunk: int = LOG2_CHUNK) -> list[tuple[int, int]]:
    """Contiguous whole chunks per rank, balanced by chunk count: [(start, count)].
    (Not one power-of-two range per rank, which strands ranks at 100k, §8e.)"""
    C = 1 << log2_chunk
    chunks = -(-n_total // C)
    out = []
    for r in range(world):
        c0, c1 = chunks * r // world, chunks * (r + 1) // world
        s, e = min(c0 * C, n_total), min(c1 * C, n_total)
        out.append((s, e - s))
    return out


def n_chunks(count: int, log2_chunk: int) -> int:
    return -(-count // (1 << log2_chunk))


@dataclass
class DeviceBlock:
    """A block (or one rank's slice of it) resident in device memory."""
    payloads: "object"   # torch.uint8 [bytes (+pad)]
    offs: "object"       # torch.int64 [n+1] (uint64 bit pattern), rebased to payloads
    atts: "object"       # torch.uint8 [n*104]
    header: "object"     # torch.uint8 [256]
    n: int
    revs: "object" = None       # torch.uint8 [32*users]
    rev_index: "object" = None  # torch.int32 [n]
    witnesses: "object" = None  # torch.uint8 [n*256] (Groth16 mode)

    @staticmethod
    def upload(fb, start: int = 0, count: int | None = None, revs=None, rev_index=None,
               device=None, pin: bool = True) -> "DeviceBlock":
        """Host FlatBlock slice [start, start+count) -> device tensors."""
        import torch
        count = fb.n - start if count is None else count
        dev = torch.device("cuda", N.default_device() if device is None else device)
        b0 = int(fb.offs[start]) if count else 0
        b1 = int(fb.offs[start + count]) if count else 0
        offs = (fb.offs[start:start + count + 1].astype(np.int64) - b0) if count else np.zeros(1, np.int64)

        def put(a):
            t = torch.from_numpy(np.ascontiguousarray(a))
            if pin:
                t = t.pin_memory()
            return t.to(dev, non_blocking=True)
        pl = np.zeros(b1 - b0 + 16, np.uint8)
        pl[:b1 - b0] = fb.payloads[b0:b1]
        at = fb.atts[104 * start:104 * (start + count)] if count else np.zeros(8, np.uint8)
        hdr = fb.header if isinstance(fb.header, np.ndarray) else np.frombuffer(fb.header, np.uint8)
        db = DeviceBlock(put(pl), put(offs), put(at), put(np.ascontiguousarray(hdr)), count)
        if revs is not None:
            db.revs = put(np.ascontiguousarray(revs, np.uint8))
            ri = np.ascontiguousarray(rev_index, np.uint32)[start:start + count]
            db.rev_index = put(ri.view(np.int32) if count else np.zeros(1, np.int32))
        return db


def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream():
    import torch
    return torch.cuda.current_stream().cuda_stream


class GpuBackend:
    """Chunk roots and their combination on the local GPU (libacegpu)."""

    def __init__(self, ctx: N.Context | None = None):
        self.ctx = ctx or N.context()

    def shard_roots(self, db: DeviceBlock, n_total: int, log2_chunk: int, codes=None):
        import torch
        c = n_chunks(db.n, log2_chunk)
        roots = torch.empty(max(c, 1) * 289, dtype=torch.uint8, device=db.atts.device)
        merk = torch.empty(max(c, 1) * 32, dtype=torch.uint8, device=db.atts.device)
        if db.n:
            self.ctx.call("acegpu_shard_roots_dev", _stream(), _ptr(db.payloads), _ptr(db.offs),
                          _ptr(db.atts), db.n, n_total, log2_chunk, _ptr(db.revs),
                          0 if db.revs is None else db.revs.numel() // 32,
                          _ptr(db.rev_index), _ptr(codes), _ptr(roots), _ptr(merk))
        return roots[:c * 289], merk[:c * 32]

    def combine(self, roots, merk, chunks: int, n_total: int, header):
        import torch
        out = torch.empty(289 + 15 + 328, dtype=torch.uint8, device=header.device)
        self.ctx.call("acegpu_combine_roots_dev", _stream(), _ptr(roots) if chunks else None,
                      _ptr(merk) if chunks else None, chunks, n_total, _ptr(header), _ptr(out),
                      out.data_ptr() + 304)
        return out[:289], out[304:304 + 328]


class G16Backend(GpuBackend):
    """Groth16 mode: each aligned chunk of T = pk.T txs is one Groth16 proof
    (acegpu_g16_shard_roots_dev); the tree above the chunks and the FC are
    the reference's rules (acegpu_combine_roots_dev). `witnesses` is the
    rank's n x 256-B witness tensor (build_witness layout)."""

    def __init__(self, pk, ctx: N.Context | None = None):
        super().__init__(ctx or pk.ctx)
        self.pk = pk

    def shard_roots(self, db: DeviceBlock, n_total: int, log2_chunk: int, codes=None):
        import torch
        # chunks of pk.T txs, or one chunk for the whole block (a block-size key)
        assert (1 << log2_chunk) == self.pk.T or (
            n_total <= self.pk.T <= (1 << log2_chunk)), "chunk size must equal the circuit's txs/chunk"
        c = n_chunks(db.n, log2_chunk)
        roots = torch.empty(max(c, 1) * 289, dtype=torch.uint8, device=db.atts.device)
        merk = torch.empty(max(c, 1) * 32, dtype=torch.uint8, device=db.atts.device)
        if db.n:
            self.ctx.call("acegpu_g16_shard_roots_dev", _stream(), self.pk.h, _ptr(db.payloads),
                          _ptr(db.offs), _ptr(db.atts), db.n, n_total, _ptr(db.revs),
                          0 if db.revs is None else db.revs.numel() // 32,
                          _ptr(db.rev_index), _ptr(codes), _ptr(db.witnesses), _ptr(roots),
                          _ptr(merk))
        return roots[:c * 289], merk[:c * 32]


def gather_roots(roots, merk, counts: list[int], group=None):
    """All-gather each rank's chunk roots (padded to the largest rank) and
    return them concatenated in rank order."""
    import torch
    import torch.distributed as dist
    world = len(counts)
    mx = max(max(counts), 1)
    pr = torch.zeros(mx * 289, dtype=torch.uint8, device=roots.device)
    pm = torch.zeros(mx * 32, dtype=torch.uint8, device=merk.device)
    pr[:roots.numel()] = roots
    pm[:merk.numel()] = merk
    dev = pr.device
    if dist.get_backend(group) == "gloo" and dev.type == "cuda":
        # gloo (the CPU-side functional runs: ranks sharing one GPU) gathers
        # host tensors; NCCL gathers the device tensors directly
        pr, pm = pr.cpu(), pm.cpu()
    gr = [torch.empty_like(pr) for _ in range(world)]
    gm = [torch.empty_like(pm) for _ in range(world)]
    dist.all_gather(gr, pr, group=group)
    dist.all_gather(gm, pm, group=group)
    allr = torch.cat([g[:c * 289] for g, c in zip(gr, counts)]).to(dev)
    allm = torch.cat([g[:c * 32] for g, c in zip(gm, counts)]).to(dev)
    return allr, allm


def prove_sharded(local: DeviceBlock, n_total: int, rank: int, world: int,
                  log2_chunk: int = LOG2_CHUNK, backend=None, group=None, codes=None,
                  return_roots: bool = False):
    """One rank's part of a sharded block proof; every rank returns the same
    (proof289, fc328) device tensors (+ all chunk roots, n_chunks x 289 B,
    with return_roots: their first 256 B are the chunk proofs)."""
    backend = backend or GpuBackend()
    parts = partition(n_total, world, log2_chunk)
    counts = [n_chunks(c, log2_chunk) for _, c in parts]
    assert local.n == parts[rank][1]
    roots, merk = backend.shard_roots(local, n_total, log2_chunk, codes)
    if world > 1:
        roots, merk = gather_roots(roots, merk, counts, group)
    out = backend.combine(roots, merk, sum(counts), n_total, local.header)
    return out + (roots,) if return_roots else out


def one_proof_partial(local_full: DeviceBlock, pk, codes=None):
    """One rank's part of ONE Groth16 proof for the whole block (block-size
    key, T >= n; a split key holds the rank's slice of the bases): the
    block's inputs (verdicts, Merkle root, w, pub — every rank holds the whole
    block) and the rank's partial points -> (part384, merkle32) device tensors."""
    import torch
    db = local_full
    dev = db.atts.device
    w = torch.empty(32 * pk.T, dtype=torch.uint8, device=dev)
    pub = torch.empty(32 * pk.T, dtype=torch.uint8, device=dev)
    merk = torch.empty(32, dtype=torch.uint8, device=dev)
    part = torch.empty(384, dtype=torch.uint8, device=dev)
    sp = _stream()
    pk.ctx.call("acegpu_g16_block_inputs_dev", sp, pk.h, _ptr(db.payloads), _ptr(db.offs),
                _ptr(db.atts), db.n, _ptr(db.revs),
                0 if db.revs is None else db.revs.numel() // 32, _ptr(db.rev_index),
                _ptr(codes), _ptr(db.witnesses), _ptr(w), _ptr(pub), _ptr(merk))
    pk.ctx.call("acegpu_g16_prove_partial_dev", sp, pk.h, _ptr(w), _ptr(pub), _ptr(part))
    return part, merk


def owned_mask(rank: int, world: int) -> int:
    """H-polynomial vectors a, b, c (bits 0..2) owned by `rank`: k mod world."""
    return sum(1 << k for k in range(3) if k % world == rank)


def slice_bounds(N: int, rank: int, world: int, shares=None) -> tuple[int, int]:
    """Rank `rank`'s slice of an N-entry array (acegpu_g16_setup_slice's rule)."""
    if shares is None:
        return N * rank // world, N * (rank + 1) // world
    sh = [int(x) for x in shares]
    pre, tot = sum(sh[:rank]), sum(sh)
    return N * pre // tot, N * (pre + sh[rank]) // tot


# Measured per-world shares (‰) for the 100k-tx block (3 x 2^26 domain) on
# B200, evening the slowest owner and non-owner ranks; the last measurement
# (bench.bench_one_proof_split, owner / non-owner): world 8 [70 x3, 158 x5]
# 429 / 421 ms, world 4 [214 x3, 358] 837 / 863 ms, world 2 [472, 528]
# 1,755 / 1,763 ms — the table moves each toward even. The formula's
# fractions differ per world because the MSM window size and efficiency
# change with the slice size.
_MEASURED_SHARES = {2: [472, 528], 4: [217, 217, 217, 349], 8: [70, 70, 70, 158, 158, 158, 158, 158]}


def balanced_shares(world: int, ntt_frac: float | None = None, unit: int = 1000) -> list[int]:
    """Shares of the bases that even out the ranks when vector k of the H
    polynomial is transformed on rank k mod world: an owned vector (its iNTT
    + coset NTT, run concurrently with the rank's MSMs) costs ~ntt_frac of
    the whole proof's MSM work (~0.1 at 100k txs), so owners take fewer
    bases. Without ntt_frac, the measured table for the worlds it holds."""
    if ntt_frac is None:
        if world in _MEASURED_SHARES:
            return list(_MEASURED_SHARES[world])
        ntt_frac = 0.095
    own = [bin(owned_mask(r, world)).count("1") for r in range(world)]
    t = (1.0 + ntt_frac * sum(own)) / world  # per-rank budget, MSM-work units
    w = [max(t - ntt_frac * o, 0.01) for o in own]
    tot = sum(w)
    return [max(1, round(unit * x / tot)) for x in w]


def one_proof_phase1(local_full: DeviceBlock, pk, rank: int, world: int, codes=None):
    """Owner split, phase 1: inputs + witness + this rank's A/B1/B2/L slice
    MSMs (running) + the coset evaluations of its owned vectors ->
    (own (k x N x 32 B), merkle32)."""
    import torch
    db = local_full
    dev = db.atts.device
    N = pk.domain
    mask = owned_mask(rank, world)
    w = torch.empty(32 * pk.T, dtype=torch.uint8, device=dev)
    pub = torch.empty(32 * pk.T, dtype=torch.uint8, device=dev)
    merk = torch.empty(32, dtype=torch.uint8, device=dev)
    own = torch.empty(max(bin(mask).count("1"), 1) * 32 * N, dtype=torch.uint8, device=dev)
    sp = _stream()
    pk.ctx.call("acegpu_g16_block_inputs_dev", sp, pk.h, _ptr(db.payloads), _ptr(db.offs),
                _ptr(db.atts), db.n, _ptr(db.revs),
                0 if db.revs is None else db.revs.numel() // 32, _ptr(db.rev_index),
                _ptr(codes), _ptr(db.witnesses), _ptr(w), _ptr(pub), _ptr(merk))
    pk.ctx.call("acegpu_g16_prove_phase1_dev", sp, pk.h, _ptr(w), _ptr(pub), mask, _ptr(own))
    return own, merk


def one_proof_phase2(slices, pk):
    """Owner split, phase 2: this rank's a | b | c slices -> partial record."""
    import torch
    part = torch.empty(384, dtype=torch.uint8, device=slices.device)
    pk.ctx.call("acegpu_g16_prove_phase2_dev", _stream(), pk.h, _ptr(slices), _ptr(part))
    return part


def exchange_slices(own, rank: int, world: int, N: int, group=None, shares=None):
    """Every owner sends slice r of each of its vectors to rank r (the key's
    share bounds) -> this rank's a | b | c slices (S x 32 B each). Equal
    shares: one scatter per vector; weighted: point-to-point sends."""
    import torch
    import torch.distributed as dist
    lo, hi = slice_bounds(N, rank, world, shares)
    S = hi - lo
    dev = own.device
    gloo = dist.get_backend(group) == "gloo"
    out = torch.empty(3 * 32 * S, dtype=torch.uint8, device=dev)
    idx = 0
    for k in range(3):
        o = k % world
        dst = torch.empty(32 * S, dtype=torch.uint8, device="cpu" if gloo else dev)
        vec = None
        if rank == o:
            vec = own[32 * N * idx:32 * N * (idx + 1)]
            idx += 1
        if shares is None:
            lst = None
            if rank == o:
                lst = []
                for r in range(world):
                    a, b = slice_bounds(N, r, world)
                    t = vec[32 * a:32 * b]
                    lst.append(t.cpu() if gloo else t)
            dist.scatter(dst, lst, src=o, group=group)
        elif rank == o:
            reqs = []
            for r in range(world):
                a, b = slice_bounds(N, r, world, shares)
                t = vec[32 * a:32 * b]
                if r == rank:
                    dst.copy_(t)
                else:
                    reqs.append(dist.isend(t.cpu() if gloo else t.contiguous(), r, group=group))
            for q in reqs:
                q.wait()
        else:
            dist.recv(dst, o, group=group)
        out[32 * S * k:32 * S * (k + 1)] = dst.to(dev)
    return out


def one_proof_finish(parts, world: int, merk, n_total: int, header, pk):
    """Sum the ranks' partial points (world x 384 B, rank order) into the
    block's proof -> (proof289, fc328) via the reference's tree rule over the
    one root."""
    import torch
    root = torch.empty(289, dtype=torch.uint8, device=merk.device)
    pk.ctx.call("acegpu_g16_finish_dev", _stream(), pk.h, _ptr(parts), world, None, None, None,
                _ptr(root))
    return GpuBackend(pk.ctx).combine(root, merk, 1, n_total, header)


def prove_one_proof(local_full: DeviceBlock, n_total: int, rank: int, world: int, pk,
                    group=None, codes=None):
    """ONE Groth16 proof for the whole block across `world` ranks (DIZK-style
    split): every rank computes the witness and the MSMs over its slice of the
    bases; the H polynomial's vectors a, b, c are transformed by their owners
    (rank k mod world) and scattered by slices, so each rank forms
    (a b - c) / Z and [h] on its slice only; one all-gather of 384-B partial
    records; every rank sums them in rank order and returns the same
    (proof289, fc328)."""
    import torch
    import torch.distributed as dist
    if world > 1:
        # the H polynomial's three vectors are computed by their owners and
        # exchanged by slices (each rank then does 2 of the 6 NTTs, not 6)
        own, merk = one_proof_phase1(local_full, pk, rank, world, codes)
        slices = exchange_slices(own, rank, world, pk.domain, group, pk.shares)
        del own
        part = one_proof_phase2(slices, pk)
    else:
        part, merk = one_proof_partial(local_full, pk, codes)
    if world > 1:
        dev = part.device
        src = part.cpu() if dist.get_backend(group) == "gloo" else part
        out = [torch.empty_like(src) for _ in range(world)]
        dist.all_gather(out, src, group=group)
        parts = torch.cat(out).to(dev)
    else:
        parts = part
    return one_proof_finish(parts, world, merk, n_total, local_full.header, pk)


def prove_sharded_single_process(fb, world: int, log2_chunk: int, ctx=None, pk=None,
                                 witnesses=None, return_roots: bool = False):
    """Emulates `world` ranks one after another on one GPU (no collective):
    used to check shard/combine bit-exactness with a single device.
    With a Groth16 proving key `pk`, chunks are Groth16 proofs. return_roots
    adds the chunk roots (n_chunks x 289 B: proof | digest | kind)."""
    import torch
    be = G16Backend(pk, ctx) if pk is not None else GpuBackend(ctx)
    parts = partition(fb.n, world, log2_chunk)
    rs, ms = [], []
    for s, c in parts:
        db = DeviceBlock.upload(fb, s, c)
        if witnesses is not None:
            db.witnesses = torch.from_numpy(
                np.ascontiguousarray(witnesses[256 * s:256 * (s + c)])).to(db.atts.device)
        r, m = be.shard_roots(db, fb.n, log2_chunk)
        rs.append(r)
        ms.append(m)
        hdr = db.header
    roots, merk = torch.cat(rs), torch.cat(ms)
    proof, fc = be.combine(roots, merk, sum(n_chunks(c, log2_chunk) for _, c in parts), fb.n, hdr)
    torch.cuda.synchronize()
    out = (proof.cpu().numpy().tobytes(), fc.cpu().numpy().tobytes())
    return out + (roots.cpu().numpy().tobytes(),) if return_roots else out
