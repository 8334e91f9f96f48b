"""Pipelined block prover: the sustained-stream form of ProverService
(prover.hpp:141-172, prover.cpp:301-359).

The reference's worker proves one block at a time. Here blocks are spread
over `lanes` independent libacegpu contexts, each with its own CUDA stream,
device workspace and pinned output buffers, so block n+1's host->device copy
and attestation run while block n's proof tree is still being hashed (a
12,800-tx block's upper tree levels are latency chains that leave most SMs
idle). Everything is stream-ordered and asynchronous from the submitting
thread, one C-ABI call per block (acegpu_attest_prove_certify_async: H2D of
the pinned inputs, the pipeline, D2H of verdicts / proof / FC); per-block
latency is taken from CUDA events on the lane's stream (H2D start -> FC and
verdicts back in pinned host memory).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .wire import FlatBlock


@dataclass
class StreamResult:
    ticket: int
    codes: np.ndarray      # n verdicts (AttestationCheck)
    proof289: bytes
    fc328: bytes
    latency_ms: float      # device timeline: H2D start -> results in host memory


class _Lane:
    def __init__(self, device: int, max_tx: int, max_payload: int, max_revs: int):
        import torch
        self.ctx = N.Context(device)
        self.dev = torch.device("cuda", device)
        self.stream = torch.cuda.Stream(device=self.dev)
        self.h_codes = torch.empty(max(max_tx, 1), dtype=torch.uint8).pin_memory()
        self.h_out = torch.empty(640, dtype=torch.uint8).pin_memory()
        self.ev0 = torch.cuda.Event(enable_timing=True)
        self.ev1 = torch.cuda.Event(enable_timing=True)
        self.ticket = None
        self.n = 0
        self.pinned = None


class PipelinedProver:
    """submit() enqueues a block (host FlatBlock, ideally in pinned memory) and
    returns a ticket; result(ticket) waits for it. A lane is reused only after
    its previous block's results were collected (FIFO per lane)."""

    def __init__(self, lanes: int = 4, max_tx: int = 16384, max_payload: int | None = None,
                 max_revs: int = 64, device: int | None = None, graphs: bool = True):
        dev = N.default_device() if device is None else device
        self.max_tx = max_tx
        self.max_payload = max_payload or 256 * max_tx
        self.max_revs = max_revs
        self.lanes = [_Lane(dev, max_tx, self.max_payload, max_revs) for _ in range(lanes)]
        self.next_ticket = 0
        # CUDA-graph replay per lane for consecutive blocks of one shape
        self.entry = ("acegpu_attest_prove_certify_graph" if graphs
                      else "acegpu_attest_prove_certify_async")
        self.done: dict[int, StreamResult] = {}

    def _collect(self, lane: _Lane) -> None:
        if lane.ticket is None:
            return
        lane.ev1.synchronize()
        n = lane.n
        out = lane.h_out.numpy()
        self.done[lane.ticket] = StreamResult(
            lane.ticket, lane.h_codes.numpy()[:n].copy(), out[:289].tobytes(),
            out[304:304 + 328].tobytes(), lane.ev0.elapsed_time(lane.ev1))
        lane.ticket = None
        lane.pinned = None

    def submit(self, fb: FlatBlock, revs: np.ndarray, rev_index: np.ndarray,
               pinned: dict | None = None) -> int:
        """pinned: optional dict of torch pinned CPU tensors with keys
        payloads/offs/atts/header/revs/rev_index (skips staging copies)."""
        import torch
        n = fb.n
        nb = int(fb.offs[n]) if n else 0
        if n > self.max_tx or nb > self.max_payload or len(revs) > 32 * self.max_revs:
            raise ValueError("block exceeds the PipelinedProver capacity")
        t = self.next_ticket
        self.next_ticket += 1
        lane = self.lanes[t % len(self.lanes)]
        self._collect(lane)
        if pinned is None:
            pinned = pin_block(fb, revs, rev_index)
        nr = len(revs) // 32
        lane.ev0.record(lane.stream)
        # one C-ABI call per block: H2D (pinned), attestation + proof + FC,
        # D2H of verdicts / proof / FC, all stream-ordered on the lane's stream
        lane.ctx.call(self.entry, lane.stream.cuda_stream,
                      pinned["payloads"].data_ptr(), pinned["offs"].data_ptr(),
                      pinned["atts"].data_ptr(), n, pinned["header"].data_ptr(),
                      pinned["revs"].data_ptr() if n else None, nr if n else 0,
                      pinned["rev_index"].data_ptr() if n else None,
                      lane.h_codes.data_ptr() if n else None, lane.h_out.data_ptr(),
                      lane.h_out.data_ptr() + 304)
        lane.ev1.record(lane.stream)
        lane.pinned = pinned  # inputs must outlive the asynchronous copies
        lane.ticket, lane.n = t, n
        return t

    def result(self, ticket: int) -> StreamResult:
        if ticket not in self.done:
            lane = self.lanes[ticket % len(self.lanes)]
            if lane.ticket != ticket:
                raise KeyError(f"ticket {ticket} unknown or already collected")
            self._collect(lane)
        return self.done.pop(ticket)

    def drain(self) -> list[StreamResult]:
        for lane in self.lanes:
            self._collect(lane)
        out = [self.done.pop(k) for k in sorted(self.done)]
        return out

    def close(self) -> None:
        for lane in self.lanes:
            lane.ctx.close()


def pin_block(fb: FlatBlock, revs: np.ndarray, rev_index: np.ndarray) -> dict:
    """Host block -> pinned torch tensors (done once per block, off the hot loop)."""
    import torch

    def pin(a, dtype=None):
        t = torch.from_numpy(np.ascontiguousarray(a if dtype is None else a.view(dtype)))
        return t.pin_memory()
    n = fb.n
    return {
        "payloads": pin(fb.payloads),
        "offs": pin(np.ascontiguousarray(fb.offs, np.uint64), np.int64),
        "atts": pin(fb.atts),
        "header": pin(fb.header if isinstance(fb.header, np.ndarray)
                      else np.frombuffer(bytes(fb.header), np.uint8)),
        "revs": pin(np.ascontiguousarray(revs, np.uint8)),
        "rev_index": pin(np.ascontiguousarray(rev_index[:max(n, 1)] if n else np.zeros(1),
                                              np.uint32), np.int32),
    }
