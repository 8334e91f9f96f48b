"""Phase 1a on the GPU, mirroring ace::pipeline
(proj/include/ace/pipeline.hpp, proj/src/pipeline.cpp): the leader's light
admission check and block assembly, feeding the prover with device-resident
blocks (no host round trip for the transactions).

Same names and semantics as the reference: ``IdentityRegistry``
(pipeline.hpp:22-30), ``LightCheck`` (:32-37), ``LightCheckCounters``
(:41-52), ``PipelineConfig`` (:16-21), ``attest_check_light`` (pipeline.cpp:
20-42). The batched ``attest_check_light_batch`` is the B200-native form; the
single-transaction call keeps the reference's signature on top of it.
Execution (Phase 1b) and the state root are outside the Prove path and come
in through the header template.
"""
from __future__ import annotations

import bisect
import enum
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .wire import BlockHeader, FlatBlock, Transaction


class LightCheck(enum.IntEnum):
    AcceptPendingProof = 0
    PayloadBinding = 1
    UnknownIdentity = 2
    StaleDomain = 3


def to_string(c: LightCheck) -> str:
    return LightCheck(c).name


@dataclass
class PipelineConfig:
    max_txs_per_block: int = 2000
    domain_window_slots: int = 2
    slot_duration_ms: int = 400
    parallelism: int = 0


@dataclass
class LightCheckCounters:
    sha256_ops: int = 0
    registry_probes: int = 0
    window_checks: int = 0

    def __iadd__(self, o: "LightCheckCounters") -> "LightCheckCounters":
        self.sha256_ops += o.sha256_ops
        self.registry_probes += o.registry_probes
        self.window_checks += o.window_checks
        return self


class IdentityRegistry:
    """Set of 32-B identity commitments. Kept sorted (the std::set order) so
    the device probe is a binary search over a flat HBM array."""

    def __init__(self):
        self._ids: list[bytes] = []

    def add(self, id_com: bytes) -> None:
        id_com = bytes(id_com)
        assert len(id_com) == 32
        i = bisect.bisect_left(self._ids, id_com)
        if i == len(self._ids) or self._ids[i] != id_com:
            self._ids.insert(i, id_com)

    def contains(self, id_com: bytes) -> bool:
        id_com = bytes(id_com)
        i = bisect.bisect_left(self._ids, id_com)
        return i < len(self._ids) and self._ids[i] == id_com

    def size(self) -> int:
        return len(self._ids)

    def array(self) -> np.ndarray:
        """n x 32 sorted commitments as one flat uint8 array (the device layout)."""
        if not self._ids:
            return np.zeros(32, np.uint8)
        return np.frombuffer(b"".join(self._ids), np.uint8).copy()


def attest_check_light_batch(fb: FlatBlock, registry: IdentityRegistry, current_slot: int,
                             cfg: PipelineConfig | None = None,
                             counters: LightCheckCounters | None = None, ctx=None) -> np.ndarray:
    """attest_check_light over every tx of a flat block (one GPU launch)."""
    cfg = cfg or PipelineConfig()
    ctx = ctx or N.context()
    codes = np.zeros(max(fb.n, 1), np.uint8)
    c3 = np.zeros(3, np.uint64)
    reg = registry.array()
    ctx.call("acegpu_light_check", N.addr(fb.payloads), N.addr(fb.offs), N.addr(fb.atts), fb.n,
             N.addr(reg), registry.size(), int(current_slot), int(cfg.domain_window_slots),
             N.addr(codes), c3.ctypes.data_as(N.u64p))
    if counters is not None:
        counters += LightCheckCounters(int(c3[0]), int(c3[1]), int(c3[2]))
    return codes[:fb.n]


def attest_check_light(tx: Transaction, registry: IdentityRegistry, current_slot: int,
                       cfg: PipelineConfig | None = None,
                       counters: LightCheckCounters | None = None, ctx=None) -> LightCheck:
    """pipeline.cpp:20-42 for one transaction."""
    fb = FlatBlock.from_lists([tx.payload], [tx.attestation.encode()], b"\0" * 256)
    return LightCheck(int(attest_check_light_batch(fb, registry, current_slot, cfg, counters,
                                                   ctx)[0]))


@dataclass
class DeviceBuiltBlock:
    """A block assembled on the device (torch tensors), ready for
    acegpu_attest_prove_certify_dev / shard.DeviceBlock."""
    payloads: "object"
    offs: "object"
    atts: "object"
    header: "object"
    n: int
    codes: "object"   # the light-check verdicts of the candidate txs


def _upload(fb: FlatBlock, dev):
    import torch

    def put(a):
        return torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    n = fb.n
    return (put(np.concatenate([fb.payloads, np.zeros(16, np.uint8)])),
            put(np.ascontiguousarray(fb.offs, np.uint64).view(np.int64)),
            put(np.concatenate([fb.atts[:104 * n], np.zeros(8, np.uint8)])))


def _build(ctx, dev, pay, offs, atts, n, codes, tmpl):
    import torch
    u8 = dict(dtype=torch.uint8, device=dev)
    out_pay = torch.empty(pay.numel(), **u8)
    out_offs = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    out_atts = torch.empty(atts.numel(), **u8)
    out_hdr = torch.empty(256, **u8)
    cnt = N.C.c_uint64()
    ctx.call("acegpu_build_block_dev", torch.cuda.current_stream(dev).cuda_stream,
             pay.data_ptr(), offs.data_ptr(), atts.data_ptr(), n,
             None if codes is None else codes.data_ptr(), tmpl.data_ptr(), out_pay.data_ptr(),
             out_offs.data_ptr(), out_atts.data_ptr(), out_hdr.data_ptr(), N.C.byref(cnt))
    k = cnt.value
    return out_pay, out_offs[:k + 1], out_atts, out_hdr, k


def build_block_device(candidates: FlatBlock, registry: IdentityRegistry, header: BlockHeader,
                       cfg: PipelineConfig | None = None, device=None,
                       ctx=None) -> DeviceBuiltBlock:
    """Phase 1a of process_slot (pipeline.cpp:99-145) on the GPU: light-check
    the candidate txs, keep the accepted ones in order, and fill the header's
    tx_count / tx_merkle_root / attest_merkle_root. `header` supplies the
    rest (slot, parent, state root, PoH, leader, timestamp); its slot_number
    is the light check's current slot."""
    import torch
    cfg = cfg or PipelineConfig()
    ctx = ctx or N.context()
    dev = torch.device("cuda", N.default_device() if device is None else device)
    n = candidates.n
    pay, offs, atts = _upload(candidates, dev)
    reg = torch.from_numpy(registry.array()).to(dev)
    tmpl = torch.from_numpy(np.frombuffer(header.encode(), np.uint8).copy()).to(dev)
    codes = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    if n:
        ctx.call("acegpu_light_check_dev", torch.cuda.current_stream(dev).cuda_stream,
                 pay.data_ptr(), offs.data_ptr(), atts.data_ptr(), n, reg.data_ptr(),
                 registry.size(), int(header.slot_number), int(cfg.domain_window_slots),
                 codes.data_ptr(), None)
    out = _build(ctx, dev, pay, offs, atts, n, codes if n else None, tmpl)
    return DeviceBuiltBlock(*out, codes=codes[:n])


def tx_merkle_roots(fb: FlatBlock, ctx=None) -> tuple[bytes, bytes]:
    """(tx_merkle_root, attest_merkle_root) of a flat block (wire.cpp:257-273),
    via the device block builder with every tx kept."""
    import torch
    ctx = ctx or N.context()
    dev = torch.device("cuda", N.default_device())
    pay, offs, atts = _upload(fb, dev)
    tmpl = torch.zeros(256, dtype=torch.uint8, device=dev)
    _, _, _, hdr, _ = _build(ctx, dev, pay, offs, atts, fb.n, None, tmpl)
    h = BlockHeader.decode(hdr.cpu().numpy().tobytes())
    return h.tx_merkle_root, h.attest_merkle_root
