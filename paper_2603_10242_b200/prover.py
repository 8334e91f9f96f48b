"""Python mirror of the reference prover API (proj/include/ace/prover.hpp),
every proof computed on the GPU through libacegpu (include/acegpu.h).

Same names, argument meaning and error behaviour as ``ace::prover``:
``aggregate_tree([])`` and ``WitnessScheme(0, ...)`` raise ``ValueError`` (the
reference throws std::invalid_argument); verdicts are enums; backup shortfall
is a ``BackupUnavailable`` value instead of a ``std::variant`` alternative.
Work counters advance exactly as the reference's (prover.cpp:60-63,83,102).
"""
from __future__ import annotations

import enum
import queue
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .crypto import Rev
from .wire import (Block, FinalityCertificate, FlatBlock, Transaction, ZERO32, sha256,
                   sha256_many)

K_WITNESS_BYTES = 256          # prover.hpp:83
K_FC_VERIFY_COST_UNITS = 1     # prover.hpp:77
PROOF_BYTES = 289              # bytes(256) | digest(32) | kind(1)


class ProofKind(enum.IntEnum):
    Tx = 0
    Aggregate = 1


@dataclass
class MockProof:
    """prover.hpp:33-43; equality compares all three fields."""
    bytes: bytes = b"\0" * 256
    public_inputs_digest: bytes = ZERO32
    kind: ProofKind = ProofKind.Tx

    def to_bytes(self) -> bytes:
        return self.bytes + self.public_inputs_digest + bytes([int(self.kind)])

    @staticmethod
    def from_bytes(b) -> "MockProof":
        b = bytes(b)
        return MockProof(b[:256], b[256:288], ProofKind(b[288]))


@dataclass
class PublicInputs:
    """Five 32-B words (prover.hpp:22-31)."""
    id_com: bytes = ZERO32
    tx_hash: bytes = ZERO32
    domain: bytes = ZERO32
    target: bytes = ZERO32
    rp_com: bytes = ZERO32

    @staticmethod
    def for_tx(tx: Transaction) -> "PublicInputs":
        """prover.cpp:65-72."""
        return PublicInputs(tx.attestation.id_com, sha256(tx.payload),
                            tx.attestation.domain.encode().ljust(32, b"\0"))

    def encode(self) -> bytes:
        return self.id_com + self.tx_hash + self.domain + self.target + self.rp_com

    def digest(self) -> bytes:
        return sha256(self.encode())


@dataclass
class AggregationStats:
    levels: int = 0
    pair_ops: int = 0


class WorkCounters:
    """prover.hpp:45-50 (relaxed atomics there; a lock here)."""

    def __init__(self):
        self._lock = threading.Lock()
        self.tx_proofs = 0
        self.aggregations = 0

    def add(self, tx_proofs: int = 0, aggregations: int = 0) -> None:
        with self._lock:
            self.tx_proofs += tx_proofs
            self.aggregations += aggregations


_counters = WorkCounters()


def work_counters() -> WorkCounters:
    return _counters


class FcCheck(enum.IntEnum):
    Valid = 0
    SlotMismatch = 1
    HashMismatch = 2
    ProofMismatch = 3


def to_string(c) -> str:
    return type(c)(c).name


def _proofs_array(proofs: list[MockProof]) -> np.ndarray:
    return np.frombuffer(b"".join(p.to_bytes() for p in proofs), np.uint8).copy()


def _split(arr: np.ndarray, n: int) -> list[MockProof]:
    return [MockProof.from_bytes(arr[289 * i:289 * (i + 1)]) for i in range(n)]


# ------------------------------------------------------------- proving
def prove_public_inputs_batch(pubs: list[PublicInputs], ctx=None) -> list[MockProof]:
    if not pubs:
        return []
    ctx = ctx or N.context()
    arr = np.frombuffer(b"".join(p.encode() for p in pubs), np.uint8).copy()
    out = np.zeros(289 * len(pubs), np.uint8)
    ctx.call("acegpu_prove_public_inputs", N.addr(arr), len(pubs), N.addr(out))
    _counters.add(tx_proofs=len(pubs))
    return _split(out, len(pubs))


def prove_public_inputs(pub: PublicInputs, ctx=None) -> MockProof:
    """prover.cpp:78-85."""
    return prove_public_inputs_batch([pub], ctx)[0]


def prove_txs(fb: FlatBlock, ctx=None) -> list[MockProof]:
    """prove_tx over every tx of a flat block (prover.cpp:87-89, batched)."""
    if fb.n == 0:
        return []
    ctx = ctx or N.context()
    out = np.zeros(289 * fb.n, np.uint8)
    ctx.call("acegpu_prove_txs", N.addr(fb.payloads), N.addr(fb.offs), N.addr(fb.atts), fb.n,
             N.addr(out))
    _counters.add(tx_proofs=fb.n)
    return _split(out, fb.n)


def prove_tx(tx: Transaction, ctx=None) -> MockProof:
    return prove_txs(FlatBlock.from_lists([tx.payload], [tx.attestation.encode()], b"\0" * 256),
                     ctx)[0]


def verify_mock_batch(proofs: list[MockProof], ctx=None) -> list[bool]:
    if not proofs:
        return []
    ctx = ctx or N.context()
    arr = _proofs_array(proofs)
    ok = np.zeros(len(proofs), np.uint8)
    ctx.call("acegpu_verify_mock", N.addr(arr), len(proofs), N.addr(ok))
    return [bool(x) for x in ok]


def verify_mock(proof: MockProof, ctx=None) -> bool:
    """prover.cpp:91-95."""
    return verify_mock_batch([proof], ctx)[0]


def aggregate_pairs(a: list[MockProof], b: list[MockProof], ctx=None) -> list[MockProof]:
    assert len(a) == len(b)
    if not a:
        return []
    ctx = ctx or N.context()
    out = np.zeros(289 * len(a), np.uint8)
    ctx.call("acegpu_aggregate_pairs", _proofs_array(a), _proofs_array(b),
             len(a), N.addr(out))
    _counters.add(aggregations=len(a))
    return _split(out, len(a))


def aggregate_pair(a: MockProof, b: MockProof, ctx=None) -> MockProof:
    """prover.cpp:97-104."""
    return aggregate_pairs([a], [b], ctx)[0]


def aggregate_tree(proofs: list[MockProof], stats: AggregationStats | None = None,
                   ctx=None) -> MockProof:
    """prover.cpp:106-127. Raises ValueError on an empty list."""
    if not proofs:
        raise ValueError("aggregate_tree: empty proof list")
    ctx = ctx or N.context()
    out = np.zeros(289, np.uint8)
    lv, pr = N.C.c_uint64(), N.C.c_uint64()
    ctx.call("acegpu_aggregate_tree", _proofs_array(proofs), len(proofs), N.addr(out),
             N.C.byref(lv), N.C.byref(pr))
    _counters.add(aggregations=pr.value)
    if stats is not None:
        stats.levels, stats.pair_ops = lv.value, pr.value
    return MockProof.from_bytes(out)


def _flat(block) -> FlatBlock:
    return block if isinstance(block, FlatBlock) else block.flatten()


@dataclass
class ProveResult:
    proof: MockProof
    fc: FinalityCertificate
    stats: AggregationStats
    codes: np.ndarray | None = None


def attest_prove_certify(block, revs: np.ndarray | None = None,
                         rev_index: np.ndarray | None = None, ctx=None) -> ProveResult:
    """The Phase-2 step in one GPU pipeline: batched full attestation check
    (when a REV table is given), prove_block and build_finality_certificate
    (ProverService::run body, prover.cpp:350-351)."""
    fb = _flat(block)
    ctx = ctx or N.context()
    proof = np.zeros(289, np.uint8)
    fc = np.zeros(328, np.uint8)
    codes = np.zeros(max(fb.n, 1), np.uint8) if revs is not None else None
    lv, pr = N.C.c_uint64(), N.C.c_uint64()
    ri = None if rev_index is None else np.ascontiguousarray(rev_index, np.uint32)
    ctx.call("acegpu_attest_prove_certify", N.addr(fb.payloads), N.addr(fb.offs), N.addr(fb.atts),
             fb.n, N.addr(fb.header), N.addr(revs), 0 if revs is None else len(revs) // 32,
             N.addr(ri), N.addr(codes), N.addr(proof), N.addr(fc), N.C.byref(lv), N.C.byref(pr))
    _counters.add(tx_proofs=max(fb.n, 1), aggregations=pr.value)
    return ProveResult(MockProof.from_bytes(proof), FinalityCertificate.decode(fc.tobytes()),
                       AggregationStats(lv.value, pr.value),
                       None if codes is None else codes[:fb.n])


def prove_block(block, stats: AggregationStats | None = None, ctx=None) -> MockProof:
    """prover.cpp:129-142 (the empty block proves PublicInputs{tx_hash = block_hash})."""
    r = attest_prove_certify(block, ctx=ctx)
    if stats is not None:
        stats.levels, stats.pair_ops = r.stats.levels, r.stats.pair_ops
    return r.proof


def build_finality_certificate(block, aggregate: MockProof, ctx=None) -> FinalityCertificate:
    """prover.cpp:144-156."""
    fb = _flat(block)
    ctx = ctx or N.context()
    out = np.zeros(328, np.uint8)
    ctx.call("acegpu_build_fc", N.addr(fb.atts), fb.n, N.addr(fb.header),
             np.frombuffer(aggregate.to_bytes(), np.uint8).copy(), N.addr(out))
    return FinalityCertificate.decode(out.tobytes())


class CostUnits:
    def __init__(self):
        self.value = 0


def verify_finality_certificate(fc: FinalityCertificate, block, cost_units: CostUnits | None = None,
                                ctx=None) -> FcCheck:
    """prover.cpp:158-169 (full recompute)."""
    if cost_units is not None:
        cost_units.value += K_FC_VERIFY_COST_UNITS
    fb = _flat(block)
    ctx = ctx or N.context()
    res = N.C.c_int()
    ctx.call("acegpu_verify_fc", np.frombuffer(fc.encode(), np.uint8).copy(),
             N.addr(fb.payloads), N.addr(fb.offs), N.addr(fb.atts), fb.n, N.addr(fb.header),
             N.C.byref(res))
    if res.value == FcCheck.Valid or res.value == FcCheck.ProofMismatch:
        _counters.add(tx_proofs=max(fb.n, 1), aggregations=max(fb.n - 1, 0))
    return FcCheck(res.value)


# ------------------------------------------------------------- witnesses
def build_witnesses(keys: list[bytes], tx_hashes: list[bytes], ctx=None) -> list[bytes]:
    if not keys:
        return []
    ctx = ctx or N.context()
    k = np.frombuffer(b"".join(keys), np.uint8).copy()
    t = np.frombuffer(b"".join(tx_hashes), np.uint8).copy()
    out = np.zeros(256 * len(keys), np.uint8)
    ctx.call("acegpu_build_witness", N.addr(k), N.addr(t), len(keys), N.addr(out))
    return [out[256 * i:256 * i + 256].tobytes() for i in range(len(keys))]


def build_witness(attest_key: bytes, tx_hash: bytes, ctx=None) -> bytes:
    """prover.cpp:181-188."""
    return build_witnesses([attest_key], [tx_hash], ctx)[0]


def witnesses_match(witnesses: list[bytes], txs: list[Transaction], ctx=None) -> list[bool]:
    """witness_matches_tx (prover.cpp:190-197) over a batch."""
    if not txs:
        return []
    ctx = ctx or N.context()
    w = np.zeros(256 * len(txs), np.uint8)
    lens = np.zeros(len(txs), np.uint32)
    for i, x in enumerate(witnesses):
        lens[i] = len(x)
        w[256 * i:256 * i + min(len(x), 256)] = np.frombuffer(x[:256], np.uint8)
    atts = np.frombuffer(b"".join(t.attestation.encode() for t in txs), np.uint8).copy()
    ok = np.zeros(len(txs), np.uint8)
    ctx.call("acegpu_witness_check", N.addr(w), N.addr(lens), N.addr(atts), len(txs), N.addr(ok))
    return [bool(x) for x in ok]


def witness_matches_tx(witness: bytes, tx: Transaction, ctx=None) -> bool:
    return witnesses_match([witness], [tx], ctx)[0]


@dataclass
class WitnessBundle:
    tx_hash: bytes = ZERO32
    ciphertext: bytes = b""
    share_threshold: int = 0


class WitnessScheme:
    """Mock XOR threshold scheme (prover.hpp:99-123, prover.cpp:199-264)."""

    def __init__(self, n_validators: int, master_seed: bytes):
        if n_validators == 0:
            raise ValueError("WitnessScheme: need at least one validator")
        if n_validators > 64:
            raise ValueError("WitnessScheme: at most 64 validators (share mask width)")
        self.n_ = n_validators
        self.t_ = (2 * n_validators + 2) // 3
        self.master_ = bytes(master_seed)

    def validators(self) -> int:
        return self.n_

    def threshold(self) -> int:
        return self.t_

    def share_indices(self, validator: int) -> list[int]:
        span = self.n_ - self.t_
        return [j for j in range(self.t_) if (validator + self.n_ - j) % self.n_ <= span]

    def share_value(self, tx_hash: bytes, index: int) -> bytes:
        return sha256(b"witness-share-v1" + self.master_ + tx_hash + index.to_bytes(4, "big"))

    def _xor(self, tx_hashes: list[bytes], masks: list[int], data: list[bytes], ctx=None):
        if not data:
            return []
        ctx = ctx or N.context()
        L = len(data[0])
        assert all(len(d) == L for d in data)
        inp = np.frombuffer(b"".join(data), np.uint8).copy()
        out = np.zeros(len(inp), np.uint8)
        ctx.call("acegpu_witness_xor", np.frombuffer(self.master_, np.uint8).copy(),
                 np.frombuffer(b"".join(tx_hashes), np.uint8).copy(),
                 np.asarray(masks, np.uint64), inp, L, len(data), out)
        return [out[L * i:L * (i + 1)].tobytes() for i in range(len(data))]

    def encapsulate(self, tx_hash: bytes, witness: bytes, ctx=None) -> WitnessBundle:
        full = (1 << self.t_) - 1
        ct = self._xor([tx_hash], [full], [witness], ctx)[0] if witness else b""
        return WitnessBundle(tx_hash, ct, self.t_)

    def covered_mask(self, contributors) -> int:
        m = 0
        for v in contributors:
            for j in self.share_indices(v % self.n_):
                m |= 1 << j
        return m

    def decrypt_many(self, bundles: list[WitnessBundle], contributors: list[list[int]],
                     ctx=None) -> list[bytes]:
        """decrypt (prover.cpp:245-264) over a batch of equal-length bundles."""
        return self._xor([b.tx_hash for b in bundles],
                         [self.covered_mask(c) for c in contributors],
                         [b.ciphertext for b in bundles], ctx)

    def decrypt(self, bundle: WitnessBundle, contributors, ctx=None) -> bytes:
        if not bundle.ciphertext:
            return b""
        return self.decrypt_many([bundle], [list(contributors)], ctx)[0]


@dataclass
class BackupUnavailable:
    missing_tx_hashes: list[bytes] = field(default_factory=list)


def backup_prove(block: Block, bundles: dict, holders: dict, scheme: WitnessScheme,
                 ctx=None):
    """prover.cpp:266-299: decrypt every bundle with its holders' shares
    (batched keystream XOR on the GPU), validate every witness (batched HMAC
    check), then re-prove. Returns a FinalityCertificate byte-identical to the
    builder's, or BackupUnavailable listing the missing tx hashes in order."""
    t = scheme.threshold()
    txs = block.transactions
    hashes = sha256_many([tx.payload for tx in txs], ctx)
    missing, todo = [], []
    for i, h in enumerate(hashes):
        contributors = [v for v, held in sorted(holders.items()) if h in held]
        if h not in bundles or len(contributors) < t:
            missing.append(i)
        else:
            todo.append((i, contributors))
    ok_idx = set()
    by_len: dict[int, list] = {}
    for i, contrib in todo:
        by_len.setdefault(len(bundles[hashes[i]].ciphertext), []).append((i, contrib))
    for L, items in by_len.items():
        plain = scheme.decrypt_many([bundles[hashes[i]] for i, _ in items], [c for _, c in items],
                                    ctx) if L else [b""] * len(items)
        good = witnesses_match(plain, [txs[i] for i, _ in items], ctx)
        ok_idx.update(i for (i, _), g in zip(items, good) if g)
    missing = sorted(set(missing) | {i for i, _ in todo if i not in ok_idx})
    if missing:
        return BackupUnavailable([hashes[i] for i in missing])
    r = attest_prove_certify(block, ctx=ctx)
    return r.fc


# ------------------------------------------------------------- service
class ProverService:
    """SPSC hand-off between the slot scheduler and the proving thread
    (prover.hpp:141-172, prover.cpp:301-359); the worker runs the GPU
    pipeline, one block at a time, FIFO."""

    @dataclass
    class Result:
        block: Block
        fc: FinalityCertificate

    def __init__(self, ctx=None):
        self._ctx = ctx
        self._in: queue.Queue = queue.Queue()
        self._out: queue.Queue = queue.Queue()
        self._enq = 0
        self._proved = 0
        self._lock = threading.Lock()
        self._worker = threading.Thread(target=self._run, daemon=True)
        self._worker.start()

    def enqueue(self, block: Block) -> None:
        with self._lock:
            self._enq += 1
        self._in.put(block)

    def try_pop_result(self):
        try:
            return self._out.get_nowait()
        except queue.Empty:
            return None

    def wait_result(self) -> "ProverService.Result":
        return self._out.get()

    def blocks_enqueued(self) -> int:
        return self._enq

    def blocks_proved(self) -> int:
        return self._proved

    def _run(self) -> None:
        while True:
            block = self._in.get()
            if block is None:
                return
            r = attest_prove_certify(block, ctx=self._ctx)
            with self._lock:
                self._proved += 1
            self._out.put(ProverService.Result(block, r.fc))

    def close(self) -> None:
        self._in.put(None)
        self._worker.join()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
