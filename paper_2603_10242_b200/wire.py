"""Wire formats the Prove path consumes and produces (reference
proj/include/ace/wire.hpp, proj/src/wire.cpp).

Encodings are host-side byte layout only; every hash (block_hash,
merkle_root, tx/attest roots) runs on the GPU through libacegpu.

``FlatBlock`` is the device-friendly layout shared with the C ABI: one
concatenated payload buffer + u64 offsets, n x 104-B attestation records and
the 256-B header. ``Block`` is the object mirror of ``wire::Block``.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

from . import _native as N

CANONICAL_TRANSFER_PAYLOAD_SIZE = 154  # wire.hpp:47
HEADER_BYTES = 256                     # wire.hpp:79
FC_BYTES = 328                         # wire.hpp:91
ATTESTATION_BYTES = 104                # crypto.hpp:76
ZERO32 = b"\0" * 32


@dataclass(frozen=True)
class Domain:
    """2-byte chain id + 48-bit slot (crypto.hpp:49-59)."""
    chain_id: int = 0
    slot: int = 0
    MAX_SLOT = (1 << 48) - 1

    def encode(self) -> bytes:
        return struct.pack(">H", self.chain_id) + (self.slot & self.MAX_SLOT).to_bytes(6, "big")

    @staticmethod
    def decode(b: bytes) -> "Domain | None":
        if len(b) != 8:
            return None
        return Domain(struct.unpack(">H", b[:2])[0], int.from_bytes(b[2:8], "big"))


@dataclass
class Attestation:
    """obj_hash | id_com | domain | credential, 104 B (crypto.cpp:56-76)."""
    obj_hash: bytes = ZERO32
    id_com: bytes = ZERO32
    domain: Domain = field(default_factory=Domain)
    credential: bytes = ZERO32

    def encode(self) -> bytes:
        return self.obj_hash + self.id_com + self.domain.encode() + self.credential

    @staticmethod
    def decode(b: bytes) -> "Attestation | None":
        if len(b) != ATTESTATION_BYTES:
            return None
        return Attestation(bytes(b[:32]), bytes(b[32:64]), Domain.decode(bytes(b[64:72])),
                           bytes(b[72:104]))


@dataclass
class Transaction:
    payload: bytes = b""
    attestation: Attestation = field(default_factory=Attestation)
    context_tag: bytes = b""


@dataclass
class BlockHeader:
    slot_number: int = 0
    parent_hash: bytes = ZERO32
    state_root: bytes = ZERO32
    tx_merkle_root: bytes = ZERO32
    attest_merkle_root: bytes = ZERO32
    poh_hash: bytes = ZERO32
    leader_id_com: bytes = ZERO32
    timestamp_ms: int = 0
    tx_count: int = 0

    def encode(self) -> bytes:
        """212 field bytes zero-padded to 256 (wire.cpp:74-98)."""
        h = (struct.pack(">Q", self.slot_number) + self.parent_hash + self.state_root
             + self.tx_merkle_root + self.attest_merkle_root + self.poh_hash + self.leader_id_com
             + struct.pack(">QI", self.timestamp_ms, self.tx_count))
        assert len(h) == 212
        return h + b"\0" * 44

    @staticmethod
    def decode(b: bytes) -> "BlockHeader | None":
        if len(b) != HEADER_BYTES or any(b[212:]):
            return None
        f = [b[8 + 32 * i: 40 + 32 * i] for i in range(6)]
        ts, cnt = struct.unpack(">QI", b[200:212])
        return BlockHeader(struct.unpack(">Q", b[:8])[0], *map(bytes, f), ts, cnt)


@dataclass
class Block:
    header: BlockHeader = field(default_factory=BlockHeader)
    transactions: list[Transaction] = field(default_factory=list)

    def flatten(self) -> "FlatBlock":
        return FlatBlock.from_lists([t.payload for t in self.transactions],
                                    [t.attestation.encode() for t in self.transactions],
                                    self.header.encode())


@dataclass
class FinalityCertificate:
    block_hash: bytes = ZERO32
    slot_number: int = 0
    proof: bytes = b"\0" * 256
    public_inputs_commitment: bytes = ZERO32

    def encode(self) -> bytes:
        """block_hash | slot_be64 | proof | commitment = 328 B (wire.cpp:125-133)."""
        return (self.block_hash + struct.pack(">Q", self.slot_number) + self.proof
                + self.public_inputs_commitment)

    @staticmethod
    def decode(b: bytes) -> "FinalityCertificate | None":
        if len(b) != FC_BYTES:
            return None
        return FinalityCertificate(bytes(b[:32]), struct.unpack(">Q", b[32:40])[0],
                                   bytes(b[40:296]), bytes(b[296:328]))


@dataclass
class FlatBlock:
    """The C-ABI block layout (include/acegpu.h)."""
    payloads: np.ndarray   # uint8 concatenated payloads
    offs: np.ndarray       # uint64, n+1
    atts: np.ndarray       # uint8, n*104
    header: np.ndarray     # uint8, 256

    @property
    def n(self) -> int:
        return len(self.offs) - 1

    @staticmethod
    def from_lists(payloads: list[bytes], atts: list[bytes], header: bytes) -> "FlatBlock":
        offs = np.zeros(len(payloads) + 1, np.uint64)
        if payloads:
            offs[1:] = np.cumsum([len(p) for p in payloads])
        pl = np.frombuffer(b"".join(payloads) + b"\0" * 16, np.uint8).copy()
        at = np.frombuffer(b"".join(atts) + b"\0" * 8, np.uint8).copy()
        return FlatBlock(pl, offs, at, np.frombuffer(header, np.uint8).copy())

    def to_block(self) -> Block:
        txs = []
        for i in range(self.n):
            p = self.payloads[self.offs[i]:self.offs[i + 1]].tobytes()
            txs.append(Transaction(p, Attestation.decode(self.atts[104 * i:104 * i + 104].tobytes())))
        return Block(BlockHeader.decode(self.header.tobytes()), txs)


# ------------------------------------------------------------------ codecs
def make_transfer_payload(frm: bytes, to: bytes, amount: int, nonce: int,
                          recent_blockhash: bytes) -> bytes:
    """TxPayload::encode of the 2-account transfer (wire.cpp:7-22, :59-72)."""
    return (struct.pack(">HQB", 1, nonce, 2) + frm + b"\x01" + to + b"\x01" + ZERO32
            + recent_blockhash + struct.pack(">H", 11) + bytes([1, 0, 1])
            + struct.pack(">Q", amount))


def encode_transaction_record(tx: Transaction) -> bytes:
    """u32 record_len | u16 payload_len | payload | u8 tag_len | tag | att (wire.cpp:145-158)."""
    body = (struct.pack(">H", len(tx.payload)) + tx.payload + bytes([len(tx.context_tag)])
            + tx.context_tag + tx.attestation.encode())
    return struct.pack(">I", len(body)) + body


def encode_block(b: Block) -> bytes:
    return b.header.encode() + b"".join(encode_transaction_record(t) for t in b.transactions)


def decode_block(raw: bytes) -> Block | None:
    """wire.cpp:160-212."""
    if len(raw) < HEADER_BYTES:
        return None
    h = BlockHeader.decode(raw[:HEADER_BYTES])
    if h is None:
        return None
    off, txs = HEADER_BYTES, []
    while off < len(raw):
        if off + 4 > len(raw):
            return None
        blen = struct.unpack(">I", raw[off:off + 4])[0]
        rec = raw[off + 4: off + 4 + blen]
        if len(rec) != blen or blen < 3:
            return None
        plen = struct.unpack(">H", rec[:2])[0]
        if 2 + plen + 1 > blen:
            return None
        p = rec[2:2 + plen]
        tl = rec[2 + plen]
        if 3 + plen + tl + ATTESTATION_BYTES != blen:
            return None
        tag = rec[3 + plen:3 + plen + tl]
        att = Attestation.decode(rec[3 + plen + tl:])
        if att is None:
            return None
        txs.append(Transaction(bytes(p), att, bytes(tag)))
        off += 4 + blen
    if len(txs) != h.tx_count:
        return None
    return Block(h, txs)


# ------------------------------------------------------------- GPU hashing
def sha256_many(msgs: list[bytes], ctx: N.Context | None = None) -> list[bytes]:
    """sha256::digest over many messages in one GPU batch."""
    if not msgs:
        return []
    ctx = ctx or N.context()
    offs = np.zeros(len(msgs) + 1, np.uint64)
    offs[1:] = np.cumsum([len(m) for m in msgs])
    data = np.frombuffer(b"".join(msgs) + b"\0" * 16, np.uint8).copy()
    out = np.zeros(32 * len(msgs), np.uint8)
    ctx.call("acegpu_sha256_varlen", N.addr(data), N.addr(offs), len(msgs), N.addr(out))
    return [out[32 * i:32 * i + 32].tobytes() for i in range(len(msgs))]


def sha256(data: bytes, ctx: N.Context | None = None) -> bytes:
    return sha256_many([data], ctx)[0]


def merkle_root(leaves: list[bytes], ctx: N.Context | None = None) -> bytes:
    """Domain-separated binary Merkle root; odd level duplicates its last node;
    empty = 0^32 (wire.cpp:223-255)."""
    if not leaves:
        return ZERO32
    ctx = ctx or N.context()
    arr = np.frombuffer(b"".join(leaves), np.uint8).copy()
    out = np.zeros(32, np.uint8)
    ctx.call("acegpu_merkle_root", N.addr(arr), len(leaves), N.addr(out))
    return out.tobytes()


def block_hash(b: "Block | BlockHeader | bytes", ctx: N.Context | None = None) -> bytes:
    """SHA-256 of the 256-B header encoding (wire.cpp:214-221)."""
    if isinstance(b, Block):
        b = b.header
    if isinstance(b, BlockHeader):
        b = b.encode()
    ctx = ctx or N.context()
    hdr = np.frombuffer(bytes(b), np.uint8).copy()
    out = np.zeros(32, np.uint8)
    ctx.call("acegpu_block_hash", N.addr(hdr), N.addr(out))
    return out.tobytes()


def tx_merkle_root(txs: list[Transaction], ctx: N.Context | None = None) -> bytes:
    return merkle_root(sha256_many([t.payload for t in txs], ctx), ctx)


def attest_merkle_root(txs: list[Transaction], ctx: N.Context | None = None) -> bytes:
    return merkle_root(sha256_many([t.attestation.encode() for t in txs], ctx), ctx)
