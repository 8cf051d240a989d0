"""Party transport across processes / GPUs.

The co-resident runtime (net.py) hands device tensors between threads.  When
the three servers run as separate processes -- one per GPU, or on different
hosts -- :class:`DistPartyRuntime` carries the same ``rt`` protocol
(src/net.py:236-289) over ``torch.distributed`` point-to-point:

* party i is rank ``ranks[i-1]`` of a process group;
* a message is a fixed-size int64 header tensor (session, round, op, head
  length, payload element count, payload dtype) + the head bytes + the
  payload tensor;
* with NCCL the payload moves device-to-device over NVLink; with gloo it is
  staged through host memory (CPU-only tests; several party processes on one
  GPU);
* round counters, session/op checks and their ProtocolError messages, the
  Meter and the reference-format transcript are the same as net.py's, so a
  distributed run's transcript digests equal the co-resident run's.
"""

from __future__ import annotations

import hashlib

import torch
import torch.distributed as dist

from .errors import ProtocolError
from .net import _HEADER, FRAME_MAGIC, OP_NAMES, Message, Meter, PartyConfig, as_message, next_party, prev_party

_DTYPES = [torch.int32, torch.uint8, torch.int64]
_HDR_LEN = 8


class DistLink:
    """Link to one peer rank with per-op round counters (src/net.py:131-165)."""

    def __init__(self, peer_rank: int, session: int, transcript, device, group=None):
        self.peer = peer_rank
        self.session = session
        self._tx: dict = {}
        self._rx: dict = {}
        self._transcript = transcript
        self.device = device
        self.group = group
        self.staged = dist.get_backend(group) != "nccl"
        self.pending: list = []

    def flush(self) -> None:
        for w, _ in self.pending:
            w.wait()
        self.pending = []

    def _frame(self, rnd, op, msg: Message) -> bytes:
        body = msg.payload_bytes()
        return _HEADER.pack(FRAME_MAGIC, self.session, rnd, op, len(body)) + body

    def _dev(self, t: torch.Tensor) -> torch.Tensor:
        return t.cpu() if self.staged else t.to(self.device)

    def send(self, op: int, msg: Message) -> int:
        rnd = self._tx.get(op, 0)
        self._tx[op] = rnd + 1
        payload = msg.tensor.contiguous() if msg.tensor is not None else None
        code = _DTYPES.index(payload.dtype) if payload is not None else -1
        hdr = torch.tensor([self.session, rnd, op, len(msg.head), payload.numel() if payload is not None else -1,
                            code, 0, 0], dtype=torch.int64)
        # asynchronous: every party sends before it receives (ring patterns),
        # so a blocking send would deadlock; buffers stay referenced until done
        parts = [self._dev(hdr)]
        if msg.head:
            parts.append(self._dev(torch.frombuffer(bytearray(msg.head), dtype=torch.uint8)))
        if payload is not None and payload.numel():
            parts.append(self._dev(payload))
        for t in parts:
            self.pending.append((dist.isend(t, self.peer, group=self.group), t))
        self.pending = [(w, t) for w, t in self.pending if not w.is_completed()]
        if self._transcript is not None:
            self._transcript.update(b"S" + self._frame(rnd, op, msg))
        return _HEADER.size + msg.nbytes

    def recv(self, op: int) -> Message:
        hdr = self._dev(torch.zeros(_HDR_LEN, dtype=torch.int64))
        dist.recv(hdr, self.peer, group=self.group)
        session, rnd, fop, hlen, numel, code = (int(v) for v in hdr.cpu()[:6])
        head = b""
        if hlen:
            hb = self._dev(torch.zeros(hlen, dtype=torch.uint8))
            dist.recv(hb, self.peer, group=self.group)
            head = bytes(hb.cpu().numpy())
        tensor = None
        if numel >= 0:
            t = torch.empty(numel, dtype=_DTYPES[code], device="cpu" if self.staged else self.device)
            if numel:
                dist.recv(t, self.peer, group=self.group)
            tensor = t.to(self.device) if self.staged else t
        if session != self.session:
            raise ProtocolError(f"session mismatch: got {session}, expected {self.session}")
        if fop != op:
            raise ProtocolError(f"expected op {OP_NAMES.get(op, op)}, got {OP_NAMES.get(fop, fop)}")
        expected = self._rx.get(op, 0)
        if rnd != expected:
            raise ProtocolError(f"round skew on op {OP_NAMES.get(op, op)}: got {rnd}, expected {expected}")
        self._rx[op] = expected + 1
        msg = Message(head, tensor)
        if self._transcript is not None:
            self._transcript.update(b"R" + self._frame(rnd, op, msg))
        return msg


class DistPartyRuntime:
    """Party ``config.party_index`` of a session whose parties are ranks
    ``ranks`` (party i = ranks[i-1]) of ``group``; same interface as
    net.PartyRuntime, so engine.sec_match runs unchanged."""

    def __init__(self, config: PartyConfig, ranks=(0, 1, 2), group=None, transcript: bool = False, device=None):
        from .rss import ZeroShareContext

        self.index = config.party_index
        self.session = config.session
        self.config = config
        self.zs = ZeroShareContext(config.zero_key_own, config.zero_key_prev)
        self.seed_with_next = config.seed_with_next
        self.seed_with_prev = config.seed_with_prev
        self.meter = Meter()
        self.opened: list = []
        self._table_counter = 0
        if transcript:
            self._transcript = hashlib.sha256()
            self._transcript.update(b"OGM-transcript:%d:%d" % (config.session, config.party_index))
        else:
            self._transcript = None
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu"))
        self._next = next_party(self.index)
        self._prev = prev_party(self.index)
        self.links = {p: DistLink(ranks[p - 1], self.session, self._transcript, self.device, group)
                      for p in (self._next, self._prev)}

    def _send(self, peer: int, op: int, payload, logical_bits: int) -> None:
        self.meter.record_send(self.links[peer].send(op, as_message(payload)), logical_bits)

    def send_next(self, op: int, payload, logical_bits: int = 0) -> None:
        self._send(self._next, op, payload, logical_bits)

    def send_prev(self, op: int, payload, logical_bits: int = 0) -> None:
        self._send(self._prev, op, payload, logical_bits)

    def recv_next(self, op: int) -> Message:
        return self.links[self._next].recv(op)

    def recv_prev(self, op: int) -> Message:
        return self.links[self._prev].recv(op)

    def zero_share(self, nbits: int):
        return self.zs.next_share(nbits)

    def alloc_table_id(self) -> int:
        tid = self._table_counter
        self._table_counter += 1
        return tid

    def note_opened(self, label: int, plaintext) -> None:
        self.opened.append((label, plaintext))

    def flush(self) -> None:
        """Wait for this party's outstanding sends."""
        for link in self.links.values():
            link.flush()

    def transcript_digest(self) -> str:
        if self._transcript is None:
            raise RuntimeError("runtime was created without transcript hashing")
        return self._transcript.hexdigest()
