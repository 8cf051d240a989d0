"""Three-party runtime with device-resident messages (src/net.py, device side).

The reference runs each party on a thread and moves bytes through framed
queues or TCP (src/net.py:27-165).  Here the three logical servers share one
GPU: a message is a device tensor handed to the peer's thread together with a
CUDA event, so nothing crosses PCIe.  What the reference's runtime guarantees
is kept:

* per-(link, op) round counters with the same ProtocolError messages
  (src/net.py:150-165), session ids, op codes;
* the Meter's byte / frame / logical-bit accounting per phase, counting
  exactly the bytes the reference frames would carry (src/net.py:168-199);
* optional transcript hashing: with ``transcript=True`` every message is
  copied to the host and hashed in the reference's frame encoding, so
  ``transcript_digest()`` is byte-comparable with the reference's
  (src/net.py:288-295) -- used by the parity tests;
* run_trio poisons peers when one party fails (src/net.py:320-373).

Each party runs on its own CUDA stream (one per thread); ctypes calls into
libogm_b200.so release the GIL.
"""

from __future__ import annotations

import hashlib
import queue
import struct
import threading
from contextlib import contextmanager
from dataclasses import dataclass, field

import numpy as np
import torch

from .errors import ProtocolError
from .prf import derive_key

FRAME_MAGIC = b"OGMF"
_HEADER = struct.Struct("<4sIIHI")

OP_SETUP = 1
OP_RESHARE = 2
OP_OPEN = 3
OP_SHUFFLE = 4
OP_NAMES = {OP_SETUP: "setup", OP_RESHARE: "reshare", OP_OPEN: "open", OP_SHUFFLE: "shuffle"}


@dataclass
class Message:
    """Payload = ``head`` bytes followed by the bytes of ``tensor`` (if any)."""

    head: bytes
    tensor: torch.Tensor | None = None
    event: torch.cuda.Event | None = None

    @property
    def nbytes(self) -> int:
        t = 0 if self.tensor is None else self.tensor.numel() * self.tensor.element_size()
        return len(self.head) + t

    def payload_bytes(self) -> bytes:
        if self.tensor is None:
            return self.head
        return self.head + self.tensor.detach().contiguous().cpu().numpy().tobytes()


def as_message(payload) -> Message:
    if isinstance(payload, Message):
        return payload
    if isinstance(payload, torch.Tensor):
        return Message(b"", payload)
    return Message(bytes(payload))


class DeviceChannel:
    """One direction of an in-process link (thread-safe queue of messages)."""

    _CLOSE = object()

    def __init__(self):
        self._q: queue.Queue = queue.Queue()

    def put(self, item) -> None:
        self._q.put(item)

    def get(self, timeout: float):
        try:
            item = self._q.get(timeout=timeout)
        except queue.Empty:
            raise ProtocolError("receive timed out") from None
        if item is self._CLOSE:
            raise ProtocolError("channel closed by peer failure")
        return item

    def close(self) -> None:
        self._q.put(self._CLOSE)


class PeerLink:
    """Link to one peer with per-op round counters (src/net.py:131-165)."""

    def __init__(self, send_ch: DeviceChannel, recv_ch: DeviceChannel, session: int, transcript):
        self._send_ch = send_ch
        self._recv_ch = recv_ch
        self.session = session
        self._tx: dict[int, int] = {}
        self._rx: dict[int, int] = {}
        self._transcript = transcript

    def _frame(self, rnd: int, op: int, msg: Message) -> bytes:
        body = msg.payload_bytes()
        return _HEADER.pack(FRAME_MAGIC, self.session, rnd, op, len(body)) + body

    def send(self, op: int, msg: Message) -> int:
        rnd = self._tx.get(op, 0)
        self._tx[op] = rnd + 1
        if msg.tensor is not None and msg.tensor.is_cuda:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(msg.tensor.device))
            msg.event = ev
        if self._transcript is not None:
            self._transcript.update(b"S" + self._frame(rnd, op, msg))
        self._send_ch.put((self.session, rnd, op, msg))
        return _HEADER.size + msg.nbytes

    def recv(self, op: int, timeout: float) -> Message:
        session, rnd, fop, msg = self._recv_ch.get(timeout)
        if session != self.session:
            raise ProtocolError(f"session mismatch: got {session}, expected {self.session}")
        if fop != op:
            raise ProtocolError(f"expected op {OP_NAMES.get(op, op)}, got {OP_NAMES.get(fop, fop)}")
        expected = self._rx.get(op, 0)
        if rnd != expected:
            raise ProtocolError(f"round skew on op {OP_NAMES.get(op, op)}: got {rnd}, expected {expected}")
        self._rx[op] = expected + 1
        if msg.tensor is not None and msg.tensor.is_cuda:
            cur = torch.cuda.current_stream(msg.tensor.device)
            if msg.event is not None:
                cur.wait_event(msg.event)
            msg.tensor.record_stream(cur)
        if self._transcript is not None:
            self._transcript.update(b"R" + self._frame(rnd, op, msg))
        return msg


@dataclass
class PhaseStats:
    """Frames, wire bytes and logical bits sent (src/net.py:168-178)."""

    bytes_sent: int = 0
    frames_sent: int = 0
    logical_bits: int = 0

    def add(self, nbytes: int, bits: int) -> None:
        self.bytes_sent, self.frames_sent, self.logical_bits = (
            self.bytes_sent + nbytes, self.frames_sent + 1, self.logical_bits + bits)


class Meter:
    """Per-party traffic accounting by protocol phase (src/net.py:180-199):
    sends count toward the total and toward the innermost open phase
    ("(none)" outside every phase)."""

    def __init__(self):
        self.total = PhaseStats()
        self.phases: dict[str, PhaseStats] = {}
        self._open: list[str] = []

    @contextmanager
    def phase(self, name: str):
        depth = len(self._open)
        self._open.append(name)
        try:
            yield
        finally:
            del self._open[depth:]

    def record_send(self, nbytes: int, logical_bits: int) -> None:
        current = self._open[-1] if self._open else "(none)"
        for stats in (self.total, self.phases.setdefault(current, PhaseStats())):
            stats.add(nbytes, logical_bits)


@dataclass
class PartyConfig:
    """Key material for one party (src/net.py:202-218)."""

    party_index: int
    session: int
    zero_key_own: bytes
    zero_key_prev: bytes
    seed_with_next: bytes
    seed_with_prev: bytes
    bind: str | None = None
    peers: dict[int, str] = field(default_factory=dict)


def make_session_configs(master: bytes, session: int = 1) -> list[PartyConfig]:
    """src/net.py:221-233 (same derivation, so the same master gives the same keys)."""
    k = {i: derive_key(master, f"zero-key-{i}") for i in (1, 2, 3)}
    s = {(1, 2): derive_key(master, "pair-seed-12"), (2, 3): derive_key(master, "pair-seed-23"),
         (3, 1): derive_key(master, "pair-seed-31")}
    return [
        PartyConfig(1, session, k[1], k[3], s[(1, 2)], s[(3, 1)]),
        PartyConfig(2, session, k[2], k[1], s[(2, 3)], s[(1, 2)]),
        PartyConfig(3, session, k[3], k[2], s[(3, 1)], s[(2, 3)]),
    ]


def next_party(i: int) -> int:
    return i % 3 + 1


def prev_party(i: int) -> int:
    return (i + 1) % 3 + 1


_STREAMS: dict = {}
_STREAMS_LOCK = threading.Lock()


def _party_stream(device: torch.device, party: int) -> torch.cuda.Stream:
    """One CUDA stream per (device, party index), reused by every session:
    the caching allocator pools blocks per stream, so a fresh stream per
    session would start from an empty pool (cudaMalloc on every query)."""
    key = (device.index, party)
    with _STREAMS_LOCK:
        st = _STREAMS.get(key)
        if st is None:
            st = _STREAMS[key] = torch.cuda.Stream(device=device)
    return st


class PartyRuntime:
    """One party's handle on a live session (src/net.py:236-289), device messages."""

    def __init__(self, config: PartyConfig, links: dict[int, PeerLink], transcript=None,
                 recv_timeout: float = 120.0, device: int | None = None):
        from .rss import ZeroShareContext

        self.config, self.links, self.recv_timeout = config, links, recv_timeout
        self.index, self.session = config.party_index, config.session
        self.seed_with_next, self.seed_with_prev = config.seed_with_next, config.seed_with_prev
        self.zs = ZeroShareContext(config.zero_key_own, config.zero_key_prev)   # src/rss.py:129-154
        self.meter = Meter()
        self.opened: list[tuple[int, object]] = []   # (label, plaintext) of every open, in order
        self._next, self._prev = next_party(self.index), prev_party(self.index)
        self._table_counter = 0
        self._transcript = transcript
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.stream = _party_stream(self.device, self.index)

    def _send(self, peer: int, op: int, payload, logical_bits: int) -> None:
        nbytes = self.links[peer].send(op, as_message(payload))
        self.meter.record_send(nbytes, logical_bits)

    def send_next(self, op: int, payload, logical_bits: int = 0) -> None:
        self._send(self._next, op, payload, logical_bits)

    def send_prev(self, op: int, payload, logical_bits: int = 0) -> None:
        self._send(self._prev, op, payload, logical_bits)

    def recv_next(self, op: int) -> Message:
        return self.links[self._next].recv(op, self.recv_timeout)

    def recv_prev(self, op: int) -> Message:
        return self.links[self._prev].recv(op, self.recv_timeout)

    def zero_share(self, nbits: int):
        return self.zs.next_share(nbits)

    def alloc_table_id(self) -> int:
        tid = self._table_counter
        self._table_counter += 1
        return tid

    def note_opened(self, label: int, plaintext) -> None:
        self.opened.append((label, plaintext))

    def transcript_digest(self) -> str:
        if self._transcript is None:
            raise RuntimeError("runtime was created without transcript hashing")
        return self._transcript.hexdigest()


def _new_transcript(config: PartyConfig):
    h = hashlib.sha256()
    h.update(b"OGM-transcript:%d:%d" % (config.session, config.party_index))
    return h


def local_runtimes(configs: list[PartyConfig], recv_timeout: float = 120.0,
                   transcript: bool = False, device: int | None = None) -> list[PartyRuntime]:
    """Wire three co-resident parties (src/net.py:298-317)."""
    if sorted(c.party_index for c in configs) != [1, 2, 3]:
        raise ValueError("configs must cover party indices 1, 2, 3 exactly")
    configs = sorted(configs, key=lambda c: c.party_index)
    if len({c.session for c in configs}) != 1:
        raise ValueError("configs disagree on session id")
    q = {(i, j): DeviceChannel() for i in (1, 2, 3) for j in (1, 2, 3) if i != j}
    out = []
    for cfg in configs:
        i = cfg.party_index
        tr = _new_transcript(cfg) if transcript else None
        links = {j: PeerLink(q[(i, j)], q[(j, i)], cfg.session, tr) for j in (1, 2, 3) if j != i}
        out.append(PartyRuntime(cfg, links, tr, recv_timeout, device))
    meeting = CoResidentMeeting()
    for rt in out:
        rt.meeting = meeting   # engine.sec_match's co-resident fast path (off with transcripts)
    return out


class CoResidentMeeting:
    """Where the three co-resident runtimes of one local session meet.

    Each party thread calls ``meet(rt, item, fn)``; the third arrival runs
    ``fn({1: item1, 2: item2, 3: item3})`` once (on its own CUDA stream, which
    it synchronises) and every caller gets the result -- or the exception it
    raised.  A caller whose peers do not arrive within ``rt.recv_timeout``
    gets a ProtocolError, like a receive that times out."""

    def __init__(self):
        self._cv = threading.Condition()
        self._pending: dict = {}
        self._done: dict = {}    # round -> [result, callers still to collect]
        self._round = 0

    def meet(self, rt, item, fn):
        with self._cv:
            rnd = self._round
            if rt.index in self._pending:
                raise ProtocolError(f"party {rt.index} entered the co-resident meeting twice")
            self._pending[rt.index] = item
            if len(self._pending) == 3:
                calls, self._pending = self._pending, {}
                try:
                    res = fn(calls)
                    torch.cuda.current_stream().synchronize()
                except BaseException as exc:  # noqa: BLE001
                    res = exc
                self._done[rnd] = [res, 3]
                self._round += 1
                self._cv.notify_all()
            elif not self._cv.wait_for(lambda: self._round > rnd, timeout=rt.recv_timeout):
                self._pending.pop(rt.index, None)
                raise ProtocolError(f"party {rt.index}: co-resident peers did not reach sec_match (timeout)")
            entry = self._done[rnd]
            entry[1] -= 1
            if entry[1] == 0:
                del self._done[rnd]
        if isinstance(entry[0], BaseException):
            raise entry[0]
        return entry[0]


def _is_channel_closed(exc: BaseException) -> bool:
    return isinstance(exc, ProtocolError) and "closed" in str(exc)


class _PartyThreads:
    """Three long-lived party threads reused by run_trio: starting and
    joining three fresh threads cost ~0.4 ms per call (measured on the C1
    query, 2.4 ms end to end).  One call at a time; a call that finds them
    busy (e.g. run_trio from inside a party) starts fresh threads."""

    def __init__(self):
        self.lock = threading.Lock()
        self.jobs = [queue.SimpleQueue() for _ in range(3)]
        self.done = queue.SimpleQueue()
        for i in range(3):
            threading.Thread(target=self._loop, args=(i,), name=f"party-{i + 1}", daemon=True).start()

    def _loop(self, i: int):
        while True:
            job = self.jobs[i].get()
            job()
            self.done.put(i)

    def run(self, jobs: list) -> bool:
        if not self.lock.acquire(blocking=False):
            return False
        try:
            for q, job in zip(self.jobs, jobs):
                q.put(job)
            for _ in jobs:
                self.done.get()
        finally:
            self.lock.release()
        return True


# run_trio on the three long-lived party threads (False: fresh threads per call, as
# the reference); measured on the C1 per-party query: 1.89 vs 2.27 ms
USE_PARTY_THREADS = True
_PARTY_THREADS: _PartyThreads | None = None
_PARTY_THREADS_LOCK = threading.Lock()


def _party_threads() -> _PartyThreads:
    global _PARTY_THREADS
    with _PARTY_THREADS_LOCK:
        if _PARTY_THREADS is None:
            _PARTY_THREADS = _PartyThreads()
        return _PARTY_THREADS


def run_trio(worker, runtimes: list[PartyRuntime], close_channels=None):
    """Run ``worker(rt)`` for the three parties on threads, each on its own
    CUDA stream (src/net.py:320-351); re-raises the root-cause failure."""
    results: list = [None, None, None]
    errors: list = [None, None, None]
    if close_channels is None:
        chans = [link._send_ch for rt in runtimes for link in rt.links.values()]  # noqa: SLF001

        def close_channels():
            for ch in chans:
                ch.close()

    def run(idx: int, rt: PartyRuntime):
        try:
            torch.cuda.set_device(rt.device)
            with torch.cuda.stream(rt.stream):
                results[idx] = worker(rt)
                rt.stream.synchronize()
        except BaseException as exc:  # noqa: BLE001
            errors[idx] = exc
            close_channels()

    jobs = [(lambda i=i, rt=rt: run(i, rt)) for i, rt in enumerate(runtimes)]
    if len(jobs) != 3 or not USE_PARTY_THREADS or not _party_threads().run(jobs):
        threads = [threading.Thread(target=job, name=f"party-{rt.index}", daemon=True)
                   for job, rt in zip(jobs, runtimes)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    # the root cause first: a party that failed on its own, not on a channel another party closed
    failures = sorted((e for e in errors if e is not None), key=_is_channel_closed)
    if failures:
        raise failures[0]
    return results


def run_local_trio(worker, configs: list[PartyConfig] | None = None, master: bytes = b"\x00" * 16,
                   recv_timeout: float = 120.0, transcript: bool = False):
    """src/net.py:358-373."""
    if configs is None:
        configs = make_session_configs(master)
    return run_trio(worker, local_runtimes(configs, recv_timeout, transcript))


def u32le(x: int) -> bytes:
    return int(x).to_bytes(4, "little")


def tensor_words(t: torch.Tensor) -> np.ndarray:
    return t.detach().contiguous().cpu().numpy().view(np.uint32)
