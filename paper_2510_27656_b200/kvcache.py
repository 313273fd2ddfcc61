"""Paged KV-cache layer-by-layer transfer, prefill -> decode GPU (data path
of railtx.kvcache, kvcache.py:57-132, 477-507, 670-768).

Same layout contract as the reference: a region holds layers x heads x
slots pages, page (l, h, s) at index (l*heads + h)*slots + s
(kvcache.py:57-98); the prefiller ships each (chunk, layer) step as ONE
paged write carrying the request's immediate, plus one context write; the
decoder arms `expect_imm_count(imm, layers*chunks + 1)` before the request
can be seen, so completion never runs ahead of any payload byte
(kvcache.py:715-728).

On B200 the pages move with device stores straight into the decoder GPU's
page pool over NVLink, and the CTA that completes a step releases its
receipt on the decoder's ImmCounter.  Two ways to drive it:

  * `send_step` / `send_all`: one kernel per (chunk, layer) step, the host
    calling it as the reference's LayerClock advances;
  * `stream_all` with a `DeviceClock`: ONE persistent kernel for the whole
    request that moves step k as soon as the compute stream has advanced
    the clock to k (`clock.advance(stream)` after each layer's compute) --
    the reference's watcher-driven LayerClock (kvcache.py:317-334, 477-500)
    with the host taken out of the loop.

The host control plane of the reference (request messages, heartbeats,
cancellation) is out of scope: `KvRequest` is handed over
in-process (or pickled by the caller).
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .engine import CompletionFlag, DeviceClock, ImmFlag, MrDesc, MrHandle, Pages, TransferEngine
from .errors import ProtocolError, ScheduleError

IMM_RING_SIZE = 1 << 16   # kvcache.py:48


class ImmRing:
    """Allocator over a ring of imm values; a value stays out until retired
    (kvcache.py:289-314).  Bounds the distinct imms a decoder ever arms, so
    the engine's ImmCounter table never fills however many requests run."""

    def __init__(self, base: int = 0, size: int = IMM_RING_SIZE) -> None:
        if base < 0 or base + size > (1 << 32):
            raise ProtocolError("imm ring outside the u32 range")
        self._base = base
        self._size = size
        self._next = 0
        self._inuse: set[int] = set()
        self._lock = threading.Lock()

    def take(self) -> int:
        with self._lock:
            if len(self._inuse) >= self._size:
                raise ProtocolError("imm ring exhausted")
            while True:
                imm = self._base + self._next % self._size
                self._next += 1
                if imm not in self._inuse:
                    self._inuse.add(imm)
                    return imm

    def retire(self, imm: int) -> None:
        with self._lock:
            self._inuse.discard(imm)


@dataclass(frozen=True)
class KvLayout:
    """Shape of one request's KV payload (kvcache.py:57-98)."""

    layers: int
    chunks: int
    pages_per_chunk: int
    page_len: int

    def __post_init__(self) -> None:
        if self.layers < 0 or self.chunks < 0:
            raise ProtocolError("negative layer or chunk count")
        if self.pages_per_chunk <= 0 or self.page_len <= 0:
            raise ProtocolError("pages per chunk and page length must be positive")

    @property
    def steps(self) -> int:
        return self.layers * self.chunks

    @property
    def slots(self) -> int:
        return self.chunks * self.pages_per_chunk

    @property
    def expected_transfers(self) -> int:
        """One paged write per (chunk, layer) plus the context write."""
        return self.steps + 1

    def chunk_slots(self, chunk: int) -> range:
        k = self.pages_per_chunk
        return range(chunk * k, (chunk + 1) * k)

    def region_bytes(self, heads: int, slots: int) -> int:
        return self.layers * heads * slots * self.page_len

    def page_index(self, heads: int, slots: int, layer: int, head: int, slot: int) -> int:
        return (layer * heads + head) * slots + slot


@dataclass(frozen=True)
class ShardMap:
    """How attention heads map onto decoder ranks (kvcache.py:101-132):
    `mla` replicates all heads, `gqa` slices contiguous head ranges."""

    mode: str
    heads: int
    ranks: int

    def __post_init__(self) -> None:
        if self.mode not in ("mla", "gqa"):
            raise ProtocolError(f"unknown shard mode {self.mode!r}")
        if self.heads <= 0 or self.ranks <= 0:
            raise ProtocolError("heads and ranks must be positive")
        if self.mode == "gqa" and self.heads % self.ranks:
            raise ProtocolError(f"{self.heads} heads do not slice evenly over {self.ranks} ranks")

    def head_range(self, rank: int) -> tuple[int, int]:
        if not 0 <= rank < self.ranks:
            raise ProtocolError(f"rank {rank} outside 0..{self.ranks - 1}")
        if self.mode == "mla":
            return 0, self.heads
        per = self.heads // self.ranks
        return rank * per, (rank + 1) * per

    def local_heads(self, rank: int) -> int:
        lo, hi = self.head_range(rank)
        return hi - lo


@dataclass(frozen=True)
class KvRequest:
    """The fields of PrefillRequest (kvcache.py:179-244) the data path needs."""

    request_id: int
    layout: KvLayout
    head_lo: int
    head_hi: int
    dst_heads: int
    dst_slots: int
    kv_desc: MrDesc
    slot_list: tuple
    ctx_desc: MrDesc
    ctx_off: int
    ctx_len: int
    imm: int
    expected: int


@dataclass
class KvTicket:
    request: KvRequest
    flag: ImmFlag
    slots: tuple

    def wait(self, timeout: float | None = 30.0) -> bool:
        return self.flag.wait(timeout)

    def wait_device(self, stream=None) -> None:
        """Make GPU work queued on `stream` (attention over the new pages)
        wait for the transfer on the device, no host round trip."""
        self.flag.wait_device(stream)


class KvReceiver:
    """Decoder side: the page pool and the arming of the completion count
    (DecoderNode, kvcache.py:600-768, data path only)."""

    def __init__(self, engine: TransferEngine, layout: KvLayout, pool_slots: int, local_heads: int,
                 ctx_bytes: int = 1 << 20, imm_base: int = 1 << 20) -> None:
        if pool_slots < layout.slots:
            raise ScheduleError(f"pool of {pool_slots} slots cannot hold a {layout.slots}-slot request")
        self.engine = engine
        self.layout = layout
        self.pool_slots = pool_slots
        self.local_heads = local_heads
        nbytes = layout.region_bytes(local_heads, pool_slots)
        self.kv = engine.alloc_buffer(max(nbytes, 16))
        self.kv_handle, self.kv_desc = engine.reg_mr(self.kv)
        self.ctx = engine.alloc_buffer(ctx_bytes)
        self.ctx_handle, self.ctx_desc = engine.reg_mr(self.ctx)
        self._free = list(range(pool_slots))[::-1]
        self._next_rid = 1
        self._ring = ImmRing(base=imm_base)

    def open_request(self, head_lo: int = 0, ctx_len: int = 4096) -> KvTicket:
        """Reserve pool slots, arm the completion count, describe the
        destination (DecoderNode.request_prefill, kvcache.py:670-729)."""
        layout = self.layout
        if len(self._free) < layout.slots:
            raise ScheduleError(f"{len(self._free)} free KV slots, request needs {layout.slots}")
        if ctx_len > self.ctx.numel():
            raise ProtocolError("context slice outside its region")
        slots = tuple(self._free.pop() for _ in range(layout.slots))
        rid = self._next_rid
        self._next_rid += 1
        imm = self._ring.take()
        req = KvRequest(rid, layout, head_lo, head_lo + self.local_heads, self.local_heads,
                        self.pool_slots, self.kv_desc, slots, self.ctx_desc, 0, ctx_len, imm,
                        layout.expected_transfers)
        # the expectation exists before the prefiller can see the request
        flag = self.engine.expect_imm_count(imm, req.expected)
        return KvTicket(req, flag, slots)

    def release(self, ticket: KvTicket) -> None:
        """Return the pages and retire the imm (DecoderNode on fire /
        cancel, kvcache.py:741-768).  The imm's receipts were consumed by
        the fired expectation, so the value can be armed again."""
        self._free.extend(ticket.slots)
        self._ring.retire(ticket.request.imm)

    def page_view(self, ticket: KvTicket, layer: int, head: int, i: int) -> torch.Tensor:
        L = self.layout
        idx = L.page_index(self.local_heads, self.pool_slots, layer, head, ticket.slots[i])
        return self.kv[idx * L.page_len:(idx + 1) * L.page_len]


class KvSender:
    """Prefiller side: one paged write per (chunk, layer) step plus the
    context write (PrefillerNode._on_progress / _send_context,
    kvcache.py:477-507)."""

    def __init__(self, engine: TransferEngine, kv: torch.Tensor, ctx: torch.Tensor | None = None) -> None:
        self.engine = engine
        self.kv = kv
        self.kv_handle, _ = engine.reg_mr(kv)
        self.ctx_handle = engine.reg_mr(ctx)[0] if ctx is not None else None

    def step_pages(self, req: KvRequest, step: int) -> tuple[Pages, Pages]:
        """Source and destination pages of one (chunk, layer) step
        (kvcache.py:484-498)."""
        layout = req.layout
        if not 1 <= step <= layout.steps:
            raise ProtocolError(f"step {step} outside 1..{layout.steps}")
        nh = req.head_hi - req.head_lo
        chunk, layer = divmod(step - 1, layout.layers)
        src, dst = [], []
        for j in range(nh):
            for slot in layout.chunk_slots(chunk):
                src.append(layout.page_index(nh, layout.slots, layer, j, slot))
                dst.append((layer * req.dst_heads + j) * req.dst_slots + req.slot_list[slot])
        return Pages(tuple(src), layout.page_len), Pages(tuple(dst), layout.page_len)

    def prepare(self, req: KvRequest) -> None:
        """Precompute every step's page lists and upload their indices once,
        so each layer step is a single kernel launch."""
        L = req.layout
        si, di = self.step_indices(req)
        dev = torch.device("cuda", self.engine.device)
        si_d = torch.from_numpy(si).to(dev)
        di_d = torch.from_numpy(di).to(dev)
        pps = (req.head_hi - req.head_lo) * L.pages_per_chunk
        self._plan = {}
        for k in range(1, L.steps + 1):
            lo, hi = (k - 1) * pps, k * pps
            sp = Pages(tuple(si[lo:hi].tolist()), L.page_len)
            dp = Pages(tuple(di[lo:hi].tolist()), L.page_len)
            self._plan[(req.request_id, k)] = (sp, dp, (si_d[lo:hi], di_d[lo:hi]))

    def send_step(self, req: KvRequest, step: int):
        """Step in 1..layout.steps: chunk, layer = divmod(step - 1, layers)."""
        plan = getattr(self, "_plan", {}).get((req.request_id, step))
        if plan is None:
            sp, dp = self.step_pages(req, step)
            dev = None
        else:
            sp, dp, dev = plan
        return self.engine.submit_paged_writes(
            req.layout.page_len, (self.kv_handle, sp), (req.kv_desc, dp), imm=req.imm, device_indices=dev)

    def send_context(self, req: KvRequest):
        if self.ctx_handle is None:
            raise ProtocolError("no context buffer registered")
        return self.engine.submit_single_write(req.ctx_len, (self.ctx_handle, 0), (req.ctx_desc, req.ctx_off),
                                               imm=req.imm)

    def send_all(self, req: KvRequest):
        """Every step then the context (the order _on_progress produces)."""
        flags = [self.send_step(req, k) for k in range(1, req.layout.steps + 1)]
        flags.append(self.send_context(req))
        return flags

    def step_indices(self, req: KvRequest) -> tuple[np.ndarray, np.ndarray]:
        """Source / destination page numbers of every step, step-major
        ([steps * pages_per_step]); the same lists as step_pages, built with
        array arithmetic (kvcache.py:484-498)."""
        L = req.layout
        nh = req.head_hi - req.head_lo
        steps = np.arange(L.steps)
        chunk, layer = np.divmod(steps, L.layers)
        j = np.arange(nh)
        k = np.arange(L.pages_per_chunk)
        slot = chunk[:, None, None] * L.pages_per_chunk + k[None, None, :]          # [S, 1, K]
        src = (layer[:, None, None] * nh + j[None, :, None]) * L.slots + slot         # [S, nh, K]
        sl = np.asarray(req.slot_list, dtype=np.int64)
        dst = (layer[:, None, None] * req.dst_heads + j[None, :, None]) * req.dst_slots + sl[slot]
        return src.reshape(-1).astype(np.int64), dst.reshape(-1).astype(np.int64)

    def prepare_stream(self, req: KvRequest):
        """Device page lists and step tickets of a request for stream_all,
        built once (the host arithmetic and the upload stay out of the
        transfer)."""
        cache = getattr(self, "_stream_plan", None)
        if cache is not None and cache[0] == req.request_id and cache[1] is req:
            return cache[2]
        L = req.layout
        si, di = self.step_indices(req)
        dev = torch.device("cuda", self.engine.device)
        plan = (torch.from_numpy(si).to(dev), torch.from_numpy(di).to(dev),
                torch.zeros(max(1, L.steps), dtype=torch.int32, device=dev))
        self._stream_plan = (req.request_id, req, plan)
        return plan

    def stream_all(self, req: KvRequest, clock: DeviceClock, grid: int = 0, use_tma: bool | None = None,
                   timeout: float = 60.0) -> CompletionFlag:
        """Enqueue the whole request as ONE persistent kernel on the engine's
        stream: step k (1-based) moves once `clock` has reached k, and its
        receipt is released as soon as its pages are visible.  `grid` CTAs
        (default: every SM) -- fewer leave SMs to the compute that advances
        the clock.  Send the context with send_context afterwards (it is
        stream-ordered behind the last step, as in _on_progress)."""
        eng = self.engine
        L = req.layout
        if L.page_len % 16 or self.kv.data_ptr() % 16:
            raise ProtocolError("streamed pages must be 16-byte aligned")
        si_d, di_d, tickets = self.prepare_stream(req)
        dst_base, dst_imm = eng._peer_base(req.kv_desc)
        nh = req.head_hi - req.head_lo
        j = _lib.StreamJob()
        j.src, j.dst, j.page_len = self.kv.data_ptr(), dst_base, L.page_len
        j.src_idx, j.dst_idx = si_d.data_ptr(), di_d.data_ptr()
        j.pages_per_step, j.nsteps = nh * L.pages_per_chunk, L.steps
        j.use_tma = int(eng.use_tma if use_tma is None else use_tma)
        j.clock, j.clock_base = clock.ptr, 0
        j.imm_ctr = eng._imm_slot_ptr(req.imm, dst_imm)
        j.tickets = tickets.data_ptr()
        j.timeout_ns = int(timeout * 1e9)
        j.err = eng._err.data_ptr()
        j.single_device = eng._single_device(req.kv_desc)
        if eng.trace.enabled:  # one traced transfer per step (1280 Python calls at cfg5: only when traced)
            for k in range(L.steps):
                eng.post_op(f"kv.{req.request_id}.s{k + 1}", req.kv_desc.owner,
                            L.page_len * nh * L.pages_per_chunk, req.imm)
        with torch.cuda.device(eng.device):
            eng._after_current()
            for t in (si_d, di_d, tickets):
                t.record_stream(eng._stream)
            _lib.call("txb_kv_stream", C.byref(j), int(grid), C.c_void_p(eng._stream.cuda_stream))
            ev = torch.cuda.Event()
            ev.record(eng._stream)
        return CompletionFlag(ev)
