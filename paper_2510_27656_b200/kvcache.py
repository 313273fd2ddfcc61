"""Paged KV-cache layer-by-layer transfer, prefill -> decode GPU (data path
of railtx.kvcache, kvcache.py:57-132, 477-507, 670-768).

Same layout contract as the reference: a region holds layers x heads x
slots pages, page (l, h, s) at index (l*heads + h)*slots + s
(kvcache.py:57-98); the prefiller ships each (chunk, layer) step as ONE
paged write carrying the request's immediate, plus one context write; the
decoder arms `expect_imm_count(imm, layers*chunks + 1)` before the request
can be seen, so completion never runs ahead of any payload byte
(kvcache.py:715-728).

On B200 each step is one sm_100a kernel on the prefiller's engine stream:
the 8-KiB pages move with TMA bulk copies straight into the decoder GPU's
page pool over NVLink, and the last CTA releases the receipt on the
decoder's ImmCounter slot.  The host control plane of the reference
(request messages, heartbeats, cancellation, the watcher-driven layer
clock) is out of scope: `KvRequest` is handed over
in-process (or pickled by the caller), and `LayerClock.advance` is the
caller invoking `send_step`.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .engine import ImmFlag, MrDesc, MrHandle, Pages, TransferEngine
from .errors import ProtocolError, ScheduleError


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
        self._imm_base = imm_base

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
        imm = self._imm_base + rid
        req = KvRequest(rid, layout, head_lo, head_lo + self.local_heads, self.local_heads,
                        self.pool_slots, self.kv_desc, slots, self.ctx_desc, 0, ctx_len, imm,
                        layout.expected_transfers)
        # the expectation exists before the prefiller can see the request
        flag = self.engine.expect_imm_count(imm, req.expected)
        return KvTicket(req, flag, slots)

    def release(self, ticket: KvTicket) -> None:
        self._free.extend(ticket.slots)

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
        self._plan = {}
        for k in range(1, req.layout.steps + 1):
            sp, dp = self.step_pages(req, k)
            self._plan[(req.request_id, k)] = (sp, dp, (self.engine.page_indices(sp), self.engine.page_indices(dp)))

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
