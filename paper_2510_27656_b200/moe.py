"""Expert-parallel token dispatch and combine on B200 (drop-in for railtx.moe).

Same public surface as the reference module (railtx/moe.py:36-939):
RoutingSpec, PrivateBufferConfig, RouteMatrix, DispatchLayout,
compute_layout, encode_tokens, decode_tokens, GroupedTokens, StepStats,
MoeRank.{dispatch_send, dispatch_recv, combine_send, combine_recv, close},
build_mesh -- with the same routing, buffer and grouped-layout conventions,
so outputs are byte-identical to the reference on the same inputs.

What changes underneath:
  * every step runs as five sm_100a kernels of libtxb200 (route/count,
    dispatch, receive, combine-send, combine-recv) on the caller's current
    CUDA stream; no host proxy, worker thread or CPU fallback;
  * tokens are stored by the sending GPU straight into their final grouped
    row on the receiving GPU (the reference's recv slab + pack_rows
    regroup, moe.py:699-722, collapses into one peer store), and completion
    is a release-add on the receiver's counter (the ImmCounter);
  * the speculative private-buffer round (moe.py:556-582) runs on the
    device: the first PrivateBufferConfig.tokens rows of each source's slab
    for a peer are stored into that peer's private slab before the route
    exchange completes, and moved to their grouped rows by the receiver.

Inputs may be numpy arrays (host mode: results come back as numpy, exactly
like the reference) or CUDA tensors (device mode: results stay on the GPU;
payload may also be f32/bf16 values, encoded inside the dispatch kernel).
"""

from __future__ import annotations

import dataclasses
import threading
import time
from dataclasses import dataclass
from typing import Sequence

import ctypes as C
import numpy as np
import torch

from . import _lib
from .engine import RegionDesc, TransferEngine
from .errors import ProtocolError
from .memory import Region, enable_peer_access, view

GROUP_PAD = 8           # moe.py:27
DEFAULT_PRIVATE = 32    # moe.py:28


# ----------------------------------------------------------- configuration


@dataclass(frozen=True)
class RoutingSpec:
    """Static shape of one expert-parallel deployment (moe.py:36-89).

    `elem_size` 1 carries fp8 e4m3 bytes plus f32 scale slots, 4 raw f32;
    2 (bf16 rows) is an extension.  `comb_elem_size`/`comb_scales` (also
    extensions) select the wire format of combine rows; by default combine
    rows use the dispatch format, as in the reference.
    """

    ranks: int
    experts: int
    max_tokens: int
    topk: int
    hidden: int = 256
    elem_size: int = 1
    scales: int = 8
    comb_elem_size: int | None = None
    comb_scales: int | None = None

    def __post_init__(self) -> None:
        if self.ranks < 1:
            raise ProtocolError("rank count must be positive")
        if self.experts < 1 or self.experts % self.ranks:
            raise ProtocolError(
                f"expert count {self.experts} is not a positive multiple of "
                f"{self.ranks} ranks")
        if not 1 <= self.topk <= self.experts:
            raise ProtocolError(f"topk {self.topk} outside 1..{self.experts}")
        if self.max_tokens < 1:
            raise ProtocolError("max_tokens must be positive")
        if self.hidden < 1:
            raise ProtocolError("hidden size must be positive")
        if self.elem_size not in (1, 2, 4):
            raise ProtocolError(f"element size {self.elem_size} not in (1, 2, 4)")
        if self.scales < 0:
            raise ProtocolError("scale count must be non-negative")
        if self.elem_size == 1 and self.scales < 1:
            raise ProtocolError("quantized payloads need at least one scale slot")
        ce, cs = self.comb_format
        if ce not in (1, 2, 4):
            raise ProtocolError(f"combine element size {ce} not in (1, 2, 4)")
        if cs < 0 or (ce == 1 and cs < 1):
            raise ProtocolError("combine rows need a non-negative scale count (>=1 for fp8)")

    @property
    def local_experts(self) -> int:
        return self.experts // self.ranks

    @property
    def payload_bytes(self) -> int:
        return self.hidden * self.elem_size + 4 * self.scales

    @property
    def comb_format(self) -> tuple[int, int]:
        if self.comb_elem_size is None:
            return self.elem_size, self.scales
        return self.comb_elem_size, (self.comb_scales if self.comb_scales is not None else 0)

    @property
    def comb_payload_bytes(self) -> int:
        ce, cs = self.comb_format
        return self.hidden * ce + 4 * cs

    def comb_spec(self) -> "RoutingSpec":
        ce, cs = self.comb_format
        return RoutingSpec(self.ranks, self.experts, self.max_tokens, self.topk,
                           self.hidden, ce, cs)

    @property
    def capacity(self) -> int:
        """Receive-slot upper bound per rank, valid for any admissible matrix."""
        return self.ranks * self.max_tokens * max(self.topk, self.local_experts)

    def owner(self, expert: int) -> int:
        return expert // self.local_experts

    def local_index(self, expert: int) -> int:
        return expert % self.local_experts


@dataclass(frozen=True)
class PrivateBufferConfig:
    """Per-source speculative receive slots (moe.py:92-102).  A source
    stores the first `tokens` rows of its slab for a peer into that peer's
    private slab before the route exchange completes (moe.py:556-582); the
    receiver moves them to their grouped rows once the layout is known."""

    tokens: int = DEFAULT_PRIVATE

    def validate(self, spec: RoutingSpec) -> None:
        if not 0 <= self.tokens <= spec.max_tokens:
            raise ProtocolError(
                f"private buffer of {self.tokens} tokens outside "
                f"0..{spec.max_tokens}")


@dataclass(frozen=True)
class RouteMatrix:
    """Per-source-rank, per-expert token copy counts (moe.py:105-139)."""

    spec: RoutingSpec
    counts: np.ndarray

    def __post_init__(self) -> None:
        spec = self.spec
        c = np.asarray(self.counts, dtype=np.int64)
        if c.shape != (spec.ranks, spec.experts):
            raise ProtocolError(f"count matrix shape {c.shape} != ({spec.ranks}, {spec.experts})")
        if (c < 0).any():
            raise ProtocolError("negative route count")
        limit = spec.max_tokens * spec.topk
        tot = c.sum(axis=1)
        for s in range(spec.ranks):
            if int(tot[s]) > limit:
                raise ProtocolError(f"source {s} routes {int(tot[s])} copies, limit {limit}")
        object.__setattr__(self, "counts", c)

    @classmethod
    def from_routes(cls, spec: RoutingSpec, routes_by_rank: Sequence[np.ndarray]) -> "RouteMatrix":
        if len(routes_by_rank) != spec.ranks:
            raise ProtocolError("one route array per rank required")
        counts = np.zeros((spec.ranks, spec.experts), dtype=np.int64)
        for s, routes in enumerate(routes_by_rank):
            r = _check_routes(spec, routes)
            if r.size:
                counts[s] = np.bincount(r.ravel(), minlength=spec.experts)
        return cls(spec, counts)


def _check_routes(spec: RoutingSpec, routes) -> np.ndarray:
    """moe.py:142-155 (vectorised; same checks, same messages)."""
    r = np.asarray(routes, dtype=np.int64)
    if r.ndim != 2 or r.shape[1] != spec.topk:
        raise ProtocolError(f"route array shape {r.shape} is not (tokens, {spec.topk})")
    if r.shape[0] > spec.max_tokens:
        raise ProtocolError(f"{r.shape[0]} tokens exceed the {spec.max_tokens}-token limit")
    if r.size and (r.min() < 0 or r.max() >= spec.experts):
        raise ProtocolError("expert index out of range")
    if r.shape[0] and spec.topk > 1:
        srt = np.sort(r, axis=1)
        dup = (srt[:, 1:] == srt[:, :-1]).any(axis=1)
        if dup.any():
            raise ProtocolError(f"token {int(np.argmax(dup))} routes to a duplicate expert")
    return r


# ------------------------------------------------------------------ layout


@dataclass(frozen=True, eq=False)
class DispatchLayout:
    """Dense receive-buffer ranges derived from one route matrix (moe.py:161-197)."""

    spec: RoutingSpec
    counts: np.ndarray
    assigned: np.ndarray
    recv_start: np.ndarray
    recv_total: np.ndarray
    send_start: np.ndarray

    def range_of(self, dst: int, local_expert: int, src: int) -> tuple[int, int]:
        base = dst * self.spec.local_experts
        e = base + local_expert
        start = int(self.recv_start[dst, src] + self.counts[src, base:e].sum())
        return start, int(self.counts[src, e])

    def ranges(self, dst: int) -> list[tuple[tuple[int, int], int, int]]:
        out = []
        for le in range(self.spec.local_experts):
            for s in range(self.spec.ranks):
                start, length = self.range_of(dst, le, s)
                out.append(((le, s), start, length))
        return out

    def private_take(self, private_tokens: int) -> np.ndarray:
        return np.minimum(self.assigned, private_tokens)


def compute_layout(spec: RoutingSpec, counts) -> DispatchLayout:
    """moe.py:200-225 (host helper; the device derives the same layout)."""
    matrix = counts if isinstance(counts, RouteMatrix) else RouteMatrix(spec, counts)
    c = matrix.counts
    n = spec.ranks
    assigned = c.reshape(n, n, spec.local_experts).sum(axis=2)
    recv_start = (np.cumsum(assigned, axis=0) - assigned).T.copy()
    recv_total = assigned.sum(axis=0)
    for d in range(n):
        if recv_total[d] > spec.capacity:
            raise ProtocolError(
                f"destination {d} needs {int(recv_total[d])} slots, capacity {spec.capacity}")
    send_start = np.cumsum(assigned, axis=1) - assigned
    return DispatchLayout(spec=spec, counts=c, assigned=assigned, recv_start=recv_start,
                          recv_total=recv_total, send_start=send_start)


# ----------------------------------------------------------- token payloads


def _stream(device: int):
    return torch.cuda.current_stream(device)


def _sp(t: torch.Tensor | None) -> C.c_void_p:
    return C.c_void_p(t.data_ptr() if t is not None else 0)


def _pinned(t) -> bool:
    """A page-locked CPU tensor the kernels can address in place."""
    return isinstance(t, torch.Tensor) and not t.is_cuda and t.is_pinned() and t.is_contiguous()


def _mapped(t: torch.Tensor) -> C.c_void_p:
    """Device address of a pinned host tensor (zero-copy over PCIe)."""
    out = C.c_void_p()
    _lib.call("txb_host_device_ptr", C.c_void_p(t.data_ptr()), C.byref(out))
    return out


def encode_tokens(spec: RoutingSpec, values):
    """[n, hidden] values -> [n, payload_bytes] wire rows (moe.py:231-246),
    on the GPU.  numpy in -> numpy out (current device); CUDA f32/bf16
    tensor in -> CUDA uint8 tensor out."""
    host = not isinstance(values, torch.Tensor)
    v = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float32)).cuda() if host \
        else values.contiguous()
    if v.ndim != 2 or v.shape[1] != spec.hidden:
        raise ProtocolError(f"value shape {tuple(v.shape)} is not (n, {spec.hidden})")
    if v.dtype not in (torch.float32, torch.bfloat16):
        v = v.float()
    kind = _lib.SRC_F32 if v.dtype == torch.float32 else _lib.SRC_BF16
    out = torch.empty((v.shape[0], spec.payload_bytes), dtype=torch.uint8, device=v.device)
    _lib.call("txb_encode_rows", _sp(v), kind, v.shape[0], spec.hidden, spec.elem_size,
              spec.scales, _sp(out), C.c_void_p(_stream(v.device.index).cuda_stream))
    return out.cpu().numpy() if host else out


def decode_tokens(spec: RoutingSpec, payload):
    """[m, payload_bytes] wire rows -> [m, hidden] f32 (moe.py:249-262)."""
    host = not isinstance(payload, torch.Tensor)
    p = torch.from_numpy(np.ascontiguousarray(payload, dtype=np.uint8)).cuda() if host \
        else payload.contiguous()
    if p.ndim != 2 or p.shape[1] != spec.payload_bytes:
        raise ProtocolError(f"payload shape {tuple(p.shape)} is not (n, {spec.payload_bytes})")
    out = torch.empty((p.shape[0], spec.hidden), dtype=torch.float32, device=p.device)
    _lib.call("txb_decode_rows", _sp(p), p.shape[0], spec.hidden, spec.elem_size, spec.scales,
              _sp(out), C.c_void_p(_stream(p.device.index).cuda_stream))
    return out.cpu().numpy() if host else out


# ----------------------------------------------------------------- results


@dataclass
class GroupedTokens:
    """Receive-side tokens regrouped per local expert (moe.py:268-285).

    Device mode: `data`, `rows`, `sources` are CUDA tensors that alias the
    rank's receive region (valid until the next dispatch_send);
    group_sizes/group_starts are host int64 tensors.  Host mode: numpy
    copies, exactly as the reference returns them.  In no-sync mode
    (dispatch_recv(sync=False)) data/rows/sources span the whole receive
    region, group_sizes/group_starts are device tensors and
    `padded_total` is a 0-d device tensor.
    """

    data: object
    group_sizes: object
    group_starts: object
    rows: object
    sources: object
    padded_total: object = None

    def group(self, local_expert: int):
        s = int(self.group_starts[local_expert])
        return self.data[s:s + int(self.group_sizes[local_expert])]


@dataclass(frozen=True)
class StepStats:
    """Spans of one dispatch/combine round (moe.py:288-307); the *_vtime
    fields hold device-event microseconds relative to the step start."""

    step: int
    start_vtime: float
    dispatch_vtime: float
    combine_vtime: float

    @property
    def dispatch_us(self) -> float:
        return self.dispatch_vtime - self.start_vtime

    @property
    def combine_us(self) -> float:
        return self.combine_vtime - self.dispatch_vtime

    @property
    def total_us(self) -> float:
        return self.combine_vtime - self.start_vtime


# ------------------------------------------------------------- rank object


class _Step:
    __slots__ = ("step", "n", "host", "grouped", "keep", "ev", "sync", "fused", "out", "ld")

    def __init__(self, step: int, n: int, host: bool) -> None:
        self.step = step
        self.n = n
        self.host = host
        self.grouped: GroupedTokens | None = None
        self.keep: list = []
        self.ev: list = []
        self.sync = True
        self.fused = False
        self.out = None
        self.ld = 0


_WAIT_WHAT = (
    (_lib.EV_ROUTE_RANGE, "expert index out of range"),
    (_lib.EV_ROUTE_DUP, "a token routes to a duplicate expert"),
    (_lib.EV_CAPACITY, "a destination needs more slots than its capacity"),
    (_lib.EV_WAIT_ROUTE, "route counts"),
    (_lib.EV_WAIT_BARRIER, "dispatch barrier"),
    (_lib.EV_WAIT_PRIV, "speculative private rows"),
    (_lib.EV_WAIT_TOKEN, "token writes"),
    (_lib.EV_WAIT_COMBINE, "combine writes"),
)


class MoeRank:
    """One rank's send/receive half of the dispatch/combine protocol.

    Drive it with dispatch_send -> dispatch_recv -> combine_send ->
    combine_recv; one step may be in flight at a time (moe.py:366-373).
    """

    def __init__(self, rank: int, engine: TransferEngine, spec: RoutingSpec,
                 private: PrivateBufferConfig, node: int, *, timeout: float = 30.0) -> None:
        private.validate(spec)
        self.rank = rank
        self.engine = engine
        self.spec = spec
        self.node = node
        self.private_tokens = private.tokens
        self.device = engine.device
        self.timeout = timeout
        ce, cs = spec.comb_format
        sh = _lib.Shape(ranks=spec.ranks, experts=spec.experts, max_tokens=spec.max_tokens,
                        topk=spec.topk, hidden=spec.hidden, elem_size=spec.elem_size,
                        scales=spec.scales, comb_elem_size=ce, comb_scales=cs, me=rank,
                        device=self.device, priv_tokens=private.tokens)
        _lib.call("txb_moe_plan", C.byref(sh))
        self._shape = sh
        self._shape_p = C.byref(sh)
        self.region: Region = engine.alloc_region(int(sh.region_bytes))
        dev = torch.device("cuda", self.device)
        T, R, L = spec.max_tokens, spec.topk, spec.local_experts
        G = int(sh.grouped_rows)
        self._pos = torch.empty(max(1, T * R), dtype=torch.int64, device=dev)
        self._rank_scratch = torch.empty(max(1, T * R), dtype=torch.int32, device=dev)
        self._rows = torch.empty(G, dtype=torch.int64, device=dev)
        self._sources = torch.empty(G, dtype=torch.int64, device=dev)
        self._ret = torch.empty(G, dtype=torch.int32, device=dev)
        self._gidx = torch.empty(max(1, T * R), dtype=torch.int32, device=dev)
        # receive rows that may hold data (the region starts zeroed)
        self._dirty = torch.zeros(G, dtype=torch.uint8, device=dev)
        self._cta_hist = torch.zeros(_lib.TXB_MAX_CTAS * spec.experts, dtype=torch.int32, device=dev)
        self._cta_bad = torch.zeros(_lib.TXB_MAX_CTAS, dtype=torch.int32, device=dev)
        self._send_list = torch.zeros(G, dtype=torch.int32, device=dev)
        self._info = torch.zeros(2 * L + 3, dtype=torch.int64, device=dev)
        self._routes_in = torch.zeros((max(1, T), R), dtype=torch.int64, device=dev)
        self._info_host = torch.zeros(2 * L + 3, dtype=torch.int64).pin_memory()
        self._grouped = self.region.tensor(int(sh.off_grouped), (G, int(sh.payload_bytes)), torch.uint8)
        self._route_views = [self.region.tensor(int(sh.off_route) + k * spec.ranks * spec.experts * 8,
                                                (spec.ranks, spec.experts), torch.int64) for k in (0, 1)]
        self._peer_regions: list[Region] = []
        self._peer_ptrs: list[int] = []
        self._peer_table: torch.Tensor | None = None
        self._peer_table_p = C.c_void_p(0)
        self.host_gated = False
        self.fused = True           # fused kernels when one GPU per rank
        self._bufs = _lib.Bufs()
        self._bufs_p = C.byref(self._bufs)
        self._lock = threading.Lock()
        self._cur: _Step | None = None
        self._error: str | None = None
        self._step_no = 0
        self._slot = 0
        self.step_stats: list[StepStats] = []
        self.record_stats = True
        self._last_counts: np.ndarray | None = None
        self._closed = False

    # -------------------------------------------------------------- wiring

    def _set_peers(self, ptrs: Sequence[int], gated: bool, single_device: bool = False) -> None:
        self._peer_ptrs = [int(p) for p in ptrs]
        self._peer_table = torch.tensor(self._peer_ptrs, dtype=torch.int64,
                                        device=torch.device("cuda", self.device))
        self._peer_table_p = C.c_void_p(self._peer_table.data_ptr())
        self.host_gated = gated
        self._shape.single_device = 1 if single_device else 0
        b = self._bufs
        b.region = self.region.ptr
        b.peers = self._peer_table.data_ptr()
        b.rank_scratch = self._rank_scratch.data_ptr()
        b.pos = self._pos.data_ptr()
        b.gidx = self._gidx.data_ptr()
        b.rows = self._rows.data_ptr()
        b.sources = self._sources.data_ptr()
        b.ret_slot = self._ret.data_ptr()
        b.info = self._info.data_ptr()
        b.dirty = self._dirty.data_ptr()
        b.cta_hist = self._cta_hist.data_ptr()
        b.cta_bad = self._cta_bad.data_ptr()
        b.send_list = self._send_list.data_ptr()

    def _connect(self, mesh: Sequence["MoeRank"]) -> None:
        """In-process wiring: peers are addressed directly (peer access)."""
        devs = [m.device for m in mesh]
        gated = len(set(devs)) < len(devs)
        self._set_peers([m.region.ptr for m in sorted(mesh, key=lambda m: m.rank)], gated,
                        single_device=len(set(devs)) == 1)

    @property
    def peer_ptrs(self) -> list[int]:
        return list(self._peer_ptrs)

    # ------------------------------------------------------------ helpers

    def _sid(self) -> C.c_void_p:
        return C.c_void_p(_stream(self.device).cuda_stream)

    def _tmo(self, timeout: float | None) -> int:
        t = self.timeout if timeout is None else timeout
        return int(max(0.0, t) * 1e9) if t is not None else (1 << 62)

    def _raise_if_failed(self) -> None:
        if self._error is not None:
            raise ProtocolError(self._error)

    def _fail(self, msg: str) -> ProtocolError:
        if self._error is None:
            self._error = msg
        return ProtocolError(msg)

    def status(self) -> tuple[int, dict]:
        """(error word, counters) read from the device (synchronous); layout
        as documented at txb_moe_status in include/txb200.h."""
        N = self.spec.ranks
        cnt = (C.c_uint64 * (10 + 9 * N))()
        err = C.c_uint32(0)
        _lib.call("txb_moe_status", self._shape_p, C.c_void_p(self.region.ptr), C.byref(err),
                  cnt, len(cnt))
        v = list(cnt)
        out = {"step": v[0], "tok_ctr": v[1], "tok_target": v[2], "comb_ctr": v[3],
               "comb_target": v[4], "priv_ctr": v[5:7], "priv_target": v[7:9], "priv_step": v[9],
               "route_tag": [v[10:10 + N], v[10 + N:10 + 2 * N]]}
        k = 10 + 2 * N
        for name in ("done", "tok_src", "tok_src_target", "comb_src", "comb_src_target",
                     "priv_src", "priv_src_target"):
            out[name] = v[k:k + N]
            k += N
        return int(err.value), out

    # signal lanes in the order a step passes them; a timeout reports the
    # lanes up to the one it waited on (later lanes are not due yet)
    _LANES = {"route counts": 1, "dispatch barrier": 1, "speculative private rows": 3,
              "token writes": 3, "combine writes": 4}

    def _diagnose(self, step: int, c: dict, what: str = "combine writes") -> dict:
        """Which source ranks have not delivered, per signal lane
        (moe.py:874-899): route rows and the buffer-reuse barrier from the
        step tags, token / private / combine rows from the per-source
        counters against the per-source expectations the kernels booked."""
        upto = self._LANES.get(what, 4)
        slot = step & 1
        diag: dict = {}
        miss = [q for q, v in enumerate(c["route_tag"][slot]) if v < step]
        if miss:
            diag["route"] = miss
        miss = [q for q, v in enumerate(c["done"]) if v < step - 1]
        if miss:
            diag["barrier"] = miss
        for lane, got, want, lv in (("token", "tok_src", "tok_src_target", 3),
                                    ("private", "priv_src", "priv_src_target", 3),
                                    ("combine", "comb_src", "comb_src_target", 4)):
            if lv > upto:
                continue
            miss = [q for q, (g, w) in enumerate(zip(c[got], c[want])) if g < w]
            if miss:
                diag[lane] = miss
        return diag

    def _check_err(self, err: int, step: int) -> None:
        if not err:
            return
        _, c = self.status()
        for bit, what in _WAIT_WHAT:
            if err & bit:
                if bit in (_lib.EV_ROUTE_RANGE, _lib.EV_ROUTE_DUP, _lib.EV_CAPACITY):
                    raise self._fail(f"rank {self.rank} step {step - 1}: {what}")
                raise self._fail(f"rank {self.rank} step {step - 1} timed out waiting for {what}; "
                                 f"missing: {self._diagnose(step, c, what)}")
        raise self._fail(f"rank {self.rank}: device error word {err:#x}")

    def _gate(self, cond, step: int, what: str, timeout: float | None) -> None:
        """Host-gated mode (several ranks on one device): launch a waiting
        kernel only once its condition already holds on the device, so no
        kernel ever spins on a rank queued behind it on the same GPU."""
        torch.cuda.current_stream(self.device).synchronize()
        t = self.timeout if timeout is None else timeout
        deadline = None if t is None else time.monotonic() + t
        sleep = 2e-5
        while True:
            err, c = self.status()
            if err:
                self._check_err(err, step)
            if cond(c):
                return
            if deadline is not None and time.monotonic() > deadline:
                raise self._fail(f"rank {self.rank} step {step - 1} timed out waiting for {what}; "
                                 f"missing: {self._diagnose(step, c, what)}")
            time.sleep(sleep)
            sleep = min(sleep * 2, 1e-3)

    def _event(self, st: _Step) -> None:
        if self.record_stats and st.sync:
            e = torch.cuda.Event(enable_timing=True)
            e.record(_stream(self.device))
            st.ev.append(e)

    # ------------------------------------------------------------ dispatch

    def dispatch_send(self, payload, routes, *, sync: bool = True, _between=None) -> None:
        """Count, exchange route rows and store every token copy at its final
        grouped row on the owning rank (moe.py:470-497, 538-643)."""
        spec = self.spec
        dev = torch.device("cuda", self.device)
        host = not isinstance(routes, torch.Tensor) or not isinstance(payload, torch.Tensor)
        if _pinned(routes) and routes.dtype == torch.int64:
            # page-locked host routes: one async copy into a resident device
            # buffer; range / duplicate checks run on the device
            if routes.ndim != 2 or routes.shape[1] != spec.topk:
                raise ProtocolError(f"route array shape {tuple(routes.shape)} is not (tokens, {spec.topk})")
            if routes.shape[0] > spec.max_tokens:
                raise ProtocolError(f"{routes.shape[0]} tokens exceed the {spec.max_tokens}-token limit")
            r_dev = self._routes_in[:routes.shape[0]]
            r_dev.copy_(routes, non_blocking=True)
        elif isinstance(routes, torch.Tensor) and routes.is_cuda:
            if routes.ndim != 2 or routes.shape[1] != spec.topk:
                raise ProtocolError(f"route array shape {tuple(routes.shape)} is not (tokens, {spec.topk})")
            if routes.shape[0] > spec.max_tokens:
                raise ProtocolError(f"{routes.shape[0]} tokens exceed the {spec.max_tokens}-token limit")
            r_dev = routes.long().contiguous()   # int64, like railtx
        else:
            r = _check_routes(spec, routes.cpu().numpy() if isinstance(routes, torch.Tensor) else routes)
            r_dev = torch.from_numpy(np.ascontiguousarray(r)).to(dev)
        n = int(r_dev.shape[0])
        p_ptr = None
        if isinstance(payload, torch.Tensor) and (payload.is_cuda or _pinned(payload)):
            # device tensors, or page-locked host tensors the dispatch kernel
            # reads in place over PCIe (no separate host-to-device copy)
            p = payload if not payload.is_cuda else payload.contiguous()
            if not p.is_cuda:
                p_ptr = _mapped(p)
            if p.dtype == torch.uint8:
                if tuple(p.shape) != (n, spec.payload_bytes):
                    raise ProtocolError(f"payload shape {tuple(p.shape)} is not ({n}, {spec.payload_bytes})")
                kind = _lib.SRC_ROWS
            elif p.dtype in (torch.float32, torch.bfloat16):
                if tuple(p.shape) != (n, spec.hidden):
                    raise ProtocolError(f"value shape {tuple(p.shape)} is not ({n}, {spec.hidden})")
                kind = _lib.SRC_F32 if p.dtype == torch.float32 else _lib.SRC_BF16
            else:
                raise ProtocolError(f"unsupported payload dtype {p.dtype}")
        else:
            pa = np.ascontiguousarray(payload.cpu().numpy() if isinstance(payload, torch.Tensor)
                                      else payload, dtype=np.uint8)
            if pa.ndim != 2 or pa.shape != (n, spec.payload_bytes):
                raise ProtocolError(f"payload shape {pa.shape} is not ({n}, {spec.payload_bytes})")
            p = torch.from_numpy(pa).to(dev)
            kind = _lib.SRC_ROWS
        with self._lock:
            self._raise_if_failed()
            if self._cur is not None:
                raise ProtocolError("previous step still in flight")
            self._step_no += 1
            st = _Step(self._step_no, n, host)
            st.sync = sync or host
            self._cur = st
        st.keep = [r_dev, p]
        self._event(st)
        self._trace_dispatch(st)
        sid = self._sid()
        st.fused = self.fused and not self.host_gated and _between is None
        if st.fused:
            # route + dispatch + receive metadata in one cooperative kernel
            _lib.call("txb_moe_dispatch_fused", self._shape_p, self._bufs_p, p_ptr or _sp(p), kind, n,
                      _sp(r_dev), self._tmo(None), sid)
            return
        _lib.call("txb_moe_route", self._shape_p, self._bufs_p, _sp(r_dev), n, sid)
        if _between is not None:      # bench hook: split route / dispatch launches
            _between()
        if self.host_gated:
            step = st.step
            self._gate(lambda c: all(v >= step for v in c["route_tag"][step & 1])
                       and all(v >= step - 1 for v in c["done"]), step, "route counts", None)
        _lib.call("txb_moe_dispatch", self._shape_p, self._bufs_p, p_ptr or _sp(p), kind, n, _sp(r_dev),
                  self._tmo(None), 0, sid)
        if self.host_gated:
            torch.cuda.current_stream(self.device).synchronize()

    def dispatch_recv(self, timeout: float | None = 30.0, *, sync: bool | None = None) -> GroupedTokens:
        """Wait for every expected row, return the grouped tokens
        (moe.py:665-735).  sync=False skips the host round trip: outputs are
        max-shape device views with device-side sizes (graph-capturable)."""
        st = self._cur
        if st is None:
            raise ProtocolError("no step in flight")
        self._raise_if_failed()
        sync = st.sync if sync is None else (sync or st.host)
        if not st.fused:
            if self.host_gated:
                par = st.step & 1
                self._gate(lambda c: c["tok_ctr"] >= c["tok_target"]
                           and c["priv_ctr"][par] >= c["priv_target"][par] + c["priv_step"],
                           st.step, "token writes", timeout)
            _lib.call("txb_moe_dispatch_recv", self._shape_p, self._bufs_p, self._tmo(timeout), self._sid())
        L = self.spec.local_experts
        if not sync:
            st.grouped = GroupedTokens(self._grouped, self._info[:L], self._info[L:2 * L],
                                       self._rows, self._sources, self._info[2 * L])
            return st.grouped
        self._event(st)
        self._info_host.copy_(self._info, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        info = self._info_host.numpy().copy()
        err = int(info[2 * L + 2])
        if not err:
            # the decode kernels latch per-CTA route checks into the rank's
            # error word, possibly after CTA 0 copied it into info
            err, _ = self.status()
        if err:
            self._check_err(err, st.step)
        total = int(info[2 * L])
        sizes = torch.from_numpy(info[:L].copy())
        starts = torch.from_numpy(info[L:2 * L].copy())
        data = self._grouped[:total]
        rows = self._rows[:total]
        srcs = self._sources[:total]
        if self.engine.trace.enabled:
            self.engine.trace.record("moe_dispatch_done", step=st.step, tokens=int(sizes.sum()),
                                     used=int(info[2 * L + 1]), capacity=self.spec.capacity)
        if st.host:
            g = GroupedTokens(data.cpu().numpy(), sizes.numpy(), starts.numpy(),
                              rows.cpu().numpy(), srcs.cpu().numpy())
        else:
            g = GroupedTokens(data, sizes, starts, rows, srcs)
        st.grouped = g
        return g

    # ------------------------------------------------------------- tracing

    def _trace_dispatch(self, st: "_Step") -> None:
        """Host view of the step's fabric writes (docs/trace.md, moe.*):
        per peer one route-row write and one token write; the kernel does
        both with device stores, so these are logical posts."""
        eng = self.engine
        if not eng.trace.enabled:
            return
        eng.trace.record("moe_host_signal", step=st.step, tokens=st.n)
        E = self.spec.experts
        for q in range(self.spec.ranks):
            if q != self.rank:
                eng.post_op("moe.route", f"r{q}", 8 * E)
                eng.post_op("moe.tok.main", f"r{q}", 0)

    def _trace_combine(self, st: "_Step") -> None:
        eng = self.engine
        if not eng.trace.enabled:
            return
        for q in range(self.spec.ranks):
            if q != self.rank:
                eng.post_op("moe.comb", f"r{q}", 0)
                eng.post_op("moe.dbar", f"r{q}", 0)

    @property
    def last_layout(self) -> DispatchLayout | None:
        """Layout of the most recent step, from the device route matrix."""
        if self._step_no == 0:
            return None
        m = self._route_views[self._step_no & 1].cpu().numpy() & 0xFFFFFFFF
        return compute_layout(self.spec, m)

    # ------------------------------------------------------------- combine

    def combine_send(self, outputs) -> None:
        """Return expert outputs to their source ranks (moe.py:739-796).

        Host mode (numpy) snapshots `outputs` here, as the reference does.
        Device mode is stream-ordered instead: on the fused path the combine
        kernel, launched by combine_recv, reads the CUDA tensor `outputs` when
        it runs -- a caller that rewrites the tensor in between must order
        that write after combine_recv."""
        st = self._cur
        self._raise_if_failed()
        if st is None or st.grouped is None:
            raise ProtocolError("combine before dispatch completed")
        spec = self.spec
        Pc = spec.comb_payload_bytes
        ce, cs = spec.comb_format
        dev = torch.device("cuda", self.device)
        g = st.grouped
        if isinstance(outputs, torch.Tensor) and outputs.is_cuda:
            out = outputs
        else:
            oa = np.ascontiguousarray(outputs.cpu().numpy() if isinstance(outputs, torch.Tensor)
                                      else outputs, dtype=np.uint8)
            want = (g.data.shape[0], Pc)
            if oa.shape != want:
                raise ProtocolError(f"output shape {oa.shape} != {want}")
            out = torch.from_numpy(oa).to(dev)
        if out.dtype == torch.uint8:
            width = Pc
        elif (out.dtype == torch.bfloat16 and ce == 2) or (out.dtype == torch.float32 and ce == 4):
            if cs:
                raise ProtocolError("typed combine outputs need comb_scales == 0")
            width = spec.hidden
        else:
            raise ProtocolError(f"output dtype {out.dtype} does not match combine element size {ce}")
        rows_needed = g.data.shape[0]
        if out.ndim != 2 or out.shape[1] != width or (out.numel() and out.stride(1) != 1):
            raise ProtocolError(f"output shape {tuple(out.shape)} != ({rows_needed}, {width})")
        if g.padded_total is None and out.shape[0] != rows_needed:
            raise ProtocolError(f"output shape {tuple(out.shape)} != ({rows_needed}, {width})")
        if out.shape[0] < rows_needed and g.padded_total is not None:
            raise ProtocolError(f"output rows {out.shape[0]} below the receive capacity {rows_needed}")
        ld = (out.stride(0) if out.numel() else width) * out.element_size()
        g0 = self.region.ptr + int(self._shape.off_grouped)
        g1 = g0 + int(self._shape.grouped_rows) * int(self._shape.payload_bytes)
        if out.numel() and g0 <= out.data_ptr() < g1:
            # outputs written in place into the receive region: any row may now
            # hold data, so the next step re-zeroes every padding row
            self._dirty.fill_(1)
        st.keep.append(out)
        st.out, st.ld = out, ld
        self.engine.trace.record("moe_combine_store", step=st.step)
        if st.fused:
            return                    # sent by the fused combine kernel in combine_recv
        _lib.call("txb_moe_combine_send", self._shape_p, self._bufs_p, _sp(out), ld, 0, self._sid())
        if self.host_gated:
            torch.cuda.current_stream(self.device).synchronize()

    def combine_recv(self, weights, timeout: float | None = 30.0, *,
                     out_dtype: torch.dtype = torch.float32, sync: bool | None = None,
                     out: torch.Tensor | None = None):
        """Weighted fp32 sum of the returned expert outputs per token
        (moe.py:802-833); out_dtype bf16 rounds RNE at the end.

        `weights` and `out` may be page-locked host tensors: the combine
        kernel then reads the weights and writes the result rows in place
        over PCIe.  `out` (device or pinned host, (n, hidden), out_dtype,
        contiguous) is returned when given."""
        st = self._cur
        if st is None or st.grouped is None:
            raise ProtocolError("combine before dispatch completed")
        self._raise_if_failed()
        spec = self.spec
        dev = torch.device("cuda", self.device)
        w_ptr = None
        if _pinned(weights) and weights.dtype == torch.float32:
            w = weights
            wshape = tuple(w.shape)
            w_ptr = _mapped(w)
        elif isinstance(weights, torch.Tensor) and weights.is_cuda:
            w = weights
            if w.dtype != torch.float32:
                w = w.float()
            w = w.contiguous()
            wshape = tuple(w.shape)
        else:
            wa = np.ascontiguousarray(weights.cpu().numpy() if isinstance(weights, torch.Tensor)
                                      else weights, dtype=np.float32)
            wshape = wa.shape
            w = torch.from_numpy(wa).to(dev)
        if wshape != (st.n, spec.topk):
            raise ProtocolError(f"weight shape {wshape} is not ({st.n}, {spec.topk})")
        if out_dtype not in (torch.float32, torch.bfloat16):
            raise ProtocolError(f"out_dtype {out_dtype} not in (float32, bfloat16)")
        o_ptr = None
        if out is None:
            out = torch.empty((st.n, spec.hidden), dtype=out_dtype, device=dev)
        else:
            if tuple(out.shape) != (st.n, spec.hidden) or out.dtype != out_dtype or not out.is_contiguous():
                raise ProtocolError(f"out must be a contiguous ({st.n}, {spec.hidden}) {out_dtype} tensor")
            if out.is_cuda:
                if out.device.index != self.device:
                    raise ProtocolError(f"out on {out.device}, rank runs on cuda:{self.device}")
            elif _pinned(out):
                o_ptr = _mapped(out)
            else:
                raise ProtocolError("out must be a CUDA tensor or a page-locked host tensor")
        sync = st.sync if sync is None else (sync or st.host)
        if st.out is None:
            raise ProtocolError("combine_recv before combine_send")
        bf = 1 if out_dtype == torch.bfloat16 else 0
        if st.fused:
            _lib.call("txb_moe_combine_fused", self._shape_p, self._bufs_p, _sp(st.out), st.ld, w_ptr or _sp(w),
                      st.n, o_ptr or _sp(out), bf, self._tmo(timeout), self._sid())
        else:
            if self.host_gated:
                self._gate(lambda c: c["comb_ctr"] >= c["comb_target"], st.step, "combine writes", timeout)
            _lib.call("txb_moe_combine_recv", self._shape_p, self._bufs_p, _sp(st.out), st.ld, w_ptr or _sp(w),
                      st.n, o_ptr or _sp(out), bf, self._tmo(timeout), self._sid())
        st.keep.append(w)
        self._trace_combine(st)
        if sync:
            self._event(st)
            torch.cuda.current_stream(self.device).synchronize()
            err, _ = self.status()
            if err:
                self._check_err(err, st.step)
            self.engine.trace.record("moe_combine_done", step=st.step, tokens=st.n)
            if len(st.ev) == 3:
                t1 = st.ev[0].elapsed_time(st.ev[1]) * 1e3
                t2 = st.ev[0].elapsed_time(st.ev[2]) * 1e3
                self.step_stats.append(StepStats(st.step - 1, 0.0, t1, t2))
        with self._lock:
            self._cur = None
        if st.host:
            # host mode returns numpy f32 like the reference (moe.py:821-833); a
            # bf16 result is widened exactly (every bf16 value is an f32 value)
            return out.float().cpu().numpy()
        return out

    def barrier(self, timeout: float | None = None) -> None:
        """Device-side barrier across the mesh on the current stream
        (launch only; a later stream operation observes completion)."""
        if self.host_gated:
            raise ProtocolError("device barrier needs one device per rank")
        _lib.call("txb_moe_barrier", self._shape_p, self._bufs_p, self._tmo(timeout), self._sid())

    @property
    def pos(self) -> torch.Tensor:
        """Send-slot index of every (token, copy) of the current/last step
        (the reference's _Step.pos, moe.py:510-520)."""
        n = self._cur.n if self._cur is not None else 0
        return self._pos[:n * self.spec.topk].view(n, self.spec.topk)

    # ---------------------------------------------------------------- close

    def close(self) -> None:
        if self._closed:
            return
        self._closed = True
        torch.cuda.synchronize(self.device)
        for r in self._peer_regions:
            r.close()
        self._peer_regions.clear()
        try:
            self.engine.free_region(self.region)
        except Exception:
            pass


def build_mesh(engines: Sequence[TransferEngine], spec: RoutingSpec, *,
               private: PrivateBufferConfig | None = None,
               ranks_per_node: int = 1, timeout: float = 30.0) -> list[MoeRank]:
    """Wire one MoeRank per engine in this process (moe.py:925-939).

    `ranks_per_node` is accepted for API compatibility; every rank on one
    NVSwitch box is reachable by peer stores, so there is a single lane.
    Ranks that share a device (single-GPU emulation of EP>1) run host-gated.
    """
    if len(engines) != spec.ranks:
        raise ProtocolError(f"{len(engines)} engines for {spec.ranks} ranks")
    if ranks_per_node < 1:
        raise ProtocolError("ranks_per_node must be positive")
    if private is None:
        private = PrivateBufferConfig(min(DEFAULT_PRIVATE, spec.max_tokens))
    enable_peer_access([e.device for e in engines])
    mesh = [MoeRank(r, engines[r], spec, private, node=r // ranks_per_node, timeout=timeout)
            for r in range(spec.ranks)]
    for rank in mesh:
        rank._connect(mesh)
    return mesh


def connect_process_group(engine: TransferEngine, spec: RoutingSpec, *,
                          private: PrivateBufferConfig | None = None, group=None,
                          ranks_per_node: int = 1, timeout: float = 30.0) -> MoeRank:
    """Multi-process wiring: one MoeRank per process (torchrun), peers'
    regions opened from CUDA IPC handles all-gathered over `group`
    (setup only; the data path never touches the process group)."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    if world != spec.ranks:
        raise ProtocolError(f"{world} processes for {spec.ranks} ranks")
    if private is None:
        private = PrivateBufferConfig(min(DEFAULT_PRIVATE, spec.max_tokens))
    me = MoeRank(rank, engine, spec, private, node=rank // max(1, ranks_per_node), timeout=timeout)
    import socket
    mine = RegionDesc(rank, socket.gethostname(), engine.device, me.region.ipc_handle(),
                      me.region.nbytes, spec_key=dataclasses.astuple(spec))
    ptrs = []
    for d in engine.fabric.exchange(mine):
        if d.rank == rank:
            ptrs.append(me.region.ptr)
            continue
        reg = Region.open_ipc(engine.device, d.handle, d.nbytes)
        me._peer_regions.append(reg)
        ptrs.append(reg.ptr)
    me._set_peers(ptrs, gated=False)
    engine.fabric.barrier()
    return me
