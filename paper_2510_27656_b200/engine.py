"""TransferEngine over NVLink peer memory (B200 stand-in for railtx.engine).

In the reference an engine owns NIC rails, a worker thread that posts work
requests, and an ImmCounterTable (engine.py:260-850).  On one NVSwitch box
every peer is a load/store away, so the B200 engine is thin: it binds a
rank to a CUDA device, owns that rank's registered regions, and knows how
to reach peer regions -- directly (same process, peer access enabled) or
through CUDA IPC handles exchanged over a torch.distributed process group
(multi-process).  Data movement and completion counting happen inside the
sm_100a kernels (device-initiated stores + release/acquire counters); there
is no host proxy and no worker thread.
"""

from __future__ import annotations

import ctypes as C
import itertools
import os
import threading
import time
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np
import torch

from . import _lib, memory
from .errors import ProtocolError, RegionError, TransferError
from .trace import TraceRecorder


@dataclass(frozen=True)
class NetAddr:
    """Engine address (wire.py:26-61): here (host id, process rank, device)."""

    host: str
    proc: int
    device: int

    @property
    def data(self) -> bytes:
        return f"{self.host}/{self.proc}/{self.device}".encode()


@dataclass(frozen=True)
class RegionDesc:
    """What a peer needs to reach one rank's symmetric region (the MrDesc
    analog, wire.py:64-87): owner rank, host, device, the 64-byte CUDA IPC
    handle, the region size and a key of the spec that laid it out."""

    rank: int
    host: str
    device: int
    handle: bytes
    nbytes: int
    spec_key: tuple = ()


def check_descs(descs: Sequence[RegionDesc], world: int) -> list[RegionDesc]:
    """Validate an all-gathered descriptor set (sorted by rank): ranks
    0..world-1 exactly once, one spec and region size for everyone, and no
    two ranks on one GPU (ranks that wait on each other must not be separate
    processes on one device)."""
    ds = sorted(descs, key=lambda d: d.rank)
    if [d.rank for d in ds] != list(range(world)):
        raise RegionError(f"region descriptors for ranks {[d.rank for d in ds]}, expected 0..{world - 1}")
    if len({d.spec_key for d in ds}) != 1:
        raise RegionError("ranks disagree on the routing spec: "
                          + "; ".join(f"rank {d.rank}: {d.spec_key}" for d in ds))
    if len({d.nbytes for d in ds}) != 1:
        raise RegionError("ranks disagree on the region size")
    seen: dict = {}
    for d in ds:
        k = (d.host, d.device)
        if k in seen:
            raise RegionError(f"ranks {seen[k]} and {d.rank} share GPU {d.device} on {d.host}: "
                              "use build_mesh in one process for several ranks per GPU")
        seen[k] = d.rank
    return ds


class NvlinkFabric:
    """The set of engines that can reach each other over NVLink.

    Single process: engines register here and address each other's regions
    directly.  Multi-process: `group` is a torch.distributed process group
    (any backend) used only at setup to all-gather IPC handles -- never on
    the data path.
    """

    def __init__(self, group=None) -> None:
        self.group = group
        self._ids = itertools.count()
        self.engines: list["TransferEngine"] = []

    @property
    def multiprocess(self) -> bool:
        return self.group is not None or (torch.distributed.is_available()
                                          and torch.distributed.is_initialized()
                                          and torch.distributed.get_world_size() > 1)

    def allocate_engine_id(self) -> int:
        return next(self._ids)

    def all_gather(self, obj):
        """Setup-time exchange (IPC handles, ranks, nodes)."""
        import torch.distributed as dist
        world = dist.get_world_size(self.group)
        out = [None] * world
        dist.all_gather_object(out, obj, group=self.group)
        return out

    def exchange(self, mine: RegionDesc) -> list[RegionDesc]:
        """All-gather every rank's region descriptor and validate the set."""
        import torch.distributed as dist
        return check_descs(self.all_gather(mine), dist.get_world_size(self.group))

    def barrier(self) -> None:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.barrier(group=self.group)


# ------------------------------------------------------------- wire types


@dataclass(frozen=True)
class MrHandle:
    """Local handle of a registered region (wire.py:90-97)."""

    region_id: int
    base: int          # device address
    length: int
    device: int


@dataclass(frozen=True)
class MrDesc:
    """What a peer needs to write into a region and count receipts
    (wire.py:64-87): the owner engine, the region's device address and
    length, and the owner's ImmCounter table.  `ipc`/`imm_ipc` carry CUDA
    IPC handles for peers in other processes (regions allocated by the
    engine); in-process peers use the addresses directly."""

    owner: str
    device: int
    base: int
    length: int
    imm_base: int
    pid: int
    ipc: bytes | None = None
    ipc_offset: int = 0
    imm_ipc: bytes | None = None


@dataclass(frozen=True)
class Pages:
    """Indirect page addressing: page i lives at offset + indices[i] * stride
    (wire.py:100-112)."""

    indices: tuple
    stride: int
    offset: int = 0

    def __post_init__(self) -> None:
        object.__setattr__(self, "indices", tuple(int(i) for i in self.indices))

    def page_offset(self, i: int) -> int:
        return self.offset + self.indices[i] * self.stride


@dataclass(frozen=True)
class ScatterDst:
    """One peer's slice in a scatter: src offset -> (desc, offset), `length`
    bytes (wire.py:115-122)."""

    length: int
    src: int
    desc: MrDesc
    offset: int


class CompletionFlag:
    """Completion of one submitted operation (engine.py:48-77): a CUDA event
    recorded after the operation's kernel on the engine's stream."""

    def __init__(self, event=None, ok: bool = True, error: str | None = None) -> None:
        self._ev = event
        self.ok = ok
        self.error = error
        self.vtime = 0.0

    def done(self) -> bool:
        return self._ev is None or self._ev.query()

    def wait(self, timeout: float | None = None) -> bool:
        if self._ev is None:
            return True
        if timeout is None:
            self._ev.synchronize()
            return True
        deadline = time.monotonic() + timeout
        while not self._ev.query():
            if time.monotonic() > deadline:
                return False
            time.sleep(2e-5)
        return True

    def result(self, timeout: float | None = None) -> float:
        if not self.wait(timeout):
            raise TransferError("timed out waiting for completion")
        if not self.ok:
            raise TransferError(self.error or "operation failed")
        return self.vtime


class ImmFlag:
    """Fires when an armed immediate count is reached (engine.py:80-103).

    Receipts are counted on the device (one u64 counter per imm value, in
    the engine's full-u32 ImmCounter table); the flag holds the threshold
    `consumed + count` fixed when it was armed.  A flag armed with a
    callback is watched by the engine's callback thread, which runs the
    callback when the count is reached (engine.py:527-543); a flag that
    fires in a caller's wait()/done() also hands its callback to that
    thread.  `wait_device(stream)` makes GPU work queued behind it wait on
    the device instead of the host."""

    def __init__(self, engine: "TransferEngine", imm: int, threshold: int,
                 cb: Callable | None = None) -> None:
        self.engine = engine
        self.imm = imm
        self.threshold = threshold
        self.cb = cb
        self.vtime = 0.0
        self._fired = False

    def _check(self, total: int | None = None) -> bool:
        if self._fired:
            return True
        if total is None:
            total = self.engine.imm_received_total(self.imm)
        if total >= self.threshold:
            with self.engine._lock:
                if self._fired:
                    return True
                self._fired = True
            self.engine._disarm(self.imm, self)
            self.engine.trace.record("imm_fire", imm=self.imm)
            if self.cb is not None:
                self.engine._callbacks().post(lambda: self.cb(self))
        return self._fired

    def done(self) -> bool:
        return self._check()

    def wait(self, timeout: float | None = None) -> bool:
        # back-to-back checks for the first 2 ms (each one is a device read,
        # ~10 us, so this is not a hot spin), then a backoff to 1 ms: a
        # doubling sleep from the start put the detection of a ~80 us write
        # at ~150 us (tools/bench_weights.py publish_us)
        t0 = time.monotonic()
        deadline = None if timeout is None else t0 + timeout
        sleep = 2e-5
        while not self._check():
            now = time.monotonic()
            if deadline is not None and now > deadline:
                return False
            if now - t0 > 2e-3:
                time.sleep(sleep)
                sleep = min(2 * sleep, 1e-3)
        return True

    def result(self, timeout: float | None = None) -> float:
        if not self.wait(timeout):
            raise TransferError(f"timed out waiting for imm {self.imm}")
        return self.vtime

    def wait_device(self, stream=None, timeout: float = 30.0) -> None:
        st = stream or torch.cuda.current_stream(self.engine.device)
        _lib.call("txb_imm_wait", C.c_void_p(self.engine._imm_slot_ptr(self.imm)), self.threshold,
                  int(timeout * 1e9), C.c_void_p(self.engine._err.data_ptr()), C.c_void_p(st.cuda_stream))


class Watcher:
    """Shared word the application side bumps to trigger engine callbacks
    (engine.py:106-121).  The word lives in page-locked host memory mapped
    into the GPU: `store(v)` from the host, or a device store through
    `device_ptr` from any kernel or stream (txb_stream_write_value64), and
    the engine's callback thread calls cb(old, new) with a strictly
    increasing subsequence of the values, ending at the latest one."""

    __slots__ = ("_word", "device_ptr", "last_seen", "cb")

    def __init__(self, cb: Callable[[int, int], None], initial: int = 0) -> None:
        self._word = torch.full((1,), int(initial), dtype=torch.int64).pin_memory()
        out = C.c_void_p()
        _lib.call("txb_host_device_ptr", C.c_void_p(self._word.data_ptr()), C.byref(out))
        self.device_ptr = int(out.value)
        self.last_seen = int(initial)
        self.cb = cb

    @property
    def value(self) -> int:
        return int(self._word[0])

    def store(self, v: int) -> None:
        self._word[0] = int(v)


class _CallbackThread:
    """The engine's callback thread (the reference runs callbacks, watcher
    polling and completion delivery off its worker, engine.py:642-813):
    watches armed ImmFlags that carry a callback, pending on_done
    completions and watchers, and runs every callback in order.  Callbacks
    must not block."""

    def __init__(self, engine: "TransferEngine") -> None:
        self.engine = engine
        self._cv = threading.Condition()
        self._flags: list[ImmFlag] = []
        self._done: list[tuple[CompletionFlag, Callable]] = []
        self._watchers: list[Watcher] = []
        self._queue: list[Callable[[], None]] = []
        self._stop = False
        self.errors: list[BaseException] = []
        self._th = threading.Thread(target=self._run, name=f"{engine.name}-callbacks", daemon=True)
        self._th.start()

    def post(self, fn: Callable[[], None]) -> None:
        with self._cv:
            self._queue.append(fn)
            self._cv.notify()

    def watch_flag(self, flag: ImmFlag) -> None:
        with self._cv:
            self._flags.append(flag)
            self._cv.notify()

    def watch_done(self, flag: CompletionFlag, cb: Callable) -> None:
        with self._cv:
            self._done.append((flag, cb))
            self._cv.notify()

    def add_watcher(self, w: Watcher) -> None:
        with self._cv:
            self._watchers.append(w)
            self._cv.notify()

    def remove_watcher(self, w: Watcher) -> None:
        with self._cv:
            if w in self._watchers:
                self._watchers.remove(w)

    def close(self) -> None:
        with self._cv:
            self._stop = True
            self._cv.notify()
        if threading.current_thread() is not self._th:
            self._th.join(5.0)

    def _run(self) -> None:
        sleep = 2e-5
        while True:
            with self._cv:
                if self._stop:
                    return
                if not (self._flags or self._done or self._watchers or self._queue):
                    self._cv.wait(0.05)
                    sleep = 2e-5
                    continue
                flags, done, watchers = list(self._flags), list(self._done), list(self._watchers)
            busy = False
            if flags:
                totals = self.engine.imm_received_totals([f.imm for f in flags])
                fired = [f for f, t in zip(flags, totals) if f._check(t)]
                if fired:
                    busy = True
                    with self._cv:
                        self._flags = [f for f in self._flags if f not in fired]
            for cf, cb in done:
                if cf.done():
                    busy = True
                    with self._cv:
                        self._done.remove((cf, cb))
                    self.post(lambda cf=cf, cb=cb: cb(cf))
            for w in watchers:
                v = w.value
                if v != w.last_seen:
                    busy = True
                    old, w.last_seen = w.last_seen, v
                    self.post(lambda w=w, old=old, v=v: w.cb(old, v))
            with self._cv:
                queue, self._queue = self._queue, []
            for fn in queue:
                busy = True
                try:
                    fn()
                except BaseException as exc:  # noqa: BLE001  (a callback must not kill the thread)
                    self.errors.append(exc)
            sleep = 2e-5 if busy else min(sleep * 2, 1e-3)
            time.sleep(sleep)


class DeviceClock:
    """A monotone u64 word in device memory, advanced in stream order and
    waited on in stream order (the LayerClock of kvcache.py:317-334 moved
    onto the GPU): `advance(stream)` appends a write of the next value to
    the compute stream; consumers queued on other streams -- or a running
    kernel polling the word -- see it without a host round trip."""

    def __init__(self, engine: "TransferEngine", steps: int | None = None) -> None:
        self.engine = engine
        self.steps = steps
        self._t = torch.zeros(1, dtype=torch.int64, device=torch.device("cuda", engine.device))
        self.ptr = self._t.data_ptr()
        self._value = 0

    @property
    def value(self) -> int:
        """Value as last advanced from the host (stream order may lag)."""
        return self._value

    def device_value(self) -> int:
        return int(self._t.cpu()[0])

    def advance(self, stream=None, by: int = 1) -> int:
        if self.steps is not None and self._value + by > self.steps:
            raise ProtocolError(f"layer clock past its final value {self.steps}")
        self._value += by
        st = stream or torch.cuda.current_stream(self.engine.device)
        _lib.call("txb_stream_write_value64", C.c_void_p(self.ptr), self._value, C.c_void_p(st.cuda_stream))
        return self._value

    def wait_device(self, value: int, stream=None, timeout: float = 30.0) -> None:
        st = stream or torch.cuda.current_stream(self.engine.device)
        _lib.call("txb_stream_wait_value64", C.c_void_p(self.ptr), int(value), int(timeout * 1e9),
                  C.c_void_p(self.engine._err.data_ptr()), C.c_void_p(st.cuda_stream))


class TransferEngine:
    """One rank's endpoint on one CUDA device.

    Mirrors the submission API of railtx.engine.TransferEngine
    (engine.py:260-850): reg_mr / dereg_mr, submit_single_write,
    submit_paged_writes, submit_scatter, submit_barrier, expect_imm_count,
    add_peer_group.  Every submission is one sm_100a kernel on the engine's
    stream that moves the bytes with device-initiated stores (TMA bulk copies
    for aligned pages) and releases one increment on the destination's
    ImmCounter slot after the payload is visible.  There are no rails, no
    worker thread and no host proxy."""

    _TICKETS = 256

    def __init__(self, fabric: NvlinkFabric | None = None, *, device: int = 0,
                 name: str | None = None, rails: int = 1, engine_id: int | None = None,
                 trace: bool = False) -> None:
        if not 1 <= rails <= 4:
            raise TransferError(f"rail count {rails} outside 1..4")
        self.fabric = fabric or NvlinkFabric()
        self.engine_id = engine_id if engine_id is not None else self.fabric.allocate_engine_id()
        self.name = name or f"e{self.engine_id}"
        self.device = int(device)
        self.fabric.engines.append(self)
        self._regions: dict[int, memory.Region] = {}
        self._mrs: dict[int, tuple[MrHandle, MrDesc, object]] = {}
        self._ids = itertools.count(1)
        self._lock = threading.Lock()
        self._closed = False
        self._imm = None           # lazily: ImmCounter table region
        self._stream = None
        self._order_tl = threading.local()
        self._consumed: dict[int, int] = {}
        self._armed: dict[int, ImmFlag] = {}
        self._groups: dict[int, tuple] = {}
        self._opened: dict[tuple, memory.Region] = {}
        # 16-byte vector copies by default: at layer-step sizes they beat the
        # TMA bulk-copy pipeline (profiles/r02/kv); TMA stays selectable
        self.use_tma = False
        self._slots: dict[tuple[int, int], int] = {}
        self._cbt: _CallbackThread | None = None
        self._own_streams: list[int] = []
        self.timing: list | None = None
        self.trace = TraceRecorder(self.name, enabled=trace)
        self._op_ids = itertools.count(1)
        # every library kernel loaded now, not at its first launch (txb_preload)
        if torch.cuda.is_available():
            _lib.call("txb_preload", self.device)

    def main_address(self) -> NetAddr:
        import socket
        proc = 0
        if torch.distributed.is_available() and torch.distributed.is_initialized():
            proc = torch.distributed.get_rank()
        return NetAddr(socket.gethostname(), proc, self.device)

    # ------------------------------------------------------------- regions

    def alloc_region(self, nbytes: int) -> memory.Region:
        if self._closed:
            raise RegionError("engine closed")
        r = memory.Region.alloc(self.device, nbytes)
        self._regions[r.ptr] = r
        return r

    def free_region(self, region: memory.Region) -> None:
        if self._regions.pop(region.ptr, None) is None:
            raise RegionError("region not registered with this engine")
        region.close()

    def _callbacks(self) -> _CallbackThread:
        with self._lock:
            if self._cbt is None:
                self._cbt = _CallbackThread(self)
            return self._cbt

    def _ensure_imm(self) -> None:
        if self._imm is None:
            # full-u32 ImmCounter table: keys[SLOTS] then counts[SLOTS]
            self._imm = self.alloc_region(2 * _lib.TXB_IMM_SLOTS * 8 + 4096)
            dev = torch.device("cuda", self.device)
            self._tickets = torch.zeros(self._TICKETS, dtype=torch.int32, device=dev)
            self._ticket_i = 0
            self._err = torch.zeros(1, dtype=torch.int32, device=dev)
            # dedicated streams (torch's pooled streams can alias a caller's)
            self._stream = self._own_stream()
            self._read_stream = self._own_stream()    # counter snapshots

    def _own_stream(self):
        out = C.c_void_p()
        _lib.call("txb_stream_create", self.device, C.byref(out))
        self._own_streams.append(int(out.value))
        return torch.cuda.ExternalStream(int(out.value), device=torch.device("cuda", self.device))

    @property
    def stream(self):
        self._ensure_imm()
        return self._stream

    def alloc_buffer(self, nbytes: int) -> torch.Tensor:
        """A uint8 device buffer whose region can be exported to peers in
        other processes (CUDA IPC); register it with reg_mr."""
        r = self.alloc_region(nbytes)
        t = r.tensor(0, (nbytes,), torch.uint8)
        t._txb_region = r  # keep the region reachable from the tensor
        return t

    def reg_mr(self, buf, device: int | None = None) -> tuple[MrHandle, MrDesc]:
        """Register a writable contiguous CUDA tensor (engine.py:314-341)."""
        self._ensure_imm()
        if device is not None and device != self.device:
            raise RegionError(f"unknown device {device}")
        if not isinstance(buf, torch.Tensor) or not buf.is_cuda:
            raise RegionError("region must be a CUDA tensor on the engine's device")
        if buf.device.index != self.device:
            raise RegionError(f"region lives on cuda:{buf.device.index}, engine on cuda:{self.device}")
        if not buf.is_contiguous():
            raise RegionError("region must be contiguous")
        base, length = buf.data_ptr(), buf.numel() * buf.element_size()
        with self._lock:
            if any(h.base == base for h, _, _ in self._mrs.values()):
                raise RegionError("buffer already registered")
            rid = next(self._ids)
        ipc, ipc_off = None, 0
        reg = getattr(buf, "_txb_region", None)
        if reg is not None:
            ipc, ipc_off = reg.ipc_handle(), base - reg.ptr
        h = MrHandle(rid, base, length, self.device)
        d = MrDesc(self.name, self.device, base, length, self._imm.ptr, os.getpid(), ipc, ipc_off,
                   self._imm.ipc_handle())
        with self._lock:
            self._mrs[rid] = (h, d, buf)
        self.trace.record("reg_mr", region=rid, nbytes=length)
        return h, d

    def dereg_mr(self, handle: MrHandle) -> None:
        with self._lock:
            if self._mrs.pop(handle.region_id, None) is None:
                raise RegionError(f"region {handle.region_id} not registered")

    def desc_of(self, handle: MrHandle) -> MrDesc:
        with self._lock:
            rec = self._mrs.get(handle.region_id)
        if rec is None:
            raise RegionError(f"region {handle.region_id} not registered")
        return rec[1]

    def _get(self, handle: MrHandle) -> MrHandle:
        with self._lock:
            rec = self._mrs.get(handle.region_id)
        if rec is None:
            raise RegionError(f"region {handle.region_id} not registered")
        return rec[0]

    def _peer_base(self, desc: MrDesc) -> tuple[int, int]:
        """(region address, ImmCounter table address) of `desc` as seen from
        this process."""
        if desc.pid == os.getpid():
            return desc.base, desc.imm_base
        if desc.ipc is None or desc.imm_ipc is None:
            raise RegionError("remote region was not allocated with alloc_buffer (no IPC handle)")
        key = (desc.pid, desc.ipc, desc.imm_ipc)
        with self._lock:
            got = self._opened.get(key)
            if got is None:
                reg = memory.Region.open_ipc(self.device, desc.ipc, desc.ipc_offset + desc.length)
                imm = memory.Region.open_ipc(self.device, desc.imm_ipc, 2 * _lib.TXB_IMM_SLOTS * 8)
                got = self._opened[key] = (reg, imm)
        return got[0].ptr + desc.ipc_offset, got[1].ptr

    def _imm_slot(self, imm: int, imm_base: int | None = None) -> int:
        """Slot of `imm` in an ImmCounter table (own, or a peer's), claimed
        on first use with a system-scope CAS on the table; cached."""
        self._ensure_imm()
        base = self._imm.ptr if imm_base is None else imm_base
        key = (base, int(imm))
        slot = self._slots.get(key)
        if slot is None:
            out = C.c_int64(-1)
            _lib.call("txb_imm_slot", C.c_void_p(base), C.c_uint32(int(imm)), 1, C.byref(out))
            slot = self._slots[key] = int(out.value)
        return slot

    def _imm_slot_ptr(self, imm: int, imm_base: int | None = None) -> int:
        """Address of imm's receipt counter in a table (counts follow keys)."""
        base = self._imm.ptr if imm_base is None else imm_base
        return base + (_lib.TXB_IMM_SLOTS + self._imm_slot(imm, base)) * 8

    # --------------------------------------------------------- submissions

    def _single_device(self, desc: MrDesc) -> int:
        return 1 if desc.pid == os.getpid() and desc.device == self.device else 0

    def page_indices(self, pages: Pages) -> torch.Tensor:
        """Device copy of a page index list (reusable across submissions)."""
        t = torch.from_numpy(np.asarray(pages.indices, dtype=np.int64)).pin_memory()
        return t.to(torch.device("cuda", self.device), non_blocking=True)

    def post_op(self, label: str, dst: str, nbytes: int, imm: int | None = None, posts: int = 1) -> int:
        """Trace one submitted transfer: op_submit with its label and one
        wr_post per logical write it performs on the fabric (the events
        check_moe / check_kvcache audit, docs/trace.md)."""
        op = next(self._op_ids)
        if self.trace.enabled:
            if label:
                self.trace.label_transfer(op, label)
            self.trace.record("op_submit", transfer=op, dst=dst, nbytes=int(nbytes), imm=imm)
            for _ in range(posts):
                self.trace.record("wr_post", transfer=op, dst=dst)
        return op

    def _after_current(self) -> None:
        """Order the engine stream after the caller's current stream (where
        the payload was produced): one reused event per calling thread
        instead of wait_stream's fresh one."""
        tl = self._order_tl
        ev = getattr(tl, "ev", None)
        if ev is None:
            ev = tl.ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        self._stream.wait_event(ev)

    def _launch_pages(self, src_base: int, src_pages: Pages, desc: MrDesc, dst_pages: Pages,
                      page_len: int, npages: int, imm: int | None,
                      idx: tuple | None = None, label: str = "") -> CompletionFlag:
        self._ensure_imm()
        self.post_op(label, desc.owner, page_len * npages, imm)
        dst_base, dst_imm = self._peer_base(desc)
        j = _lib.Pages()
        j.src_base, j.src_offset, j.src_stride = src_base, src_pages.offset, src_pages.stride
        j.dst_base, j.dst_offset, j.dst_stride = dst_base, dst_pages.offset, dst_pages.stride
        keep = []
        if idx is not None:
            si, di = idx if isinstance(idx[0], torch.Tensor) else \
                (self.page_indices(src_pages), self.page_indices(dst_pages))
            keep = [si, di]
            j.src_idx, j.dst_idx = si.data_ptr(), di.data_ptr()
        j.npages, j.page_len = npages, page_len
        j.imm_ctr = self._imm_slot_ptr(imm, dst_imm) if imm is not None else None
        with self._lock:
            t = self._ticket_i
            self._ticket_i = (t + 1) % self._TICKETS
        j.ticket = self._tickets.data_ptr() + 4 * t
        aligned = all(v % 16 == 0 for v in (src_base + src_pages.offset, dst_base + dst_pages.offset,
                                            src_pages.stride, dst_pages.stride, page_len))
        j.use_tma = 1 if aligned and page_len >= 1024 and self.use_tma else 0
        j.single_device = self._single_device(desc)
        # every call below names its stream: no `with torch.cuda.stream`
        # (~10 us of host time per launch on this image)
        with torch.cuda.device(self.device):
            # the payload was produced on the caller's stream
            self._after_current()
            for k in keep:
                k.record_stream(self._stream)
            if self.timing is not None:              # bench hook: device time of the copy kernel
                with torch.cuda.stream(self._stream):
                    torch.cuda._sleep(200000)         # keep the GPU busy past the host launch
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(self._stream)
            _lib.call("txb_copy_pages", C.byref(j), 0, C.c_void_p(self._stream.cuda_stream))
            if self.timing is not None:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(self._stream)
                self.timing.append((e0, e1))
            ev = torch.cuda.Event()
            ev.record(self._stream)
        return CompletionFlag(ev)

    def _launch_jobs(self, jobs: list, label: str = "") -> CompletionFlag:
        """Several contiguous writes (src_base, src Pages, desc, dst Pages,
        page_len, npages, imm) in ONE kernel launch (txb_copy_jobs): the
        per-peer slices of a scatter, each completing on its own."""
        self._ensure_imm()
        out = []
        for k in range(0, len(jobs), _lib.TXB_MAX_JOBS):
            chunk = jobs[k:k + _lib.TXB_MAX_JOBS]
            arr = (_lib.Pages * len(chunk))()
            for j, (src_base, sp, desc, dp, page_len, npages, imm) in zip(arr, chunk):
                self.post_op(label, desc.owner, page_len * npages, imm)
                dst_base, dst_imm = self._peer_base(desc)
                j.src_base, j.src_offset, j.src_stride = src_base, sp.offset, sp.stride
                j.dst_base, j.dst_offset, j.dst_stride = dst_base, dp.offset, dp.stride
                j.npages, j.page_len = npages, page_len
                j.imm_ctr = self._imm_slot_ptr(imm, dst_imm) if imm is not None else None
                with self._lock:
                    t = self._ticket_i
                    self._ticket_i = (t + 1) % self._TICKETS
                j.ticket = self._tickets.data_ptr() + 4 * t
                aligned = all(v % 16 == 0 for v in (src_base + sp.offset, dst_base + dp.offset, page_len))
                j.use_tma = 1 if aligned and page_len >= 1024 and self.use_tma else 0
                j.single_device = self._single_device(desc)
            with torch.cuda.device(self.device):
                self._after_current()
                _lib.call("txb_copy_jobs", arr, len(chunk), 0, C.c_void_p(self._stream.cuda_stream))
                ev = torch.cuda.Event()
                ev.record(self._stream)
            out.append(ev)
        return CompletionFlag(out[-1])

    @staticmethod
    def _check_imm(imm) -> None:
        if imm is not None and not 0 <= imm < (1 << 32):
            raise TransferError(f"imm {imm} is not a u32")

    def submit_single_write(self, length: int, src: tuple, dst: tuple, imm: int | None = None,
                            on_done: Callable | None = None, not_before: float = 0.0,
                            label: str = "") -> CompletionFlag:
        """engine.py:397-436 -- bounds, then one device copy + one receipt."""
        handle, src_off = src
        desc, dst_off = dst
        rec = self._get(handle)
        if length < 0 or src_off < 0 or dst_off < 0:
            raise TransferError("negative length or offset")
        if src_off + length > rec.length:
            raise TransferError(f"source range [{src_off},{src_off + length}) outside region of {rec.length}")
        if dst_off + length > desc.length:
            raise TransferError(f"destination range [{dst_off},{dst_off + length}) outside region of {desc.length}")
        if length == 0 and imm is None:
            raise TransferError("zero-length write requires an immediate")
        self._check_imm(imm)
        flag = self._launch_pages(rec.base, Pages((0,), 0, src_off), desc, Pages((0,), 0, dst_off),
                                  length, 1 if length else 0, imm, label=label)
        return self._done(flag, on_done)

    def submit_paged_writes(self, page_len: int, src: tuple, dst: tuple, imm: int | None = None,
                            on_done: Callable | None = None, not_before: float = 0.0,
                            label: str = "", device_indices: tuple | None = None) -> CompletionFlag:
        """engine.py:438-466 -- one kernel moves every page, one receipt.
        `device_indices` = (src, dst) int64 CUDA tensors equal to the Pages
        indices (from page_indices) skip the per-call index upload."""
        handle, src_pages = src
        desc, dst_pages = dst
        rec = self._get(handle)
        if len(src_pages.indices) != len(dst_pages.indices):
            raise TransferError(f"{len(src_pages.indices)} source pages vs "
                                f"{len(dst_pages.indices)} destination pages")
        if page_len <= 0:
            raise TransferError("page length must be positive")
        self._check_pages(src_pages, page_len, rec.length, "source")
        self._check_pages(dst_pages, page_len, desc.length, "destination")
        self._check_imm(imm)
        flag = self._launch_pages(rec.base, src_pages, desc, dst_pages, page_len,
                                  len(src_pages.indices), imm, idx=device_indices or (True,), label=label)
        return self._done(flag, on_done)

    @staticmethod
    def _check_pages(pages: Pages, page_len: int, region_len: int, side: str) -> None:
        if not pages.indices:
            return
        idx = np.asarray(pages.indices, dtype=np.int64)
        lo, hi = int(idx.min()), int(idx.max())
        if lo < 0 or hi >= (1 << 32):
            raise TransferError(f"{side} page index {lo if lo < 0 else hi} is not a u32")
        worst = pages.offset + hi * pages.stride + page_len
        if worst > region_len:
            raise TransferError(f"{side} page ends at {worst}, outside region of {region_len}")

    def add_peer_group(self, addrs: Sequence) -> int:
        if not addrs:
            raise TransferError("empty peer group")
        with self._lock:
            h = next(self._ids)
            self._groups[h] = tuple(addrs)
        return h

    def _group(self, group: int, n: int, what: str) -> tuple:
        with self._lock:
            peers = self._groups.get(group)
        if peers is None:
            raise TransferError(f"unknown peer group {group}")
        if n != len(peers):
            raise TransferError(f"{what} carries {n} entries for a group of {len(peers)}")
        return peers

    def submit_scatter(self, group: int, src: MrHandle, dsts: Sequence[ScatterDst], imm: int | None = None,
                       on_done: Callable | None = None, not_before: float = 0.0,
                       label: str = "") -> CompletionFlag:
        """engine.py:563-597 -- one slice per peer, each carrying the imm."""
        self._group(group, len(dsts), "scatter")
        rec = self._get(src)
        self._check_imm(imm)
        flag = CompletionFlag()
        for i, d in enumerate(dsts):
            if d.length < 0 or d.src < 0 or d.offset < 0:
                raise TransferError("negative length or offset in scatter entry")
            if d.src + d.length > rec.length:
                raise TransferError(f"scatter source slice {i} out of bounds")
            if d.offset + d.length > d.desc.length:
                raise TransferError(f"scatter destination slice {i} out of bounds")
        live = [d for d in dsts if d.length or imm is not None]
        if live:
            flag = self._launch_jobs([(rec.base, Pages((0,), 0, d.src), d.desc, Pages((0,), 0, d.offset),
                                       d.length, 1 if d.length else 0, imm) for d in live], label)
        return self._done(flag, on_done)

    def submit_barrier(self, group: int, imm: int, dsts: Sequence[tuple], on_done: Callable | None = None,
                       not_before: float = 0.0, label: str = "") -> CompletionFlag:
        """engine.py:599-619 -- a zero-length write with the imm per peer."""
        self._group(group, len(dsts), "barrier")
        if not 0 <= imm < (1 << 32):
            raise TransferError(f"imm {imm} is not a u32")
        self._ensure_imm()
        ptrs = []
        for desc, off in dsts:
            if not 0 <= off <= desc.length:
                raise TransferError(f"barrier offset {off} out of bounds")
            ptrs.append(self._imm_slot_ptr(imm, self._peer_base(desc)[1]))
        for desc, _ in dsts:
            self.post_op(label, desc.owner, 0, imm)
        dev = torch.device("cuda", self.device)
        tab = torch.tensor(ptrs, dtype=torch.int64).to(dev, non_blocking=True)
        sd = 1 if all(self._single_device(d) for d, _ in dsts) else 0
        with torch.cuda.device(self.device):
            self._after_current()
            tab.record_stream(self._stream)
            _lib.call("txb_imm_add", C.c_void_p(tab.data_ptr()), len(ptrs), 1, sd,
                      C.c_void_p(self._stream.cuda_stream))
            ev = torch.cuda.Event()
            ev.record(self._stream)
        return self._done(CompletionFlag(ev), on_done)

    def _done(self, flag: CompletionFlag, on_done: Callable | None) -> CompletionFlag:
        """on_done runs on the engine's callback thread once the operation
        has completed (engine.py:563-619); the submitter never blocks."""
        if on_done is not None:
            self._callbacks().watch_done(flag, on_done)
        return flag

    # ----------------------------------------------------------- ImmCounter

    def imm_received_total(self, imm: int) -> int:
        """Receipts counted for `imm` so far (ImmCounterTable.received_total)."""
        return self.imm_received_totals([imm])[0]

    def imm_received_totals(self, imms: Sequence[int]) -> list[int]:
        """Receipt counts of several imms with one device gather and one
        device-to-host copy (what the callback thread polls)."""
        self._ensure_imm()
        if not imms:
            return []
        if len(imms) <= 64:
            # one small copy per counter on the library's private stream: a
            # few us, where a torch gather + .cpu() cost ~30 us per poll
            ptrs = (C.c_void_p * len(imms))(*[self._imm_slot_ptr(i) for i in imms])
            vals = (C.c_uint64 * len(imms))()
            _lib.call("txb_read_u64", ptrs, len(imms), vals)
            return [int(v) for v in vals]
        slots = [self._imm_slot(i) for i in imms]
        with torch.cuda.device(self.device), torch.cuda.stream(self._read_stream):
            counts = self._imm.tensor(_lib.TXB_IMM_SLOTS * 8, (_lib.TXB_IMM_SLOTS,), torch.int64)
            if len(slots) == 1:
                out = counts[slots[0]:slots[0] + 1].cpu()
            else:
                idx = torch.tensor(slots, dtype=torch.int64).to(counts.device, non_blocking=True)
                out = counts.index_select(0, idx).cpu()
        return [int(v) for v in out.tolist()]

    def expect_imm_count(self, imm: int, count: int, cb: Callable | None = None) -> ImmFlag:
        """Arm a threshold (engine.py:527-543 / ImmCounterTable.arm): fires
        once `count` receipts beyond those already consumed have arrived and
        consumes them, so the same imm can be re-armed round after round."""
        if not 0 <= imm < (1 << 32):
            raise TransferError(f"imm {imm} is not a u32")
        if count < 0:
            raise ProtocolError("negative imm count")
        self._ensure_imm()
        with self._lock:
            if imm in self._armed:
                raise ProtocolError(f"imm {imm} already armed")
            base = self._consumed.get(imm, 0)
            self._consumed[imm] = base + count
            flag = ImmFlag(self, imm, base + count, cb)
            self._armed[imm] = flag
        self.trace.record("imm_arm", imm=imm, count=count)
        if not flag._check() and cb is not None:
            self._callbacks().watch_flag(flag)
        return flag

    def _disarm(self, imm: int, flag: ImmFlag) -> None:
        with self._lock:
            if self._armed.get(imm) is flag:
                del self._armed[imm]

    def alloc_watcher(self, cb: Callable[[int, int], None], initial: int = 0) -> Watcher:
        """engine.py:621-632: a word the application bumps (host store or a
        device store through Watcher.device_ptr); the callback thread calls
        cb(old, new) when it changes."""
        w = Watcher(cb, initial)
        self._callbacks().add_watcher(w)
        return w

    def free_watcher(self, w: Watcher) -> None:
        """engine.py:634-638."""
        if self._cbt is not None:
            self._cbt.remove_watcher(w)

    def device_clock(self, steps: int | None = None) -> DeviceClock:
        """A device layer clock on this engine's GPU (kvcache LayerClock)."""
        self._ensure_imm()
        return DeviceClock(self, steps)

    def cancel_imm(self, imm: int) -> None:
        """ImmCounterTable.cancel: drop the expectation and realign the
        consumed count with the receipts seen so far."""
        total = self.imm_received_total(imm)
        with self._lock:
            self._armed.pop(imm, None)
            self._consumed[imm] = total

    # ---------------------------------------------------------------- close

    def close(self) -> None:
        if self._closed:
            return
        if self._cbt is not None:
            self._cbt.close()
        if self._stream is not None:
            self._stream.synchronize()
        for reg, imm in self._opened.values():
            reg.close()
            imm.close()
        self._opened.clear()
        for r in list(self._regions.values()):
            r.close()
        self._regions.clear()
        # the engine's streams stay alive with the process: tensors that
        # recorded use on them (record_stream) may be freed after close()
        self._closed = True
        if self in self.fabric.engines:
            self.fabric.engines.remove(self)

    def __enter__(self) -> "TransferEngine":
        return self

    def __exit__(self, *exc) -> None:
        self.close()


def local_engines(devices: Sequence[int], fabric: NvlinkFabric | None = None,
                  trace: bool = False) -> list[TransferEngine]:
    """One engine per device in this process (the single-box analog of the
    reference test harness's `engines(cfg, n)`, tests/_fabric.py:35-44)."""
    fab = fabric or NvlinkFabric()
    return [TransferEngine(fab, device=d, name=f"e{i}", trace=trace) for i, d in enumerate(devices)]
