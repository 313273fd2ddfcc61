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

import itertools
from dataclasses import dataclass
from typing import Sequence

import torch

from . import memory
from .errors import RegionError, TransferError


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


class TransferEngine:
    """One rank's endpoint on one CUDA device."""

    def __init__(self, fabric: NvlinkFabric | None = None, *, device: int = 0,
                 name: str | None = None, rails: int = 1, engine_id: int | None = None) -> None:
        if not 1 <= rails <= 4:
            raise TransferError(f"rail count {rails} outside 1..4")
        self.fabric = fabric or NvlinkFabric()
        self.engine_id = engine_id if engine_id is not None else self.fabric.allocate_engine_id()
        self.name = name or f"e{self.engine_id}"
        self.device = int(device)
        self.fabric.engines.append(self)
        self._regions: dict[int, memory.Region] = {}
        self._closed = False

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

    def close(self) -> None:
        if self._closed:
            return
        for r in list(self._regions.values()):
            r.close()
        self._regions.clear()
        self._closed = True
        if self in self.fabric.engines:
            self.fabric.engines.remove(self)

    def __enter__(self) -> "TransferEngine":
        return self

    def __exit__(self, *exc) -> None:
        self.close()


def local_engines(devices: Sequence[int], fabric: NvlinkFabric | None = None) -> list[TransferEngine]:
    """One engine per device in this process (the single-box analog of the
    reference test harness's `engines(cfg, n)`, tests/_fabric.py:35-44)."""
    fab = fabric or NvlinkFabric()
    return [TransferEngine(fab, device=d, name=f"e{i}") for i, d in enumerate(devices)]
