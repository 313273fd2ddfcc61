"""RL weight publication on B200 (data path of railtx.weights: `prepare`
narrowing, weights.py:370-387, and the per-destination single writes,
weights.py:570-590).

`prepare_device` turns one task's assembled bf16 words into wire bytes on
the GPU: bf16 passes through, fp8 is a per-TENSOR e4m3 quantisation
(amax over finite values / 448, IEEE division, RNE satfinite) followed by
the 4-byte f32 scale footer -- byte-identical to the reference `prepare`.
`publish` writes the prepared bytes to every destination with one
WriteImm each.  The schedule builder, shard store and pipeline threads of
the reference are host control plane and out of scope.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

import torch

from . import _lib
from .engine import MrDesc, MrHandle, Pages, TransferEngine
from .errors import ScheduleError

DT_BF16 = "bf16"
DT_FP8 = "fp8"
_ESIZE = {DT_BF16: 2, DT_FP8: 1}
_SCALE_BYTES = 4


@dataclass(frozen=True)
class ParamMeta:
    """One parameter as seen by one rank (weights.py:41-96)."""

    name: str
    shape: tuple
    dtype: str
    group: int = 0
    axis: int = 0
    shard_index: int = 0
    shard_count: int = 1
    offload: bool = False

    def __post_init__(self) -> None:
        if self.dtype not in _ESIZE:
            raise ScheduleError(f"{self.name}: unknown dtype {self.dtype!r}")
        if not self.shape or any(d <= 0 for d in self.shape):
            raise ScheduleError(f"{self.name}: bad shape {self.shape}")
        if not 0 <= self.axis < len(self.shape):
            raise ScheduleError(f"{self.name}: shard axis {self.axis} outside shape {self.shape}")
        if self.shard_count < 1 or not 0 <= self.shard_index < self.shard_count:
            raise ScheduleError(f"{self.name}: shard {self.shard_index} of {self.shard_count} is invalid")
        if self.shape[self.axis] % self.shard_count:
            raise ScheduleError(f"{self.name}: axis {self.axis} of {self.shape[self.axis]} "
                                f"does not tile into {self.shard_count} shards")

    @property
    def nelems(self) -> int:
        n = 1
        for d in self.shape:
            n *= d
        return n

    @property
    def shard_nelems(self) -> int:
        return self.nelems // self.shard_count

    def payload_bytes(self) -> int:
        n = self.shard_nelems * _ESIZE[self.dtype]
        return n + _SCALE_BYTES if self.dtype == DT_FP8 else n


def prepare_device(words: torch.Tensor, dtype: str, out: torch.Tensor | None = None) -> torch.Tensor:
    """bf16 words (CUDA int16/uint16 view of the sliced tensor, any shape)
    -> wire bytes (uint8 CUDA tensor): raw for bf16, fp8 + f32 footer for
    fp8 (weights.py:383-387)."""
    if dtype not in _ESIZE:
        raise ScheduleError(f"unknown dtype {dtype!r}")
    w = words.contiguous().view(torch.int16).reshape(-1)
    n = w.numel()
    if dtype == DT_BF16:
        b = w.view(torch.uint8)
        if out is None:
            return b.clone()
        out[:2 * n].copy_(b)
        return out
    dev = w.device
    if out is None:
        out = torch.empty(n + _SCALE_BYTES, dtype=torch.uint8, device=dev)
    scratch = torch.empty(1, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream(dev)
    _lib.call("txb_fp8_quantize_tensor", C.c_void_p(w.data_ptr()), n, C.c_void_p(scratch.data_ptr()),
              C.c_void_p(out.data_ptr()), C.c_void_p(st.cuda_stream))
    return out


def publish(engine: TransferEngine, prepared: torch.Tensor, dsts: Sequence[tuple[MrDesc, int]],
            imm: int | None = None, handle: MrHandle | None = None, wait: bool = True):
    """One WriteImm of the prepared bytes to each destination
    (RankExecutor._lane_write, weights.py:570-590), all destinations in ONE
    kernel launch (k_copy_jobs), each releasing its own receipt.  `handle`:
    the prepared buffer's registration, reused across updates (registered and
    released here when None).  wait=False returns as soon as the copy is
    enqueued; the caller waits on the returned flag (or the receivers on
    their ImmFlags)."""
    own = handle is None
    h = engine.reg_mr(prepared)[0] if own else handle
    try:
        n = prepared.numel() * prepared.element_size()
        flag = engine._launch_jobs([(h.base, Pages((0,), 0, 0), d, Pages((0,), 0, off), n, 1 if n else 0, imm)
                                    for d, off in dsts], label="weights.publish")
        if wait:
            flag.wait()
    finally:
        if own:
            engine.dereg_mr(h)   # host bookkeeping only: the memory stays with the caller
    return [flag]
