"""Device regions: symmetric allocations, IPC descriptors, tensor views.

A region is one cudaMalloc allocation owned by libtxb200 (so its CUDA IPC
handle names the whole allocation).  Peers in the same process address it
directly once peer access is enabled; peers in other processes open its
64-byte IPC handle.  This stands in for the reference's registered memory
region and its rkey descriptor (engine.py:314-350, wire.py:64-97).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib

_TYPESTR = {
    torch.uint8: "|u1", torch.int8: "|i1", torch.int32: "<i4", torch.int64: "<i8",
    torch.float32: "<f4", torch.bfloat16: "<V2", torch.float16: "<f2", torch.int16: "<i2",
}


class _CAI:
    """Minimal __cuda_array_interface__ carrier for zero-copy torch views."""

    def __init__(self, ptr: int, shape: tuple, typestr: str, owner) -> None:
        self._owner = owner
        self.__cuda_array_interface__ = {
            "data": (int(ptr), False), "shape": tuple(int(s) for s in shape),
            "typestr": typestr, "strides": None, "version": 3}


def view(ptr: int, shape: tuple, dtype: torch.dtype, device: int, owner=None) -> torch.Tensor:
    """A torch tensor aliasing device memory at `ptr` (no copy)."""
    if dtype == torch.bfloat16:
        t = view(ptr, shape, torch.int16, device, owner)
        return t.view(torch.bfloat16)
    with torch.cuda.device(device):
        return torch.as_tensor(_CAI(ptr, shape, _TYPESTR[dtype], owner), device=f"cuda:{device}")


@dataclass
class Region:
    """One device allocation (owned, or imported from a peer process)."""

    device: int
    ptr: int
    nbytes: int
    imported: bool = False
    _closed: bool = False

    @classmethod
    def alloc(cls, device: int, nbytes: int) -> "Region":
        out = C.c_void_p()
        _lib.call("txb_alloc", device, nbytes, C.byref(out))
        return cls(device, int(out.value), nbytes)

    @classmethod
    def open_ipc(cls, device: int, handle: bytes, nbytes: int) -> "Region":
        out = C.c_void_p()
        _lib.call("txb_ipc_import", device, C.c_char_p(bytes(handle)), C.byref(out))
        return cls(device, int(out.value), nbytes, imported=True)

    def ipc_handle(self) -> bytes:
        buf = C.create_string_buffer(64)
        _lib.call("txb_ipc_export", self.device, C.c_void_p(self.ptr), buf)
        return buf.raw

    def tensor(self, offset: int, shape: tuple, dtype: torch.dtype) -> torch.Tensor:
        return view(self.ptr + offset, shape, dtype, self.device, owner=self)

    def close(self) -> None:
        if self._closed:
            return
        self._closed = True
        if self.imported:
            _lib.call("txb_ipc_close", self.device, C.c_void_p(self.ptr))
        else:
            _lib.call("txb_free", self.device, C.c_void_p(self.ptr))


def enable_peer_access(devices: list[int]) -> None:
    """All-pairs peer access between the devices of one process."""
    devs = sorted(set(devices))
    for a in devs:
        for b in devs:
            if a != b:
                _lib.call("txb_enable_peer", a, b)


def device_count() -> int:
    n = C.c_int(0)
    _lib.call("txb_device_count", C.byref(n))
    return int(n.value)
