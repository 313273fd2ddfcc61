"""Numeric kernels on the GPU -- the "cuda" entry of the reference kernel
registry (railtx/kernels.py:245-264).

Same functions and semantics as the reference numpy/numba variants:
e4m3 encode/decode (RNE, satfinite 448, NaN -> 0x7F), bf16 RNE encode,
pack_rows gather and the fp32 weighted combine (j-ordered, no FMA).  Inputs
may be numpy arrays (copied to the current device, result copied back) or
CUDA tensors (result stays on the device).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib

FP8_MAX = 448.0
FP8_NAN = 0x7F


def _dev(x, dtype: torch.dtype) -> tuple[torch.Tensor, bool]:
    if isinstance(x, torch.Tensor) and x.is_cuda:
        return x.to(dtype).contiguous(), False
    a = np.ascontiguousarray(x.cpu().numpy() if isinstance(x, torch.Tensor) else x)
    return torch.from_numpy(a).to(device="cuda", dtype=dtype), True


def _sid(t: torch.Tensor) -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _ret(t: torch.Tensor, host: bool):
    return t.cpu().numpy() if host else t


def fp8_encode(x):
    xt, host = _dev(x, torch.float32)
    out = torch.empty(xt.shape, dtype=torch.uint8, device=xt.device)
    _lib.call("txb_fp8_encode", C.c_void_p(xt.data_ptr()), xt.numel(), C.c_void_p(out.data_ptr()), _sid(xt))
    return _ret(out, host)


def fp8_decode(b):
    bt, host = _dev(b, torch.uint8)
    out = torch.empty(bt.shape, dtype=torch.float32, device=bt.device)
    _lib.call("txb_fp8_decode", C.c_void_p(bt.data_ptr()), bt.numel(), C.c_void_p(out.data_ptr()), _sid(bt))
    return _ret(out, host)


def bf16_encode(x):
    xt, host = _dev(x, torch.float32)
    out = torch.empty(xt.shape, dtype=torch.int16, device=xt.device)
    _lib.call("txb_bf16_encode", C.c_void_p(xt.data_ptr()), xt.numel(), C.c_void_p(out.data_ptr()), _sid(xt))
    if host:
        return out.cpu().numpy().view(np.uint16)
    return out


def bf16_decode(h):
    if isinstance(h, torch.Tensor) and h.is_cuda:
        return (h.to(torch.int32) << 16).view(torch.float32)
    return (np.asarray(h, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def pack_rows(src, rows):
    st, host = _dev(src, torch.uint8) if not (isinstance(src, torch.Tensor) and src.is_cuda) \
        else (src.contiguous(), False)
    rt, _ = _dev(rows, torch.int64)
    width = st.shape[1] * st.element_size()
    out = torch.empty((rt.shape[0],) + tuple(st.shape[1:]), dtype=st.dtype, device=st.device)
    _lib.call("txb_pack_rows", C.c_void_p(st.data_ptr()), width, C.c_void_p(rt.data_ptr()),
              rt.shape[0], C.c_void_p(out.data_ptr()), _sid(st))
    return _ret(out, host)


def weighted_combine(y, rows, weights):
    yt, host = _dev(y, torch.float32)
    rt, _ = _dev(rows, torch.int64)
    wt, _ = _dev(weights, torch.float32)
    n, r = rt.shape
    out = torch.empty((n, yt.shape[1]), dtype=torch.float32, device=yt.device)
    _lib.call("txb_weighted_combine", C.c_void_p(yt.data_ptr()), yt.shape[1], C.c_void_p(rt.data_ptr()),
              C.c_void_p(wt.data_ptr()), n, r, C.c_void_p(out.data_ptr()), _sid(yt))
    return _ret(out, host)


def implementations() -> dict[str, dict[str, object]]:
    """The registry entry a railtx caller would select (kernels.py:245-264)."""
    return {"cuda": {
        "fp8_encode": fp8_encode,
        "fp8_decode": fp8_decode,
        "bf16_encode": bf16_encode,
        "pack_rows": pack_rows,
        "weighted_combine": weighted_combine,
    }}
