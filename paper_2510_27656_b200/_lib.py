"""ctypes binding of libtxb200.so (the C ABI declared in include/txb200.h).

The library is built in-tree (`make` / __graft_entry__.build()).  There is
no fallback: if it is missing, importing the hot path raises immediately.
ctypes.CDLL releases the GIL for the duration of every call, so ranks
driven from threads launch concurrently.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import ProtocolError, RailtxError, RegionError, TransferError

LIB_PATH = Path(__file__).resolve().parent / "libtxb200.so"

TXB_OK = 0
TXB_ERR_PROTOCOL = -1
TXB_ERR_TRANSFER = -2
TXB_ERR_REGION = -3
TXB_ERR_CUDA = -4

TXB_MAX_RANKS = 128
TXB_MAX_CTAS = 1024

EV_ROUTE_RANGE = 0x1
EV_ROUTE_DUP = 0x2
EV_WAIT_ROUTE = 0x4
EV_WAIT_TOKEN = 0x8
EV_WAIT_BARRIER = 0x10
EV_WAIT_COMBINE = 0x20
EV_CAPACITY = 0x40
EV_WAIT_IMM = 0x80
EV_WAIT_PRIV = 0x100

SRC_ROWS, SRC_F32, SRC_BF16 = 0, 1, 2


class Shape(C.Structure):
    """txb_moe_shape (include/txb200.h)."""

    _fields_ = [
        ("ranks", C.c_int32), ("experts", C.c_int32), ("max_tokens", C.c_int32),
        ("topk", C.c_int32), ("hidden", C.c_int32), ("elem_size", C.c_int32),
        ("scales", C.c_int32), ("comb_elem_size", C.c_int32), ("comb_scales", C.c_int32),
        ("me", C.c_int32), ("device", C.c_int32), ("single_device", C.c_int32),
        ("priv_tokens", C.c_int32), ("local_experts", C.c_int32),
        ("payload_bytes", C.c_int64), ("comb_bytes", C.c_int64), ("capacity", C.c_int64),
        ("grouped_rows", C.c_int64), ("comb_rows", C.c_int64),
        ("off_flags", C.c_uint64), ("off_route", C.c_uint64), ("off_grouped", C.c_uint64),
        ("off_comb", C.c_uint64), ("off_priv", C.c_uint64), ("region_bytes", C.c_uint64),
    ]


class Bufs(C.Structure):
    """txb_moe_bufs (include/txb200.h)."""

    _fields_ = [("region", C.c_void_p), ("peers", C.c_void_p), ("rank_scratch", C.c_void_p),
                ("pos", C.c_void_p), ("gidx", C.c_void_p), ("rows", C.c_void_p),
                ("sources", C.c_void_p), ("ret_slot", C.c_void_p), ("info", C.c_void_p),
                ("dirty", C.c_void_p), ("cta_hist", C.c_void_p), ("cta_bad", C.c_void_p),
                ("send_list", C.c_void_p), ("prof", C.c_void_p)]


class Pages(C.Structure):
    """txb_pages (include/txb200.h)."""

    _fields_ = [("src_base", C.c_void_p), ("src_offset", C.c_int64), ("src_stride", C.c_int64),
                ("src_idx", C.c_void_p), ("dst_base", C.c_void_p), ("dst_offset", C.c_int64),
                ("dst_stride", C.c_int64), ("dst_idx", C.c_void_p), ("npages", C.c_int64),
                ("page_len", C.c_int64), ("imm_ctr", C.c_void_p), ("ticket", C.c_void_p),
                ("use_tma", C.c_int32), ("single_device", C.c_int32)]


class StreamJob(C.Structure):
    """txb_stream_job (include/txb200.h): the persistent KV layer stream."""

    _fields_ = [("src", C.c_void_p), ("dst", C.c_void_p), ("page_len", C.c_int64),
                ("src_idx", C.c_void_p), ("dst_idx", C.c_void_p), ("pages_per_step", C.c_int64),
                ("nsteps", C.c_int32), ("use_tma", C.c_int32), ("clock", C.c_void_p),
                ("clock_base", C.c_uint64), ("imm_ctr", C.c_void_p), ("tickets", C.c_void_p),
                ("timeout_ns", C.c_uint64), ("err", C.c_void_p), ("single_device", C.c_int32),
                ("pad", C.c_int32)]


TXB_IMM_SLOTS = 131072
TXB_MAX_JOBS = 64

_VP = C.c_void_p
_I64 = C.c_int64
_U64 = C.c_uint64
_I32 = C.c_int32
_INT = C.c_int

# (name, argtypes) for every exported symbol; the ABI test checks this list
# against include/txb200.h.
SIGNATURES: dict[str, list] = {
    "txb_last_error": [],
    "txb_version": [],
    "txb_device_count": [C.POINTER(C.c_int)],
    "txb_alloc": [_INT, _U64, C.POINTER(_VP)],
    "txb_free": [_INT, _VP],
    "txb_memset": [_INT, _VP, _INT, _U64, _VP],
    "txb_ipc_export": [_INT, _VP, C.c_char_p],
    "txb_ipc_import": [_INT, C.c_char_p, C.POINTER(_VP)],
    "txb_ipc_close": [_INT, _VP],
    "txb_enable_peer": [_INT, _INT],
    "txb_stream_create": [_INT, C.POINTER(_VP)],
    "txb_preload": [_INT],
    "txb_check_failures": [_INT, C.POINTER(C.c_uint32)],
    "txb_stream_destroy": [_INT, _VP],
    "txb_host_device_ptr": [_VP, C.POINTER(_VP)],
    "txb_moe_plan": [C.POINTER(Shape)],
    "txb_moe_dispatch_fused": [C.POINTER(Shape), C.POINTER(Bufs), _VP, _INT, _I64, _VP, _U64, _VP],
    "txb_moe_combine_fused": [C.POINTER(Shape), C.POINTER(Bufs), _VP, _I64, _VP, _I64, _VP, _INT, _U64, _VP],
    "txb_moe_route": [C.POINTER(Shape), C.POINTER(Bufs), _VP, _I64, _VP],
    "txb_moe_dispatch": [C.POINTER(Shape), C.POINTER(Bufs), _VP, _INT, _I64, _VP, _U64, _INT, _VP],
    "txb_moe_dispatch_recv": [C.POINTER(Shape), C.POINTER(Bufs), _U64, _VP],
    "txb_moe_combine_send": [C.POINTER(Shape), C.POINTER(Bufs), _VP, _I64, _INT, _VP],
    "txb_moe_combine_recv": [C.POINTER(Shape), C.POINTER(Bufs), _VP, _I64, _VP, _I64, _VP, _INT, _U64, _VP],
    "txb_moe_barrier": [C.POINTER(Shape), C.POINTER(Bufs), _U64, _VP],
    "txb_moe_status": [C.POINTER(Shape), _VP, C.POINTER(C.c_uint32), C.POINTER(_U64), _I64],
    "txb_imm_table_slots": [],
    "txb_copy_pages": [C.POINTER(Pages), _INT, _VP],
    "txb_copy_jobs": [C.POINTER(Pages), _INT, _INT, _VP],
    "txb_kv_stream": [C.POINTER(StreamJob), _INT, _VP],
    "txb_imm_slot": [_VP, C.c_uint32, _INT, C.POINTER(_I64)],
    "txb_read_u64": [_VP, _INT, _VP],
    "txb_stream_write_value64": [_VP, _U64, _VP],
    "txb_stream_wait_value64": [_VP, _U64, _U64, _VP, _VP],
    "txb_imm_add": [_VP, _INT, _U64, _INT, _VP],
    "txb_imm_wait": [_VP, _U64, _U64, _VP, _VP],
    "txb_globaltimer": [_VP, _VP],
    "txb_fp8_quantize_tensor": [_VP, _I64, _VP, _VP, _VP],
    "txb_encode_rows": [_VP, _INT, _I64, _I32, _I32, _I32, _VP, _VP],
    "txb_decode_rows": [_VP, _I64, _I32, _I32, _I32, _VP, _VP],
    "txb_pack_rows": [_VP, _I64, _VP, _I64, _VP, _VP],
    "txb_weighted_combine": [_VP, _I64, _VP, _VP, _I64, _I32, _VP, _VP],
    "txb_fp8_encode": [_VP, _I64, _VP, _VP],
    "txb_fp8_decode": [_VP, _I64, _VP, _VP],
    "txb_bf16_encode": [_VP, _I64, _VP, _VP],
}

_lib: C.CDLL | None = None


def load() -> C.CDLL:
    """Load the in-tree library; raise loudly if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("TXB200_LIB", LIB_PATH))
    if not path.exists():
        raise RailtxError(
            f"{path} not found: build the sm_100a extension first "
            "(`make` or `python -c 'import __graft_entry__ as g; g.build()'`); "
            "there is no CPU fallback")
    lib = C.CDLL(str(path))
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_char_p if name == "txb_last_error" else C.c_int
    _lib = lib
    return lib


def last_error() -> str:
    return load().txb_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    """Map a txb status code onto the reference exception classes."""
    if rc == TXB_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == TXB_ERR_PROTOCOL:
        raise ProtocolError(msg)
    if rc == TXB_ERR_TRANSFER:
        raise TransferError(msg)
    if rc == TXB_ERR_REGION:
        raise RegionError(msg)
    raise RailtxError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
