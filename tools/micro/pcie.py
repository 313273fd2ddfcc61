"""Host link micro: copy-engine H2D / D2H vs SM zero-copy reads / writes of
page-locked host memory (txb_copy_pages on the mapped host address), at the
decode step's sizes.  Prints one line per case (us, GB/s).

python tools/micro/pcie.py
"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

import torch

from paper_2510_27656_b200 import _lib

dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
ticket = torch.zeros(4, dtype=torch.int32, device=dev)


def timed(fn, reps=30):
    ts = []
    for k in range(reps + 3):
        torch.cuda.synchronize()
        torch.cuda._sleep(100000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        if k >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def mapped(t):
    out = C.c_void_p()
    _lib.call("txb_host_device_ptr", C.c_void_p(t.data_ptr()), C.byref(out))
    return out.value


def sm_copy(dst_ptr, src_ptr, nbytes, page, tma, grid=0):
    j = _lib.Pages()
    j.src_base, j.src_offset, j.src_stride = src_ptr, 0, page
    j.dst_base, j.dst_offset, j.dst_stride = dst_ptr, 0, page
    j.npages, j.page_len = nbytes // page, page
    j.imm_ctr = None
    j.ticket = ticket.data_ptr()
    j.use_tma = tma
    j.single_device = 1
    _lib.call("txb_copy_pages", C.byref(j), grid, C.c_void_p(st.cuda_stream))


for nbytes in (1835008, 1 << 24, 1 << 26):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    hp = mapped(h)
    rows = [("CE H2D", timed(lambda: d.copy_(h, non_blocking=True))),
            ("CE D2H", timed(lambda: h.copy_(d, non_blocking=True)))]
    for page in (14336, 65536):
        if nbytes % page:
            continue
        for tma in (0, 1):
            rows.append((f"SM read  page={page} tma={tma}", timed(lambda: sm_copy(d.data_ptr(), hp, nbytes, page, tma))))
            rows.append((f"SM write page={page} tma={tma}", timed(lambda: sm_copy(hp, d.data_ptr(), nbytes, page, tma))))
    for name, us in rows:
        print(f"{nbytes:>10} B  {name:<28} {us:8.2f} us  {nbytes / us / 1e3:7.1f} GB/s", flush=True)
