"""NVLink peer-write micro: txb_copy_pages from cuda:0 HBM into cuda:1 HBM
(peer-mapped pointer), at the MoE step sizes, TMA bulk vs 16-byte vector
stores, grid sizes 1-4 CTAs per SM.  Also the copy-engine peer copy.  The
span is device time of one copy kernel (launch hidden behind a sleep).

python tools/micro/peer.py
"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

import torch

from paper_2510_27656_b200 import _lib
from paper_2510_27656_b200.memory import enable_peer_access

enable_peer_access([0, 1])
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
ticket = torch.zeros(4, dtype=torch.int32, device=dev)
sms = torch.cuda.get_device_properties(0).multi_processor_count


def timed(fn, reps=20):
    ts = []
    for k in range(reps + 3):
        torch.cuda.synchronize(0)
        torch.cuda._sleep(100000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize(0)
        if k >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def sm_copy(dst_ptr, src_ptr, nbytes, page, tma, grid):
    j = _lib.Pages()
    j.src_base, j.src_offset, j.src_stride = src_ptr, 0, page
    j.dst_base, j.dst_offset, j.dst_stride = dst_ptr, 0, page
    j.npages, j.page_len = nbytes // page, page
    j.imm_ctr = None
    j.ticket = ticket.data_ptr()
    j.use_tma = tma
    j.single_device = 0
    _lib.call("txb_copy_pages", C.byref(j), grid, C.c_void_p(st.cuda_stream))


for nbytes in (7392 * 512, 14336 * 512, 14336 * 896, 1 << 24, 1 << 26):
    s = torch.empty(nbytes, dtype=torch.uint8, device=dev).fill_(3)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda:1")
    page = 7392 if nbytes % 14336 else 14336
    rows = [("CE peer", timed(lambda: d.copy_(s, non_blocking=True)))]
    for tma in (0, 1):
        for g in (sms, 2 * sms, 4 * sms):
            rows.append((f"SM tma={tma} grid={g}", timed(lambda: sm_copy(d.data_ptr(), s.data_ptr(), nbytes, page, tma, g))))
    for name, us in rows:
        print(f"{nbytes:>10} B  {name:<24} {us:8.2f} us  {nbytes / us / 1e3:7.1f} GB/s", flush=True)
