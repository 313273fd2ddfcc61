"""Probe: do NVML's NVLink byte counters see device peer writes, and at what
granularity?  Copies a known number of bytes cuda:0 -> cuda:1 (peer pointer,
torch copy = copy engine, and an SM copy kernel) and prints the counter deltas
(fields DATA_TX/RX 138/139 in KiB, RAW_TX/RX 140/141, COUNT_XMIT/RCV 202/204)
per device, scope = all links (scopeId UINT_MAX) and link 0.

python tools/micro/nvml_nvlink.py
"""
import time

import pynvml as nv
import torch

nv.nvmlInit()
h = [nv.nvmlDeviceGetHandleByIndex(i) for i in range(2)]
FIELDS = {"DATA_TX": 138, "DATA_RX": 139, "RAW_TX": 140, "RAW_RX": 141, "XMIT_B": 202, "RCV_B": 204}


def read(dev):
    ids = [(fid, scope) for fid in FIELDS.values() for scope in (0xFFFFFFFF, 0)]
    vals = nv.nvmlDeviceGetFieldValues(dev, ids)
    out = {}
    k = 0
    for name in FIELDS:
        for scope in (0xFFFFFFFF, 0):
            r = vals[k]
            k += 1
            out[(name, scope)] = r.value.ullVal if r.nvmlReturn == 0 else f"err{r.nvmlReturn}"
    return out


a = torch.empty(64 << 20, dtype=torch.uint8, device="cuda:0")
b = torch.empty(64 << 20, dtype=torch.uint8, device="cuda:1")
torch.cuda.synchronize(0)
for nbytes in (64 << 20, 8 << 20):
    for reps in (1, 10):
        before = [read(x) for x in h]
        for _ in range(reps):
            b[:nbytes].copy_(a[:nbytes])
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        time.sleep(0.2)
        after = [read(x) for x in h]
        print(f"copy {nbytes} B x{reps} = {nbytes * reps} B")
        for d in range(2):
            row = []
            for k in before[d]:
                x, y = before[d][k], after[d][k]
                row.append(f"{k[0]}@{'all' if k[1] else 'l0'}={(y - x) if isinstance(x, int) and isinstance(y, int) else (x, y)}")
            print(f"  dev{d}: " + " ".join(row))
