"""Which compute-stream pattern lets a running k_kv_stream see the device
layer clock?  Small request, four ways of advancing the clock."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import torch

from paper_2510_27656_b200 import kvcache
from paper_2510_27656_b200.engine import NvlinkFabric, TransferEngine
from paper_2510_27656_b200.memory import enable_peer_access

d1 = 1 if torch.cuda.device_count() > 1 else 0
if d1:
    enable_peer_access([0, 1])
fab = NvlinkFabric()
a, b = TransferEngine(fab, device=0, name="p"), TransferEngine(fab, device=d1, name="d")
layout = kvcache.KvLayout(10, 5, 16, 8192)
dec = kvcache.KvReceiver(b, layout, pool_slots=layout.slots, local_heads=2, ctx_bytes=4096)
kv = a.alloc_buffer(layout.region_bytes(2, layout.slots))
send = kvcache.KvSender(a, kv, a.alloc_buffer(4096))
comp = torch.cuda.Stream(0)
if "--warm" in sys.argv:           # load torch's kernels before any stream kernel runs
    with torch.cuda.stream(comp):
        torch.cuda._sleep(10)
    torch.zeros(1, device="cuda:0").fill_(1)
    torch.cuda.synchronize()
for variant in ["memop_only", "memop_sync", "sleep_memop", "sleep_memop_sync", "kernelwrite_sleep"]:
    t = dec.open_request(ctx_len=64)
    clock = a.device_clock(layout.steps)
    send.prepare_stream(t.request)
    torch.cuda.synchronize()
    f = send.stream_all(t.request, clock, grid=8, timeout=5.0)
    time.sleep(0.05)
    for k in range(layout.steps):
        if "sleep" in variant:
            with torch.cuda.stream(comp):
                torch.cuda._sleep(20000)
        if variant.startswith("kernelwrite"):
            with torch.cuda.stream(comp):
                clock._t.fill_(k + 1)
            clock._value += 1
        else:
            clock.advance(comp)
        if variant.endswith("sync"):
            comp.synchronize()
    t_end = time.monotonic() + 3.0
    while b.imm_received_total(t.request.imm) < layout.steps and time.monotonic() < t_end:
        time.sleep(0.01)
    got = b.imm_received_total(t.request.imm)
    print(f"{variant:20s} receipts {got}/{layout.steps}  clock {clock.device_value()}  err {int(a._err.cpu()[0])}",
          flush=True)
    torch.cuda.synchronize()
    a._err.zero_()
    send.send_context(t.request).result(10)
    t.wait(5)
    dec.release(t)
