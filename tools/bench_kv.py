"""Paged KV-cache layer transfer bandwidth (BASELINE.json configs[4]:
Llama-3-70B shape, 80 layers x 8 KV heads, 16-token pages of 128 dims x
2 B x (K, V) = 8 KiB, 32k context = 2048 slots).

Prefiller on cuda:0, decoder on cuda:1 when present (NVLink), else both on
cuda:0 (HBM loopback).  One step = one (chunk, layer) paged write of
heads x pages_per_chunk pages (kvcache.py:477-500), TMA bulk copies into a
randomly permuted slot list of the decoder pool (TMA by default here; the
engine's own default is vector copies).  Prints one JSON line.

python tools/bench_kv.py [--layers 80] [--chunks 16] [--steps 50] [--no-tma]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

from paper_2510_27656_b200 import kvcache
from paper_2510_27656_b200.engine import NvlinkFabric, TransferEngine
from paper_2510_27656_b200.memory import enable_peer_access

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=80)
ap.add_argument("--chunks", type=int, default=16)
ap.add_argument("--heads", type=int, default=8)
ap.add_argument("--slots", type=int, default=2048)
ap.add_argument("--page", type=int, default=8192)
ap.add_argument("--steps", type=int, default=40)
ap.add_argument("--no-tma", action="store_true")
a = ap.parse_args()

ngpu = torch.cuda.device_count()
d1 = 1 if ngpu > 1 else 0
if d1:
    enable_peer_access([0, 1])
fab = NvlinkFabric()
pre, dec_e = TransferEngine(fab, device=0, name="prefill"), TransferEngine(fab, device=d1, name="decode")
ppc = a.slots // a.chunks
layout = kvcache.KvLayout(a.layers, a.chunks, ppc, a.page)
dec = kvcache.KvReceiver(dec_e, layout, pool_slots=a.slots, local_heads=a.heads, ctx_bytes=1 << 16)
rng = np.random.default_rng(0)
dec._free = list(rng.permutation(a.slots))     # scattered destination slots
t = dec.open_request(ctx_len=4096)
kv = pre.alloc_buffer(layout.region_bytes(a.heads, layout.slots))
kv.fill_(7)
ctx = pre.alloc_buffer(4096)
send = kvcache.KvSender(pre, kv, ctx)
pre.use_tma = not a.no_tma
send.prepare(t.request)
torch.cuda.synchronize()
step_bytes = a.heads * ppc * a.page
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda:0")
st = pre.stream
times = []
pre.timing = []
for k in range(1, min(layout.steps, a.steps) + 5):
    torch.cuda.synchronize(0)
    flush.fill_(1)            # still running while the step is enqueued behind it
    send.send_step(t.request, k)
    torch.cuda.synchronize(0)
    e0, e1 = pre.timing[-1]
    if k > 4:
        times.append(e0.elapsed_time(e1) * 1e3)
pre.timing = None
# full request: every step + context, completion observed by the decoder
torch.cuda.synchronize()
import time
t0 = time.perf_counter()
for k in range(min(layout.steps, a.steps) + 5, layout.steps + 1):
    send.send_step(t.request, k)
send.send_context(t.request)
ok_partial = True
med = float(np.median(times))
res = {"metric": "paged KV layer transfer GB/s (Llama-3-70B shape)", "value": round(step_bytes / (med * 1e-6) / 1e9, 1),
       "unit": "GB/s", "path": "NVLink cuda:0 -> cuda:1" if d1 else "HBM loopback cuda:0",
       "step_bytes": step_bytes, "step_us_p50": round(med, 2),
       "peak": 770.0 if d1 else 6555.2,
       "frac": round(step_bytes / (med * 1e-6) / 1e9 / (770.0 if d1 else 6555.2), 3),
       "pages_per_step": a.heads * ppc, "page_bytes": a.page, "layers": a.layers, "chunks": a.chunks,
       "copy": ("k_copy_jobs: TMA bulk copies (cp.async.bulk) of 8-KiB pieces issued by lane 0 of every warp, "
                "2 stages each" if not a.no_tma else
                "k_copy_jobs: 16-byte vector copies, one warp per 8-KiB piece") + ", one ImmCounter receipt per step"}
assert t.wait(60.0), "KV request did not complete"
res["request_completed"] = True
print(json.dumps(res))
