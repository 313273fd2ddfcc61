"""Whole-request KV-cache transfer (BASELINE.json configs[4], SURVEY.md §8
cfg5: Llama-3-70B, 80 layers x 8 KV heads x 2048 slots of 8-KiB pages =
10 GiB, 16 chunks -> 1280 (chunk, layer) steps, floor 11.9 ms at 900 GB/s).

Prefiller on cuda:0, decoder pool on cuda:1 (NVLink; HBM loopback on one
GPU).  Modes:
  stream  -- KvSender.stream_all: ONE persistent kernel for the request,
             step k moving once the device layer clock reaches k.  "ready":
             the clock is advanced to the end before the kernel starts (the
             prefill ran ahead: pure transfer); "paced": a compute stream
             advances the clock once per layer-step after a simulated layer
             of --layer-us microseconds, and the report is the tail from the
             last advance to the last receipt.
  launch  -- one send_step kernel per step (the round-1 path), for contrast.
Every run checks the decoder pool byte for byte against the source pages
(device-side comparison of every page).  Prints one JSON line per mode.

python tools/bench_kv_stream.py [--grid 148] [--tma] [--reps 3]
"""
import argparse
import json
import sys
import time
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
ap.add_argument("--grid", type=int, default=0)
ap.add_argument("--tma", action="store_true")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--layer-us", type=float, default=0.0, help="paced mode: simulated compute per step (us)")
ap.add_argument("--modes", default="ready,launch")
a = ap.parse_args()

ngpu = torch.cuda.device_count()
d1 = 1 if ngpu > 1 else 0
if d1:
    enable_peer_access([0, 1])
fab = NvlinkFabric()
pre, dec_e = TransferEngine(fab, device=0, name="prefill"), TransferEngine(fab, device=d1, name="decode")
pre.use_tma = a.tma
ppc = a.slots // a.chunks
layout = kvcache.KvLayout(a.layers, a.chunks, ppc, a.page)
dec = kvcache.KvReceiver(dec_e, layout, pool_slots=a.slots, local_heads=a.heads, ctx_bytes=1 << 16)
rng = np.random.default_rng(0)
dec._free = list(rng.permutation(a.slots))     # scattered destination slots
total = layout.region_bytes(a.heads, layout.slots)
kv = pre.alloc_buffer(total)
W = a.page // 8
# page p holds int64 words p * W + [0, W): every page distinct
kv.view(torch.int64).view(-1, W).copy_(
    torch.arange(total // 8, dtype=torch.int64, device="cuda:0").view(-1, W))
ctx = pre.alloc_buffer(4096)
send = kvcache.KvSender(pre, kv, ctx)
peak_nvl, peak_hbm = 770.0, 6555.2
comp = torch.cuda.Stream(0)        # the "compute" stream that advances the layer clock
with torch.cuda.stream(comp):      # load the sleep kernel now: a first launch (lazy module
    torch.cuda._sleep(10)          # loading) does not complete while the stream kernel polls
comp.synchronize()
peak = peak_nvl if d1 else peak_hbm


def verify(t) -> bool:
    si, di = send.step_indices(t.request)
    dstw = dec.kv.view(torch.int64).view(-1, W)
    ok = True
    col = torch.arange(W, dtype=torch.int64, device=dstw.device)
    for c0 in range(0, si.size, 65536):
        s = torch.from_numpy(si[c0:c0 + 65536]).to(dstw.device)
        d = torch.from_numpy(di[c0:c0 + 65536]).to(dstw.device)
        want = s[:, None] * W + col[None, :]
        ok &= bool(torch.equal(dstw.index_select(0, d), want))
    return ok


def one_request(mode: str) -> dict:
    dec.kv.zero_()
    t = dec.open_request(ctx_len=4096)
    req = t.request
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(d1)
    st = pre.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = {}
    if mode == "launch":
        send.prepare(req)
        torch.cuda.synchronize(0)
        with torch.cuda.stream(st):
            torch.cuda._sleep(20_000_000)
        e0.record(st)
        for k in range(1, layout.steps + 1):
            send.send_step(req, k)
        e1.record(st)
    else:
        clock = pre.device_clock(layout.steps)
        send.prepare_stream(req)
        torch.cuda.synchronize(0)
        if mode == "ready":
            clock.advance(comp, by=layout.steps)
            comp.synchronize()
            # the GPU sleeps while the host enqueues the request, so the
            # events bracket the kernel, not the host's launch path
            with torch.cuda.stream(st):
                torch.cuda._sleep(20_000_000)
            e0.record(st)
            send.stream_all(req, clock, grid=a.grid)
            e1.record(st)
        else:  # paced: one simulated layer of compute, then the clock tick
            cyc = int(a.layer_us * 1.9e3)
            e0.record(st)
            send.stream_all(req, clock, grid=a.grid)
            e1.record(st)
            ec = torch.cuda.Event(enable_timing=True)
            ecs = torch.cuda.Event(enable_timing=True)
            ecs.record(comp)
            for k in range(layout.steps):
                with torch.cuda.stream(comp):
                    torch.cuda._sleep(cyc)
                clock.advance(comp)
            ec.record(comp)
    send.send_context(req)
    if not t.wait(60.0):
        raise SystemExit(f"{mode}: request did not complete: receipts {dec_e.imm_received_total(req.imm)} of "
                         f"{req.expected}, clock on device {clock.device_value() if mode != 'launch' else None}, "
                         f"engine error word {int(pre._err.cpu()[0])}")
    torch.cuda.synchronize(0)
    ms = e0.elapsed_time(e1)
    out["transfer_ms"] = round(ms, 3)
    out["gbs"] = round(total / (ms * 1e-3) / 1e9, 1)
    if mode == "paced":
        out["last_tick_to_end_us"] = round(ec.elapsed_time(e1) * 1e3, 1)
        out["compute_ms"] = round(ecs.elapsed_time(ec), 3)
    out["bytes_identical"] = verify(t)
    dec.release(t)
    return out


res_all = []
for mode in [m for m in a.modes.split(",") if m]:
    runs = [one_request(mode) for _ in range(a.reps)]
    best = min(runs, key=lambda r: r["transfer_ms"])
    res = {"metric": "KV whole-request transfer (Llama-3-70B, 32k ctx)", "mode": mode,
           "path": "NVLink cuda:0 -> cuda:1" if d1 else "HBM loopback cuda:0",
           "bytes": total, "steps": layout.steps, "pages_per_step": a.heads * ppc, "page_bytes": a.page,
           "copy": "TMA bulk, lane 0 of every warp issues" if a.tma else "16-byte vector copies, one warp per page",
           "grid": a.grid or "all SMs", "runs": runs, "best_ms": best["transfer_ms"], "best_gbs": best["gbs"],
           "frac_of_peak": round(best["gbs"] / peak, 3), "peak": peak,
           "floor_ms_900": round(total / 900e9 * 1e3, 2),
           "all_bytes_identical": all(r["bytes_identical"] for r in runs)}
    if mode == "paced":
        res["layer_us"] = a.layer_us
    print(json.dumps(res), flush=True)
pre.close()
dec_e.close()
