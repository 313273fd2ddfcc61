"""Where the bench step's time goes at EP=N, one process per GPU (the bench's
own launch shape): every rank replays a CUDA graph of the public-API step
bracketed by %globaltimer samples, with the kernels' phase stamps on, after
the same L2 flush + device barrier as bench.py.  Per rank it reports the
event span and, in the device clock, graph start -> dispatch start ->
dispatch end -> combine start -> combine end -> graph end.

python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
    --master-port 29533 tools/prof_torchrun.py [--config decode] [--reps 50]
"""
import argparse
import ctypes as C
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch
import torch.distributed as dist

import bench
from paper_2510_27656_b200 import _lib, moe
from paper_2510_27656_b200.engine import NvlinkFabric, TransferEngine

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="decode")
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--mode", default="graph", choices=["graph", "eager", "empty"])
ap.add_argument("--noflush", action="store_true")
ap.add_argument("--mid", action="store_true", help="a %globaltimer kernel between dispatch and combine")
ap.add_argument("--sleep", type=int, default=0, help="GPU sleep cycles queued before the graph (host runs ahead)")
ap.add_argument("--private", type=int, default=None, help="PrivateBufferConfig.tokens")
ap.add_argument("--cta", type=int, nargs="*", default=[], help="also print these CTAs' own stamps")
a = ap.parse_args()

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
wl = bench.WORKLOADS[a.config]
T, E, R, H = wl["tokens"], wl["experts"], wl["topk"], wl["hidden"]
spec = moe.RoutingSpec(ranks=world, experts=E, max_tokens=T, topk=R, hidden=H, elem_size=wl["elem"],
                       scales=wl["scales"], comb_elem_size=2, comb_scales=0)
priv = None if a.private is None else moe.PrivateBufferConfig(a.private)
if world > 1:
    dist.init_process_group("gloo")
    rk = moe.connect_process_group(TransferEngine(NvlinkFabric(group=dist.group.WORLD), device=local), spec,
                                   private=priv)
else:
    rk = moe.build_mesh([TransferEngine(NvlinkFabric(), device=local)], spec, private=priv)[0]
rk.record_stats = False
x, routes, w = bench._inputs(wl, rank, T)
xd = torch.from_numpy(x).to(dev).to(torch.bfloat16)
rd = torch.from_numpy(routes).to(dev)
wd = torch.from_numpy(w).to(dev)
y = torch.randn(int(rk._shape.grouped_rows), H, device=dev).to(torch.bfloat16)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
NS = _lib.TXB_MAX_CTAS  # stamp rows: one per CTA of the largest launch (<= TXB_MAX_CTAS)
prof = torch.zeros(NS * 32, dtype=torch.int64, device=dev)
gt = torch.zeros(4, dtype=torch.int64, device=dev)
sid = C.c_void_p(stream.cuda_stream)


def step():
    rk.dispatch_send(xd, rd, sync=False)
    rk.dispatch_recv(sync=False)
    if a.mid:
        _lib.call("txb_globaltimer", C.c_void_p(gt.data_ptr() + 24), sid)
    rk.combine_send(y)
    rk.combine_recv(wd, out_dtype=torch.bfloat16, sync=False)


for _ in range(5):
    step()
torch.cuda.synchronize()
rk._bufs.prof = prof.data_ptr()


def stamped():
    _lib.call("txb_globaltimer", C.c_void_p(gt.data_ptr()), sid)
    if a.mode != "empty":
        step()
    _lib.call("txb_globaltimer", C.c_void_p(gt.data_ptr() + 8), sid)


if a.mode == "eager":
    run = stamped
else:
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        stamped()
    rk._bufs.prof = 0
    run = g.replay
rows = []
detail = []
lastcta = []
ctarows = []
ORDER = [0, 19, 22, 27, 28, 24, 25, 14, 1, 2, 26, 3, 15, 20, 16, 17, 18, 4, 7, 5, 6, 8, 9, 10, 11, 23, 12, 13]
STAMP = {27: "dups checked", 28: "ids synced", 26: "priv stored", 24: "seg prefix", 25: "seg sync2", 0: "start", 19: "own routes in", 22: "hist done", 14: "counted(+loads)", 1: "encoded", 2: "published+pos", 3: "routes-in", 15: "dests",
         5: "joined", 20: "tok stored", 16: "T:loaded", 17: "T:srcpre", 18: "T:scan", 4: "tables", 6: "signalled", 7: "metadata", 8: "tokens-in", 9: "c:start", 10: "c:sent",
         11: "c:signalled", 23: "c:waited", 12: "c:reduced", 13: "c:end"}
for k in range(a.reps + 5):
    if not a.noflush:
        flush.fill_(k & 0xFF)
    if world > 1:
        rk.barrier()
    _lib.call("txb_globaltimer", C.c_void_p(gt.data_ptr() + 16), sid)   # barrier done
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prof.zero_()
    if a.sleep:
        torch.cuda._sleep(a.sleep)
    e0.record(stream)
    run()
    e1.record(stream)
    torch.cuda.synchronize()
    if k < 5:
        continue
    p = prof.view(NS, 32).cpu().numpy().astype(np.float64)
    t = gt.cpu().numpy().astype(np.float64)
    base = t[0]

    def lo(i):
        v = p[:, i][p[:, i] > 0]
        return (v.min() - base) / 1e3 if v.size else np.nan

    def hi(i):
        v = p[:, i][p[:, i] > 0]
        return (v.max() - base) / 1e3 if v.size else np.nan

    det, amax = [], []
    for kk in ORDER:
        v = p[:, kk][p[:, kk] > 0]
        det.append(((np.median(v) - base) / 1e3, (v.max() - base) / 1e3) if v.size else (np.nan, np.nan))
        amax.append(int(np.argmax(p[:, kk])) if v.size else -1)
    detail.append(det)
    lastcta.append(amax)
    ctarows.append([[(p[c, kk] - base) / 1e3 if p[c, kk] > 0 else np.nan for kk in ORDER] for c in a.cta])
    rows.append([e0.elapsed_time(e1) * 1e3, (t[2] - base) / 1e3, lo(0), hi(3), hi(8), lo(9), hi(11), hi(13),
                 (t[1] - base) / 1e3, (t[3] - base) / 1e3 if a.mid else np.nan])
med = np.median(np.asarray(rows), axis=0).tolist()
names = ["event_span", "barrier_done", "disp_start", "routes_in_last", "disp_end", "comb_start",
         "comb_signalled_last", "comb_end", "graph_end", "mid_stamp"]
mine = dict(zip(names, [round(v, 2) for v in med]))
allr = [None] * world
if world > 1:
    dist.all_gather_object(allr, mine)
else:
    allr = [mine]
dmed = np.nanmedian(np.asarray(detail), axis=0)
lc = np.asarray(lastcta)


def _mode(col):
    vals, cnt = np.unique(col, return_counts=True)
    return int(vals[np.argmax(cnt)]), int(cnt.max())


lines = [f"  {STAMP[k]:16s} median CTA {m:7.2f}  last CTA {x:7.2f}  (last is CTA {_mode(lc[:, i])[0]:>3} "
         f"in {_mode(lc[:, i])[1]}/{lc.shape[0]} reps)"
         for i, (k, (m, x)) in enumerate(zip(ORDER, dmed.tolist()))]
if a.cta:
    cm = np.nanmedian(np.asarray(ctarows), axis=0)  # [len(cta)][ORDER]
    for ci, c in enumerate(a.cta):
        lines.append(f"  -- CTA {c}: " + ", ".join(f"{STAMP[k]} {v:.2f}" for k, v in zip(ORDER, cm[ci].tolist())
                                                 if not np.isnan(v)))
alld = [None] * world
if world > 1:
    dist.all_gather_object(alld, lines)
else:
    alld = [lines]
if rank == 0:
    for r, ls in enumerate(alld):
        print(f"rank {r} phase stamps (us from graph start, median over reps)")
        print("\n".join(ls))
if rank == 0:
    print("us, device clock of each rank relative to its graph start (median over reps)")
    print("rank " + " ".join(f"{n:>18}" for n in names))
    for r, d in enumerate(allr):
        print(f"{r:>4} " + " ".join(f"{d[n]:>18.2f}" for n in names))
    print(json.dumps({"config": a.config, "mode": a.mode, "ranks": world, "per_rank": allr}))
rk.close()
if world > 1:
    dist.barrier()
    dist.destroy_process_group()
