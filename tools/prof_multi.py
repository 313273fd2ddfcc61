"""Phase stamps of the fused kernels at EP=N (one rank per GPU, threads in
one process, CUDA-graph replays, L2 flushed before each step).

python tools/prof_multi.py [--ranks N] [--tokens T] [--reps K]
"""
import argparse
import sys
import threading
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

from paper_2510_27656_b200 import _lib, moe
from paper_2510_27656_b200.engine import local_engines

ap = argparse.ArgumentParser()
ap.add_argument("--ranks", type=int, default=torch.cuda.device_count())
ap.add_argument("--tokens", type=int, default=128)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--noflush", action="store_true")
a = ap.parse_args()
N, T, H, E, R = a.ranks, a.tokens, 7168, 256, 8
spec = moe.RoutingSpec(N, E, T, R, hidden=H, elem_size=1, scales=56, comb_elem_size=2, comb_scales=0)
mesh = moe.build_mesh(local_engines(list(range(N))), spec, timeout=20.0)
names = {0: "start", 14: "counted(+loads)", 1: "encoded", 2: "published+pos", 3: "routes-in",
         15: "dests", 5: "stored", 4: "tables", 6: "signalled", 7: "metadata", 8: "tokens-in",
         9: "c:start", 10: "c:sent", 11: "c:signalled", 12: "c:reduced", 13: "c:end"}
order = [0, 14, 1, 2, 3, 15, 5, 4, 6, 7, 8, 9, 10, 11, 12, 13]
stamps = [None] * N
times = [None] * N
bar = threading.Barrier(N)
CAPTURE = threading.Lock()


def worker(r):
    torch.cuda.set_device(r)
    rk = mesh[r]
    rng = np.random.default_rng(r)
    x = torch.from_numpy(rng.standard_normal((T, H)).astype(np.float32)).cuda().to(torch.bfloat16)
    rt = torch.from_numpy(np.argsort(rng.random((T, E)), axis=1)[:, :R].astype(np.int64)).cuda()
    w = torch.rand(T, R, device="cuda")
    y = torch.randn(int(rk._shape.grouped_rows), H, device="cuda").to(torch.bfloat16)
    side = torch.cuda.Stream()
    torch.cuda.set_stream(side)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    prof = torch.zeros(_lib.TXB_MAX_CTAS * 32, dtype=torch.int64, device="cuda")  # [grid][32], grid <= TXB_MAX_CTAS

    def one():
        rk.dispatch_send(x, rt, sync=False)
        rk.dispatch_recv(sync=False)
        rk.combine_send(y)
        rk.combine_recv(w, out_dtype=torch.bfloat16, sync=False)

    for _ in range(3):
        one()
    torch.cuda.synchronize()
    bar.wait()
    g = torch.cuda.CUDAGraph()
    rk._bufs.prof = prof.data_ptr()
    with CAPTURE:
        with torch.cuda.graph(g, stream=side, capture_error_mode="thread_local"):
            one()
    res, ts = [], []
    for _ in range(a.reps):
        if not a.noflush:
            flush.fill_(1)
        prof.zero_()
        torch.cuda.synchronize()
        bar.wait()
        rk.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        res.append(prof.view(_lib.TXB_MAX_CTAS, 32).cpu().numpy().astype(np.float64))
        ts.append(e0.elapsed_time(e1) * 1e3)
    rk._bufs.prof = 0
    stamps[r] = res[-1]
    times[r] = ts


th = [threading.Thread(target=worker, args=(r,)) for r in range(N)]
for t in th:
    t.start()
for t in th:
    t.join()
print(f"EP={N} step us per rep (max over ranks):",
      [round(max(times[r][k] for r in range(N)), 2) for k in range(a.reps)])
t0 = min(p[p[:, 0] > 0, 0].min() for p in stamps)
for k in order:
    vals = []
    for p in stamps:
        col = p[:, k]
        col = col[col > 0]
        if col.size:
            vals.append((np.median(col) - t0, col.max() - t0))
    if vals:
        print(f"{names[k]:12s} med(max over ranks) {max(v[0] for v in vals)/1e3:8.2f}us"
              f"  max {max(v[1] for v in vals)/1e3:8.2f}us")
for m in mesh:
    m.close()
# slowest CTAs per phase on rank 0 (relative to rank 0's earliest start)
p0 = stamps[0]
t00 = p0[p0[:, 0] > 0, 0].min()
for k in (6, 7, 8, 12, 13):
    col = p0[:, k]
    idx = np.argsort(-col)[:5]
    print(names[k], "slowest CTAs (rank 0)", [(int(i), round((col[i] - t00) / 1e3, 2)) for i in idx if col[i] > 0])
