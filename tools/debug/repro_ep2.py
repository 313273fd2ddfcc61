"""Debug repro: EP=2 decode steps in one process (thread mesh over cuda:0/1),
graph-free, many steps; --experts / --skew select the shape."""
import argparse, sys, threading
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np, torch
import bench
from paper_2510_27656_b200 import moe
from paper_2510_27656_b200.engine import local_engines
ap = argparse.ArgumentParser()
ap.add_argument("--experts", type=int, default=384)
ap.add_argument("--skew", type=int, default=1)
ap.add_argument("--steps", type=int, default=200)
ap.add_argument("--sync", type=int, default=0)
a = ap.parse_args()
wl = dict(bench.WORKLOADS["kimi"]); wl["experts"] = a.experts; wl["routing"] = "skewed" if a.skew else "uniform"
N = 2
spec = moe.RoutingSpec(ranks=N, experts=a.experts, max_tokens=128, topk=8, hidden=7168, elem_size=1, scales=56,
                       comb_elem_size=2, comb_scales=0)
mesh = moe.build_mesh(local_engines([0, 1]), spec, timeout=20.0)
ins = []
for r in range(N):
    dev = torch.device("cuda", r)
    x, routes, w = bench._inputs(wl, r, 128)
    G = int(mesh[r]._shape.grouped_rows)
    ins.append((torch.from_numpy(x).to(dev).to(torch.bfloat16), torch.from_numpy(routes).to(dev),
                torch.from_numpy(w).to(dev), torch.randn(G, 7168, device=dev).to(torch.bfloat16)))
errs = []
def worker(r):
    try:
        torch.cuda.set_device(r)
        xd, rd, wd, y = ins[r]
        for k in range(a.steps):
            mesh[r].dispatch_send(xd, rd, sync=False)
            mesh[r].dispatch_recv(sync=False)
            mesh[r].combine_send(y)
            mesh[r].combine_recv(wd, out_dtype=torch.bfloat16, sync=False)
            if a.sync:
                torch.cuda.synchronize(r)
        torch.cuda.synchronize(r)
        e, _ = mesh[r].status()
        assert e == 0, hex(e)
    except Exception as exc:
        errs.append(f"rank {r}: {exc!r}"[:300])
th = [threading.Thread(target=worker, args=(r,)) for r in range(N)]
[t.start() for t in th]; [t.join() for t in th]
print(f"E={a.experts} skew={a.skew} sync={a.sync}:", "OK" if not errs else errs)
