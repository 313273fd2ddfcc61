"""Eager DeepSeek-V3 decode steps at EP=1 for ncu captures (no graphs, no
flush): python tools/prof_step.py [--steps N] [--tokens T]."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

from paper_2510_27656_b200 import _lib, moe
from paper_2510_27656_b200.engine import local_engines

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--tokens", type=int, default=128)
ap.add_argument("--comb", type=int, default=2)
ap.add_argument("--graph", action="store_true", help="stamps from CUDA-graph replays with an L2 flush")
a = ap.parse_args()
T, H, E, R = a.tokens, 7168, 256, 8
spec = moe.RoutingSpec(1, E, T, R, hidden=H, elem_size=1, scales=56, comb_elem_size=a.comb, comb_scales=0)
rk = moe.build_mesh(local_engines([0]), spec)[0]
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.standard_normal((T, H)).astype(np.float32)).cuda().to(torch.bfloat16)
r = torch.from_numpy(np.argsort(rng.random((T, E)), axis=1)[:, :R].astype(np.int64)).cuda()
w = torch.rand(T, R, device="cuda")
y = torch.randn(int(rk._shape.grouped_rows), H, device="cuda").to(torch.bfloat16)
for _ in range(a.steps):
    rk.dispatch_send(x, r, sync=False)
    rk.dispatch_recv(sync=False)
    rk.combine_send(y)
    rk.combine_recv(w, out_dtype=torch.bfloat16, sync=False)
torch.cuda.synchronize()
err, _ = rk.status()
assert err == 0, hex(err)
print("ok")

# phase stamps of the fused kernels (%globaltimer, per CTA)
prof = torch.zeros(_lib.TXB_MAX_CTAS * 32, dtype=torch.int64, device="cuda")  # [grid][32], grid <= TXB_MAX_CTAS
rk._bufs.prof = prof.data_ptr()
names = ["start", "counted", "positions", "routes-in", "layout", "stored", "signalled", "metadata",
         "tokens-in", "c:start", "c:sent", "c:signalled", "c:reduced", "c:end"]
def one():
    rk.dispatch_send(x, r, sync=False)
    rk.dispatch_recv(sync=False)
    rk.combine_send(y)
    rk.combine_recv(w, out_dtype=torch.bfloat16, sync=False)

if a.graph:
    side = torch.cuda.Stream()
    torch.cuda.set_stream(side)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    one(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        one()
    for _ in range(3):
        flush.fill_(1)
        prof.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record()
        torch.cuda.synchronize()
    print(f"graph step {e0.elapsed_time(e1)*1e3:.2f} us (events)")
else:
    for _ in range(3):
        prof.zero_()
        one()
        torch.cuda.synchronize()
p = prof.view(_lib.TXB_MAX_CTAS, 32).cpu().numpy().astype(np.float64)
rk._bufs.prof = 0
act = p[:, 0] > 0
t0 = p[act, 0].min()
for k, nm in list(enumerate(names)) + [(14, "pre-encoded")]:
    col = p[:, k]
    col = col[col > 0] - t0
    if col.size:
        print(f"{nm:12s} min {col.min()/1e3:8.2f}us  med {np.median(col)/1e3:8.2f}us  max {col.max()/1e3:8.2f}us  n={col.size}")

for k in (3, 4, 5, 6, 7, 8):
    col = p[:, k] - t0
    idx = np.argsort(-col)[:4]
    print(names[k], "slowest CTAs", [(int(i), round(col[i] / 1e3, 2)) for i in idx])
