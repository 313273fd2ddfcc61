"""NVLink bytes of the MoE data movement, measured by ncu on two GPUs.

The fused cooperative kernels spin on their peers, so they cannot be
replayed by ncu inside a multi-rank job.  This driver runs the same EP=2
step (bench.py's DSv3 decode or prefill workload, bf16 values in, fp8 or
bf16 rows, bf16 combine) in ONE process over cuda:0 and cuda:1 with the mesh
forced host-gated: the split kernels, each waiting kernel launched only once
its condition holds, so ncu may serialise and replay them.  k_dispatch
(token stores + release-add) and k_comb_send (row returns + release-add)
move exactly the bytes the fused kernels move; ncu's nvltx/nvlrx counters
on them give the link-level bytes per launch (user data vs protocol).

ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,... \
    -k regex:"k_(dispatch|comb_send)<" python tools/prof_nvlink.py [--config decode]
"""
import argparse
import json
import sys
import threading
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

import bench
from paper_2510_27656_b200 import moe
from paper_2510_27656_b200.engine import local_engines

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="decode", choices=sorted(bench.WORKLOADS))
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()

wl = bench.WORKLOADS[a.config]
N = 2
spec = moe.RoutingSpec(ranks=N, experts=wl["experts"], max_tokens=wl["tokens"], topk=wl["topk"],
                       hidden=wl["hidden"], elem_size=wl["elem"], scales=wl["scales"], comb_elem_size=2,
                       comb_scales=0)
mesh = moe.build_mesh(local_engines([0, 1]), spec, timeout=120.0)
for m in mesh:
    m.host_gated = True          # split kernels, host-gated launches (replay-safe)
inputs = []
for r in range(N):
    dev = torch.device("cuda", r)
    x, routes, w = bench._inputs(wl, r, wl["tokens"])
    G = int(mesh[r]._shape.grouped_rows)
    inputs.append((torch.from_numpy(x).to(dev).to(torch.bfloat16), torch.from_numpy(routes).to(dev),
                   torch.from_numpy(w).to(dev), torch.randn(G, wl["hidden"], device=dev).to(torch.bfloat16)))
expect = [bench.expected_rows(wl, r, N, wl["tokens"]) for r in range(N)]


def worker(r: int, errs: list) -> None:
    try:
        torch.cuda.set_device(r)
        xd, rd, wd, y = inputs[r]
        for _ in range(a.steps):
            mesh[r].dispatch_send(xd, rd)
            g = mesh[r].dispatch_recv()
            mesh[r].combine_send(y[:g.data.shape[0]])
            mesh[r].combine_recv(wd, out_dtype=torch.bfloat16)
        torch.cuda.synchronize(r)
    except Exception as exc:  # reported below
        errs.append(exc)


errs: list = []
th = [threading.Thread(target=worker, args=(r, errs)) for r in range(N)]
for t in th:
    t.start()
for t in th:
    t.join()
print(json.dumps({"config": a.config, "ep": N, "steps": a.steps, "errors": [repr(e) for e in errs],
                  "algorithmic": expect}))
for m in mesh:
    m.close()
