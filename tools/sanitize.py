"""Small dispatch/combine scenarios for compute-sanitizer (racecheck,
synccheck, memcheck).  Each scenario runs a few steps through the public
API and checks the result against the CPU oracle, so a sanitizer run also
proves the kernels it watched produced the right bytes.

    compute-sanitizer --tool racecheck python tools/sanitize.py decode1
    compute-sanitizer --tool memcheck  python tools/sanitize.py gated2

Scenarios:
  decode1   EP=1, DeepSeek-V3 decode shape (fp8 from bf16 values, bf16 combine)
  prefill1  EP=1, large batch (generic fused path), bf16 rows
  gated2    EP=2 with both ranks on cuda:0 (host-gated split kernels)
  ep2       EP=2 over two GPUs (fused cooperative kernels, one thread per rank)
"""

from __future__ import annotations

import sys
import threading
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import moe_oracle as mo  # noqa: E402  (checker only)
from paper_2510_27656_b200 import moe  # noqa: E402
from paper_2510_27656_b200.engine import local_engines  # noqa: E402


def run(name: str, steps: int = 2) -> None:
    if name == "decode1":
        ranks, devs, T, E, H, elem, sc, priv = 1, [0], 128, 256, 7168, 1, 56, None
    elif name == "prefill1":
        ranks, devs, T, E, H, elem, sc, priv = 1, [0], 1024, 256, 2048, 2, 0, None
    elif name == "gated2":
        ranks, devs, T, E, H, elem, sc, priv = 2, [0, 0], 64, 64, 1024, 1, 8, 16
    elif name == "ep2":
        ranks, devs, T, E, H, elem, sc, priv = 2, [0, 1], 128, 256, 7168, 1, 56, 32
    else:
        raise SystemExit(f"unknown scenario {name}")
    spec = moe.RoutingSpec(ranks=ranks, experts=E, max_tokens=T, topk=8, hidden=H, elem_size=elem,
                           scales=sc, comb_elem_size=2, comb_scales=0)
    os_ = mo.Spec(ranks, E, T, 8, hidden=H, elem_size=elem, scales=sc)
    cs = mo.Spec(ranks, E, T, 8, hidden=H, elem_size=2, scales=0)
    pv = None if priv is None else moe.PrivateBufferConfig(priv)
    mesh = moe.build_mesh(local_engines(devs), spec, private=pv, timeout=120.0)
    try:
        for step in range(steps):
            rng = np.random.default_rng(31 + step)
            routes, values, weights = mo.random_step(os_, rng, tokens=T)
            xb = [torch.from_numpy(v).to(torch.bfloat16) for v in values]
            ref = mo.dispatch(os_, routes, [mo.encode_tokens(os_, x.float().numpy()) for x in xb])
            outs = [None] * ranks
            errs: list = []

            def worker(r: int) -> None:
                try:
                    rk = mesh[r]
                    torch.cuda.set_device(rk.device)
                    dev = torch.device("cuda", rk.device)
                    rk.dispatch_send(xb[r].to(dev), torch.from_numpy(routes[r]).to(dev))
                    g = rk.dispatch_recv(120.0)
                    want = ref.ranks[r].grouped
                    assert np.array_equal(g.data.cpu().numpy(), want.data), f"rank {r} grouped data"
                    assert np.array_equal(g.rows.cpu().numpy(), want.rows), f"rank {r} rows"
                    y = torch.from_numpy(mo.bf16_decode(mo.bf16_encode(
                        mo.decode_tokens(os_, want.data)))).to(dev).to(torch.bfloat16)
                    rk.combine_send(y)
                    outs[r] = rk.combine_recv(torch.from_numpy(weights[r]).to(dev), 120.0,
                                              out_dtype=torch.bfloat16).view(torch.int16).cpu().numpy()
                except Exception as exc:  # noqa: BLE001
                    errs.append(exc)

            th = [threading.Thread(target=worker, args=(r,)) for r in range(ranks)]
            for t in th:
                t.start()
            for t in th:
                t.join()
            if errs:
                raise errs[0]
            ys = [mo.bf16_decode(mo.bf16_encode(mo.decode_tokens(os_, ref.ranks[d].grouped.data)))
                  for d in range(ranks)]
            outs_b = [mo.bf16_encode(y).view(np.uint8).reshape(y.shape[0], -1) for y in ys]
            want = mo.combine(os_, ref, outs_b, weights, comb_spec=cs)
            for r in range(ranks):
                assert np.array_equal(outs[r].view(np.uint16), mo.bf16_encode(want[r])), f"rank {r} combine"
    finally:
        for m in mesh:
            m.close()
    print(f"sanitize scenario {name}: {steps} steps bit-exact vs oracle")


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["decode1"]:
        run(nm)
