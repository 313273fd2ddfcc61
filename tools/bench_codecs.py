"""Kernel-registry codecs on the GPU (kernels.implementations()["cuda"],
kernels.py:245-264) at the DeepSeek-V3 decode/prefill sizes: device time per
call (CUDA events, L2 flushed) and HBM GB/s of the algorithmic bytes.

python tools/bench_codecs.py
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

from paper_2510_27656_b200 import kernels

dev = torch.device("cuda", 0)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)


def timed(fn, reps=20):
    ts = []
    for k in range(reps + 3):
        flush.fill_(k & 0xFF)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if k >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


res = {}
for T in (128, 4096):
    H, R = 7168, 8
    x = torch.randn(T * R, H, device=dev)
    b = kernels.fp8_encode(x)
    res[f"fp8_encode_{T*R}x{H}"] = (timed(lambda: kernels.fp8_encode(x)), x.numel() * 5)
    res[f"fp8_decode_{T*R}x{H}"] = (timed(lambda: kernels.fp8_decode(b)), x.numel() * 5)
    res[f"bf16_encode_{T*R}x{H}"] = (timed(lambda: kernels.bf16_encode(x)), x.numel() * 6)
    rows = torch.randint(0, T * R, (T * R,), device=dev)
    src = torch.randint(0, 255, (T * R, H), dtype=torch.uint8, device=dev)
    res[f"pack_rows_{T*R}x{H}B"] = (timed(lambda: kernels.pack_rows(src, rows)), 2 * T * R * H)
    pos = torch.arange(T * R, device=dev).reshape(T, R)
    w = torch.rand(T, R, device=dev)
    res[f"weighted_combine_{T}x{R}x{H}"] = (timed(lambda: kernels.weighted_combine(x, pos, w)),
                                           T * R * H * 4 + T * H * 4)
out = {k: {"us": round(t, 2), "gbs": round(by / (t * 1e-6) / 1e9, 1)} for k, (t, by) in res.items()}
print(json.dumps(out))
