import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2510_27656_b200 import weights
n = 7168 * 2048 * 3
words = (torch.randn(n, device="cuda:0") * 0.02).to(torch.bfloat16).view(torch.int16)
out = torch.empty(n + 4, dtype=torch.uint8, device="cuda:0")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda:0")
for mode in ("plain", "sleep"):
    ts = []
    for k in range(23):
        flush.fill_(k & 0xFF)
        if mode == "sleep":
            torch.cuda._sleep(200000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); weights.prepare_device(words, "fp8", out=out); e1.record()
        torch.cuda.synchronize()
        if k >= 3: ts.append(e0.elapsed_time(e1) * 1e3)
    print(mode, np.median(ts))
t0 = time.perf_counter()
for _ in range(100): weights.prepare_device(words, "fp8", out=out)
t1 = time.perf_counter(); torch.cuda.synchronize()
print("host us per call", (t1 - t0) / 100 * 1e6)
