"""HBM write-only vs copy bandwidth on this B200 (event-timed, best of 10):
the roofline a write-dominated kernel (the prefill dispatch writes 8 rows
per row read) can reach."""
import torch
n = 1 << 30
a = torch.empty(n, dtype=torch.uint8, device="cuda")
b = torch.empty(n, dtype=torch.uint8, device="cuda")
def best(fn, nbytes):
    ts = []
    for _ in range(12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return nbytes / (min(ts[2:]) * 1e-3) / 1e9
print(f"write-only (fill_) {best(lambda: a.fill_(7), n):8.1f} GB/s")
print(f"copy (read+write)  {best(lambda: b.copy_(a), 2 * n):8.1f} GB/s")
print(f"read-only (sum)    {best(lambda: a.view(torch.int32).sum(), n):8.1f} GB/s")
