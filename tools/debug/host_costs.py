"""Per-call host cost of the torch stream/event plumbing around a launch."""
import time, torch
dev = 0
torch.cuda.set_device(dev)
s = torch.cuda.Stream(dev)
def t(name, fn, n=2000):
    for _ in range(50): fn()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    print(f"{name:36s} {(time.perf_counter() - t0) / n * 1e6:7.2f} us")
t("current_stream", lambda: torch.cuda.current_stream(dev))
cur = torch.cuda.current_stream(dev)
t("wait_stream", lambda: s.wait_stream(cur))
def ctx_dev():
    with torch.cuda.device(dev): pass
t("with torch.cuda.device", ctx_dev)
def ctx_st():
    with torch.cuda.stream(s): pass
t("with torch.cuda.stream", ctx_st)
def ev():
    e = torch.cuda.Event(); e.record(s)
t("Event() + record", ev)
e = torch.cuda.Event(); e.record(s)
t("Event.query", lambda: e.query())
import ctypes
lib = ctypes.CDLL(None)
t("python no-op", lambda: None)
