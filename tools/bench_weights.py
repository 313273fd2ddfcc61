"""RL weight-update path on B200 (BASELINE §8(f) row 2): per-tensor fp8
narrowing of bf16 weights on the GPU (`weights.prepare_device`: amax pass +
quantise pass + f32 footer, weights.py:370-387) and the WriteImm of the
prepared bytes to a peer GPU (`weights.publish`, one single write per
destination, weights.py:570-590).

Shape: one DeepSeek-V3 routed expert's three matrices (7168 x 2048 x 3 bf16,
88 MB), prepared, then published to cuda:1 (NVLink) when present, else to
cuda:0 (HBM loopback).  Device time with CUDA events after an L2 flush.
Prints one JSON line.

python tools/bench_weights.py [--reps 20]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

from paper_2510_27656_b200 import weights
from paper_2510_27656_b200.engine import NvlinkFabric, TransferEngine
from paper_2510_27656_b200.memory import enable_peer_access

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--elems", type=int, default=7168 * 2048 * 3)
a = ap.parse_args()

ngpu = torch.cuda.device_count()
d1 = 1 if ngpu > 1 else 0
if d1:
    enable_peer_access([0, 1])
fab = NvlinkFabric()
src, dst = TransferEngine(fab, device=0, name="trainer"), TransferEngine(fab, device=d1, name="inference")
n = a.elems
words = (torch.randn(n, device="cuda:0") * 0.02).to(torch.bfloat16).view(torch.int16)
out = torch.empty(n + 4, dtype=torch.uint8, device="cuda:0")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda:0")
landing = dst.alloc_buffer(n + 4 + 64)
_, desc = dst.reg_mr(landing)


def timed(fn):
    ts = []
    for k in range(a.reps + 3):
        flush.fill_(k & 0xFF)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if k >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


prep_us = timed(lambda: weights.prepare_device(words, "fp8", out=out))
# algorithmic HBM bytes of the narrowing: amax pass reads 2n, quantise pass
# reads 2n and writes n + 4
prep_bytes = 2 * n + 2 * n + n + 4
imm = 4242
k_pub = [0]
# the prepared buffer is registered outside the timed write, as the
# reference's pipeline does (its prepare lane registers the payload,
# weights.py:563-565; the write lane only submits, weights.py:570-590)
h_out = src.reg_mr(out)[0]


def pub():
    # one imm re-armed every update (its ImmCounter slot is claimed once)
    k_pub[0] += 1
    f = dst.expect_imm_count(imm, 1)
    weights.publish(src, out, [(desc, 0)], imm=imm, handle=h_out)
    assert f.wait(10.0)


pub_us = timed(pub)
torch.cuda.synchronize()

# device time of the copy kernel itself: the publish enqueued without
# waiting, events on the engine stream around it
dev_ts = []
for k in range(a.reps + 3):
    flush.fill_(k & 0xFF)
    st = src.stream
    st.wait_stream(torch.cuda.current_stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    weights.publish(src, out, [(desc, 0)], imm=None, handle=h_out, wait=False)
    e1.record(st)
    torch.cuda.synchronize()
    if k >= 3:
        dev_ts.append(e0.elapsed_time(e1) * 1e3)
pub_dev_us = float(np.median(dev_ts))
ok = bool(torch.equal(landing[:n + 4].cpu(), out.cpu()))
res = {"metric": "RL weight update: fp8 prepare + publish (DSv3 expert, 88 MB bf16)",
       "elems": n, "prepare_us_p50": round(prep_us, 2),
       "prepare_hbm_gbs": round(prep_bytes / (prep_us * 1e-6) / 1e9, 1), "prepare_peak_gbs": 6555.2,
       "publish_bytes": n + 4, "publish_us_p50": round(pub_us, 2),
       "publish_gbs": round((n + 4) / (pub_us * 1e-6) / 1e9, 1),
       "publish_path": "NVLink cuda:0 -> cuda:1" if d1 else "HBM loopback cuda:0",
       "publish_peak_gbs": 770.0 if d1 else 6555.2,
       "publish_device_us_p50": round(pub_dev_us, 2),
       "publish_device_gbs": round((n + 4) / (pub_dev_us * 1e-6) / 1e9, 1),
       "note": "publish_us: end to end through the host calls (arm the receiver's ImmFlag, one k_copy_jobs "
               "launch, the ImmFlag wait on the host; the prepared buffer registered and the imm's counter slot "
               "claimed once); "
               "publish_device_us: the copy kernel on the engine stream (no host wait)",
       "landing_bit_exact": ok}
print(json.dumps(res))
