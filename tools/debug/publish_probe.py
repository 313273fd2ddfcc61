"""Host-side cost of one weights.publish round (arm, launch, wait), to see
where the end-to-end publish time goes beyond the copy kernel."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np, torch
from paper_2510_27656_b200 import weights
from paper_2510_27656_b200.engine import NvlinkFabric, TransferEngine
from paper_2510_27656_b200.memory import enable_peer_access
enable_peer_access([0, 1])
fab = NvlinkFabric()
src, dst = TransferEngine(fab, device=0, name="t"), TransferEngine(fab, device=1, name="i")
n = 7168 * 2048 * 3
out = torch.zeros(n + 4, dtype=torch.uint8, device="cuda:0")
landing = dst.alloc_buffer(n + 4 + 64)
_, desc = dst.reg_mr(landing)
h = src.reg_mr(out)[0]
imm = 77
rows = []
for k in range(30):
    torch.cuda.synchronize(0); torch.cuda.synchronize(1)
    t0 = time.perf_counter()
    f = dst.expect_imm_count(imm, 1)
    t1 = time.perf_counter()
    flag = weights.publish(src, out, [(desc, 0)], imm=imm, handle=h, wait=False)
    t2 = time.perf_counter()
    checks = 0
    while not f.done():
        checks += 1
    t3 = time.perf_counter()
    c0 = time.perf_counter(); f.done(); dst.imm_received_total(imm); c1 = time.perf_counter()
    if k >= 5:
        rows.append(((t1 - t0) * 1e6, (t2 - t1) * 1e6, (t3 - t2) * 1e6, checks, (c1 - c0) * 1e6))
r = np.median(np.asarray(rows), axis=0)
print(f"arm {r[0]:.1f} us, publish launch {r[1]:.1f} us, wait {r[2]:.1f} us ({r[3]:.0f} checks), one check {r[4]:.1f} us")
