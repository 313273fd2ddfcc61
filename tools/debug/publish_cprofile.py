import sys, cProfile, pstats
sys.path.insert(0, '.')
import torch
from paper_2510_27656_b200 import weights
from paper_2510_27656_b200.engine import NvlinkFabric, TransferEngine
from paper_2510_27656_b200.memory import enable_peer_access
enable_peer_access([0, 1])
fab = NvlinkFabric()
src, dst = TransferEngine(fab, device=0, name="t"), TransferEngine(fab, device=1, name="i")
n = 1 << 20
out = torch.zeros(n, dtype=torch.uint8, device="cuda:0")
landing = dst.alloc_buffer(n + 64)
_, desc = dst.reg_mr(landing)
h = src.reg_mr(out)[0]
for _ in range(20):
    weights.publish(src, out, [(desc, 0)], imm=5, handle=h, wait=False)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(300):
    weights.publish(src, out, [(desc, 0)], imm=5, handle=h, wait=False)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
