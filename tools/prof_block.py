"""Run block-mode K1 launches of one config a few times (for ncu captures):
K=2 L=7 Q=4 EPI=store|resid python tools/prof_block.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_06700_b200.fem import build_hierarchy
from paper_2209_06700_b200 import measure

k = int(os.environ.get("K", 2)); L = int(os.environ.get("L", 7)); Q = int(os.environ.get("Q", 4))
h = build_hierarchy(3, L, k)
n = h.levels[L].n_dofs
u = torch.rand((Q, n), dtype=torch.float64, device="cuda")
v = torch.empty_like(u)
lams = [1.5, 2.5, 3.5, 4.5][:Q]
f = lambda: h.apply_block(L, lams, 1e-3, u, out=v)
for _ in range(3):
    f()
torch.cuda.synchronize()
ms = sorted(measure.event_time(f) for _ in range(5))[2]
print(f"block STORE k={k} L={L} Q={Q}: {ms*1e3:.1f} us  {16*Q*n/ms/1e6:.1f} GB/s")
