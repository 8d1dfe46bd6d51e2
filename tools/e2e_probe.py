"""Probe the host-buffer pipeline: PCIe H2D/D2H bandwidth and HostStageOperator chunk counts."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2209_06700_b200.fem import build_hierarchy
from paper_2209_06700_b200.pipeline import HostStageOperator
from paper_2209_06700_b200.tableau import radau_iia
from paper_2209_06700_b200 import measure
h = build_hierarchy(3, 6, 4); L = 6; Q = 3
n = h.levels[L].n_dofs
uh = torch.rand((Q, n), dtype=torch.float64).pin_memory(); vh = torch.empty_like(uh).pin_memory()
ud = uh.cuda(); torch.cuda.synchronize()
ms = measure.event_time(lambda: ud.copy_(uh, non_blocking=True)); print(f"H2D {uh.numel()*8/ms/1e6:.1f} GB/s")
ms = measure.event_time(lambda: vh.copy_(ud, non_blocking=True)); print(f"D2H {uh.numel()*8/ms/1e6:.1f} GB/s")
s2 = torch.cuda.Stream()
def both():
    with torch.cuda.stream(s2):
        vh.copy_(ud, non_blocking=True)
    ud.copy_(uh, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)
ms = measure.event_time(both); print(f"H2D+D2H concurrent {ms:.2f} ms")
DM, DK = np.eye(Q), 1e-3 * radau_iia(Q).A
for ch in (4, 8, 16, 32):
    op = HostStageOperator(h, L, DM, DK, chunks=ch)
    op.apply(uh, vh); torch.cuda.synchronize()
    t = sorted(measure.event_time(lambda: op.apply(uh, vh)) for _ in range(5))[2]
    print(f"chunks={ch}: {t:.2f} ms/apply")
# steady state: back-to-back applies (double-buffered device sets overlap call i's D2H with i+1's H2D)
for ch in (4, 8, 16):
    op = HostStageOperator(h, L, DM, DK, chunks=ch)
    for _ in range(2):
        op.apply(uh, vh)
    torch.cuda.synchronize()
    def loop():
        for _ in range(10):
            op.apply(uh, vh)
    t = measure.event_time(loop) / 10
    print(f"steady chunks={ch}: {t:.2f} ms/apply")
