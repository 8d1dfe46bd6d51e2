"""Run the C2 stage operator a few times (for ncu captures) and print per-variant timings."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2209_06700_b200.fem import build_hierarchy
from paper_2209_06700_b200.tableau import radau_iia
from paper_2209_06700_b200 import _lib, measure

k = int(os.environ.get("K", 4)); L = int(os.environ.get("L", 6)); Q = int(os.environ.get("Q", 3))
reps = int(os.environ.get("REPS", 3))
h = build_hierarchy(3, L, k)
n = h.levels[L].n_dofs
u = torch.rand((Q, n), dtype=torch.float64, device="cuda")
v = torch.empty_like(u)
DM, DK = np.eye(Q), 1e-3 * radau_iia(Q).A
for t in [int(x) for x in os.environ.get("TARGETS", "0").split(",")]:
    _lib.load().spk_set_chunks(h.ctx, t)
    for _ in range(reps):
        h.apply_stage_operator(L, DM, DK, u, out=v)
    torch.cuda.synchronize()
    ms = sorted(measure.event_time(lambda: h.apply_stage_operator(L, DM, DK, u, out=v)) for _ in range(5))[2]
    print(f"k={k} L={L} Q={Q} target_ctas={t}: {ms*1e3:.1f} us  {16*Q*n/ms/1e6:.1f} GB/s")
