"""Small workload for compute-sanitizer (racecheck / synccheck / memcheck, one tool per run): the
fused coarse V-cycle (single CTA per block, shared-memory levels), the cooperative MGS column (grid
barriers), K1 coupled / block launches and the small-level gather kernel, one un-graphed Radau IIA
step. usage: compute-sanitizer --tool racecheck python tools/sanitize_small.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2209_06700_b200.fem import build_hierarchy  # noqa: E402
from paper_2209_06700_b200.irk import StageSystem  # noqa: E402
from paper_2209_06700_b200.multigrid import MultiBlockSolver, VCycleConfig  # noqa: E402

h = build_hierarchy(3, 3, 2)
cfg = VCycleConfig(smoother_degree=3)
mb = MultiBlockSolver(h, [3.2, 2.1, 9.0], 0.01, cfg)
b = torch.rand((3, h.levels[3].n_dofs), dtype=torch.float64, device="cuda")
x = mb.apply_device(b)
ss = StageSystem(h, 3, 0.01, config=cfg)
ss.use_graphs = False
ss.speculate = False
u = ss.initial_condition()
u, rep = ss.step(0.0, u)
h4 = build_hierarchy(3, 2, 4)
n4 = h4.levels[2].n_dofs
v = h4.apply_stage_operator(2, np.eye(3), 1e-3 * np.ones((3, 3)), torch.rand((3, n4), dtype=torch.float64,
                                                                            device="cuda"))
torch.cuda.synchronize()
print("sanitize workload ok", rep.iterations, float(x.abs().max()), float(v.abs().max()))
