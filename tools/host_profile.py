"""Host-side (Python) profile of a few Radau IIA steps: python tools/host_profile.py C3"""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from tools.bench_steps import CONFIGS
from paper_2209_06700_b200.fem import build_hierarchy
from paper_2209_06700_b200.irk import StageSystem
from paper_2209_06700_b200.multigrid import VCycleConfig
c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
h = build_hierarchy(c["dim"], c["L"], c["k"])
s = StageSystem(h, c["Q"], c["tau"], config=VCycleConfig(smoother_degree=c["deg"]), rel_tol=c["rtol"])
u = s.initial_condition()
u, _ = s.step(0.0, u)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for i in range(3):
    u, rep = s.step(c["tau"] * (i + 1), u)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
