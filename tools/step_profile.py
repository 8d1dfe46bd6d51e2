"""One timed step of a config (for an ncu launch list): python tools/step_profile.py C4"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from tools.bench_steps import CONFIGS
from paper_2209_06700_b200.fem import build_hierarchy
from paper_2209_06700_b200.irk import StageSystem
from paper_2209_06700_b200.complex_solver import DirectComplexSystem
from paper_2209_06700_b200.multigrid import VCycleConfig
c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
h = build_hierarchy(c["dim"], c["L"], c["k"])
cfg = VCycleConfig(smoother_degree=c["deg"])
s = StageSystem(h, c["Q"], c["tau"], config=cfg, rel_tol=c["rtol"]) if c["path"] == "real" else \
    DirectComplexSystem(h, c["Q"], c["tau"], variant=c["path"], config=cfg, rel_tol=c["rtol"])
u = s.initial_condition()
u, _ = s.step(0.0, u)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
u, rep = s.step(c["tau"], u)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("iterations", rep.iterations)
