"""GPU busy vs idle time inside one Radau IIA step (torch.profiler / CUPTI kernel timeline):
python tools/gpu_idle.py C3"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
from tools.bench_steps import CONFIGS
from paper_2209_06700_b200.fem import build_hierarchy
from paper_2209_06700_b200.irk import StageSystem
from paper_2209_06700_b200.complex_solver import DirectComplexSystem
from paper_2209_06700_b200.multigrid import VCycleConfig
c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
h = build_hierarchy(c["dim"], c["L"], c["k"])
cfg = VCycleConfig(smoother_degree=c["deg"])
s = StageSystem(h, c["Q"], c["tau"], config=cfg, rel_tol=c["rtol"]) if c["path"] == "real" else \
    DirectComplexSystem(h, c["Q"], c["tau"], variant=c["path"], config=cfg, rel_tol=c["rtol"])
u = s.initial_condition()
u, _ = s.step(0.0, u)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    u, rep = s.step(c["tau"], u)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
iv = sorted((e.time_range.start, e.time_range.end) for e in ev)
busy, cur_s, cur_e = 0.0, None, None
for a, b in iv:
    if cur_e is None or a > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = a, b
    else:
        cur_e = max(cur_e, b)
busy += cur_e - cur_s
span = iv[-1][1] - iv[0][0]
print(f"{sys.argv[1] if len(sys.argv) > 1 else 'C3'}: {len(iv)} GPU activities, span {span/1e3:.2f} ms, "
      f"busy {busy/1e3:.2f} ms ({100*busy/span:.0f} %), iterations {rep.iterations}")
