"""CUDA runtime calls that block the host inside one step (torch.profiler CPU + CUDA activities):
python tools/sync_count.py C3"""
import collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
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
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    u, rep = s.step(c["tau"], u)
    torch.cuda.synchronize()
agg = collections.Counter()
dur = collections.Counter()
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CPU and e.name.startswith("cuda"):
        agg[e.name] += 1
        dur[e.name] += e.cpu_time_total
for k, v in agg.most_common(20):
    print(f"{k:40s} {v:5d} calls  {dur[k]/1e3:8.2f} ms")
