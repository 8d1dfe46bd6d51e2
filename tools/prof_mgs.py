"""Time one MGS sweep (spk_mgs) on N doubles: N=67898372 python tools/prof_mgs.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_06700_b200 import _lib, measure
from paper_2209_06700_b200._device import ptr, stream_ptr
from paper_2209_06700_b200.fem import build_hierarchy
n = int(os.environ.get("N", 67898372))
h = build_hierarchy(3, 2, 1)
w, vp, vc = (torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(3))
hh = torch.tensor([1e-3], dtype=torch.float64, device="cuda")
out = torch.zeros(1, dtype=torch.float64, device="cuda")
st = stream_ptr(w.device)
for name, a, b, B in [("w-=h vp; <vc,w>", vp, vc, 32), ("<vc,w>", None, vc, 16), ("||w||", None, None, 8)]:
    f = lambda: _lib.call("spk_mgs", h.ctx, n, ptr(w), ptr(a), ptr(hh), ptr(b), ptr(out), st)
    for _ in range(3):
        f()
    ms = sorted(measure.event_time(f) for _ in range(7))[3]
    print(f"{name:18s} {ms*1e3:8.1f} us  {B*n/ms/1e6:8.1f} GB/s")
