"""Time dense_combine (spk_combine) on (Q, n) stage vectors: Q=4 N=16974593 python tools/prof_combine.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2209_06700_b200 import measure
from paper_2209_06700_b200.tensor_ops import dense_combine
Q = int(os.environ.get("Q", 4)); n = int(os.environ.get("N", 16974593))
u = torch.rand((Q, n), dtype=torch.float64, device="cuda")
out = torch.empty_like(u)
D = np.random.default_rng(1).standard_normal((Q, Q))
for acc in (False, True):
    f = lambda: dense_combine(D, u, out=out, accumulate=acc)
    for _ in range(3):
        f()
    ms = sorted(measure.event_time(f) for _ in range(7))[3]
    B = 8 * Q * n * (3 if acc else 2)
    print(f"Q={Q} accumulate={acc}: {ms*1e3:8.1f} us  {B/ms/1e6:8.1f} GB/s")
