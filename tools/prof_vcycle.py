"""Per-kernel timings of the V-cycle building blocks at the finest level of a config (CUDA events):
block STORE apply, residual(+d), Chebyshev step, cheb_init, restriction, prolongation, one full
MultiBlockSolver V-cycle.   K=2 L=7 NB=4 DEG=2 python tools/prof_vcycle.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2209_06700_b200 import _lib, measure
from paper_2209_06700_b200._device import ptr, stream_ptr
from paper_2209_06700_b200.fem import build_hierarchy
from paper_2209_06700_b200.multigrid import MultiBlockSolver, VCycleConfig

k = int(os.environ.get("K", 2)); L = int(os.environ.get("L", 7)); nb = int(os.environ.get("NB", 4))
deg = int(os.environ.get("DEG", 3))
h = build_hierarchy(3, L, k)
if "TARGET" in os.environ:  # K1 x-chunking target (CTAs per launch; 0 = automatic)
    _lib.load().spk_set_chunks(h.ctx, int(os.environ["TARGET"]))
if "SPLIT" in os.environ:  # Chebyshev split threshold (block-DoFs); 0 = always split
    _lib.call("spk_set_cheb_split", h.ctx, int(os.environ["SPLIT"]))
n = h.levels[L].n_dofs
lams = [5.6, 2.9, 3.2, 16.0][:nb]
tau = 1e-3
st = stream_ptr(h.device)
mk = lambda: torch.rand((nb, n), dtype=torch.float64, device="cuda")
x, b, r, d, d2 = mk(), mk(), mk(), mk(), mk()
la = _lib.dbl_array(lams)
c1 = _lib.dbl_array([0.5] * nb); c2 = _lib.dbl_array([0.1] * nb)
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
def t(f, bytes_per):
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    ms = sorted(measure.event_time(f) for _ in range(5))[2]
    return ms, bytes_per * nb * n / ms / 1e6
res = {}
res["block STORE"] = t(lambda: h.apply_block(L, lams, tau, x, constrained=True, out=d2), 16)
res["residual+d"] = t(lambda: _lib.call("spk_residual", h.ctx, L, nb, la, tau, ptr(x), ptr(b), ptr(r), ptr(d), c1, st), 40)
res["residual"] = t(lambda: _lib.call("spk_residual", h.ctx, L, nb, la, tau, ptr(x), ptr(b), ptr(r), None, None, st), 24)
res["cheb step"] = t(lambda: _lib.call("spk_cheb_step", h.ctx, L, nb, la, tau, c1, c2, ptr(d), ptr(r), ptr(x), ptr(d2), 0, ptr(flag), st), 48)
res["cheb final"] = t(lambda: _lib.call("spk_cheb_step", h.ctx, L, nb, la, tau, c1, c2, ptr(d), ptr(r), ptr(x), ptr(d2), 1, ptr(flag), st), 32)
res["cheb_init"] = t(lambda: _lib.call("spk_cheb_init", h.ctx, L, nb, la, tau, c1, ptr(b), ptr(r), ptr(x), ptr(d), st), 32)
rc = torch.zeros((nb, h.levels[L - 1].n_dofs), dtype=torch.float64, device="cuda")
res["restrict"] = t(lambda: h.restrict_into(L, r, rc, mask=True), 8 * (1 + 1 / 8))
res["prolong+acc"] = t(lambda: h.prolong_into(L - 1, rc, x, accumulate=True), 8 * (2 + 1 / 8))
sv = MultiBlockSolver(h, lams, tau, VCycleConfig(smoother_degree=deg))
res["V-cycle"] = t(lambda: sv.apply_device(b, check=False), 0)
for kname, (ms, gbs) in res.items():
    print(f"{kname:12s} {ms*1e3:9.1f} us  {gbs:8.1f} GB/s (algorithmic)")
