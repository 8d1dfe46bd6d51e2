"""Debug: where does the constrained stage operator differ from the oracle (small 3D level)?"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_06700_b200.fem import build_hierarchy
from paper_2209_06700_b200.tableau import radau_iia
from oracle import fem_qk

k = int(os.environ.get("K", 4)); L = int(os.environ.get("L", 3)); Q = int(os.environ.get("Q", 3))
h = build_hierarchy(3, L, k)
n = h.levels[L].n_dofs
nax = round(n ** (1 / 3))
rng = np.random.default_rng(0)
u = rng.uniform(-1, 1, (Q, n))
DM, DK = np.eye(Q), 1e-3 * radau_iia(Q).A
for constrained in (False, True):
    v = h.apply_stage_operator(L, DM, DK, torch.tensor(u, device="cuda"), constrained=constrained).cpu().numpy()
    ho = fem_qk.Hierarchy(3, L, k)
    ref = np.zeros_like(u)
    for i in range(Q):
        for j in range(Q):
            w = u[j]
            Mu = ho.apply_constrained_mass(L, w) if hasattr(ho, "apply_constrained_mass") else None
    # reference through the package's own generic path is not available: use the oracle operators
    M = lambda w: ho.apply_mass(L, w)
    Kf = lambda w: ho.apply_stiffness(L, w)
    mask = ho.levels[L].interior_mask.reshape(-1) if hasattr(ho.levels[L], "interior_mask") else None
    if constrained:
        if mask is None:
            g = np.ones((nax, nax, nax), bool); g[0] = g[-1] = False; g[:, 0] = g[:, -1] = False; g[:, :, 0] = g[:, :, -1] = False
            mask = g.reshape(-1)
        um = u * mask
    else:
        um = u
    for i in range(Q):
        acc = np.zeros(n)
        for j in range(Q):
            acc += DM[i, j] * M(um[j]) + DK[i, j] * Kf(um[j])
        ref[i] = np.where(mask, acc, u[i]) if constrained else acc
    d = np.abs(v - ref).reshape(Q, nax, nax, nax)
    print("constrained", constrained, "max abs diff", d.max(), "ref max", np.abs(ref).max())
    bad = np.argwhere(d > 1e-12 * np.abs(ref).max())
    print(" mismatches", len(bad))
    if len(bad):
        for ax, nm in ((1, "x"), (2, "y"), (3, "z")):
            print("  ", nm, sorted(set(bad[:, ax].tolist()))[:40])
        print("  first", bad[:10].tolist())
