"""Parity at the BASELINE.json sizes through size-independent properties (the oracle's dense 1D
contractions do not finish in seconds at 257^3 nodes):

* C2 (64^3 Q4, Q = 3): separable stage inputs u_q = f_q (x) g_q (x) h_q make the exact operator a sum
  of outer products of 1D matvecs with the oracle's assembled 1D matrices -> full-size reference;
* C4 (128^3 Q2, Q = 4 blocks): the V-cycle is linear and symmetric in the energy-free sense the
  reference tests (test_multigrid.py:143-163): V(a a + b b) = a V(a) + b V(b), <V a, b> = <a, V b>.
"""

import numpy as np
import pytest
import torch

from oracle.fem_qk import Level
from oracle.tableau_ref import radau_iia
from paper_2209_06700_b200.fem import build_hierarchy

pytestmark = pytest.mark.gpu


def _outer3(a, b, c):
    return (a[:, None, None] * b[None, :, None] * c[None, None, :]).reshape(-1)


@pytest.mark.parametrize("cfg,constrained", [("C2", False), ("C2", True), ("C4", True), ("C5", True)])
def test_full_size_separable_stage_operator(cuda, cfg, constrained):
    """C2: I (x) M + tau A (x) K (the microbench); C4 / C5: the GMRES operator A^-1 (x) M + tau I (x) K."""
    k, L, Q, tau = {"C2": (4, 6, 3, 1e-3), "C4": (2, 7, 4, 1e-3), "C5": (3, 6, 3, 5e-3)}[cfg]
    lvl = Level(L, 3, k)
    x = lvl.coords
    M1, K1 = lvl.mass_1d, lvl.stiffness_1d
    inter = np.ones_like(x, dtype=bool)
    inter[0] = inter[-1] = False
    fs = [(np.sin(np.pi * (q + 1) * x), np.cos(2 * q * x) + x ** 2, np.exp(-x) * (1 + q * x)) for q in range(Q)]
    if constrained:  # the constrained operator sees where(mask, u, 0): zero the 1D boundary values
        fs = [tuple(np.where(inter, f, 0.0) for f in t) for t in fs]
    tab = radau_iia(Q)
    if cfg == "C2":
        DM, DK = np.eye(Q), tau * np.asarray(tab["A"])
    else:
        DM, DK = np.asarray(tab["Ainv"]), tau * np.eye(Q)
    u = np.stack([_outer3(*t) for t in fs])
    Mu = [(M1 @ f, M1 @ g, M1 @ h) for f, g, h in fs]
    Ku = [(K1 @ f, K1 @ g, K1 @ h) for f, g, h in fs]
    ref = np.zeros_like(u)
    for i in range(Q):
        for j in range(Q):
            (mf, mg, mh), (kf, kg, kh) = Mu[j], Ku[j]
            ref[i] += DM[i, j] * _outer3(mf, mg, mh)
            ref[i] += DK[i, j] * (_outer3(kf, mg, mh) + _outer3(mf, kg, mh) + _outer3(mf, mg, kh))
    if constrained:  # boundary rows are the identity on the (zero) boundary values
        ref[:, ~lvl.interior_mask] = u[:, ~lvl.interior_mask]
    h = build_hierarchy(3, L, k)
    v = h.apply_stage_operator(L, DM, DK, torch.from_numpy(u).cuda(), constrained=constrained).cpu().numpy()
    err = np.abs(v - ref).max() / np.abs(ref).max()
    assert err < 1e-12, err


def test_c4_full_size_vcycle_linear_and_symmetric(cuda):
    from paper_2209_06700_b200.multigrid import MultiBlockSolver, VCycleConfig

    k, L = 2, 7
    h = build_hierarchy(3, L, k)
    lams = [5.644108, 2.941868, 3.161847, 16.0]  # radau_iia(4) L~ diagonal
    sv = MultiBlockSolver(h, lams, 1e-3, VCycleConfig(smoother_degree=3))
    mask = h.mask_tensor(L)
    g = torch.Generator(device="cuda").manual_seed(4)
    a = torch.where(mask, torch.randn((4, h.n), generator=g, device="cuda", dtype=torch.float64), 0.0)
    b = torch.where(mask, torch.randn((4, h.n), generator=g, device="cuda", dtype=torch.float64), 0.0)
    Va, Vb = sv.apply_device(a), sv.apply_device(b)
    Vab = sv.apply_device(2.0 * a - 3.0 * b)
    lin = (Vab - (2.0 * Va - 3.0 * Vb)).abs().max() / Vab.abs().max()
    assert float(lin) < 1e-12, float(lin)
    for q in range(4):
        s1 = float(torch.dot(Va[q], b[q]))
        s2 = float(torch.dot(a[q], Vb[q]))
        assert abs(s1 - s2) <= 1e-10 * max(abs(s1), abs(s2)), (q, s1, s2)
