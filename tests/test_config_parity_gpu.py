"""Radau IIA steps at the BASELINE.json config sizes vs the CPU oracle (north_star: per-step
solution within relative 1e-9, GMRES iterations within +-1).

C3 runs all 20 of its steps at full size (32^3 Q2 cells), C4 one step at full size (128^3 Q2 cells,
17M DoFs per stage, Q=4), C5 three steps at full size (64^3 Q3 cells, 7.2M DoFs per stage). The
oracle uses its banded fast path (oracle/fastband.c) on the 129- and 257-node axes: the same
contractions as the dense reference form over their nonzero band only, checked against the dense
form in tests/test_oracle_fast.py; the dense form would need ~12 minutes of host time per C4 step.
C1 at full size is in test_solvers_gpu.py.
"""

import numpy as np
import pytest

from oracle import solvers as OS
from oracle import stepper as OST
from oracle.fem_qk import Hierarchy
from oracle.tableau_ref import radau_iia as ref_radau
from paper_2209_06700_b200.complex_solver import DirectComplexSystem
from paper_2209_06700_b200.fem import build_hierarchy
from paper_2209_06700_b200.irk import StageSystem
from paper_2209_06700_b200.multigrid import VCycleConfig

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _real_steps(L, k, Q, tau, deg, steps):
    tab = ref_radau(Q)
    dev = StageSystem(build_hierarchy(3, L, k), Q, tau, config=VCycleConfig(smoother_degree=deg), tableau=tab)
    ora = OST.RealLU(Hierarchy(3, L, k, fast=True), Q, tau, OS.Config(smoother_degree=deg), tab=tab)
    u, uo = dev.initial_condition(), ora.initial()
    for s in range(steps):
        u, rep = dev.step(s * tau, u)
        uo, its, _ = ora.step(s * tau, uo)
        err = rel(u.cpu().numpy(), uo)
        print(f"L={L} k={k} Q={Q} step {s}: GMRES its device {rep.iterations} oracle {its}, rel err {err:.2e}")
        assert abs(rep.iterations - its) <= 1, (s, rep.iterations, its)
        assert err < 1e-9, s
    return rep.iterations


def test_c3_full_size_steps():
    """C3: 32^3 Q2 hex, Radau IIA Q=3, tau=0.01, Chebyshev degree 3, rtol 1e-12 (all 20 steps)."""
    its = _real_steps(L=5, k=2, Q=3, tau=0.01, deg=3, steps=20)
    assert 10 <= its <= 13


def test_c5_full_size_presb_steps():
    """C5: 64^3 Q3 hex, Radau IIA Q=3 diagonalised (one complex pair with PRESB + one real block),
    tau=5e-3, degree 3, rtol 1e-12 (3 of its 10 steps)."""
    tab = ref_radau(3)
    L, k, tau = 6, 3, 5e-3
    cfg = VCycleConfig(smoother_degree=3)
    dev = DirectComplexSystem(build_hierarchy(3, L, k), 3, tau, variant="presb", config=cfg, tableau=tab)
    ora = OST.DirectComplex(Hierarchy(3, L, k, fast=True), 3, tau, variant="presb",
                            cfg=OS.Config(smoother_degree=3), tab=tab)
    u, uo = dev.initial_condition(), ora.initial()
    for s in range(3):
        u, rep = dev.step(s * tau, u)
        uo, its = ora.step(s * tau, uo)
        err = rel(u.cpu().numpy(), uo)
        print(f"C5 full step {s}: block its device {rep.block_iterations} oracle {its}, rel err {err:.2e}")
        assert all(abs(a - b) <= 1 for a, b in zip(rep.block_iterations, its)), (rep.block_iterations, its)
        assert err < 1e-9


def test_c2_full_size_seeded_operator():
    """C2 exactly as benchmarked: 64^3 Q4 hex, Q=3, D_M = I, D_K = 1e-3 A, u ~ U[-1,1] from
    default_rng(42), applied once on the device and once by the oracle (relative 1e-12)."""
    import torch

    from paper_2209_06700_b200.tableau import radau_iia

    L, k, Q = 6, 4, 3
    h = build_hierarchy(3, L, k)
    n = h.levels[L].n_dofs
    u = np.random.default_rng(42).uniform(-1.0, 1.0, size=(Q, n))
    DM, DK = np.eye(Q), 1e-3 * radau_iia(Q).A
    v = h.apply_stage_operator(L, DM, DK, torch.from_numpy(u).cuda()).cpu().numpy()
    import oracle.fem_qk as F
    F.FAST = False  # the reference's dense contraction form, as benchmarked on the CPU
    ref = Hierarchy(3, L, k).apply_stage(L, DM, DK, u)
    print(f"C2 full seeded operator: rel err {rel(v, ref):.2e}")
    assert rel(v, ref) < 1e-12


def test_c4_full_size_step():
    """C4: 128^3 Q2 hex, Radau IIA Q=4, tau=1e-3, degree 3, rtol 1e-12 (1 of its 5 steps)."""
    _real_steps(L=7, k=2, Q=4, tau=1e-3, deg=3, steps=1)
