"""K1 parity: device Q_k operators vs the CPU oracle (relative 1e-12, north_star tolerance)."""

import numpy as np
import pytest
import torch

from oracle.fem_qk import Hierarchy
from paper_2209_06700_b200.fem import build_hierarchy
from paper_2209_06700_b200.tableau import radau_iia

pytestmark = pytest.mark.gpu
TOL = 1e-12


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))


CASES = [(1, 1, 4), (2, 1, 3), (3, 1, 3), (1, 2, 3), (2, 2, 3), (3, 2, 3), (1, 3, 3), (2, 3, 2),
         (3, 3, 2), (1, 4, 3), (2, 4, 2), (3, 4, 2), (3, 1, 5), (3, 2, 4), (3, 4, 3)]


@pytest.mark.parametrize("dim,k,L", CASES)
def test_mass_stiffness_shifted_constrained(cuda, dim, k, L):
    h = build_hierarchy(dim, L, k)
    o = Hierarchy(dim, L, k)
    rng = np.random.default_rng(7 + dim + 10 * k)
    u = rng.standard_normal((3, h.n))
    assert rel(h.apply_mass(L, u), o.apply_mass(L, u)) < TOL
    assert rel(h.apply_stiffness(L, u), o.apply_stiffness(L, u)) < TOL
    lam = np.array([0.5, 2.0, 7.0])
    assert rel(h.apply_shifted(L, lam, 0.1, u), o.apply_shifted(L, lam, 0.1, u)) < TOL
    assert rel(h.apply_constrained(L, 1.3, 0.01, u[0]), o.apply_constrained(L, 1.3, 0.01, u[0])) < TOL
    assert rel(h.operator_diagonal(L, 2.0, 0.1), o.operator_diagonal(L, 2.0, 0.1)) < TOL


@pytest.mark.parametrize("dim,k,L", CASES)
def test_transfers(cuda, dim, k, L):
    h = build_hierarchy(dim, L, k)
    o = Hierarchy(dim, L, k)
    rng = np.random.default_rng(3)
    uc = rng.standard_normal((2, h.levels[L - 1].n_dofs))
    rf = rng.standard_normal((2, h.n))
    assert rel(h.prolong(L - 1, uc), o.prolong(L - 1, uc)) < TOL
    assert rel(h.restrict(L, rf), o.restrict(L, rf)) < TOL


@pytest.mark.parametrize("Q", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_stage_operator(cuda, Q, k):
    L = 3 if k <= 2 else 2
    h = build_hierarchy(3, L, k)
    o = Hierarchy(3, L, k)
    A = radau_iia(Q).A
    rng = np.random.default_rng(42)
    u = rng.uniform(-1, 1, (Q, h.n))
    for DM, DK, cons in [(np.eye(Q), 1e-3 * A, False), (np.linalg.inv(A), 0.05 * np.eye(Q), True)]:
        v = h.apply_stage_operator(L, DM, DK, u, constrained=cons)
        assert rel(v, o.apply_stage(L, DM, DK, u, constrained=cons)) < TOL


def test_stage_operator_2d(cuda):
    h = build_hierarchy(2, 4, 2)
    o = Hierarchy(2, 4, 2)
    A = radau_iia(2).A
    u = np.random.default_rng(1).uniform(-1, 1, (2, h.n))
    assert rel(h.apply_stage_operator(4, np.eye(2), 0.05 * A, u),
               o.apply_stage(4, np.eye(2), 0.05 * A, u)) < TOL


def _sep(vecs, dim):
    out = vecs[0]
    for v in vecs[1:dim]:
        out = np.multiply.outer(out, v)
    return out.ravel()


@pytest.mark.parametrize("k,L", [(4, 6), (2, 7)])
def test_full_size_separable_and_linear(cuda, k, L):
    """C2 / C4 sizes: separable inputs have exact 1D Kronecker answers; random inputs are checked
    through linearity and the adjoint identity <w, Op u> = <Op^T w, u>."""
    h = build_hierarchy(3, L, k)
    lvl = h.levels[L]
    M1, K1 = lvl.mass_1d, lvl.stiffness_1d
    rng = np.random.default_rng(5)
    Q = 3
    A = radau_iia(Q).A
    DM, DK = np.eye(Q), 1e-3 * A
    a = [rng.standard_normal(lvl.n_per_axis) for _ in range(3)]
    u1 = _sep(a, 3)
    Ma = [M1 @ x for x in a]
    Ka = [K1 @ x for x in a]
    Mu = _sep(Ma, 3)
    Ku = _sep([Ka[0], Ma[1], Ma[2]], 3) + _sep([Ma[0], Ka[1], Ma[2]], 3) + _sep([Ma[0], Ma[1], Ka[2]], 3)
    coef = rng.standard_normal(Q)
    U = torch.from_numpy(np.outer(coef, u1)).cuda()
    V = h.apply_stage_operator(L, DM, DK, U).cpu().numpy()
    ref = np.outer(DM @ coef, Mu) + np.outer(DK @ coef, Ku)
    assert rel(V, ref) < TOL
    # linearity and adjointness on random data
    x = torch.rand((Q, h.n), dtype=torch.float64, device="cuda") * 2 - 1
    y = torch.rand((Q, h.n), dtype=torch.float64, device="cuda") * 2 - 1
    ox = h.apply_stage_operator(L, DM, DK, x)
    oy = h.apply_stage_operator(L, DM, DK, y)
    oxy = h.apply_stage_operator(L, DM, DK, 2.5 * x - 0.75 * y)
    assert float((oxy - (2.5 * ox - 0.75 * oy)).abs().max() / oxy.abs().max()) < 1e-13
    oty = h.apply_stage_operator(L, DM.T, DK.T, y)
    lhs = float(torch.sum(y * ox))
    rhs = float(torch.sum(oty * x))
    assert abs(lhs - rhs) < 1e-11 * max(abs(lhs), 1.0)


@pytest.mark.parametrize("k,L", [(1, 4), (2, 3), (3, 3), (4, 3), (2, 4)])
def test_single_block_virtual_xsplit(cuda, k, L):
    """One block runs as 4 x-ranges per CTA (virtual x-split): unconstrained / constrained applies,
    the residual epilogue and a V-cycle agree with the oracle and with the plain Q = 1 launch."""
    from paper_2209_06700_b200 import _lib
    from paper_2209_06700_b200.multigrid import BlockSolver, VCycleConfig
    from oracle import solvers as OS

    h, o = build_hierarchy(3, L, k), Hierarchy(3, L, k)
    rng = np.random.default_rng(31)
    u = rng.standard_normal(o.n)
    outs = {}
    for on in (1, 0):
        _lib.call("spk_set_vsplit", h.ctx, on)
        ud = torch.from_numpy(u).cuda().reshape(1, -1)
        outs[on] = (h.apply_block(L, 1.3, 0.07, ud).cpu().numpy()[0],
                    h.apply_block(L, 1.3, 0.07, ud, constrained=True).cpu().numpy()[0],
                    BlockSolver(h, 2.5, 0.03, VCycleConfig(smoother_degree=3)).apply(
                        np.where(o.finest.interior_mask, u, 0.0)))
    ref = (o.apply_shifted(L, 1.3, 0.07, u), o.apply_constrained(L, 1.3, 0.07, u),
           OS.VCycle(o, [2.5], 0.03, OS.Config(smoother_degree=3)).apply(np.where(o.finest.interior_mask, u, 0.0)))
    for a, b, r in zip(outs[1], outs[0], ref):
        assert rel(a, r) < 1e-11
        assert rel(a, b) < 1e-13
