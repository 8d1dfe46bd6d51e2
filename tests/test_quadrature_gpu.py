"""Device load vector and L2 error (reference fem.py:220-273) against the
oracle's quadratures: general callables (host evaluation at the Gauss points + the device
Gauss-to-node / node-to-Gauss kernels) and separable solutions (the reference's manufactured() family
and the configs' sin(pi x) e^{-t}, formed and evaluated on the device), k = 1..4, d = 1..3."""

import numpy as np
import pytest

from oracle.fem_qk import Hierarchy
from paper_2209_06700_b200.fem import SeparableSolution, build_hierarchy, manufactured

pytestmark = pytest.mark.gpu

CASES = [(1, 5, 1), (1, 4, 3), (2, 3, 2), (2, 3, 4), (3, 2, 1), (3, 2, 2), (3, 2, 3), (3, 1, 4)]


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))


def general_f(x, t):
    """non-separable, with every coordinate present"""
    return x[:, 0] ** 2 + 3.0 * x[:, -1] + np.cos(2.0 * x.sum(axis=1)) * (1.0 + t)


@pytest.mark.parametrize("dim,L,k", CASES)
def test_load_vector_general_and_manufactured(dim, L, k):
    h, o = build_hierarchy(dim, L, k), Hierarchy(dim, L, k)
    for t in (0.0, 0.37):
        assert rel(h.load_vector(L, general_f, t), o.load_vector(L, general_f, t)) < 1e-13
        u_ex, f_src, _ = manufactured(dim)
        assert f_src.separable is not None  # device path
        plain = lambda x, tt: f_src(x, tt)   # same function without the separable tag: oracle input
        assert rel(h.load_vector(L, f_src, t), o.load_vector(L, plain, t)) < 1e-13


@pytest.mark.parametrize("dim,L,k", CASES)
def test_l2_error_general_and_separable(dim, L, k):
    h, o = build_hierarchy(dim, L, k), Hierarchy(dim, L, k)
    n = h.levels[L].n_dofs
    uh = np.random.default_rng(dim * 10 + k).standard_normal(n)
    for u_ex in (manufactured(dim)[0], SeparableSolution(dim).callables()[0]):
        plain = lambda x, t, u_ex=u_ex: u_ex(x, t)
        for t in (0.0, 0.5):
            ref = o.l2_error(L, uh, plain, t)
            assert abs(h.l2_error(L, uh, u_ex, t) - ref) <= 1e-13 * ref
            assert abs(h.l2_error(L, uh, plain, t) - ref) <= 1e-13 * ref
    # interpolant of the exact solution: the error converges at order k+1 (here: small and positive)
    u_ex = manufactured(dim)[0]
    ui = u_ex(h.node_coords(L), 0.2)
    e = h.l2_error(L, ui, u_ex, 0.2)
    # (e is small by cancellation: compare at the scale of the quadrature of u itself)
    scale = o.l2_error(L, np.zeros(n), lambda x, t: u_ex(x, t), 0.2)
    assert 0.0 < e < 0.5 and abs(e - o.l2_error(L, ui, lambda x, t: u_ex(x, t), 0.2)) <= 1e-13 * scale


def test_manufactured_step_uses_device_rhs():
    """A Radau IIA step with the reference's manufactured() callables (HeatProblem default) runs the
    separable device RHS and matches the step driven by the general (host-evaluated) callable."""
    import torch

    from paper_2209_06700_b200.irk import StageSystem
    from paper_2209_06700_b200.multigrid import VCycleConfig

    h = build_hierarchy(2, 3, 2)
    cb = manufactured(2)
    plain = tuple(lambda x, t, f=f: f(x, t) for f in cb)
    cfg = VCycleConfig(smoother_degree=3)
    a = StageSystem(h, 2, 0.01, config=cfg, source=cb)
    b = StageSystem(h, 2, 0.01, config=cfg, source=plain)
    assert isinstance(a.source, SeparableSolution) and isinstance(b.source, tuple)
    u0 = torch.from_numpy(cb[0](h.node_coords(3), 0.0)).cuda()
    ua, ra = a.step(0.0, u0)
    ub, rb = b.step(0.0, u0)
    assert ra.iterations == rb.iterations
    assert rel(ua.cpu().numpy(), ub.cpu().numpy()) < 1e-12
