"""The oracle's banded fast path (oracle/fastband.c, used for the full-size C4 / C3 / C5 parity runs)
against the oracle's dense reference-form contractions (fem.py:37-41 as written) at <= 65^3 nodes
per axis-product, and once at the real 129-node-axis threshold."""

import numpy as np
import pytest

import oracle.fem_qk as F


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))


@pytest.fixture
def fast_everywhere(monkeypatch):
    monkeypatch.setattr(F, "FAST_MIN", 0)
    monkeypatch.setattr(F, "FAST_MIN_AXIS", 2)
    yield
    F.FAST = False


def _both(fn):
    F.FAST = False
    ref = fn()
    F.FAST = True
    try:
        fast = fn()
    finally:
        F.FAST = False
    return fast, ref


@pytest.mark.parametrize("dim,L,k", [(3, 4, 4), (3, 5, 2), (3, 4, 3), (2, 5, 3), (1, 5, 2), (3, 3, 1)])
def test_fast_matches_dense(dim, L, k, fast_everywhere):
    h = F.Hierarchy(dim, L, k)
    n = h.levels[L].n_dofs
    rng = np.random.default_rng(3)
    Q = 3
    u = rng.standard_normal((Q, n))
    DM, DK = rng.standard_normal((Q, Q)), rng.standard_normal((Q, Q))
    lams = np.array([1.5, 2.0, 9.0])
    checks = {
        "stage": lambda: h.apply_stage(L, DM, DK, u),
        "stage_constrained": lambda: h.apply_stage(L, DM, DK, u, constrained=True),
        "shifted": lambda: h.apply_shifted(L, lams, 0.01, u),
        "constrained": lambda: h.apply_constrained(L, 2.0, 0.01, u[0]),
        "mass": lambda: h.apply_mass(L, u),
        "stiffness": lambda: h.apply_stiffness(L, u),
        "restrict": lambda: h.restrict(L, u),
        "prolong": lambda: h.prolong(L - 1, h.restrict(L, u)),
    }
    for name, fn in checks.items():
        fast, ref = _both(fn)
        assert rel(fast, ref) <= 1e-13, (name, rel(fast, ref))
    src = lambda x, t: np.prod(np.sin(np.pi * x), axis=1) * np.exp(-t)
    fast, ref = _both(lambda: h.load_vector(L, src, 0.3))
    assert rel(fast, ref) <= 1e-13
    fast, ref = _both(lambda: h.l2_error(L, u[0], src, 0.3))
    assert abs(fast - ref) <= 1e-13 * abs(ref)


def test_fast_at_real_threshold():
    """n_ax = 129 (3D, level 5, k = 4): the configuration size where the fast path switches on."""
    h = F.Hierarchy(3, 5, 4)
    L = 5
    u = np.random.default_rng(4).standard_normal((2, h.levels[L].n_dofs))
    DM, DK = np.eye(2), 1e-3 * np.array([[0.4, -0.1], [0.7, 0.3]])
    fast, ref = _both(lambda: h.apply_stage(L, DM, DK, u, constrained=True))
    assert rel(fast, ref) <= 1e-13
