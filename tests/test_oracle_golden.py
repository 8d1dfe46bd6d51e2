"""Pin the CPU oracle against golden vectors produced by the reference package itself
(tests/golden/make_golden.py); also pins the product's host-side tableau. No GPU."""

import os

import numpy as np
import pytest

from oracle import solvers, stepper
from oracle.fem_qk import Hierarchy
from oracle.tableau_ref import crout_lu, radau_iia, spectral_complex, spectral_real

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_k1.npz"))


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def f_load(x, t):
    return np.sin(3.0 * x[:, 0]) + x[:, -1] ** 2 + t


def u_err(x, t):
    return np.cos(2.0 * x[:, 0]) * (1.0 + t)


@pytest.mark.parametrize("dim,L", [(1, 4), (2, 3), (3, 2)])
def test_fem_k1_matches_reference(dim, L):
    h = Hierarchy(dim, L, 1)
    key = f"fem_d{dim}_L{L}"
    u, uc = G[key + "_u"], G[key + "_uc"]
    assert rel(h.apply_mass(L, u), G[key + "_mass"]) < 1e-13
    assert rel(h.apply_stiffness(L, u), G[key + "_stiff"]) < 1e-13
    assert rel(h.apply_shifted(L, np.array([0.5, 2.0, 7.0]), 0.1, u), G[key + "_shifted"]) < 1e-13
    assert rel(h.apply_constrained(L, 1.3, 0.01, u[0]), G[key + "_constrained"]) < 1e-13
    assert rel(h.operator_diagonal(L, 2.0, 0.1), G[key + "_diag"]) < 1e-14
    assert rel(h.prolong(L - 1, uc), G[key + "_prolong"]) < 1e-14
    assert rel(h.restrict(L, u[:2]), G[key + "_restrict"]) < 1e-14
    assert rel(h.load_vector(L, f_load, 0.3), G[key + "_load"]) < 1e-13
    assert abs(h.l2_error(L, u[0], u_err, 0.2) - G[key + "_l2"][0]) < 1e-13 * G[key + "_l2"][0]
    assert np.array_equal(h.node_coords(L), G[key + "_coords"])


@pytest.mark.parametrize("dim,L", [(1, 4), (2, 3), (3, 3)])
def test_vcycles_match_reference(dim, L):
    h = Hierarchy(dim, L, 1)
    key = f"mg_d{dim}_L{L}"
    b = G[key + "_b"]
    bs = solvers.VCycle(h, [1.7], 0.05)
    assert rel(bs.apply(b[0]), G[key + "_block"]) < 1e-12
    lmax = [bs.sm[l][0].theta * 2 / (1 + 1 / 20.0) for l in range(L + 1)]
    assert rel(np.array(lmax), G[key + "_block_lmax"]) < 1e-12
    b3 = solvers.VCycle(h, [2.5], 0.01, solvers.Config(smoother_degree=3))
    assert rel(b3.apply(b[1]), G[key + "_block3"]) < 1e-12
    bb = solvers.VCycle(h, [1.5, 4.0], 0.05, shared=True)
    assert rel(bb.apply(b), G[key + "_batched"]) < 1e-12
    assert rel(np.array([bb.sm[l][0].theta for l in range(L + 1)]), G[key + "_batched_theta"]) < 1e-13
    pb = solvers.VCycle(h, tau=0.05, pair=(2.0, np.sqrt(2.0)))
    assert rel(pb.apply(b), G[key + "_pair"]) < 1e-12
    assert rel(np.array([pb.sm[l].theta for l in range(L + 1)]), G[key + "_pair_theta"]) < 1e-13
    x, its, hist, conv = solvers.gmres(lambda v: h.apply_constrained(L, 1.7, 0.05, v), bs.apply, b[0])
    assert its == int(G[key + "_gmres_its"][0]) and conv
    assert rel(x, G[key + "_gmres_x"]) < 1e-9
    assert rel(np.array(hist), G[key + "_gmres_hist"]) < 1e-6
    xp, itp, _, _ = solvers.gmres(lambda v: pb.op(L, v), pb.apply, b, rel_tol=1e-10)
    assert itp == int(G[key + "_pair_gmres_its"][0])
    assert rel(xp, G[key + "_pair_gmres_x"]) < 1e-9


def test_krylov_matches_reference():
    A, b = G["kry_A"], G["kry_b"]
    x, its, hist, conv = solvers.gmres(lambda v: A @ v, None, b)
    assert rel(x, G["kry_x"]) < 1e-12 and conv
    assert len(hist) == len(G["kry_hist"])
    Ac, bc = G["kryc_A"], G["kryc_b"]
    xc, itc, _, _ = solvers.gmres(lambda v: Ac @ v, None, bc)
    assert itc == int(G["kryc_its"][0])
    assert rel(xc, G["kryc_x"]) < 1e-12


@pytest.mark.parametrize("Q", range(1, 10))
def test_oracle_tableau_matches_reference(Q):
    t = radau_iia(Q)
    for nm in ("A", "b", "c", "Ainv"):
        assert np.array_equal(t[nm], G[f"tab_Q{Q}_{nm}"]), nm
    L, U = crout_lu(t["Ainv"])
    assert np.array_equal(L, G[f"tab_Q{Q}_L"]) and np.array_equal(U, G[f"tab_Q{Q}_U"])
    lam, S, Si = spectral_real(L)
    assert np.array_equal(S, G[f"tab_Q{Q}_S"]) and np.array_equal(Si, G[f"tab_Q{Q}_Sinv"])
    cl, cS, cSi, pairs = spectral_complex(t["Ainv"])
    assert np.array_equal(cl, G[f"tab_Q{Q}_clam"]) and np.array_equal(cS, G[f"tab_Q{Q}_cS"])
    assert np.allclose(np.array(pairs), G[f"tab_Q{Q}_pairs"], rtol=0, atol=0)


@pytest.mark.parametrize("Q", range(1, 10))
def test_product_tableau_matches_reference(Q):
    from paper_2209_06700_b200 import tableau as T

    t = T.radau_iia(Q)
    scale = np.abs(G[f"tab_Q{Q}_Ainv"]).max()
    assert rel(t.A, G[f"tab_Q{Q}_A"]) < 2e-11
    assert np.abs(t.Ainv - G[f"tab_Q{Q}_Ainv"]).max() < 2e-11 * scale
    assert t.c[-1] == 1.0 and np.array_equal(t.b, t.A[-1])
    lu = T.crout_lu(G[f"tab_Q{Q}_Ainv"])
    assert rel(lu.L, G[f"tab_Q{Q}_L"]) < 1e-13
    sr = T.spectral_real(G[f"tab_Q{Q}_L"])
    assert rel(sr.S, G[f"tab_Q{Q}_S"]) < 1e-13 and rel(sr.Sinv, G[f"tab_Q{Q}_Sinv"]) < 1e-13
    sc = T.spectral_complex(G[f"tab_Q{Q}_Ainv"])
    assert rel(sc.S, G[f"tab_Q{Q}_cS"]) < 1e-12
    assert np.allclose([[p.re, p.im, p.index, p.partner_index] for p in sc.pairs], G[f"tab_Q{Q}_pairs"],
                       rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("dim,L,Q,tau,steps,deg", [(2, 4, 2, 0.05, 3, 5), (3, 3, 3, 0.01, 2, 3)])
def test_oracle_step_matches_reference_composition(dim, L, Q, tau, steps, deg):
    h = Hierarchy(dim, L, 1)
    s = stepper.RealLU(h, Q, tau, solvers.Config(smoother_degree=deg))
    u = s.initial()
    its = []
    for i in range(steps):
        u, k, conv = s.step(i * tau, u)
        its.append(k)
    key = f"step_d{dim}_L{L}_Q{Q}"
    assert its == list(G[key + "_its"])
    assert rel(u, G[key + "_u"]) < 1e-10
