"""Generate golden vectors from the reference package itself (run in the build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the unmodified reference `spirk` (pkg/src/spirk) and records the outputs of its own public
functions on small seeded inputs: fem operators/transfers/load/L2 (fem.py), the three V-cycle
solvers and their lambda_max (multigrid.py), GMRES (krylov.py), the tableau factors for Q = 1..9
(tableau.py), and a time step composed from reference pieces exactly as SPEC.md:448-483 describes
(the survey's §3.4 probe). The oracle (oracle/) is pinned against this file in
tests/test_oracle_golden.py; /root/reference is never read at test time.
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("SPIRK_SRC", "/root/reference/pkg/src"))
from spirk import fem, krylov, multigrid, tableau  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_k1.npz")
g = {}


def f_load(x, t):
    return np.sin(3.0 * x[:, 0]) + x[:, -1] ** 2 + t


def u_err(x, t):
    return np.cos(2.0 * x[:, 0]) * (1.0 + t)


rng = np.random.default_rng(2024)
for dim, L in [(1, 4), (2, 3), (3, 2)]:
    h = fem.build_hierarchy(dim, L)
    n = h.n
    key = f"fem_d{dim}_L{L}"
    u = rng.standard_normal((3, n))
    uc = rng.standard_normal((2, h.levels[L - 1].n_dofs))
    lam = np.array([0.5, 2.0, 7.0])
    g[key + "_u"] = u
    g[key + "_uc"] = uc
    g[key + "_mass"] = h.apply_mass(L, u)
    g[key + "_stiff"] = h.apply_stiffness(L, u)
    g[key + "_shifted"] = h.apply_shifted(L, lam, 0.1, u)
    g[key + "_constrained"] = h.apply_constrained(L, 1.3, 0.01, u[0])
    g[key + "_diag"] = h.operator_diagonal(L, 2.0, 0.1)
    g[key + "_prolong"] = h.prolong(L - 1, uc)
    g[key + "_restrict"] = h.restrict(L, u[:2])
    g[key + "_load"] = h.load_vector(L, f_load, 0.3)
    g[key + "_l2"] = np.array([h.l2_error(L, u[0], u_err, 0.2)])
    g[key + "_coords"] = h.node_coords(L)

# multigrid: BlockSolver / BatchedBlockSolver / PairBlockSolver (k = 1)
for dim, L in [(1, 4), (2, 3), (3, 3)]:
    h = fem.build_hierarchy(dim, L)
    mask = h.finest.interior_mask
    key = f"mg_d{dim}_L{L}"
    b = np.where(mask, rng.standard_normal((2, h.n)), 0.0)
    g[key + "_b"] = b
    bs = multigrid.BlockSolver(h, 1.7, 0.05)
    g[key + "_block"] = bs.apply(b[0])
    g[key + "_block_lmax"] = np.array([bs.lambda_max[l] for l in range(L + 1)])
    cfg3 = multigrid.VCycleConfig(smoother_degree=3)
    g[key + "_block3"] = multigrid.BlockSolver(h, 2.5, 0.01, cfg3).apply(b[1])
    bb = multigrid.BatchedBlockSolver(h, [1.5, 4.0], 0.05)
    g[key + "_batched"] = bb.apply(b)
    g[key + "_batched_theta"] = np.array([bb.smoothers[l].theta for l in range(L + 1)])
    pb = multigrid.PairBlockSolver(h, 2.0, np.sqrt(2.0), 0.05)
    g[key + "_pair"] = pb.apply(b)
    g[key + "_pair_theta"] = np.array([pb.smoothers[l].theta for l in range(L + 1)])
    # GMRES + V-cycle on the block operator
    x, rep = krylov.gmres(lambda v: h.apply_constrained(L, 1.7, 0.05, v), bs.apply, b[0], rel_tol=1e-12)
    g[key + "_gmres_x"] = x
    g[key + "_gmres_its"] = np.array([rep.iterations])
    g[key + "_gmres_hist"] = np.array(rep.residual_history)
    xp, repp = krylov.gmres(lambda v: pb._apply(L, v), pb.apply, b, rel_tol=1e-10)
    g[key + "_pair_gmres_x"] = xp
    g[key + "_pair_gmres_its"] = np.array([repp.iterations])

# krylov on dense systems
A = rng.standard_normal((40, 40)) + 8.0 * np.eye(40)
bvec = rng.standard_normal(40)
x, rep = krylov.gmres(lambda v: A @ v, None, bvec, rel_tol=1e-12)
g["kry_A"], g["kry_b"], g["kry_x"] = A, bvec, x
g["kry_hist"] = np.array(rep.residual_history)
Ac = rng.standard_normal((20, 20)) + 1j * rng.standard_normal((20, 20)) + 10 * np.eye(20)
bc = rng.standard_normal(20) + 1j * rng.standard_normal(20)
xc, repc = krylov.gmres(lambda v: Ac @ v, None, bc, rel_tol=1e-12)
g["kryc_A"], g["kryc_b"], g["kryc_x"] = Ac, bc, xc
g["kryc_its"] = np.array([repc.iterations])

# tableau Q = 1..9
for Q in range(1, 10):
    t = tableau.radau_iia(Q)
    lu = tableau.crout_lu(t.Ainv)
    sr = tableau.spectral_real(lu.L)
    sc = tableau.spectral_complex(t.Ainv)
    for nm, v in [("A", t.A), ("b", t.b), ("c", t.c), ("Ainv", t.Ainv), ("L", lu.L), ("U", lu.U),
                  ("lam", sr.lambdas), ("S", sr.S), ("Sinv", sr.Sinv), ("clam", sc.lambdas), ("cS", sc.S),
                  ("cSinv", sc.Sinv)]:
        g[f"tab_Q{Q}_{nm}"] = v
    g[f"tab_Q{Q}_pairs"] = np.array([[p.re, p.im, p.index, p.partner_index] for p in sc.pairs])


# composed real-LU step from reference pieces, k = 1
def composed_steps(dim, L, Q, tau, steps, degree):
    h = fem.build_hierarchy(dim, L)
    t = tableau.radau_iia(Q)
    sp = tableau.spectral_real(tableau.crout_lu(t.Ainv).L)
    cfg = multigrid.VCycleConfig(smoother_degree=degree)
    blocks = [multigrid.BlockSolver(h, lam, tau, cfg) for lam in sp.lambdas]
    mask = h.finest.interior_mask
    sfun = lambda x: np.prod(np.sin(np.pi * x), axis=1)
    F = lambda x, tt: sfun(x) * (dim * np.pi ** 2 - 1.0) * np.exp(-tt)
    u = sfun(h.node_coords(L))
    its = []
    for s in range(steps):
        tn = s * tau
        Ku = h.apply_stiffness(L, np.where(mask, u, 0.0))
        w = np.stack([h.load_vector(L, F, tn + c * tau) - Ku for c in t.c])
        rhs = np.where(mask, t.Ainv @ w, 0.0)

        def A_op(k):
            ki = np.where(mask, k, 0.0)
            v = t.Ainv @ h.apply_mass(L, ki) + tau * h.apply_stiffness(L, ki)
            return np.where(mask, v, k)

        def P(r):
            z = sp.Sinv @ r
            return sp.S @ np.stack([blocks[i].apply(z[i]) for i in range(Q)])

        k, rep = krylov.gmres(A_op, P, rhs, rel_tol=1e-12)
        u = u + tau * (t.b @ k)
        its.append(rep.iterations)
    return u, np.array(its)


for dim, L, Q, tau, steps, deg in [(2, 4, 2, 0.05, 3, 5), (3, 3, 3, 0.01, 2, 3)]:
    u, its = composed_steps(dim, L, Q, tau, steps, deg)
    key = f"step_d{dim}_L{L}_Q{Q}"
    g[key + "_u"] = u
    g[key + "_its"] = its

np.savez_compressed(OUT, **g)
print("wrote", OUT, os.path.getsize(OUT), "bytes,", len(g), "arrays")
