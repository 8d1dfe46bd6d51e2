"""Oracle: Radau IIA time steps composed from the restated pieces (TEST ONLY).

Real LU path (SPEC irk_solver; survey §3.4 composition):
  w_j = F(t_n + c_j tau) - K (mask u_n)        RHS sign pinned by reference test_fem.py:268-274
  rhs = mask * (Ainv w)                          eq. irk:A
  A(k)   = mask * (Ainv M(mask k) + tau K(mask k)) + (1 - mask) k
  P^-1 r = S~ [V-cycle_i((S~^-1 r)_i)]_i        eq. irk:P with L = S~ Lambda~ S~^-1, blocks lam~_i M + tau K
  k = GMRES(A, P^-1, rhs); u_{n+1} = u_n + tau sum_i b_i k_i
Direct complex path (SPEC complex_solver):
  rhs as above; w = S^-1 rhs; per pair block (lam_p M + tau K) z_p = w_p by GMRES on the real 2x2 form
  with PRESB ([I,-I;0,I] blocktri(K'+M')^-1 [I,I;0,I], two V-cycles) or the 2x2 GMG V-cycle; an odd-Q
  real eigenvalue uses the plain V-cycle; k = S z (conjugate partners by symmetry).
"""

import numpy as np

from . import solvers
from .tableau_ref import crout_lu, radau_iia, spectral_complex, spectral_real


class Separable:
    """u = T(t) prod_d s(x_d), f = F(t) prod_d s(x_d); default: the configs' sin(pi x).. e^{-t}."""

    def __init__(self, dim):
        self.dim = dim
        self.s = lambda x: np.sin(np.pi * np.asarray(x))
        self.T = lambda t: np.exp(-t)
        self.F = lambda t: (dim * np.pi ** 2 - 1.0) * np.exp(-t)

    def _sp(self, x):
        x = np.atleast_2d(x)
        v = np.ones(x.shape[0])
        for d in range(self.dim):
            v = v * self.s(x[:, d])
        return v

    def u(self, x, t):
        return self._sp(x) * self.T(t)

    def f(self, x, t):
        return self._sp(x) * self.F(t)


class RealLU:
    def __init__(self, hier, Q, tau, cfg=None, rel_tol=1e-12, max_iter=200, tab=None, shared=False, src=None):
        self.h, self.Q, self.tau, self.rel_tol, self.max_iter = hier, Q, tau, rel_tol, max_iter
        self.tab = tab or radau_iia(Q)
        L, _ = crout_lu(self.tab["Ainv"])
        self.lam, self.S, self.Si = spectral_real(L)
        self.src = src or Separable(hier.dim)
        self.pc = solvers.VCycle(hier, self.lam, tau, cfg, shared=shared)
        self.Lv = hier.max_level
        self.mask = hier.levels[self.Lv].interior_mask

    def rhs(self, t, u):
        Ku = self.h.apply_stiffness(self.Lv, np.where(self.mask, u, 0.0))
        w = np.stack([self.h.load_vector(self.Lv, self.src.f, t + c * self.tau) - Ku for c in self.tab["c"]])
        return np.where(self.mask, self.tab["Ainv"] @ w, 0.0)

    def A(self, k):
        return self.h.apply_stage(self.Lv, self.tab["Ainv"], self.tau * np.eye(self.Q), k, constrained=True)

    def Pinv(self, r):
        return self.S @ self.pc.apply(self.Si @ r)

    def step(self, t, u):
        k, its, hist, conv = solvers.gmres(self.A, self.Pinv, self.rhs(t, u), self.rel_tol, self.max_iter)
        return u + self.tau * (self.tab["b"] @ k), its, conv

    def initial(self):
        return self.src.u(self.h.node_coords(self.Lv), 0.0)


class DirectComplex:
    """Per-pair solves after the complex basis change; variant 'presb' or 'gmg'."""

    def __init__(self, hier, Q, tau, variant="presb", cfg=None, rel_tol=1e-12, max_iter=200, tab=None, src=None):
        self.h, self.Q, self.tau, self.variant = hier, Q, tau, variant
        self.rel_tol, self.max_iter = rel_tol, max_iter
        self.tab = tab or radau_iia(Q)
        self.lam, self.S, self.Si, self.pairs = spectral_complex(self.tab["Ainv"])
        self.src = src or Separable(hier.dim)
        self.Lv = hier.max_level
        self.mask = hier.levels[self.Lv].interior_mask
        self.blocks = []
        for re, im, idx, partner in self.pairs:
            if idx == partner:
                self.blocks.append(("real", re, solvers.VCycle(hier, [re], tau, cfg)))
            elif variant == "presb":
                self.blocks.append(("presb", (re, im), solvers.VCycle(hier, [re + im], tau, cfg)))
            else:
                self.blocks.append(("gmg", (re, im), solvers.VCycle(hier, tau=tau, cfg=cfg, pair=(re, im))))

    rhs = RealLU.rhs
    initial = RealLU.initial

    def _pair_op(self, re, im, u):
        h, l = self.h, self.Lv
        ui = np.where(self.mask, u, 0.0)
        mr, mi = h.apply_mass(l, ui[0]), h.apply_mass(l, ui[1])
        kr, ki = h.apply_stiffness(l, ui[0]), h.apply_stiffness(l, ui[1])
        out = np.stack([re * mr + self.tau * kr - im * mi, im * mr + re * mi + self.tau * ki])
        return np.where(self.mask, out, u)

    def _presb(self, re, im, vc, r):
        s1 = r[0] + r[1]
        y1 = vc.apply(s1)
        y2 = vc.apply(r[1] - self.h.apply_constrained(self.Lv, im, 0.0, y1))
        return np.stack([y1 - y2, y2])

    def step(self, t, u):
        rhs = self.rhs(t, u)
        iters = []
        ks = np.zeros_like(rhs)
        for (kind, par, vc), (re, im, idx, partner) in zip(self.blocks, self.pairs):
            w = self.Si[idx] @ rhs  # complex block right-hand side (n,)
            if kind == "real":
                z, its, _, _ = solvers.gmres(lambda v: self.h.apply_constrained(self.Lv, re, self.tau, v), vc.apply,
                                             w.real, self.rel_tol, self.max_iter)
                ks += np.outer(self.S[:, idx].real, z)
            else:
                b2 = np.stack([w.real, w.imag])
                op = lambda v, re=re, im=im: self._pair_op(re, im, v)
                pc = (lambda v, re=re, im=im, vc=vc: self._presb(re, im, vc, v)) if kind == "presb" else vc.apply
                z, its, _, _ = solvers.gmres(op, pc, b2, self.rel_tol, self.max_iter)
                zc = z[0] + 1j * z[1]
                ks += 2.0 * np.real(np.outer(self.S[:, idx], zc))
            iters.append(its)
        return u + self.tau * (self.tab["b"] @ ks), iters
