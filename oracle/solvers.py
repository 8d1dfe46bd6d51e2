"""Oracle: restated V-cycle solvers and GMRES (TEST ONLY; numpy/scipy on the host).

Follows reference multigrid.py (VCycleConfig :26-42, estimate_lambda_max :45-62, Chebyshev :65-88,
recursive V-cycle :110-140, BlockSolver :143-186, BatchedBlockSolver :189-256, PairBlockSolver
:259-353) and krylov.py (gmres :28-103, Hessenberg least squares :106-110), operating on any
hierarchy exposing the reference GridHierarchy interface (oracle.fem_qk.Hierarchy for Q_k).
"""

import numpy as np
import scipy.linalg

POWER_SEED = 202206


class Config:
    def __init__(self, smoother_degree=5, smoothing_range=20.0, eig_iters=20, eig_safety=1.2,
                 coarse_solver="direct"):
        self.smoother_degree = smoother_degree
        self.smoothing_range = smoothing_range
        self.eig_iters = eig_iters
        self.eig_safety = eig_safety
        self.coarse_solver = coarse_solver


def lambda_max(op, inv_diag, n, cfg, seed=POWER_SEED):
    """Seeded power iteration on Dinv*A, times the safety factor."""
    v = np.random.default_rng(seed).standard_normal(n)
    v = v / np.linalg.norm(v)
    est = 1.0
    for _ in range(cfg.eig_iters):
        w = inv_diag * op(v)
        est = np.linalg.norm(w)
        if not np.isfinite(est) or est <= 0.0:
            raise FloatingPointError(f"power iteration estimate {est}")
        v = w / est
    return est * cfg.eig_safety


class Cheb:
    def __init__(self, lmax, cfg):
        self.deg = cfg.smoother_degree
        lmin = lmax / cfg.smoothing_range
        self.theta = 0.5 * (lmax + lmin)
        self.delta = 0.5 * (lmax - lmin)

    def smooth(self, op, dinv, x, b):
        r = b - op(x)
        d = (dinv * r) / self.theta
        if self.deg == 1:
            return x + d
        sigma = self.theta / self.delta
        rho = 1.0 / sigma
        for _ in range(self.deg - 1):
            x = x + d
            r = r - op(d)
            rn = 1.0 / (2.0 * sigma - rho)
            d = rn * rho * d + (2.0 * rn / self.delta) * (dinv * r)
            rho = rn
        return x + d


class _Pair2x2Jacobi:
    def __init__(self, a, b):
        self.a, self.b = a, b

    def __mul__(self, r):
        return np.stack([self.a * r[0] + self.b * r[1], -self.b * r[0] + self.a * r[1]])

    __rmul__ = __mul__


class VCycle:
    """kind: 'block' (lams: one or per-block shifts, shared or per-block Chebyshev) or 'pair'."""

    def __init__(self, hier, lams=None, tau=0.0, cfg=None, min_level=0, shared=False, pair=None):
        self.h, self.cfg, self.min_level = hier, cfg or Config(), min_level
        self.tau = float(tau)
        self.pair = pair
        self.cycles = 0
        self.sm, self.dinv, self._coarse = {}, {}, None
        if pair is None:
            self.lams = np.atleast_1d(np.asarray(lams, dtype=float))
            for l in range(min_level, hier.max_level + 1):
                d = np.stack([1.0 / hier.operator_diagonal(l, lam, self.tau) for lam in self.lams])
                self.dinv[l] = d
                ests = [lambda_max(lambda u, l=l, lam=lam: hier.apply_constrained(l, lam, self.tau, u), d[i],
                                   hier.levels[l].n_dofs, self.cfg) for i, lam in enumerate(self.lams)]
                if shared:
                    self.sm[l] = [Cheb(max(ests), self.cfg)] * len(self.lams)
                else:
                    self.sm[l] = [Cheb(e, self.cfg) for e in ests]
        else:
            re, im = pair
            for l in range(min_level, hier.max_level + 1):
                a = hier.operator_diagonal(l, re, self.tau)
                b = np.where(hier.levels[l].interior_mask, im * hier.operator_diagonal(l, 1.0, 0.0), 0.0)
                det = a * a + b * b
                jac = _Pair2x2Jacobi(a / det, b / det)
                self.dinv[l] = jac
                n = hier.levels[l].n_dofs
                flat_jac = lambda r, jac=jac, n=n: (jac * r.reshape(2, n)).ravel()

                class _F:
                    def __mul__(s, r):
                        return flat_jac(r)
                    __rmul__ = __mul__
                est = lambda_max(lambda u, l=l, n=n: self.op(l, u.reshape(2, n)).ravel(), _F(), 2 * n, self.cfg,
                                 seed=POWER_SEED + 1)
                self.sm[l] = Cheb(est, self.cfg)

    def op(self, level, u):
        h = self.h
        if self.pair is None:
            if len(self.lams) == 1 and np.ndim(u) == 1:
                return h.apply_constrained(level, self.lams[0], self.tau, u)
            mask = h.levels[level].interior_mask
            v = h.apply_shifted(level, self.lams, self.tau, np.where(mask, u, 0.0))
            return np.where(mask, v, u)
        re, im = self.pair
        mask = h.levels[level].interior_mask
        ui = np.where(mask, u, 0.0)
        mr, mi = h.apply_mass(level, ui[0]), h.apply_mass(level, ui[1])
        kr, ki = h.apply_stiffness(level, ui[0]), h.apply_stiffness(level, ui[1])
        out = np.stack([re * mr + self.tau * kr - im * mi, im * mr + re * mi + self.tau * ki])
        return np.where(mask, out, u)

    def _smooth(self, level, x, b):
        if self.pair is not None:
            return self.sm[level].smooth(lambda u: self.op(level, u), self.dinv[level], x, b)
        if np.ndim(b) == 1:
            return self.sm[level][0].smooth(lambda u: self.op(level, u), self.dinv[level][0], x, b)
        # per-block coefficients: smooth each block with its own smoother (independent blocks)
        out = np.empty_like(b)
        for i in range(b.shape[0]):
            lam = self.lams[i]
            op = lambda u, lam=lam: self.h.apply_constrained(level, lam, self.tau, u)
            out[i] = self.sm[level][i].smooth(op, self.dinv[level][i], x[i], b[i])
        return out

    def _coarse_solve(self, b):
        l = self.min_level
        if self.cfg.coarse_solver == "chebyshev":
            return self._smooth(l, np.zeros_like(b), b)
        if self._coarse is None:
            nc = self.h.levels[l].n_dofs
            if self.pair is not None:
                cols = [self.op(l, e.reshape(2, nc)).ravel() for e in np.eye(2 * nc)]
                self._coarse = [scipy.linalg.lu_factor(np.column_stack(cols))]
            else:
                self._coarse = []
                for lam in self.lams:
                    cols = [self.h.apply_constrained(l, lam, self.tau, e) for e in np.eye(nc)]
                    self._coarse.append(scipy.linalg.lu_factor(np.column_stack(cols)))
        if self.pair is not None:
            return scipy.linalg.lu_solve(self._coarse[0], b.ravel()).reshape(b.shape)
        if np.ndim(b) == 1:
            return scipy.linalg.lu_solve(self._coarse[0], b)
        return np.stack([scipy.linalg.lu_solve(self._coarse[i], b[i]) for i in range(b.shape[0])])

    def _cycle(self, level, b):
        if level == self.min_level:
            return self._coarse_solve(b)
        x = self._smooth(level, np.zeros_like(b), b)
        r = b - self.op(level, x)
        rc = np.where(self.h.levels[level - 1].interior_mask, self.h.restrict(level, r), 0.0)
        x = x + self.h.prolong(level - 1, self._cycle(level - 1, rc))
        x = self._smooth(level, x, b)
        if not np.all(np.isfinite(x)):
            raise FloatingPointError(f"non-finite V-cycle iterate at level {level}")
        return x

    def apply(self, b):
        self.cycles += 1
        return self._cycle(self.h.max_level, np.asarray(b, dtype=float))


def hessenberg_lstsq(Hk, gk):
    y, *_ = np.linalg.lstsq(Hk, gk, rcond=None)
    return y, float(np.linalg.norm(gk - Hk @ y))


def gmres(A, Pinv, rhs, rel_tol=1e-12, max_iter=200):
    """Right-preconditioned MGS GMRES without restart; returns (x, iterations, history, converged)."""
    Pinv = Pinv or (lambda v: v)
    b = np.array(rhs, dtype=np.complex128 if np.iscomplexobj(rhs) else np.float64)
    beta = float(np.linalg.norm(b.ravel()))
    hist = [beta]
    if beta == 0.0:
        return np.zeros_like(b), 0, hist, True
    target = rel_tol * beta
    V = [b / beta]
    H = np.zeros((max_iter + 1, max_iter), dtype=b.dtype)
    g = np.zeros(max_iter + 1, dtype=b.dtype)
    g[0] = beta
    k, happy = 0, False
    for j in range(max_iter):
        w = np.asarray(A(Pinv(V[j])), dtype=b.dtype)
        if not np.all(np.isfinite(w.view(np.float64))):
            raise FloatingPointError("non-finite GMRES operator output")
        for i in range(j + 1):
            H[i, j] = np.vdot(V[i], w)
            w = w - H[i, j] * V[i]
        H[j + 1, j] = np.linalg.norm(w.ravel())
        k = j + 1
        if abs(H[j + 1, j]) < 1e-30:
            happy = True
        else:
            V.append(w / H[j + 1, j])
        y, res = hessenberg_lstsq(H[: k + 1, :k], g[: k + 1])
        hist.append(res)
        if happy or res <= target:
            break
    y, _ = hessenberg_lstsq(H[: k + 1, :k], g[: k + 1])
    z = np.zeros_like(b)
    for i in range(k):
        z = z + y[i] * V[i]
    x = np.asarray(Pinv(z), dtype=b.dtype)
    true_res = float(np.linalg.norm((b - np.asarray(A(x), dtype=b.dtype)).ravel()))
    conv = happy or true_res <= target * (1 + 1e-9) or hist[-1] <= target
    return x, k, hist, conv
