"""Device geometric multigrid for the blocks (lam M + tau K): one V-cycle as the approximate block
inverse inside the stage preconditioner.

Mirrors the reference multigrid module (VCycleConfig multigrid.py:26-42, estimate_lambda_max :45-62,
ChebyshevSmoother :65-88, _VCycleBase :91-140, BlockSolver :143-186, BatchedBlockSolver :189-256,
PairBlockSolver :259-353, chebyshev_smooth / v_cycle / v_cycle_2x2 :356-373) with the same numerics:
seeded power iteration (seed 202206, pair: 202207 on the 2n vector), frozen Chebyshev coefficients,
V(deg, deg) from a zero guess, masked restriction, direct coarse solve (LU of the assembled coarse
operator). Every level operation runs on the device:

  smoothing start      spk_cheb_init / spk_residual(+d)    r = b - A x, d = Dinv r / theta
  Chebyshev step       spk_cheb_step (K1 + fused epilogue)  x += d, r -= A d, d = c1 d + c2 Dinv r
  x + d (+NaN flag)    spk_axpy_flag
  restriction          spk_transfer (P^T, masked)
  prolongation         spk_transfer (P, accumulate)
  coarse solve         x_c = LU^{-1} b_c (inverse of the assembled coarse operator, device GEMV)

`MultiBlockSolver` batches independent per-stage BlockSolvers (per-block Chebyshev coefficients) in
the same launches: numerically identical to Q separate BlockSolvers, Q times fewer launches.
"""

from dataclasses import dataclass

import os

import numpy as np
import scipy.linalg
import torch

from . import _lib
from ._device import is_host, like_input, ptr, stream_ptr, to_device
from .errors import ConfigurationError, NumericalFailureError, SpectralFailureError

_POWER_SEED = 202206


@dataclass
class VCycleConfig:
    smoother_degree: int = 5
    smoothing_range: float = 20.0
    eig_iters: int = 20
    eig_safety: float = 1.2
    coarse_solver: str = "direct"  # "direct" | "chebyshev"

    def __post_init__(self):
        if self.smoother_degree < 1:
            raise ConfigurationError("smoother_degree must be >= 1")
        if self.smoothing_range <= 1.0:
            raise ConfigurationError("smoothing_range must exceed 1")
        if self.eig_safety < 1.0:
            raise ConfigurationError("eig_safety must be >= 1")
        if self.coarse_solver not in ("direct", "chebyshev"):
            raise ConfigurationError(f"unknown coarse solver {self.coarse_solver!r}")


def _norm(v):
    if isinstance(v, torch.Tensor):
        return float(torch.linalg.vector_norm(v.reshape(-1)).item())
    return float(np.linalg.norm(np.asarray(v).ravel()))


def estimate_lambda_max(apply_op, inv_diag, n, config=None, seed=_POWER_SEED):
    """Power iteration on the Jacobi-preconditioned operator (generic callables, host or device);
    returns the estimate times eig_safety (reference multigrid.py:45-62)."""
    config = config or VCycleConfig()
    v = np.random.default_rng(seed).standard_normal(n)
    v /= np.linalg.norm(v)
    if isinstance(inv_diag, torch.Tensor):
        v = torch.from_numpy(v).to(inv_diag.device)
    est = 1.0
    for _ in range(config.eig_iters):
        w = inv_diag * apply_op(v)
        est = _norm(w)
        if not np.isfinite(est) or est <= 0.0:
            raise SpectralFailureError(f"power iteration produced estimate {est}")
        v = w / est
    return est * config.eig_safety


class ChebyshevSmoother:
    """Fixed-coefficient Chebyshev iteration around point Jacobi (reference multigrid.py:65-88)."""

    def __init__(self, lam_max, config):
        self.degree = config.smoother_degree
        self.lam_max = float(lam_max)
        lam_min = lam_max / config.smoothing_range
        self.theta = 0.5 * (lam_max + lam_min)
        self.delta = 0.5 * (lam_max - lam_min)

    def coefficients(self):
        """(c1_k, c2_k) of the deg-1 inner steps: d = c1 d + c2 Dinv r."""
        sigma = self.theta / self.delta
        rho = 1.0 / sigma
        out = []
        for _ in range(self.degree - 1):
            rho_new = 1.0 / (2.0 * sigma - rho)
            out.append((rho_new * rho, 2.0 * rho_new / self.delta))
            rho = rho_new
        return out

    def apply(self, apply_op, inv_diag, x, b):
        """Generic (callable) smoothing, returns the updated x."""
        r = b - apply_op(x)
        d = (inv_diag * r) / self.theta
        if self.degree == 1:
            return x + d
        for c1, c2 in self.coefficients():
            x = x + d
            r = r - apply_op(d)
            d = c1 * d + c2 * (inv_diag * r)
        return x + d


def chebyshev_smooth(apply_op, inv_diag, x, b, lam_max, config=None):
    """Standalone Chebyshev smoothing step (testing hook, reference multigrid.py:356-359)."""
    config = config or VCycleConfig()
    return ChebyshevSmoother(lam_max, config).apply(apply_op, inv_diag, x, b)


class _Level:
    def __init__(self, nblk, n, device, need_b):
        mk = lambda: torch.zeros((nblk, n), dtype=torch.float64, device=device)
        self.x, self.r, self.d, self.d2 = mk(), mk(), mk(), mk()
        self.b = mk() if need_b else None


class _DeviceVCycle:
    """V-cycle engine over nblk independent blocks (or one 2x2 pair) on the device."""

    pair = False
    # the coarsest levels (a few thousand nodes per block) run as ONE fused launch
    # (spk_coarse_vcycle: the same cycle inside one CTA per block, vectors in shared memory)
    _fuse_coarse = os.environ.get("SPK_FUSE_COARSE", "1") != "0"
    _cv_level = -1

    def __init__(self, hierarchy, config, min_level):
        if not (0 <= min_level <= hierarchy.max_level):
            raise ConfigurationError("min_level outside hierarchy range")
        self.hierarchy = hierarchy
        self.config = config or VCycleConfig()
        self.min_level = min_level
        self.smoothers = {}
        self.cycles_applied = 0
        self._bufs = None
        self._coarse_inv = None

    # ---- subclass hooks ----
    @property
    def nrows(self):
        """rows of the (rows, n) device vectors the cycle works on"""
        raise NotImplementedError

    def _block_lams(self):
        raise NotImplementedError

    def _halo(self, level, t):
        """refresh the halo planes of t before an operator application / transfer reads them
        (no-op on a whole-mesh hierarchy; slab.DistMultiBlockSolver exchanges them)"""

    # ---- device kernels per level ----
    def _thetas(self, level):
        return [sm.theta for sm in self._level_smoothers(level)]

    def _level_smoothers(self, level):
        s = self.smoothers[level]
        return s if isinstance(s, list) else [s] * self.nrows

    def _smooth(self, level, b, lv, zero_start):
        h = self.hierarchy
        st = stream_ptr(h.device)
        sms = self._level_smoothers(level)
        thetas = _lib.dbl_array([sm.theta for sm in sms])
        if self.pair:
            re, im = self.re_lam, self.im_lam
            if zero_start:
                _lib.call("spk_pair_cheb_init", h.ctx, level, re, im, self.tau, sms[0].theta, ptr(b), ptr(lv.r),
                          ptr(lv.x), ptr(lv.d), st)
            else:
                _lib.call("spk_pair_residual", h.ctx, level, re, im, self.tau, ptr(lv.x), ptr(b), ptr(lv.r),
                          ptr(lv.d), sms[0].theta, st)
        else:
            lams = _lib.dbl_array(self._block_lams())
            nb = self.nrows
            deg = self.config.smoother_degree
            if zero_start and deg >= 2 and _lib.load().spk_cheb_split(h.ctx, level, nb) == 1:
                # large level: d = Dinv b / theta, then the first step with r = b, x = 0 implicit
                _lib.call("spk_cheb_start", h.ctx, level, nb, lams, self.tau, thetas, ptr(b), ptr(lv.d), st)
                coefs = [sm.coefficients() for sm in sms]
                self._halo(level, lv.d)
                _lib.call("spk_cheb_first_step", h.ctx, level, nb, lams, self.tau,
                          _lib.dbl_array([c[0][0] for c in coefs]), _lib.dbl_array([c[0][1] for c in coefs]),
                          ptr(b), ptr(lv.d), ptr(lv.r), ptr(lv.x), ptr(lv.d2), 1 if deg == 2 else 0,
                          ptr(self._flags[level:]), st)
                lv.d, lv.d2 = lv.d2, lv.d
                self._cheb_steps(level, lv, coefs, first=1)
                return
            if zero_start:
                _lib.call("spk_cheb_init", h.ctx, level, nb, lams, self.tau, thetas, ptr(b), ptr(lv.r), ptr(lv.x),
                          ptr(lv.d), st)
            else:
                self._halo(level, lv.x)
                _lib.call("spk_residual", h.ctx, level, nb, lams, self.tau, ptr(lv.x), ptr(b), ptr(lv.r),
                          ptr(lv.d), thetas, st)
        deg = self.config.smoother_degree
        flag = ptr(self._flags[level:])
        if deg == 1:
            _lib.call("spk_axpy_flag", lv.x.numel(), ptr(lv.x), ptr(lv.d), flag, st)
            return
        self._cheb_steps(level, lv, [sm.coefficients() for sm in sms], first=0)

    def _cheb_steps(self, level, lv, coefs, first):
        """Chebyshev steps first .. deg-2 (the last one fused with "return x + d")."""
        h = self.hierarchy
        st = stream_ptr(h.device)
        deg = self.config.smoother_degree
        flag = ptr(self._flags[level:])
        for k in range(first, deg - 1):
            final = 1 if k == deg - 2 else 0  # last step also performs "return x + d" (fused)
            self._halo(level, lv.d)
            if self.pair:
                c1, c2 = coefs[0][k]
                _lib.call("spk_pair_cheb_step", h.ctx, level, self.re_lam, self.im_lam, self.tau, c1, c2,
                          ptr(lv.d), ptr(lv.r), ptr(lv.x), ptr(lv.d2), final, flag, st)
            else:
                c1s = _lib.dbl_array([c[k][0] for c in coefs])
                c2s = _lib.dbl_array([c[k][1] for c in coefs])
                _lib.call("spk_cheb_step", h.ctx, level, self.nrows, _lib.dbl_array(self._block_lams()),
                          self.tau, c1s, c2s, ptr(lv.d), ptr(lv.r), ptr(lv.x), ptr(lv.d2), final, flag, st)
            lv.d, lv.d2 = lv.d2, lv.d

    def _residual_restrict(self, level, b, lv):
        h = self.hierarchy
        st = stream_ptr(h.device)
        if self.pair:
            _lib.call("spk_pair_residual", h.ctx, level, self.re_lam, self.im_lam, self.tau, ptr(lv.x), ptr(b),
                      ptr(lv.r), None, 1.0, st)
        else:
            self._halo(level, lv.x)
            _lib.call("spk_residual", h.ctx, level, self.nrows, _lib.dbl_array(self._block_lams()), self.tau,
                      ptr(lv.x), ptr(b), ptr(lv.r), None, None, st)
        self._halo(level, lv.r)
        h.restrict_into(level, lv.r, self._bufs[level - 1].b, mask=True)

    def _ensure(self):
        if self._bufs is not None:
            return
        h = self.hierarchy
        self._bufs = {}
        for level in range(self.min_level, h.max_level + 1):
            self._bufs[level] = _Level(self.nrows, h.levels[level].n_dofs, h.device, level < h.max_level)
        self._flags = torch.zeros(h.max_level + 1, dtype=torch.int32, device=h.device)
        self._cv_level = -1
        if (self._fuse_coarse and not self.pair and h.dim >= 2 and self.min_level == 0
                and self.config.coarse_solver == "direct" and self.nrows <= 16):
            lc = min(int(_lib.load().spk_coarse_vcycle_level(h.ctx)), h.max_level)
            if lc >= 1:
                deg = self.config.smoother_degree
                rows = []
                for level in range(lc + 1):
                    for b in range(self.nrows):
                        if level == 0:
                            rows.append([0.0] * (2 * deg - 1))
                            continue
                        sm = self._level_smoothers(level)[b]
                        row = [sm.theta]
                        for c1, c2 in sm.coefficients():
                            row += [c1, c2]
                        rows.append(row)
                self._cv_coef = torch.tensor(rows, dtype=torch.float64, device=h.device).contiguous()
                self._cv_lams = _lib.dbl_array(self._block_lams())
                self._cv_scratch = torch.zeros((self.nrows, 3 * h.levels[lc].n_dofs), dtype=torch.float64,
                                               device=h.device)
                self._cv_level = lc

    def _coarse(self, b):
        """Coarse solve: direct (inverse of the assembled coarse operator) or Chebyshev."""
        lv = self._bufs[self.min_level]
        if self.config.coarse_solver == "chebyshev":
            self._smooth(self.min_level, b, lv, zero_start=True)
            return lv.x
        if self._coarse_inv is None:
            self._coarse_inv = self._build_coarse_inverse()
        if self.pair:
            out = (self._coarse_inv @ b.reshape(-1, 1)).reshape(2, -1)
        else:
            out = torch.bmm(self._coarse_inv, b.unsqueeze(-1)).squeeze(-1)
        lv.x.copy_(out)
        return lv.x

    def _build_coarse_inverse(self):
        """Assemble the constrained coarse operator column by column on the device, LU-factor it on
        the host (scipy, as the reference multigrid.py:179-186), return the inverse on the device."""
        h = self.hierarchy
        nc = h.levels[self.min_level].n_dofs
        if self.pair:
            cols = []
            for j in range(2 * nc):
                e = torch.zeros((2, nc), dtype=torch.float64, device=h.device)
                e.view(-1)[j] = 1.0
                v = torch.empty_like(e)
                _lib.call("spk_pair_apply", h.ctx, self.min_level, self.re_lam, self.im_lam, self.tau, 1,
                          ptr(e), ptr(v), stream_ptr(h.device))
                cols.append(v.reshape(-1))
            mat = torch.stack(cols, dim=1).cpu().numpy()
            lu = scipy.linalg.lu_factor(mat)
            inv = scipy.linalg.lu_solve(lu, np.eye(2 * nc))
            return torch.from_numpy(inv).to(h.device)
        eye = torch.eye(nc, dtype=torch.float64, device=h.device)
        invs = []
        for lam in self._block_lams():
            cols = h.apply_block(self.min_level, lam, self.tau, eye, constrained=True)  # row j = A e_j
            mat = cols.T.contiguous().cpu().numpy()
            lu = scipy.linalg.lu_factor(mat)
            invs.append(scipy.linalg.lu_solve(lu, np.eye(nc)))
        return torch.from_numpy(np.stack(invs)).to(h.device)

    def _coarse_fused(self, level, b):
        """Levels 0..level in one launch (spk_coarse_vcycle)."""
        h = self.hierarchy
        lv = self._bufs[level]
        if self._coarse_inv is None:
            self._coarse_inv = self._build_coarse_inverse().contiguous()
        _lib.call("spk_coarse_vcycle", h.ctx, level, self.nrows, self._cv_lams, self.tau,
                  self.config.smoother_degree, ptr(self._cv_coef), ptr(self._coarse_inv), ptr(b), ptr(lv.x),
                  ptr(self._cv_scratch), ptr(self._flags), stream_ptr(h.device))
        return lv.x

    def _cycle(self, level, b):
        if level == self._cv_level:
            return self._coarse_fused(level, b)
        if level == self.min_level:
            return self._coarse(b)
        lv = self._bufs[level]
        self._smooth(level, b, lv, zero_start=True)
        self._residual_restrict(level, b, lv)
        ec = self._cycle(level - 1, self._bufs[level - 1].b)
        self.hierarchy.prolong_into(level - 1, ec, lv.x, accumulate=True)
        self._smooth(level, b, lv, zero_start=False)
        return lv.x

    def apply_device(self, b, out=None, check=True):
        """One V-cycle from the zero guess on device rows b (nrows, n); returns a device tensor."""
        self._ensure()
        self._flags.zero_()
        x = self._cycle(self.hierarchy.max_level, b)
        if out is None:
            out = x.clone()
        else:
            out.copy_(x)
        self.cycles_applied += 1
        if check:
            self.check_finite()
        return out

    def check_finite(self):
        flags = self._flags.cpu().numpy()
        bad = [l for l in range(self.min_level + 1, len(flags)) if flags[l]]
        if bad:
            raise NumericalFailureError("non-finite V-cycle iterate", level=min(bad))

    def apply(self, b):
        """One V-cycle from the zero initial guess (reference multigrid.py:110-114)."""
        h = self.hierarchy
        n = h.finest.n_dofs
        shape = tuple(b.shape)
        bd = to_device(b, h.device).reshape(self.nrows, n)
        x = self.apply_device(bd)
        return like_input(x.reshape(shape), b)


class _BlockFamily(_DeviceVCycle):
    def __init__(self, hierarchy, lams, tau, config, min_level, shared):
        super().__init__(hierarchy, config, min_level)
        self.lams = np.atleast_1d(np.asarray(lams, dtype=float))
        self.tau = float(tau)
        self.shared = shared
        self.lambda_max = {}
        self._diag = {}
        for level in range(self.min_level, hierarchy.max_level + 1):
            per_block = [self._estimate(level, lam) for lam in self.lams]
            if shared:
                est = max(per_block)
                self.lambda_max[level] = est
                self.smoothers[level] = ChebyshevSmoother(est, self.config)
            else:
                self.lambda_max[level] = per_block if len(per_block) > 1 else per_block[0]
                sm = [ChebyshevSmoother(e, self.config) for e in per_block]
                self.smoothers[level] = sm if len(sm) > 1 else sm[0]

    @property
    def nrows(self):
        return len(self.lams)

    def _block_lams(self):
        return list(self.lams)

    def _estimate(self, level, lam):
        """Device power iteration (estimate_lambda_max semantics, one sync at the end)."""
        h = self.hierarchy
        n = h.levels[level].n_dofs
        v0 = np.random.default_rng(_POWER_SEED).standard_normal(n)
        v0 /= np.linalg.norm(v0)
        v = torch.from_numpy(v0).to(h.device)
        w = torch.empty_like(v)
        ests = torch.zeros(self.config.eig_iters, dtype=torch.float64, device=h.device)
        st = stream_ptr(h.device)
        for it in range(self.config.eig_iters):
            est_ptr = ests.data_ptr() + 8 * it
            _lib.call("spk_dinv_norm", h.ctx, level, 0, float(lam), 0.0, self.tau, ptr(v), ptr(w), est_ptr, st)
            _lib.call("spk_scale_div", n, ptr(w), est_ptr, ptr(v), st)
        e = ests.cpu().numpy()
        for est in e:
            if not np.isfinite(est) or est <= 0.0:
                raise SpectralFailureError(f"power iteration produced estimate {est}")
        return float(e[-1]) * self.config.eig_safety

    def _inv_diag(self, level):
        if level not in self._diag:
            self._diag[level] = np.stack([1.0 / self.hierarchy.operator_diagonal(level, lam, self.tau)
                                          for lam in self.lams])
        d = self._diag[level]
        return d[0] if len(self.lams) == 1 else d

    def _apply(self, level, u):
        """Constrained block operator (host or device input)."""
        return self.hierarchy.apply_constrained(level, self.lams if len(self.lams) > 1 else self.lams[0],
                                                self.tau, u)


class BlockSolver(_BlockFamily):
    """V-cycle approximate inverse of one constrained block (lam M + tau K) (multigrid.py:143-186)."""

    def __init__(self, hierarchy, lam, tau, config=None, min_level=0):
        super().__init__(hierarchy, [float(lam)], tau, config, min_level, shared=False)
        self.lam = float(lam)


class BatchedBlockSolver(_BlockFamily):
    """All Q blocks in one sweep with a shared Chebyshev coefficient set from the max lambda_max
    over blocks (paper §5.3; multigrid.py:189-256)."""

    def __init__(self, hierarchy, lams, tau, config=None, min_level=0):
        super().__init__(hierarchy, lams, tau, config, min_level, shared=True)


class MultiBlockSolver(_BlockFamily):
    """Q independent BlockSolvers (per-block coefficients) executed in the same launches: the
    stage-parallel preconditioner of eq. irk:P on one device."""

    def __init__(self, hierarchy, lams, tau, config=None, min_level=0):
        super().__init__(hierarchy, lams, tau, config, min_level, shared=False)


class PairBlockSolver(_DeviceVCycle):
    """V-cycle on the coupled real form [[K', -M'], [M', K']] with 2x2 block Jacobi smoothing
    (multigrid.py:259-353); K' = re M + tau K, M' = im M."""

    pair = True

    def __init__(self, hierarchy, re_lam, im_lam, tau, config=None, min_level=0):
        super().__init__(hierarchy, config, min_level)
        self.re_lam, self.im_lam, self.tau = float(re_lam), float(im_lam), float(tau)
        self.lambda_max = {}
        for level in range(self.min_level, hierarchy.max_level + 1):
            est = self._estimate(level)
            self.lambda_max[level] = est
            self.smoothers[level] = ChebyshevSmoother(est, self.config)

    @property
    def nrows(self):
        return 2

    def _estimate(self, level):
        h = self.hierarchy
        n = h.levels[level].n_dofs
        v0 = np.random.default_rng(_POWER_SEED + 1).standard_normal(2 * n)
        v0 /= np.linalg.norm(v0)
        v = torch.from_numpy(v0).to(h.device)
        w = torch.empty_like(v)
        ests = torch.zeros(self.config.eig_iters, dtype=torch.float64, device=h.device)
        st = stream_ptr(h.device)
        for it in range(self.config.eig_iters):
            est_ptr = ests.data_ptr() + 8 * it
            _lib.call("spk_dinv_norm", h.ctx, level, 1, self.re_lam, self.im_lam, self.tau, ptr(v), ptr(w),
                      est_ptr, st)
            _lib.call("spk_scale_div", 2 * n, ptr(w), est_ptr, ptr(v), st)
        e = ests.cpu().numpy()
        for est in e:
            if not np.isfinite(est) or est <= 0.0:
                raise SpectralFailureError(f"power iteration produced estimate {est}")
        return float(e[-1]) * self.config.eig_safety

    def _apply(self, level, u):
        """Coupled 2x2 operator on (2, n), constrained (multigrid.py:292-304)."""
        h = self.hierarchy
        n = h.levels[level].n_dofs
        ud = to_device(u, h.device).reshape(2, n)
        v = torch.empty_like(ud)
        _lib.call("spk_pair_apply", h.ctx, level, self.re_lam, self.im_lam, self.tau, 1, ptr(ud), ptr(v),
                  stream_ptr(h.device))
        return like_input(v.reshape(tuple(u.shape)), u)

    def apply_device_flat(self, b):
        return self.apply_device(b.reshape(2, -1))


def v_cycle(hierarchy, lambda_shift, tau, b, config=None, min_level=0):
    """One-shot V-cycle (reference multigrid.py:362-367)."""
    if lambda_shift <= 0.0:
        raise ConfigurationError("lambda_shift must be positive")
    return BlockSolver(hierarchy, lambda_shift, tau, config, min_level).apply(b)


def v_cycle_2x2(hierarchy, re_lam, im_lam, tau, b_pair, config=None, min_level=0):
    """One V-cycle on the coupled 2x2 system (reference multigrid.py:370-373)."""
    return PairBlockSolver(hierarchy, re_lam, im_lam, tau, config, min_level).apply(b_pair)
