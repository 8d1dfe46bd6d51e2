"""Radau IIA time stepper on the device (SPEC irk_solver; no reference code exists,
the composition follows the survey's §3.4 probe built from reference pieces).

One step, all vectors device-resident (Q, n) fp64:
  rhs_i = mask * sum_j Ainv_ij (F(t_n + c_j tau) - K(mask u_n))      spk_rhs (separable source) or
                                                                      load_vector + combine (general f)
  A(k)  = (Ainv (x) M + tau I (x) K) k, constrained                   K1 coupled (spk_stage_apply)
  P^-1  = (S~ (x) I) blockdiag(V-cycle(lam~_i M + tau K)) (S~^-1 (x) I)  combines + MultiBlockSolver
          (mode 'batched': BatchedBlockSolver with shared Chebyshev coefficients, paper §5.3)
  k = gmres(A, P^-1, rhs); u_{n+1} = u_n + tau sum_i b_i k_i        spk_update
The RHS sign g - K u_n is the one pinned by the reference test test_fem.py:268-274.
"""

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._device import capture_graph, ptr, stream_ptr
from .errors import ConfigurationError, StepFailureError
from .fem import SeparableSolution
from .krylov import GraphedIterations, gmres
from .multigrid import BatchedBlockSolver, MultiBlockSolver, VCycleConfig
from .tableau import crout_lu, radau_iia, spectral_real
from .tensor_ops import dense_combine


# stage-DoFs below which a step is host-bound (GMRES with speculation; measured: C3 is, C5 / C4 are not)
SPECULATE_MAX_DOFS = 1 << 22


@dataclass
class SolveReport:
    """Per-step record: outer GMRES iterations, V-cycles per stage (= its + 1), history."""

    iterations: int = 0
    vcycles_per_stage: int = 0
    vcycles_total: int = 0
    residual_history: list = field(default_factory=list)
    converged: bool = False
    block_iterations: list = field(default_factory=list)  # complex path: per pair block


class StageSystem:
    """Stage system of eq. irk:A with the LU-based block preconditioner of eq. irk:P."""

    _real_path = True

    def __init__(self, hierarchy, Q, tau, mode="stage_parallel", config=None, rel_tol=1e-12, max_iter=200,
                 source=None, tableau=None):
        if mode not in ("stage_parallel", "sequential", "batched"):
            raise ConfigurationError(f"unknown mode {mode!r}")
        self.h, self.Q, self.tau, self.mode = hierarchy, int(Q), float(tau), mode
        self.rel_tol, self.max_iter = rel_tol, max_iter
        self.config = config or VCycleConfig()
        self.tab = tableau if tableau is not None else radau_iia(Q)
        Ainv = np.asarray(self.tab.Ainv if hasattr(self.tab, "Ainv") else self.tab["Ainv"])
        self.Ainv = Ainv
        self.A_ = np.asarray(self.tab.A if hasattr(self.tab, "A") else self.tab["A"])
        self.b = np.asarray(self.tab.b if hasattr(self.tab, "b") else self.tab["b"])
        self.c = np.asarray(self.tab.c if hasattr(self.tab, "c") else self.tab["c"])
        L = crout_lu(Ainv).L
        sp = spectral_real(L)
        self.lams, self.S, self.Sinv = sp.lambdas, sp.S, sp.Sinv
        self.source = source if source is not None else SeparableSolution(hierarchy.dim)
        if isinstance(self.source, tuple) and getattr(self.source[1], "solution", None) is not None:
            # callables of a separable solution (the reference's manufactured(), HeatProblem
            # defaults): the device right-hand side kernel (spk_rhs) serves them
            self.source = self.source[1].solution
        self.level = hierarchy.max_level
        lvl = hierarchy.levels[self.level]
        self.n = lvl.n_dofs
        dev = hierarchy.device
        solver_cls = BatchedBlockSolver if mode == "batched" else MultiBlockSolver
        self.precond = solver_cls(hierarchy, self.lams, self.tau, self.config) if self._real_path else None
        self._tmp = torch.zeros((self.Q, self.n), dtype=torch.float64, device=dev)
        self._bw = torch.from_numpy(self.b.copy()).to(dev)
        if isinstance(self.source, SeparableSolution):
            self._g1 = torch.from_numpy(hierarchy.load_vector_1d(self.level, self.source.s)).to(dev)
        self.vcycles = 0
        self.use_graphs = True
        self._graph = None
        # host-bound small problems: overlap the host least squares with the next A P^{-1} product
        # (krylov.gmres(speculate=True); costs one discarded application per solve)
        self.speculate = self.Q * self.n <= SPECULATE_MAX_DOFS
        # ... and run their GMRES iterations as replayed per-iteration CUDA graphs with the residual
        # test on the device (krylov.GraphedIterations); large problems are device-bound already
        self.graph_iterations = self.speculate and self._real_path
        self._gi = None

    # ---- pieces ----
    def assemble_rhs(self, t_n, u_n):
        h, L = self.h, self.level
        um = h.constrain(L, u_n.reshape(1, -1))
        ku = h.apply_block(L, 0.0, 1.0, um)
        out = torch.empty((self.Q, self.n), dtype=torch.float64, device=h.device)
        if isinstance(self.source, SeparableSolution):
            T = _lib.dbl_array([self.source.F(t_n + cj * self.tau) for cj in self.c])
            A = np.ascontiguousarray(self.Ainv)
            _lib.call("spk_rhs", h.ctx, L, self.Q, ptr(self._g1), T, A.ctypes.data_as(_lib.P_dbl), ptr(ku),
                      ptr(out), stream_ptr(h.device))
        else:
            f = self.source[1] if isinstance(self.source, tuple) else self.source.f_source
            w = torch.stack([h.load_vector_device(L, f, t_n + cj * self.tau) - ku[0] for cj in self.c])
            dense_combine(self.Ainv, w, out=out, mask_level=L, hierarchy=h)
        return out

    def apply_system_operator(self, k):
        return self.h.apply_stage_operator(self.level, self.Ainv, self.tau * np.eye(self.Q), k, constrained=True)

    def _precond_body(self, r, out):
        w = dense_combine(self.Sinv, r.reshape(self.Q, self.n), hierarchy=self.h)
        z = self.precond.apply_device(w, check=False)
        return dense_combine(self.S, z, out=out, hierarchy=self.h)

    def apply_preconditioner(self, r):
        """P^-1 r: combine(S~^-1) -> Q V-cycles -> combine(S~). The whole chain (tens of small
        launches per level) is captured once as a CUDA graph and replayed."""
        self.vcycles += 1
        if not self.use_graphs:
            return self._precond_body(r, None)
        if self._graph is None:
            self._g_in = torch.zeros((self.Q, self.n), dtype=torch.float64, device=self.h.device)
            self._g_out = torch.zeros_like(self._g_in)
            self._precond_body(self._g_in, self._g_out)  # warm-up: configures kernels, allocates
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with capture_graph(g):
                self._precond_body(self._g_in, self._g_out)
            self._graph = g
        self._g_in.copy_(r.reshape(self.Q, self.n))
        self._graph.replay()
        return self._g_out

    def _graphed_iterations(self):
        if not (self.graph_iterations and self.use_graphs):
            return None
        if self._gi is None:
            self._gi = GraphedIterations(self.apply_system_operator, lambda r: self._precond_body(r, None),
                                         (self.Q, self.n), self.h.device, self.max_iter)
        return self._gi

    def step(self, t_n, u_n, check=True):
        """u_{n+1} for device u_n (n,), and the SolveReport."""
        nvtx = torch.cuda.nvtx
        nvtx.range_push("radau_step")
        nvtx.range_push("assemble_rhs")
        rhs = self.assemble_rhs(t_n, u_n)
        nvtx.range_pop()
        v0 = self.vcycles
        gi = self._graphed_iterations()
        nvtx.range_push("gmres")
        k, rep = gmres(self.apply_system_operator, self.apply_preconditioner, rhs, self.rel_tol, self.max_iter,
                       speculate=self.speculate, graphs=gi, owns_output=True)
        nvtx.range_pop()
        if gi is not None:
            self.vcycles += rep.iterations  # the in-graph P^-1 applications (the final one counted itself)
        else:
            self.vcycles -= rep.speculative_applies
        if check:
            self.precond.check_finite()
        u_next = u_n.clone()
        _lib.call("spk_update", self.n, self.Q, ptr(k), ptr(self._bw), self.tau, ptr(u_next),
                  stream_ptr(self.h.device))
        nvtx.range_pop()
        report = SolveReport(iterations=rep.iterations, vcycles_per_stage=self.vcycles - v0,
                             vcycles_total=self.Q * (self.vcycles - v0),
                             residual_history=rep.residual_history, converged=rep.converged)
        if not rep.converged:
            raise StepFailureError("stage solve did not converge", report=report)
        return u_next, report

    def initial_condition(self, t0=0.0):
        h = self.h
        s1 = torch.from_numpy(self.source.s(h.levels[self.level].nodes_1d) * 1.0).to(h.device)
        u = torch.empty(self.n, dtype=torch.float64, device=h.device)
        _lib.call("spk_outer3", h.ctx, self.level, ptr(s1), ptr(u), stream_ptr(h.device))
        return u * self.source.T(t0)

    def run(self, steps, t0=0.0, u0=None):
        u = self.initial_condition(t0) if u0 is None else u0
        t = t0
        reports = []
        for _ in range(steps):
            u, rep = self.step(t, u)
            t += self.tau
            reports.append(rep)
        return u, t, reports
