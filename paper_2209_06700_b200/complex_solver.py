"""Directly diagonalised A_Q^{-1} (eq. irk:Ainv) on the device: per conjugate pair, the block
(lam_p M + tau K) z_p = w_p is solved by GMRES on its real 2x2 form (eq. complex:twobytwo) with the
PRESB preconditioner (eq. presb:p; two sequential V-cycles on K' + M') or one 2x2 GMG V-cycle
(PairBlockSolver); an odd-Q real eigenvalue uses the plain real V-cycle.

GMRES runs on the real (2, n) form: PRESB is only R-linear, so a complex-arithmetic Krylov method
would mis-combine its images; the real form keeps GMRES exact for both preconditioners.
Basis changes: w = S^{-1} rhs and k = S z are real (2P x Q) / (Q x 2P) combines (tensor_ops).
"""

import numpy as np
import torch

from . import _lib
from ._device import capture_graph, ptr, stream_ptr
from .errors import StepFailureError
from .irk import SolveReport, StageSystem
from .krylov import gmres
from .multigrid import BlockSolver, PairBlockSolver
from .tableau import spectral_complex
from .tensor_ops import dense_combine, paired_back_matrix, paired_forward_matrix


class DirectComplexSystem(StageSystem):
    """Stage-pair parallel solve of eq. irk:Ainv; variant 'presb' or 'gmg'."""

    _real_path = False

    def __init__(self, hierarchy, Q, tau, variant="presb", config=None, rel_tol=1e-12, max_iter=200,
                 source=None, tableau=None):
        # reuse RHS / update / initial condition plumbing of the real path (no real preconditioner)
        self.variant = variant
        super().__init__(hierarchy, Q, tau, "stage_parallel", config, rel_tol, max_iter, source, tableau)
        sp = spectral_complex(self.Ainv)
        self.spec = sp
        self.Wf = paired_forward_matrix(sp.Sinv, sp.pairs)
        self.Wb = paired_back_matrix(sp.S, sp.pairs)
        self.blocks = []
        for p in sp.pairs:
            if p.is_real:
                self.blocks.append(("real", p, BlockSolver(hierarchy, p.re, tau, self.config)))
            elif variant == "presb":
                self.blocks.append(("presb", p, BlockSolver(hierarchy, p.re + p.im, tau, self.config)))
            else:
                self.blocks.append(("gmg", p, PairBlockSolver(hierarchy, p.re, p.im, tau, self.config)))

    def _build_preconditioner(self):
        return None

    def _graphed(self, key, fn):
        """fn (a preconditioner: tens of small launches per V-cycle level) captured once as a CUDA
        graph on static buffers and replayed; returns a fresh tensor per call."""
        cache = self.__dict__.setdefault("_graphs", {})
        if not self.use_graphs:
            return fn

        def run(x):
            ent = cache.get(key)
            if ent is None or ent[0].shape != x.shape:
                g_in = torch.zeros_like(x)
                fn(g_in)  # warm-up: configures kernels, allocates
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with capture_graph(g):
                    g_out = fn(g_in).clone()
                ent = (g_in, g, g_out)
                cache[key] = ent
            ent[0].copy_(x)
            ent[1].replay()
            return ent[2].clone()

        return run

    def _pair_op(self, re, im, u):
        h = self.h
        v = torch.empty_like(u)
        _lib.call("spk_pair_apply", h.ctx, self.level, re, im, self.tau, 1, ptr(u), ptr(v), stream_ptr(h.device))
        return v

    def _presb(self, p, vc, r):
        """P^-1 (r1, r2) = [I,-I;0,I] blocktri(K'+M')^-1 [I,I;0,I] (eq. presb:p), 2 V-cycles."""
        h, L = self.h, self.level
        s1 = (r[0] + r[1]).reshape(1, -1)
        y1 = vc.apply_device(s1, check=False)
        By1 = h.apply_block(L, p.im, 0.0, y1, constrained=True)
        y2 = vc.apply_device((r[1].reshape(1, -1) - By1), check=False)
        return torch.cat([y1 - y2, y2], dim=0)

    def step(self, t_n, u_n, check=True):
        rhs = self.assemble_rhs(t_n, u_n)
        w = dense_combine(self.Wf, rhs, hierarchy=self.h)  # (2P, n): (re, im) rows per pair
        z = torch.zeros_like(w)
        its = []
        for bi, (kind, p, vc) in enumerate(self.blocks):
            if kind == "real":
                op = lambda v, lam=p.re: self.h.apply_block(self.level, lam, self.tau, v.reshape(1, -1),
                                                            constrained=True).reshape(v.shape)
                pc = self._graphed(("real", bi), lambda v, vc=vc: vc.apply_device(v.reshape(1, -1),
                                                                                   check=False).reshape(v.shape))
                zi, rep = gmres(op, pc, w[2 * bi].contiguous(), self.rel_tol, self.max_iter,
                                speculate=self.speculate)
                z[2 * bi].copy_(zi)
            else:
                op = lambda v, re=p.re, im=p.im: self._pair_op(re, im, v.contiguous())
                if kind == "presb":
                    pc = self._graphed(("presb", bi), lambda v, p=p, vc=vc: self._presb(p, vc, v))
                else:
                    pc = self._graphed(("gmg", bi), lambda v, vc=vc: vc.apply_device(v.contiguous(), check=False))
                zi, rep = gmres(op, pc, w[2 * bi : 2 * bi + 2].contiguous(), self.rel_tol, self.max_iter,
                                speculate=self.speculate)
                z[2 * bi : 2 * bi + 2].copy_(zi)
            its.append(rep.iterations)
            if not rep.converged:
                raise StepFailureError(f"pair block {bi} did not converge", report=rep)
        k = dense_combine(self.Wb, z, hierarchy=self.h)
        u_next = u_n.clone()
        _lib.call("spk_update", self.n, self.Q, ptr(k), ptr(self._bw), self.tau, ptr(u_next),
                  stream_ptr(self.h.device))
        return u_next, SolveReport(iterations=max(its), converged=True, block_iterations=its)
