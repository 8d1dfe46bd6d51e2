"""Right-preconditioned GMRES (modified Gram-Schmidt, no restart) on device vectors.

Same contract as the reference krylov.gmres (krylov.py:28-103): signature, KrylovReport fields,
stopping rule (lstsq residual <= rel_tol * beta), happy breakdown below 1e-30, final x =
P^{-1}(sum_i y_i v_i), true residual recomputed, NumericalFailureError on non-finite values.

The Krylov basis lives in HBM; every MGS step is one fused sweep (spk_mgs: w -= h_prev v_prev and
the next dot, deterministic two-level reduction) whose result stays in a device Hessenberg array,
so an iteration costs j+2 memory-bound launches and ONE device->host copy (the new Hessenberg column
for the host least-squares solve, done with numpy like the reference, krylov.py:106-110).

Host (numpy) right-hand sides and callables are accepted for drop-in use: the vectors still live on
the device and the callables are bridged. Complex fields use the real (re, im) interleaved view with
the complex inner product computed on device.
"""

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._device import capture_graph, ptr, require_cuda, stream_ptr
from .errors import NumericalFailureError

BREAKDOWN_TOL = 1e-30


@dataclass
class KrylovReport:
    """Convergence record of one GMRES solve."""

    iterations: int = 0
    residual_history: list = field(default_factory=list)
    converged: bool = False
    reduction_achieved: float = 1.0
    speculative_applies: int = 0   # discarded A P^{-1} applications (gmres(speculate=True))


_NULL_CTX = None


def _ctx():
    global _NULL_CTX
    if _NULL_CTX is None:
        c = _lib.c_vp()
        _lib.check(_lib.load().spk_ctx_create(1, 1, 1, _lib.ctypes.byref(c)))
        _NULL_CTX = c
    return _NULL_CTX


def _solve_hessenberg(Hk, gk):
    y, *_ = np.linalg.lstsq(Hk, gk, rcond=None)
    res = float(np.linalg.norm(gk - Hk @ y))
    return y, res


class _Bridge:
    """Adapts user callables to device tensors of one fixed shape/dtype."""

    def __init__(self, fn, shape, host, complex_, device):
        self.fn, self.shape, self.host, self.complex, self.device = fn, shape, host, complex_, device

    def to_user(self, v):
        x = v.reshape(self.shape + ((2,) if self.complex else ()))
        if self.complex:
            x = torch.view_as_complex(x)
        return x.cpu().numpy() if self.host else x

    def from_user(self, y):
        if self.host:
            arr = np.asarray(y)
            t = torch.from_numpy(np.ascontiguousarray(arr.astype(np.complex128 if self.complex else np.float64)))
            t = t.to(self.device)
        else:
            t = y if isinstance(y, torch.Tensor) else torch.as_tensor(y, device=self.device)
            t = t.to(torch.complex128 if self.complex else torch.float64)
        if self.complex:
            t = torch.view_as_real(t.contiguous())
        return t.contiguous().reshape(-1)

    def __call__(self, v):
        if self.fn is None:
            return v
        return self.from_user(self.fn(self.to_user(v)))


class _Ops:
    """Device inner products / updates for real vectors or complex vectors in (re, im) view."""

    def __init__(self, n, complex_, device, max_iter):
        self.n, self.complex, self.device = n, complex_, device
        self.st = stream_ptr(device)
        self.ctx = _ctx()
        # Hessenberg columns: col j holds H[0..j+1, j]; complex: (re, im) pairs
        w = 2 if complex_ else 1
        self.H = torch.zeros((max_iter + 2) * (max_iter + 2) * w, dtype=torch.float64, device=device)
        self.scal = torch.zeros(8, dtype=torch.float64, device=device)
        self.scal[0] = 1.0
        self.cols = max_iter + 2

    def hptr(self, i, j):
        w = 2 if self.complex else 1
        return self.H.data_ptr() + 8 * w * (j * self.cols + i)

    def col(self, j, k):
        w = 2 if self.complex else 1
        c = self.H[w * j * self.cols : w * (j * self.cols + k)].cpu().numpy()
        return c.view(np.complex128) if self.complex else c

    def mgs_step(self, w, v_prev, h_prev_ptr, v_cur, out_ptr):
        if not self.complex:
            _lib.call("spk_mgs", self.ctx, self.n, ptr(w), ptr(v_prev) if v_prev is not None else None,
                      h_prev_ptr, ptr(v_cur) if v_cur is not None else None, out_ptr, self.st)
            return
        # complex: w -= h v (complex h), <v, w> = sum conj(v) w (np.vdot), ||w||
        wc = torch.view_as_complex(w.view(-1, 2))
        if v_prev is not None:
            h = torch.view_as_complex(self._h_view(h_prev_ptr))
            wc -= h * torch.view_as_complex(v_prev.view(-1, 2))
        if v_cur is not None:
            val = torch.vdot(torch.view_as_complex(v_cur.view(-1, 2)), wc)
            self._h_view(out_ptr).copy_(torch.view_as_real(val.reshape(1)).reshape(2))
        else:
            nrm = torch.linalg.vector_norm(wc)
            self._h_view(out_ptr).copy_(torch.stack([nrm, torch.zeros_like(nrm)]))

    def _h_view(self, p):
        off = (p - self.H.data_ptr()) // 8
        return self.H[off : off + 2]

    def norm_into(self, w, out_ptr):
        self.mgs_step(w, None, None, None, out_ptr)

    def scale_div(self, w, h_ptr, out):
        if not self.complex:
            _lib.call("spk_scale_div", self.n, ptr(w), h_ptr, ptr(out), self.st)
        else:
            h = self._h_view(h_ptr)[0]
            torch.div(w, h, out=out)


class GraphedIterations:
    """Host-free GMRES iterations for small, host-bound problems (C1 / C3): fixed basis buffers and
    ONE captured CUDA graph per iteration index j, holding w = A P^-1 v_j, the MGS column
    (spk_mgs_column), v_{j+1} = w / h, the device Givens update of the least-squares residual
    (spk_givens, krylov.py:84-87) and its copy into pinned host memory. A solve replays graph j, then
    (speculatively) graph j + 1 before it waits for iteration j's residual, so the host only reads
    two scalars per iteration; the final y is the reference's lstsq on the raw Hessenberg
    (krylov.py:89, :106-110), copied to the host once. Graphs are captured on first use and reused by
    every later solve of the same owner (same shapes, same buffers).

    A and P must be capture-safe device callables returning fresh tensors (irk.StageSystem passes
    its system operator and its un-graphed preconditioner body)."""

    def __init__(self, A, P, shape, device, max_iter):
        self.A, self.P, self.shape, self.device = A, P, tuple(shape), device
        self.N = int(np.prod(self.shape))
        self.max_iter = max_iter
        self.cols = max_iter + 2
        f64 = dict(dtype=torch.float64, device=device)
        self.H = torch.zeros(self.cols * self.cols, **f64)
        self.R = torch.zeros(self.cols * self.cols, **f64)
        self.cs = torch.zeros(2 * self.cols, **f64)
        self.g = torch.zeros(self.cols, **f64)
        self.res = torch.zeros(self.cols, **f64)
        self.scal = torch.zeros(4, **f64)
        self.host = torch.zeros(2 * self.cols, dtype=torch.float64, pin_memory=True)
        self.basis = [torch.zeros(self.N, **f64)]
        self.ptrs = (_lib.ctypes.c_void_p * (max_iter + 2))()
        self.ptrs[0] = self.basis[0].data_ptr()
        self.graphs, self.outs = {}, {}
        self.events = [torch.cuda.Event() for _ in range(self.cols)]
        self.ctx = _ctx()
        self.st = None
        self._warm()

    def _warm(self):
        """one un-captured pass of every piece (lazy allocations, kernel attributes)"""
        st = stream_ptr(self.device)
        w = self.A(self.P(self.basis[0].reshape(self.shape))).reshape(-1).contiguous()
        tmp = torch.zeros_like(self.basis[0])
        _lib.call("spk_mgs_column", self.ctx, self.N, 0, _lib.ctypes.addressof(self.ptrs), ptr(w), ptr(self.R),
                  ptr(tmp), st)
        _lib.call("spk_mgs", self.ctx, self.N, ptr(w), None, None, None, ptr(self.scal), st)
        _lib.call("spk_givens", ptr(self.R), ptr(self.R[self.cols:]), ptr(self.cs), ptr(self.g), ptr(self.res), 0, st)
        torch.cuda.synchronize()

    def hptr(self, i, j):
        return self.H.data_ptr() + 8 * (j * self.cols + i)

    def _body(self, j):
        st = stream_ptr(self.device)
        w = self.A(self.P(self.basis[j].reshape(self.shape))).reshape(-1)
        if not w.is_contiguous():
            w = w.contiguous()
        _lib.call("spk_mgs_column", self.ctx, self.N, j, _lib.ctypes.addressof(self.ptrs), ptr(w), self.hptr(0, j),
                  ptr(self.basis[j + 1]), st)
        _lib.call("spk_givens", self.hptr(0, j), self.R.data_ptr() + 8 * j * self.cols, ptr(self.cs), ptr(self.g),
                  self.res.data_ptr() + 8 * j, j, st)
        self.host[2 * j : 2 * j + 1].copy_(self.res[j : j + 1], non_blocking=True)
        self.host[2 * j + 1 : 2 * j + 2].copy_(self.H[j * self.cols + j + 1 : j * self.cols + j + 2], non_blocking=True)
        return w

    def launch(self, j):
        if j + 1 >= len(self.basis):
            self.basis.append(torch.zeros(self.N, dtype=torch.float64, device=self.device))
            self.ptrs[j + 1] = self.basis[j + 1].data_ptr()
        g = self.graphs.get(j)
        if g is None:
            g = torch.cuda.CUDAGraph()
            with capture_graph(g):
                self.outs[j] = self._body(j)
            self.graphs[j] = g
        g.replay()
        self.events[j].record()

    def solve(self, b, rel_tol, report):
        """GMRES on the device-resident (N,) rhs b; returns (k, happy) with basis / H filled."""
        st = stream_ptr(self.device)
        nb = self.scal.data_ptr()
        _lib.call("spk_mgs", self.ctx, self.N, ptr(b), None, None, None, nb, st)
        beta = float(self.scal[0].item())
        report.residual_history.append(beta)
        if beta == 0.0:
            return 0, False, beta
        _lib.call("spk_scale_div", self.N, ptr(b), nb, ptr(self.basis[0]), st)
        self.g.zero_()
        self.g[0:1].copy_(self.scal[0:1])
        target = rel_tol * beta
        k, happy, launched = 0, False, -1
        self.launch(0)
        launched = 0
        hist = report.residual_history
        for j in range(self.max_iter):
            likely_last = len(hist) >= 2 and hist[-2] > 0 and hist[-1] * (hist[-1] / hist[-2]) <= target
            if j + 1 < self.max_iter and launched == j and not likely_last:
                self.launch(j + 1)
                launched = j + 1
            self.events[j].synchronize()
            res, hsub = float(self.host[2 * j]), float(self.host[2 * j + 1])
            if not (np.isfinite(res) and np.isfinite(hsub)):
                raise NumericalFailureError("non-finite value in GMRES operator output")
            k = j + 1
            happy = abs(hsub) < BREAKDOWN_TOL
            hist.append(res)
            if happy or res <= target:
                report.speculative_applies = 1 if launched > j else 0
                break
            if launched == j and j + 1 < self.max_iter:
                self.launch(j + 1)
                launched = j + 1
        return k, happy, beta

    def hessenberg(self, k):
        Hc = self.H[: k * self.cols].reshape(k, self.cols)[:, : k + 1].cpu().numpy()
        return Hc.T.copy()  # (k+1, k): column j = H[0..k, j]


def gmres(apply_A, apply_Pinv, rhs, rel_tol=1e-12, max_iter=200, dtype=None, speculate=False, graphs=None,
          owns_output=False):
    """Solve A x = rhs with right preconditioning A P^{-1} y = rhs, x = P^{-1} y.

    rhs: torch CUDA tensor (device path) or numpy array (bridged). Returns (x, KrylovReport) with x in
    the container type of rhs.

    graphs: a GraphedIterations of the caller (device path, real field): the iterations run as replayed
    per-iteration CUDA graphs with the residual test on the device (see GraphedIterations).
    owns_output: apply_A returns a fresh tensor per call, so its output is orthogonalised in place
    (no defensive copy).

    speculate (device path): enqueue iteration j+1's A P^{-1} v_{j+1} before waiting for iteration j's
    Hessenberg column, so the host least-squares solve and the next launches overlap device work
    (small problems are host-bound). Same arithmetic in the same stream order, so the iterates are
    unchanged. Not done when the residual trend predicts convergence at the current iteration; an
    application issued after the last iteration anyway is discarded and reported in
    KrylovReport.speculative_applies.
    """
    if not (0.0 < rel_tol < 1.0):
        raise ValueError("rel_tol must lie in (0, 1)")
    require_cuda()
    host = not isinstance(rhs, torch.Tensor)
    if host:
        arr = np.asarray(rhs)
        complex_ = np.iscomplexobj(arr) if dtype is None else np.dtype(dtype).kind == "c"
        device = torch.device("cuda", torch.cuda.current_device())
        shape = arr.shape
        bt = torch.from_numpy(np.ascontiguousarray(arr.astype(np.complex128 if complex_ else np.float64)))
        bt = bt.to(device)
    else:
        complex_ = rhs.is_complex() if dtype is None else (np.dtype(dtype).kind == "c")
        device = rhs.device
        shape = tuple(rhs.shape)
        bt = rhs.to(torch.complex128 if complex_ else torch.float64)
    b = (torch.view_as_real(bt.contiguous()) if complex_ else bt.contiguous()).reshape(-1).clone()
    n = b.numel()
    A = _Bridge(apply_A, shape, host, complex_, device)
    P = _Bridge(apply_Pinv, shape, host, complex_, device)
    ops = _Ops(n, complex_, device, max_iter)

    def out_of(v):
        x = v.reshape(shape + ((2,) if complex_ else ()))
        if complex_:
            x = torch.view_as_complex(x.contiguous())
        return x.cpu().numpy() if host else x

    report = KrylovReport()
    if graphs is not None and not host and not complex_:
        return _gmres_graphed(graphs, A, P, b, n, shape, rel_tol, report, ops, out_of, device)
    beta_ptr = ops.hptr(0, max_iter + 1)  # scratch slot outside the used columns
    ops.norm_into(b, beta_ptr)
    beta = float(ops.col(max_iter + 1, 1)[0].real)
    report.residual_history.append(beta)
    if beta == 0.0:
        report.converged = True
        report.reduction_achieved = 0.0
        z = torch.zeros_like(b)
        return out_of(z), report
    target = rel_tol * beta

    basis = [torch.empty_like(b)]
    ops.scale_div(b, beta_ptr, basis[0])
    Hh = np.zeros((max_iter + 1, max_iter), dtype=np.complex128 if complex_ else np.float64)
    g = np.zeros(max_iter + 1, dtype=Hh.dtype)
    g[0] = beta
    k = 0
    happy = False
    spec = bool(speculate) and not host and not complex_
    if spec:
        col_host = torch.empty(max_iter + 2, dtype=torch.float64, pin_memory=True)
        col_ev = torch.cuda.Event()
    w_next = None
    # real device path: one C call per MGS column (the j+2 fused sweeps and v_{j+1} = w / h)
    basis_ptrs = (_lib.ctypes.c_void_p * (max_iter + 1))() if not complex_ else None
    for j in range(max_iter):
        w = w_next if w_next is not None else A(P(basis[j]))
        if w_next is None and not owns_output:
            w = w.clone()
        w_next = None
        vcol = None
        if not complex_:
            basis_ptrs[j] = basis[j].data_ptr()
            vcol = torch.empty_like(b)
            _lib.call("spk_mgs_column", ops.ctx, n, j, _lib.ctypes.addressof(basis_ptrs), ptr(w), ops.hptr(0, j),
                      ptr(vcol), ops.st)
        else:
            # modified Gram-Schmidt: h_ij = <v_i, w>; w -= h_ij v_i  (fused pairwise on device)
            ops.mgs_step(w, None, None, basis[0], ops.hptr(0, j))
            for i in range(1, j + 1):
                ops.mgs_step(w, basis[i - 1], ops.hptr(i - 1, j), basis[i], ops.hptr(i, j))
            ops.mgs_step(w, basis[j], ops.hptr(j, j), None, ops.hptr(j + 1, j))
        # skip the speculation when the residual trend predicts convergence at this iteration (the
        # product would be discarded; a wrong guess only loses the overlap of one iteration)
        hist = report.residual_history
        likely_last = len(hist) >= 2 and hist[-2] > 0 and hist[-1] * (hist[-1] / hist[-2]) <= target
        if spec and j + 1 < max_iter and not likely_last:
            # column j to pinned memory, then the next basis vector and its A P^{-1} product are queued
            # behind it; the host waits only for the column
            col_host[: j + 2].copy_(ops.H[j * ops.cols : j * ops.cols + j + 2], non_blocking=True)
            col_ev.record()
            vnext = vcol
            w_next = A(P(vnext))
            if not owns_output:
                w_next = w_next.clone()
            col_ev.synchronize()
            col = col_host[: j + 2].numpy().copy()
        else:
            vnext = vcol
            col = ops.col(j, j + 2)
        if not np.all(np.isfinite(col.view(np.float64) if complex_ else col)):
            raise NumericalFailureError("non-finite value in GMRES operator output")
        Hh[: j + 2, j] = col
        k = j + 1
        if abs(Hh[j + 1, j]) < BREAKDOWN_TOL:
            happy = True
        else:
            if vnext is None:
                vnext = torch.empty_like(b)
                ops.scale_div(w, ops.hptr(j + 1, j), vnext)
            basis.append(vnext)
        y, res = _solve_hessenberg(Hh[: k + 1, :k], g[: k + 1])
        report.residual_history.append(res)
        if happy or res <= target:
            report.speculative_applies = 1 if w_next is not None else 0
            w_next = None
            break

    y, _ = _solve_hessenberg(Hh[: k + 1, :k], g[: k + 1])
    z = torch.empty_like(b)
    if complex_:
        zc = torch.zeros(n // 2, dtype=torch.complex128, device=device)
        for i in range(k):
            zc = zc + complex(y[i]) * torch.view_as_complex(basis[i].view(-1, 2))
        z = torch.view_as_real(zc).reshape(-1).contiguous()
    else:
        yd = torch.from_numpy(np.ascontiguousarray(y[:k].astype(np.float64))).to(device)
        tbl = torch.tensor([v.data_ptr() for v in basis[:k]], dtype=torch.int64, device=device)
        _lib.call("spk_lincomb", n, k, tbl.data_ptr(), ptr(yd), ptr(z), ops.st)
    x = P(z).clone()
    r = A(x)
    if not owns_output:
        r = r.clone()
    # ||b - A x|| : r -= 1 * b, then the norm (fused)
    one = ops.scal.data_ptr()
    res_ptr = ops.hptr(1, max_iter + 1)
    if complex_:
        rc = torch.view_as_complex(r.view(-1, 2)) - torch.view_as_complex(b.view(-1, 2))
        true_res = float(torch.linalg.vector_norm(rc).item())
    else:
        _lib.call("spk_mgs", ops.ctx, n, ptr(r), ptr(b), one, None, res_ptr, ops.st)
        true_res = float(ops.H[(max_iter + 1) * ops.cols + 1].item())
    report.iterations = k
    report.reduction_achieved = true_res / beta
    report.converged = happy or true_res <= target * (1.0 + 1e-9) or report.residual_history[-1] <= target
    if not np.isfinite(true_res):  # a non-finite x reaches ||b - A x|| (A is the identity on boundary rows)
        raise NumericalFailureError("non-finite GMRES solution")
    return out_of(x), report


def _gmres_graphed(gi, A, P, b, n, shape, rel_tol, report, ops, out_of, device):
    """Device-resident iterations (GraphedIterations), then the reference's final update: y from
    lstsq on the raw Hessenberg (krylov.py:89), z = sum_i y_i v_i, x = P^-1 z, true residual."""
    k, happy, beta = gi.solve(b, rel_tol, report)
    if beta == 0.0:
        report.converged = True
        report.reduction_achieved = 0.0
        return out_of(torch.zeros_like(b)), report
    Hk = gi.hessenberg(k)
    g = np.zeros(k + 1)
    g[0] = beta
    y, _ = _solve_hessenberg(Hk, g)
    yd = torch.from_numpy(np.ascontiguousarray(y[:k].astype(np.float64))).to(device)
    tbl = torch.tensor([v.data_ptr() for v in gi.basis[:k]], dtype=torch.int64, device=device)
    z = torch.empty_like(b)
    _lib.call("spk_lincomb", n, k, tbl.data_ptr(), ptr(yd), ptr(z), ops.st)
    x = P(z).clone()
    r = A(x)
    one = ops.scal.data_ptr()
    res_ptr = ops.hptr(1, gi.max_iter + 1)
    _lib.call("spk_mgs", ops.ctx, n, ptr(r), ptr(b), one, None, res_ptr, ops.st)
    true_res = float(ops.H[(gi.max_iter + 1) * ops.cols + 1].item())
    target = rel_tol * beta
    report.iterations = k
    report.reduction_achieved = true_res / beta
    report.converged = happy or true_res <= target * (1.0 + 1e-9) or report.residual_history[-1] <= target
    if not np.isfinite(true_res):
        raise NumericalFailureError("non-finite GMRES solution")
    return out_of(x), report
