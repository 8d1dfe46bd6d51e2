"""Stage-parallel Radau IIA step across GPUs (the paper's layout).

Rank (s, b) of a `runtime.RankGrid` owns stage group s (a contiguous range of the Q stages) of mesh
partition b (B = 1: the whole mesh; B > 1: an x-slab, `slab.SlabPartition`), so every block solve
of eq. irk:P runs inside its column group with no inter-stage traffic. The exchanges are:

* stage combines (D (x) I) u for D in {S~^-1, S~, A^-1}: a Cannon-like ring (`RingCombiner`): in round
  s rank r holds the stage group of rank (r + s) mod world, adds D[own, held] @ held, and passes it on
  (world - 1 shifts of one stage group; grouped isend/irecv, NCCL over NVLink on the GPU path);
* GMRES inner products: local partial dot + all-reduce (fixed order, deterministic per run);
* halo planes on the column group before each operator application (B > 1 only);
* the update u + tau sum_i b_i k_i: partial sums all-reduced on the row group.

The driver is backend-agnostic: `backend` supplies the stage-local operators. `GPUStageBackend` uses
the device kernels (K1 block mode, MultiBlockSolver, spk_rhs); tests/test_stage_parallel_gloo.py runs the
same driver with a CPU backend built on the oracle over gloo and checks it against the single-process
oracle stepper.
"""

import numpy as np
import torch
import torch.distributed as dist

from .errors import NumericalFailureError
from .runtime import Counters, RankGrid, all_reduce_sum, host_staged, stage_groups  # noqa: F401
from .tableau import crout_lu, radau_iia, spectral_real


def _combine_into(out, D, rows, accumulate):
    """out (+)= D @ rows: the device kernel (spk_combine, K7) for CUDA tensors, torch for the CPU
    test doubles."""
    if out.is_cuda:
        from . import _lib
        from ._device import stream_ptr
        Dc = np.ascontiguousarray(D, dtype=np.float64)
        _lib.call("spk_combine", None, -1, out.shape[-1], Dc.shape[1], Dc.shape[0], Dc.ctypes.data_as(_lib.P_dbl),
                  rows.data_ptr(), rows.stride(0), out.data_ptr(), out.stride(0), 1 if accumulate else 0,
                  stream_ptr(out.device))
        return
    blk = torch.from_numpy(np.ascontiguousarray(D)).to(out.dtype)
    if accumulate:
        out.addmm_(blk, rows)
    else:
        torch.mm(blk, rows, out=out)


class RingCombiner:
    """v_own = sum_j D[own, j] x_j with x distributed by stage groups (Cannon-like rotation,
    PAPER.md:481-548; SPEC tensor_ops rotate_combine).

    `rank` is the position in the ring (the stage group index), `world` the ring length; `ranks`
    maps ring positions to global ranks (default: identity, the default group).

    Double-buffered: in round s the transfer of the held stage group to the left neighbour (and the
    receive of the next one from the right) is posted BEFORE round s's combine kernel is queued, so
    on NCCL the NVLink transfer of round s+1's operand overlaps round s's FMA; the received buffer is
    only read after the request completes. Two persistent wire buffers per shape, no per-round
    allocation or zero-fill. Groups may be uneven or empty (Q not a multiple of the ring length)."""

    def __init__(self, groups, rank, world, group=None, ranks=None, counters=None):
        self.groups, self.rank, self.world, self.group = groups, rank, world, group
        self.ranks = list(ranks) if ranks is not None else list(range(world))
        self.counters = counters if counters is not None else Counters()
        self.shift_rounds = 0
        self._wires = {}

    def _buffers(self, rows, n, dtype, device):
        key = (rows, n, dtype, str(device))
        if key not in self._wires:
            self._wires[key] = [torch.zeros((rows, n), dtype=dtype, device=device) for _ in range(2)]
        return self._wires[key]

    def __call__(self, D, x_local, in_groups=None, out_groups=None):
        """in_groups / out_groups: row ranges of D's columns / rows owned by each rank (default:
        the stage groups for both)."""
        D = np.asarray(D, dtype=np.float64)
        ig = in_groups or self.groups
        og = out_groups or self.groups
        r, W = self.rank, self.world
        lo, hi = og[r]
        n = x_local.shape[-1]
        dev = x_local.device
        out = torch.zeros((hi - lo, n), dtype=x_local.dtype, device=dev)
        maxg = max(max(g[1] - g[0] for g in ig), 1)
        ilo, ihi = ig[r]
        if W == 1:
            if hi > lo and ihi > ilo:
                _combine_into(out, D[lo:hi, ilo:ihi], x_local[: ihi - ilo].contiguous(), False)
            return out
        # gloo moves host memory only: stage the wire buffers on the host for CUDA tensors
        host = x_local.is_cuda and dist.get_backend(self.group) == "gloo"
        cur, nxt = self._buffers(maxg, n, x_local.dtype, "cpu" if host else dev)
        if ihi > ilo:
            cur[: ihi - ilo].copy_(x_local[: ihi - ilo])
        held_owner = r
        first = True
        for s in range(W):
            reqs = []
            if s < W - 1:  # post round s+1's exchange before round s's combine
                ops = [dist.P2POp(dist.isend, cur, self.groups_rank((r - 1) % W), self.group),
                       dist.P2POp(dist.irecv, nxt, self.groups_rank((r + 1) % W), self.group)]
                reqs = dist.batch_isend_irecv(ops)
                self.shift_rounds += 1
                self.counters.shift_rounds += 1
                self.counters.add_send(cur)
            hlo, hhi = ig[held_owner]
            if hhi > hlo and hi > lo:
                rows = cur[: hhi - hlo]
                if host:
                    rows = rows.to(dev)
                _combine_into(out, D[lo:hi, hlo:hhi], rows, not first)
                first = False
            for req in reqs:
                req.wait()
            cur, nxt = nxt, cur
            held_owner = (held_owner + 1) % W
        return out

    def groups_rank(self, r):
        return self.ranks[r]


class CudaIpcWindows:
    """Peer windows in device memory: cudaMalloc'd buffers exported / imported with CUDA IPC
    (`spk_ipc_*`); peers map them over NVLink (lazy peer access)."""

    def __init__(self, device):
        self.device = device

    def create(self, nbytes):
        from . import _lib
        p = _lib.c_vp()
        h = (_lib.ctypes.c_char * 64)()
        _lib.call("spk_ipc_alloc", int(nbytes), _lib.ctypes.byref(p), h)
        return p.value, bytes(h)

    def open(self, handle):
        from . import _lib
        p = _lib.c_vp()
        buf = (_lib.ctypes.c_char * 64).from_buffer_copy(handle)
        _lib.call("spk_ipc_open", buf, _lib.ctypes.byref(p))
        return p.value

    def row(self, ptr, i, n):
        return ptr + i * n * 8

    def write(self, ptr, x):
        from . import _lib
        from ._device import stream_ptr
        x = x.contiguous()
        _lib.call("spk_copy_d2d", ptr, x.data_ptr(), x.numel() * 8, stream_ptr(self.device))

    def combine(self, n, rows, D, out):
        from . import _lib
        from ._device import stream_ptr
        D = np.ascontiguousarray(D, dtype=float)
        table = (_lib.c_vp * len(rows))(*rows)
        _lib.call("spk_peer_combine", n, len(rows), table, D.shape[0], D.ctypes.data_as(_lib.P_dbl),
                  out.data_ptr(), out.stride(0), 0, stream_ptr(self.device))

    def sync(self):
        torch.cuda.current_stream(self.device).synchronize()

    def close(self, peer_ptrs, own):
        from . import _lib
        for p in peer_ptrs:
            _lib.call("spk_ipc_close", p)
        _lib.call("spk_ipc_free", own)


class PeerCombiner:
    """Shared-memory stage combine (SPEC tensor_ops sharedmem_combine; the paper's
    shared-memory virtual topology): every rank of the row group exposes its
    stage group in a peer window; between two row barriers each rank reads the peers' rows directly
    and combines them in ONE kernel (`spk_peer_combine`: the loads over NVLink are the exchange).
    No messages, 2 barriers per call. Same interface as RingCombiner."""

    def __init__(self, groups, rank, world, group=None, ranks=None, counters=None, windows=None, device=None):
        self.groups, self.rank, self.world, self.group = groups, rank, world, group
        self.ranks = list(ranks) if ranks is not None else list(range(world))
        self.counters = counters if counters is not None else Counters()
        self.windows = windows if windows is not None else CudaIpcWindows(device)
        self.shift_rounds = 0
        self._own = None
        self._n = None

    def _setup(self, n, rows_max):
        own, handle = self.windows.create(rows_max * n * 8)
        handles = [None] * self.world
        if self.world > 1:
            dist.all_gather_object(handles, handle, group=self.group)
        else:
            handles = [handle]
        self._own = own
        self._peers = [own if r == self.rank else self.windows.open(h) for r, h in enumerate(handles)]
        self._n, self._rows_max = n, rows_max

    def _barrier(self):
        if self.world > 1:
            dist.barrier(group=self.group)
        self.counters.barrier_count += 1

    def __call__(self, D, x_local, in_groups=None, out_groups=None):
        D = np.asarray(D)
        ig = in_groups or self.groups
        og = out_groups or self.groups
        lo, hi = og[self.rank]
        n = x_local.shape[-1]
        rows_max = max(max(g[1] - g[0] for g in ig), 1)
        if self._own is None or self._n != n or self._rows_max < rows_max:
            if self._own is not None:
                self.close()
            self._setup(n, rows_max)
        ilo, ihi = ig[self.rank]
        if ihi > ilo:
            self.windows.write(self._own, x_local[: ihi - ilo])
        self.windows.sync()
        self._barrier()  # every window holds its rank's current rows
        out = torch.zeros((hi - lo, n), dtype=x_local.dtype, device=x_local.device)
        rows = []
        for r, (a, b) in enumerate(ig):
            rows.extend(self.windows.row(self._peers[r], i, n) for i in range(b - a))
        if hi > lo and rows:
            self.windows.combine(n, rows, D[lo:hi, : len(rows)], out)
        self.windows.sync()
        self._barrier()  # nobody overwrites a window before every rank has read it
        return out

    def close(self):
        """Collective: release the peer mappings and the own window."""
        if self._own is None:
            return
        self._barrier()
        self.windows.close([p for r, p in enumerate(self._peers) if r != self.rank], self._own)
        self._own = None


class DistKrylov:
    """Right-preconditioned MGS GMRES (krylov.py:28-103 semantics) with all-reduced inner products.

    `owned(v)` selects the entries a rank owns (slab halos excluded from the dots).

    Device path (CUDA vectors, every entry owned): each MGS sweep is one fused `spk_mgs_partial`
    launch (w -= h_prev v_prev; local <v_cur, w>) writing this rank's partial straight into the
    device Hessenberg slot, which is then all-reduced in place (NCCL: 8 bytes on the stream, no host
    sync); the next sweep reads the reduced h from device memory. The norm slot is all-reduced as a
    sum of squares and square-rooted on device. The host sees ONE copy per iteration: the finished
    column for the least-squares solve (np.linalg.lstsq as in krylov.py:106-110). Slab partitions
    (halo entries excluded) compute the partials with torch on device, same order, still without a
    host sync per dot. CPU tensors (gloo tests) take the host path."""

    def __init__(self, group=None, owned=None, counters=None, ctx=None):
        self.group = group
        self.owned = owned
        self.counters = counters
        self.ctx = ctx

    def _own(self, v):
        return self.owned(v) if self.owned is not None else v

    def dot(self, a, b):
        t = torch.sum(self._own(a) * self._own(b)).reshape(1).to(torch.float64)
        all_reduce_sum(t, self.group, self.counters)
        return float(t.item())

    def _lstsq(self, H, g, k):
        y, *_ = np.linalg.lstsq(H[: k + 1, :k], g[: k + 1], rcond=None)
        res = float(np.linalg.norm(g[: k + 1] - H[: k + 1, :k] @ y))
        return y, res

    def solve(self, A, P, b, rel_tol=1e-12, max_iter=200):
        if b.is_cuda:
            return self._solve_device(A, P, b, rel_tol, max_iter)
        beta = np.sqrt(self.dot(b, b))
        hist = [beta]
        if beta == 0.0:
            return torch.zeros_like(b), 0, hist, True
        target = rel_tol * beta
        V = [b / beta]
        H = np.zeros((max_iter + 1, max_iter))
        g = np.zeros(max_iter + 1)
        g[0] = beta
        k, happy = 0, False
        for j in range(max_iter):
            w = A(P(V[j]))
            for i in range(j + 1):
                H[i, j] = self.dot(V[i], w)
                w = w - H[i, j] * V[i]
            H[j + 1, j] = np.sqrt(self.dot(w, w))
            if not np.all(np.isfinite(H[: j + 2, j])):
                raise NumericalFailureError("non-finite value in distributed GMRES")
            k = j + 1
            if abs(H[j + 1, j]) < 1e-30:
                happy = True
            else:
                V.append(w / H[j + 1, j])
            y, res = self._lstsq(H, g, k)
            hist.append(res)
            if happy or res <= target:
                break
        y, _ = self._lstsq(H, g, k)
        z = torch.zeros_like(b)
        for i in range(k):
            z = z + float(y[i]) * V[i]
        x = P(z)
        r = b - A(x)
        true_res = np.sqrt(self.dot(r, r))
        conv = happy or true_res <= target * (1 + 1e-9) or hist[-1] <= target
        return x, k, hist, conv

    # ---- device path ----
    def _sweep(self, Hd, w, v_prev, hp, v_cur, out):
        """Hd[out] = local <v_cur, w - Hd[hp] v_prev> (or local sum w^2 if v_cur is None); w updated."""
        if self.owned is None:
            from . import _lib
            from ._device import stream_ptr
            _lib.call("spk_mgs_partial", self.ctx, w.numel(), w.data_ptr(),
                      v_prev.data_ptr() if v_prev is not None else None,
                      Hd[hp:].data_ptr() if v_prev is not None else None,
                      v_cur.data_ptr() if v_cur is not None else None, Hd[out:].data_ptr(), stream_ptr(w.device))
            return
        if v_prev is not None:
            w.sub_(Hd[hp] * v_prev)
        wo = self._own(w)
        c = self._own(v_cur) if v_cur is not None else wo
        Hd[out : out + 1].copy_(torch.sum(c * wo).reshape(1))

    def _solve_device(self, A, P, b, rel_tol, max_iter):
        if self.owned is None and self.ctx is None:
            from .krylov import _ctx
            self.ctx = _ctx()
        b = b.contiguous()
        Hd = torch.zeros((max_iter + 2) * (max_iter + 2), dtype=torch.float64, device=b.device)
        cols = max_iter + 2
        # beta = ||b||: sum of squares, all-reduced, square-rooted on device
        nb = (max_iter + 1) * cols
        self._sweep(Hd, b, None, 0, None, nb)
        all_reduce_sum(Hd[nb : nb + 1], self.group, self.counters)
        from . import _lib
        from ._device import stream_ptr
        st = stream_ptr(b.device)
        _lib.call("spk_sqrt_dev", Hd[nb:].data_ptr(), 1, st)
        beta = float(Hd[nb].item())
        hist = [beta]
        if beta == 0.0:
            return torch.zeros_like(b), 0, hist, True
        target = rel_tol * beta
        V = [b / Hd[nb]]
        H = np.zeros((max_iter + 1, max_iter))
        g = np.zeros(max_iter + 1)
        g[0] = beta
        k, happy = 0, False
        for j in range(max_iter):
            w = A(P(V[j])).contiguous().clone()
            c0 = j * cols
            for i in range(j + 1):
                self._sweep(Hd, w, V[i - 1] if i > 0 else None, c0 + i - 1, V[i], c0 + i)
                all_reduce_sum(Hd[c0 + i : c0 + i + 1], self.group, self.counters)
            self._sweep(Hd, w, V[j], c0 + j, None, c0 + j + 1)
            all_reduce_sum(Hd[c0 + j + 1 : c0 + j + 2], self.group, self.counters)
            _lib.call("spk_sqrt_dev", Hd[c0 + j + 1 :].data_ptr(), 1, st)
            col = Hd[c0 : c0 + j + 2].cpu().numpy()   # the one host copy of the iteration
            if not np.all(np.isfinite(col)):
                raise NumericalFailureError("non-finite value in distributed GMRES")
            H[: j + 2, j] = col
            k = j + 1
            if abs(H[j + 1, j]) < 1e-30:
                happy = True
            else:
                V.append(w / Hd[c0 + j + 1])
            y, res = self._lstsq(H, g, k)
            hist.append(res)
            if happy or res <= target:
                break
        y, _ = self._lstsq(H, g, k)
        z = torch.zeros_like(b)
        for i in range(k):
            z.add_(V[i], alpha=float(y[i]))
        x = P(z)
        r = b - A(x)
        nr = (max_iter + 1) * cols + 1
        self._sweep(Hd, r, None, 0, None, nr)
        all_reduce_sum(Hd[nr : nr + 1], self.group, self.counters)
        true_res = float(np.sqrt(Hd[nr].item()))
        conv = happy or true_res <= target * (1 + 1e-9) or hist[-1] <= target
        return x, k, hist, conv


class StageParallelStepper:
    """eq. irk:A solved by GMRES with the eq. irk:P preconditioner, stages distributed over ranks."""

    def __init__(self, backend, Q, tau, rank, world, group=None, tableau=None, rel_tol=1e-12, max_iter=200,
                 grid=None, combine="ring", windows=None):
        self.be, self.Q, self.tau = backend, Q, float(tau)
        self.rank, self.world = rank, world
        self.rel_tol, self.max_iter = rel_tol, max_iter
        tab = tableau if tableau is not None else radau_iia(Q)
        get = lambda t, k: np.asarray(t[k] if isinstance(t, dict) else getattr(t, k))
        self.A, self.b, self.c, self.Ainv = get(tab, "A"), get(tab, "b"), get(tab, "c"), get(tab, "Ainv")
        sp = spectral_real(crout_lu(self.Ainv).L)
        self.lams, self.S, self.Sinv = sp.lambdas, sp.S, sp.Sinv
        # rank grid: default = every rank its own stage group, one mesh partition (B = 1)
        self.grid = grid if grid is not None else RankGrid(world, 1)
        if self.grid.size != world and self.grid.topology != "row_major_padded":
            raise ValueError(f"rank grid spans {self.grid.size} ranks, world has {world}")
        sb = self.grid.coords(rank)
        if sb is None:
            raise ValueError(f"rank {rank} is idle in the {self.grid.topology} grid")
        self.s_idx, self.b_idx = sb
        S = self.grid.S
        if S > 1 and self.grid.B > 1:
            # the row groups carry the stage combines and the update all-reduce; without them those
            # would run on the world group and silently add different x-slabs together
            self.grid.init_groups()
        self.groups = stage_groups(Q, S)
        self.lo, self.hi = self.groups[self.s_idx]
        row_group = self.grid.row_group(self.b_idx) if self.grid.B > 1 else group
        self.row_group = row_group
        if combine == "ring":
            self.ring = RingCombiner(self.groups, self.s_idx, S, row_group, ranks=self.grid.row_ranks(self.b_idx),
                                     counters=self.grid.counters)
        elif combine == "peer":
            self.ring = PeerCombiner(self.groups, self.s_idx, S, row_group, ranks=self.grid.row_ranks(self.b_idx),
                                     counters=self.grid.counters, windows=windows,
                                     device=getattr(getattr(backend, "h", None), "device", None))
        else:
            raise ValueError(f"unknown combine backend {combine!r}")
        self.kry = DistKrylov(group, owned=getattr(backend, "owned", None), counters=self.grid.counters,
                              ctx=getattr(getattr(backend, "h", None), "ctx", None))
        backend.setup(self.lams[self.lo : self.hi], self.tau)

    def A_op(self, k):
        """mask (Ainv M (mask k) + tau K (mask k)) + (1 - mask) k, own stages."""
        mk, kk = self.be.mass_stiff(k)
        v = self.ring(self.Ainv, mk) + self.tau * kk
        return self.be.boundary_identity(v, k)

    def P_op(self, r):
        w = self.ring(self.Sinv, r)
        z = self.be.vcycle(w)
        return self.ring(self.S, z)

    def step(self, t_n, u_n):
        w = self.be.stage_rhs(t_n, u_n, self.c[self.lo : self.hi] * self.tau)  # (own, n): F_j - K u_n
        rhs = self.be.mask(self.ring(self.Ainv, w))
        k, its, hist, conv = self.kry.solve(self.A_op, self.P_op, rhs, self.rel_tol, self.max_iter)
        # u_{n+1} = u_n + tau sum_i b_i k_i: partial sum over own stages, all-reduced
        part = self.tau * torch.einsum("i,in->n", torch.as_tensor(self.b[self.lo : self.hi], dtype=k.dtype,
                                                                  device=k.device), k)
        if self.grid.S > 1:
            all_reduce_sum(part, self.row_group, self.grid.counters)
        return u_n + part, its, conv


class GPUStageBackend:
    """Stage-local device operators for StageParallelStepper (one GPU per rank)."""

    def __init__(self, hierarchy, config=None, source=None):
        from .fem import SeparableSolution
        from .multigrid import VCycleConfig

        self.h = hierarchy
        self.L = hierarchy.max_level
        self.config = config or VCycleConfig()
        self.source = source or SeparableSolution(hierarchy.dim)

    def setup(self, lams, tau):
        from .multigrid import MultiBlockSolver

        self.tau = tau
        self.solver = MultiBlockSolver(self.h, lams, tau, self.config) if len(lams) else None
        self.g1 = torch.from_numpy(self.h.load_vector_1d(self.L, self.source.s)).to(self.h.device)
        self.maskt = self.h.mask_tensor(self.L)

    def mass_stiff(self, k):
        km = torch.where(self.maskt, k, torch.zeros_like(k))
        return (self.h.apply_block(self.L, 1.0, 0.0, km), self.h.apply_block(self.L, 0.0, 1.0, km))

    def boundary_identity(self, v, k):
        return torch.where(self.maskt, v, k)

    def mask(self, v):
        return torch.where(self.maskt, v, torch.zeros_like(v))

    def vcycle(self, w):
        return self.solver.apply_device(w.contiguous(), check=False)

    def stage_rhs(self, t_n, u_n, ctau):
        """w_j = F(t_n + c_j tau) - K (mask u_n) for the own stages, one spk_rhs launch (identity mix:
        masking w here does not change mask * (A^-1 w), which the stepper forms next)."""
        um = torch.where(self.maskt, u_n, torch.zeros_like(u_n)).reshape(1, -1)
        self._exchange_rhs(um)
        ku = self.h.apply_block(self.L, 0.0, 1.0, um)
        return self._rhs(t_n, ctau, ku, u_n)

    def _exchange_rhs(self, um):
        pass

    def _rhs(self, t_n, ctau, ku, u_n):
        from . import _lib
        from ._device import ptr, stream_ptr
        q = len(ctau)
        out = torch.empty((q, u_n.numel()), dtype=torch.float64, device=u_n.device)
        if q == 0:
            return out
        T = _lib.dbl_array([self.source.F(t_n + ct) for ct in ctau])
        eye = np.ascontiguousarray(np.eye(q))
        _lib.call("spk_rhs", self.h.ctx, self.L, q, ptr(self.g1), T, eye.ctypes.data_as(_lib.P_dbl), ptr(ku),
                  ptr(out), stream_ptr(self.h.device))
        return out


class GPUSlabStageBackend(GPUStageBackend):
    """Stage-local device operators on an x-slab of the mesh (B > 1): halo exchange on the column
    group before each operator application, distributed V-cycles (slab.DistMultiBlockSolver), dots
    over the owned planes only."""

    def __init__(self, slab_hierarchy, config=None, source=None):
        super().__init__(slab_hierarchy, config, source)
        self.part = slab_hierarchy.part
        self.win = slab_hierarchy.window(self.L)

    def setup(self, lams, tau):
        from .slab import DistMultiBlockSolver

        self.tau = tau
        self.solver = DistMultiBlockSolver(self.h, lams, tau, self.config) if len(lams) else None
        self.g1 = torch.from_numpy(self.h.load_vector_1d(self.L, self.source.s)).to(self.h.device)
        self.maskt = self.h.mask_tensor(self.L)

    def owned(self, v):
        return self.win.owned(v)

    def mass_stiff(self, k):
        km = torch.where(self.maskt, k, torch.zeros_like(k))
        self.part.exchange(km, self.L)
        return (self.h.apply_block(self.L, 1.0, 0.0, km), self.h.apply_block(self.L, 0.0, 1.0, km))

    def _exchange_rhs(self, um):
        self.part.exchange(um, self.L)


class DirectComplexParallelStepper:
    """eq. irk:Ainv with the conjugate-pair blocks distributed over ranks (SPEC complex_solver
    stage-pair parallelism): w = S^-1 rhs and k = S z are ring combines between the stage groups and
    the pair groups; each rank solves its own pair blocks (GMRES on the real 2x2 form with PRESB or
    the 2x2 GMG V-cycle; the odd-Q real eigenvalue with the plain V-cycle) with no further traffic."""

    def __init__(self, backend, Q, tau, rank, world, group=None, tableau=None, variant="presb",
                 rel_tol=1e-12, max_iter=200):
        from .tableau import spectral_complex
        from .tensor_ops import paired_back_matrix, paired_forward_matrix

        self.be, self.Q, self.tau, self.rank, self.world = backend, Q, float(tau), rank, world
        self.rel_tol, self.max_iter = rel_tol, max_iter
        tab = tableau if tableau is not None else radau_iia(Q)
        get = lambda t, k: np.asarray(t[k] if isinstance(t, dict) else getattr(t, k))
        self.b, self.c, self.Ainv = get(tab, "b"), get(tab, "c"), get(tab, "Ainv")
        sp = spectral_complex(self.Ainv)
        self.pairs = sp.pairs
        self.Wf = paired_forward_matrix(sp.Sinv, sp.pairs)
        self.Wb = paired_back_matrix(sp.S, sp.pairs)
        P = len(sp.pairs)
        self.groups = stage_groups(Q, world)
        pg = stage_groups(P, world)
        self.pair_groups = pg
        self.row_groups = [(2 * a, 2 * b) for a, b in pg]
        self.lo, self.hi = self.groups[rank]
        self.ring = RingCombiner(self.groups, rank, world, group)
        self.group = group
        own = [self.pairs[i] for i in range(*pg[rank])]
        backend.setup_pairs(own, self.tau, variant)

    def step(self, t_n, u_n):
        w = self.be.stage_rhs(t_n, u_n, self.c[self.lo : self.hi] * self.tau)
        rhs = self.be.mask(self.ring(self.Ainv, w))
        wp = self.ring(self.Wf, rhs, in_groups=self.groups, out_groups=self.row_groups)
        z = torch.zeros_like(wp)
        its = []
        for i in range(wp.shape[0] // 2):
            zi, k = self.be.solve_pair(i, wp[2 * i : 2 * i + 2])
            z[2 * i : 2 * i + 2] = zi
            its.append(k)
        kst = self.ring(self.Wb, z, in_groups=self.row_groups, out_groups=self.groups)
        part = self.tau * torch.einsum("i,in->n", torch.as_tensor(self.b[self.lo : self.hi], dtype=kst.dtype,
                                                                  device=kst.device), kst)
        if self.world > 1:
            all_reduce_sum(part, self.group)
        return u_n + part, its


def _gpu_setup_pairs(self, own_pairs, tau, variant):
    """Pair-block solvers for DirectComplexParallelStepper (GPUStageBackend extension)."""
    from .multigrid import BlockSolver, PairBlockSolver

    self.tau = tau
    self.g1 = torch.from_numpy(self.h.load_vector_1d(self.L, self.source.s)).to(self.h.device)
    self.maskt = self.h.mask_tensor(self.L)
    self.pair_blocks = []
    for p in own_pairs:
        if p.is_real:
            self.pair_blocks.append(("real", p, BlockSolver(self.h, p.re, tau, self.config)))
        elif variant == "presb":
            self.pair_blocks.append(("presb", p, BlockSolver(self.h, p.re + p.im, tau, self.config)))
        else:
            self.pair_blocks.append(("gmg", p, PairBlockSolver(self.h, p.re, p.im, tau, self.config)))


def _gpu_solve_pair(self, i, rows):
    """GMRES on the real 2x2 form of pair block i (rows: (2, n) re/im right-hand side)."""
    from . import _lib
    from ._device import ptr, stream_ptr
    from .krylov import gmres

    kind, p, vc = self.pair_blocks[i]
    h, L = self.h, self.L
    if kind == "real":
        op = lambda v: h.apply_block(L, p.re, self.tau, v.reshape(1, -1), constrained=True).reshape(v.shape)
        pc = lambda v: vc.apply_device(v.reshape(1, -1), check=False).reshape(v.shape)
        z, rep = gmres(op, pc, rows[0].contiguous(), self.rel_tol, self.max_iter)
        out = torch.zeros_like(rows)
        out[0] = z
        return out, rep.iterations

    def op(v):
        v = v.contiguous()
        w = torch.empty_like(v)
        _lib.call("spk_pair_apply", h.ctx, L, p.re, p.im, self.tau, 1, ptr(v), ptr(w), stream_ptr(h.device))
        return w

    if kind == "presb":
        def pc(r):
            y1 = vc.apply_device((r[0] + r[1]).reshape(1, -1), check=False)
            y2 = vc.apply_device(r[1].reshape(1, -1) - h.apply_block(L, p.im, 0.0, y1, constrained=True),
                                 check=False)
            return torch.cat([y1 - y2, y2], dim=0)
    else:
        pc = lambda r: vc.apply_device(r.contiguous(), check=False)
    z, rep = gmres(op, pc, rows.contiguous(), self.rel_tol, self.max_iter)
    return z, rep.iterations


GPUStageBackend.setup_pairs = _gpu_setup_pairs
GPUStageBackend.solve_pair = _gpu_solve_pair
GPUStageBackend.rel_tol = 1e-12
GPUStageBackend.max_iter = 200
