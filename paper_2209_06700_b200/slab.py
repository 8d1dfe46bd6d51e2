"""Mesh partition inside a stage group: x-slabs of whole elements on B ranks (the
spatial partition b of rank (q, b); SPEC RankGrid SPEC.md:303-318), with a distributed V-cycle.

Layout of a distributed level l (2^l elements per axis, E = 2^l / B per rank, partition b owns
elements [e0, e0 + E), e0 = b E): the local arrays hold the planes of elements [e0 - 2, e0 + E), i.e.
K (E + 2) + 1 x-planes whose plane 0 is global plane K (e0 - 2):

    [ 2K halo planes | K E owned planes | 1 plane: right halo, or the global boundary on the last slab ]

On the first slab the 2K halo planes are padding (global planes < 0, never produced or read as
data). Two halo elements on the left are what the restriction P^T needs (a coarse vertex gathers
the fine nodes of both adjacent coarse elements = 2 fine elements); the operator needs one. The
kernels see the window through `spk_ctx_set_slab` and compute boundary rows, Jacobi classes and
sources at global positions, so every entry point produces exactly the owned nodes of the global
operation (bit-identical per node to the whole-mesh launch).

Halo planes are refreshed (`SlabPartition.exchange`, grouped isend/irecv on the column group) before
every operator application and transfer that reads them. Levels with fewer than `min_elems`
elements per slab are not partitioned: at the coarsest distributed level the residual is
all-gathered over the column group and every rank runs the rest of the V-cycle redundantly on a
whole-mesh replica hierarchy (identical arithmetic on every rank, no further traffic), then keeps
its owned planes of the prolongated correction.
"""

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from ._device import ptr, stream_ptr
from .errors import ConfigurationError, SpectralFailureError
from .fem import GridHierarchy
from .multigrid import MultiBlockSolver, VCycleConfig, _BlockFamily, _Level, _POWER_SEED
from .runtime import Counters, all_reduce_sum


@dataclass(frozen=True)
class SlabWindow:
    level: int
    k: int
    nax: int        # nodes per axis of the global level
    E: int          # owned elements along x
    e0: int         # first owned element (global)
    last: bool      # owns the global boundary plane x = 1

    @property
    def x_elems(self):
        return self.E + 2

    @property
    def x0(self):
        """global plane index of local plane 0 (negative on the first slab)"""
        return self.k * (self.e0 - 2)

    @property
    def nplanes(self):
        return self.k * self.x_elems + 1

    @property
    def plane(self):
        return self.nax * self.nax

    @property
    def local_numel(self):
        return self.nplanes * self.plane

    @property
    def n_owned_planes(self):
        return self.k * self.E + (1 if self.last else 0)

    @property
    def owned_planes(self):
        """local plane range of the owned nodes"""
        return 2 * self.k, 2 * self.k + self.n_owned_planes

    @property
    def global_owned_planes(self):
        return self.k * self.e0, self.k * self.e0 + self.n_owned_planes

    def owned(self, v):
        """view of the owned nodes of a (rows, local_numel) buffer: (rows, n_owned_planes * plane)"""
        a, b = self.owned_planes
        return v[..., a * self.plane : b * self.plane]

    def interior_mask(self, device):
        """bool (local_numel,) True on owned-or-halo nodes that are interior in the global mesh"""
        gx = self.x0 + torch.arange(self.nplanes, device=device)
        mx = (gx > 0) & (gx < self.nax - 1)
        r = torch.arange(self.nax, device=device)
        my = (r > 0) & (r < self.nax - 1)
        return (mx[:, None, None] & my[None, :, None] & my[None, None, :]).reshape(-1)


class SlabPartition:
    """Per-level windows of partition b out of B (B a power of two) and the halo / gather
    exchanges on the column group (`ranks`: global ranks of partitions 0..B-1 of this stage group)."""

    def __init__(self, k, max_level, B, b, ranks=None, group=None, min_elems=2, counters=None):
        if B < 1 or B & (B - 1):
            raise ConfigurationError(f"number of slabs must be a power of two, got {B}")
        if not 0 <= b < B:
            raise ConfigurationError(f"slab index {b} outside [0, {B})")
        self.k, self.max_level, self.B, self.b = k, max_level, B, b
        self.ranks = list(ranks) if ranks is not None else list(range(B))
        self.group = group
        self.counters = counters if counters is not None else Counters()
        self.dist_levels = [l for l in range(max_level + 1) if (1 << l) >= B * min_elems]
        if max_level not in self.dist_levels:
            raise ConfigurationError(f"level {max_level} has fewer than {min_elems} elements per slab "
                                     f"with {B} slabs")
        self.gather_level = min(self.dist_levels)

    def window(self, level):
        E = (1 << level) // self.B
        return SlabWindow(level, self.k, self.k * (1 << level) + 1, E, self.b * E, self.b == self.B - 1)

    def apply_windows(self, ctx):
        """Install the windows of the distributed levels into a libspk context."""
        for l in self.dist_levels:
            w = self.window(l)
            _lib.call("spk_ctx_set_slab", ctx, l, w.x_elems, w.x0, 2, w.x_elems, 1 if w.last else 0)

    # ---- exchanges on the column group ----
    def _wire(self, t):
        return t.cpu() if (t.is_cuda and dist.get_backend(self.group) == "gloo") else t.contiguous()

    def exchange(self, buf, level):
        """Refresh the halo planes of buf (rows, local_numel) at a distributed level: the left
        neighbour's last 2K owned planes and the right neighbour's first owned plane."""
        if self.B == 1:
            return 0
        w = self.window(level)
        k, P = self.k, w.plane
        rows = buf.reshape(-1, w.local_numel)
        ops, recvs = [], []
        host = rows.is_cuda and dist.get_backend(self.group) == "gloo"
        dev = "cpu" if host else rows.device
        if self.b + 1 < self.B:  # right neighbour
            peer = self.ranks[self.b + 1]
            s = self._wire(rows[:, (k * w.E) * P : (k * w.E + 2 * k) * P])
            ops.append(dist.P2POp(dist.isend, s, peer, self.group))
            self.counters.add_send(s)
            r = torch.empty((rows.shape[0], P), dtype=rows.dtype, device=dev)
            ops.append(dist.P2POp(dist.irecv, r, peer, self.group))
            recvs.append((slice((w.nplanes - 1) * P, w.nplanes * P), r))
        if self.b > 0:  # left neighbour
            peer = self.ranks[self.b - 1]
            s = self._wire(rows[:, 2 * k * P : (2 * k + 1) * P])
            ops.append(dist.P2POp(dist.isend, s, peer, self.group))
            self.counters.add_send(s)
            r = torch.empty((rows.shape[0], 2 * k * P), dtype=rows.dtype, device=dev)
            ops.append(dist.P2POp(dist.irecv, r, peer, self.group))
            recvs.append((slice(0, 2 * k * P), r))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        for sl, r in recvs:
            rows[:, sl].copy_(r)
        self.counters.halo_exchanges += 1
        return len(ops)

    def gather(self, buf, level):
        """All-gather the owned planes of buf (rows, local_numel) into whole-level vectors
        (rows, nax^3) on every rank of the column group."""
        w = self.window(level)
        P, k, E = w.plane, self.k, w.E
        rows = buf.reshape(-1, w.local_numel)
        a = 2 * k
        # every slab sends K E + 1 planes (its owned planes + the next vertex plane; only the last
        # slab's copy of the global boundary plane is used)
        part = self._wire(rows[:, a * P : (a + k * E + 1) * P])
        if self.B == 1:
            parts = [part]
        else:
            parts = [torch.empty_like(part) for _ in range(self.B)]
            dist.all_gather(parts, part, group=self.group)
            self.counters.messages_sent += self.B - 1
            self.counters.bytes_sent += (self.B - 1) * part.numel() * part.element_size()
        full = torch.empty((rows.shape[0], w.nax * P), dtype=rows.dtype, device=rows.device)
        for bb, p in enumerate(parts):
            lo = k * E * bb
            cnt = k * E + (1 if bb == self.B - 1 else 0)
            full[:, lo * P : (lo + cnt) * P].copy_(p[:, : cnt * P])
        return full

    def scatter(self, full, level, out=None):
        """Local (rows, local_numel) buffer from whole-level vectors: owned + halo planes that
        exist in the global mesh (padding planes zero)."""
        w = self.window(level)
        P = w.plane
        full = full.reshape(-1, w.nax * P)
        if out is None:
            out = torch.zeros((full.shape[0], w.local_numel), dtype=full.dtype, device=full.device)
        g0 = max(w.x0, 0)
        g1 = min(w.x0 + w.nplanes, w.nax)
        out[:, (g0 - w.x0) * P : (g1 - w.x0) * P].copy_(full[:, g0 * P : g1 * P])
        return out


class SlabHierarchy(GridHierarchy):
    """GridHierarchy (3D) whose distributed levels are x-slab windows of partition b."""

    def __init__(self, max_level, degree, partition, device=None):
        super().__init__(3, max_level, degree, device)
        if partition.k != degree or partition.max_level != max_level:
            raise ConfigurationError("partition does not match the hierarchy")
        self.part = partition
        partition.apply_windows(self.ctx)
        self._wmasks = {}

    def local_numel(self, level):
        if level in self.part.dist_levels:
            return self.part.window(level).local_numel
        return self.levels[level].n_dofs

    def window(self, level):
        return self.part.window(level)

    def mask_tensor(self, level):
        if level not in self.part.dist_levels:
            return super().mask_tensor(level)
        if level not in self._wmasks:
            self._wmasks[level] = self.window(level).interior_mask(self.device)
        return self._wmasks[level]

    def _check(self, level, u):
        n = self.local_numel(level)
        if u.shape[-1] != n:
            from .errors import DimensionMismatchError
            raise DimensionMismatchError(f"level {level} slab expects {n} local DoFs, got {u.shape[-1]}")
        return self.levels[level]

    def prolong_into(self, coarse_level, uc, out, accumulate=False):
        nblk = uc.shape[0]
        nf = max(self.local_numel(coarse_level + 1), self.local_numel(coarse_level))
        scr = self.scratch(("transfer", nblk), 2 * nblk * nf)
        _lib.call("spk_transfer", self.ctx, coarse_level + 1, nblk, 1, ptr(uc), ptr(out), ptr(scr),
                  1 if accumulate else 0, 0, stream_ptr(self.device))
        return out

    def restrict_into(self, fine_level, rf, out, mask=False):
        nblk = rf.shape[0]
        nf = max(self.local_numel(fine_level), self.local_numel(fine_level - 1))
        scr = self.scratch(("transfer", nblk), 2 * nblk * nf)
        _lib.call("spk_transfer", self.ctx, fine_level, nblk, 0, ptr(rf), ptr(out), ptr(scr), 0,
                  1 if mask else 0, stream_ptr(self.device))
        return out

    def owned(self, level, v):
        if level not in self.part.dist_levels:
            return v
        return self.window(level).owned(v)


class DistMultiBlockSolver(_BlockFamily):
    """MultiBlockSolver (per-block Chebyshev coefficients, one V-cycle per stage block) on an x-slab
    partition: distributed levels exchange halos before every operator application; the levels
    at and below the coarsest distributed one run redundantly on a whole-mesh replica.

    lambda_max: levels at or below the gather level come from the replica (the same global
    operator and start vector); finer levels run the power iteration on the slabs with the norms
    all-reduced over the column group (sqrt of the summed squares)."""

    _fuse_coarse = False  # windowed levels: the replica coarse cycle (self.rep) fuses instead

    def __init__(self, slab_h, lams, tau, config=None):
        self.part = slab_h.part
        self.rep = MultiBlockSolver(GridHierarchy(3, self.part.gather_level, slab_h.degree, slab_h.device),
                                    lams, tau, config)
        super().__init__(slab_h, lams, tau, config, self.part.gather_level, shared=False)

    # ---- lambda_max ----
    def _estimate(self, level, lam):
        if level <= self.part.gather_level:
            ests = self.rep.lambda_max[level]
            i = list(self.rep.lams).index(lam)
            return ests[i] if isinstance(ests, list) else ests
        h, part = self.hierarchy, self.part
        w = part.window(level)
        if not hasattr(self, "_v0"):
            self._v0 = {}
        if level not in self._v0:
            v0 = np.random.default_rng(_POWER_SEED).standard_normal(w.nax ** 3)
            v0 /= np.linalg.norm(v0)
            self._v0[level] = part.scatter(torch.from_numpy(v0).to(h.device), level)[0]
        v = self._v0[level].clone()
        wv = torch.zeros_like(v)
        ests = torch.zeros(self.config.eig_iters, dtype=torch.float64, device=h.device)
        st = stream_ptr(h.device)
        for it in range(self.config.eig_iters):
            part.exchange(v, level)
            est = ests[it : it + 1]
            _lib.call("spk_dinv_norm", h.ctx, level, 0, float(lam), 0.0, self.tau, ptr(v), ptr(wv), ptr(est), st)
            sq = est * est
            all_reduce_sum(sq, part.group, part.counters)
            est.copy_(torch.sqrt(sq))
            _lib.call("spk_scale_div", v.numel(), ptr(wv), ptr(est), ptr(v), st)
        e = ests.cpu().numpy()
        for x in e:
            if not np.isfinite(x) or x <= 0.0:
                raise SpectralFailureError(f"power iteration produced estimate {x}")
        return float(e[-1]) * self.config.eig_safety

    # ---- engine hooks ----
    def _halo(self, level, t):
        if level in self.part.dist_levels:
            self.part.exchange(t, level)

    def _ensure(self):
        if self._bufs is not None:
            return
        h = self.hierarchy
        self._bufs = {}
        for level in range(self.min_level, h.max_level + 1):
            self._bufs[level] = _Level(self.nrows, h.local_numel(level), h.device, level < h.max_level)
        self._flags = torch.zeros(h.max_level + 1, dtype=torch.int32, device=h.device)

    def _coarse(self, b):
        raise AssertionError("the distributed cycle hands the coarse part to the replica")

    def _cycle(self, level, b):
        lv = self._bufs[level]
        self._smooth(level, b, lv, zero_start=True)
        if level > self.part.gather_level:
            self._residual_restrict(level, b, lv)
            ec = self._cycle(level - 1, self._bufs[level - 1].b)
            self._halo(level - 1, ec)
            self.hierarchy.prolong_into(level - 1, ec, lv.x, accumulate=True)
        else:
            # gather level: whole-level residual on every rank, replica V-cycle below it
            self._halo(level, lv.x)
            _lib.call("spk_residual", self.hierarchy.ctx, level, self.nrows, _lib.dbl_array(self._block_lams()),
                      self.tau, ptr(lv.x), ptr(b), ptr(lv.r), None, None, stream_ptr(self.hierarchy.device))
            rep, rh = self.rep, self.rep.hierarchy
            rep._ensure()
            r_full = self.part.gather(lv.r, level)
            if level == 0:
                raise ConfigurationError("gather level 0 has no coarser level")
            rh.restrict_into(level, r_full, rep._bufs[level - 1].b, mask=True)
            ec = rep._cycle(level - 1, rep._bufs[level - 1].b)
            e_full = torch.zeros_like(r_full)
            rh.prolong_into(level - 1, ec, e_full)
            w = self.part.window(level)
            e_loc = self.part.scatter(e_full, level)
            w.owned(lv.x).add_(w.owned(e_loc))
        self._smooth(level, b, lv, zero_start=False)
        return lv.x

    def apply_device(self, b, out=None, check=True):
        self.rep._ensure()
        self.rep._flags.zero_()
        return super().apply_device(b, out, check)

    def check_finite(self):
        super().check_finite()
        self.rep.check_finite()
