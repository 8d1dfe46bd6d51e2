"""Multi-GPU layouts of the stage-parallel method (one process per GPU, torch.distributed/NCCL).

* Mesh partitioning (the paper's spatial partition inside a stage group): x-slabs of
  whole elements. A slab needs one element of halo planes from its left neighbour and one vertex
  plane from its right neighbour; `exchange_halo` moves them with grouped point-to-point sends.
* Stage partitioning (SPEC RankGrid): rank (q, b) = q*B + b holds stage q of
  partition b; the stage combine (D (x) I) u is the Cannon-like rotation of PAPER.md:481-548
  (`rotate_combine`): Q rounds, Q-1 ring shifts of the held source block on the row group.

The host logic (plane bookkeeping, ring schedule) is backend-agnostic and is exercised with gloo on
CPU tensors in tests/test_parallel_gloo.py; on the GPU path the same calls run over NCCL.
"""

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from ._device import ptr, stream_ptr


# ----------------------------------------------------------------------------------------------
# x-slab mesh partition
# ----------------------------------------------------------------------------------------------
class SlabLayout:
    """Owned planes of rank r in a global mesh of world*E elements along x (degree k).

    Local buffer planes: [0, k) left halo | [k, k + k*E) owned | k + k*E right halo (or, on the
    last rank, its own global boundary plane).
    """

    def __init__(self, k, E, plane, world, rank):
        self.k, self.E, self.plane, self.world, self.rank = k, E, plane, world, rank
        self.nplanes = k * (E + 1) + 1
        self.first = k
        self.n_owned_planes = k * E + (1 if rank == world - 1 else 0)

    @property
    def local_numel(self):
        return self.nplanes * self.plane

    def owned_slice(self):
        return slice(self.first * self.plane, (self.first + self.n_owned_planes) * self.plane)

    def plane_slice(self, p0, p1):
        return slice(p0 * self.plane, p1 * self.plane)


def exchange_halo_start(buf, layout, group=None):
    """Post the halo exchange of buf (Q, local_numel) (grouped P2P; on NCCL the transfers run on
    the communicator's stream): right neighbour receives my last k owned planes into its left halo,
    left neighbour receives my first owned plane into its right halo plane. Returns the pending
    state for exchange_halo_finish."""
    k, E, r, W = layout.k, layout.E, layout.rank, layout.world
    ops = []
    recv_bufs = []
    Q = buf.shape[0]
    # gloo moves host memory only: stage device halos through the host (functional testing)
    host = buf.is_cuda and dist.get_backend(group) == "gloo"
    wire = (lambda t: t.cpu()) if host else (lambda t: t.contiguous())
    for q in range(Q):
        row = buf[q]
        if r + 1 < W:
            send = row[layout.plane_slice(k + k * E - k, k + k * E)]
            ops.append(dist.P2POp(dist.isend, wire(send), r + 1, group))
            rv = row[layout.plane_slice(k + k * E, k + k * E + 1)]
            tmp = torch.empty_like(rv, device="cpu" if host else rv.device)
            recv_bufs.append((rv, tmp))
            ops.append(dist.P2POp(dist.irecv, tmp, r + 1, group))
        if r > 0:
            send = row[layout.plane_slice(k, k + 1)]
            ops.append(dist.P2POp(dist.isend, wire(send), r - 1, group))
            lv = row[layout.plane_slice(0, k)]
            tmp = torch.empty_like(lv, device="cpu" if host else lv.device)
            recv_bufs.append((lv, tmp))
            ops.append(dist.P2POp(dist.irecv, tmp, r - 1, group))
    reqs = dist.batch_isend_irecv(ops) if ops else []
    return reqs, recv_bufs, len(ops)


def exchange_halo_finish(pending):
    """Wait for the posted exchange (stream-ordered on NCCL) and write the received halo planes."""
    reqs, recv_bufs, nops = pending
    for req in reqs:
        req.wait()
    for dst, tmp in recv_bufs:
        dst.copy_(tmp)
    return nops


def exchange_halo(buf, layout, group=None):
    """Blocking form: fill the halo planes of buf (Q, local_numel) from the neighbouring ranks."""
    return exchange_halo_finish(exchange_halo_start(buf, layout, group))


class SlabOperator:
    """K1 on an x-slab of a world*E x E x E element mesh. An apply posts the halo exchange, runs K1
    on the interior elements (they read owned planes only) while the planes are in flight, then the
    two edge elements once the halos have landed: the exchange overlaps the bulk of the operator.
    Every node is produced with the same arithmetic as one launch over the whole slab."""

    def __init__(self, hier, level, DM, DK, world, rank, group=None):
        if hier.dim != 3:
            raise ValueError("slab partitioning is implemented for 3D")
        self.hier, self.level = hier, level
        self.DM = np.ascontiguousarray(np.asarray(DM, dtype=float))
        self.DK = np.ascontiguousarray(np.asarray(DK, dtype=float))
        self.Q = self.DM.shape[0]
        lvl = hier.levels[level]
        self.k, self.E = hier.degree, lvl.n_elements
        self.plane = lvl.n_per_axis ** 2
        self.layout = SlabLayout(self.k, self.E, self.plane, world, rank)
        self.world, self.rank, self.group = world, rank, group
        self.overlap = self.E >= 4
        self.launches_per_apply = 3 if self.overlap else 1

    def alloc(self):
        n = self.layout.local_numel
        return (torch.zeros((self.Q, n), dtype=torch.float64, device=self.hier.device),
                torch.zeros((self.Q, n), dtype=torch.float64, device=self.hier.device))

    def apply(self, u, v):
        if not self.overlap:
            exchange_halo(u, self.layout, self.group)
            return self.launch(u, v)
        pending = exchange_halo_start(u, self.layout, self.group)
        eb, ee = self._range()
        self.launch(u, v, eb + 1, ee - 1)   # interior: planes K eb .. K (ee - 1), all owned
        exchange_halo_finish(pending)
        self.launch(u, v, eb, eb + 1)       # first owned element: reads the left halo element
        self.launch(u, v, ee - 1, ee)       # last one: reads the right halo plane
        return v

    def _range(self):
        return (0, self.E) if self.rank == 0 else (1, self.E + 1)

    def launch(self, u, v, eb=None, ee=None):
        """A windowed K1 launch over local elements [eb, ee) (default: the whole slab; halos
        already in place)."""
        lay = self.layout
        n = lay.local_numel
        if self.rank == 0:
            base_u = u[:, lay.plane_slice(self.k, lay.nplanes)]
            base_v = v[:, lay.plane_slice(self.k, lay.nplanes)]
            x_elems = self.E
        else:
            base_u, base_v = u, v
            x_elems = self.E + 1
        e0, e1 = self._range()
        eb = e0 if eb is None else eb
        ee = e1 if ee is None else ee
        store_last = 1 if (self.rank == self.world - 1 and ee == e1) else 0
        _lib.call("spk_stage_apply_slab", self.hier.ctx, self.level, self.Q,
                  self.DM.ctypes.data_as(_lib.P_dbl), self.DK.ctypes.data_as(_lib.P_dbl),
                  ptr(base_u), n, ptr(base_v), n, x_elems, eb, ee, store_last,
                  stream_ptr(self.hier.device))
        return v


# ----------------------------------------------------------------------------------------------
# stage partition: Cannon-like rotation of the stage combine
# ----------------------------------------------------------------------------------------------
def rotate_combine(D, u_local, q, Q, group=None, group_ranks=None, counters=None):
    """v_q = sum_j D[q, j] u_j on the row group holding one stage per rank.

    Round r adds D[q, (q+r) mod Q] * (held block), then the held block is shifted one rank "up"
    (received from q+1, sent to q-1); Q-1 shifts in total. Deterministic summation order (by round).
    """
    D = np.asarray(D)
    held = u_local.clone()
    out = torch.zeros_like(u_local)
    ranks = group_ranks if group_ranks is not None else list(range(Q))
    up, down = ranks[(q + 1) % Q], ranks[(q - 1) % Q]
    shifts = 0
    for r in range(Q):
        j = (q + r) % Q
        out.add_(held, alpha=float(D[q, j]))
        if r < Q - 1:
            nxt = torch.empty_like(held)
            ops = [dist.P2POp(dist.isend, held, down, group), dist.P2POp(dist.irecv, nxt, up, group)]
            for req in dist.batch_isend_irecv(ops):
                req.wait()
            held = nxt
            shifts += 1
    if counters is not None:
        counters["shift_rounds"] = counters.get("shift_rounds", 0) + shifts
    return out
