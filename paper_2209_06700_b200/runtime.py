"""Rank grid of the stage-parallel layout and its communication counters (SPEC runtime module,
SPEC.md:298-359, Fig. comm and the virtual topologies of §5.2).

N = S * B processes, one per GPU. Rank (s, b) holds stage group s (a contiguous range of the Q
stages, `stage_groups`) of mesh partition b (an x-slab of whole elements, `slab.SlabPartition`).

* row group of (s, b):    the S ranks sharing partition b  -> stage combines (ring), the update
* column group of (s, b): the B ranks sharing stage group s -> halo planes, lambda_max norms
* world:                  every rank                        -> GMRES inner products

Topologies map (s, b) to a global rank (SPEC create_rank_grid): ``row_major`` rank = s*B + b,
``column_major`` rank = b*S + s, ``row_major_padded`` = row-major with each stage group padded to
``node_size`` ranks so a group never straddles a node (idle ranks take part in world barriers only).
Results do not depend on the topology; only locality does.

`Counters` tracks messages / bytes / barriers / ring shift rounds per rank and writes the CSV of
SPEC.md:356 (rank, q, b, messages, bytes, barriers, shift_rounds).
"""

import csv
import io
from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from .errors import ConfigurationError

TOPOLOGIES = ("row_major", "column_major", "row_major_padded")


def stage_groups(Q, S):
    """Contiguous stage ranges per stage group (as equal as possible, larger groups first)."""
    if S < 1:
        raise ConfigurationError("need at least one stage group")
    base, extra = divmod(Q, S)
    out, s = [], 0
    for r in range(S):
        c = base + (1 if r < extra else 0)
        out.append((s, s + c))
        s += c
    return out


@dataclass
class Counters:
    messages_sent: int = 0
    bytes_sent: int = 0
    barrier_count: int = 0
    shift_rounds: int = 0
    halo_exchanges: int = 0
    allreduces: int = 0

    def add_send(self, t):
        self.messages_sent += 1
        self.bytes_sent += t.numel() * t.element_size()

    def as_dict(self):
        return dict(messages=self.messages_sent, bytes=self.bytes_sent, barriers=self.barrier_count,
                    shift_rounds=self.shift_rounds, halo_exchanges=self.halo_exchanges,
                    allreduces=self.allreduces)


@dataclass
class RankGrid:
    """(stage group, partition) <-> rank bijection and the three communicators."""

    S: int
    B: int
    topology: str = "row_major"
    node_size: int = 0
    counters: Counters = field(default_factory=Counters)

    def __post_init__(self):
        if self.S < 1 or self.B < 1:
            raise ConfigurationError("S and B must be >= 1")
        if self.topology not in TOPOLOGIES:
            raise ConfigurationError(f"unknown topology {self.topology!r}")
        if self.topology == "row_major_padded":
            if self.node_size < self.B:
                raise ConfigurationError("padded topology needs node_size >= B")
        self._groups = None

    # ---- mapping (SPEC create_rank_grid) ----
    @property
    def size(self):
        """ranks the mapping spans (padded topologies include idle ranks)"""
        if self.topology == "row_major_padded":
            return self.S * self.node_size
        return self.S * self.B

    def rank_of(self, s, b):
        if not (0 <= s < self.S and 0 <= b < self.B):
            raise ConfigurationError(f"(s, b) = ({s}, {b}) outside the {self.S} x {self.B} grid")
        if self.topology == "row_major":
            return s * self.B + b
        if self.topology == "column_major":
            return b * self.S + s
        return s * self.node_size + b

    def coords(self, rank):
        """(s, b) of a rank, or None for an idle (padding) rank."""
        for s in range(self.S):
            for b in range(self.B):
                if self.rank_of(s, b) == rank:
                    return s, b
        return None

    def row_ranks(self, b):
        """global ranks of partition b's stage groups, in stage-group order"""
        return [self.rank_of(s, b) for s in range(self.S)]

    def col_ranks(self, s):
        """global ranks of stage group s's partitions, in partition order"""
        return [self.rank_of(s, b) for b in range(self.B)]

    # ---- communicators ----
    def init_groups(self):
        """Create the row and column process groups (collective over the default group: every
        rank calls this in the same order). Returns self."""
        if self._groups is not None:
            return self
        rows = [dist.new_group(self.row_ranks(b)) if self.S > 1 else None for b in range(self.B)]
        cols = [dist.new_group(self.col_ranks(s)) if self.B > 1 else None for s in range(self.S)]
        self._groups = (rows, cols)
        return self

    def row_group(self, b):
        return self._groups[0][b] if self._groups else None

    def col_group(self, s):
        return self._groups[1][s] if self._groups else None

    def barrier(self, group=None):
        dist.barrier(group=group)
        self.counters.barrier_count += 1

    # ---- counters (SPEC CounterSnapshot, CSV of SPEC.md:356) ----
    def snapshot(self, rank):
        sb = self.coords(rank)
        q, b = sb if sb is not None else (-1, -1)
        return dict(rank=rank, q=q, b=b, **self.counters.as_dict())

    def gather_csv(self, rank, world):
        """Counter snapshots of every rank as CSV text (collective; rank 0 gets the text)."""
        snap = self.snapshot(rank)
        allv = [None] * world
        dist.all_gather_object(allv, snap)
        buf = io.StringIO()
        w = csv.DictWriter(buf, fieldnames=list(snap.keys()))
        w.writeheader()
        for row in allv:
            w.writerow(row)
        return buf.getvalue()


def host_staged(t, group):
    """gloo moves host memory only: the wire copy of t (a CPU clone when t is a CUDA tensor)."""
    if t.is_cuda and dist.get_backend(group) == "gloo":
        return t.cpu()
    return t.contiguous()


def all_reduce_sum(t, group=None, counters=None):
    """In-place sum all-reduce that also works for CUDA tensors over gloo (host staging)."""
    if counters is not None:
        counters.allreduces += 1
    if t.is_cuda and dist.get_backend(group) == "gloo":
        h = t.cpu()
        dist.all_reduce(h, group=group)
        t.copy_(h)
        return t
    dist.all_reduce(t, group=group)
    return t
