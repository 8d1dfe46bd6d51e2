"""Rank grid (SPEC runtime) and the x-slab halo / gather exchanges on CPU with gloo."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2209_06700_b200.errors import ConfigurationError
from paper_2209_06700_b200.runtime import RankGrid, stage_groups
from paper_2209_06700_b200.slab import SlabPartition


def test_rank_grid_mappings():
    # SPEC create_rank_grid examples
    g = RankGrid(6, 4, "row_major")
    assert g.rank_of(1, 2) == 6  # stage 2, partition 3 (1-based) -> rank 6
    g = RankGrid(2, 3, "column_major")
    assert [g.rank_of(0, 0), g.rank_of(1, 0), g.rank_of(0, 1)] == [0, 1, 2]
    g = RankGrid(4, 3, "row_major_padded", node_size=4)
    for s in range(4):
        ranks = g.row_ranks(0)
        assert g.col_ranks(s) == [4 * s, 4 * s + 1, 4 * s + 2]
        assert all(r // 4 == s for r in g.col_ranks(s))  # a stage group never straddles a node
    assert g.coords(3) is None and g.size == 16  # idle padding rank
    for topo in ("row_major", "column_major"):
        g = RankGrid(3, 4, topo)
        ranks = sorted(g.rank_of(s, b) for s in range(3) for b in range(4))
        assert ranks == list(range(12))  # bijection
        for r in range(12):
            s, b = g.coords(r)
            assert g.rank_of(s, b) == r and r in g.row_ranks(b) and r in g.col_ranks(s)
    with pytest.raises(ConfigurationError):
        RankGrid(2, 3, "row_major_padded", node_size=2)
    with pytest.raises(ConfigurationError):
        RankGrid(2, 2, "hexagonal")


def test_stage_groups():
    assert stage_groups(4, 2) == [(0, 2), (2, 4)]
    assert stage_groups(3, 2) == [(0, 2), (2, 3)]
    assert stage_groups(3, 3) == [(0, 1), (1, 2), (2, 3)]


def test_slab_windows_tile_the_mesh():
    for k, L, B in [(1, 4, 4), (2, 3, 2), (4, 5, 8), (3, 3, 4)]:
        covered = []
        for b in range(B):
            part = SlabPartition(k, L, B, b)
            for level in part.dist_levels:
                w = part.window(level)
                assert w.x0 == k * (w.e0 - 2) and w.nplanes == k * (w.E + 2) + 1
                if level == L:
                    covered.extend(range(*w.global_owned_planes))
            assert part.gather_level == min(part.dist_levels) and (1 << part.gather_level) >= 2 * B
        assert covered == list(range(k * (1 << L) + 1))  # owned planes partition the global planes
    with pytest.raises(ConfigurationError):
        SlabPartition(2, 3, 3, 0)  # not a power of two
    with pytest.raises(ConfigurationError):
        SlabPartition(2, 2, 4, 0)  # finest level too coarse for 4 slabs


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        # grid 2 x 2 (world 4): groups and counters
        grid = RankGrid(2, world // 2, "column_major").init_groups()
        s, b = grid.coords(rank)
        k, L, B = 2, 3, world // 2
        part = SlabPartition(k, L, B, b, ranks=grid.col_ranks(s), group=grid.col_group(s),
                             counters=grid.counters)
        for level in part.dist_levels:
            w = part.window(level)
            nax = w.nax
            full = torch.arange(3 * nax ** 3, dtype=torch.float64).reshape(3, -1) * (1 + s)
            loc = torch.full((3, w.local_numel), -1.0, dtype=torch.float64)
            # fill owned planes only, then exchange: every non-padding plane must equal the global one
            ref = part.scatter(full, level)
            w.owned(loc).copy_(w.owned(ref))
            part.exchange(loc, level)
            g0 = max(w.x0, 0)
            ok = torch.equal(loc[:, (g0 - w.x0) * w.plane :], ref[:, (g0 - w.x0) * w.plane :])
            out[("halo", level)] = ok
            out[("gather", level)] = torch.equal(part.gather(loc, level), full)
        csv_text = grid.gather_csv(rank, world)
        q.put((rank, out, csv_text, grid.snapshot(rank)))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc(), None, None))
    finally:
        dist.destroy_process_group()


def test_slab_exchange_and_counters_gloo():
    world = 4
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get() for _ in range(world)]
    for p in procs:
        p.join(120)
    for rank, out, csv_text, snap in res:
        assert isinstance(out, dict), out
        assert all(out.values()), (rank, out)
        assert snap["halo_exchanges"] == 2 and snap["messages"] > 0  # 2 distributed levels
        if rank == 0:
            lines = csv_text.strip().splitlines()
            assert lines[0].startswith("rank,q,b,messages,bytes,barriers,shift_rounds")
            assert len(lines) == world + 1
