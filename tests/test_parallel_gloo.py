"""Multi-rank host logic of parallel.py on CPU with the gloo backend (world sizes 2 and 4):
halo exchange of the x-slab partition and the Cannon-like stage rotation."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _halo_worker(rank, world, port, q, errs):
    from paper_2209_06700_b200.parallel import SlabLayout, exchange_halo

    _init(rank, world, port)
    try:
        k, E, plane, Q = 2, 3, 5, 2
        lay = SlabLayout(k, E, plane, world, rank)
        buf = torch.full((Q, lay.local_numel), -1.0, dtype=torch.float64)
        # owned planes carry (global plane index * 100 + stage * 10 + rank) in every slot
        for p in range(lay.n_owned_planes):
            gp = rank * k * E + p
            for qq in range(Q):
                buf[qq, lay.plane_slice(k + p, k + p + 1)] = gp * 100 + qq * 10
        exchange_halo(buf, lay)
        for qq in range(Q):
            if rank > 0:
                for h in range(k):
                    gp = rank * k * E - k + h
                    got = buf[qq, lay.plane_slice(h, h + 1)]
                    assert torch.all(got == gp * 100 + qq * 10), (rank, h, got[0])
            if rank + 1 < world:
                gp = (rank + 1) * k * E
                got = buf[qq, lay.plane_slice(k + k * E, k + k * E + 1)]
                assert torch.all(got == gp * 100 + qq * 10)
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(f"rank {rank}: {e!r}")
    finally:
        dist.destroy_process_group()


def _rotate_worker(rank, world, port, q, errs):
    from paper_2209_06700_b200.parallel import rotate_combine

    _init(rank, world, port)
    try:
        Q, n = world, 50
        rng = np.random.default_rng(7)
        D = rng.standard_normal((Q, Q))
        U = rng.standard_normal((Q, n))
        counters = {}
        out = rotate_combine(D, torch.from_numpy(U[rank].copy()), rank, Q, counters=counters)
        ref = D @ U
        err = float(np.abs(out.numpy() - ref[rank]).max() / np.abs(ref).max())
        assert err < 1e-13, err
        assert counters["shift_rounds"] == Q - 1
    except Exception as e:  # pragma: no cover
        q.put(f"rank {rank}: {e!r}")
    finally:
        dist.destroy_process_group()


def _run(fn, world):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, world, port, q, None)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    errs = []
    while not q.empty():
        errs.append(q.get())
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs)


@pytest.mark.parametrize("world", [2, 4])
def test_halo_exchange_gloo(world):
    _run(_halo_worker, world)


@pytest.mark.parametrize("world", [2, 4])
def test_rotate_combine_gloo(world):
    _run(_rotate_worker, world)
