"""The stage-parallel data plane over NCCL on >= 2 GPUs (one process per GPU): the double-buffered
device ring combine (RingCombiner + spk_combine), the device-resident distributed GMRES dots
(DistKrylov + spk_mgs_partial + NCCL all-reduce) and the S x B stepper, against the single-GPU
StageSystem. Skips when fewer than 2 GPUs are visible (the round's GPU box has one); the same code
paths run over gloo in test_stage_parallel_gloo.py / test_slab_dist_gpu.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                                 reason="needs >= 2 GPUs for NCCL")]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _entry(rank, world, port, q, S, B):
    import traceback

    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        from oracle.tableau_ref import radau_iia
        from paper_2209_06700_b200.fem import build_hierarchy
        from paper_2209_06700_b200.irk import StageSystem
        from paper_2209_06700_b200.multigrid import VCycleConfig
        from paper_2209_06700_b200.runtime import RankGrid, stage_groups
        from paper_2209_06700_b200.slab import SlabHierarchy, SlabPartition
        from paper_2209_06700_b200.stage_parallel import (GPUSlabStageBackend, GPUStageBackend, RingCombiner,
                                                          StageParallelStepper)

        # ring combine with uneven groups (Q = 5 on world ranks)
        Q, n = 5, 1000
        X = torch.from_numpy(np.random.default_rng(3).standard_normal((Q, n))).to(dev)
        D = np.random.default_rng(4).standard_normal((Q, Q))
        groups = stage_groups(Q, world)
        lo, hi = groups[rank]
        got = RingCombiner(groups, rank, world)(D, X[lo:hi].contiguous())
        ring_err = float((got - torch.from_numpy(D).to(dev)[lo:hi] @ X).abs().max())

        k, L, Qs, tau = 2, 4, 4, 0.01
        cfg = VCycleConfig(smoother_degree=3)
        tab = radau_iia(Qs)
        grid = RankGrid(S, B).init_groups()
        s_idx, b_idx = grid.coords(rank)
        full = build_hierarchy(3, L, k, device=dev)
        ss = StageSystem(full, Qs, tau, config=cfg, tableau=tab)
        u_ref = ss.initial_condition()
        if B > 1:
            part = SlabPartition(k, L, B, b_idx, ranks=grid.col_ranks(s_idx), group=grid.col_group(s_idx),
                                 counters=grid.counters)
            be = GPUSlabStageBackend(SlabHierarchy(L, k, part, device=dev), cfg)
            u = part.scatter(u_ref.reshape(1, -1), L)[0]
        else:
            part = None
            be = GPUStageBackend(build_hierarchy(3, L, k, device=dev), cfg)
            u = u_ref.clone()
        sp = StageParallelStepper(be, Qs, tau, rank, world, tableau=tab, grid=grid)
        its = []
        for st in range(2):
            u_ref, rep = ss.step(st * tau, u_ref)
            u, k_it, conv = sp.step(st * tau, u)
            its.append((k_it, rep.iterations, conv))
        ug = part.gather(u.reshape(1, -1), L)[0] if part is not None else u
        err = float((ug - u_ref).abs().max() / u_ref.abs().max())
        q.put((rank, (ring_err, err, its)))
    except Exception:  # pragma: no cover
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("S,B", [(2, 1), (4, 1), (4, 2), (2, 2)])
def test_stage_parallel_over_nccl(S, B):
    world = S * B
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _port()
    procs = [ctx.Process(target=_entry, args=(r, world, port, q, S, B)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get() for _ in range(world))
    for p in procs:
        p.join(300)
    for r, v in res.items():
        assert not isinstance(v, str), f"rank {r}: {v}"
        ring_err, err, its = v
        assert ring_err < 1e-12
        assert err < 1e-9, (r, err)
        for k_it, k_ref, conv in its:
            assert conv and abs(k_it - k_ref) <= 1
