"""x-slab mesh partition on the device (B > 1): windowed kernels, distributed V-cycle and the
(S x B) stage-parallel stepper, against the whole-mesh device path (itself pinned to the oracle).

The ranks are processes sharing cuda:0 with gloo (host-staged halos and reductions): the kernels
never wait on one another (every exchange is a host-side rendezvous), so this checks the data
path of the multi-GPU layout on the single GPU the test box has.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(fn, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _port()
    procs = [ctx.Process(target=_entry, args=(fn, r, world, port, q, args)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, val = q.get()
        res[r] = val
    for p in procs:
        p.join(120)
    for r, v in res.items():
        assert not isinstance(v, str), f"rank {r}: {v}"
    return res


def _entry(fn, rank, world, port, q, args):
    import traceback

    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        q.put((rank, fn(rank, world, *args)))
    except Exception:  # pragma: no cover
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------------------------
def _ops_worker(rank, world, k, L):
    from paper_2209_06700_b200.fem import build_hierarchy
    from paper_2209_06700_b200.slab import SlabHierarchy, SlabPartition

    part = SlabPartition(k, L, world, rank)
    sh = SlabHierarchy(L, k, part, device="cuda:0")
    full = build_hierarchy(3, L, k, device="cuda:0")
    out = {}
    g = torch.Generator().manual_seed(7)
    lams = [1.7, 0.3]
    for level in part.dist_levels:
        n = full.levels[level].n_dofs
        u = torch.rand((2, n), generator=g, dtype=torch.float64).cuda()
        ul = part.scatter(u, level)
        for cons in (False, True):
            v_ref = full.apply_block(level, lams, 0.02, u, constrained=cons)
            ul_m = ul.clone()
            if not cons:  # unconstrained operator: apply to masked input (the stepper's use)
                m = sh.mask_tensor(level)
                ul_m = torch.where(m, ul_m, torch.zeros_like(ul_m))
                v_ref = full.apply_block(level, lams, 0.02, torch.where(full.mask_tensor(level), u,
                                                                        torch.zeros_like(u)))
            part.exchange(ul_m, level)
            v = sh.apply_block(level, lams, 0.02, ul_m, constrained=cons)
            out[(level, cons)] = float((part.gather(v, level) - v_ref).abs().max() / v_ref.abs().max())
        if level - 1 in part.dist_levels:
            # restriction and prolongation across slab boundaries
            uc = torch.rand((2, full.levels[level - 1].n_dofs), generator=g, dtype=torch.float64).cuda()
            r_ref = full.restrict(level, u)
            full.restrict_into(level, u, r_ref, mask=True)
            rc = torch.zeros((2, sh.local_numel(level - 1)), dtype=torch.float64, device="cuda:0")
            part.exchange(ul, level)
            sh.restrict_into(level, ul, rc, mask=True)
            out[(level, "R")] = float((part.gather(rc, level - 1) - r_ref).abs().max() / r_ref.abs().max())
            p_ref = full.prolong(level - 1, uc)
            ucl = part.scatter(uc, level - 1)
            part.exchange(ucl, level - 1)
            pf = torch.zeros((2, sh.local_numel(level)), dtype=torch.float64, device="cuda:0")
            sh.prolong_into(level - 1, ucl, pf)
            out[(level, "P")] = float((part.gather(pf, level) - p_ref).abs().max() / p_ref.abs().max())
    return out


@pytest.mark.parametrize("k,L,world", [(2, 3, 2), (4, 3, 2), (1, 4, 4), (3, 3, 2)])
def test_slab_operators_and_transfers(cuda, k, L, world):
    res = _run(_ops_worker, world, k, L)
    for r, errs in res.items():
        for key, e in errs.items():
            assert e <= 1e-14, (r, key, e)


# ---------------------------------------------------------------------------------------------
def _vcycle_worker(rank, world, k, L, deg, split=1 << 62):
    from paper_2209_06700_b200 import _lib
    from paper_2209_06700_b200.fem import build_hierarchy
    from paper_2209_06700_b200.multigrid import MultiBlockSolver, VCycleConfig
    from paper_2209_06700_b200.slab import DistMultiBlockSolver, SlabHierarchy, SlabPartition

    cfg = VCycleConfig(smoother_degree=deg)
    lams = [3.2, 2.1]
    part = SlabPartition(k, L, world, rank)
    sh = SlabHierarchy(L, k, part, device="cuda:0")
    _lib.call("spk_set_cheb_split", sh.ctx, split)  # 0: split Chebyshev steps on the slab windows
    full = build_hierarchy(3, L, k, device="cuda:0")
    ref = MultiBlockSolver(full, lams, 1e-2, cfg)
    dsv = DistMultiBlockSolver(sh, lams, 1e-2, cfg)
    lam_err = max(abs(np.asarray(dsv.lambda_max[l]) - np.asarray(ref.lambda_max[l])).max() /
                  np.abs(ref.lambda_max[l]).max() for l in range(part.gather_level, L + 1))
    b = torch.rand((2, full.n), generator=torch.Generator().manual_seed(3), dtype=torch.float64).cuda()
    x_ref = ref.apply_device(b)
    x = dsv.apply_device(part.scatter(b, L))
    xg = part.gather(x, L)
    return lam_err, float((xg - x_ref).abs().max() / x_ref.abs().max()), part.counters.halo_exchanges


@pytest.mark.parametrize("k,L,world,deg,split", [(2, 4, 2, 3, 1 << 62), (1, 4, 4, 5, 1 << 62), (4, 3, 2, 2, 1 << 62),
                                                 (2, 4, 2, 3, 0), (3, 3, 2, 5, 0)])
def test_distributed_vcycle_matches_whole_mesh(cuda, k, L, world, deg, split):
    res = _run(_vcycle_worker, world, k, L, deg, split)
    for r, (lam_err, err, nex) in res.items():
        assert lam_err < 1e-12, (r, lam_err)
        assert err < 1e-12, (r, err)
        assert nex > 0


# ---------------------------------------------------------------------------------------------
def _stepper_worker(rank, world, S, B, topology, combine="ring"):
    from oracle.tableau_ref import radau_iia
    from paper_2209_06700_b200.fem import build_hierarchy
    from paper_2209_06700_b200.irk import StageSystem
    from paper_2209_06700_b200.multigrid import VCycleConfig
    from paper_2209_06700_b200.runtime import RankGrid
    from paper_2209_06700_b200.slab import SlabHierarchy, SlabPartition
    from paper_2209_06700_b200.stage_parallel import GPUSlabStageBackend, StageParallelStepper

    k, L, Q, tau = 2, 3, 3, 0.01
    grid = RankGrid(S, B, topology).init_groups()
    s_idx, b_idx = grid.coords(rank)
    part = SlabPartition(k, L, B, b_idx, ranks=grid.col_ranks(s_idx), group=grid.col_group(s_idx),
                         counters=grid.counters)
    sh = SlabHierarchy(L, k, part, device="cuda:0")
    cfg = VCycleConfig(smoother_degree=3)
    tab = radau_iia(Q)
    sp = StageParallelStepper(GPUSlabStageBackend(sh, cfg), Q, tau, rank, world, tableau=tab, grid=grid,
                              combine=combine)
    ss = StageSystem(build_hierarchy(3, L, k, device="cuda:0"), Q, tau, config=cfg, tableau=tab)
    u_ref = ss.initial_condition()
    u = part.scatter(u_ref.reshape(1, -1), L)[0]
    its = []
    for st in range(2):
        u_ref, rep = ss.step(st * tau, u_ref)
        u, k_it, conv = sp.step(st * tau, u)
        its.append((k_it, rep.iterations, conv))
    ug = part.gather(u.reshape(1, -1), L)[0]
    if combine == "peer":
        sp.ring.close()
    return (float((ug - u_ref).abs().max() / u_ref.abs().max()), its, grid.snapshot(rank))


@pytest.mark.parametrize("S,B,topology,combine", [(1, 2, "row_major", "ring"), (3, 2, "row_major", "ring"),
                                                  (2, 2, "column_major", "ring"), (3, 1, "row_major", "peer"),
                                                  (2, 2, "row_major", "peer")])
def test_stage_parallel_slab_stepper(cuda, S, B, topology, combine):
    if B == 1:
        pytest.skip("B = 1 runs through the whole-mesh backend below")
    res = _run(_stepper_worker, S * B, S, B, topology, combine)
    for r, (err, its, snap) in res.items():
        assert err < 1e-9, (r, err)
        for k_it, k_ref, conv in its:
            assert conv and abs(k_it - k_ref) <= 1, its
        assert snap["halo_exchanges"] > 0
        if S > 1 and combine == "ring":
            assert snap["shift_rounds"] > 0 and snap["shift_rounds"] % (S - 1) == 0
        if combine == "peer":
            assert snap["shift_rounds"] == 0 and snap["barriers"] > 0


def _peer_worker(rank, world, Q):
    """B = 1, one stage group per rank: peer-window combines (CUDA IPC) vs the ring vs one GPU."""
    from oracle.tableau_ref import radau_iia
    from paper_2209_06700_b200.fem import build_hierarchy
    from paper_2209_06700_b200.irk import StageSystem
    from paper_2209_06700_b200.multigrid import VCycleConfig
    from paper_2209_06700_b200.stage_parallel import (GPUStageBackend, PeerCombiner, RingCombiner,
                                                      StageParallelStepper, stage_groups)

    h = build_hierarchy(3, 3, 2, device="cuda:0")
    cfg = VCycleConfig(smoother_degree=3)
    tab = radau_iia(Q)
    # raw combines: random D, x
    groups = stage_groups(Q, world)
    lo, hi = groups[rank]
    g = torch.Generator().manual_seed(11)
    D = torch.rand((Q, Q), generator=g, dtype=torch.float64).numpy()
    X = torch.rand((Q, 5000), generator=g, dtype=torch.float64).cuda()
    pc = PeerCombiner(groups, rank, world, device=torch.device("cuda", 0))
    rc = RingCombiner(groups, rank, world)
    vp = pc(D, X[lo:hi])
    vr = rc(D, X[lo:hi])
    vd = torch.from_numpy(D[lo:hi]).cuda() @ X
    comb_err = max(float((vp - vd).abs().max() / vd.abs().max()), float((vr - vd).abs().max() / vd.abs().max()))
    sp = StageParallelStepper(GPUStageBackend(h, cfg), Q, 0.01, rank, world, tableau=tab, combine="peer")
    ss = StageSystem(h, Q, 0.01, config=cfg, tableau=tab)
    u1 = ss.initial_condition()
    u2 = u1.clone()
    its = []
    for st in range(2):
        u1, rep = ss.step(st * 0.01, u1)
        u2, k_it, conv = sp.step(st * 0.01, u2)
        its.append((k_it, rep.iterations, conv))
    sp.ring.close()
    pc.close()
    return comb_err, float((u2 - u1).abs().max() / u1.abs().max()), its


@pytest.mark.parametrize("Q,world", [(3, 3), (4, 2)])
def test_peer_window_combine_stepper(cuda, Q, world):
    res = _run(_peer_worker, world, Q)
    for r, (comb_err, err, its) in res.items():
        assert comb_err < 1e-14, (r, comb_err)
        assert err < 1e-9, (r, err)
        for k_it, k_ref, conv in its:
            assert conv and abs(k_it - k_ref) <= 1


def _slab_overlap_worker(rank, world):
    from paper_2209_06700_b200.fem import build_hierarchy
    from paper_2209_06700_b200.parallel import SlabOperator

    h = build_hierarchy(3, 3, 2, device="cuda:0")
    DM, DK = np.eye(3), 1e-2 * np.arange(1.0, 10.0).reshape(3, 3)
    op = SlabOperator(h, 3, DM, DK, world=world, rank=rank)
    assert op.overlap and op.launches_per_apply == 3
    u, v1 = op.alloc()
    own = op.layout.owned_slice()
    g = torch.Generator(device="cuda").manual_seed(10 + rank)
    u[:, own] = torch.rand((3, own.stop - own.start), dtype=torch.float64, device="cuda", generator=g)
    v2 = torch.zeros_like(v1)
    op.apply(u, v1)                      # exchange overlapped with the interior launch
    op.overlap = False
    op.apply(u, v2)                      # blocking exchange, one launch
    return float((v1[:, own] - v2[:, own]).abs().max()), float(v2[:, own].abs().max())


@pytest.mark.parametrize("world", [2, 3])
def test_slab_operator_overlap_is_exact(cuda, world):
    """SlabOperator's interior/edge split (halo exchange overlapped with the interior elements)
    produces exactly the single-launch result on every rank."""
    res = _run(_slab_overlap_worker, world)
    for r, (d, scale) in res.items():
        assert d == 0.0 and scale > 0, (r, d)
