"""Device multigrid / GMRES / time steps vs the CPU oracle (north_star: solutions 1e-9, iterations +-1)."""

import numpy as np
import pytest
import torch

from oracle import solvers as OS
from oracle import stepper as OST
from oracle.fem_qk import Hierarchy
from oracle.tableau_ref import radau_iia as ref_radau
from paper_2209_06700_b200.complex_solver import DirectComplexSystem
from paper_2209_06700_b200.errors import NumericalFailureError
from paper_2209_06700_b200.fem import build_hierarchy
from paper_2209_06700_b200.irk import StageSystem
from paper_2209_06700_b200.krylov import gmres
from paper_2209_06700_b200.multigrid import (BatchedBlockSolver, BlockSolver, MultiBlockSolver, PairBlockSolver,
                                             VCycleConfig)

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


MG_CASES = [(1, 1, 4), (2, 1, 3), (3, 1, 3), (2, 2, 3), (3, 2, 2), (3, 3, 2), (3, 4, 2), (2, 4, 2)]


@pytest.mark.parametrize("dim,k,L", MG_CASES)
def test_block_vcycle_matches_oracle(cuda, dim, k, L):
    h, o = build_hierarchy(dim, L, k), Hierarchy(dim, L, k)
    b = np.where(o.finest.interior_mask, np.random.default_rng(5).standard_normal(o.n), 0.0)
    for deg in (5, 3, 1):
        cfg = VCycleConfig(smoother_degree=deg)
        dev = BlockSolver(h, 1.7, 0.05, cfg)
        ref = OS.VCycle(o, [1.7], 0.05, OS.Config(smoother_degree=deg))
        for l in range(L + 1):
            assert abs(dev.smoothers[l].theta - ref.sm[l][0].theta) < 1e-12 * ref.sm[l][0].theta
        assert rel(dev.apply(b), ref.apply(b)) < 1e-11


@pytest.mark.parametrize("dim,k,L", [(1, 1, 4), (3, 2, 2), (3, 4, 2)])
def test_batched_multi_pair_match_oracle(cuda, dim, k, L):
    h, o = build_hierarchy(dim, L, k), Hierarchy(dim, L, k)
    rng = np.random.default_rng(9)
    b = np.where(o.finest.interior_mask, rng.standard_normal((3, o.n)), 0.0)
    lams = [1.5, 4.0, 9.0]
    assert rel(BatchedBlockSolver(h, lams, 0.02).apply(b), OS.VCycle(o, lams, 0.02, shared=True).apply(b)) < 1e-11
    assert rel(MultiBlockSolver(h, lams, 0.02).apply(b), OS.VCycle(o, lams, 0.02).apply(b)) < 1e-11
    pb, po = PairBlockSolver(h, 2.0, np.sqrt(2.0), 0.05), OS.VCycle(o, tau=0.05, pair=(2.0, np.sqrt(2.0)))
    assert rel(pb.apply(b[:2]), po.apply(b[:2])) < 1e-11
    for l in range(L + 1):
        assert abs(pb.smoothers[l].theta - po.sm[l].theta) < 1e-12 * po.sm[l].theta


def test_vcycle_linear_and_symmetric(cuda):
    h = build_hierarchy(2, 3, 2)
    mask = h.finest.interior_mask
    rng = np.random.default_rng(23)
    s = BlockSolver(h, 2.0, 0.1)
    b1, b2 = (np.where(mask, rng.standard_normal(h.n), 0.0) for _ in range(2))
    lhs, rhs = s.apply(3.0 * b1 - 0.5 * b2), 3.0 * s.apply(b1) - 0.5 * s.apply(b2)
    assert np.abs(lhs - rhs).max() < 1e-12 * max(np.abs(lhs).max(), 1.0)
    v1, v2 = s.apply(b1), s.apply(b2)
    assert abs(v1 @ b2 - b1 @ v2) < 1e-10 * max(abs(v1 @ b2), 1.0)
    assert np.all(PairBlockSolver(h, 2.0, 1.5, 0.1).apply(np.zeros((2, h.n))) == 0.0)


def test_vcycle_nan_raises(cuda):
    h = build_hierarchy(2, 3, 1)
    b = np.zeros(h.n)
    b[h.n // 2] = np.nan
    with pytest.raises(NumericalFailureError):
        BlockSolver(h, 1.0, 0.1).apply(b)


def test_gmres_vcycle_mesh_independence_and_dense(cuda):
    its = []
    for L in (4, 5):
        h = build_hierarchy(1, L)
        o = Hierarchy(1, L)
        s = BlockSolver(h, 1.0, 0.1)
        b = np.where(h.finest.interior_mask, np.random.default_rng(3).standard_normal(h.n), 0.0)
        x, rep = gmres(lambda v: h.apply_constrained(L, 1.0, 0.1, v), s.apply, b, rel_tol=1e-12)
        its.append(rep.iterations)
        A = np.column_stack([o.apply_constrained(L, 1.0, 0.1, e) for e in np.eye(h.n)])
        assert np.allclose(x, np.linalg.solve(A, b), atol=1e-9)
    assert its[0] <= 10 and abs(its[0] - its[1]) <= 1


@pytest.mark.parametrize("dim,k,L", [(2, 2, 3), (3, 3, 2)])
def test_device_gmres_matches_oracle(cuda, dim, k, L):
    h, o = build_hierarchy(dim, L, k), Hierarchy(dim, L, k)
    b = np.where(o.finest.interior_mask, np.random.default_rng(1).standard_normal(o.n), 0.0)
    s, so = BlockSolver(h, 1.7, 0.05), OS.VCycle(o, [1.7], 0.05)
    bt = torch.from_numpy(b).cuda()
    x, rep = gmres(lambda v: h.apply_constrained(L, 1.7, 0.05, v), lambda v: s.apply(v), bt, rel_tol=1e-12)
    xo, its, hist, conv = OS.gmres(lambda v: o.apply_constrained(L, 1.7, 0.05, v), so.apply, b)
    assert rep.iterations == its and rep.converged
    assert rel(x.cpu().numpy(), xo) < 1e-9
    assert rel(np.array(rep.residual_history), np.array(hist)) < 1e-6


def test_gmres_reference_contract(cuda):
    rng = np.random.default_rng(11)
    b = rng.standard_normal(20)
    x, rep = gmres(lambda v: v, None, b)
    assert rep.iterations == 1 and rep.converged and np.allclose(x, b, atol=1e-12)
    A = rng.standard_normal((40, 40)) + 8.0 * np.eye(40)
    b = rng.standard_normal(40)
    x, rep = gmres(lambda v: A @ v, None, b, rel_tol=1e-12)
    hist = np.array(rep.residual_history)
    assert np.all(hist[1:] <= hist[:-1] * (1 + 1e-14))
    assert abs(hist[-1] - np.linalg.norm(b - A @ x)) <= 1e-12 * hist[0] + 1e-12 * np.linalg.norm(b - A @ x)
    xd, repd = gmres(lambda v: np.diag([2.0, 3.0, 4.0]) @ v, None, np.array([1.0, 0.0, 0.0]), rel_tol=1e-15)
    assert repd.converged and np.allclose(xd, [0.5, 0, 0], atol=1e-14)
    _, repn = gmres(lambda v: A @ v, None, b, rel_tol=1e-14, max_iter=3)
    assert not repn.converged and repn.iterations == 3
    with pytest.raises(NumericalFailureError):
        gmres(lambda v: np.full_like(v, np.nan), None, np.ones(4))
    with pytest.raises(ValueError):
        gmres(lambda v: v, None, np.ones(3), rel_tol=0.0)
    Ac = rng.standard_normal((25, 25)) + 1j * rng.standard_normal((25, 25)) + 10 * np.eye(25)
    bc = rng.standard_normal(25) + 1j * rng.standard_normal(25)
    xc, repc = gmres(lambda v: Ac @ v, None, bc, rel_tol=1e-12)
    assert repc.converged and np.allclose(xc, np.linalg.solve(Ac, bc), atol=1e-9)


def _run_pair(dev_sys, ora_sys, steps, tau):
    u = dev_sys.initial_condition()
    uo = ora_sys.initial()
    assert rel(u.cpu().numpy(), uo) < 1e-15
    its_d, its_o = [], []
    for s in range(steps):
        u, rep = dev_sys.step(s * tau, u)
        uo, ito, conv = ora_sys.step(s * tau, uo)
        its_d.append(rep.iterations)
        its_o.append(ito)
    return u.cpu().numpy(), uo, its_d, its_o


def test_config1_steps_match_oracle(cuda):
    """C1: 2D, 16x16 Q2 cells, Radau IIA Q=2, tau=0.05, 10 steps, GMRES rtol 1e-10."""
    h, o = build_hierarchy(2, 4, 2), Hierarchy(2, 4, 2)
    tab = ref_radau(2)
    dev = StageSystem(h, 2, 0.05, rel_tol=1e-10, tableau=tab)
    ora = OST.RealLU(o, 2, 0.05, rel_tol=1e-10, tab=tab)
    u, uo, itd, ito = _run_pair(dev, ora, 10, 0.05)
    assert all(abs(a - b) <= 1 for a, b in zip(itd, ito)), (itd, ito)
    assert rel(u, uo) < 1e-9
    err = h.l2_error(4, u, lambda x, t: np.prod(np.sin(np.pi * x), axis=1) * np.exp(-t), 0.5)
    assert err < 1e-4


@pytest.mark.parametrize("dim,L,k,Q", [(2, 4, 2, 2), (3, 3, 2, 3)])
def test_graphed_iterations_match_host_iterations(cuda, dim, L, k, Q):
    """GMRES iterations as replayed per-iteration CUDA graphs with the device Givens residual
    (krylov.GraphedIterations) vs the host-driven loop with lstsq every iteration (krylov.py:84-87):
    same iteration counts and V-cycle counts, solutions to 1e-12, over several steps (graph reuse)."""
    tab = ref_radau(Q)
    cfg = VCycleConfig(smoother_degree=3)
    h = build_hierarchy(dim, L, k)
    a = StageSystem(h, Q, 0.02, config=cfg, tableau=tab)
    b = StageSystem(h, Q, 0.02, config=cfg, tableau=tab)
    b.graph_iterations = False
    assert a.graph_iterations
    ua, ub = a.initial_condition(), b.initial_condition()
    for s in range(3):
        ua, ra = a.step(s * 0.02, ua)
        ub, rb = b.step(s * 0.02, ub)
        assert ra.iterations == rb.iterations and ra.vcycles_per_stage == rb.vcycles_per_stage == ra.iterations + 1
        assert rel(ua.cpu().numpy(), ub.cpu().numpy()) < 1e-12
        hs_a, hs_b = np.array(ra.residual_history), np.array(rb.residual_history)
        assert np.allclose(hs_a, hs_b, rtol=1e-8, atol=1e-14 * hs_b[0])
    assert len(a._gi.graphs) >= ra.iterations


def test_config3_like_steps_match_oracle(cuda):
    """C3 settings (Q2, Radau Q=3, tau=0.01, Chebyshev degree 3) on a 8^3 mesh, 3 steps."""
    h, o = build_hierarchy(3, 3, 2), Hierarchy(3, 3, 2)
    tab = ref_radau(3)
    cfg = VCycleConfig(smoother_degree=3)
    dev = StageSystem(h, 3, 0.01, config=cfg, tableau=tab)
    ora = OST.RealLU(o, 3, 0.01, OS.Config(smoother_degree=3), tab=tab)
    u, uo, itd, ito = _run_pair(dev, ora, 3, 0.01)
    assert all(abs(a - b) <= 1 for a, b in zip(itd, ito)), (itd, ito)
    assert rel(u, uo) < 1e-9


def test_batched_mode_matches_oracle(cuda):
    h, o = build_hierarchy(3, 3, 1), Hierarchy(3, 3, 1)
    tab = ref_radau(4)
    dev = StageSystem(h, 4, 0.1, mode="batched", tableau=tab)
    ora = OST.RealLU(o, 4, 0.1, tab=tab, shared=True)
    u, uo, itd, ito = _run_pair(dev, ora, 2, 0.1)
    assert all(abs(a - b) <= 1 for a, b in zip(itd, ito)), (itd, ito)
    assert rel(u, uo) < 1e-9


@pytest.mark.parametrize("variant", ["presb", "gmg"])
def test_complex_path_matches_oracle(cuda, variant):
    """C5 settings (Q3 elements, Radau Q=3 = one real + one complex pair, tau=5e-3) on 4^3 cells."""
    h, o = build_hierarchy(3, 2, 3), Hierarchy(3, 2, 3)
    tab = ref_radau(3)
    dev = DirectComplexSystem(h, 3, 5e-3, variant=variant, tableau=tab)
    ora = OST.DirectComplex(o, 3, 5e-3, variant=variant, tab=tab)
    u = dev.initial_condition()
    uo = ora.initial()
    for s in range(2):
        u, rep = dev.step(s * 5e-3, u)
        uo, ito = ora.step(s * 5e-3, uo)
        assert all(abs(a - b) <= 1 for a, b in zip(rep.block_iterations, ito)), (rep.block_iterations, ito)
    assert rel(u.cpu().numpy(), uo) < 1e-9


def test_real_and_complex_paths_agree(cuda):
    h = build_hierarchy(3, 3, 1)
    tab = ref_radau(2)
    a = StageSystem(h, 2, 0.1, tableau=tab)
    b = DirectComplexSystem(h, 2, 0.1, variant="presb", tableau=tab)
    ua, _, _ = a.run(3)
    ub, _, _ = b.run(3)
    assert rel(ub.cpu().numpy(), ua.cpu().numpy()) < 1e-8


def test_stage_parallel_gpu_backend_single_rank(cuda):
    """GPUStageBackend + StageParallelStepper on one rank (NCCL world of 1) == StageSystem."""
    import os
    import torch.distributed as dist
    from paper_2209_06700_b200.stage_parallel import GPUStageBackend, StageParallelStepper

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        h = build_hierarchy(3, 3, 2)
        tab = ref_radau(3)
        cfg = VCycleConfig(smoother_degree=3)
        sp = StageParallelStepper(GPUStageBackend(h, cfg), 3, 0.01, 0, 1, tableau=tab)
        ss = StageSystem(h, 3, 0.01, config=cfg, tableau=tab)
        u1 = ss.initial_condition()
        u2 = u1.clone()
        for s in range(2):
            u1, rep = ss.step(s * 0.01, u1)
            u2, its, conv = sp.step(s * 0.01, u2)
            assert abs(its - rep.iterations) <= 1 and conv
        assert rel(u2.cpu().numpy(), u1.cpu().numpy()) < 1e-9
    finally:
        dist.destroy_process_group()


def test_direct_complex_parallel_gpu_backend_single_rank(cuda):
    import os
    import torch.distributed as dist
    from paper_2209_06700_b200.stage_parallel import DirectComplexParallelStepper, GPUStageBackend

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = "29534"
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        h = build_hierarchy(3, 2, 3)
        tab = ref_radau(3)
        sp = DirectComplexParallelStepper(GPUStageBackend(h), 3, 5e-3, 0, 1, tableau=tab, variant="presb")
        ds = DirectComplexSystem(h, 3, 5e-3, variant="presb", tableau=tab)
        u1 = ds.initial_condition()
        u2 = u1.clone()
        for s in range(2):
            u1, rep = ds.step(s * 5e-3, u1)
            u2, its = sp.step(s * 5e-3, u2)
        assert rel(u2.cpu().numpy(), u1.cpu().numpy()) < 1e-9
    finally:
        dist.destroy_process_group()


def test_perfmodel_counters_on_device_steps(cuda):
    """#V = Q (#G + 1) per step in the real-LU path; predicted stage-parallel speedup = Q."""
    from paper_2209_06700_b200.perfmodel import validate_against_counters

    h = build_hierarchy(3, 3, 2)
    ss = StageSystem(h, 4, 0.01, config=VCycleConfig(smoother_degree=3), tableau=ref_radau(4))
    u = ss.initial_condition()
    reps = []
    for s in range(2):
        u, rep = ss.step(s * 0.01, u)
        reps.append(rep)
    v = validate_against_counters(reps, 4)
    assert v.ok, v.mismatches
    assert v.predicted_speedup == 4


@pytest.mark.parametrize("dim,k,L,nblk", [(3, 2, 3, 3), (3, 4, 2, 1), (2, 3, 3, 2), (1, 2, 4, 4), (3, 1, 4, 2)])
@pytest.mark.parametrize("split", [0, 1 << 62])
def test_vcycle_split_and_fused_chebyshev_match_oracle(cuda, dim, k, L, nblk, split):
    """Large levels run each Chebyshev step as K1 STORE + pointwise update (zero start without
    materialising r = b, x = 0); small ones keep the fused K1 epilogue. Force each path on every
    level and check both against the oracle (degrees 1, 2, 3, 5: the first / final-step variants)."""
    from paper_2209_06700_b200 import _lib

    h, o = build_hierarchy(dim, L, k), Hierarchy(dim, L, k)
    _lib.call("spk_set_cheb_split", h.ctx, split)
    rng = np.random.default_rng(21)
    lams = [1.7, 3.1, 0.6, 8.0][:nblk]
    b = np.where(o.finest.interior_mask, rng.standard_normal((nblk, o.n)), 0.0)
    for deg in (1, 2, 3, 5):
        cfg = VCycleConfig(smoother_degree=deg)
        dev = MultiBlockSolver(h, lams, 0.03, cfg)
        ref = OS.VCycle(o, lams, 0.03, OS.Config(smoother_degree=deg))
        assert rel(dev.apply(b), ref.apply(b)) < 1e-11, (deg, split)
