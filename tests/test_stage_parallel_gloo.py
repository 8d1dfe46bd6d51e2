"""Stage-parallel stepper (stage groups over ranks, ring combines, all-reduced GMRES dots) on CPU
with gloo, against the single-process oracle stepper."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class OracleStageBackend:
    """Stage-local operators from the CPU oracle (test double of GPUStageBackend)."""

    def __init__(self, dim, L, k, deg):
        from oracle.fem_qk import Hierarchy
        from oracle.stepper import Separable

        self.h = Hierarchy(dim, L, k)
        self.L, self.deg = L, deg
        self.src = Separable(dim)
        self.mask_np = self.h.levels[L].interior_mask

    def setup(self, lams, tau):
        from oracle import solvers

        self.tau = tau
        self.vc = solvers.VCycle(self.h, lams, tau, solvers.Config(smoother_degree=self.deg))
        self.m = torch.from_numpy(self.mask_np)

    def mass_stiff(self, k):
        km = np.where(self.mask_np, k.numpy(), 0.0)
        return (torch.from_numpy(self.h.apply_mass(self.L, km)), torch.from_numpy(self.h.apply_stiffness(self.L, km)))

    def boundary_identity(self, v, k):
        return torch.where(self.m, v, k)

    def mask(self, v):
        return torch.where(self.m, v, torch.zeros_like(v))

    def vcycle(self, w):
        return torch.from_numpy(self.vc.apply(w.numpy()))

    def stage_rhs(self, t_n, u_n, ctau):
        ku = self.h.apply_stiffness(self.L, np.where(self.mask_np, u_n.numpy(), 0.0))
        return torch.from_numpy(np.stack([self.h.load_vector(self.L, self.src.f, t_n + ct) - ku for ct in ctau]))


class HostShmWindows:
    """Test double of CudaIpcWindows: POSIX shared memory between the gloo processes."""

    def __init__(self):
        self._shm = {}

    def _arr(self, name):
        shm = self._shm[name]
        return np.ndarray((shm.size // 8,), dtype=np.float64, buffer=shm.buf)

    def create(self, nbytes):
        from multiprocessing import shared_memory
        shm = shared_memory.SharedMemory(create=True, size=nbytes)
        self._shm[shm.name] = shm
        return shm.name, shm.name.encode()

    def open(self, handle):
        from multiprocessing import shared_memory
        name = handle.decode()
        self._shm[name] = shared_memory.SharedMemory(name=name)
        return name

    def row(self, ptr, i, n):
        return (ptr, i * n, n)

    def write(self, ptr, x):
        x = x.reshape(-1).numpy()
        self._arr(ptr)[: x.size] = x

    def combine(self, n, rows, D, out):
        X = np.stack([self._arr(p)[o : o + m] for p, o, m in rows])
        out.copy_(torch.from_numpy(np.asarray(D) @ X))

    def sync(self):
        pass

    def close(self, peer_ptrs, own):
        for p in peer_ptrs:
            self._shm.pop(p).close()
        shm = self._shm.pop(own)
        shm.close()
        shm.unlink()


def _worker(rank, world, port, Q, q_out, combine="ring"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.tableau_ref import radau_iia
        from paper_2209_06700_b200.stage_parallel import StageParallelStepper

        be = OracleStageBackend(3, 3, 1, 5)
        tab = radau_iia(Q)
        sp = StageParallelStepper(be, Q, 0.05, rank, world, tableau=tab, combine=combine,
                                  windows=HostShmWindows() if combine == "peer" else None)
        u = torch.from_numpy(be.src.u(be.h.node_coords(be.L), 0.0))
        its = []
        for s in range(2):
            u, k, conv = sp.step(s * 0.05, u)
            its.append(k)
        if combine == "peer":
            sp.ring.close()
        if rank == 0:
            q_out.put((u.numpy(), its, sp.ring.shift_rounds, sp.grid.counters.as_dict()))
    except Exception as e:  # pragma: no cover
        q_out.put(repr(e))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("Q,world,combine", [(2, 2, "ring"), (3, 2, "ring"), (4, 2, "ring"), (4, 4, "peer"),
                                              (3, 2, "peer")])
def test_stage_parallel_matches_oracle(Q, world, combine):
    from oracle import stepper
    from oracle.fem_qk import Hierarchy
    from oracle.tableau_ref import radau_iia

    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = [ctx.Process(target=_worker, args=(r, world, port, Q, q, combine)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    res = q.get()
    assert not isinstance(res, str), res
    u_dist, its_dist, shifts, counters = res
    ref = stepper.RealLU(Hierarchy(3, 3, 1), Q, 0.05, tab=radau_iia(Q))
    u = ref.initial()
    its = []
    for i in range(2):
        u, k, _ = ref.step(i * 0.05, u)
        its.append(k)
    assert all(abs(a - b) <= 1 for a, b in zip(its_dist, its)), (its_dist, its)
    assert np.abs(u_dist - u).max() / np.abs(u).max() < 1e-9
    if combine == "ring":
        # (world - 1) ring shifts per combine, 3 combines per GMRES iteration (+ 1 for the RHS, the
        # final P^-1 and A) -> strictly positive and a multiple of world - 1
        assert shifts > 0 and shifts % (world - 1) == 0
    else:
        # shared-memory backend: no messages for the combines, 2 barriers per combine
        assert shifts == 0 and counters["shift_rounds"] == 0
        assert counters["barriers"] > 0 and counters["barriers"] % 2 == 1  # + 1 for close()


class OracleComplexBackend(OracleStageBackend):
    def setup_pairs(self, own_pairs, tau, variant):
        from oracle import solvers

        self.tau = tau
        self.m = torch.from_numpy(self.mask_np)
        cfg = solvers.Config(smoother_degree=self.deg)
        self.blocks = []
        for p in own_pairs:
            if p.is_real:
                self.blocks.append(("real", p, solvers.VCycle(self.h, [p.re], tau, cfg)))
            elif variant == "presb":
                self.blocks.append(("presb", p, solvers.VCycle(self.h, [p.re + p.im], tau, cfg)))
            else:
                self.blocks.append(("gmg", p, solvers.VCycle(self.h, tau=tau, cfg=cfg, pair=(p.re, p.im))))

    def solve_pair(self, i, rows):
        from oracle import solvers

        kind, p, vc = self.blocks[i]
        h, L, tau = self.h, self.L, self.tau
        r = rows.numpy()
        if kind == "real":
            z, its, _, _ = solvers.gmres(lambda v: h.apply_constrained(L, p.re, tau, v), vc.apply, r[0])
            out = np.zeros_like(r)
            out[0] = z
            return torch.from_numpy(out), its

        def op(u):
            ui = np.where(self.mask_np, u, 0.0)
            mr, mi = h.apply_mass(L, ui[0]), h.apply_mass(L, ui[1])
            kr, ki = h.apply_stiffness(L, ui[0]), h.apply_stiffness(L, ui[1])
            out = np.stack([p.re * mr + tau * kr - p.im * mi, p.im * mr + p.re * mi + tau * ki])
            return np.where(self.mask_np, out, u)

        if kind == "presb":
            def pc(v):
                y1 = vc.apply(v[0] + v[1])
                y2 = vc.apply(v[1] - h.apply_constrained(L, p.im, 0.0, y1))
                return np.stack([y1 - y2, y2])
        else:
            pc = vc.apply
        z, its, _, _ = solvers.gmres(op, pc, r)
        return torch.from_numpy(z), its


def _cworker(rank, world, port, Q, variant, q_out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.tableau_ref import radau_iia
        from paper_2209_06700_b200.stage_parallel import DirectComplexParallelStepper

        be = OracleComplexBackend(3, 2, 2, 3)
        sp = DirectComplexParallelStepper(be, Q, 5e-3, rank, world, tableau=radau_iia(Q), variant=variant)
        u = torch.from_numpy(be.src.u(be.h.node_coords(be.L), 0.0))
        for s in range(2):
            u, its = sp.step(s * 5e-3, u)
        if rank == 0:
            q_out.put(u.numpy())
    except Exception as e:  # pragma: no cover
        q_out.put(repr(e))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("Q,variant", [(3, "presb"), (4, "gmg")])
def test_direct_complex_parallel_matches_oracle(Q, variant):
    from oracle import solvers, stepper
    from oracle.fem_qk import Hierarchy
    from oracle.tableau_ref import radau_iia

    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world = 2
    procs = [ctx.Process(target=_cworker, args=(r, world, port, Q, variant, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    res = q.get()
    assert not isinstance(res, str), res
    ref = stepper.DirectComplex(Hierarchy(3, 2, 2), Q, 5e-3, variant, solvers.Config(smoother_degree=3),
                                tab=radau_iia(Q))
    u = ref.initial()
    for i in range(2):
        u, _ = ref.step(i * 5e-3, u)
    assert np.abs(res - u).max() / np.abs(u).max() < 1e-9


def _ring_worker(rank, world, port, Q, pairs, q_out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2209_06700_b200.runtime import stage_groups
        from paper_2209_06700_b200.stage_parallel import RingCombiner

        rng = np.random.default_rng(5)
        n = 37
        X = rng.standard_normal((Q, n))
        groups = stage_groups(Q, world)
        ring = RingCombiner(groups, rank, world)
        lo, hi = groups[rank]
        out = {}
        D = rng.standard_normal((Q, Q))
        out["square"] = ring(D, torch.from_numpy(X[lo:hi].copy())).numpy()
        if pairs:  # stage groups -> paired rows (the complex path's S^-1 combine) and back
            P = (Q + 1) // 2
            pg = [(2 * a, 2 * b) for a, b in stage_groups(P, world)]
            Wf = rng.standard_normal((2 * P, Q))
            out["fwd"] = ring(Wf, torch.from_numpy(X[lo:hi].copy()), in_groups=groups, out_groups=pg).numpy()
            Y = rng.standard_normal((2 * P, n))
            plo, phi = pg[rank]
            Wb = rng.standard_normal((Q, 2 * P))
            out["back"] = ring(Wb, torch.from_numpy(Y[plo:phi].copy()), in_groups=pg, out_groups=groups).numpy()
        q_out.put((rank, out))
    except Exception as e:  # pragma: no cover
        q_out.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("Q,world", [(7, 3), (3, 4), (5, 2)])
def test_ring_combiner_uneven_and_empty_groups(Q, world):
    """Stage groups of different sizes (Q=7 on 3 ranks) and empty groups (Q=3 on 4 ranks: the
    complex path at 4 GPUs) through the double-buffered ring, against D @ x."""
    from paper_2209_06700_b200.runtime import stage_groups

    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = [ctx.Process(target=_ring_worker, args=(r, world, port, Q, True, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    res = dict(q.get() for _ in range(world))
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
    rng = np.random.default_rng(5)
    n = 37
    X = rng.standard_normal((Q, n))
    D = rng.standard_normal((Q, Q))
    P = (Q + 1) // 2
    Wf = rng.standard_normal((2 * P, Q))
    Y = rng.standard_normal((2 * P, n))
    Wb = rng.standard_normal((Q, 2 * P))
    groups = stage_groups(Q, world)
    pg = [(2 * a, 2 * b) for a, b in stage_groups(P, world)]
    for r in range(world):
        lo, hi = groups[r]
        plo, phi = pg[r]
        np.testing.assert_allclose(res[r]["square"], (D @ X)[lo:hi], rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(res[r]["fwd"], (Wf @ X)[plo:phi], rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(res[r]["back"], (Wb @ Y)[lo:hi], rtol=1e-13, atol=1e-13)
