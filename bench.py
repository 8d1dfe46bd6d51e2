#!/usr/bin/env python
"""Headline benchmark: BASELINE.json configs[1] (C2), the batched stage-coupled operator.

  v = (I (x) M + tau A_Q (x) K) u   on 64^3 hex cells, Q4 elements (n = 257^3 = 16,974,593 DoFs per
  stage), Radau IIA Q = 3, tau = 1e-3, u ~ U[-1,1] fp64 from seed 42.

One "step" is one apply of the operator to the Q stage vectors. Metric: stage-DoFs/s (whole job).
  value : device-resident input, CUDA-event time of the K1 kernel, inputs (407 MB) > L2 (126 MB)
  e2e   : same apply through the public API with pinned host buffers, H2D + apply + D2H per step
  roofline: 16 B per stage-DoF (read u, write v) / kernel time vs measured HBM copy bandwidth
  cpu_baseline: the oracle (dense 1D Kronecker contractions, reference fem.py:37-41 generalised to
    Q_k) on all host cores, bounded sample (see `sample`)
Multi-GPU (torchrun): each rank owns an x-slab of a global mesh of N*64 x 64 x 64 cells and
exchanges its halo planes with its neighbours every apply (weak scaling).
`--impl reference` times the reference CPU path (oracle port) on the host cores instead.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CFG = dict(dim=3, cells=64, level=6, degree=4, Q=3, tau=1e-3, seed=42)
STEP_CONFIGS_C4_LEVEL = 7
METRIC = "stage-DoFs/s of batched matrix-free apply (C2: 64^3 Q4 hex, Radau IIA Q=3)"
UNIT = "stage-DoF/s"
FLOPS_PER_SDOF = 2 * (8 * (CFG["degree"] + 2) + 2 * CFG["Q"])  # 108 for C2


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    p.add_argument("--no-step", action="store_true", help="skip the Radau IIA step timings")
    p.add_argument("--step-configs", default="C1,C3,C4,C5,C5-gmg,C5-LU",
                   help="comma-separated Radau IIA step workloads timed at N=1")
    p.add_argument("--sp-level", type=int, default=STEP_CONFIGS_C4_LEVEL,
                   help="mesh level of the N>1 stage-parallel C4 step (7 = the config's 128^3 cells)")
    p.add_argument("--level", type=int, default=CFG["level"])
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def config_dict(args, world, extra=None):
    d = {"workload": "C2 batched operator microbench (BASELINE.json configs[1])",
         "mesh": f"{CFG['cells'] * world}x{CFG['cells']}x{CFG['cells']} hex" if world > 1 else "64^3 hex",
         "degree": CFG["degree"], "stages": CFG["Q"], "tau": CFG["tau"], "seed": CFG["seed"],
         "dofs_per_stage_per_gpu": (CFG["degree"] * 2 ** args.level + 1) ** 3,
         "operator": "I(x)M + tau*A_Q(x)K, unconstrained",
         "l2": "inputs 407 MB > 126 MB L2 (no flush needed)",
         "parallelism": f"x-slab mesh partition x{world}" if world > 1 else "single GPU"}
    if extra:
        d.update(extra)
    return d


# BASELINE.json configs as time-per-step workloads (C2 is the operator microbench above)
STEP_CONFIGS = {
    "C1": dict(dim=2, L=4, k=2, Q=2, tau=0.05, steps=10, rtol=1e-10, deg=5, path="real",
               desc="2D 16^2 Q2 quad, Radau IIA Q=2, tau=0.05, rtol 1e-10, LU block preconditioner (V-cycle)"),
    "C3": dict(dim=3, L=5, k=2, Q=3, tau=0.01, steps=20, rtol=1e-12, deg=3, path="real",
               desc="3D 32^3 Q2 hex, Radau IIA Q=3, tau=0.01, GMG V-cycle Chebyshev deg 3"),
    "C4": dict(dim=3, L=7, k=2, Q=4, tau=1e-3, steps=5, rtol=1e-12, deg=3, path="real",
               desc="3D 128^3 Q2 hex, Radau IIA Q=4, tau=1e-3, GMG V-cycle Chebyshev deg 3"),
    "C5": dict(dim=3, L=6, k=3, Q=3, tau=5e-3, steps=10, rtol=1e-12, deg=3, path="presb",
               desc="3D 64^3 Q3 hex, Radau IIA Q=3 diagonalised: complex pair by PRESB + real block"),
    "C5-gmg": dict(dim=3, L=6, k=3, Q=3, tau=5e-3, steps=10, rtol=1e-12, deg=3, path="gmg",
                   desc="C5 with the 2x2 GMG V-cycle for the pair instead of PRESB"),
    "C5-LU": dict(dim=3, L=6, k=3, Q=3, tau=5e-3, steps=10, rtol=1e-12, deg=3, path="real",
                  desc="C5 mesh and tableau through the LU-based (real, stage-parallel) variant"),
}
# one CPU oracle step per config on the host cores (the reference algorithm, dense 1D contractions);
# C4 / C5 take minutes per step there: not timed in the bench (their parity runs are in tests/)
CPU_STEP_CONFIGS = ("C1", "C3")


def cpu_info():
    """Core count, CPU model and BLAS backend of this host (threadpoolctl)."""
    import threadpoolctl

    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = [{k: d.get(k) for k in ("internal_api", "version", "num_threads", "architecture")}
            for d in threadpoolctl.threadpool_info() if d.get("user_api") == "blas"]
    return {"cores": len(os.sched_getaffinity(0)), "cpu_model": model, "blas": blas}


def _level_dofs(c):
    return [(c["k"] * 2 ** l + 1) ** c["dim"] for l in range(c["L"] + 1)]


def radau_steps(names, cpu=True, bw_gbs=None):
    """Time per Radau IIA step (the metric's second half) of each config on this GPU:
    device-resident state, one untimed warm-up step (graph capture), then the config's remaining
    steps between CUDA events. Each entry: GMRES iterations, V-cycles per stage (= its + 1),
    algorithmic bytes of the step (perfmodel) and the step-level HBM fraction."""
    import torch

    from paper_2209_06700_b200 import perfmodel
    from paper_2209_06700_b200.complex_solver import DirectComplexSystem
    from paper_2209_06700_b200.fem import build_hierarchy
    from paper_2209_06700_b200.irk import StageSystem
    from paper_2209_06700_b200.multigrid import VCycleConfig

    out = {}
    for name in names:
        c = STEP_CONFIGS[name]
        h = build_hierarchy(c["dim"], c["L"], c["k"])
        cfg = VCycleConfig(smoother_degree=c["deg"])
        t0 = time.perf_counter()
        if c["path"] == "real":
            ss = StageSystem(h, c["Q"], c["tau"], config=cfg, rel_tol=c["rtol"])
        else:
            ss = DirectComplexSystem(h, c["Q"], c["tau"], variant=c["path"], config=cfg, rel_tol=c["rtol"])
        u = ss.initial_condition()
        u, _ = ss.step(0.0, u)
        torch.cuda.synchronize()
        setup_s = time.perf_counter() - t0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        its, vcs, t = [], [], c["tau"]
        e0.record()
        for _ in range(c["steps"] - 1):
            u, rep = ss.step(t, u)
            its.append(rep.block_iterations if rep.block_iterations else rep.iterations)
            vcs.append(rep.vcycles_per_stage)
            t += c["tau"]
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / (c["steps"] - 1)
        err = h.l2_error(c["L"], u, lambda x, tt: np.prod(np.sin(np.pi * x), axis=1) * np.exp(-tt), t)
        lv = _level_dofs(c)
        fused = int(getattr(getattr(ss, "precond", None), "_cv_level", -1) or -1)
        if c["path"] == "real":
            byts = float(np.mean([perfmodel.real_step_bytes(lv, c["Q"], c["deg"], i, fused) for i in its]))
        else:
            byts = float(np.mean([perfmodel.complex_step_bytes(lv, c["Q"], c["deg"], i, c["path"], fused)
                                  for i in its]))
        ent = {"config": c["desc"], "n_per_stage": lv[-1], "Q": c["Q"], "ms_per_step": ms,
               "steps_timed": c["steps"] - 1, "warmup_steps": 1, "gmres_iterations": its,
               "vcycles_per_stage": vcs, "l2_error": err, "setup_and_first_step_s": setup_s,
               "alg_bytes_per_step": byts}
        if bw_gbs:
            ent["hbm_frac"] = byts / (ms * 1e-3) / (bw_gbs * 1e9)
        if cpu and name in CPU_STEP_CONFIGS:
            ent["cpu_baseline"] = cpu_step_sample(c)
        out[name] = ent
        del ss, h, u
        torch.cuda.empty_cache()
    return out


def cpu_step_sample(c):
    """The oracle (the reference's algorithm: dense-1D contractions, numpy/OpenBLAS) running one step
    of the same config on all host cores (the first step from the initial condition)."""
    import threadpoolctl
    from oracle import solvers as OS
    from oracle import stepper as OST
    from oracle.fem_qk import Hierarchy
    from oracle.tableau_ref import radau_iia as ref_radau

    cores = len(os.sched_getaffinity(0))
    with threadpoolctl.threadpool_limits(cores):
        ocfg = OS.Config(smoother_degree=c["deg"])
        ora = OST.RealLU(Hierarchy(c["dim"], c["L"], c["k"]), c["Q"], c["tau"], ocfg, rel_tol=c["rtol"],
                         tab=ref_radau(c["Q"]))
        uo = ora.initial()
        t0 = time.perf_counter()
        uo, its, _ = ora.step(0.0, uo)
        dt = time.perf_counter() - t0
    return {"ms_per_step": dt * 1e3, "cores": cores, "kind": "port", "gmres_iterations": its,
            "sample": "one step of the oracle (first step from the initial condition)"}


def c2_cpu_apply(Q, degree, tau, level, warm, reps):
    """The oracle on the full C2 configuration: the reference's algorithm as written (dense 1D
    Kronecker contractions via moveaxis/matmul, fem.py:37-41 and 120-151, generalised to Q_k) with
    the stage coupling matrix from the oracle's own tableau (oracle/tableau_ref.py), all host cores."""
    import threadpoolctl
    import oracle.fem_qk as F
    from oracle.tableau_ref import radau_iia as ref_radau

    F.FAST = False  # the dense reference form, not the oracle's banded test fast path
    cores = len(os.sched_getaffinity(0))
    with threadpoolctl.threadpool_limits(cores):
        h = F.Hierarchy(3, level, degree)
        n = h.levels[level].n_dofs
        u = np.random.default_rng(CFG["seed"]).uniform(-1.0, 1.0, size=(Q, n))
        DM, DK = np.eye(Q), tau * np.asarray(ref_radau(Q)["A"])
        for _ in range(warm):
            h.apply_stage(level, DM, DK, u)
        t0 = time.perf_counter()
        for _ in range(reps):
            h.apply_stage(level, DM, DK, u)
        dt = (time.perf_counter() - t0) / reps
    return n, dt, cores


def cpu_sample(Q, degree, tau, level, reps=3):
    """cpu_baseline of our arm: the C2 workload itself (same mesh, seed, operator) on the host."""
    n, dt, cores = c2_cpu_apply(Q, degree, tau, level, 1, reps)
    info = cpu_info()
    return {"value": Q * n / dt, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{reps} timed oracle applies (+1 warm-up) of the full C2 workload: 64^3 Q4 hex, "
                      f"n={n}/stage, Q={Q}, seed {CFG['seed']}, dense 1D contractions (reference form)",
            "seconds_per_apply": dt, "same_config": True, "cpu_model": info["cpu_model"], "blas": info["blas"]}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    Q, k, tau = CFG["Q"], CFG["degree"], CFG["tau"]
    level = args.level
    warm = min(args.warmup, 2)  # CPU warm-up beyond the first apply changes nothing (page faults only)
    n, dt, cores = c2_cpu_apply(Q, k, tau, level, warm, args.steps)
    val = Q * n / dt
    info = cpu_info()
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": warm, "ms_per_step": dt * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic U[-1,1] seed 42",
            "config": config_dict(args, 1),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"each step = one oracle apply of the full C2 workload (64^3 Q4 hex, "
                                       f"n={n}/stage, Q={Q}, seed {CFG['seed']}); the reference is pure numpy "
                                       f"(k=1 only, fem.py:37-41 dense contractions): the oracle is that "
                                       f"algorithm generalised to Q_k, coupling matrix from oracle/tableau_ref",
                             "same_config": True, "cpu_model": info["cpu_model"], "blas": info["blas"]},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def stage_parallel_c4(args, rank, world, dev, bw_gbs, combine="ring"):
    """C4 (BASELINE.json configs[3]) in the paper's stage-parallel layout on N = S x B GPUs: stage
    group s of mesh partition b per rank (row-major), ring stage combines over NCCL, distributed
    V-cycles on x-slabs when B > 1, all-reduced GMRES dots (stage_parallel.StageParallelStepper).
    One untimed warm-up step, then the config's remaining steps; time = max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2209_06700_b200.fem import build_hierarchy
    from paper_2209_06700_b200.multigrid import VCycleConfig
    from paper_2209_06700_b200.runtime import RankGrid
    from paper_2209_06700_b200.slab import SlabHierarchy, SlabPartition
    from paper_2209_06700_b200.stage_parallel import GPUSlabStageBackend, GPUStageBackend, StageParallelStepper
    from paper_2209_06700_b200.tableau import radau_iia

    c = dict(STEP_CONFIGS["C4"], L=args.sp_level)
    Q = c["Q"]
    S = min(world, Q)
    B = world // S
    if S * B != world:
        return {"skipped": f"{world} GPUs do not factor as S x B with S <= Q = {Q}"}
    grid = RankGrid(S, B).init_groups()
    s_idx, b_idx = grid.coords(rank)
    cfg = VCycleConfig(smoother_degree=c["deg"])
    if B > 1:
        part = SlabPartition(c["k"], c["L"], B, b_idx, ranks=grid.col_ranks(s_idx), group=grid.col_group(s_idx),
                             counters=grid.counters)
        be = GPUSlabStageBackend(SlabHierarchy(c["L"], c["k"], part, device=dev), cfg)
    else:
        part = None
        be = GPUStageBackend(build_hierarchy(3, c["L"], c["k"], device=dev), cfg)
    sp = StageParallelStepper(be, Q, c["tau"], rank, world, tableau=radau_iia(Q), rel_tol=c["rtol"], grid=grid,
                              combine=combine)
    # initial condition: nodal interpolant of prod_d sin(pi x_d) (the configs' manufactured solution)
    s1 = np.sin(np.pi * build_hierarchy(3, c["L"], c["k"], device=dev).levels[c["L"]].nodes_1d)
    full = torch.from_numpy(np.multiply.outer(np.multiply.outer(s1, s1), s1).reshape(1, -1)).to(dev)
    u = full[0] if part is None else part.scatter(full, c["L"])[0]
    del full
    u, its0, _ = sp.step(0.0, u)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    its, t = [], c["tau"]
    e0.record()
    for _ in range(c["steps"] - 1):
        u, k, conv = sp.step(t, u)
        its.append(k)
        t += c["tau"]
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (c["steps"] - 1)
    tt = torch.tensor([ms], device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms = float(tt.item())
    return {"config": c["desc"] + ("" if c["L"] == 7 else f" [mesh level {c['L']}]"),
            "grid": f"S={S} x B={B} (row-major)", "combine": combine, "ms_per_step": ms,
            "steps_timed": c["steps"] - 1, "warmup_steps": 1, "gmres_iterations": its,
            "stage_dofs_per_s": Q * (c["k"] * 2 ** c["L"] + 1) ** 3 / (ms * 1e-3), "counters": grid.snapshot(rank)}


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2209_06700_b200 import measure
    from paper_2209_06700_b200.fem import build_hierarchy
    from paper_2209_06700_b200.parallel import SlabOperator
    from paper_2209_06700_b200.tableau import radau_iia

    rank, world, local = dist_env()
    if os.environ.get("BENCH_SHARE_GPU"):  # functional multi-rank test on one GPU (gloo only)
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    Q, k, tau, L = CFG["Q"], CFG["degree"], CFG["tau"], args.level
    hier = build_hierarchy(3, L, k, device=dev)
    n = hier.levels[L].n_dofs
    DM = np.eye(Q)
    DK = tau * radau_iia(Q).A
    rng = np.random.default_rng(CFG["seed"] + rank)
    u_host = torch.from_numpy(rng.uniform(-1.0, 1.0, size=(Q, n))).pin_memory()
    v_host = torch.empty_like(u_host).pin_memory()
    op = SlabOperator(hier, L, DM, DK, world=world, rank=rank) if world > 1 else None
    if op is None:
        u = u_host.to(dev)
        v = torch.empty_like(u)
    else:
        # slab buffers: [k halo planes | owned planes | 1 halo plane]; this rank's 64^3-cell block
        # fills the owned planes (the last rank also owns the global boundary plane)
        u, v = op.alloc()
        lay = op.layout
        own = lay.owned_slice()
        u[:, own] = u_host[:, : own.stop - own.start].to(dev)

    def apply_dev():
        if op is None:
            hier.apply_stage_operator(L, DM, DK, u, out=v)
        else:
            op.apply(u, v)

    for _ in range(max(3, args.warmup)):
        apply_dev()
    torch.cuda.synchronize()

    # ---- device-resident timed region ----
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with measure.ClockSampler(local) as clk:
        e0.record(s)
        for _ in range(args.steps):
            apply_dev()
        e1.record(s)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    ms_local = ms
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * Q * n / (ms * 1e-3)

    # ---- kernel-only time of K1 (single launch, same stream) ----
    kern_ms = []
    for _ in range(5):
        if op is None:
            kern_ms.append(measure.event_time(lambda: hier.apply_stage_operator(L, DM, DK, u, out=v)))
        else:
            kern_ms.append(measure.event_time(lambda: op.launch(u, v)))
    kern_best = min(kern_ms)
    kern_single = sorted(kern_ms)[len(kern_ms) // 2]
    # roofline: K1's AVERAGE launch duration over the timed region (one K1 launch per step at N = 1,
    # CUDA events on the launching stream); an isolated launch (event pair around one launch) is
    # reported beside it. With slabs (N > 1) a step also exchanges halos: the isolated launch is used.
    kern_ms = ms_local if op is None else kern_single
    # the constrained variant of the same operator (report both)
    cons_ms = None
    if op is None:
        hier.apply_stage_operator(L, DM, DK, u, out=v, constrained=True)
        cons_ms = sorted(measure.event_time(
            lambda: hier.apply_stage_operator(L, DM, DK, u, out=v, constrained=True)) for _ in range(5))[2]
    peak, peak_kind = measure.measured_peaks()
    alg_bytes = 16.0 * Q * n
    achieved = alg_bytes / (kern_ms * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(REPO, "profiles", "stage_apply_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- end-to-end through the public API with host buffers ----
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world == 1:
        # public host-buffer entry point: chunked H2D / K1 / D2H overlap (pipeline.py)
        from paper_2209_06700_b200.pipeline import HostStageOperator
        hop = HostStageOperator(hier, L, DM, DK, chunks=4)  # steady-state optimum (tools/e2e_probe.py)
        hop.apply(u_host, v_host)
        torch.cuda.synchronize()
        e2.record(s)
        for _ in range(args.steps):
            hop.apply(u_host, v_host)
        e3.record(s)
    else:
        e2.record(s)
        for _ in range(args.steps):
            own = op.layout.owned_slice()
            m = own.stop - own.start
            for q in range(Q):
                u[q, own].copy_(u_host[q, :m], non_blocking=True)
            apply_dev()
            for q in range(Q):
                v_host[q, :m].copy_(v[q, own], non_blocking=True)
        e3.record(s)
    torch.cuda.synchronize()
    e2e_ms = e2.elapsed_time(e3) / args.steps
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_val = world * Q * n / (e2e_ms * 1e-3)

    fp64_peak = measure.fp64_peak_tflops()
    steps = None
    if world == 1 and not args.no_step:
        names = [x for x in args.step_configs.split(",") if x]
        steps = radau_steps(names, cpu=not args.no_cpu, bw_gbs=peak)
    par = None
    if world > 1 and not args.no_step:
        par = stage_parallel_c4(args, rank, world, dev, peak)

    cpu = None
    if rank == 0 and not args.no_cpu and world == 1:
        cpu = cpu_sample(Q, k, tau, L)

    if rank == 0:
        launches_per_apply = 1 if op is None else op.launches_per_apply
        line = {"impl": "ours", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic U[-1,1] fp64, seed 42 (+rank)",
                "config": config_dict(args, world),
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "traffic": traffic,
                             "peak_source": peak_kind, "kernel": "stage_apply_kernel<4,3,coupled,store>",
                             "kernel_ms": kern_ms, "alg_bytes_per_launch": alg_bytes},
                # k = 4 in fp64 is co-bound by the FP64 pipe: algorithmic flops of
                # the flop-minimal Kronecker form, 2*(8(k+2)+2Q) per stage-DoF,
                # against the measured DFMA peak (tools/ubench/fp64.cu)
                "fp64_pipe": {"achieved": FLOPS_PER_SDOF * Q * n / (kern_ms * 1e-3) / 1e12,
                              "peak": fp64_peak, "unit": "TFLOP/s",
                              "frac": FLOPS_PER_SDOF * Q * n / (kern_ms * 1e-3) / 1e12 / fp64_peak,
                              "flops_per_stage_dof": FLOPS_PER_SDOF,
                              "peak_source": "measured in this run: DFMA throughput (spk_fp64_probe)"},
                "kernel_ms_single_launch": kern_single,
                "kernel_ms_best": kern_best,
                "constrained": None if cons_ms is None else {
                    "kernel_ms": cons_ms, "value": Q * n / (cons_ms * 1e-3), "unit": UNIT},
                "cpu_baseline": cpu,
                "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(u_host.numel() * 8),
                        "d2h_bytes_per_step": int(v_host.numel() * 8), "ms_per_step": e2e_ms},
                "gpu_launches": args.steps * launches_per_apply,
                "clocks": clk.summary(),
                "radau_steps": steps,
                "stage_parallel_step": par}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
