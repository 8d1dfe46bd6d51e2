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
METRIC = "stage-DoFs/s of batched matrix-free apply (C2: 64^3 Q4 hex, Radau IIA Q=3)"
UNIT = "stage-DoF/s"
FLOPS_PER_SDOF = 2 * (8 * (CFG["degree"] + 2) + 2 * CFG["Q"])  # 108 for C2
FP64_PEAK_TFS = 34.2


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    p.add_argument("--no-step", action="store_true", help="skip the Radau IIA step timing (C3)")
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


def radau_step_sample(steps=4, cpu=True):
    """Time per Radau IIA step of C3 (BASELINE.json configs[2]: 32^3 Q2 hex, Q=3, tau=0.01, GMRES
    rtol 1e-12, Chebyshev degree 3) on this GPU: the second half of the metric ("time per Radau IIA
    step"). Device-resident state, CUDA events around `steps` steps after one warm-up step."""
    import torch

    from paper_2209_06700_b200.fem import build_hierarchy
    from paper_2209_06700_b200.irk import StageSystem
    from paper_2209_06700_b200.multigrid import VCycleConfig

    tau = 0.01
    ss = StageSystem(build_hierarchy(3, 5, 2), 3, tau, config=VCycleConfig(smoother_degree=3))
    u = ss.initial_condition()
    u, _ = ss.step(0.0, u)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    its = []
    e0.record()
    for i in range(steps):
        u, rep = ss.step((i + 1) * tau, u)
        its.append(rep.iterations)
    e1.record()
    torch.cuda.synchronize()
    out = {"config": "C3 (32^3 Q2 hex, Radau IIA Q=3, tau=0.01, rtol 1e-12, Chebyshev deg 3)",
           "ms_per_step": e0.elapsed_time(e1) / steps, "steps": steps, "gmres_iterations": its,
           "n_gpus": 1, "note": "per-config step times (C1, C3, C4, C5): tools/bench_steps.py, "
                                "profiles/r01_steps.jsonl"}
    if cpu:
        out["cpu_baseline"] = cpu_step_sample(tau)
    return out


def cpu_step_sample(tau):
    """The oracle (the reference's algorithm: dense-1D contractions, numpy) running the same C3 step
    on all host cores: one step after setup (~5-10 s)."""
    import threadpoolctl
    from oracle import solvers as OS
    from oracle import stepper as OST
    from oracle.fem_qk import Hierarchy
    from oracle.tableau_ref import radau_iia as ref_radau

    cores = len(os.sched_getaffinity(0))
    with threadpoolctl.threadpool_limits(cores):
        ora = OST.RealLU(Hierarchy(3, 5, 2), 3, tau, OS.Config(smoother_degree=3), tab=ref_radau(3))
        uo = ora.initial()
        t0 = time.perf_counter()
        uo, its, _ = ora.step(0.0, uo)
        dt = time.perf_counter() - t0
    return {"ms_per_step": dt * 1e3, "cores": cores, "kind": "port", "gmres_iterations": its,
            "sample": "one C3 step of the oracle (first step from the initial condition)"}


def cpu_sample(Q, degree, tau, seconds=10.0):
    """Oracle (reference-as-written algorithm, numpy/OpenBLAS) on a bounded sample."""
    import threadpoolctl
    from oracle.fem_qk import Hierarchy
    from paper_2209_06700_b200.tableau import radau_iia

    cores = len(os.sched_getaffinity(0))
    lvl = 5
    with threadpoolctl.threadpool_limits(cores):
        h = Hierarchy(3, lvl, degree)
        n = h.levels[lvl].n_dofs
        u = np.random.default_rng(CFG["seed"]).uniform(-1.0, 1.0, size=(Q, n))
        A = radau_iia(Q).A
        DM, DK = np.eye(Q), tau * A
        h.apply_stage(lvl, DM, DK, u)  # warm
        t0 = time.perf_counter()
        reps = 0
        while True:
            h.apply_stage(lvl, DM, DK, u)
            reps += 1
            if time.perf_counter() - t0 > seconds:
                break
        dt = (time.perf_counter() - t0) / reps
    return {"value": Q * n / dt, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{reps} oracle applies at 32^3 cells (level 5, n={n}/stage, k={degree}, Q={Q}); "
                      f"dense-1D contraction cost per DoF grows with n_ax, so the full 64^3 CPU rate is "
                      f"about 2x lower than this sample", "seconds_per_apply": dt}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    Q, k, tau = CFG["Q"], CFG["degree"], CFG["tau"]
    import threadpoolctl
    from oracle.fem_qk import Hierarchy
    from paper_2209_06700_b200.tableau import radau_iia

    cores = len(os.sched_getaffinity(0))
    lvl = 5
    with threadpoolctl.threadpool_limits(cores):
        h = Hierarchy(3, lvl, k)
        n = h.levels[lvl].n_dofs
        u = np.random.default_rng(CFG["seed"]).uniform(-1.0, 1.0, size=(Q, n))
        DM, DK = np.eye(Q), tau * radau_iia(Q).A
        for _ in range(args.warmup):
            h.apply_stage(lvl, DM, DK, u)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            h.apply_stage(lvl, DM, DK, u)
        dt = (time.perf_counter() - t0) / args.steps
    val = Q * n / dt
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic U[-1,1] seed 42",
            "config": config_dict(args, 1, {"cpu_level": lvl}),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"each step = one oracle apply at 32^3 cells (n={n}/stage, k={k}, "
                                       f"Q={Q}); the reference is pure numpy (k=1 only), the oracle is its "
                                       f"algorithm generalised to Q_k"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


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
    kern_ms = sorted(kern_ms)[len(kern_ms) // 2]
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

    cpu = None
    if rank == 0 and not args.no_cpu and world == 1:
        cpu = cpu_sample(Q, k, tau)

    step = None
    if rank == 0 and world == 1 and not args.no_step:
        step = radau_step_sample(cpu=not args.no_cpu)

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
                              "peak": FP64_PEAK_TFS, "unit": "TFLOP/s",
                              "frac": FLOPS_PER_SDOF * Q * n / (kern_ms * 1e-3) / 1e12 / FP64_PEAK_TFS,
                              "flops_per_stage_dof": FLOPS_PER_SDOF,
                              "peak_source": "measured DFMA throughput, tools/ubench/fp64.cu"},
                "kernel_ms_best": kern_best,
                "constrained": None if cons_ms is None else {
                    "kernel_ms": cons_ms, "value": Q * n / (cons_ms * 1e-3), "unit": UNIT},
                "cpu_baseline": cpu,
                "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(u_host.numel() * 8),
                        "d2h_bytes_per_step": int(v_host.numel() * 8), "ms_per_step": e2e_ms},
                "gpu_launches": args.steps * launches_per_apply,
                "clocks": clk.summary(),
                "radau_step": step}
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
