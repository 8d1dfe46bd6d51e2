"""Time per Radau IIA step for the BASELINE.json configs (C1, C3, C4, C5) on one GPU.

usage: python tools/bench_steps.py [C1 C3 C4 C5] [--steps N] [--oracle-steps M]
Prints one JSON line per config: ms/step (CUDA events, device-resident state), GMRES iterations per
step, V-cycles, L2 error vs the manufactured solution, and optionally the CPU oracle's time for M
steps on the host cores (bounded sample).
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_06700_b200.complex_solver import DirectComplexSystem  # noqa: E402
from paper_2209_06700_b200.fem import build_hierarchy  # noqa: E402
from paper_2209_06700_b200.irk import StageSystem  # noqa: E402
from paper_2209_06700_b200.multigrid import VCycleConfig  # noqa: E402

CONFIGS = {
    "C1": dict(dim=2, L=4, k=2, Q=2, tau=0.05, steps=10, rtol=1e-10, deg=5, path="real"),
    "C3": dict(dim=3, L=5, k=2, Q=3, tau=0.01, steps=20, rtol=1e-12, deg=3, path="real"),
    "C4": dict(dim=3, L=7, k=2, Q=4, tau=1e-3, steps=5, rtol=1e-12, deg=3, path="real"),
    "C5": dict(dim=3, L=6, k=3, Q=3, tau=5e-3, steps=10, rtol=1e-12, deg=3, path="presb"),
}


def exact(dim):
    return lambda x, t: np.prod(np.sin(np.pi * x), axis=1) * np.exp(-t)


def run(name, steps=None, oracle_steps=0):
    c = CONFIGS[name]
    steps = steps or c["steps"]
    h = build_hierarchy(c["dim"], c["L"], c["k"])
    cfg = VCycleConfig(smoother_degree=c["deg"])
    t0 = time.perf_counter()
    if c["path"] == "real":
        sys_ = StageSystem(h, c["Q"], c["tau"], config=cfg, rel_tol=c["rtol"])
    else:
        sys_ = DirectComplexSystem(h, c["Q"], c["tau"], variant=c["path"], config=cfg, rel_tol=c["rtol"])
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    u = sys_.initial_condition()
    # warm-up step (not timed), then the timed steps from t = tau
    u, _ = sys_.step(0.0, u)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    its = []
    e0.record()
    t = c["tau"]
    for _ in range(steps - 1):
        u, rep = sys_.step(t, u)
        its.append(rep.block_iterations if rep.block_iterations else rep.iterations)
        t += c["tau"]
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / max(1, steps - 1)
    err = h.l2_error(c["L"], u, exact(c["dim"]), t)
    n = h.levels[c["L"]].n_dofs
    out = {"config": name, "n_per_stage": n, "Q": c["Q"], "degree": c["k"], "ms_per_step": ms,
           "stage_dofs_per_s_step": c["Q"] * n / (ms * 1e-3), "iterations": its, "l2_error": err,
           "setup_s": setup_s, "steps_timed": steps - 1}
    if oracle_steps:
        import threadpoolctl
        from oracle import solvers as OS
        from oracle import stepper as OST
        from oracle.fem_qk import Hierarchy
        cores = len(os.sched_getaffinity(0))
        with threadpoolctl.threadpool_limits(cores):
            o = Hierarchy(c["dim"], c["L"], c["k"])
            ocfg = OS.Config(smoother_degree=c["deg"])
            if c["path"] == "real":
                osys = OST.RealLU(o, c["Q"], c["tau"], ocfg, rel_tol=c["rtol"])
            else:
                osys = OST.DirectComplex(o, c["Q"], c["tau"], c["path"], ocfg, rel_tol=c["rtol"])
            uo = osys.initial()
            t1 = time.perf_counter()
            for s in range(oracle_steps):
                res = osys.step(s * c["tau"], uo)
                uo = res[0]
            out["cpu_oracle_s_per_step"] = (time.perf_counter() - t1) / oracle_steps
            out["cpu_cores"] = cores
    print(json.dumps(out), flush=True)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["C1", "C3", "C5", "C4"])
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--oracle-steps", type=int, default=0)
    a = ap.parse_args()
    for name in a.configs:
        run(name, a.steps, a.oracle_steps)
