"""bench.py contract: one JSON line with the driver's keys, on 1 GPU, on 2 ranks (torchrun, two
processes sharing the test box's GPU over gloo -- functional only), and the reference arm under
torchrun (rank 0 alone prints)."""

import json
import os
import socket
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config"]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(args, nproc=1, env=None, timeout=600):
    e = dict(os.environ)
    e.update(env or {})
    if nproc > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", *args]
    else:
        cmd = [sys.executable, "bench.py", *args]
    r = subprocess.run(cmd, cwd=REPO, env=e, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    return json.loads(lines[0])


def test_reference_arm_under_torchrun():
    d = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1", "--level", "3"], nproc=2)
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["same_config"] and d["cpu_baseline"]["cores"] >= 1
    for k in KEYS:
        assert k in d, k
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"


@pytest.mark.gpu
def test_bench_single_gpu_line():
    d = _run(["--steps", "3", "--warmup", "3", "--level", "4", "--no-cpu", "--no-step"])
    for k in KEYS + ["roofline", "e2e", "gpu_launches", "clocks", "fp64_pipe"]:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] == 3
    assert 0 < d["roofline"]["frac"] < 1 and d["e2e"]["h2d_bytes_per_step"] > 0


@pytest.mark.gpu
def test_bench_step_entries():
    """Per-config Radau IIA step entries (C1 here: the smallest) with iterations, V-cycles and the
    step-level HBM fraction, plus the C1 CPU oracle step."""
    d = _run(["--steps", "3", "--warmup", "3", "--level", "4", "--step-configs", "C1"])
    e = d["radau_steps"]["C1"]
    assert e["ms_per_step"] > 0 and len(e["gmres_iterations"]) == e["steps_timed"] == 9
    assert all(v == i + 1 for v, i in zip(e["vcycles_per_stage"], e["gmres_iterations"]))
    assert 0 < e["hbm_frac"] < 1.5 and e["cpu_baseline"]["ms_per_step"] > 0
    assert d["cpu_baseline"]["same_config"] and d["fp64_pipe"]["peak"] > 10


@pytest.mark.gpu
def test_bench_two_ranks_shared_gpu():
    d = _run(["--gpus", "2", "--steps", "3", "--warmup", "3", "--level", "4", "--no-cpu", "--sp-level", "3"],
             nproc=2, env={"BENCH_SHARE_GPU": "1", "BENCH_DIST_BACKEND": "gloo"})
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["parallelism"].startswith("x-slab")
    sp = d["stage_parallel_step"]
    assert sp["grid"].startswith("S=2 x B=1") and sp["ms_per_step"] > 0 and len(sp["gmres_iterations"]) == 4
