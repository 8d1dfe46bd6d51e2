"""Timing model of the stage-parallel method (SPEC perfmodel; §4,
eq. time:irk / time:spirk) and its validation against the solver's V-cycle counters.

Model time is in cost units (V-cycle counts, or measured milliseconds when the caller has them):

  predict_irk    T = 2 T_S + sum_q T_Bq          (one process handles all stages)
  predict_spirk  T = 2 T_S' + max_q T_Bq         (stage groups in parallel)
  speedup_bound  sum_q T_Bq / max_q T_Bq <= Q

Per-stage block costs are either given directly (t_block) or as per-iteration cost x iteration count
(t_iter, n_iter: the "limit" form of §4). `validate_against_counters` checks the V-cycle bookkeeping
of a run (#V = Q (#G + 1) per step in the real-LU path, critical path = max over stage groups) and
`write_solve_log` emits the per-step CSV (step, t, iterations, V-cycles, converged, error).
"""

import csv
from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigurationError


@dataclass
class CostModel:
    t_basis: float = 0.0
    t_block: list = field(default_factory=list)
    t_iter: list = None
    n_iter: list = None

    def __post_init__(self):
        if self.t_iter is not None or self.n_iter is not None:
            if self.t_iter is None or self.n_iter is None or len(self.t_iter) != len(self.n_iter):
                raise ConfigurationError("iteration form needs t_iter and n_iter of equal length")
            self.t_block = [float(a) * float(b) for a, b in zip(self.t_iter, self.n_iter)]
        if self.t_basis < 0 or any(t < 0 for t in self.t_block):
            raise ConfigurationError("costs must be non-negative")
        if not self.t_block:
            raise ConfigurationError("need at least one block cost")

    @property
    def Q(self):
        return len(self.t_block)


def predict_irk(model):
    """eq. time:irk: total runtime when one process handles every stage."""
    return 2.0 * model.t_basis + float(np.sum(model.t_block))


def predict_spirk(model):
    """eq. time:spirk: runtime with the stage blocks in parallel (critical path)."""
    return 2.0 * model.t_basis + float(np.max(model.t_block))


def speedup_bound(model):
    """sum_q T_Bq / max_q T_Bq (<= Q; equal blocks reach Q)."""
    m = float(np.max(model.t_block))
    return float(np.sum(model.t_block)) / m if m > 0 else 1.0


@dataclass
class Validation:
    ok: bool
    steps: int
    avg_gmres: float
    critical_vcycles: float
    sequential_vcycles: float
    predicted_speedup: float
    mismatches: list


def validate_against_counters(reports, Q, per_group_vcycles=None):
    """Check the V-cycle counters of a run of real-LU steps (SolveReport list).

    Each GMRES iteration applies P^-1 once (one V-cycle per stage block) and the final
    x = P^-1(V y) once more, so per step: vcycles_per_stage = its + 1 and vcycles_total = Q (its + 1).
    With the stage blocks on separate groups the critical path is max_q of the per-group counts
    (`per_group_vcycles`, default: every group ran vcycles_per_stage) and the sequential total is
    their sum; the predicted speedup is their ratio (= Q here since the real-LU path shares the
    outer iteration count)."""
    mism = []
    its = [r.iterations for r in reports]
    for i, r in enumerate(reports):
        if r.vcycles_per_stage != r.iterations + 1:
            mism.append(f"step {i}: vcycles_per_stage {r.vcycles_per_stage} != its + 1 = {r.iterations + 1}")
        if r.vcycles_total != Q * (r.iterations + 1):
            mism.append(f"step {i}: vcycles_total {r.vcycles_total} != Q (its + 1) = {Q * (r.iterations + 1)}")
    per_group = per_group_vcycles
    if per_group is None:
        per_group = [sum(r.vcycles_per_stage for r in reports)] * Q
    if len(per_group) != Q:
        mism.append(f"{len(per_group)} group counts for Q = {Q}")
    seq = float(sum(r.vcycles_total for r in reports))
    crit = float(max(per_group)) if per_group else 0.0
    if abs(float(sum(per_group)) - seq) > 0:
        mism.append(f"sum of per-group V-cycles {sum(per_group)} != sequential total {seq}")
    if crit * Q < seq:
        mism.append("critical path x Q below the sequential total")
    n = max(len(reports), 1)
    return Validation(not mism, len(reports), float(np.mean(its)) if its else 0.0, crit / n, seq / n,
                      seq / crit if crit > 0 else 1.0, mism)


def write_solve_log(path, rows):
    """Per-step CSV (one-line header): step, t, iterations, vcycles_per_stage, vcycles_total,
    converged, l2_error (rows: dicts with those keys; missing keys are left empty)."""
    cols = ["step", "t", "iterations", "vcycles_per_stage", "vcycles_total", "converged", "l2_error"]
    with open(path, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=cols, extrasaction="ignore")
        w.writeheader()
        for r in rows:
            w.writerow(r)
    return path
