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


# ---- algorithmic HBM bytes of one Radau IIA step (SURVEY.md §8(d) "per-step model") ----------------
# Each math operation is counted at its minimal traffic (every operand vector read once, every result
# written once, 8 B per fp64 entry), whatever kernel split the device path uses; per-level Chebyshev /
# V-cycle counts follow multigrid.py:74-129. Levels at or below `fused_level` run inside one CTA
# (shared memory) and contribute nothing beyond their right-hand side and solution.

def vcycle_bytes(level_dofs, deg, fused_level=-1):
    """Bytes per block of one V-cycle over levels level_dofs[0..L] (DoFs per level, coarsest first)."""
    tot = 0.0
    for lvl in range(len(level_dofs) - 1, 0, -1):
        n = float(level_dofs[lvl])
        if lvl <= fused_level:
            tot += 16.0 * n          # the fused cycle reads b_lc, writes x_lc
            break
        pre = 16.0 + 48.0 * (deg - 1)        # d = Dinv b / theta; deg-1 steps (x, r, d read + written)
        post = 32.0 + 48.0 * (deg - 1)       # r = b - A x, d = Dinv r / theta; deg-1 steps
        resid = 24.0 + 8.0 + 8.0 / 8.0       # r = b - A x; restrict (read r, write the coarse rhs)
        prolong = 16.0 + 8.0 / 8.0           # x += P e_c
        tot += n * (pre + post + resid + prolong)
    else:
        tot += 16.0 * float(level_dofs[0])   # direct coarse solve (dense inverse: small)
    return tot


def gmres_bytes(N, its):
    """MGS columns (krylov.py:74-82), basis scaling, the final sum_i y_i v_i, the true residual."""
    tot = 16.0 * N                                     # beta = ||b||
    for j in range(its):
        tot += N * (16.0 + 32.0 * j + 24.0 + 16.0)     # <v0,w>; j fused (axpy, dot); last axpy + norm; scale
    tot += 8.0 * (its + 1) * N                         # sum_i y_i v_i
    tot += 24.0 * N                                    # ||b - A x||
    return tot


def real_step_bytes(level_dofs, Q, deg, its, fused_level=-1):
    """Real LU path (irk.StageSystem): rhs, (its + 1) x [A P^-1], GMRES, update."""
    n = float(level_dofs[-1])
    N = Q * n
    rhs = 16.0 * n + 8.0 * n + 8.0 * N                 # K u_n; source / A^-1 mix of Q rows
    pinv = 16.0 * N + Q * vcycle_bytes(level_dofs, deg, fused_level) + 16.0 * N   # S~^-1, V-cycles, S~
    op = 16.0 * N                                      # K1 coupled (A^-1 (x) M + tau I (x) K)
    update = 8.0 * (Q + 2) * n
    return rhs + (its + 1) * (pinv + op) + gmres_bytes(N, its) + update


def complex_step_bytes(level_dofs, Q, deg, block_its, variant="presb", fused_level=-1):
    """Direct complex path (complex_solver.DirectComplexSystem): rhs, S^-1, per pair block GMRES on
    the real 2x2 form with PRESB (2 V-cycles + 1 apply + 4 vector passes) or the 2x2 V-cycle, the real
    block with the plain V-cycle, S, update. block_its: GMRES iterations per block (pairs first)."""
    n = float(level_dofs[-1])
    N = Q * n
    tot = 16.0 * n + 8.0 * n + 8.0 * N + 2.0 * 16.0 * N + 8.0 * (Q + 2) * n
    npairs = Q // 2
    vc = vcycle_bytes(level_dofs, deg, fused_level)
    for b, its in enumerate(block_its):
        pair = b < npairs
        rows = 2 if pair else 1
        if pair and variant == "presb":
            pc = 2.0 * vc + 16.0 * n + 4.0 * 24.0 * n
        elif pair:
            pc = 2.0 * vc
        else:
            pc = vc
        tot += (its + 1) * (pc + 16.0 * rows * n) + gmres_bytes(rows * n, its)
    return tot
