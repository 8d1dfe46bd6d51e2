"""SPEC perfmodel examples and counter validation."""

import numpy as np
import pytest

from paper_2209_06700_b200.errors import ConfigurationError
from paper_2209_06700_b200.irk import SolveReport
from paper_2209_06700_b200.perfmodel import (CostModel, predict_irk, predict_spirk, speedup_bound,
                                             validate_against_counters, write_solve_log)


def test_closed_forms():
    assert predict_irk(CostModel(0.0, [1, 1, 1, 1])) == 4
    assert predict_irk(CostModel(0.5, [1, 2, 3])) == 7
    assert predict_irk(CostModel(t_iter=[1, 1], n_iter=[5, 5])) == 10
    assert predict_spirk(CostModel(0.0, [1, 1, 1, 1])) == 1
    assert predict_spirk(CostModel(0.5, [1, 2, 3])) == 4
    assert predict_spirk(CostModel(t_iter=[1, 1, 1, 1], n_iter=[12, 12, 13, 12])) == 13
    assert speedup_bound(CostModel(0.0, [1, 1, 1, 1])) == 4
    assert speedup_bound(CostModel(0.0, [1, 2, 3])) == 2
    rng = np.random.default_rng(5)
    for Q in range(1, 10):
        m = CostModel(float(rng.uniform()), list(rng.uniform(0, 3, Q)))
        assert speedup_bound(m) <= Q + 1e-12
        assert predict_irk(m) >= predict_spirk(m)
    with pytest.raises(ConfigurationError):
        CostModel(0.0, [-1.0])
    with pytest.raises(ConfigurationError):
        CostModel(t_iter=[1], n_iter=[1, 2])


def _rep(its, Q):
    return SolveReport(iterations=its, vcycles_per_stage=its + 1, vcycles_total=Q * (its + 1), converged=True)


def test_validate_against_counters(tmp_path):
    v = validate_against_counters([_rep(7, 4), _rep(7, 4)], 4)
    assert v.ok and v.predicted_speedup == 4 and v.avg_gmres == 7 and v.critical_vcycles == 8
    v = validate_against_counters([_rep(5, 1)], 1)
    assert v.ok and v.predicted_speedup == 1
    # synthetic per-group counts [10, 10, 20] -> critical 20, bound 40 / 20 = 2
    reps = [SolveReport(iterations=0, vcycles_per_stage=1, vcycles_total=40, converged=True)]
    v = validate_against_counters(reps, 3, per_group_vcycles=[10, 10, 20])
    assert v.critical_vcycles == 20 and v.predicted_speedup == 2
    bad = SolveReport(iterations=3, vcycles_per_stage=3, vcycles_total=12)
    assert not validate_against_counters([bad], 4).ok
    p = write_solve_log(tmp_path / "log.csv", [dict(step=0, t=0.0, iterations=7, vcycles_per_stage=8,
                                                    vcycles_total=32, converged=True, l2_error=1e-3)])
    lines = open(p).read().strip().splitlines()
    assert lines[0] == "step,t,iterations,vcycles_per_stage,vcycles_total,converged,l2_error" and len(lines) == 2
