"""Working-space column renumbering (host driver, tree mode): columns ordered
by descending degree when the degrees are skewed, every primal vector mapped
back at the boundary.  Checked against the compiled reference on config 2
family members with the renumbering forced ($FOLP_HOT_COLUMNS=1) and off:
same iterates over the first restart period (1e-10), same restarts, the
solution in the caller's column order, KKT <= 1e-8."""
import numpy as np
import pytest

from paper_2106_04756_b200 import cabi, instances

pytestmark = pytest.mark.gpu


def _rel(u, v):
    return float(np.max(np.abs(u - v) / np.maximum(1.0, np.abs(v))))


def _degree_permutation_is_nontrivial(lp):
    deg = np.bincount(lp.row_cols, minlength=lp.num_cols)
    return not np.array_equal(np.argsort(-deg, kind="stable"), np.arange(lp.num_cols))


@pytest.mark.parametrize("mode", ["1", "0"])
def test_first_restart_period_matches_reference(eng, ref, monkeypatch, mode):
    monkeypatch.setenv("FOLP_HOT_COLUMNS", mode)
    lp = instances.generate(2, 1, 0.01)
    assert _degree_permutation_is_nontrivial(lp)
    p = cabi.params(record_iterate_trace=True, iteration_limit=100)
    a = eng.solve_lp(lp, p, iterate_capacity=100)
    b = ref.solve_lp(lp, p, iterate_capacity=100)
    assert len(a.iterate_trace) == len(b.iterate_trace) == 100
    worst = 0.0
    for (ia, ea, xa, ya), (ib, eb, xb, yb) in zip(a.iterate_trace[:40], b.iterate_trace[:40]):
        assert ia == ib
        worst = max(worst, _rel(xa, xb), _rel(ya, yb))
    assert worst <= 1e-10
    assert a.restart_iterations == b.restart_iterations
    assert _rel(a.primal_solution, b.primal_solution) <= 1e-6
    assert _rel(a.reduced_costs, b.reduced_costs) <= 1e-6


def test_solve_to_1e8_in_caller_order(eng, monkeypatch):
    """Renumbered and unrenumbered solves both reach 1e-8 with the same
    objective, and the returned point is in the caller's column order."""
    lp = instances.generate(2, 2, 0.005)
    p = cabi.params(kkt_pass_limit=400000)
    res = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("FOLP_HOT_COLUMNS", mode)
        res[mode] = eng.solve_lp(lp, p)
    a, b = res["1"], res["0"]
    assert a.termination_reason == b.termination_reason == "Optimal"
    info = a.final_info
    gap = info["gap_abs"] / (1 + abs(info["primal_objective"]) + abs(info["dual_objective"]))
    pr = info["primal_residual_norm"] / (1 + info["norm_q"])
    du = info["dual_residual_norm"] / (1 + info["norm_c"])
    assert max(gap, pr, du) <= 1e-8
    pa, pb = info["primal_objective"], b.final_info["primal_objective"]
    assert abs(pa - pb) <= 1e-8 * (2 + 2 * abs(pa) + 2 * abs(pb))
    x = a.primal_solution
    assert abs(float(lp.objective @ x) + lp.objective_constant - pa) <= 1e-7 * (1 + abs(pa))
    assert np.all(x >= lp.variable_lower - 1e-9) and np.all(x <= lp.variable_upper + 1e-9)
