"""End-to-end parity of folp::solve on the B200 against the compiled
reference: per-iterate agreement (1e-10 relative over the first 100
iterations), identical restart decisions, final relative KKT <= 1e-8,
objective within 1e-8 relative, iteration counts within 5 %
(BASELINE.json north_star)."""
import numpy as np
import pytest

from paper_2106_04756_b200 import cabi, instances

pytestmark = pytest.mark.gpu


def _rel_kkt(info):
    gap = info["gap_abs"] / (1 + abs(info["primal_objective"]) + abs(info["dual_objective"]))
    pr = info["primal_residual_norm"] / (1 + info["norm_q"])
    du = info["dual_residual_norm"] / (1 + info["norm_c"])
    return max(gap, pr, du)


def _iterate_drift(a, b, count):
    worst = 0.0
    for (ia, ea, xa, ya), (ib, eb, xb, yb) in zip(a[:count], b[:count]):
        assert ia == ib
        for u, v in ((xa, xb), (ya, yb)):
            worst = max(worst, float(np.max(np.abs(u - v) / np.maximum(1.0, np.abs(v)), initial=0)))
    return worst


def test_cfg1_iterates_first_100(eng, ref):
    lp = instances.generate(1, 1, 1.0)
    p = cabi.params(record_iterate_trace=True, iteration_limit=100)
    a = eng.solve_lp(lp, p, iterate_capacity=100)
    b = ref.solve_lp(lp, p, iterate_capacity=100)
    assert len(a.iterate_trace) == len(b.iterate_trace) == 100
    assert _iterate_drift(a.iterate_trace, b.iterate_trace, 100) <= 1e-10
    assert a.restart_iterations == b.restart_iterations
    assert a.kkt_passes == b.kkt_passes


def test_cfg1_solve_to_1e8(eng, ref):
    lp = instances.generate(1, 1, 1.0)
    a = eng.solve_lp(lp)
    b = ref.solve_lp(lp)
    assert a.termination_reason == b.termination_reason == "Optimal"
    assert _rel_kkt(a.final_info) <= 1e-8
    assert a.final_info["primal_objective"] == pytest.approx(b.final_info["primal_objective"],
                                                             rel=1e-8)
    assert abs(a.iterations - b.iterations) <= 0.05 * b.iterations
    assert a.step_condition_violations == 0


def test_handcrafted_suite(eng, ref):
    from oracle import ref as R
    for lp, objective in R.handcrafted():
        a = eng.solve_lp(lp)
        b = ref.solve_lp(lp)
        assert a.termination_reason == "Optimal", lp.name
        assert abs(a.final_info["primal_objective"] - objective) <= 1e-6 * max(1, abs(objective))
        assert a.restart_iterations == b.restart_iterations, lp.name
