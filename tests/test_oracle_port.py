"""Pins the oracle: the C restatement (oracle/pdlp_port.c) must equal the
compiled reference (oracle/_ref, built from /root/reference/proj/src) bit
for bit -- iterates, step sizes, restarts, traces, solutions, ledger -- on
the reference's own instance generators and on members of the five
BASELINE families.  CPU only."""
import math

import numpy as np
import pytest

from oracle import port
from paper_2106_04756_b200 import cabi, instances


@pytest.fixture(scope="module")
def prt():
    return port.binding()


def _same_result(a, b, iterates=True):
    assert a.termination_reason == b.termination_reason
    assert a.iterations == b.iterations
    assert a.kkt_passes == b.kkt_passes
    assert a.restarts == b.restarts
    assert a.step_trials == b.step_trials
    assert a.restart_iterations == b.restart_iterations
    assert a.final_info == b.final_info
    assert np.array_equal(a.primal_solution, b.primal_solution)
    assert np.array_equal(a.dual_solution, b.dual_solution)
    assert np.array_equal(a.reduced_costs, b.reduced_costs)
    assert len(a.trace) == len(b.trace)
    for ta, tb in zip(a.trace, b.trace):
        assert ta == tb
    if iterates:
        assert len(a.iterate_trace) == len(b.iterate_trace)
        for (ia, ea, xa, ya), (ib, eb, xb, yb) in zip(a.iterate_trace, b.iterate_trace):
            assert ia == ib and ea == eb
            assert np.array_equal(xa, xb) and np.array_equal(ya, yb)


def test_port_products_and_scaling_bit_exact(ref, prt):
    lp = instances.generate(2, 3, 0.02)
    rng = np.random.default_rng(0)
    x = rng.standard_normal(lp.num_cols)
    y = rng.standard_normal(lp.num_rows)
    assert np.array_equal(prt.kx(lp, x), ref.kx(lp, x))
    assert np.array_equal(prt.kty(lp, y), ref.kty(lp, y))
    a, b = prt.rescale_lp(lp), ref.rescale_lp(lp)
    for k in a:
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("cfg,scale,seed", [(1, 0.25, 1), (1, 0.25, 2), (2, 0.005, 1),
                                            (3, 0.0001, 1), (5, 0.01, 1), (4, 0.00002, 1)])
def test_port_matches_reference_with_iterates(ref, prt, cfg, scale, seed):
    lp = instances.generate(cfg, seed, scale)
    p = cabi.params(record_iterate_trace=True, iteration_limit=300)
    _same_result(prt.solve_lp(lp, p, iterate_capacity=300), ref.solve_lp(lp, p, iterate_capacity=300))


@pytest.mark.parametrize("policy,scheme", [("adaptive", "pdlp"), ("constant", "none"),
                                           ("malitsky_pock", "pdlp"), ("adaptive", "theory"),
                                           ("adaptive", "none")])
def test_port_policies_and_schemes(ref, prt, policy, scheme):
    from oracle import ref as R
    lp = R.random_feasible(77, 6, 3, 9, 1.0)
    p = cabi.params(step_policy=policy, restart_scheme=scheme, iteration_limit=2000)
    _same_result(prt.solve_lp(lp, p), ref.solve_lp(lp, p), iterates=False)


def test_port_full_solve_config1(ref, prt):
    lp = instances.generate(1, 1, 0.25)
    _same_result(prt.solve_lp(lp), ref.solve_lp(lp), iterates=False)


def test_port_reference_generators(ref, prt):
    from oracle import ref as R
    for lp in (R.pagerank(60, 3, 5), R.random_feasible(5003, 16, 6, 15, 2.5)):
        _same_result(prt.solve_lp(lp, cabi.params(kkt_pass_limit=20000)),
                     ref.solve_lp(lp, cabi.params(kkt_pass_limit=20000)), iterates=False)


def test_port_step_level(ref, prt):
    lp = instances.generate(1, 4, 0.1)
    rng = np.random.default_rng(5)
    x = np.clip(rng.uniform(0, 3, lp.num_cols), lp.variable_lower, lp.variable_upper)
    y = rng.standard_normal(lp.num_rows)
    y[:lp.num_inequality_rows] = np.abs(y[:lp.num_inequality_rows])
    a, b = prt.step(lp, x, y, 0.7, 20.0, 3), ref.step(lp, x, y, 0.7, 20.0, 3)
    for k in a:
        assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k
    assert prt.ndg(lp, x, y, 2.0, 0.7) == ref.ndg(lp, x, y, 2.0, 0.7)
    assert prt.info(lp, x, y) == ref.info(lp, x, y)


def test_port_refuses_non_identity_presolve(prt):
    from oracle import ref as R
    from paper_2106_04756_b200.cabi import FolpError
    lp, _ = R.handcrafted()[2]  # pinned_by_equality keeps presolve trivial? check both
    fixed = cabi.LP(1, 2, 0, np.array([0, 1]), np.array([0]), np.array([1.0]),
                    np.array([1.0, 0.0]), np.array([0.5]), np.array([0.0, 0.0]),
                    np.array([1.0, 0.0]))  # column 1 fixed at 0 and empty
    with pytest.raises(FolpError):
        prt.solve_lp(fixed)
    assert math.isfinite(prt.solve_lp(lp).final_info["primal_objective"])
