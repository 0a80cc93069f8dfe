"""Golden vectors produced by the compiled reference (tools/make_golden.py ->
tests/golden/reference_solves.json).  CPU: the C restatement (oracle) must
reproduce them bit for bit (solution hashes, per-iterate hashes and step
sizes, restarts, ledger).  GPU: the B200 engine must reach the same
termination with the north_star tolerances."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import port
from paper_2106_04756_b200 import cabi, instances
from paper_2106_04756_b200.cabi import FolpError

GOLDEN = json.loads((Path(__file__).parent / "golden" / "reference_solves.json").read_text())
CASE_NAMES = sorted(k for k in GOLDEN if k != "handcrafted_suite")


def _make(name):
    if name.startswith("cfg"):
        cfg = int(name[3])
        seed = int(name.split("_s")[1].split("_")[0])
        scale = float(name.split("_x")[1].split("_")[0])
        return instances.generate(cfg, seed, scale)
    from oracle import ref as R
    if not R.available():
        pytest.skip("reference generators need oracle/_ref")
    if name == "ref_pagerank_n200_s5":
        return R.pagerank(200, 3, 5)
    if name == "ref_random_feasible_5003":
        return R.random_feasible(5003, 16, 6, 15, 2.5)
    if name == "ref_random_feasible_1000_constant":
        return R.random_feasible(1000, 4, 2, 5, 0.5)
    raise KeyError(name)


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def _check_bitwise(r, g):
    assert r.termination_reason == g["termination_reason"]
    assert r.iterations == g["iterations"]
    assert r.kkt_passes == g["kkt_passes"]
    assert r.restart_iterations == g["restart_iterations"]
    assert {k: float(v).hex() for k, v in r.final_info.items()} == g["final_info"]
    assert _digest(r.primal_solution) == g["primal_sha256"]
    assert _digest(r.dual_solution) == g["dual_sha256"]
    assert _digest(r.reduced_costs) == g["reduced_costs_sha256"]
    its = [_digest(np.concatenate([x, y])) for (_, _, x, y) in r.iterate_trace]
    assert its == g["iterate_sha256"]
    assert [float(e).hex() for (_, e, _, _) in r.iterate_trace] == g["iterate_eta"]


@pytest.mark.parametrize("name", CASE_NAMES)
def test_oracle_reproduces_reference_golden(name):
    case = GOLDEN[name]
    lp = _make(name)
    assert (lp.num_rows, lp.num_cols, lp.nnz) == (case["m"], case["n"], case["nnz"])
    n_it = len(case["result"]["iterate_sha256"])
    r = port.solve(lp, cabi.params(**case["params"]), iterate_capacity=n_it)
    _check_bitwise(r, case["result"])


def test_oracle_handcrafted_golden():
    from oracle import ref as R
    if not R.available():
        pytest.skip("handcrafted instances come from oracle/_ref")
    checked = 0
    for (lp, obj), g in zip(R.handcrafted(), GOLDEN["handcrafted_suite"]):
        assert lp.name == g["name"]
        try:
            r = port.solve(lp)
        except FolpError as e:  # presolve not restated in the port
            assert "presolve" in str(e)
            continue
        _check_bitwise(r, g["result"])
        checked += 1
    assert checked >= 6


def _rel_kkt(info):
    gap = info["gap_abs"] / (1 + abs(info["primal_objective"]) + abs(info["dual_objective"]))
    return max(gap, info["primal_residual_norm"] / (1 + info["norm_q"]),
               info["dual_residual_norm"] / (1 + info["norm_c"]))


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASE_NAMES)
def test_engine_against_reference_golden(eng, name):
    case = GOLDEN[name]
    g = case["result"]
    lp = _make(name)
    r = eng.solve_lp(lp, cabi.params(**case["params"]))
    assert r.termination_reason == g["termination_reason"]
    if g["termination_reason"] == "Optimal":
        assert _rel_kkt(r.final_info) <= case["params"].get("eps_optimal", 1e-8)
        want = float.fromhex(g["final_info"]["primal_objective"])
        assert r.final_info["primal_objective"] == pytest.approx(want, rel=1e-8, abs=1e-8)
        assert abs(r.iterations - g["iterations"]) <= max(40, 0.05 * g["iterations"])
    else:
        assert r.iterations == g["iterations"]
        assert r.restart_iterations == g["restart_iterations"]


@pytest.mark.gpu
def test_engine_handcrafted_golden(eng):
    from oracle import ref as R
    if not R.available():
        pytest.skip("handcrafted instances come from oracle/_ref")
    for (lp, obj), g in zip(R.handcrafted(), GOLDEN["handcrafted_suite"]):
        r = eng.solve_lp(lp)
        assert r.termination_reason == g["result"]["termination_reason"] == "Optimal", lp.name
        assert abs(r.final_info["primal_objective"] - obj) <= 1e-6 * max(1.0, abs(obj))
        assert _rel_kkt(r.final_info) <= 1e-8
