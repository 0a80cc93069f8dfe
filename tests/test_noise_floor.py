"""The reference's own reduction-order noise floor (test infrastructure the
tree-mode GPU tests are held to, tests/_parity.py), pinned on the CPU:

* the iteration-spread fixture (tests/golden/iteration_spread.json, from
  tools/noise_floor_iterations.py --fixture) reproduces -- the reference's
  iteration counts and those of its re-associated restatements -- on the
  instances cheap enough to re-solve here;
* re-associating the sums is all a sum order changes: order 0 of the
  restatement is bit-identical to the compiled reference, and the floor is
  zero for it;
* the floor grows with the iterate index (the step rule amplifies the
  last-bit differences), so a fixed 1e-10 over 100 iterates is not a bar
  any parallel summation can meet on these instances."""
import ctypes as C
import json
from pathlib import Path

import pytest

from paper_2106_04756_b200 import cabi, instances

from _parity import drift_curve, reference_floor

SPREAD = json.loads((Path(__file__).parent / "golden" / "iteration_spread.json").read_text())


@pytest.mark.parametrize("key", ["cfg1_s1_x1.0", "cfg5_s3_x0.02"])
def test_iteration_spread_fixture_reproduces(ref, key):
    from oracle import port
    row = SPREAD[key]
    lp = instances.generate(row["config"], row["seed"], row["scale"])
    want = ref.solve_lp(lp, trace_capacity=4096)
    assert want.iterations == row["ref"]["iterations"]
    assert want.termination_reason == row["ref"]["termination"]
    lib = port.binding().lib
    lib.folp_port_set_sum_order.argtypes = [C.c_int]
    lib.folp_port_set_sum_order(2)
    try:
        got = port.binding().solve_lp(lp, trace_capacity=4096)
    finally:
        lib.folp_port_set_sum_order(0)
    assert got.iterations == row["order2"]["iterations"]


def test_floor_is_zero_for_the_reference_order_and_grows(ref):
    from oracle import port
    lp = instances.generate(2, 1, 0.01)
    p = cabi.params(record_iterate_trace=True, iteration_limit=100)
    want = ref.solve_lp(lp, p, iterate_capacity=100)
    same = port.solve(lp, p, iterate_capacity=100)
    assert max(drift_curve(same.iterate_trace, want.iterate_trace)) == 0.0
    floor = reference_floor(lp, p, 100, want)
    assert floor[9] < 1e-9 and floor[99] > 1e-10 and floor[99] >= floor[39] >= floor[9]
