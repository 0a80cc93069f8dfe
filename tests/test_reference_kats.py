"""Known-answer tests of the reference (proj/tests/test_solver.cpp,
test_termination.cpp, test_sparse_ops.cpp, test_scaling.cpp,
acceptance_main.cpp) restated over the folp_c.h boundary and run against
both the oracle (C restatement, CPU) and the B200 engine (GPU)."""
import math

import numpy as np
import pytest

from paper_2106_04756_b200 import cabi
from paper_2106_04756_b200.cabi import LP, FolpError

INF = math.inf


@pytest.fixture(params=["oracle", pytest.param("engine", marks=pytest.mark.gpu)])
def be(request):
    if request.param == "oracle":
        from oracle import port
        return port.binding()
    from paper_2106_04756_b200 import engine
    return engine()


def make(c, rows, cols, entries, q, m1, lo, hi):
    """make_lp / from_triplets for small hand instances (test_solver.cpp:30-41)."""
    dense = np.zeros((rows, cols))
    for r, k, v in entries:
        dense[r, k] += v
    rs, rc, rv = [0], [], []
    for r in range(rows):
        for k in range(cols):
            if dense[r, k] != 0.0:
                rc.append(k)
                rv.append(dense[r, k])
        rs.append(len(rc))
    return LP(rows, cols, m1, np.array(rs), np.array(rc, dtype=np.int64), np.array(rv),
              np.array(c, dtype=float), np.array(q, dtype=float), np.array(lo, dtype=float),
              np.array(hi, dtype=float))


def tiny():  # {min x : x >= 1, x >= 0}, optimum (1, 1)
    return make([1.0], 1, 1, [(0, 0, 1.0)], [1.0], 1, [0.0], [INF])


def knapsack():  # min -x1 - 2x2 : x1 + x2 <= 1, x >= 0
    return make([-1.0, -2.0], 1, 2, [(0, 0, -1.0), (0, 1, -1.0)], [-1.0], 1, [0.0, 0.0],
                [INF, INF])


# ---- sparse products (test_sparse_ops.cpp:47-64) ----
def test_products_hand_values(be):
    k = make([0, 0], 2, 2, [(0, 0, 1), (0, 1, 2), (1, 1, 3)], [0, 0], 0, [0, 0], [1, 1])
    assert list(be.kx(k, [1, 1])) == [3, 3]
    assert list(be.kx(k, [0, 0])) == [0, 0]
    assert list(be.kty(k, [1, 1])) == [1, 5]


def test_adjoint_identity_random(be):
    rng = np.random.default_rng(7)  # test_sparse_ops.cpp:81-101
    for _ in range(10):
        r, c = rng.integers(3, 11, 2)
        ent = [(i, j, rng.uniform(-1, 1)) for i in range(r) for j in range(c) if rng.random() < 0.25]
        if not ent:
            continue
        lp = make(np.zeros(c), r, c, ent, np.zeros(r), 0, np.zeros(c), np.ones(c))
        x, y = rng.uniform(-1, 1, c), rng.uniform(-1, 1, r)
        assert np.dot(be.kx(lp, x), y) == pytest.approx(np.dot(x, be.kty(lp, y)), rel=1e-12)


# ---- convergence_info (test_termination.cpp:40-65) ----
def test_convergence_info_hand_values(be):
    i = be.info(tiny(), [1.0], [1.0])
    assert (i["primal_objective"], i["dual_objective"], i["gap_abs"]) == (1.0, 1.0, 0.0)
    assert i["primal_residual_norm"] == 0.0 and i["dual_residual_norm"] == 0.0
    i = be.info(tiny(), [0.0], [0.0])
    assert i["primal_residual_norm"] == 1.0 and i["dual_residual_norm"] == 0.0 and i["gap_abs"] == 0
    i = be.info(tiny(), [2.0], [0.0])
    assert i["primal_residual_norm"] == 0.0 and i["gap_abs"] == 2.0


# ---- adaptive step (test_solver.cpp:95-171) ----
def test_adaptive_step_at_fixed_point_grows(be):
    r = be.step(tiny(), [1.0], [1.0], 1.0, 0.25, 1)
    assert r["trials"] == 1 and r["eta_used"] == 0.25
    assert r["eta_hat_next"] == pytest.approx((1 + 2 ** -0.6) * 0.25, rel=1e-12)
    assert r["x"][0] == pytest.approx(1.0)


def test_adaptive_step_counter_is_one_based(be):
    with pytest.raises(FolpError) as e:
        be.step(tiny(), [0.0], [0.0], 1.0, 0.5, 0)
    assert e.value.kind == "InvalidArgument"


def test_adaptive_step_movement_bound(be):
    rng = np.random.default_rng(42)
    multi = 0
    for _ in range(60):
        n, m = rng.integers(2, 5, 2)
        ent = [(r, c, 2 * rng.uniform(-1, 1)) for r in range(m) for c in range(n) if rng.random() < .5]
        if not ent:
            continue
        lp = make(rng.uniform(-1, 1, n), m, n, ent, rng.uniform(-1, 1, m), m // 2, -np.ones(n),
                  np.ones(n))
        x = np.clip(0.5 * rng.uniform(-1, 1, n), -1, 1)
        y = rng.uniform(-1, 1, m)
        y[:m // 2] = np.maximum(y[:m // 2], 0)
        omega, eta_hat, k = math.exp(rng.uniform(-1, 1)), math.exp(2 * rng.uniform(-1, 1)), int(rng.integers(1, 50))
        r = be.step(lp, x, y, omega, eta_hat, k)
        multi += r["trials"] > 1
        if r["cross_term"] > 0:
            assert 2 * r["eta_used"] * r["cross_term"] <= r["movement_sq"] * (1 + 1e-9)
        eta_bar = r["movement_sq"] / (2 * r["cross_term"]) if r["cross_term"] > 0 else INF
        want = min((1 - (k + 1) ** -0.3) * eta_bar, (1 + (k + 1) ** -0.6) * r["eta_used"])
        assert r["eta_hat_next"] == pytest.approx(want, rel=1e-12)
    assert multi > 0


# ---- normalized duality gap (test_solver.cpp:219-260, acceptance_main.cpp:289-345) ----
def test_gap_zero_at_verified_optima(be):
    for lp, z in ((tiny(), ([1.0], [1.0])), (knapsack(), ([0.0, 1.0], [2.0])),
                  (make([0.0], 1, 1, [(0, 0, 1.0)], [0.3], 0, [0.0], [1.0]), ([0.3], [0.0]))):
        for radius in (0.5, 1.0, 2.0):
            assert abs(be.ndg(lp, z[0], z[1], radius, 1.3)) <= 1e-10


def _grid_gap(lp, x, y, radius, omega, step=1e-3):
    """Dense grid oracle for 1x1 problems (tests/oracles.cpp:239-278 idea)."""
    k = lp.row_values[0]
    g = np.array([k * y[0] - lp.objective[0], lp.right_hand_side[0] - k * x[0]])
    lo = [min(0.0, lp.variable_lower[0] - x[0]),
          min(0.0, -y[0]) if lp.num_inequality_rows else -INF]
    hi = [max(0.0, lp.variable_upper[0] - x[0]), INF]
    best = 0.0
    for dx in np.arange(-radius / math.sqrt(omega), radius / math.sqrt(omega) + step, step):
        if dx < lo[0] or dx > hi[0]:
            continue
        rem = radius ** 2 - omega * dx * dx
        if rem < 0:
            continue
        span = math.sqrt(rem * omega)
        for dy in (max(-span, lo[1]), min(span, hi[1]), 0.0):
            if lo[1] <= dy <= hi[1] and omega * dx * dx + dy * dy / omega <= radius ** 2 * (1 + 1e-12):
                best = max(best, g[0] * dx + g[1] * dy)
    return best / radius


def test_gap_against_grid_oracle(be):
    rng = np.random.default_rng(515)
    checked = 0
    while checked < 12:
        k00 = 0.35 * rng.uniform(-1, 1)
        if abs(k00) < 0.05:
            continue
        ineq = rng.random() < 0.5
        lp = make([0.35 * rng.uniform(-1, 1)], 1, 1, [(0, 0, k00)], [0.35 * rng.uniform(-1, 1)],
                  1 if ineq else 0, [-0.4 if rng.random() < .5 else -INF],
                  [0.4 if rng.random() < .5 else INF])
        x = np.clip([0.2 * rng.uniform(-1, 1)], lp.variable_lower, lp.variable_upper)
        y = np.array([0.2 * rng.uniform(-1, 1)])
        if ineq:
            y = np.maximum(y, 0.0)
        omega, radius = math.exp(0.5 * rng.uniform(-1, 1)), 1 + 0.5 * rng.random()
        fast = be.ndg(lp, x, y, radius, omega)
        assert fast >= 0.0
        assert abs(fast - _grid_gap(lp, x, y, radius, omega)) <= 1e-3
        checked += 1


# ---- rescaling (test_scaling.cpp:155-179, acceptance_main.cpp:506-553) ----
def test_ruiz_equilibrates(be):
    rng = np.random.default_rng(606)
    for _ in range(8):
        m, n = rng.integers(8, 16, 2)
        ent = [(r, r % n, 10 * rng.uniform(-1, 1)) for r in range(m)]
        ent += [(c % m, c, 10 * rng.uniform(-1, 1)) for c in range(n)]
        ent += [(r, c, 10 * rng.uniform(-1, 1)) for r in range(m) for c in range(n) if rng.random() < .3]
        lp = make(np.ones(n), m, n, ent, np.ones(m), m, np.zeros(n), np.full(n, INF))
        s = be.rescale_lp(lp, 10, False, 1.0)
        k = np.abs(lp.dense() * np.outer(s["row_scale"], s["col_scale"]))
        for v in list(k.max(axis=1)) + list(k.max(axis=0)):
            if v > 0:
                assert 0.99 <= v <= 1.01


# ---- solves (test_solver.cpp:388-471, 532-672) ----
def test_solve_tiny_lp(be):
    r = be.solve_lp(tiny())
    assert r.termination_reason == "Optimal"
    assert r.final_info["primal_objective"] == pytest.approx(1.0, rel=1e-6)
    assert r.primal_solution[0] == pytest.approx(1.0, rel=1e-6)
    assert r.dual_solution[0] == pytest.approx(1.0, rel=1e-4)
    assert r.step_condition_violations == 0


def test_solve_two_variable_lp(be):
    r = be.solve_lp(knapsack())
    assert r.termination_reason == "Optimal"
    assert r.final_info["primal_objective"] == pytest.approx(-2.0, rel=1e-6)
    assert r.primal_solution[0] == pytest.approx(0.0, abs=1e-5)
    assert r.primal_solution[1] == pytest.approx(1.0, rel=1e-5)


def test_start_at_optimum_stops_immediately(be):
    r = be.solve_lp(tiny(), x0=[1.0], y0=[1.0])
    assert r.termination_reason == "Optimal" and r.iterations == 0 and r.kkt_passes <= 2.0


def test_limits(be):
    assert be.solve_lp(knapsack(), cabi.params(kkt_pass_limit=1.0)).termination_reason == \
        "KktPassLimit"
    r = be.solve_lp(tiny(), cabi.params(iteration_limit=3, eps_optimal=1e-14))
    assert r.termination_reason == "IterationLimit" and r.iterations == 3


def test_kkt_ledger_formula(be):
    """test_solver.cpp:532-556: ledger = pre-check + per-iteration + evaluations
    + restarts + final reduced-cost K'."""
    r = be.solve_lp(knapsack(), cabi.params(use_presolve=False, ruiz_iterations=0,
                                            use_pock_chambolle=False))
    assert r.termination_reason == "Optimal"
    evaluations = len(r.trace) - 1
    intermediate = evaluations - 1
    k = 1 + r.iterations + r.step_trials + 4 * intermediate + 2 + r.restarts
    kt = 1 + r.iterations + 4 * intermediate + 2 + r.restarts + 1
    assert r.kkt_passes == 0.5 * (k + kt)


def test_constant_step_scale_invariance(be):
    """test_solver.cpp:558-625: (K,c,q,l,u) -> (gK, g ay c, g ax q, ax l, ax u)."""
    lp = make([1.0, -0.5, 0.25], 2, 3, [(0, 0, 1.0), (0, 1, 0.5), (1, 1, -0.75), (1, 2, 1.25)],
              [0.5, -0.25], 1, [0.0, -1.0, -INF], [2.0, 1.0, 3.0])
    g, ax, ay = 1.7, 0.6, 2.3
    sc = make(np.array([1.0, -0.5, 0.25]) * g * ay, 2, 3,
              [(0, 0, g), (0, 1, 0.5 * g), (1, 1, -0.75 * g), (1, 2, 1.25 * g)],
              np.array([0.5, -0.25]) * g * ax, 1, np.array([0.0, -1.0, -INF]) * ax,
              np.array([2.0, 1.0, 3.0]) * ax)
    p = cabi.params(step_policy="constant", restart_scheme="none", theta_smoothing=0.0,
                    use_presolve=False, ruiz_iterations=0, use_pock_chambolle=False,
                    eps_zero=0.0, eps_optimal=1e-300, iteration_limit=25,
                    record_iterate_trace=True)
    rng = np.random.default_rng(4)
    x0, y0 = 0.25 * rng.uniform(-1, 1, 3), 0.25 * rng.uniform(-1, 1, 2)
    a = be.solve_lp(lp, p, x0, y0, iterate_capacity=25)
    b = be.solve_lp(sc, p, x0 * ax, y0 * ay, iterate_capacity=25)
    assert len(a.iterate_trace) == len(b.iterate_trace) == 25
    for (_, _, xa, ya), (_, _, xb, yb) in zip(a.iterate_trace, b.iterate_trace):
        assert np.all(np.abs(xb - ax * xa) <= 1e-9 * np.maximum(1, np.abs(ax * xa)))
        assert np.all(np.abs(yb - ay * ya) <= 1e-9 * np.maximum(1, np.abs(ay * ya)))


def test_deterministic_reruns(be):
    a, b = be.solve_lp(knapsack()), be.solve_lp(knapsack())
    assert np.array_equal(a.primal_solution, b.primal_solution)
    assert np.array_equal(a.dual_solution, b.dual_solution)
    assert a.iterations == b.iterations and a.kkt_passes == b.kkt_passes
    assert a.final_info == b.final_info


def test_malitsky_pock_step_hand_values(be):
    """test_solver.cpp:173-217."""
    p0 = cabi.params(mp_interpolation_coefficient=0.0)
    r = be.mp_step(tiny(), [0.5], [0.5], 1.0, 0.25, 1.0, p0)
    assert (r["eta_next"], r["theta_next"], r["trials"]) == (0.25, 1.0, 1)
    assert be.mp_step(tiny(), [0.0], [0.0], 1.0, 0.9, 1.0, p0)["trials"] == 1
    r = be.mp_step(tiny(), [0.0], [0.0], 1.0, 1.9, 1.0, p0)
    assert r["trials"] == 2 and r["eta_next"] == pytest.approx(0.95)
    p4 = cabi.params(mp_interpolation_coefficient=0.4)
    expected = 4.0 + 0.4 * (math.sqrt(2.0) - 1.0) * 4.0
    trials = 1
    while expected > 1.0:
        expected *= 0.5
        trials += 1
    r = be.mp_step(tiny(), [0.0], [0.0], 1.0, 4.0, 1.0, p4)
    assert r["trials"] == trials
    assert r["eta_next"] == pytest.approx(expected)
    assert r["theta_next"] == pytest.approx(4.0 / expected)


@pytest.mark.parametrize("overrides", [dict(step_policy="constant"),
                                       dict(step_policy="malitsky_pock"),
                                       dict(restart_scheme="none"),
                                       dict(restart_scheme="theory")])
def test_policies_solve_tiny(be, overrides):
    r = be.solve_lp(tiny(), cabi.params(**overrides))
    assert r.termination_reason == "Optimal"
    assert r.final_info["primal_objective"] == pytest.approx(1.0, rel=1e-6)
    if overrides.get("restart_scheme") == "none":
        assert r.restarts == 0
