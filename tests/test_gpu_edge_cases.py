"""Edge cases of the solve path on the B200 against the compiled reference:
free and one-sided variables, fixed variables, empty rows and columns
(presolve removes them, postsolve restores them), duplicate and explicit-zero
triplets (SparseMatrix::from_triplets sums / drops them), equality-only and
inequality-only programs, crossed bounds, a trivially empty program.

Ordered reductions: every result must be bit-identical to the reference
(solver.cpp:818-946 with presolve.cpp:35-272 around it).  Tree reductions:
same termination and the 1e-8 KKT bar."""
import numpy as np
import pytest

from paper_2106_04756_b200 import cabi

pytestmark = pytest.mark.gpu

INF = np.inf


def _lp_from_triplets(m, n, m1, rows, cols, vals, c, q, lo, hi, const=0.0, name=""):
    """A canonical-or-not CSR straight from triplets in row order (duplicates
    and zeros kept: the C ABI routes such input through from_triplets)."""
    order = np.lexsort((np.arange(len(rows)), np.asarray(rows)))
    rows = np.asarray(rows, dtype=np.int64)[order]
    cols = np.asarray(cols, dtype=np.int64)[order]
    vals = np.asarray(vals, dtype=np.float64)[order]
    start = np.zeros(m + 1, dtype=np.int64)
    np.add.at(start, rows + 1, 1)
    start = np.cumsum(start)
    return cabi.LP(num_rows=m, num_cols=n, num_inequality_rows=m1, row_start=start,
                   row_cols=cols, row_values=vals, objective=np.asarray(c, float),
                   right_hand_side=np.asarray(q, float), variable_lower=np.asarray(lo, float),
                   variable_upper=np.asarray(hi, float), objective_constant=const, name=name)


def _random_feasible(seed, m1, m2, n, density=0.3, free_frac=0.2, fixed_frac=0.1,
                     empty_cols=2, empty_rows=2, dup=True):
    rng = np.random.default_rng(seed)
    m = m1 + m2 + empty_rows
    k = (rng.random((m1 + m2, n)) < density) * rng.standard_normal((m1 + m2, n))
    k[:, :empty_cols] = 0.0  # empty columns
    x0 = rng.uniform(-1, 3, n)
    lo = np.zeros(n)
    hi = np.full(n, 5.0)
    kind = rng.random(n)
    lo[kind < free_frac] = -INF
    hi[kind < free_frac] = INF
    one = (kind >= free_frac) & (kind < free_frac + 0.2)
    hi[one] = INF  # one-sided
    fixed = (kind >= 0.9 - fixed_frac) & (kind < 0.9)
    lo[fixed] = hi[fixed] = 1.0
    x0 = np.clip(x0, lo, hi)
    x0[fixed] = 1.0
    b = k @ x0
    q = np.concatenate([b[:m1] - rng.uniform(0, 1, m1), b[m1:], np.zeros(empty_rows)])
    y0 = rng.standard_normal(m1 + m2)
    y0[:m1] = np.abs(y0[:m1])
    z = rng.uniform(0, 1, n)
    c = k.T @ y0 + np.where(np.isinf(lo) & np.isinf(hi), 0.0, z)
    # empty columns: cost pushing to a finite bound
    c[:empty_cols] = 1.0
    lo[:empty_cols] = 0.0
    rr, cc = np.nonzero(k)
    vv = k[rr, cc]
    rr = np.where(rr >= m1, rr + 0, rr)  # equality rows after the >= rows
    if dup:  # split a few entries into duplicate triplets, add explicit zeros
        pick = rng.choice(len(vv), size=min(5, len(vv)), replace=False)
        rr = np.concatenate([rr, rr[pick], rr[pick[:2]]])
        cc = np.concatenate([cc, cc[pick], cc[pick[:2]]])
        half = vv[pick] / 2
        vv = vv.copy()
        vv[pick] = half
        vv = np.concatenate([vv, half, np.zeros(2)])
    # empty rows sit at the end (inequality rows must come first: they are
    # equality rows with q = 0, feasible)
    return _lp_from_triplets(m, n, m1, rr, cc, vv, c, q, lo, hi, const=0.5,
                             name=f"edge_{seed}")


def _same(a, b):
    assert a.termination_reason == b.termination_reason
    assert a.iterations == b.iterations and a.restart_iterations == b.restart_iterations
    assert a.kkt_passes == b.kkt_passes
    assert a.final_info == b.final_info
    assert np.array_equal(a.primal_solution, b.primal_solution)
    assert np.array_equal(a.dual_solution, b.dual_solution)
    assert np.array_equal(a.reduced_costs, b.reduced_costs)


@pytest.fixture
def ordered(eng):
    eng.lib.folp_gpu_set_default_reduction(1)
    yield
    eng.lib.folp_gpu_set_default_reduction(0)


CASES = [dict(seed=1, m1=10, m2=8, n=30),
         dict(seed=2, m1=0, m2=15, n=25),          # equality only
         dict(seed=3, m1=20, m2=0, n=25),          # inequality only
         dict(seed=4, m1=12, m2=6, n=40, free_frac=0.5),
         dict(seed=5, m1=6, m2=6, n=20, fixed_frac=0.3, dup=False)]


@pytest.mark.parametrize("case", CASES, ids=[f"s{c['seed']}" for c in CASES])
def test_edge_lps_ordered_bit_identical(eng, ref, ordered, case):
    lp = _random_feasible(**case)
    p = cabi.params(kkt_pass_limit=40000)
    a = eng.solve_lp(lp, p)
    b = ref.solve_lp(lp, p)
    _same(a, b)


@pytest.mark.parametrize("case", CASES, ids=[f"s{c['seed']}" for c in CASES])
def test_edge_lps_tree_mode(eng, ref, case):
    lp = _random_feasible(**case)
    p = cabi.params(kkt_pass_limit=40000)
    a = eng.solve_lp(lp, p)
    b = ref.solve_lp(lp, p)
    assert a.termination_reason == b.termination_reason
    assert len(a.primal_solution) == lp.num_cols and len(a.dual_solution) == lp.num_rows
    if b.termination_reason == "Optimal":
        pa, pb = a.final_info["primal_objective"], b.final_info["primal_objective"]
        assert abs(pa - pb) <= 1e-8 * (2 + 2 * abs(pa) + 2 * abs(pb))


def test_crossed_bounds_and_empty_program(eng, ref):
    lp = _lp_from_triplets(1, 2, 0, [0, 0], [0, 1], [1.0, 1.0], [1.0, 1.0], [1.0],
                           [0.0, 2.0], [1.0, 1.0])  # l > u on variable 1
    a = eng.solve_lp(lp)
    b = ref.solve_lp(lp)
    assert a.termination_reason == b.termination_reason == "PrimalInfeasibleDetected"
    # every column empty: presolve fixes them all, the solve is trivial
    lp = _lp_from_triplets(1, 3, 1, [], [], [], [1.0, -1.0, 0.0], [-1.0],
                           [0.0, 0.0, -1.0], [2.0, 3.0, 1.0], const=1.5)
    a = eng.solve_lp(lp)
    b = ref.solve_lp(lp)
    assert a.termination_reason == b.termination_reason
    assert np.array_equal(a.primal_solution, b.primal_solution)
    assert a.final_info == b.final_info
