"""GPU parity of the single kernels against the compiled reference
(oracle/_ref), on instances of every BASELINE family and the reference's own
generators.  Calls go through the C ABI (include/folp_c.h)."""
import numpy as np
import pytest

from paper_2106_04756_b200 import instances

pytestmark = pytest.mark.gpu

FAMILIES = [(1, 1.0), (2, 0.02), (3, 0.01), (4, 0.00005), (5, 0.05)]


def _lp(cfg, scale, seed=1):
    return instances.generate(cfg, seed, scale)


def _sum_abs_terms(lp, vec, transpose):
    k = np.abs(lp.row_values)
    out = np.zeros(lp.num_cols if transpose else lp.num_rows)
    rows = np.repeat(np.arange(lp.num_rows), np.diff(lp.row_start))
    if transpose:
        np.add.at(out, lp.row_cols, k * np.abs(vec[rows]))
    else:
        np.add.at(out, rows, k * np.abs(vec[lp.row_cols]))
    return out


# above 2^20 nonzeros the tree-mode plans are balanced (plans.cuh: retargeted
# tiles, chunk-level LPT order, single parts, padding slots)
LARGE = [(2, 0.4), (3, 0.06), (5, 0.04)]


@pytest.mark.parametrize("cfg,scale", FAMILIES + LARGE)
def test_products_match_reference(eng, ref, cfg, scale):
    lp = _lp(cfg, scale)
    rng = np.random.default_rng(cfg)
    x = rng.standard_normal(lp.num_cols)
    y = rng.standard_normal(lp.num_rows)
    for transpose, vec in ((False, x), (True, y)):
        got = eng.kty(lp, vec) if transpose else eng.kx(lp, vec)
        want = ref.kty(lp, vec) if transpose else ref.kx(lp, vec)
        # reordered fp64 sums: error bounded by ~len * eps * sum|terms|
        bound = 64 * np.finfo(float).eps * _sum_abs_terms(lp, vec, transpose) + 1e-300
        assert np.all(np.abs(got - want) <= bound), (cfg, transpose)


@pytest.mark.parametrize("cfg,scale", FAMILIES)
def test_rescale_bit_exact(eng, ref, cfg, scale):
    lp = _lp(cfg, scale)
    a = eng.rescale_lp(lp)
    b = ref.rescale_lp(lp)
    for key in a:
        assert np.array_equal(a[key], b[key]), key


@pytest.mark.parametrize("cfg,scale", FAMILIES)
def test_convergence_info_matches(eng, ref, cfg, scale):
    lp = _lp(cfg, scale)
    rng = np.random.default_rng(7)
    x = np.clip(rng.uniform(-1, 6, lp.num_cols), lp.variable_lower, lp.variable_upper)
    y = rng.standard_normal(lp.num_rows)
    a = eng.info(lp, x, y)
    b = ref.info(lp, x, y)
    for key in a:
        assert a[key] == pytest.approx(b[key], rel=1e-12, abs=1e-12 * (1 + abs(b[key]))), key


@pytest.mark.parametrize("cfg,scale", FAMILIES)
def test_normalized_duality_gap_matches(eng, ref, cfg, scale):
    lp = _lp(cfg, scale)
    rng = np.random.default_rng(11)
    x = np.clip(rng.uniform(0, 3, lp.num_cols), lp.variable_lower, lp.variable_upper)
    y = rng.standard_normal(lp.num_rows)
    y[:lp.num_inequality_rows] = np.abs(y[:lp.num_inequality_rows])
    for radius, omega in ((0.5, 1.0), (3.0, 0.2), (50.0, 4.0)):
        a = eng.ndg(lp, x, y, radius, omega)
        b = ref.ndg(lp, x, y, radius, omega)
        assert a == pytest.approx(b, rel=1e-9), (radius, omega)


@pytest.mark.parametrize("cfg,scale", FAMILIES)
def test_adaptive_step_matches(eng, ref, cfg, scale):
    lp = _lp(cfg, scale)
    rng = np.random.default_rng(3)
    x = np.clip(rng.uniform(0, 3, lp.num_cols), lp.variable_lower, lp.variable_upper)
    y = rng.standard_normal(lp.num_rows)
    y[:lp.num_inequality_rows] = np.abs(y[:lp.num_inequality_rows])
    a = eng.step(lp, x, y, 1.3, 50.0, 7)
    b = ref.step(lp, x, y, 1.3, 50.0, 7)
    assert a["trials"] == b["trials"]
    assert a["eta_used"] == pytest.approx(b["eta_used"], rel=1e-12)
    assert a["eta_hat_next"] == pytest.approx(b["eta_hat_next"], rel=1e-10)
    np.testing.assert_allclose(a["x"], b["x"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(a["y"], b["y"], rtol=1e-12, atol=1e-12)

