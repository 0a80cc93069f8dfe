"""Structure of the seeded BASELINE instances at reduced scale:
sizes, canonical CSR/CSC, the >= rows first, feasibility by construction."""
import numpy as np
import pytest

from paper_2106_04756_b200 import instances


def _canonical(lp):
    rs, rc = lp.row_start, lp.row_cols
    assert rs[0] == 0 and rs[-1] == lp.nnz
    for r in range(min(lp.num_rows, 2000)):
        cols = rc[rs[r]:rs[r + 1]]
        assert np.all(np.diff(cols) > 0)
    assert np.all(lp.row_values != 0) and np.all(np.isfinite(lp.row_values))


@pytest.mark.parametrize("cfg,scale", [(1, 1.0), (2, 0.01), (3, 0.001), (4, 0.0001), (5, 0.02)])
def test_family_structure(cfg, scale):
    lp = instances.generate(cfg, 1, scale)
    _canonical(lp)
    assert np.all(np.isfinite(lp.objective)) and np.all(np.isfinite(lp.right_hand_side))
    assert lp.num_inequality_rows <= lp.num_rows
    again = instances.generate(cfg, 1, scale)
    assert np.array_equal(lp.row_values, again.row_values)  # seeded, deterministic


def test_config1_full_size():
    lp = instances.generate(1, 1, 1.0)
    assert (lp.num_rows, lp.num_inequality_rows, lp.num_cols, lp.nnz) == (1000, 500, 2000, 10000)
    cols = np.bincount(lp.row_cols, minlength=lp.num_cols)
    assert np.all(cols == 5)  # 5 distinct rows per column
    assert np.all(lp.variable_lower == 0) and np.all(lp.variable_upper == 10)


def test_config2_powerlaw_degrees():
    lp = instances.generate(2, 1, 0.05)
    deg = np.bincount(lp.row_cols, minlength=lp.num_cols)
    assert deg.min() >= 2 and deg.max() <= 2000
    assert 7.5 < deg.mean() < 10.5  # discrete k^-2.1 on {2..2000}: mean 8.76
    mags = np.abs(lp.row_values)
    assert mags.min() >= 1e-3 * (1 - 1e-12) and mags.max() <= 1e3 * (1 + 1e-12)


def test_config3_pagerank_rows():
    lp = instances.generate(3, 1, 0.0005)
    n = lp.num_cols
    assert lp.num_rows == n + 1 and lp.num_inequality_rows == n
    last = lp.row_values[lp.row_start[n]:lp.row_start[n + 1]]
    assert last.size == n and np.all(last == 1.0)       # 1'x = 1
    assert lp.right_hand_side[-1] == 1.0
    assert np.allclose(lp.right_hand_side[:-1], 0.01 / n)  # (1 - 0.99) / N
    colsum = np.zeros(n)
    rows = np.repeat(np.arange(lp.num_rows), np.diff(lp.row_start))
    np.add.at(colsum, lp.row_cols, np.where(rows < n, lp.row_values, 0.0))
    assert np.allclose(colsum, 1.0 - 0.99)  # diag 1 minus lambda * column-stochastic P


def test_config5_transportation():
    lp = instances.generate(5, 1, 0.02)
    S, D = lp.num_inequality_rows, lp.num_rows - lp.num_inequality_rows
    assert lp.num_cols == S * D and lp.nnz == 2 * S * D
    supply, demand = -lp.right_hand_side[:S], lp.right_hand_side[S:]
    assert np.isclose(supply.sum(), 1.1 * demand.sum())
    assert np.all((demand >= 10) & (demand <= 40))
    assert np.all(lp.objective >= 0) and np.all(lp.objective <= np.sqrt(2))
