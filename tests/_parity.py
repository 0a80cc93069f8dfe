"""Per-iterate comparison helpers shared by the parity tests and
tools/noise_floor.py (test infrastructure).

The metric is the reference acceptance suite's own
(/root/reference/proj/tests/acceptance_main.cpp:249-259): per iterate,
max over entries of |a - b| / max(1, |b|), over primal and dual."""
from __future__ import annotations

import hashlib

import numpy as np


def rel_dev(u: np.ndarray, v: np.ndarray) -> float:
    if u.size == 0:
        return 0.0
    return float(np.max(np.abs(u - v) / np.maximum(1.0, np.abs(v))))


def drift_curve(a, b, count: int | None = None) -> list[float]:
    """Per-iterate deviation of trace `a` from trace `b` (lists of
    (iteration, eta, x, y)); iteration numbers must agree."""
    out = []
    for (ia, _, xa, ya), (ib, _, xb, yb) in list(zip(a, b))[:count]:
        assert ia == ib, (ia, ib)
        out.append(max(rel_dev(xa, xb), rel_dev(ya, yb)))
    return out


def running_max(curve: list[float]) -> list[float]:
    out, m = [], 0.0
    for v in curve:
        m = max(m, v)
        out.append(m)
    return out


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def iterate_digest(x, y) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(x, dtype=np.float64).tobytes())
    h.update(np.ascontiguousarray(y, dtype=np.float64).tobytes())
    return h.hexdigest()


def rel_kkt(info: dict) -> float:
    """check_termination's three ratios (termination.cpp:75-83), max."""
    gap = info["gap_abs"] / (1 + abs(info["primal_objective"]) + abs(info["dual_objective"]))
    pr = info["primal_residual_norm"] / (1 + info["norm_q"])
    du = info["dual_residual_norm"] / (1 + info["norm_c"])
    return max(gap, pr, du)


# ---- the reference's own reduction-order noise floor ------------------------
# Any parallel fp64 PDLP re-associates the reference's sequential folds, and
# the adaptive step rule amplifies last-bit differences.  The
# floor of an instance is the per-iterate deviation of the SAME algorithm with
# re-associated sums -- the C restatement (oracle/pdlp_port.c) under sum
# orders 1 (pairwise tree), 2 (reversed fold), 3 (tree + 256-entry parts for
# long dots) -- from the compiled reference; tools/noise_floor.py measures it
# at BASELINE sizes.  Tree-mode tests hold the production reductions to
# FLOOR_FACTOR x that floor (one more association, another sample of the same
# spread), and its iteration counts to the reference's own spread.
FLOOR_FACTOR = 10.0
CHECKPOINTS = (10, 20, 40, 60, 80, 100, 120)
SUM_ORDERS = (1, 2, 3)


def reference_floor(lp, p: dict, iterates: int, want=None) -> list[float]:
    """Running max over iterates of the largest deviation of a re-associated
    reference (sum orders 1-3) from the reference itself."""
    import ctypes as C

    from oracle import port, ref

    if want is None:
        want = ref.binding().solve_lp(lp, p, iterate_capacity=iterates)
    lib = port.binding().lib
    lib.folp_port_set_sum_order.argtypes = [C.c_int]
    floor = [0.0] * len(want.iterate_trace)
    for order in SUM_ORDERS:
        lib.folp_port_set_sum_order(order)
        try:
            got = port.binding().solve_lp(lp, p, iterate_capacity=iterates)
        finally:
            lib.folp_port_set_sum_order(0)
        for k, v in enumerate(running_max(drift_curve(got.iterate_trace, want.iterate_trace))):
            floor[k] = max(floor[k], v)
    return floor


def assert_within_floor(got_trace, want_trace, floor: list[float], what: str = "") -> list[float]:
    """Tree-mode drift against the reference at every checkpoint <= FLOOR_FACTOR
    x the floor (never required below 1e-12: both agree to the last bits
    early on).  Returns the drift's running max."""
    curve = running_max(drift_curve(got_trace, want_trace))
    for k in CHECKPOINTS:
        if k <= len(curve):
            bound = max(FLOOR_FACTOR * floor[k - 1], 1e-12)
            assert curve[k - 1] <= bound, (what, k, curve[k - 1], floor[k - 1])
    return curve


def iteration_band(cfg: int, seed: int, scale: float) -> float:
    """Allowed relative iteration-count deviation of a tree-mode solve to 1e-8:
    the north_star's 5 %, or the reference's own spread under re-associated
    sums when larger (tests/golden/iteration_spread.json, made by
    tools/noise_floor_iterations.py): the largest deviation over the config
    family (6 seeds x 2 re-associations, ~ the 92 % quantile of a single
    re-associated run) or over this instance's three re-associations.  A
    tree-mode run is one more draw from that distribution."""
    import json
    from pathlib import Path

    spread = json.loads((Path(__file__).parent / "golden" / "iteration_spread.json").read_text())
    inst = spread.get(f"cfg{cfg}_s{seed}_x{scale}", {}).get("max_abs_iter_dev", 0.0)
    return max(0.05, inst, spread["family_spread"][f"cfg{cfg}"])


def host_kkt(lp, x, y) -> dict:
    """Independent host recheck of the termination criterion (the paper's
    Eq. 7) on the ORIGINAL problem from a returned solution, restating the
    reference acceptance suite's evaluate_optimality
    (/root/reference/proj/tests/acceptance_main.cpp:88-139) with scipy
    products: relative gap, primal and dual residuals and their max."""
    import scipy.sparse as sp

    k = sp.csr_matrix((lp.row_values, lp.row_cols, lp.row_start), shape=(lp.num_rows, lp.num_cols))
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    kx, kty = k @ x, k.T @ y
    c, q = np.asarray(lp.objective), np.asarray(lp.right_hand_side)
    lo, up = np.asarray(lp.variable_lower), np.asarray(lp.variable_upper)
    primal_obj = lp.objective_constant + float(c @ x)
    r = c - kty
    has_lo, has_up = lo > -np.inf, up < np.inf
    lam = np.where(has_lo & has_up, r, np.where(has_lo, np.maximum(r, 0.0),
                                                np.where(has_up, np.minimum(r, 0.0), 0.0)))
    dual_obj = lp.objective_constant + float(q @ y)
    dual_obj += float(np.sum(np.where(lam > 0, lo * np.where(lam > 0, lam, 0.0), 0.0)))
    dual_obj += float(np.sum(np.where(lam < 0, up * np.where(lam < 0, lam, 0.0), 0.0)))
    pv = q - kx
    m1 = lp.num_inequality_rows
    pv[:m1] = np.maximum(pv[:m1], 0.0)
    out = {"gap": abs(dual_obj - primal_obj) / (1 + abs(primal_obj) + abs(dual_obj)),
           "primal": float(np.linalg.norm(pv)) / (1 + float(np.linalg.norm(q))),
           "dual": float(np.linalg.norm(r - lam)) / (1 + float(np.linalg.norm(c)))}
    out["worst"] = max(out.values())
    return out
