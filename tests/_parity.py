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
