"""Relative KKT error over time of a B200 solve (evaluation trace), to see
where a configuration stands against the 1e-8 target."""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2106_04756_b200 import cabi, engine, instances  # noqa: E402


def rel(info):
    gap = info["gap_abs"] / (1 + abs(info["primal_objective"]) + abs(info["dual_objective"]))
    pr = info["primal_residual_norm"] / (1 + info["norm_q"])
    du = info["dual_residual_norm"] / (1 + info["norm_c"])
    return max(gap, pr, du), gap, pr, du


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--seconds", type=float, default=60.0)
    ap.add_argument("--every", type=int, default=500)
    a = ap.parse_args()
    lp = instances.generate(a.config, 1, a.scale)
    t = time.perf_counter()
    r = engine().solve_lp(lp, cabi.params(time_limit_seconds=a.seconds), trace_capacity=1_000_000)
    dt = time.perf_counter() - t
    print(f"cfg{a.config} x{a.scale}: {r.termination_reason} after {r.iterations} iterations, "
          f"{dt:.1f}s, restarts {r.restarts}")
    for i, e in enumerate(r.trace):
        if i % a.every == 0 or i == len(r.trace) - 1:
            c, g, p, d = rel(e["current"])
            ca = rel(e["average"])[0]
            print(f"it {e['iteration']:9d}  cur {c:.2e} (gap {g:.1e} pr {p:.1e} du {d:.1e})  "
                  f"avg {ca:.2e}")
    print("restart iterations (last 10):", r.restart_iterations[-10:])


if __name__ == "__main__":
    main()
