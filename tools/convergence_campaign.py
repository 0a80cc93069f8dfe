"""Solve each BASELINE config toward 1e-8 relative KKT under a time limit on
the B200 and record the relative-KKT trajectory (for time-to-tolerance
evidence).  Output: one JSON line per config."""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2106_04756_b200 import cabi, engine, instances  # noqa: E402


def rel(info):
    gap = info["gap_abs"] / (1 + abs(info["primal_objective"]) + abs(info["dual_objective"]))
    pr = info["primal_residual_norm"] / (1 + info["norm_q"])
    du = info["dual_residual_norm"] / (1 + info["norm_c"])
    return max(gap, pr, du)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3,5,4")
    ap.add_argument("--seconds", default="900,600,600,900")
    a = ap.parse_args()
    eng = engine()
    for cfg, secs in zip(map(int, a.configs.split(",")), map(float, a.seconds.split(","))):
        t = time.perf_counter()
        lp = instances.generate(cfg, 1, 1.0)
        gen = time.perf_counter() - t
        t = time.perf_counter()
        r = eng.solve_lp(lp, cabi.params(eps_optimal=1e-8, time_limit_seconds=secs),
                         trace_capacity=2_000_000)
        wall = time.perf_counter() - t
        traj = []
        marks = [1e-2, 1e-3, 1e-4, 1e-5, 1e-6, 1e-7, 1e-8]
        best = 1.0
        first = {}
        for e in r.trace:
            v = min(rel(e["current"]), rel(e["average"]))
            best = min(best, v)
            for mk in marks:
                if best <= mk and mk not in first:
                    first[mk] = e["iteration"]
        step = max(1, len(r.trace) // 40)
        for i in range(0, len(r.trace), step):
            e = r.trace[i]
            traj.append([e["iteration"], min(rel(e["current"]), rel(e["average"]))])
        print(json.dumps({"config": cfg, "generate_s": gen, "time_limit_s": secs, "wall_s": wall,
                          "termination": r.termination_reason, "iterations": r.iterations,
                          "restarts": r.restarts, "final_rel_kkt": rel(r.final_info),
                          "first_iteration_reaching": {f"{k:g}": v for k, v in first.items()},
                          "trajectory": traj}), flush=True)


if __name__ == "__main__":
    main()
