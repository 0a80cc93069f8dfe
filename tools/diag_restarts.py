"""Restart schedules of the B200 tree / ordered modes against the compiled
reference on one instance (diagnostic for tree-mode decision flips)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2106_04756_b200 import cabi, engine, instances  # noqa: E402
from oracle import ref as R  # noqa: E402  (diagnostic checker only)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--scale", type=float, default=0.01)
    a = ap.parse_args()
    lp = instances.generate(a.config, 1, a.scale)
    p = cabi.params(kkt_pass_limit=300000)
    runs = {"reference": R.binding().solve_lp(lp, p, trace_capacity=100000)}
    eng = engine()
    for mode, flag in (("tree", 0), ("ordered", 1)):
        eng.lib.folp_gpu_set_default_reduction(flag)
        runs[mode] = eng.solve_lp(lp, p, trace_capacity=100000)
    eng.lib.folp_gpu_set_default_reduction(0)
    for k, r in runs.items():
        print(f"{k:9s} {r.termination_reason} it={r.iterations} restarts={r.restart_iterations}")
    ref = runs["reference"].trace
    for mode in ("tree", "ordered"):
        tr = runs[mode].trace
        for i, (e, f) in enumerate(zip(tr, ref)):
            x, y = e["current"]["gap_abs"], f["current"]["gap_abs"]
            if abs(x - y) > 1e-6 * (abs(y) + 1e-30):
                print(f"{mode}: first divergence at evaluation {i} (iteration {e['iteration']}):"
                      f" gap {x:.6e} vs {y:.6e}")
                break


if __name__ == "__main__":
    main()
