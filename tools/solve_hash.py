"""SHA-256 of the solution a fixed-iteration tree-mode solve returns: A/B of
engine switches that must not change a bit (run once per environment setting
and compare the lines)."""
import argparse
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2106_04756_b200 import cabi, engine, instances  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--scale", type=float, default=0.1)
ap.add_argument("--iterations", type=int, default=400)
a = ap.parse_args()
lp = instances.generate(a.config, 1, a.scale)
r = engine().solve_lp(lp, cabi.params(iteration_limit=a.iterations), trace_capacity=64)
h = hashlib.sha256(r.primal_solution.tobytes() + r.dual_solution.tobytes()).hexdigest()
print(f"cfg{a.config} x{a.scale} it={r.iterations} restarts={list(r.restart_iterations)} sha={h[:16]}")
