"""Short solves for compute-sanitizer (memcheck / racecheck / synccheck).

Cases cover the engine's synchronization patterns (determinism is
pinned by the reference at proj/tests/acceptance_main.cpp:652-682):
  cfg1          config 1 family, tree mode: the single-cluster chunk kernel
                (DSMEM partials, cluster barriers), evaluations, bisection
  cfg1_ordered  the same in ordered mode: exact folds (cooperative grid
                kernel, replay lists in shared memory), ordered bisection
  cfg2          config 2 x0.05, tree mode: persistent segdot products with
                last-CTA tickets and part-arrival atomics, balanced plans,
                PDL chaining, the cooperative duality-gap bisection, graphs
  cfg2_ordered  the same in ordered mode
  shard2        loopback W=2 column shards (peer exchange) on config 1
Each case prints one line; the sanitizer's exit code and summary are the
result (tools/sanitize.sh collects them into profiles/)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2106_04756_b200 import cabi, engine, instances, shard  # noqa: E402


def run(case: str) -> None:
    eng = engine()
    ordered = case.endswith("_ordered")
    eng.lib.folp_gpu_set_default_reduction(1 if ordered else 0)
    try:
        if case.startswith("cfg1"):
            lp = instances.generate(1, 1, 1.0)
            r = eng.solve_lp(lp, cabi.params(iteration_limit=200), trace_capacity=8)
        elif case.startswith("cfg2"):
            lp = instances.generate(2, 1, 0.05)
            r = eng.solve_lp(lp, cabi.params(iteration_limit=120), trace_capacity=8)
        elif case == "shard2":
            lp = instances.generate(1, 1, 1.0)
            res = shard.solve_loopback(lp, 2, cabi.params(iteration_limit=120), partition="cols")
            r = res[0]
        else:
            raise SystemExit(f"unknown case {case}")
    finally:
        eng.lib.folp_gpu_set_default_reduction(0)
    print(f"{case}: {r.termination_reason} after {r.iterations} iterations, "
          f"restarts {r.restart_iterations}", flush=True)


if __name__ == "__main__":
    run(sys.argv[1] if len(sys.argv) > 1 else "cfg1")
