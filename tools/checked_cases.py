"""Parity cases run through a given engine library (FOLP_ENGINE_LIB), one
JSON line of result digests (test infrastructure: tests/test_gpu_checked.py
runs it through the checked library -- device bounds checks, segdot.cuh
FOLP_DCHECK -- and through the product library, and compares)."""
import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2106_04756_b200 import cabi, engine, instances, shard  # noqa: E402


def digest(r) -> str:
    h = hashlib.sha256()
    for a in (r.primal_solution, r.dual_solution, r.reduced_costs):
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    h.update(json.dumps([r.iterations, r.restart_iterations, r.termination_reason,
                         {k: float(v).hex() for k, v in r.final_info.items()}]).encode())
    return h.hexdigest()


def main():
    eng = engine()
    out = {}
    cases = [("cfg1", 1, 1, 1.0, 200), ("cfg2", 2, 1, 0.05, 120), ("cfg3", 3, 1, 0.002, 120),
             ("cfg4", 4, 1, 0.0005, 120)]
    for mode in (0, 1):
        eng.lib.folp_gpu_set_default_reduction(mode)
        try:
            for name, cfg, seed, scale, its in cases:
                lp = instances.generate(cfg, seed, scale)
                out[f"{name}_{'ordered' if mode else 'tree'}"] = digest(
                    eng.solve_lp(lp, cabi.params(iteration_limit=its), trace_capacity=8))
        finally:
            eng.lib.folp_gpu_set_default_reduction(0)
    os.environ["FOLP_SELL_MIN_LEN"] = "16"  # SELL-32 groups on a small config-5 member
    lp = instances.generate(5, 1, 0.05)
    out["cfg5_sell"] = digest(eng.solve_lp(lp, cabi.params(iteration_limit=120), trace_capacity=8))
    del os.environ["FOLP_SELL_MIN_LEN"]
    lp = instances.generate(5, 1, 0.01)
    for part in ("rows", "cols"):
        res = shard.solve_loopback(lp, 3, cabi.params(iteration_limit=120), partition=part)
        out[f"shard3_{part}"] = digest(res[0])
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
