"""Generates tests/golden/*.json from the compiled reference (oracle/_ref,
built from /root/reference/proj/src by oracle/Makefile).  Run here, where the
reference exists; the JSON travels with the repo so the oracle (and the
engine) can be checked against the reference's own outputs anywhere.

    python tools/make_golden.py
"""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import ref as R  # noqa: E402
from paper_2106_04756_b200 import cabi, instances  # noqa: E402

OUT = ROOT / "tests" / "golden"


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def summarize(r) -> dict:
    return {
        "termination_reason": r.termination_reason,
        "iterations": r.iterations,
        "kkt_passes": r.kkt_passes,
        "restarts": r.restarts,
        "step_trials": r.step_trials,
        "restart_iterations": r.restart_iterations,
        "final_info": {k: float(v).hex() for k, v in r.final_info.items()},
        "primal_sha256": digest(r.primal_solution),
        "dual_sha256": digest(r.dual_solution),
        "reduced_costs_sha256": digest(r.reduced_costs),
        "primal_head": [float(v).hex() for v in r.primal_solution[:8]],
        "dual_head": [float(v).hex() for v in r.dual_solution[:8]],
        "trace_len": len(r.trace),
        "iterate_sha256": [digest(np.concatenate([x, y])) for (_, _, x, y) in r.iterate_trace],
        "iterate_eta": [float(e).hex() for (_, e, _, _) in r.iterate_trace],
    }


CASES = [
    # (name, instance factory, params overrides, iterates)
    ("cfg1_s1_x0.25_full", lambda: instances.generate(1, 1, 0.25), {}, 0),
    ("cfg1_s1_x1_iter200", lambda: instances.generate(1, 1, 1.0),
     {"iteration_limit": 200, "record_iterate_trace": True}, 200),
    ("cfg2_s1_x0.005_iter400", lambda: instances.generate(2, 1, 0.005),
     {"iteration_limit": 400, "record_iterate_trace": True}, 100),
    ("cfg3_s1_x0.0001_iter400", lambda: instances.generate(3, 1, 0.0001),
     {"iteration_limit": 400}, 0),
    ("cfg5_s1_x0.01_iter400", lambda: instances.generate(5, 1, 0.01),
     {"iteration_limit": 400}, 0),
    ("ref_pagerank_n200_s5", lambda: R.pagerank(200, 3, 5), {}, 0),
    ("ref_random_feasible_5003", lambda: R.random_feasible(5003, 16, 6, 15, 2.5),
     {"kkt_pass_limit": 100000}, 0),
    ("ref_random_feasible_1000_constant", lambda: R.random_feasible(1000, 4, 2, 5, 0.5),
     {"step_policy": "constant", "restart_scheme": "none", "theta_smoothing": 0.0,
      "use_presolve": False, "ruiz_iterations": 0, "use_pock_chambolle": False,
      "eps_zero": 0.0, "eps_optimal": 1e-300, "iteration_limit": 100,
      "record_iterate_trace": True}, 100),
]


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    b = R.binding()
    golden = {}
    for name, make, over, n_it in CASES:
        lp = make()
        p = cabi.params(**over)
        r = b.solve_lp(lp, p, iterate_capacity=n_it)
        golden[name] = {"params": over, "m": lp.num_rows, "n": lp.num_cols, "nnz": lp.nnz,
                        "result": summarize(r)}
        print(name, r.termination_reason, r.iterations)
    hc = []
    for lp, obj in R.handcrafted():
        r = b.solve_lp(lp)
        hc.append({"name": lp.name, "optimal_objective": obj, "result": summarize(r)})
    golden["handcrafted_suite"] = hc
    (OUT / "reference_solves.json").write_text(json.dumps(golden, indent=1, sort_keys=True))
    print("wrote", OUT / "reference_solves.json")


if __name__ == "__main__":
    main()
