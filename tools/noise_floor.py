"""The reference's own reduction-order noise floor (test infrastructure).

Runs the first N iterates of one instance through
  * the compiled reference (oracle/_ref, sequential folds), and
  * the C restatement (oracle/pdlp_port.c) with the SAME algorithm and the
    same per-element terms but a different association of the sums
    (folp_port_set_sum_order: 1 pairwise tree, 2 reversed fold, 3 tree plus
    256-entry parts for long segment dots),
and reports the per-iterate deviation curve (acceptance_main.cpp:249-259's
metric) and whether restart decisions / the KKT ledger agree.  Any parallel
implementation must re-associate these sums, so these curves are the floor a
parallel fp64 PDLP can be held to on that instance.

    python tools/noise_floor.py --config 2 --scale 1 --iterates 100 [--out f.json]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from _parity import drift_curve, iterate_digest, running_max  # noqa: E402
from oracle import port, ref  # noqa: E402
from paper_2106_04756_b200 import cabi, instances  # noqa: E402

CHECKPOINTS = (10, 20, 40, 60, 80, 100)


def measure(cfg: int, seed: int, scale: float, iterates: int, orders=(1, 2, 3)) -> dict:
    lp = instances.generate(cfg, seed, scale)
    p = cabi.params(record_iterate_trace=True, iteration_limit=iterates)
    t0 = time.time()
    want = ref.binding().solve_lp(lp, p, iterate_capacity=iterates, copy_iterates=False)
    out = {"config": cfg, "seed": seed, "scale": scale, "m": lp.num_rows, "n": lp.num_cols,
           "nnz": int(lp.nnz), "iterates": iterates, "ref_seconds": round(time.time() - t0, 2),
           "ref_restarts": want.restart_iterations, "orders": {},
           # golden record of the reference's own trajectory (tests/golden/fullsize_traces.json)
           "golden": {"iterations": [int(i) for (i, _, _, _) in want.iterate_trace],
                      "eta": [float(e).hex() for (_, e, _, _) in want.iterate_trace],
                      "iterate_sha256": [iterate_digest(x, y) for (_, _, x, y) in want.iterate_trace],
                      "restart_iterations": want.restart_iterations,
                      "kkt_passes": want.kkt_passes, "step_trials": want.step_trials,
                      "final_info": {k: float(v).hex() for k, v in want.final_info.items()}}}
    lib = port.binding().lib
    lib.folp_port_set_sum_order.argtypes = [C.c_int]
    for order in orders:
        lib.folp_port_set_sum_order(order)
        try:
            got = port.binding().solve_lp(lp, p, iterate_capacity=iterates, copy_iterates=False)
        finally:
            lib.folp_port_set_sum_order(0)
        curve = drift_curve(got.iterate_trace, want.iterate_trace)
        rm = running_max(curve)
        out["orders"][str(order)] = {
            "max_first_40": rm[min(39, len(rm) - 1)] if rm else 0.0,
            "max_all": rm[-1] if rm else 0.0,
            "at": {str(k): rm[k - 1] for k in CHECKPOINTS if k <= len(rm)},
            "restarts_equal": got.restart_iterations == want.restart_iterations,
            "kkt_passes_equal": got.kkt_passes == want.kkt_passes,
            "eta_equal_first": next((i for i, (a, b) in enumerate(zip(got.iterate_trace,
                                                                      want.iterate_trace))
                                     if a[1] != b[1]), None),
        }
        del got
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--iterates", type=int, default=100)
    ap.add_argument("--orders", default="1,2,3")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    r = measure(a.config, a.seed, a.scale, a.iterates,
                tuple(int(o) for o in a.orders.split(",") if o))
    line = json.dumps(r)
    short = dict(r)
    short.pop("golden")
    print(json.dumps(short))
    if a.out:
        with open(a.out, "a") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
