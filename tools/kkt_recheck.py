"""Full-size solves to 1e-8 on the B200 with an independent host recheck of
the termination criterion (Eq. 7) from the returned solution on the
original problem (tests/_parity.py host_kkt, restating the reference's
acceptance_main.cpp:88-139).  One JSON line per config.

    python tools/kkt_recheck.py --configs 1,3,5,2 --seconds 60,600,600,900
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from _parity import host_kkt, rel_kkt  # noqa: E402
from paper_2106_04756_b200 import cabi, engine, instances  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,3,5")
    ap.add_argument("--seconds", default="60,600,600")
    a = ap.parse_args()
    eng = engine()
    for cfg, secs in zip(map(int, a.configs.split(",")), map(float, a.seconds.split(","))):
        lp = instances.generate(cfg, 1, 1.0)
        t = time.perf_counter()
        r = eng.solve_lp(lp, cabi.params(eps_optimal=1e-8, time_limit_seconds=secs), trace_capacity=4)
        wall = time.perf_counter() - t
        hk = host_kkt(lp, r.primal_solution, r.dual_solution)
        print(json.dumps({"config": cfg, "termination": r.termination_reason, "iterations": r.iterations,
                          "seconds": wall, "device_rel_kkt": rel_kkt(r.final_info),
                          "host_recheck": hk, "objective": r.final_info["primal_objective"]}), flush=True)


if __name__ == "__main__":
    main()
