"""Aggregate throughput of independent small solves run concurrently on one
GPU (one host thread per solve, the reference's run_bench pattern) against
the same solves run one after another."""
import argparse
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2106_04756_b200 import cabi, engine, instances  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--solves", type=int, default=16)
    ap.add_argument("--threads", type=int, default=16)
    a = ap.parse_args()
    eng = engine()
    lps = [instances.generate(a.config, s + 1, a.scale) for s in range(a.solves)]
    p = cabi.params(eps_optimal=1e-8)
    eng.solve_lp(lps[0], p, trace_capacity=1)  # warm the process
    t = time.perf_counter()
    its = sum(eng.solve_lp(lp, p, trace_capacity=1).iterations for lp in lps)
    seq = time.perf_counter() - t
    res = [0] * len(lps)
    nxt = [0]
    lock = threading.Lock()

    def worker():
        while True:
            with lock:
                i = nxt[0]
                nxt[0] += 1
            if i >= len(lps):
                return
            res[i] = eng.solve_lp(lps[i], p, trace_capacity=1).iterations

    t = time.perf_counter()
    ths = [threading.Thread(target=worker) for _ in range(a.threads)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    par = time.perf_counter() - t
    print(f"config {a.config} x{a.scale}: {a.solves} solves to 1e-8, {its} iterations; "
          f"sequential {seq:.2f} s ({its / seq:.0f} it/s), {a.threads} threads {par:.2f} s "
          f"({sum(res) / par:.0f} it/s, {seq / par:.2f}x)")


if __name__ == "__main__":
    main()
