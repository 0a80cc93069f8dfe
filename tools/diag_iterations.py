"""Tree-mode vs reference iteration counts over seeds (how far chaotic
trajectory separation moves the iteration count)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2106_04756_b200 import cabi, engine, instances  # noqa: E402
from oracle import ref as R  # noqa: E402  (diagnostic checker only)


def main():
    eng, ref = engine(), R.binding()
    p = cabi.params(kkt_pass_limit=300000)
    for cfg, scale in ((5, 0.01), (5, 0.02), (3, 0.0005), (2, 0.01), (4, 0.0001), (1, 0.3)):
        tot_a = tot_b = 0
        for seed in range(1, 7):
            lp = instances.generate(cfg, seed, scale)
            a = eng.solve_lp(lp, p)
            b = ref.solve_lp(lp, p)
            tot_a += a.iterations
            tot_b += b.iterations
            print(f"cfg{cfg} x{scale} seed {seed}: tree {a.termination_reason} {a.iterations}  "
                  f"ref {b.termination_reason} {b.iterations}  ({100 * (a.iterations - b.iterations) / max(1, b.iterations):+.1f}%)",
                  flush=True)
        print(f"cfg{cfg} x{scale} total: tree {tot_a} ref {tot_b} ({100 * (tot_a - tot_b) / max(1, tot_b):+.1f}%)", flush=True)


if __name__ == "__main__":
    main()
