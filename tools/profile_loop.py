"""Short, profiler-friendly run of the B200 PDLP loop on a BASELINE config:
generates the LP, runs `--warmup` then `--periods` evaluation periods through
the solve session and prints the device time.  Used under ncu (launch list
and full captures of the fused step kernels)."""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2106_04756_b200 import cabi, engine, instances  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--periods", type=int, default=1)
    a = ap.parse_args()
    lp = instances.generate(a.config, 1, a.scale)
    t = time.perf_counter()
    s = engine().session(lp, cabi.params())
    print(f"setup {time.perf_counter() - t:.3f}s m={lp.num_rows} n={lp.num_cols} nnz={lp.nnz}")
    if a.warmup:
        s.advance(a.warmup)
    ms = s.advance(a.periods)
    st = s.stats()
    print(f"{a.periods} periods: {ms:.3f} ms device; stats {st}")
    s.close()


if __name__ == "__main__":
    main()
