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
    ap.add_argument("--hot-cols", action="store_true",
                    help="experiment: renumber columns by descending degree (rows keep their entry order)")
    ap.add_argument("--sort-rows", action="store_true", help="with --hot-cols: sort each row by new column")
    a = ap.parse_args()
    lp = instances.generate(a.config, 1, a.scale)
    if a.hot_cols:
        import numpy as np
        deg = np.bincount(lp.row_cols, minlength=lp.num_cols)
        order = np.argsort(-deg, kind="stable")
        rank = np.empty_like(order)
        rank[order] = np.arange(lp.num_cols)
        cols = rank[lp.row_cols]
        vals = lp.row_values
        if a.sort_rows:
            rows = np.repeat(np.arange(lp.num_rows), np.diff(lp.row_start))
            o = np.lexsort((cols, rows))
            cols, vals = cols[o], vals[o]
        lp.row_cols = np.ascontiguousarray(cols, dtype=np.int64)
        lp.row_values = np.ascontiguousarray(vals)
        for f in ("objective", "variable_lower", "variable_upper"):
            setattr(lp, f, np.ascontiguousarray(getattr(lp, f)[order]))
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
