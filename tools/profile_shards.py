"""Per-shard traffic of the sharded loop: W loopback shards of
one solve as host threads on one GPU (no kernel waits on another shard), one
warm-up evaluation period, then --periods timed ones.  Run under ncu with
dram__bytes_read/write; tools/shard_bytes.py splits the launch list by
stream (one stream per shard) into bytes per shard and trial.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --csv --log-file L.csv python tools/profile_shards.py --config 4 --scale 0.25 --world 8
"""
import argparse
import sys
import threading
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2106_04756_b200 import cabi, engine, instances, shard  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--scale", type=float, default=0.25)
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--partition", default="cols")
    ap.add_argument("--periods", type=int, default=1)
    a = ap.parse_args()
    lp = instances.generate(a.config, 1, a.scale)
    eng = engine()
    g = shard.LoopbackGroup(a.world)
    stats = [None] * a.world
    errs = [None] * a.world

    def run(r):
        try:
            s = eng.session(lp, cabi.params(), shard=g.spec(r, a.partition))
            try:
                s.advance(1)
                s0 = s.stats()
                ms = s.advance(a.periods)
                s1 = s.stats()
                stats[r] = (ms, s1["iterations"] - s0["iterations"], s1["loop_slots"] - s0["loop_slots"])
            finally:
                s.close()
        except BaseException as e:  # noqa: BLE001
            errs[r] = e

    try:
        ts = [threading.Thread(target=run, args=(r,)) for r in range(a.world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    finally:
        g.close()
    for e in errs:
        if e is not None:
            raise e
    print(f"config {a.config} x{a.scale} m={lp.num_rows} n={lp.num_cols} nnz={lp.nnz} world {a.world}: "
          f"per shard (ms, iterations, trial slots) {stats}", flush=True)


if __name__ == "__main__":
    main()
