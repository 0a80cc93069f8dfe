"""DRAM bytes per shard and trial from an ncu launch list of
tools/profile_shards.py (one CUDA stream per loopback shard).

    python tools/shard_bytes.py L.csv TRIALS [--label replicated]

TRIALS: trial slots per shard in the profiled region (profile_shards.py
prints them).  Only the step kernels of the loop are summed (the partial
products, both epilogues, the decision); evaluations are reported apart.
"""
import argparse
import collections
import csv
import io

STEP = ("EpiPrimal,", "EpiPrimal>", "EpiShardPart", "OpShardDualOwn", "OpShardDual", "k_shard_decide",
        "OpShardPrimal", "EpiDual,", "EpiDual>")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("trials", type=int)
    ap.add_argument("--label", default="")
    a = ap.parse_args()
    txt = open(a.csv).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
    launches = collections.OrderedDict()
    for r in rows:
        d = launches.setdefault(r["ID"], {"k": r["Kernel Name"], "s": r["Stream"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    per = collections.defaultdict(lambda: collections.defaultdict(lambda: [0, 0.0, 0.0]))
    for d in launches.values():
        name = d["k"].replace("folpgpu::", "").split("(")[0]
        kind = next((s.rstrip(",>") for s in STEP if s in d["k"]), None)
        if kind is None or "Residual" in name or "Ndg" in name:
            kind = "other"
        e = per[d["s"]][kind]
        e[0] += 1
        e[1] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        e[2] += d.get("gpu__time_duration.sum", 0.0)
    step_streams = [s for s in per if sum(v[0] for k, v in per[s].items() if k != "other") > 0]
    print(f"{a.label} {len(step_streams)} shard streams; per shard and trial:")
    tot = []
    for s in sorted(step_streams, key=lambda x: int(x)):
        b = sum(v[1] for k, v in per[s].items() if k != "other") / a.trials
        t = sum(v[2] for k, v in per[s].items() if k != "other") / a.trials
        tot.append(b)
        parts = ", ".join(f"{k} {v[1] / a.trials / 1e6:.1f} MB" for k, v in sorted(per[s].items())
                          if k != "other")
        print(f"  stream {s}: {b / 1e6:8.1f} MB, {t / 1e3:7.1f} us (serialized)  [{parts}]")
    if tot:
        print(f"  mean {sum(tot) / len(tot) / 1e6:.1f} MB, max {max(tot) / 1e6:.1f} MB per shard and trial")


if __name__ == "__main__":
    main()
