"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections
import csv
import sys


def main(path, top=20):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].replace("folpgpu::", "").replace("(anonymous namespace)::", "")
        name = name.split("(")[0][:80]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"{'launches':>8} {'total_us':>10} {'avg_us':>8} {'share':>6}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{v[0]:8d} {v[1] / 1e3:10.1f} {v[1] / 1e3 / v[0]:8.2f} {100 * v[1] / tot:5.1f}%  {k}")
    print(f"total {tot / 1e3:.1f} us over {sum(v[0] for v in agg.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20)
