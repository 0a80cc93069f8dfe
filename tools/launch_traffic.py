"""Per-trial DRAM traffic of the loop's step kernels from an ncu launch list
with dram__bytes_read/write (tools/gpu_profile*.sh, FOLP_NO_GRAPH=1), merged
into profiles/r2_traffic.json (bench.py roofline.traffic).  A trial = every
step-kernel launch (window phases included) divided by the kernel-A count.

    python tools/launch_traffic.py LAUNCHES.csv CONFIG [LAST_N]
"""
import collections
import csv
import io
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def main(path, config, last=None):
    txt = open(path).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
    launches = collections.OrderedDict()
    for r in rows:
        d = launches.setdefault(r["ID"], {"k": r["Kernel Name"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    ls = list(launches.values())
    if last:
        ls = ls[-int(last):]
    step = [d for d in ls if "segdot_kernel" in d["k"] and ("EpiPrimal" in d["k"] or "EpiDual" in d["k"])
            and "Residual" not in d["k"]]
    a = sum(1 for d in step if "EpiPrimal" in d["k"] and "EpiCarry<" not in d["k"])
    tot = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in step)
    per = tot / max(1, a)
    tj = ROOT / "profiles" / "r2_traffic.json"
    out = json.loads(tj.read_text()) if tj.exists() else {}
    out[f"config{config}"] = {"trial_dram_bytes": per, "trials": a,
                              "source": f"{path} (ncu launch list, dram__bytes_read+write of the step kernels, cold caches)"}
    tj.write_text(json.dumps(out, indent=1) + "\n")
    print(f"config {config}: {a} trials, {per / 1e6:.1f} MB DRAM per trial")


if __name__ == "__main__":
    main(*sys.argv[1:])
