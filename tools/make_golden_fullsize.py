"""Collects tools/noise_floor.py output lines (one per config, run here where
the reference exists) into
  * tests/golden/fullsize_traces.json -- the reference's own 100-iterate (10
    for config 4) trajectories as hashes + the noise floor per checkpoint
    (max over the re-associated orders), read by
    tests/test_gpu_fullsize_parity.py on the GPU box;
  * profiles/r2_noise_floor.json -- the full floor measurements.

    python tools/noise_floor.py --config 2 --out /tmp/nf.jsonl   (3, 5; 4 with --iterates 10 --orders "")
    python tools/make_golden_fullsize.py /tmp/nf.jsonl [...]
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def main(paths):
    gold_path = ROOT / "tests" / "golden" / "fullsize_traces.json"
    prof_path = ROOT / "profiles" / "r2_noise_floor.json"
    gold = json.loads(gold_path.read_text()) if gold_path.exists() else {}
    prof = json.loads(prof_path.read_text()) if prof_path.exists() else {}
    for p in paths:
        for line in open(p):
            r = json.loads(line)
            key = f"cfg{r['config']}"
            floor = {}
            for o in r["orders"].values():
                for k, v in o["at"].items():
                    floor[k] = max(floor.get(k, 0.0), v)
            gold[key] = {"config": r["config"], "seed": r["seed"], "scale": r["scale"],
                         "iterates": r["iterates"], "m": r["m"], "n": r["n"], "nnz": r["nnz"],
                         "golden": r["golden"], "floor": floor}
            short = dict(r)
            short.pop("golden")
            prof[key] = short
    gold_path.write_text(json.dumps(gold, indent=0, sort_keys=True))
    prof_path.write_text(json.dumps(prof, indent=1, sort_keys=True))
    print("configs:", sorted(gold))


if __name__ == "__main__":
    main(sys.argv[1:])
