"""Summarize an `ncu --set full` capture of the loop's step kernels (raw CSV
page, tools/gpu_profile_kernel.sh) into the profiles/ text format, and merge
the per-trial DRAM traffic into the JSON bench.py reports as
roofline.traffic.

    python tools/ncu_step_summary.py RAW_CSV "<header line>" OUT_TXT CONFIG [TRAFFIC_JSON]

CONFIG is the bench config number (1-5); one trial is every step-kernel
launch of the capture divided by the number of kernel-A launches (kernel B
may be several window phases)."""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__grid_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__warps_eligible.avg.per_cycle_active",
        "smsp__average_warp_latency_per_inst_issued.ratio", "smsp__inst_executed.sum",
        "smsp__cycles_active.avg", "sm__cycles_elapsed.avg",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
SCALE = {"byte": (1e-6, "Mbyte"), "Kbyte": (1e-3, "Mbyte"), "Mbyte": (1.0, "Mbyte"), "Gbyte": (1e3, "Mbyte"),
         "nsecond": (1e-3, "usecond"), "usecond": (1.0, "usecond"), "msecond": (1e3, "usecond")}


def short(name: str) -> str:
    return name.split("(")[0].replace("folpgpu::", "").replace("void ", "")


def main(path, header, out_txt, config, traffic_json="profiles/r2_traffic.json"):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ki = hdr.index("Kernel Name")
    out = [header, ""]
    total, a_launches, kernels = 0.0, 0, []
    for r in data:
        out.append(short(r[ki]))
        vals = {}
        for w in WANT:
            if w not in hdr:
                continue
            i = hdr.index(w)
            f, u = SCALE.get(units[i], (1.0, units[i]))
            v = float(r[i].replace(",", "")) * f
            vals[w] = v
            out.append(f"  {w:60s} {v:.6f}" + (f"  [{u}]" if u else ""))
        out.append("")
        b = (vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]) * 1e6
        total += b
        a_launches += "EpiPrimal" in r[ki] and "Residual" not in r[ki]
        kernels.append({"kernel": short(r[ki]), "dram_bytes": b, "duration_us": vals["gpu__time_duration.sum"]})
    per_trial = total / max(1, a_launches)
    out.append(f"per trial ({a_launches} trial(s) captured): DRAM traffic {per_trial / 1e6:.1f} MB")
    Path(out_txt).write_text("\n".join(out) + "\n")
    tj = ROOT / traffic_json
    d = json.loads(tj.read_text()) if tj.exists() else {}
    d[f"config{config}"] = {"trial_dram_bytes": per_trial, "kernels": kernels,
                            "source": f"{out_txt} (ncu --set full, cold caches)"}
    tj.write_text(json.dumps(d, indent=1) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main(*sys.argv[1:])
