"""Summarize an `ncu --set full` capture of the two step kernels (raw CSV page,
tools/gpu_profile.sh) into the profiles/ text format and the traffic JSON that
bench.py reports as roofline.traffic.

    python tools/ncu_step_summary.py gpurun_out/step_full_raw.csv "<header line>"
"""
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
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
SCALE = {"byte": (1e-6, "Mbyte"), "Kbyte": (1e-3, "Mbyte"), "Mbyte": (1.0, "Mbyte"), "Gbyte": (1e3, "Mbyte"),
         "nsecond": (1e-3, "usecond"), "usecond": (1.0, "usecond"), "msecond": (1e3, "usecond")}


def main(path, header):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ki = hdr.index("Kernel Name")
    out = [header, ""]
    kern = {}
    for r in data:
        key = "A" if "EpiPrimal" in r[ki] else "B"
        name = f"void segdot_kernel<{'EpiPrimal' if key == 'A' else 'EpiDual'}, 0, 0>"
        out.append(name)
        vals = {}
        for w in WANT:
            i = hdr.index(w)
            f, u = SCALE.get(units[i], (1.0, units[i]))
            v = float(r[i].replace(",", "")) * f
            vals[w] = v
            out.append(f"  {w:60s} {v:.6f}" + (f"  [{u}]" if u else ""))
        out.append("")
        kern[key] = {"kernel": name, "dram_read_bytes": vals["dram__bytes_read.sum"] * 1e6,
                     "dram_write_bytes": vals["dram__bytes_write.sum"] * 1e6,
                     "duration_us": vals["gpu__time_duration.sum"]}
    tot = sum(k["dram_read_bytes"] + k["dram_write_bytes"] for k in kern.values())
    out.append(f"trial (A+B) DRAM traffic {tot / 1e6:.1f} MB vs algorithmic 125.0 MB (24*nnz + 68*(m+n))")
    (ROOT / "profiles" / "r1_step_kernels_ncu_s3.txt").write_text("\n".join(out) + "\n")
    (ROOT / "profiles" / "r1_traffic.json").write_text(json.dumps(
        {"config2": {"trial_dram_bytes": tot, "kernels": kern,
                     "source": "profiles/r1_step_kernels_ncu_s3.txt (ncu --set full, cold)"}}, indent=1))
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
