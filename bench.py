#!/usr/bin/env python
"""bench.py -- PDHG iterations/s of the B200 PDLP loop (BASELINE.json metric).

Workload: BASELINE.json configs[1] (config 2): seeded synthetic LP, m=200,000
(half >= rows), n=400,000, power-law column degrees (~3.5M nonzeros), fp64.
A step = one evaluation period of the reference's loop
(SolverParams::evaluation_cadence = 40 accepted PDHG iterations, then the
evaluation / restart check), run on device through the resumable folp solve
session (include/folp_c.h folp_session_*).

  value      : PDHG iterations/s over K timed steps (CUDA events on the engine
               stream, LP resident in HBM), summed over ranks / max time
  e2e        : the same metric through folp_solve() on host arrays (C ABI):
               upload, rescaling, loop, download inside the timed region
               (three solves, the median reported, all three listed)
  roofline   : fused step kernels (K'y+primal step, Kx'+dual step) --
               algorithmic bytes per trial slot 24*nnz + 68*(m+n)
               (SURVEY.md 8d), less 8*n per bound vector that is one 0 /
               infinite value (a constant to the algorithm, not a stream),
               over their CUDA-event time, vs measured HBM peak;
               traffic = the DRAM bytes ncu measured for one trial
               (profiles/r2_traffic.json)
  cpu_baseline: the compiled reference (oracle/_ref) on 1 host core

``--impl reference`` times the reference CPU solver (oracle/_ref, compiled
from the reference sources) on all host cores: one independent solve per core,
aggregate iterations/s.  Multi-GPU (torchrun): `--parallelism replicas`
runs an independent copy of the workload per rank ("replicas only" for
configs 1-2; weak scaling); `--parallelism shards` runs ONE
solve partitioned over the ranks (NCCL collectives issued by the engine,
include/folp_gpu.h folp_gpu_shard; strong scaling) -- by rows (the north_star
layout, all-reduce of n + 3 doubles per trial) or by columns (m + 2), per
`--partition` (default: the shorter exchange).  `auto` shards configs 3-5
when N > 1.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "PDHG iters/s"
UNIT = "iter/s"
CADENCE = 40


def bytes_per_trial(m: int, n: int, nnz: int, uniform_bounds: int = 0) -> int:
    """Algorithmic HBM bytes of one trial slot (kernel A + kernel B), fp64 values,
    int32 indices/pointers, every vector touched once, less the
    bound vectors the algorithm does not need: a lower (upper) bound that is
    the same 0 / infinite value for every variable stays uniform under the
    diagonal rescaling and is a constant, not an 8-byte stream per column."""
    return 24 * nnz + 68 * (m + n) - 8 * n * uniform_bounds


def uniform_bound_count(lp) -> int:
    """How many of (lower, upper) are one scale-invariant value (0 or +-inf)."""
    count = 0
    for v in (lp.variable_lower, lp.variable_upper):
        v = np.asarray(v)
        if v.size and (v[0] == 0.0 or np.isinf(v[0])) and bool(np.all(v == v[0])):
            count += 1
    return count


def measured_traffic(config: int):
    """DRAM bytes per trial (kernel A + kernel B, window phases included) from
    the committed ncu captures (profiles/r2_traffic.json: tools/
    ncu_step_summary.py, tools/launch_traffic.py), or None."""
    for name in ("r2_traffic.json", "r1_traffic.json"):
        try:
            d = json.loads((ROOT / "profiles" / name).read_text())
            return d[f"config{config}"]["trial_dram_bytes"]
        except Exception:
            continue
    return None


def measured_peak() -> tuple[float, str]:
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML
    polled every 2 ms from a thread (the timed region of the default run is
    tens of milliseconds; nvidia-smi's 100 ms loop saw one sample), falling
    back to `nvidia-smi -lms 100`."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")
    PERIOD_S = 0.002

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.samples: list[tuple[float, float, set]] = []
        self.nvml = None
        self.stop = threading.Event()
        self.thread = None

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nvml = nv
            self.handle = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_sm = float(nv.nvmlDeviceGetMaxClockInfo(self.handle, nv.NVML_CLOCK_SM))
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _poll(self):
        nv = self.nvml
        bits = {"sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap,
                "hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown}
        while not self.stop.is_set():
            try:
                sm = float(nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
                self.samples.append((sm, self.max_sm, {k for k, b in bits.items() if r & b}))
            except Exception:
                pass
            self.stop.wait(self.PERIOD_S)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self.stop.set()
        if self.nvml is not None and self.thread is not None:
            self.thread.join(timeout=2)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for a, b, r in self.samples:
            sm.append(a)
            mx.append(b)
            reasons |= r
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[2:]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml 2 ms" if self.samples else "nvidia-smi 100 ms"}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    os.environ["FOLP_DEVICE"] = str(local)
    return world, rank, local


def allreduce_max(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int) -> None:
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def reference_loop_rate(lp, iters_small: int, iters_big: int, threads: int = 1):
    """Reference CPU solver iterations/s from two runs with different iteration
    limits (setup cancels out).  `threads` independent solves run concurrently
    (ctypes releases the GIL); returns aggregate iterations/s."""
    from oracle import ref
    from paper_2106_04756_b200 import cabi

    b = ref.binding()

    def run(limit: int, out: list, i: int):
        t = time.perf_counter()
        r = b.solve_lp(lp, cabi.params(iteration_limit=limit), trace_capacity=1)
        out[i] = (time.perf_counter() - t, r.iterations)

    def batch(limit: int):
        out = [None] * threads
        ts = [threading.Thread(target=run, args=(limit, out, i)) for i in range(threads)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        return out

    small = batch(iters_small)
    big = batch(iters_big)
    rates = []
    for (ts_, is_), (tb, ib) in zip(small, big):
        rates.append((ib - is_) / max(1e-9, tb - ts_))
    return float(sum(rates)), small, big


def run_reference(args, world, rank):
    if rank != 0:
        return
    from paper_2106_04756_b200 import instances

    lp = instances.generate(args.config, args.seed, 1.0)
    threads = args.ref_threads or (os.cpu_count() or 1)
    w_iters = CADENCE * max(1, args.warmup)
    k_iters = CADENCE * args.steps
    rate, small, big = reference_loop_rate(lp, w_iters, w_iters + k_iters, threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * CADENCE * threads / rate if rate > 0 else None,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, BASELINE.json configs[1])",
        "config": config_block(lp, args),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{threads} independent reference solves of the workload, "
                                   f"{k_iters} PDHG iterations each, timed as the difference "
                                   f"of {w_iters + k_iters}- and {w_iters}-iteration runs"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def use_shards(args, world: int) -> bool:
    if args.parallelism == "shards":
        return True
    if args.parallelism == "replicas":
        return False
    return world > 1 and args.config >= 3


def rel_kkt(info: dict) -> float:
    gap = info["gap_abs"] / (1 + abs(info["primal_objective"]) + abs(info["dual_objective"]))
    pr = info["primal_residual_norm"] / (1 + info["norm_q"])
    du = info["dual_residual_norm"] / (1 + info["norm_c"])
    return max(gap, pr, du)


def config_block(lp, args) -> dict:
    from paper_2106_04756_b200 import instances

    working_mb = (24 * lp.nnz * 2 + 8 * 16 * (lp.num_rows + lp.num_cols)) / 1e6
    return {"workload": instances.CONFIG_NAMES[args.config], "config_index": args.config - 1,
            "m": lp.num_rows, "m_inequality": lp.num_inequality_rows, "n": lp.num_cols,
            "nnz": lp.nnz, "seed": args.seed, "evaluation_cadence": CADENCE,
            "step": f"{CADENCE} accepted PDHG iterations + evaluation/restart check",
            "l2": f"resident working set ~{working_mb:.0f} MB (K~ CSR+CSC, original values, "
                  f"iterate vectors) > 126 MB L2; no flush",
            "parallelism": parallelism_name(args, lp)}


def parallelism_name(args, lp) -> str:
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if use_shards(args, world):
        return (f"cols{world} (column-sharded K, NCCL all-reduce of Kx' + trial sums)"
                if shard_partition(args, lp) == "cols" else
                f"rows{world} (row-sharded K, NCCL all-reduce of K'y + trial sums)")
    return f"replicas{world}" if world > 1 else "single"


def shard_partition(args, lp) -> str:
    """--partition auto: the engine's FOLP_SHARD_AUTO rule (columns when
    m + 2 < n), resolved here for the config name."""
    if args.partition != "auto":
        return args.partition
    return "cols" if lp.num_rows + 2 < lp.num_cols else "rows"


def run_b200(args, world, rank, local):
    from paper_2106_04756_b200 import cabi, engine, instances

    eng = engine()
    lp = instances.generate(args.config, args.seed, 1.0)
    m, n, nnz = lp.num_rows, lp.num_cols, lp.nnz
    p = cabi.params(eps_optimal=args.eps)
    sharded = use_shards(args, world)
    spec = None
    if sharded:
        from paper_2106_04756_b200 import shard
        spec = shard.nccl_spec(partition=shard_partition(args, lp))
    # replicas: every rank runs its own solve (work x world); shards: one solve
    jobs = 1 if sharded else world

    # ---- device-resident loop: W untimed + K timed evaluation periods ----
    sess = eng.session(lp, p, shard=spec)
    if args.warmup:
        sess.advance(args.warmup)
    s0 = sess.stats()
    barrier(world)
    step_ms = []
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            step_ms.append(sess.advance(1))
            if sess.finished:
                break
    s1 = sess.stats()
    finished_early = sess.finished
    sess.close()
    total_ms = float(sum(step_ms))
    iters = s1["iterations"] - s0["iterations"]
    max_ms = allreduce_max(total_ms, world)
    value = iters * jobs / (max_ms / 1000.0)
    slots = s1["loop_slots"] - s0["loop_slots"]
    loop_ms = s1["loop_ms"] - s0["loop_ms"]
    launches = s1["launches"] - s0["launches"]
    n_uniform = uniform_bound_count(lp)
    b_trial = bytes_per_trial(m, n, nnz, n_uniform)
    achieved = b_trial * slots / (loop_ms / 1000.0) / 1e9 if loop_ms > 0 else 0.0
    peak, peak_src = measured_peak()

    # ---- end to end: folp_solve() on host arrays, transfers inside --------
    # Three complete solves, the median reported (all three listed): one
    # solve is ~0.1 s of mixed host and device work, and a single sample has
    # been seen 30 % off on a busy host.
    e2e_iters = CADENCE * args.steps
    e2e_runs = []
    for _ in range(1 if sharded else 3):
        t = time.perf_counter()
        if sharded:
            spec = shard.nccl_spec(partition=shard_partition(args, lp))  # a fresh communicator
        r = eng.solve_lp(lp, cabi.params(eps_optimal=args.eps, iteration_limit=e2e_iters),
                         trace_capacity=1, shard=spec)
        e2e_runs.append(allreduce_max(time.perf_counter() - t, world))
    e2e_s = sorted(e2e_runs)[len(e2e_runs) // 2]
    # what folp_solve moves over PCIe for one solve: row starts (int64), column
    # indices (narrowed to int32 on the host), values, c / l / u / q, the
    # column order and its inverse (int32, degree-ordered contexts), the final
    # dual for the reduced costs; the CSC is built on the device and a zero
    # start point is a device memset.  Back: the final point, K'y for the
    # reduced costs, the column starts the host plans from, and 48 doubles of
    # evaluation results per period.
    h2d = 8 * (m + 1) + 12 * nnz + 8 * (3 * n + m) + 8 * n + 8 * m
    d2h = 8 * (n + m) + 8 * n + 8 * (n + 1) + 48 * 8 * args.steps

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": len(step_ms), "warmup": args.warmup,
        "ms_per_step": max_ms / max(1, len(step_ms)),
        "higher_is_better": True, "scaling": "strong" if sharded else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded generator, BASELINE.json configs[{args.config - 1}])",
        "config": config_block(lp, args),
        "iterations_timed": iters, "trial_slots_timed": slots,
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": measured_traffic(args.config),
                     "kernel": "kernel A (K'y + primal step: segdot_kernel<EpiPrimal>, pair_kernel<EpiPrimal> on "
                               "two-entry columns) + kernel B (K x' + dual step: segdot_kernel<EpiDual>), one trial",
                     "bytes_per_launch_pair": b_trial,
                     "bytes_model": "24*nnz + 68*(m+n) - 8*n per uniform (0 or infinite) bound vector: %d uniform"
                                    % n_uniform,
                     "kernel_ms_per_trial": loop_ms / max(1, slots), "peak_source": peak_src},
        "e2e": {"value": e2e_iters * jobs / e2e_s, "unit": UNIT,
                "h2d_bytes_per_step": int(h2d / args.steps), "d2h_bytes_per_step": int(d2h / args.steps),
                "seconds": e2e_s, "seconds_all_runs": e2e_runs,
                "aggregate": "median of %d solves" % len(e2e_runs), "iterations": r.iterations,
                "termination": r.termination_reason},
        "clocks": clocks.summary(),
    }
    if finished_early:
        line["note"] = "solve converged inside the timed region; fewer steps timed"

    if args.ordered_steps > 0 and not sharded:
        line["ordered"] = ordered_block(eng, lp, p, args, world, jobs, b_trial, peak)

    if rank == 0 and world == 1 and not args.skip_cpu_baseline:
        rate, small, big = reference_loop_rate(lp, CADENCE, 3 * CADENCE, 1)
        line["cpu_baseline"] = {
            "value": rate, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"oracle/_ref (reference compiled from its sources), 1 thread, same LP: "
                      f"{2 * CADENCE} PDHG iterations timed as the difference of "
                      f"{3 * CADENCE}- and {CADENCE}-iteration solves "
                      f"({big[0][0]:.1f}s - {small[0][0]:.1f}s)"}
    if args.time_to_tol and rank == 0 and world == 1:
        line["convergence"] = convergence_block(eng, lp, args)
    if rank == 0:
        print(json.dumps(line), flush=True)


def ordered_block(eng, lp, p, args, world, jobs, b_trial, peak) -> dict:
    """The same device-resident loop in the ordered reduction mode (every sum
    folded in the reference's sequential order: iterates bit-identical to the
    reference, tests/test_gpu_fullsize_parity.py), timed the same way."""
    eng.lib.folp_gpu_set_default_reduction(1)
    try:
        sess = eng.session(lp, p)
        sess.advance(1)
        s0 = sess.stats()
        barrier(world)
        ms = [sess.advance(1) for _ in range(args.ordered_steps)]
        s1 = sess.stats()
        sess.close()
    finally:
        eng.lib.folp_gpu_set_default_reduction(0)
    total = allreduce_max(float(sum(ms)), world)
    iters = s1["iterations"] - s0["iterations"]
    slots = s1["loop_slots"] - s0["loop_slots"]
    loop_ms = s1["loop_ms"] - s0["loop_ms"]
    achieved = b_trial * slots / (loop_ms / 1000.0) / 1e9 if loop_ms > 0 else 0.0
    return {"value": iters * jobs / (total / 1000.0), "unit": UNIT, "steps": len(ms),
            "ms_per_step": total / max(1, len(ms)), "kernel_ms_per_trial": loop_ms / max(1, slots),
            "roofline_frac": achieved / peak,
            "parity": "iterates bit-identical to the reference (ordered reductions)"}


def convergence_block(eng, lp, args) -> dict:
    """Solves to 1e-8 relative KKT: config 1 end to end on the B200 and on the
    reference CPU solver (1 core), and the workload itself under a time limit
    (the relative KKT error it reaches)."""
    from oracle import ref
    from paper_2106_04756_b200 import cabi, instances

    out = {}
    lp1 = instances.generate(1, args.seed, 1.0)
    t = time.perf_counter()
    a = eng.solve_lp(lp1, cabi.params(eps_optimal=1e-8), trace_capacity=1)
    gpu_s = time.perf_counter() - t
    t = time.perf_counter()
    b = ref.binding().solve_lp(lp1, cabi.params(eps_optimal=1e-8), trace_capacity=1)
    cpu_s = time.perf_counter() - t
    out["config1_to_1e-8"] = {
        "b200_seconds": gpu_s, "b200_iterations": a.iterations, "b200": a.termination_reason,
        "b200_rel_kkt": rel_kkt(a.final_info),
        "reference_cpu_seconds": cpu_s, "reference_iterations": b.iterations,
        "reference": b.termination_reason}
    t = time.perf_counter()
    r = eng.solve_lp(lp, cabi.params(eps_optimal=1e-8, time_limit_seconds=args.time_to_tol),
                     trace_capacity=1)
    out[f"config{args.config}_time_limited"] = {
        "seconds": time.perf_counter() - t, "time_limit": args.time_to_tol,
        "termination": r.termination_reason, "iterations": r.iterations,
        "rel_kkt_reached": rel_kkt(r.final_info), "restarts": r.restarts}
    return out


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--eps", type=float, default=1e-8)
    ap.add_argument("--skip-cpu-baseline", action="store_true")
    ap.add_argument("--ordered-steps", type=int, default=5,
                    help="also time this many steps in the ordered (bit-exact) reduction mode")
    ap.add_argument("--ref-threads", type=int, default=0)
    ap.add_argument("--time-to-tol", type=float, default=60.0,
                    help="also solve config 1 to 1e-8 (B200 and reference CPU) and the "
                         "workload with this time limit (s); 0 disables")
    ap.add_argument("--parallelism", choices=["auto", "replicas", "shards"], default="auto")
    ap.add_argument("--partition", choices=["auto", "rows", "cols"], default="auto")
    args = ap.parse_args()
    world, rank, local = dist_setup()
    try:
        if args.impl == "reference":
            run_reference(args, world, rank)
        else:
            run_b200(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
