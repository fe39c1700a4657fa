#!/usr/bin/env python
"""Benchmark: KS replicates/s of the untruncated cutoff-table sweep (BASELINE.json configs[1]).

Workload ("config2"): K = inf, gamma = 1.5..3.5 step 0.1 (21 values) x n in {10, 20, 50, 100,
500, 1000} = 126 cells, base_seed = 1, one repetition, R = 10^6 replicates per cell and GPU
(weak scaling: at N GPUs each cell has N*10^6 replicates, sharded by index; the exact
quantiles are selected across the shards with NCCL all-reduces of radix digit histograms).  One step = the whole 126-cell sweep:
per replicate sample -> MLE refit -> KS, then the 4 order-statistic cutoffs per cell.

  value        device time of the sweep with draw tables resident, L2 flushed between steps
  e2e          the public API paper_1305_6738_b200.build_table (parallel.build_table at N>1):
               host-built draw tables uploaded every step, cutoffs copied back to the host
  roofline     the dominant kernel (largest device time, CUDA events per launch): algorithmic
               bytes per launch over its launch time against the measured HBM peak; plus the
               FP64 / 64-bit-multiply pipe work of the replicate math against on-device probes
  cpu_baseline the CPU oracle (numpy restatement of the reference, bit-identical to it) on
               all host cores over a bounded sample of the same sweep

``--impl reference`` times the reference's CPU algorithm (the oracle port: the reference is a
Python package and cannot travel to the GPU box) on this box's cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "KS replicates/sec per (gamma,n) at 1/2/4/8 B200 vs host-CPU ref; roofline fraction"
GAMMAS = tuple(round(1.5 + 0.1 * i, 1) for i in range(21))
NS = (10, 20, 50, 100, 500, 1000)
CPU_SAMPLE_GAMMAS = (1.5, 1.9, 2.3, 2.7, 3.1, 3.5)
CLOCK_QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
               "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
               "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")


def parse_args():
    p = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("b200", "reference"), default="b200")
    p.add_argument("--replicates", type=int, default=1_000_000, help="replicates per cell per GPU")
    p.add_argument("--cpu-replicates", type=int, default=4096, help="replicates per sampled cell on the CPU")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={CLOCK_QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-f", self.path],
                stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait(timeout=10)

    def summary(self) -> dict:
        rows = []
        try:
            with open(self.path) as fh:
                for line in fh:
                    parts = [x.strip() for x in line.split(",")]
                    if len(parts) >= 9:
                        rows.append(parts)
        except OSError:
            pass
        finally:
            try:
                os.unlink(self.path)
            except OSError:
                pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------- CPU legs

def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def cpu_sample_run(replicates: int, workers: int) -> tuple[float, int, float]:
    """The oracle (numpy restatement of the reference, bit-identical to it) over the sampled
    cells of the sweep with ``workers`` processes (the reference's own Pool driver,
    montecarlo.py:151-191); returns (replicates/s, replicates, seconds)."""
    from oracle import port

    total = 0
    t0 = time.perf_counter()
    for g in CPU_SAMPLE_GAMMAS:
        for n in NS:
            port.simulate(g, None, n, 1, replicates, 1, workers=workers)
            total += replicates
    dt = time.perf_counter() - t0
    return total / dt, total, dt


def cpu_baseline(replicates: int, steps: int = 1, warmup: int = 1) -> dict:
    """Both CPU legs measure the same thing the same way: the oracle over the sampled cells
    with all host cores (W = os.cpu_count()) after ``warmup`` untimed passes, plus one pass on a
    single core (W = 1) over an eighth of the sample.  Run before CUDA is initialised in this
    process (the Pool forks)."""
    workers = os.cpu_count() or 1
    for _ in range(warmup):
        cpu_sample_run(max(replicates // 8, 512), workers)
    total, secs = 0, 0.0
    for _ in range(steps):
        _, reps, dt = cpu_sample_run(replicates, workers)
        total += reps
        secs += dt
    w1_reps = max(replicates // 8, 512)
    v1, r1, d1 = cpu_sample_run(w1_reps, 1)
    return {"value": total / secs, "unit": "replicates/s", "cores": workers, "kind": "port",
            "sample": cpu_sample_desc(replicates) + f"; {total} replicates in {secs:.1f} s after {warmup} warm-up",
            "cpu_model": cpu_model(),
            "w1": {"value": v1, "cores": 1, "sample": f"{len(CPU_SAMPLE_GAMMAS) * len(NS)} cells x {w1_reps} "
                                                      f"replicates, {r1} in {d1:.1f} s"},
            "wcores": {"value": total / secs, "cores": workers}}


def cpu_sample_desc(replicates: int) -> str:
    return (f"{len(CPU_SAMPLE_GAMMAS)} of 21 gammas {CPU_SAMPLE_GAMMAS} x n {NS} = "
            f"{len(CPU_SAMPLE_GAMMAS) * len(NS)} cells x {replicates} replicates, K=inf, base_seed=1, "
            f"1 repetition, multiprocessing pool over all cores (the reference's own parallel driver)")


def run_reference(args, world, rank):
    if rank != 0:
        return
    t0 = time.perf_counter()
    cpu = cpu_baseline(args.cpu_replicates, steps=args.steps, warmup=args.warmup)
    value = cpu["value"]
    secs = time.perf_counter() - t0
    line = {
        "metric": METRIC, "value": value, "unit": "replicates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": len(CPU_SAMPLE_GAMMAS) * len(NS) * args.cpu_replicates / value * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config2 untruncated sweep (bounded CPU sample)", "support": "inf",
                   "gammas": list(CPU_SAMPLE_GAMMAS), "ns": list(NS), "replicates_per_cell": args.cpu_replicates,
                   "repetitions": 1, "base_seed": 1},
        "impl": "reference",
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": "replicates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": secs,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- roofline

def hbm_peak_gbs() -> tuple[float, str]:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy bandwidth, burst)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "B200_PROFILING.md fallback (MEASURED_PEAKS.json absent)"


def ncu_counts() -> dict:
    """Per-sweep warp instructions and DRAM bytes of each kernel kind, from the committed ncu
    launch list of this bench command (tools/ncu_launch_table.py -> profiles/r02_launch_inst.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_launch_inst.json")) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {}


def roofline(work, ktimes, peaks, args, world, shard, R, ncells, total_ms, sm_mhz, sms) -> dict:
    """The dominant kernel (largest summed device time in the timed region, CUDA events around
    every launch on the engine stream) against the resource that binds it.

    The replicate math moves few bytes (about 40 B per replicate in and out), so
    HBM does not bind any kernel of the path; ncu shows them issue- and latency-bound (DRAM a few
    per cent).  The line therefore reports, per kernel kind, the issue-slot fraction -- warp
    instructions (the committed ncu launch list of this command) over the SM's issue slots
    (sms x 4 schedulers x the SM clock sampled during the run) in the kind's measured time -- beside
    its algorithmic HBM bytes over the measured copy bandwidth, and names the larger one as
    ``bound``.  Algorithmic bytes per sweep:
      row     148 B per pre-drawn row written (u16 counts 128, log-sum 8, min / max / tail length
              12) + 2 B per tail value
      fit     the same rows read back + 17 B per replicate written (ks, gamma_hat, status)
      batch   17 B per replicate written (n < 128: draws, fits and KS stay on chip)
      select  8 B per KS value per full radix pass (2 full passes, then candidates only)
    """
    (attempts, draws, evals, eval_terms, norm_terms, ks_terms, ks_tails, ks_tiles, keys, pre_rows, pre_tails) = work
    per_gpu = R if world == 1 else shard[1] - shard[0]
    small_cells = sum(1 for n in NS if n < 128) * len(GAMMAS)
    row_bytes = 128 + 8 + 12
    alg = {
        "row": row_bytes * pre_rows + 2.0 * pre_tails,
        "fit": row_bytes * pre_rows + 2.0 * pre_tails + 17.0 * pre_rows,
        "batch": 17.0 * small_cells * per_gpu,
        "select": 8.0 * 2 * ncells * per_gpu,
    }
    steps = max(args.steps, 1)
    clk_hz = (sm_mhz or 1965.0) * 1e6
    issue_peak = sms * 4 * clk_hz  # warp instructions per second
    hbm_peak, hbm_src = hbm_peak_gbs()
    ncu = ncu_counts()
    kern = {k: {"ms_per_sweep": ms / steps, "launches_per_sweep": n / steps} for k, (ms, n) in ktimes.items() if n}
    kernel_ms = sum(v["ms_per_sweep"] for v in kern.values())
    for k, v in kern.items():
        v["share_of_kernel_time"] = v["ms_per_sweep"] / kernel_ms if kernel_ms else None
        secs = v["ms_per_sweep"] / 1e3
        if k in alg and secs:
            v["algorithmic_gb_per_sweep"] = alg[k] / 1e9
            v["hbm_frac"] = alg[k] / secs / 1e9 / hbm_peak
        c = ncu.get("kinds", {}).get(k)
        if c and secs:
            v["warp_inst_per_sweep"] = c["warp_inst_per_sweep"]
            v["issue_frac"] = c["warp_inst_per_sweep"] / secs / issue_peak
            v["dram_bytes_per_sweep"] = c["dram_bytes_per_sweep"]
            v["dram_frac"] = c["dram_bytes_per_sweep"] / secs / 1e9 / hbm_peak
    dom = max(kern, key=lambda k: kern[k]["ms_per_sweep"])
    d = kern[dom]
    launch_ms = d["ms_per_sweep"] / max(d["launches_per_sweep"], 1)
    issue = d.get("issue_frac")
    hbm = d.get("hbm_frac", 0.0)
    if issue is not None and issue >= hbm:
        per_launch_inst = d["warp_inst_per_sweep"] / max(d["launches_per_sweep"], 1)
        achieved = per_launch_inst / (launch_ms / 1e3)
        roof = {"bound": "issue", "achieved": achieved, "peak": issue_peak, "unit": "warp-instructions/s",
                "frac": achieved / issue_peak,
                "peak_source": f"{sms} SMs x 4 schedulers x {clk_hz / 1e6:.0f} MHz (median SM clock sampled in the "
                               f"timed region): one warp instruction per scheduler per cycle",
                "achieved_source": "warp instructions per launch from the committed ncu launch list of this command "
                                   f"({ncu.get('source', '?')}) over the CUDA-event launch time"}
    else:
        per_launch_bytes = alg.get(dom, 0.0) / max(d["launches_per_sweep"], 1)
        achieved = per_launch_bytes / (launch_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                "peak_source": hbm_src}
    dram = d.get("dram_bytes_per_sweep")
    roof.update({
        "kernel": KERNEL_NAMES.get(dom, dom), "launch_ms": launch_ms,
        "traffic": dram / max(d["launches_per_sweep"], 1) if dram is not None else None,
        "traffic_unit": "DRAM bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum)",
        "hbm": {"algorithmic_bytes_per_launch": alg.get(dom, 0.0) / max(d["launches_per_sweep"], 1),
                "achieved_gbs": alg.get(dom, 0.0) / (d["ms_per_sweep"] / 1e3) / 1e9 if d["ms_per_sweep"] else None,
                "peak_gbs": hbm_peak, "frac": hbm, "peak_source": hbm_src},
        "timing": "CUDA events around every launch on the engine stream, summed over the timed steps",
    })
    # SURVEY.md 8(d)'s compute roofline of the REFERENCE algorithm on the same inputs: W_INT =
    # 5 mulhilo per draw (Philox4x64-10, n draws per replicate), T = the power terms it sums
    # (Newton moment evaluations x their m-rule / K terms, the fitted normaliser, min(kmax, 4096)
    # KS terms; counted in-kernel at the same iterates), each one exp + 3 FMA-class ops;
    # T_ideal = max(W_INT / P_INT, T c_exp / P_FP64) with the pipe peaks probed on this device.
    exp_flops = peaks["dfma_flops"] / peaks["exp_per_s"]  # DFMA-equivalent FLOP of one fp64 exp
    terms = eval_terms + norm_terms + ks_terms
    fp64_flops = terms * (exp_flops + 6.0)
    ref_draws = sum(n for n in NS) * len(GAMMAS) * per_gpu
    mul64 = 5.0 * ref_draws
    t_fp64 = fp64_flops / peaks["dfma_flops"]
    t_int = mul64 / peaks["mul64_per_s"]
    sweep_s = total_ms / steps / 1e3
    roof["compute"] = {
        "reference_algorithm_at_peak": {
            "t_ideal_ms_per_sweep": max(t_fp64, t_int) * 1e3, "bound": "fp64" if t_fp64 > t_int else "int64_mul",
            "speedup_over_reference_algorithm_at_peak": max(t_fp64, t_int) / sweep_s,
            "note": "the time the REFERENCE algorithm would need on this GPU at its FP64 / 64-bit-multiply peaks, "
                    "over the measured sweep time: > 1 means the engine does less work than the reference "
                    "algorithm (fit tables, Euler-Maclaurin KS endpoints, one stream per sweep row)",
            "power_terms": terms, "philox_mulhilo": mul64},
        "engine": {"philox_mulhilo_per_sweep": 5.0 * draws,
                   "int64_mul_frac_of_sweep": 5.0 * draws / peaks["mul64_per_s"] / sweep_s,
                   "peak_tmul_s": peaks["mul64_per_s"] / 1e12, "peak_dfma_tflops": peaks["dfma_flops"] / 1e12},
        "peak_source": "measured on this device by zks_probe_peaks (DFMA / fp64 exp / 64-bit mulhilo micro-kernels)",
        "work_per_sweep": {"replicates": ncells * per_gpu, "attempts": attempts, "philox_draws": draws,
                           "keys_bucketed": keys, "pre_drawn_rows": pre_rows, "pre_drawn_tail_values": pre_tails,
                           "moment_evals": evals,
                           "reference_power_terms": {"moments": eval_terms, "normaliser": norm_terms, "ks": ks_terms},
                           "ks_tail_endpoints": ks_tails, "fp64_exp_dfma_equiv": exp_flops},
    }
    roof["kernels"] = kern
    roof["kernel_share_of_step"] = kernel_ms / total_ms * steps if total_ms else None
    return roof


KERNEL_NAMES = {"row": "row_draw_kernel", "draw": "draw_stats_kernel", "fit": "fit_ks_kernel",
                "retry": "retry_kernel", "batch": "lane_row_kernel", "single": "replicate_kernel",
                "select": "select_kernel", "other": "other"}


# ----------------------------------------------------------------------------- GPU leg

def run_b200(args, world, rank, local):
    # the CPU leg first, before this process holds a CUDA context (the reference's Pool forks)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.cpu_replicates)

    import torch
    import torch.distributed as dist

    import paper_1305_6738_b200 as zk
    from paper_1305_6738_b200 import montecarlo as mc
    from paper_1305_6738_b200 import parallel
    from paper_1305_6738_b200.engine import get_engine

    torch.cuda.set_device(local)
    eng = get_engine(local)
    R = args.replicates * world  # weak scaling: replicates per GPU fixed
    support = zk.Support.unbounded()
    configs = [zk.SimulationConfig(n=n, support=support, gamma=g, base_seed=1, replicates=R, repetitions=1)
               for g in GAMMAS for n in NS]
    ncells = len(configs)
    shard = parallel.shard_bounds(R, world, rank) if world > 1 else None
    reduce = parallel.histogram_reducer() if world > 1 else None
    mc._slab(eng, parallel.padded_size(R, world))
    dev = torch.device("cuda", local)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()

    def sweep():
        plans = [mc._CellPlan(cfg) for cfg in configs]
        mc._enqueue_plans(eng, plans, shard=shard, reduce=reduce)
        return plans

    # warm-up (also builds and uploads the 21 draw tables)
    for _ in range(args.warmup):
        sweep()
    torch.cuda.synchronize()

    # work counters for the roofline: one instrumented sweep outside the timed region
    counters = torch.zeros(11, dtype=torch.int64, device=dev)
    eng.set_counters(counters)
    sweep()
    torch.cuda.synchronize()
    eng.set_counters(None)
    work = [int(x) for x in counters.cpu().tolist()]
    peaks = eng.probe_peaks()

    # timed region; every engine kernel launch is bracketed by CUDA events on its stream
    stream = torch.cuda.current_stream()
    total_ms = 0.0
    host_s = 0.0  # host time to enqueue the sweeps (the device must not wait on it)
    plans = None
    launches0 = eng.launches
    eng.set_timing(True)
    eng.kernel_times()  # reset
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            h0 = time.perf_counter()
            plans = sweep()
            host_s += time.perf_counter() - h0
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
            total_ms += e0.elapsed_time(e1)
    clock = clocks.summary()
    ktimes = eng.kernel_times()
    eng.set_timing(False)
    timed_launches = eng.launches - launches0
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = args.steps * ncells * R / (total_ms / 1e3)
    rows = {(p.config.gamma, p.config.n): tuple(c for _, c in mc._finish_cell(eng, p, shard=shard)) for p in plans}
    for row in rows.values():
        assert all(0.0 < c < 1.0 for c in row) and list(row) == sorted(row), row

    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    roof = roofline(work, ktimes, peaks, args, world, shard, R, ncells, total_ms, clock.get("sm_mhz"), sms)
    # per sample size: a sweep row's replicates over its span (first start to last finish of its
    # cells; the cells of a row are computed jointly, one stream per replicate for all gammas)
    per_n = {}
    for n in NS:
        mine = [p for p in plans if p.config.n == n]
        t0 = min(plans[0].started.elapsed_time(p.started) for p in mine)
        t1 = max(plans[0].started.elapsed_time(p.finished) for p in mine)
        per_n[str(n)] = len(mine) * (R if world == 1 else shard[1] - shard[0]) / ((t1 - t0) / 1e3) if t1 > t0 else None
    # end to end through the public API (host tables built + uploaded each step)
    e2e = None
    if not args.no_e2e:
        def api_call():
            eng.clear_tables()
            if world > 1:
                return parallel.build_table(NS, GAMMAS, support, base_seed=1, replicates=R, repetitions=1)
            return zk.build_table(NS, GAMMAS, support, base_seed=1, replicates=R, repetitions=1)

        api_call()
        torch.cuda.synchronize()
        secs = 0.0
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            table = api_call()
            secs += time.perf_counter() - t0
        tt = torch.tensor([secs], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        secs = float(tt.item())
        assert table.cells == rows, "public API and device sweep disagree"
        e2e = {"value": args.steps * ncells * R / secs, "unit": "replicates/s",
               "h2d_bytes_per_step": len(GAMMAS) * 65535 * 8,
               "d2h_bytes_per_step": ncells * (4 + 1) * 8 + (4 * ncells if world > 1 else 0),
               "api": "paper_1305_6738_b200.build_table" if world == 1 else "paper_1305_6738_b200.parallel.build_table"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "replicates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "config2: untruncated Zipf, gamma 1.5..3.5 step 0.1 x n {10,20,50,100,500,1000}",
                       "cells": ncells, "replicates_per_cell": R, "replicates_per_gpu_per_cell": args.replicates,
                       "repetitions": 1, "base_seed": 1, "parallelism": f"dp{world}",
                       "l2": "flushed between timed steps (256 MiB write)"},
            "roofline": roof,
            "per_n_replicates_per_s": per_n,
            "per_gamma_n": "every (gamma, n) cell of a row runs at its row's rate (one stream per replicate, "
                           "counted for all 21 gammas in the same launches)",
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": timed_launches,
            "host_enqueue_ms_per_step": host_s / args.steps * 1e3,
            "clocks": clock,
            "cutoffs_sample": {f"{g},{n}": rows[(g, n)] for g, n in ((1.5, 10), (2.5, 100), (3.5, 1000))},
        }
        print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    world, rank, local = dist_env()
    if world > 1 and args.impl == "b200":
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        if args.impl == "reference":
            run_reference(args, world, rank)
        else:
            run_b200(args, world, rank, local)
    finally:
        if world > 1 and args.impl == "b200":
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
