"""Device throughput of BASELINE.json configs 1, 3 and 4 (bench.py's line is config 2).

One untimed warm-up sweep (draw tables built and uploaded), then ``--steps`` timed sweeps,
each bracketed by CUDA events on the engine's stream with L2 flushed before it; per-cell
device times from the cell plans' own events.  Prints one JSON line per config.

    python tools/config_sweeps.py [--configs 1,3,4] [--steps 2] [--replicates 1000000]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1305_6738_b200 as zk  # noqa: E402
from paper_1305_6738_b200 import montecarlo as mc  # noqa: E402
from paper_1305_6738_b200.engine import get_engine  # noqa: E402


def grid(lo, hi, step):
    k = round((hi - lo) / step)
    return tuple(round(lo + i * step, 10) for i in range(k + 1))


def configs(replicates, ns3):
    return {
        "1": ("config1: untruncated Zipf gamma=2.5, n=100, 10^4 replicates",
              zk.Support.unbounded(), (2.5,), (100,), 10_000),
        "3": (f"config3: truncated Zipf K=1000, gamma 0.5..2.0 step 0.05 x n {{{','.join(map(str, ns3))}}}",
              zk.Support.finite(1000), grid(0.5, 2.0, 0.05), ns3, replicates),
        "4": ("config4: untruncated Zipf gamma=2.0, n {10^5, 2x10^5, 5x10^5, 10^6}, 10^5 replicates",
              zk.Support.unbounded(), (2.0,), (100_000, 200_000, 500_000, 1_000_000), 100_000),
    }


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--configs", default="1,3,4")
    p.add_argument("--steps", type=int, default=2)
    p.add_argument("--replicates", type=int, default=1_000_000, help="replicates per cell for config 3")
    p.add_argument("--rng", default="numpy", help="numpy (bit-exact, default) or philox4x32 (opt-in fast stream)")
    p.add_argument("--ns3", default="10,20,30,40,50,100,500,1000,2000,3000,4000,5000,10000",
                   help="config-3 sample sizes (the paper's grid <= 10^4)")
    args = p.parse_args()
    eng = get_engine(0)
    eng.set_rng(args.rng)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    table = configs(args.replicates, tuple(int(x) for x in args.ns3.split(",")))
    for key in args.configs.split(","):
        name, support, gammas, ns, R = table[key]
        cfgs = [zk.SimulationConfig(n=n, support=support, gamma=g, base_seed=1, replicates=R, repetitions=1)
                for g in gammas for n in ns]
        mc._slab(eng, R)

        def sweep():
            plans = [mc._CellPlan(c) for c in cfgs]
            mc._enqueue_plans(eng, plans)
            return plans

        sweep()
        torch.cuda.synchronize()
        total_ms = 0.0
        per_n = {n: 0.0 for n in ns}
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            plans = sweep()
            e1.record(stream)
            torch.cuda.synchronize()
            total_ms += e0.elapsed_time(e1)
            for n in ns:  # a row's span: its first start to its last finish (rows run back to back)
                mine = [pl for pl in plans if pl.config.n == n]
                t0 = min(e0.elapsed_time(pl.started) for pl in mine)
                t1 = max(e0.elapsed_time(pl.finished) for pl in mine)
                per_n[n] += t1 - t0
        rows = {(pl.config.gamma, pl.config.n): tuple(c for _, c in mc._finish_cell(eng, pl)) for pl in plans}
        for row in rows.values():
            assert all(0.0 < c < 1.0 for c in row) and list(row) == sorted(row), row
        reps = args.steps * len(cfgs) * R
        line = {
            "config": name, "rng": args.rng, "cells": len(cfgs), "replicates_per_cell": R, "steps": args.steps,
            "ms_per_sweep": total_ms / args.steps, "replicates_per_s": reps / (total_ms / 1e3),
            "draws_per_s": args.steps * R * len(gammas) * sum(ns) / (total_ms / 1e3),
            "per_n_replicates_per_s": {str(n): args.steps * len(gammas) * R / (ms / 1e3) for n, ms in per_n.items()},
            "cutoffs_sample": {f"{g},{n}": rows[(g, n)] for g, n in list(rows)[:: max(1, len(rows) // 4)]},
        }
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
