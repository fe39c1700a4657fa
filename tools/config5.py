"""BASELINE config 5 / the north_star "Target": the paper's whole cutoff-table sweep on one GPU.

Grids of the reference's shipped tables (pkg/src/zipfks/cli.py:24-26): K = inf x 8 gammas and
K in {20, 50, 100, 500, 1000} x 12 gammas, every n <= 10^4 of REFERENCE_NS (13 sizes; --ns to
change), filled by build_table (montecarlo.py:263-314) on the device.

Two protocols per support:
  * target: R = 10^7 replicates per cell, 1 repetition, base_seed 1 (BASELINE configs[4]);
  * paper:  R = 50,000 x 10 repetitions (the reference's default protocol and the paper's),
            whose per-repetition spread gives the Monte Carlo standard error of a published
            cutoff (std over repetitions / sqrt(10)).
Writes one table file per (support, protocol) in the reference's CSV format, and a JSON summary
with device / wall times, clocks sampled during the run, and every cell's cutoffs and sigma.

    python tools/config5.py --out-dir gpurun_out/config5
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


class Clocks:
    """nvidia-smi samples (SM clock, throttle reasons) while the sweep runs."""

    def __init__(self):
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        q = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active"
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-i", "0"],
                                     capture_output=True, text=True, timeout=10).stdout.strip()
                sm, smax, pw, reasons = [x.strip() for x in out.split(",")]
                self.samples.append((float(sm), float(smax), float(pw), reasons))
            except Exception:
                pass
            self._stop.wait(1.0)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join()

    def summary(self):
        if not self.samples:
            return None
        sm = [s[0] for s in self.samples]
        return {"sm_mhz_median": float(np.median(sm)), "sm_mhz_min": min(sm), "sm_max_mhz": self.samples[0][1],
                "power_w_max": max(s[2] for s in self.samples),
                "reasons": sorted({s[3] for s in self.samples}), "samples": len(self.samples)}


def run_support(zk, mc, support, gammas, ns, replicates, reps, seed):
    """Fill one table; returns (CutoffTable, per-cell per-repetition quantiles, device s, wall s)."""
    import torch

    eng = mc._engine()
    plans = []
    for g in gammas:
        for n in ns:
            plans.append(mc._CellPlan(mc.SimulationConfig(n=n, support=support, gamma=g, base_seed=seed,
                                                          replicates=replicates, repetitions=reps)))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    stream = eng.bind_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    mc._enqueue_plans(eng, plans)
    e1.record(stream)
    mc._fetch_plans(plans)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    device = e0.elapsed_time(e1) / 1e3
    cells, per_rep = {}, {}
    for p in plans:
        pairs = mc._finish_cell(eng, p)
        cells[(p.config.gamma, p.config.n)] = tuple(c for _, c in pairs)
        per_rep[(p.config.gamma, p.config.n)] = np.asarray(p.host[0])
    table = mc.CutoffTable(support=support, levels=mc.DEFAULT_LEVELS, gammas=tuple(gammas), ns=tuple(ns),
                           cells=cells, replicates=replicates, repetitions=reps, base_seed=seed)
    return table, per_rep, device, wall


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--out-dir", default="gpurun_out/config5")
    ap.add_argument("--ns", default="10,20,30,40,50,100,500,1000,2000,3000,4000,5000,10000")
    ap.add_argument("--supports", default="inf,20,50,100,500,1000")
    ap.add_argument("--replicates", type=int, default=10_000_000)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--paper-seed", type=int, default=2)
    ap.add_argument("--skip-paper", action="store_true")
    ap.add_argument("--no-warmup", action="store_true")
    args = ap.parse_args()

    import paper_1305_6738_b200 as zk
    from paper_1305_6738_b200 import cli, montecarlo as mc, tablefile

    os.makedirs(args.out_dir, exist_ok=True)
    ns = tuple(int(x) for x in args.ns.split(","))
    summary = {"ns": ns, "replicates": args.replicates, "seed": args.seed, "supports": {}}
    total_cells = total_reps = 0
    dev_total = wall_total = 0.0
    mc._engine()
    if not args.no_warmup:
        # untimed: the engine's scratch at its largest (the pre-drawn-row chunk of the largest row,
        # the small-n words), so the timed grid measures the steady state, not first-touch
        # allocation of tens of GB
        zk.build_table((max(ns),), cli.REFERENCE_GAMMAS_FINITE, zk.Support.finite(1000), base_seed=99,
                       replicates=400_000, repetitions=1)
        zk.build_table((min(100, max(ns)),), cli.REFERENCE_GAMMAS_FINITE, zk.Support.finite(1000), base_seed=99,
                       replicates=1_000_000, repetitions=1)
    with Clocks() as clk:
        for label in args.supports.split(","):
            support = zk.Support.unbounded() if label == "inf" else zk.Support.finite(int(label))
            gammas = cli.REFERENCE_GAMMAS_UNBOUNDED if label == "inf" else cli.REFERENCE_GAMMAS_FINITE
            entry = {}
            table, _, dev, wall = run_support(zk, mc, support, gammas, ns, args.replicates, 1, args.seed)
            path = os.path.join(args.out_dir, f"config5_k{label}_r{args.replicates}_s{args.seed}.csv")
            tablefile.write_table(table, path)
            entry["target"] = {"device_s": dev, "wall_s": wall, "cells": len(table.cells), "file": path,
                               "cutoffs": {f"{g},{n}": list(v) for (g, n), v in table.cells.items()}}
            total_cells += len(table.cells)
            total_reps += len(table.cells) * args.replicates
            dev_total += dev
            wall_total += wall
            print(f"K={label}: {len(table.cells)} cells x {args.replicates}: device {dev:.2f} s, wall {wall:.2f} s",
                  flush=True)
            if not args.skip_paper:
                ptab, per_rep, pdev, pwall = run_support(zk, mc, support, gammas, ns, 50000, 10, args.paper_seed)
                ppath = os.path.join(args.out_dir, f"config5_k{label}_r50000x10_s{args.paper_seed}.csv")
                tablefile.write_table(ptab, ppath)
                entry["paper_protocol"] = {
                    "device_s": pdev, "wall_s": pwall, "file": ppath,
                    "cutoffs": {f"{g},{n}": list(v) for (g, n), v in ptab.cells.items()},
                    # standard error of a 10-repetition average (the paper's protocol)
                    "sigma": {f"{g},{n}": list(np.std(q, axis=0, ddof=1) / np.sqrt(q.shape[0]))
                              for (g, n), q in per_rep.items()},
                }
                print(f"K={label}: paper protocol 50000x10: device {pdev:.2f} s, wall {pwall:.2f} s", flush=True)
            summary["supports"][label] = entry
    summary["total"] = {"cells": total_cells, "replicates": total_reps, "device_s": dev_total, "wall_s": wall_total,
                        "replicates_per_s": total_reps / dev_total if dev_total else None}
    summary["clocks"] = clk.summary()
    with open(os.path.join(args.out_dir, "config5_summary.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps({"total": summary["total"], "clocks": summary["clocks"]}))


if __name__ == "__main__":
    main()
