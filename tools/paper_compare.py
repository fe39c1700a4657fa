"""Compare a config-5 run (tools/config5.py summary) with the paper's published tables.

For every cell (support, gamma, n <= 10^4) and level: delta = our 10^7-replicate cutoff - the
published value (tests/golden/paper_tables.json), and
z = delta / sigma with sigma^2 = sigma_MC^2 + sigma_round^2:
  * sigma_MC: the Monte Carlo standard error of a published cutoff (the paper's protocol,
    50,000 replicates x 10 repetitions averaged), measured from the per-repetition spread of our
    own run of that protocol;
  * sigma_round: the 4-decimal rounding of the published numbers, 0.5e-4 / sqrt(3).
Also checks our own two protocols against each other (z_self = (paper-protocol cutoff - target
cutoff) / sigma_MC), which must look like N(0, 1) draws.

    python tools/paper_compare.py gpurun_out/config5/config5_summary.json --out profiles/r02_config5_vs_paper.json
"""
from __future__ import annotations

import argparse
import json
import math
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LEVELS = (0.9, 0.95, 0.99, 0.999)
SIGMA_ROUND = 0.5e-4 / math.sqrt(3.0)


def compare(summary: dict, paper: dict, z_flag: float = 4.0) -> dict:
    report = {"sigma_round": SIGMA_ROUND, "supports": {}}
    for label, entry in summary["supports"].items():
        pub = paper[label]
        tgt = entry["target"]["cutoffs"]
        prot = entry.get("paper_protocol", {})
        sig = prot.get("sigma", {})
        rows = []
        for key, ours in tgt.items():
            g, n = key.split(",")
            pkey = f"{float(g)},{int(n)}"
            if pkey not in pub:
                continue
            for li, level in enumerate(LEVELS):
                s_mc = sig[key][li] if key in sig else float("nan")
                s = math.sqrt(s_mc ** 2 + SIGMA_ROUND ** 2)
                d = ours[li] - pub[pkey][li]
                z_self = (prot["cutoffs"][key][li] - ours[li]) / s_mc if key in sig and s_mc > 0 else float("nan")
                rows.append({"gamma": float(g), "n": int(n), "level": level, "ours": ours[li],
                             "paper": pub[pkey][li], "delta": d, "sigma": s, "sigma_mc": s_mc, "z": d / s,
                             "z_self": z_self})
        z = np.array([r["z"] for r in rows])
        zs = np.array([r["z_self"] for r in rows])
        d = np.array([r["delta"] for r in rows])
        out = [r for r in rows if abs(r["z"]) > z_flag]
        report["supports"][label] = {
            "compared": len(rows),
            "max_abs_delta": float(np.max(np.abs(d))),
            "median_abs_delta": float(np.median(np.abs(d))),
            "max_abs_z": float(np.max(np.abs(z))),
            "frac_abs_z_le_2": float(np.mean(np.abs(z) <= 2.0)),
            "frac_abs_z_le_3": float(np.mean(np.abs(z) <= 3.0)),
            "mean_z": float(np.mean(z)),
            "self_max_abs_z": float(np.nanmax(np.abs(zs))),
            "self_frac_abs_z_le_2": float(np.nanmean(np.abs(zs) <= 2.0)),
            "outliers": sorted(out, key=lambda r: -abs(r["z"])),
        }
    return report


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("summary")
    ap.add_argument("--paper", default=os.path.join(ROOT, "tests", "golden", "paper_tables.json"))
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    with open(args.summary) as fh:
        summary = json.load(fh)
    with open(args.paper) as fh:
        paper = json.load(fh)["tables"]
    rep = compare(summary, paper)
    for label, r in rep["supports"].items():
        print(f"K={label:>4}: {r['compared']:4d} cutoffs, max|d| {r['max_abs_delta']:.4f}, median|d| "
              f"{r['median_abs_delta']:.5f}, |z|<=2 {r['frac_abs_z_le_2']:.2f}, |z|<=3 {r['frac_abs_z_le_3']:.2f}, "
              f"max|z| {r['max_abs_z']:.1f}, mean z {r['mean_z']:+.2f}, outliers {len(r['outliers'])}; "
              f"self-check |z|<=2 {r['self_frac_abs_z_le_2']:.2f} max {r['self_max_abs_z']:.1f}")
        for o in r["outliers"][:8]:
            print(f"    gamma={o['gamma']} n={o['n']} q={o['level']}: ours {o['ours']:.5f} paper {o['paper']:.4f} "
                  f"z={o['z']:+.1f}")
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(rep, fh, indent=1)


if __name__ == "__main__":
    main()
