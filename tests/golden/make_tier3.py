"""Full-protocol cutoffs (50,000 replicates x 10 repetitions) computed by the reference itself for
the acceptance-gate cells of pkg/tests/test_acceptance.py:119-125 (and a config-2 cell).

Run in the build container (needs /root/reference):  python tests/golden/make_tier3.py
Writes tests/golden/tier3_reference.json (committed).
"""
import json
import os
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")

from zipfks.distribution import Support  # noqa: E402
from zipfks.montecarlo import SimulationConfig, run_simulation  # noqa: E402

CELLS = [  # (K or None, gamma, n, base_seed, replicates, repetitions)
    (None, 2.0, 100, 20240001, 50000, 10),
    (20, 1.0, 1000, 20240001, 50000, 10),
    (None, 1.25, 1000, 20240001, 50000, 10),
    (None, 4.0, 1000, 20240001, 50000, 10),
    (None, 2.5, 100, 1, 10000, 1),  # BASELINE config 1
]

out = []
for k, g, n, seed, R, reps in CELLS:
    t0 = time.time()
    cfg = SimulationConfig(n=n, support=Support(k), gamma=g, base_seed=seed, replicates=R, repetitions=reps)
    pairs = run_simulation(cfg, workers=os.cpu_count())
    out.append({"K": k, "gamma": g, "n": n, "base_seed": seed, "replicates": R, "repetitions": reps,
                "cutoffs": [c for _, c in pairs], "cpu_seconds": time.time() - t0})
    print(out[-1], flush=True)
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "tier3_reference.json"), "w") as fh:
    json.dump(out, fh, indent=1)
