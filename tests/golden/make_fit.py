"""Record the reference CLI's own ``fit`` outputs (pkg/src/zipfks/cli.py:197-262) for fixed
observation files and seeds: tests/golden/fit/*.txt (observations, tables) and fit.json
(argv, exit code, stdout, stderr of the UNMODIFIED reference run as ``python -m zipfks``).

Run in the build container (where /root/reference exists):
    python tests/golden/make_fit.py
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "fit")


def run(*args):
    env = dict(os.environ, PYTHONPATH=REF)
    r = subprocess.run([sys.executable, "-m", "zipfks", *args], capture_output=True, text=True, env=env,
                       timeout=3600, cwd=OUT)
    return {"argv": list(args), "rc": r.returncode, "stdout": r.stdout, "stderr": r.stderr}


def main() -> None:
    sys.path.insert(0, REF)
    import numpy as np
    from zipfks.distribution import RandomStream, Support, ZipfModel, sample
    from zipfks.estimate import mle_gamma
    from zipfks.observations import write_observations

    os.makedirs(OUT, exist_ok=True)

    def obs(name, gamma, k, n, seed):
        drawn = sample(ZipfModel(gamma, Support(k=k)), n, RandomStream.for_replicate(seed, 0, 0))
        write_observations(drawn, os.path.join(OUT, name))
        return drawn

    obs("inf_g22_n300.txt", 2.2, None, 300, 6)
    obs("k1000_g10_n150.txt", 1.0, 1000, 150, 4)
    d = obs("k100_g20_n200.txt", 2.0, 100, 200, 6)
    obs("k100_g35_n200.txt", 3.5, 100, 200, 6)
    rng = np.random.default_rng(2)
    geo = np.minimum(rng.geometric(0.5, size=2000), 100)
    with open(os.path.join(OUT, "geo_k100.txt"), "w") as fh:
        fh.write("\n".join(str(int(v)) for v in geo))
    with open(os.path.join(OUT, "bad_token.txt"), "w") as fh:
        fh.write("1 2\n3 x5 4\n")
    with open(os.path.join(OUT, "above_support.txt"), "w") as fh:
        fh.write("1 2 300\n")
    with open(os.path.join(OUT, "tiny.txt"), "w") as fh:
        fh.write("1 1 2\n")
    # a table whose grid holds the k100 sample's (rounded) estimate, made by the reference itself
    gh = mle_gamma(d, Support.finite(100))
    cases = {
        "table_build": run("simulate", "--n", "200", "--gamma", f"{round(gh, 2)}", "--k", "100", "--replicates",
                           "400", "--reps", "1", "--seed", "11", "--out", "t_k100.csv", "--workers", "1"),
        "inf_bespoke_machine": run("fit", "--input", "inf_g22_n300.txt", "--k", "inf", "--bespoke", "--replicates",
                                   "2000", "--reps", "2", "--seed", "7", "--workers", "1", "--machine"),
        "inf_bespoke_human": run("fit", "--input", "inf_g22_n300.txt", "--k", "inf", "--bespoke", "--replicates",
                                 "2000", "--reps", "2", "--seed", "7", "--workers", "1"),
        "k1000_bespoke_machine": run("fit", "--input", "k1000_g10_n150.txt", "--k", "1000", "--bespoke",
                                     "--replicates", "1000", "--reps", "3", "--seed", "9", "--workers", "1",
                                     "--machine"),
        "geo_rejected": run("fit", "--input", "geo_k100.txt", "--k", "100", "--bespoke", "--replicates", "400",
                            "--reps", "1", "--seed", "8", "--workers", "1", "--machine"),
        "tiny_perfect": run("fit", "--input", "tiny.txt", "--k", "2", "--bespoke", "--replicates", "100", "--reps",
                            "1", "--seed", "3", "--workers", "1"),
        "bad_token": run("fit", "--input", "bad_token.txt", "--k", "100", "--bespoke"),
        "above_support": run("fit", "--input", "above_support.txt", "--k", "100", "--bespoke"),
        "missing_file": run("fit", "--input", "no_such_file.txt", "--k", "100", "--bespoke"),
    }
    cases["table_lookup"] = run("fit", "--input", "k100_g20_n200.txt", "--k", "100", "--table", "t_k100.csv")
    cases["table_wrong_support"] = run("fit", "--input", "tiny.txt", "--k", "50", "--table", "t_k100.csv")
    cases["table_no_match"] = run("fit", "--input", "k100_g35_n200.txt", "--k", "100", "--table", "t_k100.csv")
    cases["table_missing"] = run("fit", "--input", "tiny.txt", "--k", "2", "--table", "no_such_table.csv")
    with open(os.path.join(OUT, "fit.json"), "w") as fh:
        json.dump(cases, fh, indent=1, sort_keys=True)
    for k, v in cases.items():
        print(k, v["rc"], v["stdout"][:80].replace("\n", " | "), v["stderr"][:80].replace("\n", " | "))


if __name__ == "__main__":
    main()
