"""Generate cutoff-table CSV fixtures with the reference ``zipfks`` package itself.

Run in the build container (where ``/root/reference`` exists):

    python tests/golden/make_tables.py

Each fixture is the UNMODIFIED reference's ``build_table`` + ``write_table`` output (the
third through its own CLI, ``zipfks tables``).  The CSVs are committed; tests compare the
engine's tables and files against them without reading ``/root/reference``.
"""
from __future__ import annotations

import os
import sys

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))

# name -> build_table keyword arguments (support given as K, None = unbounded)
TABLES = {
    "table_k20_s5.csv": dict(ns=(20, 50), gammas=(1.0, 1.5), k=20, base_seed=5, replicates=200, repetitions=1),
    "table_inf_s3.csv": dict(ns=(10, 100, 300), gammas=(1.5, 2.5), k=None, base_seed=3, replicates=300,
                             repetitions=2),
    "table_k1000_s8.csv": dict(ns=(40, 200), gammas=(0.5, 1.25), k=1000, base_seed=8, replicates=256,
                               repetitions=1),
}
CLI_TABLE = ("tables_k20_r100_s13.csv", ["tables", "--k", "20", "--replicates", "100", "--reps", "1",
                                         "--seed", "13", "--workers", "1"])


def main() -> None:
    sys.path.insert(0, REF)
    import zipfks
    from zipfks import cli
    from zipfks.distribution import Support
    from zipfks.montecarlo import build_table
    from zipfks.tablefile import write_table

    assert zipfks.__version__ == "1.0.0"
    for name, kw in TABLES.items():
        kw = dict(kw)
        k = kw.pop("k")
        support = Support.unbounded() if k is None else Support.finite(k)
        table = build_table(support=support, workers=1, **kw)
        write_table(table, os.path.join(OUT, name))
        print("wrote", name)
    name, argv = CLI_TABLE
    assert cli.main(argv + ["--out", os.path.join(OUT, name)]) == 0
    print("wrote", name)


if __name__ == "__main__":
    main()
