"""Extract the published cutoff tables of the paper into
tests/golden/paper_tables.json: {"inf"|"20"|...: {"gamma,n": [q90, q95, q99, q999]}}.

Run in the build container (the reference tree does not travel to the GPU box):
    python tests/golden/make_paper_tables.py
"""
from __future__ import annotations

import json
import os
import re

SRC = "/root/reference/PAPER.md"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "paper_tables.json")


def parse(text: str) -> dict:
    tables: dict = {}
    support = None
    gammas: list[float] = []
    for line in text.splitlines():
        cap = re.search(r"\\caption\{KS test statistic for the (pure|truncated) power-law distribution"
                        r"(?: with \$K=(\d+)\$)?", line)
        if cap:
            support = "inf" if cap.group(1) == "pure" else cap.group(2)
            tables.setdefault(support, {})
            continue
        if support is None:
            continue
        if "multicolumn" in line and "gamma" in line:
            gammas = [float(g) for g in re.findall(r"\\gamma=([0-9.]+)", line)]
            continue
        row = re.match(r"^\s*(\d+)&(.*)\\\\\s*$", line)
        if row and gammas:
            n = int(row.group(1))
            vals = [float(v) for v in re.findall(r"\.\d+", row.group(2))]
            assert len(vals) == 4 * len(gammas), (line, gammas)
            for i, g in enumerate(gammas):
                tables[support][f"{g},{n}"] = vals[4 * i : 4 * i + 4]
        if line.startswith("\\end{table*}"):
            support = None
    return tables


def main() -> None:
    with open(SRC, encoding="utf-8") as fh:
        tables = parse(fh.read())
    counts = {k: len(v) for k, v in tables.items()}
    assert counts == {"inf": 120, "20": 180, "50": 180, "100": 180, "500": 180, "1000": 180}, counts
    with open(OUT, "w", encoding="utf-8") as fh:
        json.dump({"source": "PAPER.md:273-661 (published tables, 4 decimals)", "tables": tables}, fh, indent=0,
                  sort_keys=True)
    print(OUT, counts)


if __name__ == "__main__":
    main()
