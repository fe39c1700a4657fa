"""Per-sweep warp instructions, DRAM bytes and device time of each engine kernel kind, from an ncu
launch list of ``bench.py`` (every launch, metrics gpu__time_duration.sum, smsp__inst_executed.sum,
dram__bytes_read.sum, dram__bytes_write.sum; --clock-control none):

    ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/launches.csv \
        python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline
    python tools/ncu_launch_table.py gpurun_out/launches.csv profiles/r02_launch_inst.json

A bench run at --warmup W --steps S runs W + 1 + S sweeps (the +1: the work-counter sweep); each
sweep has 6 selection launches (one per sample size), which is how sweeps are counted here.
bench.py reads the JSON for the issue-slot and DRAM fractions of its roofline.
"""
import collections
import csv
import json
import sys

KINDS = {"row_draw_kernel": "row", "draw_stats_kernel": "draw", "fit_ks_kernel": "fit", "long_tail_kernel": "fit", "retry_kernel": "retry",
         "lane_row_kernel": "batch", "replicate_kernel": "single", "select_kernel": "select"}
SCALE_T = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
SCALE_B = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def kind_of(name: str):
    base = name.split("(")[0].split("<")[0].replace("void ", "").split("::")[-1].strip()
    return KINDS.get(base)


def main(path: str, out: str) -> None:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ix = {h: i for i, h in enumerate(hdr)}
    acc = collections.defaultdict(lambda: collections.defaultdict(float))
    launches = collections.Counter()
    counted = set()
    for r in rows[hi + 1:]:
        if len(r) < len(hdr):
            continue
        name = r[ix["Kernel Name"]]
        k = kind_of(name)
        if k is None:
            continue
        if "<1" in name or "<true" in name:  # the kCount (work-counter) variants of the counting sweep
            counted.add(k)
            continue
        metric, unit = r[ix["Metric Name"]], r[ix["Metric Unit"]]
        val = float(r[ix["Metric Value"]].replace(",", ""))
        if metric == "gpu__time_duration.sum":
            acc[k]["ms"] += val * SCALE_T[unit]
            launches[k] += 1
        elif metric == "smsp__inst_executed.sum":
            acc[k]["inst"] += val
        elif metric.startswith("dram__bytes_"):
            acc[k]["dram"] += val * SCALE_B.get(unit, 1.0)
    sweeps = launches["select"] / 6.0
    selects = sweeps
    if counted:  # one of the sweeps ran the counting variants (skipped above)
        sweeps -= 1.0
    res = {"source": f"ncu launch list {path} ({sweeps:g} sweeps of bench.py, --clock-control none; per-launch "
                     "times are cold-cache and serialised)", "sweeps": sweeps, "kinds": {}}
    for k, a in acc.items():
        n_sw = selects if k == "select" else sweeps  # the selection has no counting variant
        res["kinds"][k] = {"warp_inst_per_sweep": a["inst"] / n_sw, "dram_bytes_per_sweep": a["dram"] / n_sw,
                           "ncu_ms_per_sweep": a["ms"] / n_sw, "launches_per_sweep": launches[k] / n_sw}
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
