"""Summarise an ncu report: key throughput / occupancy / stall numbers (+ top stall lines)."""
import csv, io, subprocess, sys, collections

KEYS = ["Duration", "Elapsed Cycles", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issued Warp Per Scheduler", "No Eligible",
        "Active Warps Per Scheduler", "Eligible Warps Per Scheduler", "Registers Per Thread",
        "Theoretical Occupancy", "Achieved Occupancy", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size",
        "Warp Cycles Per Issued Instruction"]

def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    res = collections.OrderedDict()
    for r in rows[1:]:
        name = r[ix["Metric Name"]]
        if name in KEYS and name not in res:
            res[name] = (r[ix["Metric Value"]], r[ix["Metric Unit"]])
    return res, rows[1][ix["Kernel Name"]] if len(rows) > 1 else "?"

def raw(rep, pats):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals) if any(p in h for p in pats)}

if __name__ == "__main__":
    rep = sys.argv[1]
    d, kname = details(rep)
    print(f"report: {rep}\nkernel: {kname}")
    for k, (v, u) in d.items():
        print(f"  {k:40s} {v:>14s} {u}")
    pats = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak",
            "sm__inst_executed_pipe_fp64", "sm__pipe_alu_cycles_active.avg.pct", "sm__pipe_fma_cycles_active.avg.pct",
            "sm__inst_executed_pipe_lsu.avg.pct", "smsp__pcsamp_warps_issue_stalled", "sm__pipe_shared_cycles_active.avg.pct",
            "sm__pipe_fmaheavy_cycles_active.avg.pct", "smsp__inst_executed.sum", "sm__pipe_int"]
    r = raw(rep, pats)
    stalls = {k: v for k, v in r.items() if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")}
    for k, (v, u) in sorted(r.items()):
        if "pcsamp" in k:
            continue
        print(f"  {k:70s} {v:>16s} {u}")
    top = sorted(((float(v[0].replace(',', '')) if v[0] else 0.0, k) for k, v in stalls.items()), reverse=True)[:8]
    print("  top stall reasons (pc samples):")
    for v, k in top:
        print(f"    {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):40s} {v:12.0f}")
