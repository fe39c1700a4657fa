"""profiles/traffic.json from an ncu --set full report of one draw_stats launch + traffic_capture output."""
import csv, io, json, subprocess, sys

rep, cap_log, out = sys.argv[1], sys.argv[2], sys.argv[3]
cap = json.loads([l for l in open(cap_log) if l.startswith("{")][-1])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
def metric(name):
    i = hdr.index(name)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6,
             "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}
    return float(vals[i].replace(",", "")) * scale.get(units[i], 1)
rd, wr = metric("dram__bytes_read.sum"), metric("dram__bytes_write.sum")
res = {"kernel": "draw_stats_kernel", "source": f"ncu --set full --clock-control none, {rep.split('/')[-1]}: "
       f"one staged draw_stats launch, gamma={cap['gamma']} n={cap['n']} rows={cap['rows']}",
       "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes": rd + wr,
       "algorithmic_bytes": cap["algorithmic_bytes"], "launch": cap,
       "duration_s": metric("gpu__time_duration.sum")}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
