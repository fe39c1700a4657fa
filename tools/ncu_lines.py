"""Top source lines of an ncu report by warp-stall samples and by instructions executed."""
import csv, io, subprocess, sys

def lines(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    res = []
    cur = None
    hdr = None
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path" or row[0] == "File Name":
            cur = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = {h: i for i, h in enumerate(row)}
            continue
        if hdr is None or not row[0].isdigit():
            continue
        def g(name):
            v = row[hdr[name]] if name in hdr and hdr[name] < len(row) else "0"
            try:
                return float(v)
            except ValueError:
                return 0.0
        res.append((cur, int(row[0]), row[1][:90], g("Warp Stall Sampling (All Samples)"), g("Instructions Executed")))
    return res

if __name__ == "__main__":
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    L = lines(rep)
    ts = sum(x[3] for x in L) or 1
    ti = sum(x[4] for x in L) or 1
    print(f"total stall samples {ts:.0f}, warp instructions {ti:.3e}")
    print("-- by stall samples")
    for f, ln, src, s, i in sorted(L, key=lambda x: -x[3])[:n]:
        print(f"{100*s/ts:5.1f}% {100*i/ti:5.1f}%  {f}:{ln:<4d} {src}")
    print("-- by instructions executed")
    for f, ln, src, s, i in sorted(L, key=lambda x: -x[4])[:n]:
        print(f"{100*s/ts:5.1f}% {100*i/ti:5.1f}%  {f}:{ln:<4d} {src}")
