"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) into per-kernel shares."""
import collections, csv, sys

def summarise(path, title):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ix = {h: i for i, h in enumerate(hdr)}
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0]
        tot[name] += float(r[ix["Metric Value"]].replace(",", "")) * scale[r[ix["Metric Unit"]]]
        cnt[name] += 1
    T = sum(tot.values())
    out = [f"# {title}", "# gpu__time_duration.sum, --clock-control none; launches are cold-cache and serialised: compare SHARES",
           f"# total kernel time {T:.1f} ms over {sum(cnt.values())} launches", "kernel,launches,total_ms,share"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"{k},{cnt[k]},{v:.3f},{v / T:.4f}")
    return "\n".join(out) + "\n"

if __name__ == "__main__":
    text = summarise(sys.argv[1], sys.argv[3] if len(sys.argv) > 3 else sys.argv[1])
    open(sys.argv[2], "w").write(text)
    print(text)
