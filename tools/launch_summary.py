"""Summarize an ncu --metrics gpu__time_duration.sum --csv launch list: share per kernel."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, {}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            k = d["Kernel Name"].split("(")[0][:70]
            v = float(d["Metric Value"].replace(",", ""))
            unit = d.get("Metric Unit", "ns")
            v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
            a = agg.setdefault(k, [0, 0.0])
            a[0] += 1
            a[1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'share':>7} {'launches':>8} {'total ms':>10} {'avg ms':>9}  kernel")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v / tot * 100:6.2f}% {c:8d} {v:10.3f} {v / c:9.4f}  {k}")
