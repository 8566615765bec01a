"""Per-kernel DRAM traffic of one `ncu --set full` capture, as the JSON bench.py
reads for roofline.traffic:  python tools/ncu_traffic.py rep.ncu-rep "what ran" > profiles/rNN/ncu_traffic.json"""
import csv
import json
import subprocess
import sys

rep, what = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
rows = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                      text=True).stdout.splitlines()))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
tscale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}
out = {"_capture": {"report": rep, "command": what,
                    "commit": subprocess.run(["git", "rev-parse", "--short", "HEAD"], capture_output=True,
                                             text=True).stdout.strip()}}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].split("(")[0].replace("void ", "").split("<")[0].replace("pb::", "")
    u = dict(zip(hdr, units))
    rd = float(d["dram__bytes_read.sum"].replace(",", "")) * scale[u["dram__bytes_read.sum"]]
    wr = float(d["dram__bytes_write.sum"].replace(",", "")) * scale[u["dram__bytes_write.sum"]]
    t = float(d["gpu__time_duration.sum"].replace(",", "")) * tscale[u["gpu__time_duration.sum"]]
    out[name] = {"dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes": rd + wr, "duration_s": t}
print(json.dumps(out, indent=1))
