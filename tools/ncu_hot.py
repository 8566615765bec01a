"""Top SASS instructions by warp-stall samples for one kernel of an ncu report."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
hdr = rows[0]
si, wi = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for idx, r in enumerate(rows[1:]):
    try:
        data.append((float(r[wi] or 0), idx, r[si].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
print(f"{kern}: {len(data)} SASS instrs, {tot:.0f} samples")
for v, idx, s in sorted(data, reverse=True)[:n]:
    print(f"{v / tot * 100:5.1f}% #{idx:5d} {s}")
