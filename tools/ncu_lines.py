"""Per CUDA-source-line warp-stall samples for one kernel (ncu 'cuda,sass' source view)."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout.splitlines()
cur_file, rows, res = None, [], []
for line in csv.reader(out):
    if not line:
        continue
    if line[0] == "File Path":
        cur_file = line[1].split("/")[-1]
        continue
    if line[0] in ("Function Name", "Line No"):
        hdr = line if line[0] == "Line No" else None
        if hdr:
            wi = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if line[0] and line[0] != "":
        try:
            res.append((float(line[wi] or 0), cur_file, line[0], line[1][:100]))
        except (ValueError, IndexError):
            pass
tot = sum(r[0] for r in res) or 1
for v, f, l, s in sorted(res, reverse=True)[:n]:
    print(f"{v / tot * 100:5.1f}% {f}:{l}  {s}")
