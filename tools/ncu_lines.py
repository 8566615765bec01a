"""Per CUDA-source-line warp-stall samples and executed instructions for one
kernel (ncu 'cuda,sass' source view):
python tools/ncu_lines.py report.ncu-rep KERNEL_REGEX [N] [sort: stall|inst]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
key = sys.argv[4] if len(sys.argv) > 4 else "stall"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout.splitlines()
cur_file, res, wi, ii = None, [], None, None
for line in csv.reader(out):
    if not line:
        continue
    if line[0] == "File Path":
        cur_file = line[1].split("/")[-1]
        continue
    if line[0] == "Function Name":
        continue
    if line[0] == "Line No":
        wi = line.index("Warp Stall Sampling (All Samples)")
        ii = line.index("Instructions Executed")
        continue
    if line[0] and wi is not None:
        try:
            res.append((float(line[wi] or 0), float(line[ii] or 0), cur_file, line[0], line[1][:100]))
        except (ValueError, IndexError):
            pass
ts = sum(r[0] for r in res) or 1
ti = sum(r[1] for r in res) or 1
print(f"total warp-instructions {ti:.4g}")
idx = 0 if key == "stall" else 1
for v, ins, f, l, s in sorted(res, key=lambda r: -r[idx])[:n]:
    print(f"{v / ts * 100:5.1f}% stall {ins / ti * 100:5.1f}% inst  {f}:{l}  {s}")
