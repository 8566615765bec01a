"""List the loops (backward branches) of one SASS function with their body sizes
and instruction mix: python tools/sass_loops.py file.sass FUNCNAME_SUBSTR"""
import re
import sys
from collections import Counter

text = open(sys.argv[1]).read().split("Function : ")
fn = [t for t in text if t.startswith(sys.argv[2]) or sys.argv[2] in t.split("\n")[0]]
body = fn[0]
ins = []
for line in body.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
print(f"{len(ins)} instructions")
for i, (a, t) in enumerate(ins):
    m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)\s*)?.*?0x([0-9a-f]+)", t)
    if "BRA" in t:
        mm = re.search(r"0x([0-9a-f]+)", t.split("BRA")[1])
        if mm:
            tgt = int(mm.group(1), 16)
            if tgt <= a and tgt in addr:
                j = addr[tgt]
                seg = [x[1] for x in ins[j:i + 1]]
                ops = Counter(s.split()[0] if not s.startswith("@") else s.split()[1] for s in seg)
                op2 = Counter(o.split(".")[0] for o in ops.elements())
                print(f"loop {tgt:#x}-{a:#x}: {len(seg)} instr  " + " ".join(f"{k}:{v}" for k, v in op2.most_common(14)))
