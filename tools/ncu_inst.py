"""Per-source-line executed warp instructions (top N) and the SASS opcode mix of one
ncu report (source page, needs -lineinfo)."""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname = ""
lines, ops = [], Counter()
for r in csv.reader(io.StringIO(out)):
    if not r or len(r) < 8:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    try:
        inst = float(r[7])
    except ValueError:
        continue
    if r[0] != "":
        lines.append((inst, f"{fname}:{r[0]}", r[1].strip()))
    else:
        op = r[3].split()[0] if r[3].split() else "?"
        if op.startswith("@"):
            op = r[3].split()[1]
        ops[op.split(".")[0]] += inst
tot = sum(ops.values()) or 1
print("opcode mix (% of executed warp instructions):")
print("  " + ", ".join(f"{k} {100*v/tot:.1f}" for k, v in ops.most_common(22)))
tl = sum(l[0] for l in lines) or 1
for inst, loc, src in sorted(lines, reverse=True)[:n]:
    print(f"{loc:>18} {100*inst/tl:5.1f}% | {src[:110]}")
