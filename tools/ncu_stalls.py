"""Per-source-line stall-reason breakdown (top N lines by samples) of an ncu report."""
import csv
import io
import subprocess
import sys

rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, rows = "", None, []
tot = {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or r[0] == "":
        continue
    d = dict(zip(range(len(hdr)), r))
    st = {hdr[i][6:]: float(r[i] or 0) for i in range(len(hdr)) if hdr[i].startswith("stall_") and "Not Issued" not in hdr[i]}
    for k, v in st.items():
        tot[k] = tot.get(k, 0) + v
    rows.append((float(r[4] or 0), f"{fname}:{r[0]}", r[1].strip(), st))
T = sum(tot.values()) or 1
print("all lines:", ", ".join(f"{k} {100*v/T:.1f}" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
for s, loc, src, st in sorted(rows, key=lambda x: -x[0])[:n]:
    top = sorted(st.items(), key=lambda x: -x[1])[:3]
    print(f"{loc:>18} {100*s/T:5.1f}% [{', '.join(f'{k} {100*v/max(s,1):.0f}' for k, v in top)}] {src[:70]}")
