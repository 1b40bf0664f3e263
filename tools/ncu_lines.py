"""Per-source-line totals of an ncu report's source page (needs -lineinfo):
warp-stall samples and executed warp instructions, top N lines over all files."""
import csv
import io
import subprocess
import sys

rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname = ""
items = []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No") or len(r) < 8:
        continue
    if r[0] != "":  # a source line row with aggregated metrics
        try:
            items.append((float(r[4]), float(r[7]), f"{fname}:{r[0]}", r[1].strip()))
        except ValueError:
            pass
ts = sum(i[0] for i in items) or 1
ti = sum(i[1] for i in items) or 1
print(f"total stall samples {ts:.0f}, warp instructions {ti:.3e}")
for s, i, loc, src in sorted(items, reverse=True)[:n]:
    print(f"{loc:>18} {100*s/ts:5.1f}% samp {100*i/ti:5.1f}% inst | {src[:100]}")
