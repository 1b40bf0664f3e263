"""Shared-memory wavefronts per CUDA source line of an ncu report (source page, -lineinfo):
actual vs ideal (the excess is bank conflicts), top N lines by excess."""
import csv
import io
import subprocess
import sys

rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, rows = "", None, []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or r[0] == "":
        continue
    h = {k: i for i, k in enumerate(hdr)}
    try:
        wf = float(r[h["L1 Wavefronts Shared"]] or 0)
        ide = float(r[h["L1 Wavefronts Shared Ideal"]] or 0)
    except (KeyError, ValueError):
        continue
    if wf > 0:
        rows.append((wf - ide, wf, ide, f"{fname}:{r[0]}", r[1].strip()))
tw = sum(x[1] for x in rows) or 1
ti = sum(x[2] for x in rows)
print(f"shared wavefronts {tw:.4g}, ideal {ti:.4g}, excess {tw - ti:.4g} ({100 * (tw - ti) / tw:.1f}%)")
for ex, wf, ide, loc, src in sorted(rows, key=lambda x: -x[0])[:n]:
    print(f"{loc:>18} excess {ex:10.4g} ({100 * ex / tw:4.1f}% of all)  wf {wf:10.4g} ideal {ide:10.4g}  {src[:60]}")
