"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel:
launch count, total/avg device time and share of the listed time."""
import csv
import sys
from collections import defaultdict


def main(path, title=""):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("==")) if r]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui] if ui is not None else "us"
        v = v / 1e3 if unit in ("nsecond", "ns") else (v * 1e3 if unit in ("msecond", "ms") else v)
        tot[r[ki]] += v
        cnt[r[ki]] += 1
    s = sum(tot.values())
    print(title)
    print("cold-cache serialised per-launch times; compare SHARES")
    for k in sorted(tot, key=tot.get, reverse=True):
        print(f"{k[:60]:60s} launches={cnt[k]:4d} total_us={tot[k]:10.1f} avg_us={tot[k]/cnt[k]:9.1f} share={tot[k]/s:6.3f}")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
