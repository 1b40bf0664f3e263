"""One-line summaries of bench JSON lines (gpurun_out/bench_*.json)."""
import glob
import json
import sys

for f in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bench_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e)
        continue
    r = d.get("roofline", {})
    km = d.get("kernel_ms", {})
    steps = d.get("steps", 1)
    print(f.split("/")[-1], f"{d['value']:.2f} {d['unit']}", f"e2e {d['e2e']['value']:.2f}",
          f"ms/step {d['ms_per_step']:.3f}", "dom", r.get("kernel"),
          "frac", r.get("frac") and round(r["frac"], 3),
          "stage_frac", round(d.get("stage_roofline", {}).get("frac_of_hbm", 0), 3),
          "clk", d.get("clocks", {}).get("sm_mhz"), d.get("clocks", {}).get("reasons"),
          {k: round(1e3 * v / steps / 4, 1) for k, v in km.items()}, "us/stage")
