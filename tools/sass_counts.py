"""Executed fp64 work per launch of the fused kernels from an ncu --metrics CSV log
(tools/gpu_evidence_r2c.sh: smsp__sass_thread_inst_executed_op_{dfma,dmul,dadd}_pred_on,
DMMA instruction count, pipe utilisation, DRAM bytes, duration) -> JSON keyed by the
bench's kernel names:  python tools/sass_counts.py OUT.json c4=sass_c4.csv c5=... """
import csv
import json
import sys


def kname(n):
    for pre, nm in (("kt_grad", "tensor_grad(A)"), ("kt_stage", "tensor_stage(B)"), ("kt_traces", "tensor_traces"),
                    ("ks_grad", "simplex_grad(A)"), ("ks_stage", "simplex_stage(B)"), ("ks_traces", "simplex_traces")):
        if n.split("<")[0].split("::")[-1].startswith(pre) or pre in n.split("(")[0]:
            return nm
    return None


def load(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    h = {k: i for i, k in enumerate(rows[hdr])}
    per = {}
    for r in rows[hdr + 1:]:
        if len(r) != len(rows[hdr]):
            continue
        nm = kname(r[h["Kernel Name"]])
        if nm is None:
            continue
        d = per.setdefault((r[h["ID"]], nm), {})
        try:
            d[r[h["Metric Name"]]] = float(r[h["Metric Value"]].replace(",", ""))
        except ValueError:
            pass
        d["_unit_" + r[h["Metric Name"]]] = r[h["Metric Unit"]]
    out = {}
    for (_, nm), d in per.items():
        fl = 2 * d.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", 0) + \
            d.get("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", 0) + \
            d.get("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", 0)
        dmma = d.get("sm__inst_executed_pipe_tensor_subpipe_dmma.sum", 0)
        t = d.get("gpu__time_duration.sum", 0)
        tu = d.get("_unit_gpu__time_duration.sum", "ns")
        us = t / 1000.0 if tu == "ns" else (t * 1000.0 if tu == "ms" else t)
        def by(m):
            v, u = d.get(m, 0.0), d.get("_unit_" + m, "byte")
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        o = out.setdefault(nm, {"flops_per_launch": 0.0, "dmma_flops_per_launch": 0.0, "us_per_launch_ncu": 0.0,
                                "dram_bytes_per_launch": 0.0, "fp64_pipe_pct": 0.0, "dmma_pipe_pct": 0.0, "launches": 0})
        o["flops_per_launch"] += fl
        o["dmma_flops_per_launch"] += dmma * 512.0
        o["us_per_launch_ncu"] += us
        o["dram_bytes_per_launch"] += by("dram__bytes_read.sum") + by("dram__bytes_write.sum")
        o["fp64_pipe_pct"] += d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0)
        o["dmma_pipe_pct"] += d.get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", 0)
        o["launches"] += 1
    for o in out.values():
        n = o["launches"]
        for k in list(o):
            if k != "launches":
                o[k] /= n
    return out


if __name__ == "__main__":
    res = {"_how": "ncu --metrics gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_{dfma,dadd,dmul}_pred_on.sum,"
                   "sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__pipe_fp64_cycles_active,sm__pipe_tensor_op_dmma_cycles_active,"
                   "dram__bytes_{read,write}.sum --clock-control none -k regex:k[ts]_ -s 6 -c 6 (python bench.py "
                   "--config C --steps 2 --warmup 3); flops = 2 DFMA + DMUL + DADD per launch (fp64 pipe), "
                   "dmma_flops = DMMA instructions x 512 (8x8x4 FMA, zero padding included), averaged over the "
                   "profiled launches of each kernel (kernel B's count depends on the RK stage)"}
    for a in sys.argv[2:]:
        c, path = a.split("=", 1)
        res[c] = load(path)
    json.dump(res, open(sys.argv[1], "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])
