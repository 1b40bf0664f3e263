#!/usr/bin/env python
"""SDRT residual / RK4 throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl sdrt|reference]

A "step" is one classical-RK4 step (4 residual stages, every §8(a) row) of the
configuration's full mesh.  value = N_sol * N_V * K_elems * 4 * steps (summed over
ranks) / max-over-ranks device time / 1e9  [GDOF-stage/s]  (1/PM of PAPER.md
Eq. performance_per_iter_measure l.2942-2951 with N_RK = 4).

N > 1 (one rank per GPU; `--gpus N` without torchrun re-launches itself under
torch.distributed.run): weak scaling with the element-partitioned path
(paper_2105_08632_b200.dist): the global periodic mesh is the configuration's mesh
repeated pgrid times along the slow axes (3-D 2: 1x1x2, 4: 1x2x2, 8: 1x2x4; same h, so
each rank owns exactly the configuration's block) and face traces cross rank boundaries
through the library's own NCCL halo exchange (sdrt_ctx_attach_comm) every stage,
overlapped with the interior tiles.  --impl reference times the CPU oracle (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from dataclasses import replace

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from sdrt_inputs import CONFIGS, initial_state  # noqa: E402

METRIC = "SDRT residual GDOF-stage/s (fp64) and % of HBM roofline at 1/2/4/8 B200"  # BASELINE.json
# reference-arm sample size (patterns per axis) so K steps of the oracle take ~1 s each
REF_SUBBOX = {"c1": 8, "c2": 40, "c3": 6, "c4": 8, "c5": 4, "c4pri": 6}
UNIT = "GDOF-stage/s"
# ncu SASS fp64 counts of the tensor kernels at the current code (tools/sass_counts.py)
SASS_COUNTS = "r02_sass_counts.json"
WORKLOADS = {
    "c1": "c1: 2D linear advection, quad p=2, 8^2 periodic",
    "c2": "c2: 2D isentropic Euler vortex, tri p=3, 40^2x2",
    "c3": "c3: 3D linear advection-diffusion, hex p=4, 24^3",
    "c4": "c4: 3D Taylor-Green vortex NS, hex p=3, 32^3 (Re=1600, Ma=0.1)",
    "c5": "c5: 3D Taylor-Green vortex NS, tet p=3, 48^3x6",
    "c4pri": "c4 on prisms (NEXT row N3): TGV NS, prism p=3, 32^3x2, generic operator path",
}


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def dims(cfg):
    D = cfg.nd
    p = cfg.p
    if cfg.etype == "quad":
        ns, ne, nu = (p + 1) ** 2, 4 * (p + 1), 2 * p * (p + 1)
    elif cfg.etype == "hex":
        ns, ne, nu = (p + 1) ** 3, 6 * (p + 1) ** 2, 3 * p * (p + 1) ** 2
    elif cfg.etype == "tri":
        ns, ne, nu = (p + 1) * (p + 2) // 2, 3 * (p + 1), p * (p + 1) // 2
    elif cfg.etype == "pri":  # Tables A.3/A.4
        ns, ne, nu = (p + 1) ** 2 * (p + 2) // 2, (p + 1) * (4 * p + 5), p * (p + 1) * (2 * p + 3) // 2
    else:
        ns, ne, nu = (p + 1) * (p + 2) * (p + 3) // 6, 2 * (p + 1) * (p + 2), p * (p + 1) * (p + 2) // 6
    return D, ns, ne, nu


def osf(cfg):
    """One-sided flux publication: NS with beta = +1/2 on a mesh without
    far-field axes (the library's rule, kernels.cu; SDRT_OSF=0 disables it)."""
    return cfg.eq == "ns" and cfg.beta == 0.5 and os.environ.get("SDRT_OSF", "1") != "0"


def kernel_bytes(cfg, K):
    """Algorithmic bytes per launch of each kernel (each input array read once, each
    output written once; fp64; the R_int hand-over between kernels A and B is design
    overhead, not counted).  tensor_stage(B): stage input + RK registers (3 N_sol rows
    on average over the 4 stages) + neighbour U traces + viscous traces + new traces;
    tensor_grad(A): stage input + U traces + published viscous traces.  One-sided flux
    publication (osf): A reads the stage input and the N_ext/2 right-neighbour traces and
    writes N_ext/2 common fluxes; B reads/writes 3.25 N_sol RK rows on average (the stage
    input only where the RK formula reads it), gathers the common fluxes of its faces
    (tensor: the N_ext/2 x_d = -1 faces, the + faces went into R_int; simplex: all N_ext)
    and writes the N_ext/2 traces kernel A reads."""
    D, ns, ne, nu = dims(cfg)
    V = cfg.nvars
    b = 8 * V * K
    out = {
        "interp_ext(M0)": b * (ns + ne),
        "interp_int(M12)": b * (ns + nu),
        "common_value": b * (2 * ne + ne),
        "gradient(M16|M15P)": b * (ne + nu + D * ns),
        "metric_grad": b * 2 * D * ns,
        "grad_interp_ext(M5)": b * D * (ns + ne),
        "grad_interp_int(M18)": b * D * (ns + nu),
        "int_flux": b * (nu + (D * nu if cfg.eq in ("ns", "linadvdiff") else 0) + D * nu),
        "face_flux": b * (2 * ne + (2 * D * ne if cfg.eq in ("ns", "linadvdiff") else 0) + ne),
        "divergence(M14|M13M19P2)": b * (ne + D * nu + ns),
        "rk_update": b * ns * 4.25,
        # fused tensor path (each array read/written once per launch)
        "tensor_traces": b * (ns + ne),
        "tensor_grad(A)": b * (ns + ne + (ne // 2 if abs(cfg.beta) == 0.5 else ne)),
        "tensor_stage(B)": b * (ns + 3 * ns + ne + (ne if cfg.eq in ("ns", "linadvdiff") else 0) + ne),
    }
    # fused simplex path: the same data flow per element (traces of the neighbours,
    # published viscous traces of the LDG-weighted side, RK registers, new traces)
    out["simplex_traces"] = out["tensor_traces"]
    out["simplex_grad(A)"] = out["tensor_grad(A)"]
    out["simplex_stage(B)"] = out["tensor_stage(B)"]
    if osf(cfg):
        out["tensor_grad(A)"] = out["simplex_grad(A)"] = b * (ns + ne // 2 + ne // 2)
        out["tensor_stage(B)"] = b * (3.25 * ns + ne // 2 + ne // 2)
        out["simplex_stage(B)"] = b * (3.25 * ns + ne + ne // 2)
    # fused RK stage (kernel A + kernel B in one launch, SDRT_FUSE=1): both kernels' arrays
    out["tensor_fused(A+B)"] = out["tensor_grad(A)"] + out["tensor_stage(B)"]
    return out


# FP64 peak for ALU/tensor-bound kernels: 148 SMs x 64 DFMA/clk x 2 flop x 1.965 GHz
# (B200_PROFILING.md unit counts and clocks.max.sm); tools/fp64_peak measured 37.1 TF
# for both DFMA and DMMA (mma.sync m8n8k4 f64) on the pool's B200s.
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12

# pointwise flop counts per point (fp64 operations; div and sqrt count 1): convective
# flux along one direction, viscous flux along one direction, common (Rusanov/upwind)
# flux incl. the LDG combination
def _pointwise(cfg):
    D = cfg.nd
    if cfg.eq in ("linadv", "linadvdiff"):
        return 2 * D, (2 * D if cfg.eq == "linadvdiff" else 0), 2 * D + 4
    fc = 6 * D + 8
    fv = 90 if D == 3 else 50
    return fc, (fv if cfg.eq == "ns" else 0), 2 * fc + 30


def kernel_flops(cfg, K):
    """Algorithmic fp64 flops per launch of each fused kernel: 2 x the structural-nonzero
    MACs of the App. B products the kernel applies (tensor
    elements by their 1D line factors, simplices dense with the M16 face sparsity) plus
    the pointwise physics at the points it evaluates, each face point's common flux
    counted once.  A model, stated in DESIGN.md §5; not a SASS count."""
    D, ns, ne, nu = dims(cfg)
    V = cfg.nvars
    p = cfg.p
    fc, fv, fr = _pointwise(cfg)
    visc = cfg.eq in ("ns", "linadvdiff")
    nsides = 1 if abs(cfg.beta) == 0.5 else 2
    out = {}
    if cfg.etype in ("quad", "hex"):
        n = p + 1
        NL = n ** (D - 1)
        grad = 2 * D * NL * V * (2 * n + p * n + n * (p + 2)) + D * ns * V + 3 * D * NL * 2 * V
        pub = D * NL * nsides * (2 * (1 + D) * V * n + fv)
        intf = D * NL * p * (2 * ((1 + D) * V if visc else V) * n + fc + fv)
        m13 = 2 * D * NL * V * n * p
        a = grad + pub + intf + m13
        b = 2 * 2 * D * NL * V * n + D * NL * fr + 2 * D * NL * V * n * 2 + 4 * ns * V + 2 * 2 * D * NL * V * n
        if not visc:
            b += D * NL * p * (2 * V * n + fc) + m13
        if osf(cfg):  # A: + common flux and its M14 term at the + ends; B: - faces' M14, RK, - traces
            a += D * NL * fr + 2 * D * NL * V * n
            b = 2 * D * NL * V * n + 4 * ns * V + 2 * D * NL * V * n
        out["tensor_grad(A)"] = K * a
        out["tensor_stage(B)"] = K * b
        out["tensor_traces"] = K * 2 * 2 * D * NL * V * n
    else:
        grad = 2 * (ne + nu) * ns * V + 3 * ne * V + 2 * ns * D * (ne / 2 + nu) * V + 2 * ns * V * D * D
        pub = (ne / 2) * (2 * ns * D * V + fv)
        intf = 2 * nu * ns * D * V + nu * D * (fc + fv) + 2 * ns * D * nu * V
        a = grad + pub + intf
        b = 2 * ne * ns * V + (ne / 2) * fr + 2 * ns * ne * V + 4 * ns * V + 2 * ne * ns * V
        if not visc:
            b += 2 * nu * ns * V + nu * D * fc + 2 * ns * D * nu * V
        if osf(cfg):  # A: + the common flux at the left faces; B: M14, RK, right-face traces
            a += (ne / 2) * fr
            b = 2 * ns * ne * V + 4 * ns * V + ne * ns * V
        out["simplex_grad(A)"] = K * a
        out["simplex_stage(B)"] = K * b
        out["simplex_traces"] = K * 2 * ne * ns * V
    return out


def stage_model_bytes(cfg):
    """SURVEY.md §8(d) algorithmic bytes per DOF-stage (element-local data flow)."""
    D, ns, ne, nu = dims(cfg)
    V = cfg.nvars
    b = 4 * ns * V + 2 * ne * V
    if cfg.eq in ("ns", "linadvdiff"):
        ndq = D if cfg.eq == "ns" else 1
        X = ndq * ne * V * (1 if abs(cfg.beta) == 0.5 else 2)
        b += ne * V + X
    return 8.0 * b / (ns * V)


class ClockSampler:
    def __init__(self, gpu_index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = [l.strip().split(",") for l in open(self.f.name) if l.strip()]
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            if len(r) < 9:
                continue
            for k, nm in enumerate(names):
                if "Active" in r[5 + k] and "Not" not in r[5 + k]:
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def threads_used():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max([i.get("num_threads", 1) for i in info] + [1])
    except Exception:
        return os.cpu_count() or 1


def oracle_stage_rate(cfg, nstages, warm=0, N=None):
    """Time the CPU oracle: nstages residual evaluations + RK axpys on the full mesh,
    or on an N^D-pattern periodic sub-box with the same h (bounded sample)."""
    from oracle.mesh import build_mesh
    from oracle.physics import Physics
    from oracle.residual import Residual
    if N is not None and N < cfg.N:
        hi = tuple(l + (h - l) * N / cfg.N for l, h in zip(cfg.lo, cfg.hi))
        cfg = replace(cfg, N=N, hi=hi)
    m = build_mesh(cfg.etype, cfg.p, cfg.N, cfg.lo, cfg.hi)
    R = Residual(m, Physics(cfg.eq, cfg.nd, **cfg.physics_kwargs()))
    U = initial_state(cfg, m.sol_coords())
    dof = U.size
    for _ in range(warm):
        U = U + 0.0 * R(U)
    t0 = time.perf_counter()
    u = U
    for s in range(nstages):
        k = R(u)
        u = U + (0.5 * cfg.dt) * k
    t = time.perf_counter() - t0
    return dof * nstages / t / 1e9, t, dof


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    nsub = min(cfg.N, REF_SUBBOX.get(cfg.name, cfg.N))
    val, t, dof = oracle_stage_rate(cfg, args.steps, warm=args.warmup, N=nsub)
    cores = threads_used()
    sample = (f"each step = 1 RK stage (residual + RK axpy) of the {cfg.name} workload on a "
              f"{nsub}^{cfg.nd}-pattern periodic sub-box with the same h, p and physics ({dof} DOF); "
              f"{args.warmup} untimed stages first")
    out = {"metric": METRIC, "value": val, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": WORKLOADS[cfg.name], "elements": cfg.K,
                                           "dof": dof, "device": "host cpu"},
           "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


def relaunch(n):
    """`python bench.py --gpus N` outside torchrun: run the same command as N ranks of one
    node (torch.distributed.run, rendezvous on 127.0.0.1); rank 0 prints the JSON line."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="sdrt", choices=["sdrt", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=0,
                    help="e2e through Solver.host_steps with the copies in N overlapped pieces (0: whole-state "
                         "copies on the compute stream; measured on c4: 9.76 at 8 pieces vs 9.49 serial, c3 "
                         "slower from the per-piece launch overhead)")
    ap.add_argument("--scheme", default="sdrt", choices=["sdrt", "frsdrt", "frdg"],
                    help="sdrt: the path; frsdrt/frdg: flux reconstruction on the same kernels (tensor "
                         "elements; the paper's SDRT-vs-FR-DG cost comparison, Table perfo_tgv)")
    ap.add_argument("--integrator", default="rk4", choices=["rk4", "rk54"],
                    help="rk4: classical (BASELINE.json configs); rk54: the paper's PM protocol (N_RK = 5)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args.gpus)
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2105_08632_b200.build import build
    if rank == 0:
        build()
    if world > 1:
        dist.barrier()
    from paper_2105_08632_b200.solver import Solver

    if world > 1:
        from paper_2105_08632_b200.dist import DistSolver, default_pgrid
        pgrid = default_pgrid(world, cfg.nd)
        Ng = [cfg.N * g for g in pgrid]
        hi = [l + (h - l) * g for l, h, g in zip(cfg.lo, cfg.hi, pgrid)]
        S = DistSolver(cfg.etype, cfg.p, Ng, cfg.lo, hi, cfg.eq, device=dev, pgrid=pgrid, scheme=args.scheme,
                       **cfg.physics_kwargs())
        parallelism = (f"element partition {'x'.join(map(str, pgrid))} over {world} GPUs, halo exchange "
                       f"inside libsdrt over NCCL ({S.transport}), overlapped with interior tiles")
    else:
        S = Solver(cfg.etype, cfg.p, cfg.N, cfg.lo, cfg.hi, cfg.eq, device=dev, scheme=args.scheme,
                   **cfg.physics_kwargs())
        parallelism = "single"
    U0 = initial_state(cfg, S.sol_coords())
    U = S.to_device(U0)
    nsol, nv, Kp = S.shape
    K = S.K
    dof = nsol * nv * K
    stream = torch.cuda.current_stream(dev)

    def finite_now():
        torch.cuda.synchronize(dev)
        return bool(torch.isfinite(U[:, :, :K]).all().item())

    # ---------------------------------------------------------------- warm-up
    NST = 4 if args.integrator == "rk4" else 5  # stages per step

    def step_fn(solver):
        return solver.rk_step if args.integrator == "rk4" else solver.rk54_step

    step_fn(S)(U, cfg.dt, args.warmup)
    torch.cuda.synchronize(dev)
    dbg = {"after_warmup": finite_now()}
    clocks = ClockSampler(local)
    time.sleep(0.3)

    # ---------------------------------------------------------------- per-kernel pass
    # K steps with CUDA events around every kernel (sdrt_ctx_set_timing): the per-kernel
    # device times for the roofline; instrumentation, not the reported rate
    S.set_timing(True)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    step_fn(S)(U, cfg.dt, args.steps)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms_inst = e0.elapsed_time(e1)
    ktimes = S.kernel_times()
    S.set_timing(False)

    # CUDA-graph replay of the K-step call (sdrt_ctx_set_graph; off by default, measured
    # slower than the direct PDL launches): when enabled (SDRT_BENCH_GRAPH=1) the graph of
    # this K is captured here, outside the timed region
    graphs = os.environ.get("SDRT_BENCH_GRAPH") == "1"
    if graphs:
        S.set_graph(1)
        step_fn(S)(U, cfg.dt, args.steps)
        step_fn(S)(U, cfg.dt, 1)
        torch.cuda.synchronize(dev)

    # ---------------------------------------------------------------- timed region
    # K steps bracketed by a barrier + synchronize on both sides, CUDA events on the
    # launching stream, max over ranks
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # one library call for the K steps (as a K-step run is made): the stage-input traces
    # are formed once, then every stage's kernel B publishes the next ones
    e2.record(stream)
    step_fn(S)(U, cfg.dt, args.steps)
    launches = S.last_launches()  # host-side count of our kernels in the call
    e3.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms = e2.elapsed_time(e3)
    clk = clocks.stop()
    dbg["after_timed"] = finite_now()
    finite = dbg["after_timed"]

    t = torch.tensor([ms, ms_inst], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, ms_inst_max = float(t[0]), float(t[1])
    ms_clean_max = ms_max
    total_dof_stages = dof * NST * args.steps * world
    value = total_dof_stages / (ms_max * 1e-3) / 1e9

    # ---------------------------------------------------------------- e2e (host buffers)
    # A dependent trajectory through the public API with the state in host memory: every
    # step copies the state host->device from pinned memory, runs sdrt_rk_step (one step)
    # and copies the new state device->host into the same pinned buffer, which is the next
    # step's input.  Default: whole-state copies on the compute stream.  --e2e-chunks N:
    # Solver.host_steps, the copies in N pieces on two copy streams, piece k of step i+1's
    # upload ordered after piece k of step i's download by an event, the compute of step
    # i+1 after the whole upload -- measured no faster (c4 9.76 vs 9.49: the two PCIe
    # directions together do not exceed one direction's ~54 GB/s on this host).
    pin = torch.empty(S.shape, dtype=torch.float64).pin_memory()
    pin.copy_(U.cpu())
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    if not args.e2e_chunks:
        for i in range(args.steps):
            U.copy_(pin, non_blocking=True)
            step_fn(S)(U, cfg.dt, 1)
            pin.copy_(U, non_blocking=True)
    else:
        S.host_steps(pin, U, cfg.dt, args.steps, rk54=args.integrator == "rk54", chunks=args.e2e_chunks)
    a1.record(stream)
    torch.cuda.synchronize(dev)
    te = torch.tensor([a0.elapsed_time(a1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_val = total_dof_stages / (float(te[0]) * 1e-3) / 1e9
    e2e_ok = bool(torch.isfinite(pin[:, :, :K]).all())
    state_bytes = U.numel() * 8

    # ---------------------------------------------------------------- e2e, monitored run
    # The paper's own TGV workflow (l.2052-2080): the state stays resident and every step
    # the host reads back the monitored quantities <E*>, eps2, eps3 (sdrt_diagnostics with
    # the degree-10 quadrature, 24 bytes D2H, a synchronising read per step).  Reported
    # beside the state-through-host trajectory above, not instead of it.
    mon = None
    if cfg.eq == "ns" and cfg.nd == 3 and cfg.etype in ("hex", "tet") and world == 1:  # fused paths
        U.copy_(pin, non_blocking=True)
        torch.cuda.synchronize(dev)
        m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        m0.record(stream)
        last = None
        for i in range(args.steps):
            step_fn(S)(U, cfg.dt, 1)
            last = S.diagnostics(U)  # D2H of the step's monitored result
        m1.record(stream)
        torch.cuda.synchronize(dev)
        mon = {"value": total_dof_stages / (m0.elapsed_time(m1) * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 24,
               "result": [float(x) for x in last] if last is not None else None,
               "pipeline": "state resident; per step one RK step + sdrt_diagnostics (degree-10 <E*>, eps2, "
                           "eps3) read back to the host (the paper's TGV monitoring)"}

    # ---------------------------------------------------------------- roofline
    peaks = load_peaks()
    hbm = peaks.get("hbm_gbs")
    peak_note = "MEASURED_PEAKS.json hbm_gbs" if hbm else "fallback 6650 GB/s (B200_PROFILING.md)"
    hbm = hbm or 6650.0
    kb = kernel_bytes(cfg, K)
    dom, dom_ms, dom_n = None, -1.0, 0
    for nm, (tms, cnt) in ktimes.items():
        if tms > dom_ms:
            dom, dom_ms, dom_n = nm, tms, cnt
    traffic = None
    tf = os.path.join(ROOT, "profiles", f"traffic_{cfg.name}.json")
    if os.path.exists(tf):
        traffic = json.load(open(tf)).get(dom)
    kf = kernel_flops(cfg, K)
    flops_source = "model (bench.kernel_flops)"
    sc = os.path.join(ROOT, "profiles", SASS_COUNTS)
    if os.path.exists(sc) and world == 1:
        # executed fp64 flops of the tensor kernels from ncu SASS counts (2 DFMA + DMUL +
        # DADD per launch, profiles/SASS_COUNTS) replace the model
        sass = json.load(open(sc)).get(cfg.name, {})
        for kn, v in sass.items():
            if kn.startswith("tensor_") and kn in kf:
                kf[kn] = v["flops_per_launch"]
                flops_source = f"ncu SASS counts (profiles/{SASS_COUNTS}) for the tensor kernels"
    if "tensor_grad(A)" in kf and "tensor_stage(B)" in kf:  # the fused launch runs both kernels' work
        kf["tensor_fused(A+B)"] = kf["tensor_grad(A)"] + kf["tensor_stage(B)"]
    t_launch = dom_ms / dom_n * 1e-3 if dom else None
    gbs = kb[dom] / t_launch / 1e9 if dom in kb else None
    tfs = kf[dom] / t_launch / 1e12 if dom in kf else None
    f_hbm = gbs / hbm if gbs else 0.0
    f_alu = tfs / FP64_PEAK_TFLOPS if tfs else 0.0
    # the dominant kernel's binding resource: the larger of its HBM and FP64 fractions
    if f_alu > f_hbm:
        roof = {"bound": "alu", "kernel": dom, "achieved": tfs, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": f_alu, "traffic": traffic,
                "peak_source": "148 SMs x 64 DFMA/clk x 2 x 1.965 GHz (B200_PROFILING.md units and clocks); "
                               "tools/fp64_peak measured 37.1 TF (DFMA and DMMA)"}
    else:
        roof = {"bound": "hbm", "kernel": dom, "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": f_hbm,
                "traffic": traffic, "peak_source": peak_note}
    roof.update({"bytes_per_launch": kb.get(dom), "flops_per_launch": kf.get(dom), "flops_source": flops_source,
                 "hbm_frac": f_hbm, "fp64_frac": f_alu,
                 "avg_launch_ms": dom_ms / dom_n if dom else None,
                 "launches_per_step": dom_n / args.steps if dom else None,
                 "step_share": dom_ms / ms if dom else None})
    model_b = stage_model_bytes(cfg)
    stage_roof = {"model_bytes_per_dof_stage": model_b,
                  "achieved_gbs": model_b * dof * NST * args.steps / (ms_clean_max * 1e-3) / 1e9,
                  "frac_of_hbm": model_b * dof * NST * args.steps / (ms_clean_max * 1e-3) / 1e9 / hbm,
                  "ceiling_gdof_stage_s": hbm / model_b}

    # ---------------------------------------------------------------- cpu baseline
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, tt, _ = oracle_stage_rate(cfg, 1)
            cpu = {"value": v, "unit": UNIT, "cores": threads_used(), "kind": "oracle",
                   "sample": f"1 RK stage (residual + RK axpy) of the full {cfg.name} mesh, "
                             f"{tt:.1f} s of CPU time"}
        except Exception as ex:  # report, do not fail the bench
            cpu = {"value": None, "unit": UNIT, "cores": threads_used(), "kind": "oracle",
                   "sample": f"failed: {ex!r}"}

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "config": {"workload": WORKLOADS[cfg.name], "elements_per_gpu": K, "dof_per_gpu": dof,
                          "p": cfg.p, "dt": cfg.dt, "parallelism": parallelism,
                          "integrator": "classical RK4 (4 stages)" if NST == 4 else "RK54 (5 stages, 2 registers)",
                          "launch": "one CUDA graph per K-step call (replayed)" if graphs else
                                    "direct launches with programmatic dependent launch",
                          "scheme": args.scheme,
                          "l2": "working set > L2 (state 3 registers + traces >> 126 MB); no flush needed"
                          if dof * 8 * 3 > 126e6 else "working set fits L2 (small config)"},
               "roofline": roof, "stage_roofline": stage_roof, "cpu_baseline": cpu,
               "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": state_bytes,
                       "d2h_bytes_per_step": state_bytes, "result_finite": e2e_ok,
                       "pipeline": ("dependent trajectory: per step H2D state (pinned) -> sdrt_rk_step -> D2H "
                                    "state, the next step reads the host copy; serialized on one stream")
                       if not args.e2e_chunks else
                       ("dependent trajectory (Solver.host_steps): per step H2D state (pinned) -> one RK step "
                        "-> D2H state into the same host buffer, which the next step reads; copies in pieces "
                        "on two copy streams, piece k of step i+1's H2D after piece k of step i's D2H (the two "
                        "PCIe directions overlap), the step's compute after the whole H2D")},
               "e2e_monitor": mon,
               "gpu_launches": launches, "clocks": clk, "kernel_ms": {k: v[0] for k, v in ktimes.items()},
               "ms_per_step_instrumented": ms_inst_max / args.steps, "state_finite": finite,
               "finite_trace": dbg}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
