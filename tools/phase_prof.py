"""Per-phase cycle split of the fused tensor kernels (profiling build libsdrt_prof.so,
SDRT_PHASE_PROF=1).  Runs a few RK4 steps of a config and prints, per kernel, the
share of CTA time spent in each phase (thread 0's clock64 between barriers)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("SDRT_LIB", os.path.join(ROOT, "paper_2105_08632_b200", "libsdrt_prof.so"))
import torch  # noqa: E402
from paper_2105_08632_b200 import sdrt  # noqa: E402
from paper_2105_08632_b200.solver import Solver  # noqa: E402
from sdrt_inputs import CONFIGS, initial_state  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = CONFIGS[name]
S = Solver(cfg.etype, cfg.p, cfg.N, cfg.lo, cfg.hi, cfg.eq, device="cuda", **cfg.physics_kwargs())
U = S.to_device(initial_state(cfg, S.sol_coords()))
S.rk_step(U, cfg.dt, 2)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 32)()
simplex = cfg.etype in ("tri", "tet")
f = sdrt.lib.sdrt_debug_sphase_cycles if simplex else sdrt.lib.sdrt_debug_phase_cycles
f(buf, 1)
S.rk_step(U, cfg.dt, 5)
torch.cuda.synchronize()
f(buf, 1)
if simplex:
    names = {0: ["nbrs", "M0,M12", "C", "G", "metric", "M0.Q", "publish", "M12.Q", "int.flux", "M13F", "store"],
             1: ["nbrs", "M0", "faceflux+wait", "M14", "RK", "M0 new", "store"]}
    kn = ["ks_grad (A)", "ks_stage (B)"]
else:
    names = {0: ["nbrs", "tile+nb load", "gradient", "pub+Fv(0)", "div0+Fv(1)", "div1+Fv(2)", "div2"],
             1: ["nbrs", "tile load", "flux (all d)", "div (all d)", "RK+x traces"] + [""] * 10 + ["y/z traces"]}
    kn = ["kt_grad (A)", "kt_stage (B)"]
for k in range(2):
    v = [buf[16 * k + i] for i in range(16)]
    tot = sum(v) or 1
    nm = names[k] + [""] * 16
    print(kn[k], " ".join(f"{nm[i] or i}:{100*v[i]/tot:.1f}%" for i in range(16) if v[i]))
