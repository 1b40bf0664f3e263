import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_08632_b200.build import build
build()
from paper_2105_08632_b200.solver import Solver
from sdrt_inputs import CONFIGS, initial_state
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
def run(mode, n=40):
    S = Solver(cfg.etype, cfg.p, cfg.N, cfg.lo, cfg.hi, cfg.eq, **cfg.physics_kwargs())
    U = S.to_device(initial_state(cfg, S.sol_coords()))
    K = S.K
    if mode == "timing":
        S.set_timing(True)
    first_bad = None
    for i in range(n):
        S.rk_step(U, cfg.dt, 1)
        if mode == "sync":
            torch.cuda.synchronize()
        if mode in ("sync", "check") and first_bad is None:
            if not torch.isfinite(U[:, :, :K]).all():
                first_bad = i + 1
    torch.cuda.synchronize()
    ok = bool(torch.isfinite(U[:, :, :K]).all())
    if mode == "timing":
        S.kernel_times()
    print(mode, "finite after", n, "steps:", ok, "first bad:", first_bad, flush=True)
    S.close()
for m in ["nosync", "sync", "timing", "check", "nosync"]:
    run(m)
