"""Compare the fused tensor path with the generic operator path step by step."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2105_08632_b200.build import build
build()
from paper_2105_08632_b200.solver import Solver
from sdrt_inputs import CONFIGS, initial_state
cfg = CONFIGS[sys.argv[1]]
N = int(sys.argv[2]); nsteps = int(sys.argv[3])
mk = lambda: Solver(cfg.etype, cfg.p, N, cfg.lo, cfg.hi, cfg.eq, **cfg.physics_kwargs())
os.environ["SDRT_FORCE_GENERIC"] = "0"; A = mk()
os.environ["SDRT_FORCE_GENERIC"] = "1"; B = mk()
U0 = initial_state(cfg, A.sol_coords())
UA, UB = A.to_device(U0), B.to_device(U0)
K = A.K
for s in range(1, nsteps + 1):
    A.rk_step(UA, cfg.dt, 1); B.rk_step(UB, cfg.dt, 1)
    a, b = UA[:, :, :K], UB[:, :, :K]
    fa, fb = bool(torch.isfinite(a).all()), bool(torch.isfinite(b).all())
    d = (a - b).abs()
    rel = [float(d[:, v].max() / b[:, v].abs().max()) for v in range(a.shape[1])]
    if s % 4 == 0 or not fa or not fb:
        bad = torch.nonzero(~torch.isfinite(a).all(dim=0).all(dim=0)).flatten()[:10].tolist()
        print(s, 'finite', fa, fb, 'rel', ['%.1e' % r for r in rel], 'bad elems', bad, flush=True)
    if not fa and not fb: break
