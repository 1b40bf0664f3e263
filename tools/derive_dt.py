"""Derive the c2 time-step literal (sdrt_inputs.configs.C2_DT) using only oracle/.

dt = CFL * h / lambda_max with CFL = 0.1, h = 0.25 (pattern edge, tau definition
PAPER.md l.889/497) and lambda_max = max over initial solution points of |v| + a.
"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.mesh import build_mesh  # noqa: E402
from sdrt_inputs import CONFIGS, initial_state  # noqa: E402

cfg = CONFIGS["c2"]
m = build_mesh(cfg.etype, cfg.p, cfg.N, cfg.lo, cfg.hi)
U = initial_state(cfg, m.sol_coords())
rho = U[:, 0]
v = U[:, 1:3] / rho[:, None]
p = (cfg.gamma - 1) * (U[:, 3] - 0.5 * rho * (v ** 2).sum(1))
lam = np.sqrt((v ** 2).sum(1)) + np.sqrt(cfg.gamma * p / rho)
print(repr(0.1 * 0.25 / lam.max()), lam.max())
