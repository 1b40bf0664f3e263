"""Probe: advance a config on the GPU and report the first step where the state
goes non-finite / non-physical (diagnostics for stability of the dt choices)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2105_08632_b200.build import build
build()
from paper_2105_08632_b200 import sdrt
from paper_2105_08632_b200.solver import Solver
from sdrt_inputs import CONFIGS, initial_state
from dataclasses import replace
name = sys.argv[1]; nsteps = int(sys.argv[2]); scale = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
cfg = CONFIGS[name]
S = Solver(cfg.etype, cfg.p, cfg.N, cfg.lo, cfg.hi, cfg.eq, **cfg.physics_kwargs())
U = S.to_device(initial_state(cfg, S.sol_coords()))
K = S.K
for step in range(nsteps):
    try:
        S.rk_step(U, cfg.dt * scale, 1, check_every=1)
    except sdrt.SdrtError as e:
        print(name, 'dt x', scale, 'failed at step', step + 1, e, flush=True)
        break
    if step % 10 == 0 or step == nsteps - 1:
        u = U[:, :, :K]
        print(name, 'step', step + 1, 'max|U| per var', [float(u[:, a].abs().max()) for a in range(u.shape[1])], flush=True)
