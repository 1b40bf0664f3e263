"""Prisms on the GPU (NEXT row N3; App. A l.2633-2737): the generic operator
path (k_apply products + pointwise kernels) on triangular-prism meshes (N_p = 2 per
hexahedron), against the oracle's prism residual (pinned: Tables A.3/A.4 counts, RT
divergence exactness, free stream, conservation, spatial stability, the
definition-form twin; tests/test_oracle_*.py).  Tolerance as every parity test (O25)."""
from dataclasses import replace

import numpy as np
import pytest

from sdrt_inputs import CONFIGS, initial_state, random_state

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-11


def _rel(a, b):
    nv = a.shape[1]
    groups = [[0]] if nv == 1 else [[0], list(range(1, nv - 1)), [nv - 1]]
    return max(float(np.abs(a[:, g] - b[:, g]).max() / max(np.abs(b[:, g]).max(), 1e-300)) for g in groups)


@pytest.mark.parametrize("base,p,N,steps", [("c4", 3, (3, 3, 4), 3), ("c4", 2, (4, 3, 3), 3), ("c3", 2, (3, 4, 3), 3),
                                            ("c3", 1, (3, 3, 3), 5)])
def test_prism_parity(base, p, N, steps):
    from oracle.mesh import build_mesh
    from oracle.physics import Physics
    from oracle.residual import Residual, integrate
    from paper_2105_08632_b200.solver import Solver
    cfg = replace(CONFIGS[base], etype="pri", p=p)
    m = build_mesh("pri", p, N, cfg.lo, cfg.hi)
    R = Residual(m, Physics(cfg.eq, 3, **cfg.physics_kwargs()))
    S = Solver("pri", p, list(N), cfg.lo, cfg.hi, cfg.eq, device="cuda", **cfg.physics_kwargs())
    U = random_state(cfg, R.ops.nsol, m.K, seed=9, amp=0.3)
    assert _rel(S.to_host(S.residual(S.to_device(U))), R(U)) <= TOL
    U0 = initial_state(cfg, m.sol_coords())
    ref = integrate(R, U0, cfg.dt, steps)
    Ud = S.to_device(U0)
    S.rk_step(Ud, cfg.dt, steps)
    assert _rel(S.to_host(Ud), ref) <= TOL
    assert S.last_launches() > 0
