"""Far-field boundaries on the GPU (NEXT row N4; the paper's vortex
takes "the limiting values of the initial conditions" at the constant-x boundaries,
periodic in y): sdrt_mesh_create(periodic[0] = 0) + sdrt_ctx_set_farfield against the
oracle's far-field residual (pinned by the definition-form twin and free-stream
preservation, tests/test_oracle_twin.py).  Tolerance as every parity test (O25)."""
import math

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


def _farfield(cfg):
    """Free stream of the configuration (the IC's limit far from the structures)."""
    if cfg.nvars == 1:
        return np.zeros(1)
    D = cfg.nd
    if cfg.ic == "vortex":
        rho, v, p = 1.0, [0.5 * math.sqrt(cfg.gamma), 0.0], 1.0
    else:  # TGV units (reading O18): rho_inf = 1, v = 0, p_inf = 1 / (gamma Ma^2)
        rho, v, p = 1.0, [0.0] * D, 1.0 / (cfg.gamma * 0.1 ** 2)
    return np.array([rho] + [rho * x for x in v] + [p / (cfg.gamma - 1) + 0.5 * rho * sum(x * x for x in v)])


def _pair(cfg, N, **kw):
    from oracle.mesh import build_mesh
    from oracle.physics import Physics
    from oracle.residual import Residual
    from paper_2105_08632_b200.solver import Solver
    D = cfg.nd
    per = (False,) + (True,) * (D - 1)
    ff = _farfield(cfg)
    m = build_mesh(cfg.etype, cfg.p, tuple(N), cfg.lo, cfg.hi, periodic=per)
    R = Residual(m, Physics(cfg.eq, D, **cfg.physics_kwargs()), farfield=ff)
    S = Solver(cfg.etype, cfg.p, list(N), cfg.lo, cfg.hi, cfg.eq, device="cuda", periodic=per, farfield=ff,
               **kw, **cfg.physics_kwargs())
    return m, R, S


@pytest.mark.parametrize("name,N,steps", [("c1", [6, 4], 20), ("c2", [8, 6], 20), ("c3", [3, 3, 4], 3),
                                          ("c4", [4, 3, 3], 3), ("c5", [3, 3, 3], 2)])
def test_farfield_parity(name, N, steps):
    from oracle.residual import integrate
    cfg = CONFIGS[name]
    m, R, S = _pair(cfg, N)
    U = random_state(cfg, R.ops.nsol, m.K, seed=3, amp=0.2)
    assert _rel(S.to_host(S.residual(S.to_device(U))), R(U)) <= TOL
    U0 = initial_state(cfg, m.sol_coords())
    ref = integrate(R, U0, cfg.dt, steps)
    Ud = S.to_device(U0)
    S.rk_step(Ud, cfg.dt, steps)
    assert _rel(S.to_host(Ud), ref) <= TOL


def test_farfield_vortex_full_size():
    """The c2 vortex on its full 40 x 40 x 2 mesh with far-field x boundaries (the paper's
    own arrangement, l.1952), 200 RK4 steps element-wise against the oracle."""
    from oracle.residual import integrate
    cfg = CONFIGS["c2"]
    m, R, S = _pair(cfg, [cfg.N, cfg.N])
    U0 = initial_state(cfg, m.sol_coords())
    ref = integrate(R, U0, cfg.dt, 200)
    Ud = S.to_device(U0)
    S.rk_step(Ud, cfg.dt, 200)
    assert _rel(S.to_host(Ud), ref) <= TOL


def test_farfield_requires_state_and_library_exchange():
    """sdrt_rk_step refuses a far-field context before sdrt_ctx_set_farfield; with the
    periodic axes routed through the library's NCCL halo (one-rank communicator) the
    far-field run is bitwise the plain one."""
    from paper_2105_08632_b200 import sdrt
    from paper_2105_08632_b200.dist import DistSolver
    from paper_2105_08632_b200.solver import Solver
    cfg = CONFIGS["c4"]
    N = [6, 4, 4]
    per = (False, True, True)
    S0 = Solver(cfg.etype, cfg.p, N, cfg.lo, cfg.hi, cfg.eq, periodic=per, **cfg.physics_kwargs())
    U = S0.to_device(initial_state(cfg, S0.sol_coords()))
    with pytest.raises(sdrt.SdrtError) as e:
        S0.rk_step(U, cfg.dt, 1)
    assert e.value.code == -1
    ff = _farfield(cfg)
    sdrt.ctx_set_farfield(S0.ctx, ff, torch.cuda.current_stream().cuda_stream)
    S1 = DistSolver(cfg.etype, cfg.p, N, cfg.lo, cfg.hi, cfg.eq, device="cuda", force_self_halo=True,
                    transport="library", periodic=per, farfield=ff, **cfg.physics_kwargs())
    U1 = S1.to_device(initial_state(cfg, S1.sol_coords()))
    S0.rk_step(U, cfg.dt, 3)
    S1.rk_step(U1, cfg.dt, 3)
    assert np.array_equal(S0.to_host(U), S1.to_host(U1))
