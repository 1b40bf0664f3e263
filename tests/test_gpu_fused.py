"""GPU: the fused RK stage (kernel A + kernel B of one stage in ONE persistent launch,
tensor.cu kt_fused; SDRT_FUSE=1 at context creation) against the two-kernel stage and the
oracle.

The fused launch runs exactly the two kernels' per-element arithmetic, only in another
order (a job list with per-tile dependency flags), so its RK steps must be BITWISE the
two-kernel ones, and within the parity tolerance of the oracle (PAPER.md l.312-340 for the
face fluxes, l.2919-2932 for the divergence, the RK4 / RK54 updates of l.1110-1126).
Meshes: tile-aligned rows (the c4 layout), ragged rows whose tiles straddle x-rows, a
partial last tile, and the full c4 mesh (32^3)."""
import os

import numpy as np
import pytest

from sdrt_inputs import CONFIGS, random_state

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-11


def _rel(a, b):
    nv = a.shape[1]
    out = 0.0
    for g in ([[0]] if nv == 1 else [[0], list(range(1, nv - 1)), [nv - 1]]):
        out = max(out, float(np.abs(a[:, g] - b[:, g]).max() / max(np.abs(b[:, g]).max(), 1e-300)))
    return out


def _solver(cfg, N, fuse, lag=None):
    from paper_2105_08632_b200.solver import Solver
    keys = {"SDRT_FUSE": "1" if fuse else "0"}
    if lag is not None:
        keys["SDRT_FUSE_LAG"] = str(lag)
    old = {k: os.environ.get(k) for k in keys}
    os.environ.update(keys)
    try:
        return Solver(cfg.etype, cfg.p, list(N), cfg.lo, cfg.hi, cfg.eq, device="cuda", **cfg.physics_kwargs())
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


def _is_fused(S, U, dt):
    """the context runs the fused launch (its timing tag appears, the two kernels' do not)"""
    S.set_timing(True)
    Ud = S.to_device(U)
    S.rk_step(Ud, dt, 1)
    torch.cuda.synchronize()
    kt = S.kernel_times()
    S.set_timing(False)
    return "tensor_fused(A+B)" in kt and "tensor_grad(A)" not in kt


@pytest.mark.parametrize("N,lag", [((16, 4, 4), None), ((16, 4, 4), 0), ((8, 8, 8), 3), ((12, 5, 3), None),
                                   ((8, 4, 3), 1)])
def test_fused_stage_bitwise_two_kernel_and_oracle(N, lag):
    from oracle.mesh import build_mesh
    from oracle.physics import Physics
    from oracle.residual import Residual, integrate
    cfg = CONFIGS["c4"]
    m = build_mesh(cfg.etype, cfg.p, N, cfg.lo, cfg.hi)
    R = Residual(m, Physics(cfg.eq, cfg.nd, **cfg.physics_kwargs()))
    U = random_state(cfg, R.ops.nsol, m.K, seed=5, amp=0.3)
    steps = 3
    ref = integrate(R, U, cfg.dt, steps)
    out = {}
    for fuse in (True, False):
        S = _solver(cfg, N, fuse, lag)
        assert _is_fused(S, U, cfg.dt) == fuse, (N, fuse)
        Ud = S.to_device(U)
        S.rk_step(Ud, cfg.dt, steps)
        out[fuse] = S.to_host(Ud)
        Ud = S.to_device(U)
        S.rk54_step(Ud, cfg.dt, 2)
        out[(fuse, 54)] = S.to_host(Ud)
        torch.cuda.synchronize()
        S.close()
    assert np.array_equal(out[True], out[False]), np.abs(out[True] - out[False]).max()
    assert np.array_equal(out[(True, 54)], out[(False, 54)])
    assert _rel(out[True], ref) <= TOL, _rel(out[True], ref)


def test_fused_stage_full_c4_bitwise():
    """the bench configuration (32^3 hex p = 3 NS TGV, 4096 tiles on the persistent grid):
    20 RK4 steps fused == two-kernel, bit for bit, and repeated calls (the launch epoch and
    job counter reset by the last CTA) stay bitwise"""
    from sdrt_inputs import initial_state
    cfg = CONFIGS["c4"]
    res = {}
    for fuse in (True, False):
        S = _solver(cfg, (cfg.N,) * 3, fuse)
        U0 = initial_state(cfg, S.sol_coords())
        assert _is_fused(S, U0, cfg.dt) == fuse
        Ud = S.to_device(U0)
        for _ in range(4):
            S.rk_step(Ud, cfg.dt, 5)
        res[fuse] = S.to_host(Ud)
        torch.cuda.synchronize()
        S.close()
    assert np.isfinite(res[True]).all()
    assert np.array_equal(res[True], res[False]), np.abs(res[True] - res[False]).max()
