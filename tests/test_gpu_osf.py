"""GPU: the two forms of the beta = 1/2 Navier-Stokes face flux against the oracle.

With LDG weights (1/2 + beta, 1/2 - beta) = (1, 0) (the TGV settings of c4 and c5, O15) the
library evaluates each face's whole common flux once, in the face's left element, and both
sides apply the stored value (one-sided flux publication); SDRT_OSF=0 at
context creation selects the two-sided form (kernel B evaluates the common flux on both
sides from bit-identical inputs).  Both must match the oracle within
the parity tolerance, agree with each other to round-off, and keep the per-face
conservation bitwise (O28)."""
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


def _solver(cfg, Nt, osf):
    from paper_2105_08632_b200.solver import Solver
    old = os.environ.get("SDRT_OSF")
    os.environ["SDRT_OSF"] = "1" if osf else "0"
    try:
        return Solver(cfg.etype, cfg.p, list(Nt), cfg.lo, cfg.hi, cfg.eq, device="cuda", **cfg.physics_kwargs())
    finally:
        if old is None:
            del os.environ["SDRT_OSF"]
        else:
            os.environ["SDRT_OSF"] = old


@pytest.mark.parametrize("name,N", [("c4", (3, 4, 5)), ("c5", (3, 4, 3))])
def test_one_and_two_sided_flux_match_oracle(name, N):
    from oracle.mesh import build_mesh
    from oracle.physics import Physics
    from oracle.residual import Residual, integrate
    cfg = CONFIGS[name]
    m = build_mesh(cfg.etype, cfg.p, N, cfg.lo, cfg.hi)
    R = Residual(m, Physics(cfg.eq, cfg.nd, **cfg.physics_kwargs()))
    U = random_state(cfg, R.ops.nsol, m.K, seed=11, amp=0.3)
    ref_r = R(U)
    ref_u = integrate(R, U, cfg.dt, 3)
    res = {}
    for osf in (True, False):
        S = _solver(cfg, N, osf)
        r = S.to_host(S.residual(S.to_device(U)))
        Ud = S.to_device(U)
        S.rk_step(Ud, cfg.dt, 3)
        u = S.to_host(Ud)
        torch.cuda.synchronize()
        assert _rel(r, ref_r) <= TOL, (osf, _rel(r, ref_r))
        assert _rel(u, ref_u) <= TOL, (osf, _rel(u, ref_u))
        res[osf] = (r, u)
        S.close()
    assert _rel(res[True][0], res[False][0]) <= 1e-13
    assert _rel(res[True][1], res[False][1]) <= 1e-13


@pytest.mark.parametrize("osf", [True, False])
@pytest.mark.parametrize("name,N", [("c4", (3, 3, 4)), ("c5", (3, 3, 3))])
def test_face_flux_bitwise_both_forms(name, N, osf):
    """O28 under either form: the flux each side applied at every face point is bit-identical
    (one-sided: the same stored number, exported by kernel A on the left and kernel B on the
    right; two-sided: two evaluations from bit-identical inputs) and equals the oracle's
    once-per-face-point common flux."""
    from oracle.mesh import build_mesh
    from oracle.physics import Physics
    from oracle.residual import Residual
    from paper_2105_08632_b200 import sdrt
    cfg = CONFIGS[name]
    S = _solver(cfg, N, osf)
    m = build_mesh(cfg.etype, cfg.p, N, cfg.lo, cfg.hi)
    R = Residual(m, Physics(cfg.eq, cfg.nd, **cfg.physics_kwargs()))
    U = random_state(cfg, R.ops.nsol, m.K, seed=5, amp=0.3)
    dudt, F = S.face_flux(S.to_device(U))
    torch.cuda.synchronize()
    F = F.cpu().numpy()[:, :, :S.K]
    fe, fl, fp, _ = sdrt.mesh_export_maps(S.mesh)
    nfp = R.ops.nfp
    q = np.arange(nfp)
    rows_L = fl[:, 0].astype(np.int64)[:, None] * nfp + q[None, :]
    rows_R = fl[:, 1].astype(np.int64)[:, None] * nfp + fp.astype(np.int64)
    FL = F[rows_L, :, fe[:, 0][:, None]]
    FR = F[rows_R, :, fe[:, 1][:, None]]
    assert np.array_equal(FL.view(np.int64), FR.view(np.int64))
    ref = R.face_common_flux(U)
    got = FL.reshape(-1, FL.shape[2]).T
    for g in ([[0]], [list(range(1, ref.shape[0] - 1))], [[ref.shape[0] - 1]]):
        g = g[0]
        assert np.abs(got[g] - ref[g]).max() <= TOL * np.abs(ref[g]).max()
    assert _rel(S.to_host(dudt), R(U)) <= TOL
    S.close()


def _solver_env(cfg, Nt, env):
    from paper_2105_08632_b200.solver import Solver
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return Solver(cfg.etype, cfg.p, list(Nt), cfg.lo, cfg.hi, cfg.eq, device="cuda", **cfg.physics_kwargs())
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


@pytest.mark.parametrize("N,slabs", [((3, 4, 8), "4"), ((3, 3, 6), "4"), ((4, 3, 9), "8"), ((3, 3, 16), "16")])
@pytest.mark.parametrize("integrator", ["rk4", "rk54"])
def test_slab_pipeline_bitwise(N, slabs, integrator):
    """The slab-pipelined stage schedule (kernel A / kernel B of different z-slabs on two
    streams, per-slab events) gives bitwise the single-stream result: the same kernels
    and per-element arithmetic, only the launch order differs; and it matches the oracle."""
    from oracle.mesh import build_mesh
    from oracle.physics import Physics
    from oracle.residual import Residual, integrate
    cfg = CONFIGS["c4"]
    m = build_mesh(cfg.etype, cfg.p, N, cfg.lo, cfg.hi)
    U0 = random_state(cfg, (cfg.p + 1) ** 3, m.K, seed=3, amp=0.2)
    out = {}
    for sl in (slabs, "0"):
        S = _solver_env(cfg, N, {"SDRT_SLABS": sl, "SDRT_OSF": "1"})
        Ud = S.to_device(U0)
        (S.rk_step if integrator == "rk4" else S.rk54_step)(Ud, cfg.dt, 3)
        out[sl] = S.to_host(Ud)
        torch.cuda.synchronize()
        S.close()
    assert np.array_equal(out[slabs].view(np.int64), out["0"].view(np.int64))
    if integrator == "rk4":
        R = Residual(m, Physics(cfg.eq, cfg.nd, **cfg.physics_kwargs()))
        assert _rel(out[slabs], integrate(R, U0, cfg.dt, 3)) <= TOL


@pytest.mark.parametrize("name,N,integrator,steps", [("c1", 5, "rk4", 7), ("c2", 4, "rk4", 3), ("c3", 3, "rk4", 2),
                                                      ("c4", 3, "rk54", 3), ("c5", 3, "rk54", 1)])
def test_graph_replay_bitwise(name, N, integrator, steps):
    """CUDA-graph replay of repeated K-step calls (sdrt_ctx_set_graph) gives bitwise the
    direct launches, also when an odd stage count flips the trace buffer between calls."""
    cfg = CONFIGS[name]
    Nt = (N,) * cfg.nd
    from oracle.mesh import build_mesh
    m = build_mesh(cfg.etype, cfg.p, Nt, cfg.lo, cfg.hi)
    out = {}
    for mode in (1, 0):
        S = _solver_env(cfg, Nt, {})
        S.set_graph(mode)
        U0 = random_state(cfg, S.shape[0], m.K, seed=9, amp=0.2)
        Ud = S.to_device(U0)
        f = S.rk_step if integrator == "rk4" else S.rk54_step
        for _ in range(3):  # capture, then two replays (RK54: alternating trace buffers)
            f(Ud, cfg.dt, steps)
        out[mode] = S.to_host(Ud)
        torch.cuda.synchronize()
        S.close()
    assert np.isfinite(out[1]).all()
    assert np.array_equal(out[1].view(np.int64), out[0].view(np.int64))
