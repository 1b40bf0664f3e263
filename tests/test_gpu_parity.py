"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerance (north_star, reading O25): per variable group g (density; the momentum
vector, whose components share one scale; energy; or the single scalar),
    e_g = max_{alpha in g} |U_gpu - U_oracle| / max_{alpha in g} |U_oracle|  <=  1e-11.
(Per-component normalisation is ill-posed for a momentum component that starts at
zero, e.g. rho v_z of the TGV.)
Inputs are seeded (sdrt_inputs); the oracle and the product receive the same arrays.
"""
import numpy as np
import pytest

from sdrt_inputs import CONFIGS, initial_state, random_state, scaled

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-11


def _groups(nv):
    return [[0]] if nv == 1 else [[0], list(range(1, nv - 1)), [nv - 1]]


def _rel(a, b):
    """max over variable groups of max|a-b| / max|b| for arrays (N_sol, N_V, K)."""
    out = 0.0
    for g in _groups(a.shape[1]):
        num = np.abs(a[:, g] - b[:, g]).max()
        den = max(np.abs(b[:, g]).max(), 1e-300)
        out = max(out, num / den)
    return float(out)


def _pair(cfg, N):
    from oracle.mesh import build_mesh
    from oracle.physics import Physics
    from oracle.residual import Residual
    from paper_2105_08632_b200.solver import Solver
    D = cfg.nd
    Nt = tuple(N) if isinstance(N, (tuple, list)) else (N,) * D
    m = build_mesh(cfg.etype, cfg.p, Nt, cfg.lo, cfg.hi)
    R = Residual(m, Physics(cfg.eq, D, **cfg.physics_kwargs()))
    S = Solver(cfg.etype, cfg.p, list(Nt), cfg.lo, cfg.hi, cfg.eq, device="cuda", **cfg.physics_kwargs())
    return m, R, S


RES_CASES = [("c1", 5), ("c1", (3, 7)), ("c2", 5), ("c3", 3), ("c4", (3, 4, 5)), ("c5", 3), ("c5", (5, 6, 7))]


@pytest.mark.parametrize("name,N", RES_CASES)
@pytest.mark.parametrize("state", ["random", "ic"])
def test_residual_parity(name, N, state):
    cfg = CONFIGS[name]
    m, R, S = _pair(cfg, N)
    nsol = R.ops.nsol
    if state == "random":
        U = random_state(cfg, nsol, m.K, seed=7, amp=0.3)
    else:
        U = initial_state(cfg, m.sol_coords())
    ref = R(U)
    got = S.to_host(S.residual(S.to_device(U)))
    torch.cuda.synchronize()
    assert np.isfinite(got).all()
    assert _rel(got, ref) <= TOL, _rel(got, ref)
    assert S.last_launches() > 0


RK_CASES = [("c1", 8, 100), ("c2", 6, 40), ("c3", 3, 10), ("c4", 4, 10), ("c5", 3, 4)]


@pytest.mark.parametrize("name,N,steps", RK_CASES)
def test_rk4_parity(name, N, steps):
    from oracle.residual import integrate
    cfg = CONFIGS[name]
    m, R, S = _pair(cfg, N)
    U0 = initial_state(cfg, m.sol_coords())
    ref = integrate(R, U0, cfg.dt, steps)
    Ud = S.to_device(U0)
    S.rk_step(Ud, cfg.dt, steps, check_every=steps)
    got = S.to_host(Ud)
    assert _rel(got, ref) <= TOL, _rel(got, ref)


@pytest.mark.parametrize("name,steps", [("c1", 100), ("c4", 1)])
def test_full_size_parity(name, steps):
    """BASELINE.json full sizes in the bench launch configuration (c1: the full
    100-step run; c4: 32^3 hexes p=3, one RK4 step compared element-wise)."""
    from oracle.residual import integrate
    cfg = CONFIGS[name]
    m, R, S = _pair(cfg, cfg.N)
    U0 = initial_state(cfg, m.sol_coords())
    ref = integrate(R, U0, cfg.dt, steps)
    Ud = S.to_device(U0)
    S.rk_step(Ud, cfg.dt, steps)
    got = S.to_host(Ud)
    assert _rel(got, ref) <= TOL, _rel(got, ref)


@pytest.mark.parametrize("name,Ns", [("c2", 4), ("c3", 4), ("c5", 4)])
def test_full_size_tiled_parity(name, Ns):
    """BASELINE.json full sizes in the bench launch configuration, compared with the oracle
    at every element: the uniform periodic mesh is translation invariant (PAPER.md
    l.521-527), so a state with a period of Ns patterns per axis has a residual and an RK4
    step of the same period.  The oracle runs on one Ns^D period (the same h) on a seeded
    random state; its results, tiled over the full mesh, must equal the full-size GPU
    residual and RK4 step (c5: 663 552 tetrahedra)."""
    from oracle.mesh import build_mesh
    from oracle.physics import Physics
    from oracle.residual import Residual, integrate
    from paper_2105_08632_b200.solver import Solver
    cfg = CONFIGS[name]
    D, N = cfg.nd, cfg.N
    assert N % Ns == 0
    lo, hi = np.asarray(cfg.lo, dtype=float), np.asarray(cfg.hi, dtype=float)
    m = build_mesh(cfg.etype, cfg.p, Ns, list(lo), list(lo + (hi - lo) * (Ns / N)))
    R = Residual(m, Physics(cfg.eq, D, **cfg.physics_kwargs()))
    Us = random_state(cfg, R.ops.nsol, m.K, seed=7, amp=0.2)
    nsub = m.K // Ns ** D

    def tile(A):  # element order: pattern (x fastest) major, subcell innermost
        a = A.reshape(A.shape[:2] + (Ns,) * D + (nsub,))
        a = np.tile(a, (1, 1) + (N // Ns,) * D + (1,))
        return a.reshape(A.shape[:2] + (N ** D * nsub,))

    S = Solver(cfg.etype, cfg.p, N, cfg.lo, cfg.hi, cfg.eq, device="cuda", **cfg.physics_kwargs())
    K = S.K
    Uf = tile(Us)
    assert Uf.shape[2] == K
    got = S.to_host(S.residual(S.to_device(Uf)))[:, :, :K]
    assert _rel(got, tile(R(Us))) <= TOL, _rel(got, tile(R(Us)))
    Ud = S.to_device(Uf)
    S.rk_step(Ud, cfg.dt, 1)
    ref = tile(integrate(R, Us, cfg.dt, 1))
    got = S.to_host(Ud)[:, :, :K]
    assert _rel(got, ref) <= TOL, _rel(got, ref)
    S.close()


def test_divergence_is_reported():
    from paper_2105_08632_b200 import sdrt
    cfg = CONFIGS["c2"]
    m, R, S = _pair(cfg, 4)
    U = initial_state(cfg, m.sol_coords())
    U[:, 0, 5] = -1.0          # negative density in element 5
    Ud = S.to_device(U)
    with pytest.raises(sdrt.SdrtError) as e:
        S.rk_step(Ud, 0.0, 1, check_every=1)
    assert e.value.code == -7 and "element" in str(e.value)


@pytest.mark.parametrize("name", ["c2", "c3", "c5"])
def test_full_size_invariants(name):
    """BASELINE.json full sizes in the bench launch configuration, checked through
    properties that hold at any size (the oracle does not fit the c5 mesh in a test):
    freestream preservation and discrete conservation
    sum_e detJ_e sum_r w_r (dU/dt)_{r,e} = 0 to round-off (l.312-318; w from the oracle's
    quadrature weights), plus one finite RK4 step of the configuration's initial field."""
    from oracle.operators import build_operators
    from paper_2105_08632_b200 import sdrt
    from paper_2105_08632_b200.solver import Solver
    cfg = CONFIGS[name]
    S = Solver(cfg.etype, cfg.p, cfg.N, cfg.lo, cfg.hi, cfg.eq, device="cuda", **cfg.physics_kwargs())
    nsol, nv, Kp = S.shape
    K = S.K
    # freestream: constant state (Euler/NS: rho = 1, v = (0.3, -0.2, 0.1) |c|, p from the config)
    U0 = initial_state(cfg, S.sol_coords())
    const = U0[:, :, :K].mean(axis=(0, 2))
    Uc = np.broadcast_to(const[None, :, None], (nsol, nv, K)).copy()
    r = S.to_host(S.residual(S.to_device(Uc)))[:, :, :K]
    scale = np.abs(Uc).max()
    assert np.abs(r).max() <= 1e-10 * max(scale, 1.0), np.abs(r).max()
    # conservation on the initial field
    r = S.to_host(S.residual(S.to_device(U0)))[:, :, :K]
    w = build_operators(cfg.etype, cfg.p).w
    detj = sdrt.mesh_detj(S.mesh)[:K]
    total = np.einsum("r,rvk,k->v", w, r, detj)
    mag = np.einsum("r,rvk,k->v", w, np.abs(r), detj)
    assert (np.abs(total) <= 1e-12 * np.maximum(mag, 1e-300)).all(), (total, mag)
    # one RK4 step stays finite
    Ud = S.to_device(U0)
    S.rk_step(Ud, cfg.dt, 1)
    assert np.isfinite(S.to_host(Ud)[:, :, :K]).all()
    S.close()


@pytest.mark.parametrize("name,N,steps", [("c1", 8, 50), ("c2", 6, 20), ("c3", 3, 5), ("c4", 4, 5), ("c5", 3, 3)])
def test_rk54_parity(name, N, steps):
    """RK54 (NEXT row N2): the fused kernels' 2N-storage stages
    against the oracle's rk54_step (itself pinned to the paper's stability polynomial and
    tau_MAX RK54 columns)."""
    from oracle.residual import integrate_rk54
    cfg = CONFIGS[name]
    m, R, S = _pair(cfg, N)
    U0 = initial_state(cfg, m.sol_coords())
    ref = integrate_rk54(R, U0, cfg.dt, steps)
    Ud = S.to_device(U0)
    S.rk54_step(Ud, cfg.dt, steps, check_every=steps)
    got = S.to_host(Ud)
    assert _rel(got, ref) <= TOL, _rel(got, ref)


@pytest.mark.parametrize("name,N", [("c4", 4), ("c5", 3)])
@pytest.mark.parametrize("state", ["ic", "random"])
@pytest.mark.parametrize("degree", [10, 0, 6])
def test_tgv_diagnostics_parity(name, N, state, degree):
    """sdrt_diagnostics (NEXT row N4) against the oracle's tgv_diagnostics: the paper's
    degree-10 quadrature (default), a degree-6 rule and the solution-point sums (0)."""
    from oracle.diagnostics import tgv_diagnostics
    cfg = CONFIGS[name]
    m, R, S = _pair(cfg, N)
    U = initial_state(cfg, m.sol_coords()) if state == "ic" else random_state(cfg, R.ops.nsol, m.K, seed=3, amp=0.2)
    ref = np.array(tgv_diagnostics(R, U, degree or None))
    got = S.diagnostics(S.to_device(U), degree)
    scale = np.array([abs(ref[0]), abs(ref[1]), max(abs(ref[1]), abs(ref[2]))])
    assert (np.abs(got - ref) <= 1e-11 * scale).all(), (got, ref)


def test_diagnostics_rule_errors():
    """sdrt_diagnostics_rule accepts 0 (solution points) and 1..10 only; the diagnostics
    are refused on a non-NS context."""
    from paper_2105_08632_b200 import sdrt
    cfg = CONFIGS["c4"]
    m, R, S = _pair(cfg, 3)
    for bad in (-1, 11):
        with pytest.raises(sdrt.SdrtError) as e:
            sdrt.diagnostics_rule(S.ctx, bad)
        assert e.value.code == -1
    for ok in (0, 1, 10):
        sdrt.diagnostics_rule(S.ctx, ok)
    cfg2 = CONFIGS["c3"]
    _, _, S2 = _pair(cfg2, 3)
    U = S2.to_device(initial_state(cfg2, S2.sol_coords()))
    with pytest.raises(sdrt.SdrtError) as e:
        S2.diagnostics(U)
    assert e.value.code == -2


FR_CASES = [(sch, n, N, st) for sch in ("frsdrt", "frdg")
            for (n, N, st) in [("c1", 5, 20), ("c3", 3, 3), ("c4", (3, 4, 3), 3), ("c4", 4, 2)]] + \
           [(sch, n, N, st) for sch in ("frsdrt", "frdg")
            for (n, N, st) in [("c2", 5, 10), ("c5", 3, 2), ("c5", (3, 4, 3), 1)]]


@pytest.mark.parametrize("scheme,name,N,steps", FR_CASES)
def test_fr_parity(scheme, name, N, steps):
    """FR-SDRT / FR-DG (NEXT row N1) on the fused tensor and simplex kernels against the
    oracle's FRResidual (pinned to the paper's FR-DG quad/tri tau_MAX tables and the
    FR-SDRT == SDRT equivalence): residual on a random state and RK4 steps."""
    from oracle.fr import FRResidual
    from oracle.mesh import build_mesh
    from oracle.physics import Physics
    from oracle.residual import integrate
    from paper_2105_08632_b200.solver import Solver
    cfg = CONFIGS[name]
    D = cfg.nd
    Nt = tuple(N) if isinstance(N, (tuple, list)) else (N,) * D
    m = build_mesh(cfg.etype, cfg.p, Nt, cfg.lo, cfg.hi)
    R = FRResidual(m, Physics(cfg.eq, D, **cfg.physics_kwargs()), scheme)
    S = Solver(cfg.etype, cfg.p, list(Nt), cfg.lo, cfg.hi, cfg.eq, device="cuda", scheme=scheme,
               **cfg.physics_kwargs())
    U = random_state(cfg, R.ops.nsol, m.K, seed=11, amp=0.3)
    got = S.to_host(S.residual(S.to_device(U)))
    assert _rel(got, R(U)) <= TOL, _rel(got, R(U))
    U0 = initial_state(cfg, m.sol_coords())
    ref = integrate(R, U0, cfg.dt, steps)
    Ud = S.to_device(U0)
    S.rk_step(Ud, cfg.dt, steps)
    assert _rel(S.to_host(Ud), ref) <= TOL, _rel(S.to_host(Ud), ref)
