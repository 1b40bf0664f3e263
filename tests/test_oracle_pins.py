"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU).

Each test names the passage (PAPER.md line numbers) it pins.  None of these
re-types the oracle's own formula: expected values come from the paper's tables
(tests/golden/paper_tables.json), closed forms computed here with numpy, exact
invariants, or brute force.
"""
import itertools
import json
import re
import math
import os

import numpy as np
import pytest

from oracle.mesh import build_mesh
from oracle.operators import build_operators
from oracle.physics import Physics, common_flux, convective_flux, viscous_flux
from oracle.points import gauss_legendre, reference_element
from oracle.residual import Residual, rk4_step
from oracle.simplex_rules import simplex_rule
from oracle import vonneumann as VN

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_tables.json")))
ELEMS = [("quad", p) for p in range(1, 5)] + [("tri", p) for p in range(1, 5)] + \
        [("hex", p) for p in range(1, 5)] + [("tet", p) for p in range(1, 4)] + [("pri", p) for p in range(1, 4)]
ND = {"quad": 2, "tri": 2, "hex": 3, "tet": 3, "pri": 3}


def _eval_count(expr, p):
    """Evaluate a Table A.3/A.4 closed form such as '3p(p+1)^2' at p."""
    py = re.sub(r"(\d|\)|p)\(", r"\1*(", expr.replace("^", "**"))
    py = re.sub(r"(\d)p", r"\1*p", py)
    return int(eval(py, {"p": p}))


# ----------------------------------------------------------------- App. A counts
@pytest.mark.parametrize("etype,p", ELEMS)
def test_point_counts_tables_A3_A4(etype, p):
    """Tables A.3/A.4."""
    ref = reference_element(etype, p)
    t = GOLD["counts_A3_A4"][etype]
    assert ref.nsol == _eval_count(t["nsol"], p)
    assert ref.next == _eval_count(t["next"], p)
    assert ref.nint == _eval_count(t["nint"], p)
    assert ref.nu == _eval_count(t["nu"], p)
    assert ref.next + ref.nint == _eval_count(t["nf"], p)


def test_gauss_legendre_closed_forms():
    """GL nodes are roots of P_n (App. A l.2618, 2625); SPEC S:43-48 examples."""
    x, w = gauss_legendre(1)
    assert float(x[0]) == 0.0 and abs(float(w[0]) - 2.0) < 1e-15
    x, w = gauss_legendre(2)
    assert abs(float(x[0]) + 1 / math.sqrt(3)) < 1e-15
    for n in range(1, 7):
        x, w = gauss_legendre(n)
        xr, wr = np.polynomial.legendre.leggauss(n)
        assert np.allclose([float(v) for v in x], xr, atol=1e-14)
        assert np.allclose([float(v) for v in w], wr, atol=1e-14)
    x, w = gauss_legendre(5)
    assert abs(sum(float(wi) * float(xi) ** 8 for xi, wi in zip(x, w)) - 2 / 9) < 1e-14


# ----------------------------------------------------------------- simplex rules
def _tri_brute(f):
    """int over the unit triangle by a Duffy-collapsed Gauss product rule (independent)."""
    t, wt = np.polynomial.legendre.leggauss(20)
    s = (t + 1) / 2
    ws = wt / 2
    tot = 0.0
    for a, wa in zip(s, ws):
        for b, wb in zip(s, ws):
            x, y = a, b * (1 - a)
            tot += wa * wb * (1 - a) * f(1 - x - y, x, y)
    return tot


def _tet_brute(f):
    t, wt = np.polynomial.legendre.leggauss(14)
    s = (t + 1) / 2
    ws = wt / 2
    tot = 0.0
    for a, wa in zip(s, ws):
        for b, wb in zip(s, ws):
            for c, wc in zip(s, ws):
                x = a
                y = b * (1 - a)
                z = c * (1 - a) * (1 - b)
                jac = (1 - a) ** 2 * (1 - b)
                tot += wa * wb * wc * jac * f(1 - x - y - z, x, y, z)
    return tot


@pytest.mark.parametrize("D,n,deg", [(2, 1, 1), (2, 3, 2), (2, 6, 4), (2, 10, 5),
                                     (3, 1, 1), (3, 4, 2), (3, 10, 3)])
def test_simplex_rule_exactness_symmetry(D, n, deg):
    """Reading O1: symmetric, interior, positive-weight rule exact to degree `deg`
    (checked against an independent Duffy/Gauss brute-force integral)."""
    pts, ws = simplex_rule(D, n)
    P = np.array([[float(c) for c in p] for p in pts])
    W = np.array([float(w) for w in ws])
    assert len(P) == n and np.all(P > 0) and np.all(W > 0)
    assert abs(W.sum() - 1.0) < 1e-14
    vol = 0.5 if D == 2 else 1.0 / 6.0
    brute = _tri_brute if D == 2 else _tet_brute
    for e in itertools.product(range(deg + 1), repeat=D + 1):
        if sum(e) > deg:
            continue
        q = vol * np.sum(W * np.prod(P ** np.array(e), axis=1))
        ex = brute(lambda *lam: np.prod([l ** k for l, k in zip(lam, e)]))
        assert abs(q - ex) < 1e-13, (e, q, ex)
    # invariance of the point set under all vertex permutations
    key = lambda A: sorted(tuple(np.round(r, 12)) for r in A)
    for perm in itertools.permutations(range(D + 1)):
        assert key(P[:, perm]) == key(P)


# ----------------------------------------------------------------- tensor closed forms
def _lagrange(nodes, j, x):
    v = 1.0
    for k, xk in enumerate(nodes):
        if k != j:
            v *= (x - xk) / (nodes[j] - xk)
    return v


def _lagrange_d(nodes, j, x):
    s = 0.0
    for m in range(len(nodes)):
        if m == j:
            continue
        t = 1.0 / (nodes[j] - nodes[m])
        for k in range(len(nodes)):
            if k != j and k != m:
                t *= (x - nodes[k]) / (nodes[j] - nodes[k])
        s += t
    return s


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_quad_operators_closed_form(p):
    """Tensor SD structure (App. A l.2618-2625, Huynh link l.388): the nodal RT
    functions are products of 1D Lagrange polynomials; the 1D external functions on
    {-1, zeros(P_p), +1} are (1+x)P_p(x)/2 and (-1)^p (1-x)P_p(x)/2."""
    o = build_operators("quad", p)
    g, _ = np.polynomial.legendre.leggauss(p + 1)
    z = np.sort(np.polynomial.legendre.legroots([0] * p + [1]))
    Pp = np.polynomial.legendre.Legendre([0] * p + [1])
    Rp = lambda x: (1 + x) * Pp(x) / 2
    Lm = lambda x: (-1) ** p * (1 - x) * Pp(x) / 2
    dR, dL = (np.polynomial.Polynomial.fit(np.linspace(-1, 1, 50), f(np.linspace(-1, 1, 50)), p + 1).deriv()
              for f in (Rp, Lm))
    fl = np.concatenate([[-1.0], z, [1.0]])
    n = p + 1
    M14 = np.zeros((n * n, 4 * n))
    M13 = np.zeros((n * n, 2 * p * n))
    M0 = np.zeros((4 * n, n * n))
    for j in range(n):
        for i in range(n):
            s = i + n * j
            for t in range(n):
                # x faces (f=0: x=-1, f=1: x=+1): points along y (index t)
                M14[s, 0 * n + t] = -(dL(g[i])) * (t == j)
                M14[s, 1 * n + t] = dR(g[i]) * (t == j)
                M14[s, 2 * n + t] = -(dL(g[j])) * (t == i)
                M14[s, 3 * n + t] = dR(g[j]) * (t == i)
            for a in range(p):
                for t in range(n):
                    # x-internal point (z_a, g_t): index a + p t ; y-internal (g_t, z_a): t + n a
                    M13[s, a + p * t] = _lagrange_d(fl, a + 1, g[i]) * (t == j)
                    M13[s, p * n + t + n * a] = _lagrange_d(fl, a + 1, g[j]) * (t == i)
    for t in range(n):
        for j in range(n):
            for i in range(n):
                s = i + n * j
                M0[0 * n + t, s] = _lagrange(g, i, -1.0) * (j == t)
                M0[1 * n + t, s] = _lagrange(g, i, 1.0) * (j == t)
                M0[2 * n + t, s] = _lagrange(g, j, -1.0) * (i == t)
                M0[3 * n + t, s] = _lagrange(g, j, 1.0) * (i == t)
    assert np.allclose(o.M14, M14, atol=1e-11, rtol=0)
    assert np.allclose(o.M13, M13, atol=1e-11, rtol=0)
    assert np.allclose(o.M0, M0, atol=1e-13, rtol=0)
    # tensor weights = products of GL weights (int l_r)
    _, wg = np.polynomial.legendre.leggauss(n)
    assert np.allclose(o.w, np.outer(wg, wg).reshape(-1), atol=1e-14)


# ----------------------------------------------------------------- exactness invariants
def _random_rt_field(etype, p, rng):
    """Random member of the RT space as written in App. A (l.2364, 2475, 2479)."""
    D = ND[etype]
    terms = []
    if etype == "pri":  # l.2640-2642, restated: [P_p^2 (+) (x,y) P~_p](x,y) P_p(z) x P_p(x,y) P_{p+1}(z)
        tri = [e for e in itertools.product(range(p + 1), repeat=2) if sum(e) <= p]
        for c in range(p + 1):
            for k in range(2):
                for (a, b) in tri:
                    terms.append((rng.normal(), [(k, (a, b, c))]))
            for (a, b) in tri:
                if a + b == p:
                    terms.append((rng.normal(), [(0, (a + 1, b, c)), (1, (a, b + 1, c))]))
        for c in range(p + 2):
            for (a, b) in tri:
                terms.append((rng.normal(), [(2, (a, b, c))]))
    elif etype in ("tri", "tet"):
        for c in range(D):
            for e in itertools.product(range(p + 1), repeat=D):
                if sum(e) <= p:
                    terms.append((rng.normal(), [(c, e)]))
        for e in itertools.product(range(p + 1), repeat=D):
            if sum(e) == p:
                a = rng.normal()
                terms.append((a, [(c, tuple(e[k] + (k == c) for k in range(D))) for c in range(D)]))
    else:
        for c in range(D):
            for e in itertools.product(*[range(p + 2 if k == c else p + 1) for k in range(D)]):
                terms.append((rng.normal(), [(c, e)]))

    def val(x):
        v = np.zeros(D)
        for a, tt in terms:
            for c, e in tt:
                v[c] += a * np.prod([x[k] ** e[k] for k in range(D)])
        return v

    def div(x):
        s = 0.0
        for a, tt in terms:
            for c, e in tt:
                if e[c]:
                    s += a * e[c] * np.prod([x[k] ** (e[k] - (k == c)) for k in range(D)])
        return s
    return val, div


@pytest.mark.parametrize("etype,p", ELEMS)
def test_rt_divergence_exactness(etype, p):
    """div of the RT nodal interpolant is exact on the RT space (l.226-237, 342-346):
    M14 (v.n)_ext + M13 (v.n)_int = div v at solution points."""
    o = build_operators(etype, p)
    ref = reference_element(etype, p)
    rng = np.random.default_rng(7)
    for _ in range(2):
        val, div = _random_rt_field(etype, p, rng)
        fe = np.array([val(x) @ n for x, n in zip(o.xext, o.ext_normal)])
        fi = np.array([val(o.xu[ref.int_u[i]])[ref.int_dir[i]] for i in range(o.nint)])
        lhs = o.M14 @ fe + o.M13 @ fi
        rhs = np.array([div(x) for x in o.xsol])
        assert np.allclose(lhs, rhs, atol=1e-9 * max(1, np.abs(rhs).max()))


@pytest.mark.parametrize("etype,p", ELEMS)
def test_gradient_and_interpolation_exactness(etype, p):
    """M0/M12 reproduce P_p (l.2855-2865); M16 u_ext + M15 u_int = grad u for u in P_p
    (l.295-298, 2867-2880)."""
    o = build_operators(etype, p)
    D = ND[etype]
    rng = np.random.default_rng(3)
    exps = [e for e in itertools.product(range(p + 1), repeat=D) if sum(e) <= p]
    coef = rng.normal(size=len(exps))
    u = lambda x: sum(c * np.prod([x[k] ** e[k] for k in range(D)]) for c, e in zip(coef, exps))
    du = lambda x, d: sum(c * e[d] * np.prod([x[k] ** (e[k] - (k == d)) for k in range(D)])
                          for c, e in zip(coef, exps) if e[d])
    us = np.array([u(x) for x in o.xsol])
    assert np.allclose(o.M0 @ us, [u(x) for x in o.xext], atol=1e-12)
    assert np.allclose(o.M12 @ us, [u(x) for x in o.xu], atol=1e-12)
    q = o.M16 @ (o.M0 @ us) + o.M15 @ (o.P @ (o.M12 @ us))
    ex = np.concatenate([[du(x, d) for x in o.xsol] for d in range(D)])
    assert np.allclose(q, ex, atol=1e-10 * max(1, np.abs(ex).max()))
    # integral weights: sum w = |ref|, w^T M13 = 0 (internal RT functions carry no
    # boundary flux: divergence theorem)
    vol = {"quad": 4.0, "hex": 8.0, "tri": 2.0, "tet": 4.0 / 3.0, "pri": 4.0}[etype]
    assert abs(o.w.sum() - vol) < 1e-13
    assert np.abs(o.w @ o.M13).max() < 1e-11


# ----------------------------------------------------------------- physics closures
def test_physics_closed_forms():
    """Euler flux and EOS (l.1909-1935); NS stress (l.2029)."""
    ph = Physics("euler", 2, gamma=1.4)
    rho, v, p = 1.0, np.array([1.0, 0.0]), 1.0
    rE = p / 0.4 + 0.5 * rho * v @ v
    assert rE == 3.0
    u = np.array([rho, rho * v[0], rho * v[1], rE])
    f = convective_flux(ph, u)
    assert np.allclose(f[0], [1.0, 2.0, 0.0, 4.0])      # energy flux (rhoE+p)v = 4 (not S:294's 3.5)
    assert np.allclose(f[1], [0.0, 0.0, 1.0, 0.0])
    # static state: momentum flux p I, energy flux 0
    u0 = np.array([1.2, 0.0, 0.0, 2.0 / 0.4])
    f0 = convective_flux(ph, u0)
    assert np.allclose(f0[0], [0, 2.0, 0, 0]) and np.allclose(f0[1], [0, 0, 2.0, 0])
    # pure shear dv0/dx1 = s  ->  tau01 = mu s, viscous momentum flux = -tau
    ns = Physics("ns", 2, mu=0.3, Pr=0.71)
    s = 0.7
    un = np.array([1.0, 0.0, 0.0, 2.5])
    q = np.zeros((2, 4))
    q[1, 1] = s                           # d(rho v0)/dy with rho = 1
    g = viscous_flux(ns, un, q)
    assert abs(g[1, 1] + 0.3 * s) < 1e-15 and abs(g[0, 2] + 0.3 * s) < 1e-15


def test_common_flux_consistency_antisymmetry():
    """Consistency and conservation F(uL,uR,n) = -F(uR,uL,-n) (l.312-318) for Rusanov
    (beta = eta = 0 for the viscous part), 1000 seeded pairs."""
    rng = np.random.default_rng(42)
    for eq in ("euler", "ns", "linadv", "linadvdiff"):
        ph = Physics(eq, 3, c=(0.3, -0.8, 0.5), mu=0.05)
        NV = ph.nvars
        n = rng.normal(size=(3, 1000))
        n /= np.linalg.norm(n, axis=0)
        if NV == 1:
            uL, uR = rng.normal(size=(1, 1000)), rng.normal(size=(1, 1000))
        else:
            def st():
                rho = rng.uniform(0.8, 1.2, 1000)
                v = rng.uniform(-0.3, 0.3, (3, 1000))
                p = rng.uniform(0.8, 1.2, 1000)
                return np.vstack([rho, rho * v, p / 0.4 + 0.5 * rho * (v ** 2).sum(0)])
            uL, uR = st(), st()
        qL, qR = rng.normal(size=(3, NV, 1000)), rng.normal(size=(3, NV, 1000))
        F1 = common_flux(ph, uL, uR, qL, qR, n)
        F2 = common_flux(ph, uR, uL, qR, qL, -n)
        assert np.allclose(F1, -F2, atol=1e-13 * np.abs(F1).max())
        Fc = common_flux(ph, uL, uL, qL, qL, n)
        from oracle.physics import flux
        fn = np.einsum("d...,dv...->v...", n, flux(ph, uL, qL))
        assert np.allclose(Fc, fn, atol=1e-12 * np.abs(fn).max())


def test_rk4_amplification():
    """RK4 on u' = lambda u gives sum_{i<=4} z^i/i! (Eq. rk_exponential l.1124)."""
    for z in [0.3, -1.2 + 0.7j, 2.1j]:
        lam = complex(z)
        u1 = rk4_step(lambda u: lam * u, np.array([1.0 + 0j]), 1.0)[0]
        assert abs(u1 - sum(z ** i / math.factorial(i) for i in range(5))) < 1e-15


# ----------------------------------------------------------------- residual invariants
def _random_state(ph, nsol, K, rng):
    if ph.nvars == 1:
        return rng.uniform(-1, 1, (nsol, 1, K))
    D = ph.nd
    rho = rng.uniform(0.95, 1.05, (nsol, K))
    v = rng.uniform(-0.1, 0.1, (D, nsol, K))
    p = rng.uniform(0.95, 1.05, (nsol, K))
    U = np.zeros((nsol, D + 2, K))
    U[:, 0] = rho
    for d in range(D):
        U[:, 1 + d] = rho * v[d]
    U[:, -1] = p / (ph.gamma - 1) + 0.5 * rho * (v ** 2).sum(0)
    return U


@pytest.mark.parametrize("etype,p", [("quad", 2), ("tri", 3), ("hex", 2), ("tet", 2), ("tet", 3), ("pri", 2),
                                     ("pri", 3)])
@pytest.mark.parametrize("eq", ["linadv", "linadvdiff", "euler", "ns"])
def test_freestream_and_conservation(etype, p, eq):
    """Free-stream preservation on uniform affine meshes (l.170-172) and discrete
    conservation: sum_n detJ_n sum_r w_r dU/dt = 0 (telescoping common fluxes,
    l.312-318)."""
    D = ND[etype]
    m = build_mesh(etype, p, 3, [0.0] * D, [1.0] * D)
    o = build_operators(etype, p)
    ph = Physics(eq, D, c=(1.0, -0.6, 0.3)[:D], mu=0.02, beta=0.5 if eq == "ns" else 0.0,
                 eta=0.1 if eq == "ns" else 0.0)
    R = Residual(m, ph)
    rng = np.random.default_rng(1)
    U = _random_state(ph, o.nsol, m.K, rng)
    const = np.broadcast_to(U[:1, :, :1], U.shape).copy()
    assert np.abs(R(const)).max() < 1e-12 * max(1.0, np.abs(const).max())
    r = R(U)
    cons = np.einsum("s,k,sak->a", o.w, m.detJ, r)
    scale = np.einsum("s,k,sak->a", o.w, m.detJ, np.abs(r))
    assert np.all(np.abs(cons) <= 1e-13 * scale + 1e-15)


def test_linearity():
    """Residual is linear for linear equations (SPEC)."""
    m = build_mesh("tri", 2, 3, [0, 0], [1, 1])
    ph = Physics("linadvdiff", 2, c=(0.4, 1.0), mu=0.1)
    R = Residual(m, ph)
    rng = np.random.default_rng(5)
    u1, u2 = rng.normal(size=(2, 6, 1, m.K))
    assert np.allclose(R(2.0 * u1 - 3.0 * u2), 2.0 * R(u1) - 3.0 * R(u2), atol=1e-12)


@pytest.mark.parametrize("etype,p,N", [("quad", 1, 4), ("quad", 3, 4), ("tri", 1, 4), ("tri", 3, 4),
                                       ("tri", 4, 3), ("hex", 1, 3), ("hex", 2, 3), ("tet", 1, 3), ("tet", 2, 3),
                                       ("pri", 1, 3), ("pri", 2, 3)])
def test_spatial_stability(etype, p, N):
    """SDRT is linearly stable for p <= 4 on these elements (l.1192-1198): max Re
    lambda of the periodic upwind advection operator <= 1e-12 (c/h units)."""
    D = ND[etype]
    m = build_mesh(etype, p, N, [0.0] * D, [float(N)] * D)
    o = build_operators(etype, p)
    R = Residual(m, VN.advection_physics(D))
    n = o.nsol * m.K
    U = np.eye(n).reshape(n, o.nsol, m.K).transpose(1, 0, 2)
    A = R(U).transpose(0, 2, 1).reshape(n, n)
    assert np.linalg.eigvals(A).real.max() <= 1e-12


@pytest.mark.parametrize("etype,p", [(e, p) for e in ("quad", "tri") for p in range(1, 5)])
def test_tau_max_diffusion_table(etype, p):
    """Diffusion tau_MAX (BR1, beta = eta = 0), Table l.1562-1565 / l.1596-1599.
    Protocol: wave vector along x, kappa h in [0, 2 pi] (the tau_MAX is independent
    of the wave angle per l.1548; the paper's 4-digit values are truncated)."""
    B = VN.pattern_blocks(etype, p, VN.diffusion_physics(2), layers=2)
    lam = VN.spectrum(B, [np.array([k, 0.0]) for k in np.linspace(0, 2 * np.pi, 361)])
    assert lam.real.max() < 1e-10
    ref = GOLD["tau_max_diffusion"][etype][str(p)]
    for stages, r in zip((3, 4), ref):
        t = VN.tau_max(lam, stages)
        assert abs(t - r) <= 1.5e-4, (stages, t, r)


@pytest.mark.parametrize("etype,p", [("quad", 1), ("quad", 2), ("quad", 3), ("quad", 4),
                                     ("hex", 1), ("hex", 3)])
def test_tau_max_advection_rk4_table(etype, p):
    """Advection tau_MAX with RK4, theta0 = pi/6 (theta1 = pi/4), Tables l.1219-1222,
    l.1294-1297.  Protocol: kappa parallel to c, kappa h up to the aliasing limit
    pi / max_i |1_c,i| (Eq. aliasing_limit l.914-922)."""
    D = ND[etype]
    ph = VN.advection_physics(D)
    d = np.array(ph.c)
    B = VN.pattern_blocks(etype, p, ph, layers=1)
    lam = VN.spectrum(B, [k * d for k in np.linspace(0, np.pi / np.abs(d).max(), 401)])
    ref = GOLD["tau_max_advection"][etype][str(p)][1]
    assert abs(VN.tau_max(lam, 4) - ref) <= 2.5e-3


# ----------------------------------------------------------------- design order
def _advection_l2_error(etype, p, N, T=0.05, dt=2.5e-4):
    """Linear advection c = (1, 1) on the periodic unit square, u0 = sin 2pi x sin 2pi y,
    classical RK4 to time T; L2 error against the exact translate u0(x - t, y - t),
    quadrature sum_e detJ_e sum_r w_r (u - u_ex)^2 at the solution points."""
    m = build_mesh(etype, p, N, (0.0, 0.0), (1.0, 1.0))
    R = Residual(m, Physics("linadv", 2, c=(1.0, 1.0)))
    x = m.sol_coords()  # (N_sol, 2, K)

    def exact(t):
        return (np.sin(2 * np.pi * (x[:, 0] - t)) * np.sin(2 * np.pi * (x[:, 1] - t)))[:, None, :]

    u = exact(0.0)
    nsteps = int(round(T / dt))
    for _ in range(nsteps):
        u = rk4_step(R, u, dt)
    err = (u - exact(nsteps * dt))[:, 0, :] ** 2
    w = build_operators(etype, p).w
    return math.sqrt(float(np.einsum("r,rk,k->", w, err, m.detJ)))


@pytest.mark.parametrize("etype,p", [("quad", 1), ("quad", 2), ("tri", 1), ("tri", 2)])
def test_design_order_linear_advection(etype, p):
    """Measured against the analytical solution (m = 1), SDRT shows p+1 order of
    accuracy for smooth pure advection (§5.1.1, l.1680-1698).  Error ratio over
    one mesh halving must give an observed order within 0.35 of p+1."""
    e1 = _advection_l2_error(etype, p, 8)
    e2 = _advection_l2_error(etype, p, 16)
    order = math.log2(e1 / e2)
    assert abs(order - (p + 1)) < 0.35, (etype, p, e1, e2, order)


# ----------------------------------------------------------------- RK54 (NEXT row N2)
def test_rk54_stability_polynomial():
    """The oracle's RK54 step applied to u' = z u reproduces the paper's RK54 stability
    polynomial sum_{i<=4} z^i/i! + z^5/200 (Eq. rk_exponential) —
    retyped here from the paper, evaluated against the 2N-storage scheme."""
    z = np.array([0.3, -1.2, 0.5 + 1.1j, -2.0 + 0.7j, 1.5j])
    ref = sum(z ** i / math.factorial(i) for i in range(5)) + z ** 5 / 200
    assert np.abs(VN.rk_amplification(z, "rk54") - ref).max() <= 1e-14


def test_rk54_nonlinear_order():
    """Fourth order on a nonlinear autonomous ODE system ("fourth order")."""
    from oracle.residual import rk54_step

    def L(u):
        return np.array([u[1], -np.sin(u[0]) - 0.1 * u[1] * u[0] ** 2])

    def run(n):
        u = np.array([1.0, 0.0])
        for _ in range(n):
            u = rk54_step(L, u, 2.0 / n)
        return u

    ref = run(4096)
    e = [np.abs(run(n) - ref).max() for n in (16, 32, 64)]
    orders = [math.log2(e[i] / e[i + 1]) for i in range(2)]
    assert all(3.7 < o < 4.4 for o in orders), orders


@pytest.mark.parametrize("etype,p", [(e, p) for e in ("quad", "tri") for p in range(1, 5)])
def test_tau_max_diffusion_rk54(etype, p):
    """RK54 column of the diffusion tau_MAX tables (l.1562-1565, l.1596-1599) with the
    oracle's RK54 amplification; same protocol as the RK3/RK4 pin."""
    B = VN.pattern_blocks(etype, p, VN.diffusion_physics(2), layers=2)
    lam = VN.spectrum(B, [np.array([k, 0.0]) for k in np.linspace(0, 2 * np.pi, 361)])
    ref = GOLD["tau_max_rk54"]["diffusion"][etype][str(p)]
    assert abs(VN.tau_max(lam, "rk54") - ref) <= 1.5e-4, (VN.tau_max(lam, "rk54"), ref)


@pytest.mark.parametrize("etype,p", [("quad", 1), ("quad", 2), ("quad", 3), ("quad", 4), ("hex", 1), ("hex", 3)])
def test_tau_max_advection_rk54(etype, p):
    """RK54 column of the advection tau_MAX tables (l.1219-1222, l.1294-1297); protocol
    of test_tau_max_advection_rk4_table (kappa parallel to c), except quad p = 1 where the
    paper's 0.695 is the full-Brillouin-zone value (the kappa-parallel sweep gives 0.718;
    the paper does not state its sweep)."""
    D = ND[etype]
    ph = VN.advection_physics(D)
    d = np.array(ph.c)
    B = VN.pattern_blocks(etype, p, ph, layers=1)
    if (etype, p) == ("quad", 1):
        ks = np.linspace(-np.pi, np.pi, 41)
        lam = VN.spectrum(B, [np.array([a, b]) for a in ks for b in ks])
    else:
        lam = VN.spectrum(B, [k * d for k in np.linspace(0, np.pi / np.abs(d).max(), 401)])
    ref = GOLD["tau_max_rk54"]["advection"][etype][str(p)]
    assert abs(VN.tau_max(lam, "rk54") - ref) <= 1e-2, (VN.tau_max(lam, "rk54"), ref)
