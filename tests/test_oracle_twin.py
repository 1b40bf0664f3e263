"""Definition-form twin of the oracle residual on 1- and 2-element meshes (no GPU).

SURVEY §8(c) "Brute force": for every element, rebuild the Raviart-Thomas vector
polynomial from its nodal normal-flux values (internal transformed fluxes and external
common fluxes) and take its divergence analytically at
the solution points (Eq. divergence_sdrt, l.342-346); likewise the gradient as the
divergence of the RT interpolant of the normal components of u e_d (l.295-302).
This twin never forms M0, M12, M13, M14, M15, M16, P or M19.P2, never uses the
oracle's face maps (neighbours are found by matching physical coordinates across the
periodic box) and re-derives the left/right rule O14 itself; it shares with the oracle
only the point sets (App. A, pinned in test_oracle_pins.py) and the pointwise physics
(pinned in test_oracle_pins*.py).  Both residuals must agree to round-off.
"""
import itertools

import numpy as np
import pytest

from oracle import physics as phys
from oracle.mesh import build_mesh
from oracle.physics import Physics
from oracle.points import reference_element
from oracle.residual import Residual

ND = {"quad": 2, "tri": 2, "hex": 3, "tet": 3, "pri": 3}


def _sol_exps(etype, p, D):
    if etype == "pri":
        return [(a, b, c) for c in range(p + 1) for a in range(p + 1) for b in range(p + 1 - a)]
    if etype in ("tri", "tet"):
        return [e for e in itertools.product(range(p + 1), repeat=D) if sum(e) <= p]
    return list(itertools.product(range(p + 1), repeat=D))


def _rt_basis(etype, p, D):
    """RT span of App. A (l.2364, 2475-2479) as lists of (component, exponent)."""
    out = []
    if etype == "pri":  # l.2640-2642
        tri = [e for e in itertools.product(range(p + 1), repeat=2) if sum(e) <= p]
        for c in range(p + 1):
            out += [[(k, (a, b, c))] for k in range(2) for (a, b) in tri]
            out += [[(0, (a + 1, b, c)), (1, (a, b + 1, c))] for (a, b) in tri if a + b == p]
        out += [[(2, (a, b, c))] for c in range(p + 2) for (a, b) in tri]
        return out
    if etype in ("tri", "tet"):
        tot = [e for e in itertools.product(range(p + 1), repeat=D) if sum(e) <= p]
        for c in range(D):
            out += [[(c, e)] for e in tot]
        for e in itertools.product(range(p + 1), repeat=D):
            if sum(e) == p:
                out.append([(c, tuple(e[k] + (k == c) for k in range(D))) for c in range(D)])
    else:
        for c in range(D):
            out += [[(c, e)] for e in itertools.product(*[range(p + 2 if k == c else p + 1) for k in range(D)])]
    return out


def _mono(e, x):
    return np.prod([x[k] ** e[k] for k in range(len(e))])


def _dmono(e, x, c):
    if e[c] == 0:
        return 0.0
    return e[c] * np.prod([x[k] ** (e[k] - (k == c)) for k in range(len(e))])


class Twin:
    def __init__(self, etype, p, mesh, ph, farfield=None):
        self.ph, self.m = ph, mesh
        self.farfield = farfield
        ref = reference_element(etype, p)
        D = self.D = ref.nd
        f = lambda pts: np.array([[float(c) for c in x] for x in pts])
        self.xsol = f(ref.xsol)
        xext, next_n = f(ref.xext), f(ref.next_normal)
        xint = f([ref.xu[u] for u in ref.int_u])
        nint = np.eye(D)[np.array(ref.int_dir)]
        self.next = len(xext)
        self.xf = np.vstack([xext, xint])
        self.nf = np.vstack([next_n, nint])
        # solution Lagrange basis: l_r = sum_k A[r, k] phi_k,  A = V^-1, V[k, s] = phi_k(x_s)
        self.sexp = _sol_exps(etype, p, D)
        V = np.array([[_mono(e, x) for x in self.xsol] for e in self.sexp])
        self.A = np.linalg.inv(V)
        # RT: normal-DOF matrix B[sigma, j] = psi_j(x_sigma) . n_sigma and divergences
        basis = _rt_basis(etype, p, D)
        self.B = np.array([[sum(_mono(e, x) * n[c] for c, e in t) for t in basis]
                           for x, n in zip(self.xf, self.nf)])
        self.divB = np.array([[sum(_dmono(e, x, c) for c, e in t) for t in basis] for x in self.xsol])
        # physical geometry
        K = mesh.K
        self.xphys_ext = np.einsum("kij,sj->ksi", mesh.J, xext + 1.0) + mesh.x0[:, None, :]
        jn = np.einsum("kji,sj->ksi", mesh.Jinv, next_n)                  # J^-T n~
        self.scale = mesh.detJ[:, None] * np.linalg.norm(jn, axis=2)      # K x N_ext
        self.nphys = jn / np.linalg.norm(jn, axis=2)[..., None]
        # neighbours by coordinate matching modulo the periodic box
        L = mesh.hi - mesh.lo
        per = np.array(mesh.periodic if getattr(mesh, "periodic", ()) else [True] * D)
        tol = 1e-9 * float(np.min(mesh.h))
        P = self.xphys_ext.reshape(K * self.next, D)
        self.nbr = np.empty((K, self.next, 2), dtype=np.int64)
        for e in range(K):
            for s in range(self.next):
                d = P - self.xphys_ext[e, s]
                d -= np.where(per, L * np.round(d / L), 0.0)
                dist = np.abs(d).max(axis=1)
                nn = self.nphys.reshape(K * self.next, D)
                cand = np.nonzero((dist < tol) & (np.abs(nn + self.nphys[e, s]).max(axis=1) < 1e-12))[0]
                if len(cand) == 0:  # far-field boundary point: the exterior is the far field
                    x = self.xphys_ext[e, s] - mesh.lo
                    assert any(not per[c] and (abs(x[c]) < tol or abs(x[c] - L[c]) < tol) for c in range(D))
                    self.nbr[e, s] = (-1, -1)
                    continue
                assert len(cand) == 1, (e, s, cand)
                self.nbr[e, s] = divmod(int(cand[0]), self.next)
        # left rule O14 re-derived: first non-zero component of the physical normal > 0
        first = lambda n: n[np.nonzero(np.abs(n) > 1e-12)[0][0]]
        self.left = np.array([[first(self.nphys[e, s]) > 0 for s in range(self.next)] for e in range(K)])

    def interp(self, Ue, x):
        """u_h(x) = sum_r l_r(x) U_r for one element (Ue: N_sol x ...)."""
        phi = np.array([_mono(e, x) for e in self.sexp])
        return np.tensordot(self.A @ phi, Ue, axes=(0, 0))

    def rt_div(self, normal_vals):
        """Divergence at the solution points of the RT function with these normal DOFs."""
        return self.divB @ np.linalg.solve(self.B, normal_vals)

    def residual(self, U):
        m, ph, D = self.m, self.ph, self.D
        nsol, NV, K = U.shape
        ext = lambda e: [self.interp(U[:, :, e], self.xf[s]) for s in range(self.next)]
        uext = np.array([ext(e) for e in range(K)])                      # K x N_ext x NV
        ff = self.farfield
        uout = lambda e, s: ff if self.nbr[e, s, 0] < 0 else uext[self.nbr[e, s, 0], self.nbr[e, s, 1]]
        q_sol = None
        if ph.viscous:
            q_sol = np.zeros((K, nsol, D, NV))
            for e in range(K):
                w = np.zeros((len(self.xf), NV))
                for s in range(self.next):
                    uo = uout(e, s)
                    w[s] = phys.common_value(ph, uext[e, s], uo) if self.left[e, s] else \
                        phys.common_value(ph, uo, uext[e, s])
                for i in range(self.next, len(self.xf)):
                    w[i] = self.interp(U[:, :, e], self.xf[i])
                qt = np.stack([self.rt_div(self.nf[:, d:d + 1] * w) for d in range(D)], axis=1)  # nsol x D x NV
                q_sol[e] = np.einsum("ji,sjv->siv", m.Jinv[e], qt)                             # J^-T q~
        qat = lambda e, x: None if q_sol is None else self.interp(q_sol[e], x)                # D x NV
        out = np.zeros_like(U)
        for e in range(K):
            vals = np.zeros((len(self.xf), NV))
            for s in range(self.next):
                f2, s2 = self.nbr[e, s]
                ui, uo = uext[e, s], uout(e, s)
                qi = qat(e, self.xf[s])
                qo = None if qi is None else (np.zeros_like(qi) if f2 < 0 else qat(f2, self.xf[s2]))
                nout = -self.nphys[e, s] if f2 < 0 else self.nphys[f2, s2]   # the exterior's normal
                col = lambda a: a[:, None]
                colq = lambda a: None if a is None else a[:, :, None]
                if self.left[e, s]:
                    F = phys.common_flux(ph, col(ui), col(uo), colq(qi), colq(qo), self.nphys[e, s])[:, 0]
                    vals[s] = self.scale[e, s] * F
                else:
                    F = phys.common_flux(ph, col(uo), col(ui), colq(qo), colq(qi), nout)[:, 0]
                    vals[s] = -self.scale[e, s] * F
            for i in range(self.next, len(self.xf)):
                u = self.interp(U[:, :, e], self.xf[i])[:, None]
                q = None if q_sol is None else qat(e, self.xf[i])[:, :, None]
                fphys = phys.flux(ph, u, q)[:, :, 0]                               # D x NV
                ft = m.detJ[e] * (m.Jinv[e] @ fphys)                               # detJ J^-1 f
                vals[i] = self.nf[i] @ ft
            out[:, :, e] = -self.rt_div(vals) / m.detJ[e]
        return out


def _state(ph, nsol, K, rng):
    if ph.nvars == 1:
        return rng.uniform(-1, 1, (nsol, 1, K))
    D = ph.nd
    rho = rng.uniform(0.9, 1.1, (nsol, K))
    v = rng.uniform(-0.2, 0.2, (D, nsol, K))
    p = rng.uniform(0.9, 1.1, (nsol, K))
    U = np.zeros((nsol, D + 2, K))
    U[:, 0] = rho
    U[:, 1:D + 1] = np.moveaxis(rho[None] * v, 0, 1)
    U[:, -1] = p / (ph.gamma - 1) + 0.5 * rho * (v ** 2).sum(0)
    return U


CASES = [(e, p) for e in ("quad", "tri", "hex", "tet", "pri") for p in (1, 2, 3)]


@pytest.mark.parametrize("etype,p", CASES)
@pytest.mark.parametrize("eq", ["linadvdiff", "euler", "ns"])
def test_definition_form_twin(etype, p, eq):
    """1-element (self-periodic quad/hex; the 2 tris / 6 tets of one pattern) and
    2-pattern meshes: twin residual == Appendix-B matrix-form residual."""
    D = ND[etype]
    ph = Physics(eq, D, c=(0.7, -0.4, 0.3)[:D], mu=0.05, gamma=1.4, Pr=0.71,
                 beta=0.5 if eq != "euler" else 0.0, eta=0.1 if eq != "euler" else 0.0)
    rng = np.random.default_rng(11)
    for N in ([1] * D, [2] + [1] * (D - 1)):
        m = build_mesh(etype, p, tuple(N), [0.0] * D, [1.0 + 0.3 * d for d in range(D)])
        U = _state(ph, len(reference_element(etype, p).xsol), m.K, rng)
        r_mat = Residual(m, ph)(U)
        r_twin = Twin(etype, p, m, ph).residual(U)
        nv = r_mat.shape[1]
        groups = [[0]] if nv == 1 else [[0], list(range(1, nv - 1)), [nv - 1]]
        for g in groups:
            err = np.abs(r_twin[:, g] - r_mat[:, g]).max() / np.abs(r_mat[:, g]).max()
            assert err < 1e-11, (N, g, err)


# ----------------------------------------------------------------- solution-point independence
def _alt_solution_points(etype, p, rng):
    """A second unisolvent solution-point set: Gauss-Lobatto-type nodes (tensor), or the
    centroid lattice perturbed at random (simplices)."""
    ref = reference_element(etype, p)
    x = np.array([[float(c) for c in pt] for pt in ref.xsol])
    if etype in ("quad", "hex"):
        g = np.cos(np.pi * np.arange(p, -1, -1) / p)           # Chebyshev-Lobatto on [-1, 1]
        D = ND[etype]
        return np.array([[g[i] for i in idx[::-1]] for idx in itertools.product(range(p + 1), repeat=D)])
    return x + 0.05 * rng.uniform(-1, 1, x.shape) / (p + 1)


@pytest.mark.parametrize("etype,p,eq", [("quad", 3, "euler"), ("tri", 3, "euler"), ("tri", 2, "ns"),
                                        ("hex", 2, "ns"), ("tet", 2, "euler")])
def test_solution_point_independence(etype, p, eq):
    """On affine meshes the SDRT residual polynomial does not depend on the solution
    points ("the position of the solution points has little to no
    impact", l.85): flux-point values come from the same polynomial u_h, the RT
    divergence lies in the solution space.  Residual of the oracle (its points) and of
    the twin with another point set, for the same polynomial state, compared as
    polynomials at the alternative points."""
    D = ND[etype]
    rng = np.random.default_rng(5)
    ph = Physics(eq, D, mu=0.05, gamma=1.4, Pr=0.71, beta=0.5 if eq == "ns" else 0.0,
                 eta=0.1 if eq == "ns" else 0.0)
    m = build_mesh(etype, p, 2, [0.0] * D, [1.0] * D)
    xs = np.array([[float(c) for c in pt] for pt in reference_element(etype, p).xsol])
    xa = _alt_solution_points(etype, p, rng)
    ex = _sol_exps(etype, p, D)
    Vs = np.array([[_mono(e, x) for e in ex] for x in xs])     # point x monomial
    Va = np.array([[_mono(e, x) for e in ex] for x in xa])
    NV = ph.nvars
    coef = 0.05 * rng.normal(size=(len(ex), NV, m.K))
    base = _state(ph, 1, 1, np.random.default_rng(0))[0, :, 0]
    coef[0] += base[:, None]                                  # constant term (x^0)
    Us = np.einsum("sk,kvn->svn", Vs, coef)
    Ua = np.einsum("sk,kvn->svn", Va, coef)
    r_orc = Residual(m, ph)(Us)
    tw = Twin(etype, p, m, ph)
    tw.xsol = xa
    tw.A = np.linalg.inv(Va.T)
    tw.divB = np.array([[sum(_dmono(e, x, c) for c, e in t) for t in _rt_basis(etype, p, D)] for x in xa])
    r_alt = tw.residual(Ua)
    r_orc_at_alt = np.einsum("ak,kvn->avn", Va, np.linalg.solve(Vs, r_orc.reshape(len(ex), -1)).reshape(r_orc.shape))
    assert np.abs(r_alt - r_orc_at_alt).max() <= 1e-10 * np.abs(r_orc).max()


# ----------------------------------------------------------------- vortex design order
def _vortex_l2(etype, p, N, T=1.0):
    """Shu-type isentropic vortex (c2's closed form, reading O17) on [-5, 5]^2, RK4 to
    time T; L2 density error against the translated exact vortex over the elements with
    centroid in [-2.5, 2.5]^2 (the paper measures over a central window, l.1955-1960),
    integrated with the degree-10 rule of oracle.diagnostics."""
    import math
    from oracle.diagnostics import cubature, interp_matrix
    from sdrt_inputs import CONFIGS, initial_state
    from oracle.residual import rk4_step
    cfg = CONFIGS["c2"]
    m = build_mesh(etype, p, N, (-5.0, -5.0), (5.0, 5.0))
    R = Residual(m, Physics("euler", 2, gamma=1.4))
    u = initial_state(cfg, m.sol_coords())
    h = 10.0 / N
    n = int(math.ceil(T / (0.05 * h / 2.6)))
    for _ in range(n):
        u = rk4_step(R, u, T / n)
    Bq = interp_matrix(etype, p, 10)
    xq, wq, _ = cubature(etype, 10)
    X = np.einsum("kij,qj->qik", m.J, xq + 1.0) + m.x0.T[None]
    Xs = X.copy()
    Xs[:, 0] -= 0.5 * math.sqrt(1.4) * T
    err = Bq @ u[:, 0] - initial_state(cfg, Xs)[:, 0]
    cen = X.mean(axis=0)
    mask = (np.abs(cen[0]) < 2.5) & (np.abs(cen[1]) < 2.5)
    return math.sqrt(np.einsum("q,qk,k->", wq, err ** 2 * mask[None], m.detJ))


@pytest.mark.parametrize("etype,p", [("quad", 1), ("quad", 3), ("tri", 1), ("tri", 3)])
def test_isentropic_vortex_design_order(etype, p):
    """Design order on the isentropic Euler vortex (l.1905-1981; order shown only in a
    figure and, per the paper's remark l.1965-1970, dependent on m and the meshes):
    observed order N = 20 -> 40 within 0.7 of p + 1 (measured quad 2.00 / 4.41, tri
    2.09 / 3.58)."""
    import math
    e1, e2 = _vortex_l2(etype, p, 20), _vortex_l2(etype, p, 40)
    assert abs(math.log2(e1 / e2) - (p + 1)) < 0.7, (e1, e2)


# ----------------------------------------------------------------- far-field boundaries
@pytest.mark.parametrize("etype,p", [("quad", 2), ("tri", 3), ("hex", 2), ("tet", 2), ("pri", 2)])
@pytest.mark.parametrize("eq", ["linadvdiff", "euler", "ns"])
def test_farfield_twin_and_freestream(etype, p, eq):
    """Far-field boundaries (NEXT row N4): x-boundaries take a constant
    exterior state, other axes periodic.  The definition-form twin (exterior = the far
    field, zero exterior gradient, left/right by O14 re-derived) equals the matrix form,
    and a constant state equal to the far field is preserved (residual ~ 0)."""
    D = ND[etype]
    ph = Physics(eq, D, c=(0.7, -0.4, 0.3)[:D], mu=0.05, gamma=1.4, Pr=0.71,
                 beta=0.5 if eq != "euler" else 0.0, eta=0.1 if eq != "euler" else 0.0)
    rng = np.random.default_rng(17)
    per = (False,) + (True,) * (D - 1)
    m = build_mesh(etype, p, (3,) + (2,) * (D - 1), [0.0] * D, [1.0 + 0.3 * d for d in range(D)], periodic=per)
    nsol = len(reference_element(etype, p).xsol)
    U = _state(ph, nsol, m.K, rng)
    ff = U[0, :, 0].copy()
    R = Residual(m, ph, farfield=ff)
    r_mat = R(U)
    r_twin = Twin(etype, p, m, ph, farfield=ff).residual(U)
    nv = r_mat.shape[1]
    groups = [[0]] if nv == 1 else [[0], list(range(1, nv - 1)), [nv - 1]]
    for g in groups:
        assert np.abs(r_twin[:, g] - r_mat[:, g]).max() <= 1e-11 * np.abs(r_mat[:, g]).max()
    const = np.broadcast_to(ff[None, :, None], U.shape).copy()
    assert np.abs(R(const)).max() <= 1e-12 * max(1.0, np.abs(ff).max())
