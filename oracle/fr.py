"""Flux reconstruction on the SDRT data (NEXT row N1): FR-SDRT and FR-DG residuals
(oracle; test infrastructure only).

PAPER.md §2.2 "FR method" (l.353-376) and §2.3 "Connections" (l.378-434): no internal
flux points; the flux is the solution-basis interpolant of the pointwise flux at the
solution points plus corrections at the external points,
    div f~ (x_s) = sum_r f~_r . grad l_r (x_s)
                   + sum_nu [ D~_nu - (sum_r f~_r l_r(x_nu)) . n^_nu ] div g_nu (x_s)
(Eq. divergence_fr, l.400-405), with D~ the scaled common normal flux of the SDRT path.
    FR-SDRT: div g_nu = div psi_nu, the SDRT external RT basis  ->  M14     (l.407-413)
    FR-DG:   g_nu = the correction that recovers nodal DG (l.371-373); for tensor
             elements the 1D right/left Radau polynomials of degree p+1 along the face
             normal (Huynh's g_DG), i.e.
             div g_nu (x_s) = -/+ g_L/R'(xi_{s,d}) delta_tangential(s, nu);
             for simplices the DG lifting  div g_nu (x_s) = (M^-1 L)_{s nu},
             M_rs = int l_r l_s,  L_{r nu} = int_{face(nu)} l_r ell_nu dS~, with ell_nu
             the degree-p Lagrange basis of the face's flux points (dg_lift; reading in
             DESIGN.md).  For tensor elements dg_lift equals the Radau form (test pin).
The auxiliary gradient uses the same corrections (remark l.429-434):
    q~_d = sum_r u_r d_d l_r + sum_nu n^_nu,d (C_nu - u_h(x_nu)) div g_nu.
Everything else (C, common fluxes, metric terms, dU/dt = -R~/detJ) is the SDRT
residual's (residual.py).
"""
from __future__ import annotations

import itertools
import math
from fractions import Fraction
from functools import lru_cache

import numpy as np

from . import physics as phys
from .operators import _decpts, _exps_total, _f64, _inverse, _mono, _mono_integral, build_operators, sol_span
from .points import TET_FACES, TET_V, TRI_FACES, TRI_V, reference_element
from .residual import Residual


def _mono_d(e, x, d):
    """d/dx_d of the monomial x^e (extended precision)."""
    if e[d] == 0:
        return 0
    ee = list(e)
    ee[d] -= 1
    return e[d] * _mono(tuple(ee), x)


@lru_cache(maxsize=None)
def sol_derivatives(etype, p):
    """D matrices Dsol[d][s, r] = d l_r / d x~_d (x~_s) of the solution nodal basis
    (l.197-205), built in extended precision and rounded once."""
    ref = reference_element(etype, p)
    D = ref.nd
    xsol = _decpts(ref.xsol)
    sspan = sol_span(etype, p, D)
    Vu = np.array([[_mono(e, x) for x in xsol] for e in sspan], dtype=object)
    Cu = _inverse(Vu)                                   # l_r = sum_k Cu[r,k] phi_k
    out = []
    for d in range(D):
        ev = np.array([[_mono_d(e, x, d) for x in xsol] for e in sspan], dtype=object)
        out.append(_f64(Cu.dot(ev).T))                  # [s, r]
    return out


def _legendre(n, x):
    if n == 0:
        return np.ones_like(x)
    pm, pc = np.ones_like(x), x
    for k in range(1, n):
        pm, pc = pc, ((2 * k + 1) * x * pc - k * pm) / (k + 1)
    return pc


def _legendre_d(n, x):
    """P_n'(x) by the derivative recurrence (sum over P_k with matching parity)."""
    out = np.zeros_like(x)
    for k in range(n - 1, -1, -2):
        out = out + (2 * k + 1) * _legendre(k, x)
    return out


@lru_cache(maxsize=None)
def dg_correction_tensor(etype, p):
    """FR-DG correction divergence Mc[s, nu] (N_sol x N_ext) for quad/hex: along the
    face normal d, g_L(xi) = (-1)^{p+1}/2 (P_{p+1} - P_p) (g_L(-1) = 1, g_L(1) = 0) for the
    x_d = -1 face and g_R(xi) = g_L(-xi) for x_d = +1."""
    if etype not in ("quad", "hex"):
        raise ValueError("FR-DG correction implemented for tensor elements only")
    o = build_operators(etype, p)
    D = o.nd
    Mc = np.zeros((o.nsol, o.next))
    for nu in range(o.next):
        n = o.ext_normal[nu]
        d = int(np.argmax(np.abs(n)))
        side = 1 if n[d] > 0 else 0
        xn = o.xext[nu]
        for s in range(o.nsol):
            xs = o.xsol[s]
            if any(abs(xs[k] - xn[k]) > 1e-12 for k in range(D) if k != d):
                continue
            xi = np.array([xs[d]])
            # g_L'(xi) = (-1)^{p+1}/2 (P_{p+1}' - P_p')(xi);  g_R'(xi) = -g_L'(-xi)
            if side == 0:
                gl = (-1) ** (p + 1) / 2 * (_legendre_d(p + 1, xi) - _legendre_d(p, xi))
                Mc[s, nu] = -gl[0]          # div(-e_d g_L) with n^ = -e_d
            else:
                gr = -((-1) ** (p + 1) / 2 * (_legendre_d(p + 1, -xi) - _legendre_d(p, -xi)))
                Mc[s, nu] = gr[0]           # div(+e_d g_R)
    return Mc


def _pmul(a, b):
    """Product of polynomials held as {exponent tuple: coefficient}."""
    out = {}
    for ea, ca in a.items():
        for eb, cb in b.items():
            e = tuple(x + y for x, y in zip(ea, eb))
            out[e] = out.get(e, 0) + ca * cb
    return out


@lru_cache(maxsize=None)
def _unit_integral(e, simplex):
    """Exact int of t^e over the unit simplex (Dirichlet: prod e_i! / (|e| + m)!) or the
    unit box [0, 1]^m (prod 1 / (e_i + 1)), as Decimal."""
    from decimal import Decimal
    if simplex:
        num = 1
        for k in e:
            num *= math.factorial(k)
        v = Fraction(num, math.factorial(sum(e) + len(e)))
    else:
        v = Fraction(1)
        for k in e:
            v /= k + 1
    return Decimal(v.numerator) / Decimal(v.denominator)


def _faces(etype, D):
    """Per reference face: (origin x0, edge vectors T (columns), simplex parameter domain?)
    in exact integers.  Simplex faces from the vertex lists; tensor face 2d+s is x_d = 2s-1
    with the other coordinates spanning [-1, 1]."""
    if etype in ("tri", "tet"):
        V, F = (TRI_V, TRI_FACES) if etype == "tri" else (TET_V, TET_FACES)
        out = []
        for f in F:
            x0 = V[f[0]]
            T = [tuple(V[f[k]][c] - x0[c] for c in range(D)) for k in range(1, len(f))]
            out.append((x0, T, True))
        return out
    out = []
    for d in range(D):
        for sd in range(2):
            x0 = tuple((2 * sd - 1) if c == d else -1 for c in range(D))
            T = [tuple(2 if c == a else 0 for c in range(D)) for a in range(D) if a != d]
            out.append((x0, T, False))
    return out


@lru_cache(maxsize=None)
def dg_lift(etype, p):
    """Mc[s, nu] = (M^-1 L)[s, nu]: the DG lifting of the face-point values (FR-DG on any
    element type), with exact integrals (monomials over the reference element, and over
    each face in its affine parametrisation x = x0 + T t), 40-digit decimal arithmetic,
    rounded once."""
    from decimal import Decimal
    o = build_operators(etype, p)
    ref = reference_element(etype, p)
    D = o.nd
    sspan = sol_span(etype, p, D)
    xsol = _decpts(ref.xsol)
    xext = _decpts(ref.xext)
    Cu = _inverse(np.array([[_mono(e, x) for x in xsol] for e in sspan], dtype=object))
    n = len(sspan)
    # mass matrix M = Cu I Cu^T, I_km = int phi_k phi_m
    I = np.array([[_mono_integral(etype, tuple(a + b for a, b in zip(ek, em))) for em in sspan] for ek in sspan],
                 dtype=object)
    M = Cu.dot(I).dot(Cu.T)
    L = np.empty((n, o.next), dtype=object)
    L[:, :] = Decimal(0)
    for f, (x0, T, simp) in enumerate(_faces(etype, D)):
        m = len(T)
        nus = [nu for nu in range(o.next) if ref.ext_face[nu] == f]
        # face parameters of the face points: t = (T^T T)^-1 T^T (x - x0)
        G = np.array([[Decimal(sum(T[a][c] * T[b][c] for c in range(D))) for b in range(m)] for a in range(m)],
                     dtype=object)
        Gi = _inverse(G)
        ts = []
        for nu in nus:
            rhs = [sum(Decimal(T[a][c]) * (xext[nu][c] - Decimal(x0[c])) for c in range(D)) for a in range(m)]
            ts.append(tuple(sum(Gi[a, b] * rhs[b] for b in range(m)) for a in range(m)))
        fspan = _exps_total(m, p) if simp else list(itertools.product(range(p + 1), repeat=m))
        Cl = _inverse(np.array([[_mono(e, t) for t in ts] for e in fspan], dtype=object))  # ell_j = sum Cl[j,k] t^e_k
        scale = np.linalg.det(np.array([[float(G[a, b]) for b in range(m)] for a in range(m)]))
        scale = Decimal(int(round(scale))).sqrt()   # Gram determinants are integers here
        # x_c(t) = x0_c + sum_a T[a][c] t_a as polynomials in t
        xc = []
        for c in range(D):
            poly = {tuple([0] * m): Decimal(x0[c])}
            for a in range(m):
                if T[a][c]:
                    e = [0] * m
                    e[a] = 1
                    poly[tuple(e)] = poly.get(tuple(e), 0) + Decimal(T[a][c])
            xc.append(poly)
        for k, ek in enumerate(sspan):
            phi = {tuple([0] * m): Decimal(1)}
            for c in range(D):
                for _ in range(ek[c]):
                    phi = _pmul(phi, xc[c])
            # int_face phi_k ell_j dS = scale * sum Cl[j, i] int t^(e + f_i)
            for j, nu in enumerate(nus):
                v = Decimal(0)
                for i, fi in enumerate(fspan):
                    if Cl[j, i] == 0:
                        continue
                    acc = Decimal(0)
                    for te, cf in phi.items():
                        acc += cf * _unit_integral(tuple(a + b for a, b in zip(te, fi)), simp)
                    v += Cl[j, i] * acc
                for r in range(n):
                    L[r, nu] += Cu[r, k] * v * scale
    return _f64(_inverse(M).dot(L))


class FRResidual(Residual):
    """dU/dt of the FR-SDRT or FR-DG scheme on the same mesh, points and common fluxes."""

    def __init__(self, mesh, ph, scheme="frsdrt"):
        super().__init__(mesh, ph)
        o = self.ops
        self.scheme = scheme
        self.Dsol = sol_derivatives(mesh.etype, mesh.p)
        if scheme == "frsdrt":
            self.Mc = o.M14
        elif mesh.etype in ("quad", "hex"):
            self.Mc = dg_correction_tensor(mesh.etype, mesh.p)
        else:
            self.Mc = dg_lift(mesh.etype, mesh.p)
        # gradient correction per direction: (Mc_d)[s, nu] = n^_nu,d Mc[s, nu]
        self.Mcd = [self.Mc * o.ext_normal[None, :, d] for d in range(o.nd)]

    def gradient(self, U):
        o, m, ph = self.ops, self.mesh, self.ph
        nsol, NV, K = U.shape
        D = o.nd
        Uf = U.reshape(nsol, NV * K)
        Uext = (o.M0 @ Uf).reshape(o.next, NV, K)
        uL = Uext[self.pL, :, self.fL]
        uR = Uext[self.pR, :, self.fR]
        Cf = phys.common_value(ph, uL, uR)
        C = self._face_scatter(Cf, Cf, (o.next, NV, K)).reshape(o.next, NV * K)
        jump = C - Uext.reshape(o.next, NV * K)
        Qt = np.stack([(self.Dsol[d] @ Uf + self.Mcd[d] @ jump).reshape(nsol, NV, K) for d in range(D)])
        return np.einsum("kji,jsak->isak", m.Jinv, Qt)            # q_i = sum_j Jinv[j,i] q~_j

    def __call__(self, U):
        o, m, ph = self.ops, self.mesh, self.ph
        nsol, NV, K = U.shape
        D = o.nd
        Uf = U.reshape(nsol, NV * K)
        Uext = (o.M0 @ Uf).reshape(o.next, NV, K)
        Q = Qext = None
        if ph.viscous:
            Q = self.gradient(U)
            Qext = np.stack([(o.M0 @ Q[d].reshape(nsol, NV * K)).reshape(o.next, NV, K) for d in range(D)])
        # pointwise flux at the solution points, transformed: f~_d = detJ sum_j Jinv[d,j] f_j
        f = phys.flux(ph, np.moveaxis(U, 1, 0), None if Q is None else np.moveaxis(Q, 2, 1))
        ft = np.einsum("k,kdj,jask->dsak", m.detJ, m.Jinv, f)      # (D, nsol, NV, K)
        # common flux once per face point (SDRT path), D~ = +/- s F
        uL = Uext[self.pL, :, self.fL].T
        uR = Uext[self.pR, :, self.fR].T
        qL = qR = None
        if ph.viscous:
            qL = np.stack([Qext[d][self.pL, :, self.fL].T for d in range(D)])
            qR = np.stack([Qext[d][self.pR, :, self.fR].T for d in range(D)])
        Fc = phys.common_flux(ph, uL, uR, qL, qR, self.nL)
        Dt = self._face_scatter((self.s[self.pL, self.fL] * Fc).T,
                                (-self.s[self.pR, self.fR] * Fc).T, (o.next, NV, K)).reshape(o.next, NV * K)
        # interpolated discontinuous normal flux at the external points
        Dn = sum(o.ext_normal[:, d:d + 1] * (o.M0 @ ft[d].reshape(nsol, NV * K)) for d in range(D))
        R = sum(self.Dsol[d] @ ft[d].reshape(nsol, NV * K) for d in range(D)) + self.Mc @ (Dt - Dn)
        return (-R.reshape(nsol, NV, K)) / m.detJ[None, None, :]
