"""Flux reconstruction on the SDRT data (NEXT row N1): FR-SDRT and FR-DG residuals
(oracle; test infrastructure only).

PAPER.md §2.2 "FR method" (l.353-376) and §2.3 "Connections" (l.378-434): no internal
flux points; the flux is the solution-basis interpolant of the pointwise flux at the
solution points plus corrections at the external points,
    div f~ (x_s) = sum_r f~_r . grad l_r (x_s)
                   + sum_nu [ D~_nu - (sum_r f~_r l_r(x_nu)) . n^_nu ] div g_nu (x_s)
(Eq. divergence_fr, l.400-405), with D~ the scaled common normal flux of the SDRT path.
    FR-SDRT: div g_nu = div psi_nu, the SDRT external RT basis  ->  M14     (l.407-413)
    FR-DG:   g_nu = the DG correction; for tensor elements the 1D right/left Radau
             polynomials of degree p+1 along the face normal (Huynh's g_DG), i.e.
             div g_nu (x_s) = -/+ g_L/R'(xi_{s,d}) delta_tangential(s, nu)
The auxiliary gradient uses the same corrections (remark l.429-434):
    q~_d = sum_r u_r d_d l_r + sum_nu n^_nu,d (C_nu - u_h(x_nu)) div g_nu.
Everything else (C, common fluxes, metric terms, dU/dt = -R~/detJ) is the SDRT
residual's (residual.py).
"""
from __future__ import annotations

from functools import lru_cache

import numpy as np

from . import physics as phys
from .operators import _decpts, _f64, _inverse, _mono, build_operators, sol_span
from .points import reference_element
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


class FRResidual(Residual):
    """dU/dt of the FR-SDRT or FR-DG scheme on the same mesh, points and common fluxes."""

    def __init__(self, mesh, ph, scheme="frsdrt"):
        super().__init__(mesh, ph)
        o = self.ops
        self.scheme = scheme
        self.Dsol = sol_derivatives(mesh.etype, mesh.p)
        self.Mc = o.M14 if scheme == "frsdrt" else dg_correction_tensor(mesh.etype, mesh.p)
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
