"""Pointwise physics (oracle; test infrastructure only).

All functions are vectorised over trailing axes: a state u has shape (N_V, ...),
a gradient q has shape (D, N_V, ...) with q[d] = d u / d x_d (gradients of the
CONSERVED variables), a flux f has shape (D, N_V, ...).

  * linear advection-diffusion  f = c u - mu grad u
  * upwind Lax-Friedrichs common flux                          Eq. flux_advection l.491-496
  * Euler  u = (rho, rho v, rho E),  f = (rho v, rho v v + p I, (rho E + p) v)
           rho E = p/(gamma-1) + rho v.v/2                     l.1909-1935
  * Navier-Stokes viscous flux (0, -tau, -(mu c_p/Pr) grad T - tau.v),
           tau = mu (grad v + grad v^T - 2/3 div v I)          l.2012-2030
           heat term: (mu c_p/Pr) grad T = mu gamma/((gamma-1)Pr) grad(p/rho)
           (reading O18; r cancels), primitive gradients by the chain rule (O20)
  * Rusanov common convective flux                             l.324-328
           phi = max(|v_L.n| + a_L, |v_R.n| + a_R), a = sqrt(gamma p / rho)  (O13)
  * LDG common value  C = (1/2 - beta) u_L + (1/2 + beta) u_R  Eq. common_var_for_grad l.282-291
  * LDG common viscous flux
           n.[(1/2 + beta) f^v_L + (1/2 - beta) f^v_R] + eta (u_L - u_R)   l.330-335 (O10)
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

LINADV, LINADVDIFF, EULER, NS = "linadv", "linadvdiff", "euler", "ns"


@dataclass
class Physics:
    eq: str
    nd: int
    c: tuple = (0.0, 0.0, 0.0)
    mu: float = 0.0
    gamma: float = 1.4
    Pr: float = 0.71
    beta: float = 0.0
    eta: float = 0.0

    @property
    def nvars(self):
        return 1 if self.eq in (LINADV, LINADVDIFF) else self.nd + 2

    @property
    def viscous(self):
        return self.eq in (LINADVDIFF, NS)


def _dot(a, b):
    return sum(a[d] * b[d] for d in range(len(a)))


def primitives(ph, u):
    rho = u[0]
    v = [u[1 + d] / rho for d in range(ph.nd)]
    p = (ph.gamma - 1.0) * (u[ph.nd + 1] - 0.5 * rho * _dot(v, v))
    return rho, v, p


def convective_flux(ph, u):
    D = ph.nd
    if ph.eq in (LINADV, LINADVDIFF):
        return np.stack([ph.c[d] * u for d in range(D)])
    rho, v, p = primitives(ph, u)
    E = u[D + 1]
    f = np.empty((D,) + u.shape, dtype=u.dtype)
    for d in range(D):
        f[d, 0] = u[1 + d]
        for i in range(D):
            f[d, 1 + i] = u[1 + i] * v[d] + (p if i == d else 0.0)
        f[d, D + 1] = (E + p) * v[d]
    return f


def viscous_flux(ph, u, q):
    D = ph.nd
    if ph.eq == LINADVDIFF:
        return -ph.mu * q
    if ph.eq != NS:
        return np.zeros((D,) + u.shape)
    rho, v, p = primitives(ph, u)
    g = ph.gamma
    # velocity gradients dv[i][d] = d v_i / d x_d  (reading O20)
    dv = [[(q[d, 1 + i] - v[i] * q[d, 0]) / rho for d in range(D)] for i in range(D)]
    div = sum(dv[i][i] for i in range(D))
    tau = [[ph.mu * (dv[i][d] + dv[d][i] - (2.0 / 3.0) * div * (1.0 if i == d else 0.0))
            for d in range(D)] for i in range(D)]
    # d p / d x_d = (g-1) (d(rhoE) - 0.5 |v|^2 d rho - rho v.dv)
    vv = _dot(v, v)
    kappa = ph.mu * g / ((g - 1.0) * ph.Pr)
    f = np.zeros((D,) + u.shape, dtype=u.dtype)
    for d in range(D):
        dp = (g - 1.0) * (q[d, D + 1] - 0.5 * vv * q[d, 0]
                          - rho * sum(v[i] * dv[i][d] for i in range(D)))
        dT = (dp - (p / rho) * q[d, 0]) / rho          # d(p/rho)/dx_d
        for i in range(D):
            f[d, 1 + i] = -tau[i][d]
        f[d, D + 1] = -kappa * dT - sum(tau[d][i] * v[i] for i in range(D))
    return f


def flux(ph, u, q=None):
    f = convective_flux(ph, u)
    if ph.viscous:
        f = f + viscous_flux(ph, u, q)
    return f


def common_value(ph, uL, uR):
    return (0.5 - ph.beta) * uL + (0.5 + ph.beta) * uR


def common_flux(ph, uL, uR, qL, qR, n):
    """Common normal flux along n (the LEFT element's physical outward unit normal)."""
    D = ph.nd
    if ph.eq in (LINADV, LINADVDIFF):
        cn = _dot(ph.c, n)
        F = 0.5 * cn * (uL + uR) + 0.5 * np.abs(cn) * (uL - uR)
    else:
        fL = convective_flux(ph, uL)
        fR = convective_flux(ph, uR)
        rhoL, vL, pL = primitives(ph, uL)
        rhoR, vR, pR = primitives(ph, uR)
        aL = np.sqrt(ph.gamma * pL / rhoL)
        aR = np.sqrt(ph.gamma * pR / rhoR)
        phi = np.maximum(np.abs(_dot(vL, n)) + aL, np.abs(_dot(vR, n)) + aR)
        F = 0.5 * sum(n[d] * (fL[d] + fR[d]) for d in range(D)) + 0.5 * phi * (uL - uR)
    if ph.viscous:
        gL = viscous_flux(ph, uL, qL)
        gR = viscous_flux(ph, uR, qR)
        F = F + sum(n[d] * ((0.5 + ph.beta) * gL[d] + (0.5 - ph.beta) * gR[d]) for d in range(D)) \
            + ph.eta * (uL - uR)
    return F
