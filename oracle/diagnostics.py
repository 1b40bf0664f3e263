"""Taylor-Green-vortex diagnostics of the paper's compressible NS study (NEXT row N4).

Test infrastructure only (like the rest of oracle/): the product computes the same
ensemble averages on the GPU (sdrt_diagnostics); tests compare the two and pin this
module against closed forms of the TGV initial field.

PAPER.md l.2052-2080:
    <.> = (1/|Omega|) int_Omega . dOmega                         ensemble average
    E*  = rho v.v / (rho_inf v_inf^2)                             (printed without 1/2)
    eps2 = 2 mu t_c / (rho_inf v_inf^2) <S^d : S^d>,  S^d = (grad v + grad v^T)/2 - (div v / 3) I
    eps3 = - t_c / (rho_inf v_inf^2) <p div v>
    "a quadrature of degree 10 is used to assess the ensemble averages" (l.2075)
with rho_inf = v_inf = L = t_c = 1 (reading O18).  Readings: the integrand is
evaluated from the solution polynomial u_h = sum_r l_r U_r and the polynomial of the LDG
gradient Q_h = sum_r l_r Q_r (l.295-302), with grad v by the chain rule of reading O20;
the degree-10 rule is any rule exact to degree 10 on the reference element: Gauss-Legendre
products (tensor) or collapsed Gauss-Legendre (Duffy) products (simplex), mapped by the
affine element map (weights x detJ).  degree=None keeps the solution-point quadrature
sum_e detJ_e sum_r w_r.  eps1 = -d<E*>/dt is left to the caller (time differences).
"""
from functools import lru_cache

import mpmath as mp
import numpy as np

from .operators import _decpts, _f64, _inverse, _mono, sol_span
from .points import TET_V, TRI_V, gauss_legendre, reference_element


@lru_cache(maxsize=None)
def cubature(etype, degree):
    """Points (n, D) and weights (n,) of a rule on the reference element exact for
    polynomials of total degree <= degree."""
    D = 2 if etype in ("quad", "tri") else 3
    if etype in ("quad", "hex"):
        g, w = gauss_legendre(degree // 2 + 1)              # exact to 2n - 1 per axis
        pts, wts = [], []
        for idx in np.ndindex(*([len(g)] * D)):
            pts.append([g[i] for i in idx])
            wts.append(mp.fprod([w[i] for i in idx]))
    else:
        # unit simplex by the Duffy collapse t0 = a, t1 = (1-a) b, t2 = (1-a)(1-b) c with
        # Jacobian (1-a)^(D-1) (1-b)^(D-2): degree d in t is degree <= d + D - 1 in a
        nq = (degree + D - 1) // 2 + 1
        g, w = gauss_legendre(nq)
        u = [(x + 1) / 2 for x in g]
        wu = [x / 2 for x in w]
        V = TRI_V if D == 2 else TET_V
        det = 4 if D == 2 else 8                            # |det| of t -> x
        pts, wts = [], []
        for idx in np.ndindex(*([nq] * D)):
            a = [u[i] for i in idx]
            t = [a[0], (1 - a[0]) * a[1]]
            jac = (1 - a[0])
            if D == 3:
                t.append((1 - a[0]) * (1 - a[1]) * a[2])
                jac = (1 - a[0]) ** 2 * (1 - a[1])
            x = [V[0][c] + sum(t[i] * (V[i + 1][c] - V[0][c]) for i in range(D)) for c in range(D)]
            pts.append(x)
            wts.append(det * jac * mp.fprod([wu[i] for i in idx]))
    return (np.array([[float(c) for c in x] for x in pts]), np.array([float(v) for v in wts]),
            tuple(tuple(x) for x in pts))


@lru_cache(maxsize=None)
def interp_matrix(etype, p, degree):
    """B[q, r] = l_r(x_q) at the cubature points (solution nodal basis, l.197-205)."""
    ref = reference_element(etype, p)
    D = ref.nd
    sspan = sol_span(etype, p, D)
    xsol = _decpts(ref.xsol)
    Cu = _inverse(np.array([[_mono(e, x) for x in xsol] for e in sspan], dtype=object))
    xq = _decpts(cubature(etype, degree)[2])
    ev = np.array([[_mono(e, x) for x in xq] for e in sspan], dtype=object)
    return _f64(Cu.dot(ev).T)


def _averages(ph, D, Uq, Qq, wts):
    """Ensemble averages from point values Uq (npt, N_V, K), Qq (D, npt, N_V, K) and
    weights wts (npt, K) (reference weight x detJ)."""
    rho = Uq[:, 0, :]
    v = Uq[:, 1:1 + D, :] / rho[:, None, :]              # (npt, D, K)
    vv = np.einsum("sik,sik->sk", v, v)
    p = (ph.gamma - 1.0) * (Uq[:, D + 1, :] - 0.5 * rho * vv)
    # dv[j, i] = d v_i / d x_j = (d(rho v_i)/dx_j - v_i d rho/dx_j) / rho   (reading O20)
    dv = (Qq[:, :, 1:1 + D, :] - v[None, :, :, :] * Qq[:, :, 0:1, :]) / rho[None, :, None, :]
    dv = np.transpose(dv, (1, 0, 2, 3))                 # (npt, j, i, K)
    div = np.einsum("sjjk->sk", dv)
    S = 0.5 * (dv + np.transpose(dv, (0, 2, 1, 3)))
    S = S - (div / 3.0)[:, None, None, :] * np.eye(D)[None, :, :, None]
    SS = np.einsum("sjik,sjik->sk", S, S)
    vol = wts.sum()
    E = float((wts * rho * vv).sum() / vol)
    eps2 = float(2.0 * ph.mu * (wts * SS).sum() / vol)
    eps3 = float(-(wts * p * div).sum() / vol)
    return E, eps2, eps3


def tgv_diagnostics(R, U, degree=None):
    """Return (<E*>, eps2, eps3) of the state U (N_sol, N_V, K) for Residual R (NS);
    degree: None = solution-point quadrature, else the cubature exact to that degree."""
    m, o, ph = R.mesh, R.ops, R.ph
    D = o.nd
    Q = R.gradient(U)                                   # (D, N_sol, N_V, K)
    if degree is None:
        return _averages(ph, D, U, Q, o.w[:, None] * m.detJ[None, :])
    B = interp_matrix(m.etype, m.p, degree)
    W = cubature(m.etype, degree)[1]
    Uq = np.einsum("qr,rvk->qvk", B, U)
    Qq = np.einsum("qr,drvk->dqvk", B, Q)
    return _averages(ph, D, Uq, Qq, W[:, None] * m.detJ[None, :])
