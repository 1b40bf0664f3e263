"""Taylor-Green-vortex diagnostics of the paper's compressible NS study (NEXT row N4).

Test infrastructure only (like the rest of oracle/): the product computes the same
ensemble averages on the GPU (sdrt_diagnostics); tests compare the two and pin this
module against closed forms of the TGV initial field.

PAPER.md l.2052-2080:
    <.> = (1/|Omega|) int_Omega . dOmega                         ensemble average
    E*  = rho v.v / (rho_inf v_inf^2)                             (printed without 1/2)
    eps2 = 2 mu t_c / (rho_inf v_inf^2) <S^d : S^d>,  S^d = (grad v + grad v^T)/2 - (div v / 3) I
    eps3 = - t_c / (rho_inf v_inf^2) <p div v>
with rho_inf = v_inf = L = t_c = 1 (reading O18).  Readings: the averages
use the solution-point quadrature sum_e detJ_e sum_r w_r (the paper uses a degree-10
cubature, l.2075); grad v comes from the LDG gradient of the residual (l.295-302) by the
chain rule of reading O20; eps1 = -d<E*>/dt is left to the caller (time differences).
"""
import numpy as np


def tgv_diagnostics(R, U):
    """Return (<E*>, eps2, eps3) of the state U (N_sol, N_V, K) for Residual R (NS)."""
    m, o, ph = R.mesh, R.ops, R.ph
    D = o.nd
    Q = R.gradient(U)                                   # (D, N_sol, N_V, K)
    rho = U[:, 0, :]
    v = U[:, 1:1 + D, :] / rho[:, None, :]              # (N_sol, D, K)
    vv = np.einsum("sik,sik->sk", v, v)
    p = (ph.gamma - 1.0) * (U[:, D + 1, :] - 0.5 * rho * vv)
    # dv[j, i] = d v_i / d x_j = (d(rho v_i)/dx_j - v_i d rho/dx_j) / rho   (reading O20)
    dv = (Q[:, :, 1:1 + D, :] - v[None, :, :, :] * Q[:, :, 0:1, :]) / rho[None, :, None, :]
    dv = np.transpose(dv, (1, 0, 2, 3))                 # (N_sol, j, i, K)
    div = np.einsum("sjjk->sk", dv)
    S = 0.5 * (dv + np.transpose(dv, (0, 2, 1, 3)))
    S = S - (div / 3.0)[:, None, None, :] * np.eye(D)[None, :, :, None]
    SS = np.einsum("sjik,sjik->sk", S, S)
    wts = o.w[:, None] * m.detJ[None, :]
    vol = wts.sum()
    E = float((wts * rho * vv).sum() / vol)
    eps2 = float(2.0 * ph.mu * (wts * SS).sum() / vol)
    eps3 = float(-(wts * p * div).sum() / vol)
    return E, eps2, eps3
