"""Von Neumann (block-circulant) analysis of the oracle residual (test infrastructure only).

PAPER.md §3 l.521-534 and l.861-891: on a uniform periodic mesh of one element type
the RHS Jacobian is block circulant; with u_{rho n} = u^_rho exp(i kappa . x_n) the
semi-discrete system reduces, per wavenumber, to the pattern matrix G(kappa).
Blocks are obtained by probing the (linear) oracle residual with unit impulses at
the solution points of one root pattern of a periodic mesh large enough that no
impulse response wraps (advection: 1 neighbour layer, diffusion/BR1: 2 layers,
PAPER.md l.1436-1438).

  G(kappa) = sum_b  Resp_b  exp(-i kappa . h b)      (b = pattern offset)

Used for pins: spatial stability max Re lambda(G) (l.1192-1198) and tau_MAX tables
(l.1209-1282, l.1552-1623), with RK stability polynomials of Eq. rk_exponential
(l.1122-1126): RK3 1+z+z^2/2+z^3/6, RK4 ... + z^4/24.
"""
from __future__ import annotations

import numpy as np

from .mesh import build_mesh
from .operators import build_operators
from .physics import Physics
from .residual import Residual


def pattern_blocks(etype, p, ph, layers=1, residual=Residual):
    """Responses Resp_b (dict offset -> (n, n) matrix, n = N_p * N_sol) with h = 1;
    residual: the residual class (SDRT, or fr.FRResidual partial for FR schemes)."""
    D = 2 if etype in ("quad", "tri") else 3
    N = 2 * layers + 3
    m = build_mesh(etype, p, N, [0.0] * D, [float(N)] * D)
    o = build_operators(etype, p)
    R = residual(m, ph)
    nsub, nsol = m.nsub, o.nsol
    root = sum((N // 2) * N ** d for d in range(D))
    nprobe = nsub * nsol
    U = np.zeros((nsol, nprobe, m.K))
    for s in range(nsub):
        for r in range(nsol):
            U[r, s * nsol + r, root * nsub + s] = 1.0
    resp = R(U)                                    # (nsol, nprobe, K)
    blocks = {}
    for pat in range(N ** D):
        idx, t = [], pat
        for d in range(D):
            idx.append(t % N)
            t //= N
        off = tuple(i - N // 2 for i in idx)
        B = np.zeros((nprobe, nprobe))
        for s in range(nsub):
            B[s * nsol:(s + 1) * nsol, :] = resp[:, :, pat * nsub + s]
        if np.any(B != 0):
            blocks[off] = B
    return blocks


def G_of_kappa(blocks, kappa):
    kappa = np.asarray(kappa, dtype=np.float64)
    out = None
    for off, B in blocks.items():
        ph = np.exp(-1j * float(np.dot(kappa, off)))
        out = B * ph if out is None else out + B * ph
    return out


def rk_amplification(z, stages):
    """Stability polynomial of classical RK3/RK4 (Eq. rk_exponential, l.1122-1126);
    stages = "rk54": the amplification of one oracle RK54 step (residual.rk54_step)
    applied to u' = z u, u(0) = 1 (evaluated from the scheme, not from a formula)."""
    if stages == 3:
        return 1 + z + z ** 2 / 2 + z ** 3 / 6
    if stages == 4:
        return 1 + z + z ** 2 / 2 + z ** 3 / 6 + z ** 4 / 24
    if stages == "rk54":
        from .residual import rk54_step
        z = np.asarray(z, dtype=complex)
        return rk54_step(lambda u: z * u, np.ones_like(z), 1.0)
    raise ValueError(stages)


def spectrum(blocks, kappas):
    return np.concatenate([np.linalg.eigvals(G_of_kappa(blocks, k)) for k in kappas])


def tau_max(lams, stages, lo=0.0, hi=2.0, tol=1e-6):
    """Largest tau with max |R(tau lambda)| <= 1 (+1e-12) over the sampled spectrum."""
    def ok(t):
        return np.max(np.abs(rk_amplification(t * lams, stages))) <= 1.0 + 1e-12
    while ok(hi):
        hi *= 2
    while hi - lo > tol:
        mid = 0.5 * (lo + hi)
        if ok(mid):
            lo = mid
        else:
            hi = mid
    return lo


def advection_physics(D, theta0=np.pi / 6, theta1=np.pi / 4):
    """c = 1_c(theta0, theta1), PAPER.md l.474-478 (2D: theta1 = 0)."""
    if D == 2:
        c = (np.cos(theta0), np.sin(theta0))
    else:
        c = (np.cos(theta0) * np.cos(theta1), np.sin(theta0), np.cos(theta0) * np.sin(theta1))
    return Physics("linadv", D, c=c)


def diffusion_physics(D):
    """Linear diffusion with BR1 (beta = 0) and eta = 0."""
    return Physics("linadvdiff", D, c=(0.0,) * D, mu=1.0, beta=0.0, eta=0.0)
