"""SDRT residual in Appendix-B matrix form + classical RK4 (oracle; test infrastructure only).

State layout: U has shape (N_sol, N_V, K): the Appendix-B state matrix
U^(u) = N_sol x N_V|Omega_e| (PAPER.md Eq. state_matrices l.2835-2843).

Residual, step by step in the paper's order (§2.1 l.268-350, App. B l.2855-2925):
  1. U_ext = M0 U ;  U_u = M12 U ;  U_int = P U_u                 Eqs. l.2860-2865
  2. (viscous) per face point C = (1/2-beta) u_L + (1/2+beta) u_R l.282-291
     Q~ = M16 C + M15 U_int                                     l.2877-2880
     Q = J^-T Q~ (per solution point)                           l.299-302
     Q_ext = M5 Q ; Q_u = M18 Q                                 l.2882-2900
  3. F~_u[d] = (detJ J^-1 f(U_u, Q_u))_d ; F~_int = M19.P2 F~_u  Eq. normal_transformed_flux l.305-311
  4. per face point: common flux F(u_L, u_R, q_L, q_R, n_L), computed ONCE per face
     point; D~_L = +s_L F, D~_R = -s_R F, s = detJ |J^-T n~|      l.312-340 (O9, O28)
  5. R~ = M14 D~ + M13 F~_int                                    Eq. residual_sdrt_matrices l.2919-2925
  6. dU/dt = -R~ / detJ                                          l.347-350
"""
from __future__ import annotations

import numpy as np

from . import physics as phys
from .operators import build_operators


class Residual:
    """farfield: exterior state (N_V,) of the far-field boundary faces of a mesh with a
    non-periodic axis (boundaries take the limiting values of the
    initial field).  Such a face is evaluated like any other with the exterior side a
    GHOST element (column K of the trace arrays) whose traces are the far-field state
    and whose gradient is zero (the viscous flux of a constant state); left/right by the
    same rule O14."""

    def __init__(self, mesh, ph, farfield=None):
        self.mesh = mesh
        self.ph = ph
        self.ops = build_operators(mesh.etype, mesh.p)
        o, m = self.ops, mesh
        D = o.nd
        K = m.K
        # per external point reference normal and metric scale (+ a ghost column K)
        fn = o.ext_normal                                         # N_ext x D
        jn = np.einsum("kji,sj->ski", m.Jinv, fn)                 # J^-T n~  [s, k, i]
        nrm = np.linalg.norm(jn, axis=2)                          # N_ext x K
        self.s = np.concatenate([m.detJ[None, :] * nrm, np.zeros((o.next, 1))], axis=1)
        self.nphys = jn / nrm[..., None]                          # N_ext x K x D
        # face-point lists (flattened over faces x face points); -1 (far field) -> ghost K.
        # Face f's points are o.face_ptr[f] .. o.face_ptr[f+1] (prisms mix face sizes);
        # face_perm rows are padded with -1 beyond a face's own count.
        fptr = np.asarray(o.face_ptr, dtype=np.int64)
        fe = m.face_elem.astype(np.int64)
        fl = m.face_lface.astype(np.int64)
        gL, gR = fe[:, 0] < 0, fe[:, 1] < 0
        self.ghost_faces = int(gL.sum() + gR.sum())
        if self.ghost_faces and farfield is None:
            raise ValueError("the mesh has far-field faces: pass the far-field state")
        self.farfield = None if farfield is None else np.asarray(farfield, dtype=np.float64)
        inner = np.where(gL, fl[:, 1], fl[:, 0])                  # a real local face of each face
        n_of = np.diff(fptr)[inner]                                 # points per face
        rep = lambda a: np.repeat(a, n_of)
        q = np.concatenate([np.arange(n) for n in n_of]) if len(n_of) else np.zeros(0, dtype=np.int64)
        perm = m.face_perm.astype(np.int64)[rep(np.arange(len(fe))), q]
        self.fL = rep(np.where(gL, K, fe[:, 0]))
        self.fR = rep(np.where(gR, K, fe[:, 1]))
        # a ghost side takes the interior side's point index (ghost traces are constant)
        base_L = fptr[np.where(gL, fl[:, 1], fl[:, 0])]
        self.pL = rep(base_L) + q
        self.pR = np.where(rep(gL) | rep(gR), self.pL, fptr[np.maximum(rep(fl[:, 1]), 0)] + perm)
        # the left element's outward unit normal (ghost left: minus the interior's)
        gl = rep(gL)
        nin = self.nphys[np.where(gl, self.pR, self.pL), np.where(gl, self.fR, self.fL)]
        self.nL = np.where(gl[:, None], -nin, nin).T              # D x (F.nfp)

    # ---------------------------------------------------------------- helpers
    def _ghost(self, A, zero=False):
        """Append the ghost column: far-field traces (or zero gradients)."""
        g = np.zeros(A.shape[:-1] + (1,))
        if not zero and self.farfield is not None:
            g[..., :, 0] = self.farfield[None, :] if A.ndim == 3 else self.farfield[None, None, :]
        return np.concatenate([A, g], axis=-1)

    def _face_scatter(self, valL, valR, shape):
        out = np.zeros(shape[:-1] + (shape[-1] + 1,))
        out[self.pL, :, self.fL] = valL
        out[self.pR, :, self.fR] = valR
        return out[..., :-1]

    def gradient(self, U):
        """Physical gradient Q (D, N_sol, N_V, K) of the conserved variables (step 2)."""
        o, m, ph = self.ops, self.mesh, self.ph
        nsol, NV, K = U.shape
        D = o.nd
        Uf = U.reshape(nsol, NV * K)
        Uext = self._ghost((o.M0 @ Uf).reshape(o.next, NV, K))
        Uu = (o.M12 @ Uf).reshape(o.nu, NV, K)
        uL = Uext[self.pL, :, self.fL]                            # (F.nfp, NV)
        uR = Uext[self.pR, :, self.fR]
        Cf = phys.common_value(ph, uL, uR)
        C = self._face_scatter(Cf, Cf, (o.next, NV, K))
        Uint = (o.P @ Uu.reshape(o.nu, NV * K))
        Qt = o.M16 @ C.reshape(o.next, NV * K) + o.M15 @ Uint      # (D.nsol, NV.K)
        Qt = Qt.reshape(D, nsol, NV, K)
        return np.einsum("kji,jsak->isak", m.Jinv, Qt)            # q_i = sum_j Jinv[j,i] q~_j

    def _fluxes(self, U):
        """Steps 1-4: internal transformed fluxes F~_int (N_int, NV.K) and the common
        flux F (NV, F.nfp) at every face point, computed once per face point."""
        o, m, ph = self.ops, self.mesh, self.ph
        nsol, NV, K = U.shape
        D = o.nd
        Uf = U.reshape(nsol, NV * K)
        Uext = self._ghost((o.M0 @ Uf).reshape(o.next, NV, K))
        Uu = (o.M12 @ Uf).reshape(o.nu, NV, K)
        Qext = Qu = None
        if ph.viscous:
            Q = self.gradient(U)
            Qext = np.stack([self._ghost((o.M0 @ Q[d].reshape(nsol, NV * K)).reshape(o.next, NV, K), zero=True)
                             for d in range(D)])
            Qu = np.stack([(o.M12 @ Q[d].reshape(nsol, NV * K)).reshape(o.nu, NV, K)
                           for d in range(D)])
        # step 3: transformed flux at unique internal points
        f = phys.flux(ph, np.moveaxis(Uu, 1, 0), None if Qu is None else np.moveaxis(Qu, 2, 1))
        # f: (D, NV, nu, K);  f~_d = detJ sum_j Jinv[d, j] f_j
        ft = np.einsum("k,kdj,jauk->duak", m.detJ, m.Jinv, f)      # (D, nu, NV, K)
        Fint = o.M19P2 @ ft.reshape(D * o.nu, NV * K)              # (N_int, NV.K)
        # step 4: common flux once per face point
        uL = Uext[self.pL, :, self.fL].T                           # (NV, F.nfp)
        uR = Uext[self.pR, :, self.fR].T
        qL = qR = None
        if ph.viscous:
            qL = np.stack([Qext[d][self.pL, :, self.fL].T for d in range(D)])
            qR = np.stack([Qext[d][self.pR, :, self.fR].T for d in range(D)])
        Fc = phys.common_flux(ph, uL, uR, qL, qR, self.nL)         # (NV, F.nfp)
        return Fint, Fc

    def __call__(self, U):
        o, m = self.ops, self.mesh
        nsol, NV, K = U.shape
        Fint, Fc = self._fluxes(U)
        # D~_L = +s_L F, D~_R = -s_R F (O28: the same F on both sides)
        Dt = self._face_scatter((self.s[self.pL, self.fL] * Fc).T,
                                (-self.s[self.pR, self.fR] * Fc).T, (o.next, NV, K))
        # step 5-6
        R = o.M14 @ Dt.reshape(o.next, NV * K) + o.M13 @ Fint
        return (-R.reshape(nsol, NV, K)) / m.detJ[None, None, :]

    def face_common_flux(self, U):
        """Per-face-point common flux F (NV, F.nfp), faces in mesh order (left element,
        left local face), points in the left element's local order (O28): the left side
        receives D~ = +s_L F and the right side D~ = -s_R F of this one value."""
        return self._fluxes(U)[1]


def rk4_step(L, u, dt):
    """Classical RK4, c = (0, 1/2, 1/2, 1), b = (1/6, 1/3, 1/3, 1/6) (reading O22)."""
    k1 = L(u)
    k2 = L(u + 0.5 * dt * k1)
    k3 = L(u + 0.5 * dt * k2)
    k4 = L(u + dt * k3)
    return u + (dt / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)


def integrate(L, u, dt, nsteps):
    for _ in range(nsteps):
        u = rk4_step(L, u, dt)
    return u


# RK54: five stages, two registers, fourth order (Carpenter & Kennedy 1994, the paper's
# "RK54 (five stages, two registers and fourth order)"; its stability
# polynomial is P:1124's sum_{i<=4} z^i/i! + z^5/200).  2N-storage form:
#   dU <- A_s dU + dt L(U);  U <- U + B_s dU,  s = 0..4 (A_0 = 0).
# The semi-discrete SDRT operator is autonomous, so the stage times c_s are not needed.
RK54_A = (0.0,
          -567301805773.0 / 1357537059087.0,
          -2404267990393.0 / 2016746695238.0,
          -3550918686646.0 / 2091501179385.0,
          -1275806237668.0 / 842570457699.0)
RK54_B = (1432997174477.0 / 9575080441755.0,
          5161836677717.0 / 13612068292357.0,
          1720146321549.0 / 2090206949498.0,
          3134564353537.0 / 4481467310338.0,
          2277821191437.0 / 14882151754819.0)


def rk54_step(L, u, dt):
    """One RK54 step in the 2N-storage form above (two registers: u and du)."""
    du = 0.0 * u
    for a, b in zip(RK54_A, RK54_B):
        du = a * du + dt * L(u)
        u = u + b * du
    return u


def integrate_rk54(L, u, dt, nsteps):
    for _ in range(nsteps):
        u = rk54_step(L, u, dt)
    return u
