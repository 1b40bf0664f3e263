"""Exploration tool (oracle-side, test infrastructure): spatial stability of the tet p=3
SDRT scheme as a function of the free parameters of the two 10-point flux-point rules
(tet faces: triangle S3+S21+S111 degree-5 family; tet interior: S31+S22 degree-3 family).

Builds fp64 operators with plain numpy (monomial bases; cond ~1e4 at p=3, adequate
for eigenvalue screening), patches them into the oracle's mesh/residual/Von Neumann
harness and reports max Re lambda over a Brillouin-zone sample and RK4 tau_MAX with
kappa parallel to c.  Usage:  python tools/tet_rule_search.py [face_t] [int_a]
"""
from __future__ import annotations

import itertools
import sys

import numpy as np
from scipy.optimize import least_squares

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))

import oracle.mesh as OM
import oracle.residual as OR
import oracle.vonneumann as VN
from oracle import operators as OO
from oracle.operators import Operators, rt_span, sol_span
from oracle.points import TET_FACES, TET_V


def orbit(kind, par):
    if kind == "S3":
        gen, pat = (1 / 3,) * 3, (0, 0, 0)
    elif kind == "S21":
        gen, pat = (1 - 2 * par[0], par[0], par[0]), (0, 1, 1)
    elif kind == "S111":
        gen, pat = (par[0], par[1], 1 - par[0] - par[1]), (0, 1, 2)
    elif kind == "S4":
        gen, pat = (0.25,) * 4, (0, 0, 0, 0)
    elif kind == "S31":
        gen, pat = (1 - 3 * par[0], par[0], par[0], par[0]), (0, 1, 1, 1)
    elif kind == "S22":
        gen, pat = (par[0], par[0], 0.5 - par[0], 0.5 - par[0]), (0, 0, 2, 2)
    seen, out = set(), []
    for perm in itertools.permutations(range(len(gen))):
        key = tuple(pat[i] for i in perm)
        if key not in seen:
            seen.add(key)
            out.append(tuple(gen[i] for i in perm))
    return out


def exact_moment(e):
    from math import factorial
    D = len(e) - 1
    num = factorial(D)
    for k in e:
        num *= factorial(k)
    return num / factorial(sum(e) + D)


def moments(pts, ws, D, deg):
    out = []
    for e in itertools.product(range(deg + 1), repeat=D + 1):
        if sum(e) <= deg:
            s = sum(w * np.prod([l ** k for l, k in zip(p, e)]) for p, w in zip(pts, ws))
            out.append(s - exact_moment(e))
    return np.array(out)


def tri10(t, guess=(0.055, 0.07, 0.29)):
    """S3 + S21(t) + S111(a, b), degree 5; unknowns w0, w1, a, b, w2."""
    def f(x):
        w0, w1, a, b, w2 = x
        pts = orbit("S3", ()) + orbit("S21", (t,)) + orbit("S111", (a, b))
        ws = [w0] + [w1] * 3 + [w2] * 6
        return moments(pts, ws, 2, 5)
    r = least_squares(f, [0.1, 0.1, guess[1], guess[2], 0.1], xtol=1e-15, ftol=1e-15, gtol=1e-15)
    w0, w1, a, b, w2 = r.x
    pts = orbit("S3", ()) + orbit("S21", (t,)) + orbit("S111", (a, b))
    ws = [w0] + [w1] * 3 + [w2] * 6
    return pts, ws, np.abs(r.fun).max()


def tet10(a, guess=0.09):
    """S31(a) + S22(b), degree 3; unknowns w1, b, w2."""
    def f(x):
        w1, b, w2 = x
        pts = orbit("S31", (a,)) + orbit("S22", (b,))
        ws = [w1] * 4 + [w2] * 6
        return moments(pts, ws, 3, 3)
    r = least_squares(f, [0.1, guess, 0.1], xtol=1e-15, ftol=1e-15, gtol=1e-15)
    w1, b, w2 = r.x
    pts = orbit("S31", (a,)) + orbit("S22", (b,))
    return pts, [w1] * 4 + [w2] * 6, np.abs(r.fun).max()


def bary(lam, V):
    V = np.asarray(V, dtype=float)
    return tuple(np.asarray(lam) @ V)


def tet_ops(p, face_pts, int_pts):
    D = 3
    V = np.array(TET_V, dtype=float)
    # solution points: centroid lattice (irrelevant on affine meshes)
    xsol = []
    m, d = p, 0.25
    for k in range(m + 1):
        for j in range(m + 1 - k):
            for i in range(m + 1 - j - k):
                lam = np.array([m - i - j - k, i, j, k], float)
                xsol.append(tuple(((lam + d) / (m + 1)) @ V))
    s3 = 1 / np.sqrt(3)
    fn = [(0, 0, -1.0), (0, -1.0, 0), (s3, s3, s3), (-1.0, 0, 0)]
    xext, nrm, fid = [], [], []
    for f, (a, b, c) in enumerate(TET_FACES):
        for lam in face_pts:
            xext.append(bary(lam, V[[a, b, c]]))
            nrm.append(fn[f]); fid.append(f)
    xu = [bary(l, V) for l in int_pts]
    int_u, int_dir = [], []
    for u in range(len(xu)):
        for dd in range(D):
            int_u.append(u); int_dir.append(dd)
    nint = len(int_u)
    fpts = xext + [xu[u] for u in int_u]
    fnrm = nrm + [tuple(1.0 if c == int_dir[i] else 0.0 for c in range(D)) for i in range(nint)]
    span = rt_span("tet", p, D)
    mono = lambda e, x: np.prod([xi ** ei for xi, ei in zip(x, e)])
    Vf = np.array([[sum(mono(e, fpts[s]) * fnrm[s][c] for c, e in t) for s in range(len(fpts))]
                   for t in span])
    div = np.array([[sum(e[c] * mono(tuple(ee - (k == c) for k, ee in enumerate(e)), x) for c, e in t if e[c])
                     for x in xsol] for t in span])
    Cf = np.linalg.inv(Vf)         # Vf[k, s]; Cf[s, k] with sum_k Cf[r,k] Vf[k,s] = delta
    DT = Cf @ div                  # [r, s]
    Dn = DT.T
    nsol = len(xsol)
    ss = sol_span("tet", p, D)
    Vu = np.array([[mono(e, x) for x in xsol] for e in ss])
    Cu = np.linalg.inv(Vu)

    def lag(pts):
        ev = np.array([[mono(e, x) for x in pts] for e in ss])
        return (Cu @ ev).T
    next_ = len(xext)
    M14 = Dn[:, :next_].copy()
    M13 = Dn[:, next_:].copy()
    M16 = np.zeros((D * nsol, next_))
    M15 = np.zeros((D * nsol, nint))
    for dd in range(D):
        for r in range(next_):
            if nrm[r][dd] != 0:
                M16[dd * nsol:(dd + 1) * nsol, r] = nrm[r][dd] * DT[r]
        for i in range(nint):
            if int_dir[i] == dd:
                M15[dd * nsol:(dd + 1) * nsol, i] = M13[:, i]
    P = np.zeros((nint, len(xu)))
    M19P2 = np.zeros((nint, D * len(xu)))
    for i in range(nint):
        P[i, int_u[i]] = 1
        M19P2[i, int_dir[i] * len(xu) + int_u[i]] = 1
    ints = np.array([float(OO._mono_integral("tet", e)) for e in ss])
    return Operators("tet", p, D, nsol, next_, nint, len(xu), 4, len(face_pts),
                     lag(xext), lag(xu), M13, M14, M15, M16, P, M19P2, Cu @ ints,
                     np.array(nrm), np.array(fid), np.array(xsol), np.array(xext), np.array(xu),
                     float(np.linalg.cond(Vf, 1)), np.array(fn), tuple(f * len(face_pts) for f in range(5)))


def patch(ops):
    fn = lambda etype, p: ops
    OM.build_operators = fn
    OR.build_operators = fn
    VN.build_operators = fn


def analyse(face_t, int_a, nbz=10, nline=121, verbose=True):
    fp, fw, e1 = tri10(face_t)
    ip, iw, e2 = tet10(int_a)
    ok = (min(min(p) for p in fp) > 0 and min(fw) > 0 and min(min(p) for p in ip) > 0 and min(iw) > 0)
    ops = tet_ops(3, fp, ip)
    patch(ops)
    ph = VN.advection_physics(3)
    B = VN.pattern_blocks("tet", 3, ph, layers=1)
    d = np.array(ph.c)
    kl = [k * d for k in np.linspace(0, np.pi / np.abs(d).max(), nline)]
    lam_line = VN.spectrum(B, kl)
    ks = np.linspace(-np.pi, np.pi, nbz, endpoint=False)
    lam_bz = VN.spectrum(B, [np.array(k) for k in itertools.product(ks, ks, ks)])
    res = dict(face_t=face_t, int_a=int_a, valid=ok, moment_err=max(e1, e2), cond=ops.cond_flux,
               re_line=lam_line.real.max(), re_bz=lam_bz.real.max(),
               tau_rk4_line=VN.tau_max(lam_line, 4), tau_rk4_bz=VN.tau_max(lam_bz, 4),
               face=(fp, fw), interior=(ip, iw))
    if verbose:
        print(f"t={face_t:.6f} a={int_a:.6f} valid={ok} merr={res['moment_err']:.1e} cond={ops.cond_flux:.3g} "
              f"maxRe line={res['re_line']:.3e} bz={res['re_bz']:.3e} tau4 line={res['tau_rk4_line']:.4f} "
              f"bz={res['tau_rk4_bz']:.4f}", flush=True)
    return res


if __name__ == "__main__":
    t = float(sys.argv[1]) if len(sys.argv) > 1 else None
    a = float(sys.argv[2]) if len(sys.argv) > 2 else None
    if t is not None:
        analyse(t, a)
    else:
        for t in np.linspace(0.03, 0.09, 7):
            for a in np.linspace(0.04, 0.12, 9):
                try:
                    analyse(t, a, nbz=6, nline=61)
                except Exception as ex:  # noqa: BLE001
                    print(t, a, "fail", ex)
