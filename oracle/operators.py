"""Appendix-B operator matrices (oracle; test infrastructure only).

Follows PAPER.md step by step:
  * solution basis + Vandermonde  V(u)_{k s} = psi_k(x_s)            §2 l.197-205
  * RT flux span                                                   App. A l.2364, 2475-2479
      simplex : P_p^ND (+) x P~_p   (homogeneous degree p)
      tensor  : Q_{p+1,p(,p)} x Q_{p,p+1(,p)} (x Q_{p,p,p+1})
  * flux Vandermonde V(f)_{k s} = psi^_k(x_s) . n^_s                §2.1 l.231-233
  * nodal RT functions l^_r = (V(f)^-1)_{r k} psi^_k                §2.1 l.235-237
  * M0, M12 (interpolation)                                        App. B l.2855-2865
  * M13, M14 (nodal divergences at solution points)                App. B l.2902-2907
  * M15, M16 (gradient operators, n^ . div l^)                     App. B l.2867-2871
  * P (duplication), M19.P2 (normal selection)                     App. B l.2845-2853, 2915-2917
    (readings O6/O7 in DESIGN.md: only the product M19.P2, N_int x ND.N_u, is formed)

Any basis of each span gives the same nodal operators (reading O5); the oracle uses
plain monomials and solves in 40-digit decimal arithmetic (points from mpmath), then rounds each entry once to
fp64 (reading O24). Because every monomial RT function of the tensor span has a
single non-zero component, V(f) is block diagonal for tensor elements; the solve is
done per connected block (an exact property of the zero pattern, not an
approximation).
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass
from functools import lru_cache

from decimal import Decimal, getcontext
from fractions import Fraction

import mpmath as mp
import numpy as np

from .points import reference_element

getcontext().prec = 40
ONE = Decimal(1)
ZERO = Decimal(0)


# ----------------------------------------------------------------------------- spans
def _exps_total(D, p):
    return [e for e in itertools.product(range(p + 1), repeat=D) if sum(e) <= p]


def _exps_homog(D, p):
    return [e for e in itertools.product(range(p + 1), repeat=D) if sum(e) == p]


def sol_span(etype, p, D):
    """Exponents of the solution modal space: P_p (simplex), Q_p (tensor), or
    P_p(x, y) x P_p(z) (prism, l.2731-2733)."""
    if etype in ("tri", "tet"):
        return _exps_total(D, p)
    if etype == "pri":
        return [(a, b, c) for c in range(p + 1) for (a, b) in _exps_total(2, p)]
    return list(itertools.product(range(p + 1), repeat=D))


def rt_span(etype, p, D):
    """RT modal space as vector polynomials: list of [(component, exponent), ...]."""
    out = []
    if etype == "pri":
        # [P_p(x,y)^2 (+) (x,y) P~_p(x,y)] P_p(z)  x  P_p(x,y) P_{p+1}(z)   (l.2640-2642)
        for c in range(p + 1):
            for cmp_ in range(2):
                for (a, b) in _exps_total(2, p):
                    out.append([(cmp_, (a, b, c))])
            for (a, b) in _exps_homog(2, p):
                out.append([(0, (a + 1, b, c)), (1, (a, b + 1, c))])
        for c in range(p + 2):
            for (a, b) in _exps_total(2, p):
                out.append([(2, (a, b, c))])
        return out
    if etype in ("tri", "tet"):
        for c in range(D):
            for e in _exps_total(D, p):
                out.append([(c, e)])
        for e in _exps_homog(D, p):
            terms = []
            for c in range(D):
                ee = list(e)
                ee[c] += 1
                terms.append((c, tuple(ee)))
            out.append(terms)
    else:
        for c in range(D):
            rng = [range(p + 2) if a == c else range(p + 1) for a in range(D)]
            for e in itertools.product(*rng):
                out.append([(c, e)])
    return out


def _mono(e, x):
    v = ONE
    for ei, xi in zip(e, x):
        if ei:
            v *= xi ** ei
    return v


def _mono_d(e, x, a):
    """d/dx_a of the monomial."""
    if e[a] == 0:
        return ZERO
    ee = list(e)
    ee[a] -= 1
    return e[a] * _mono(ee, x)


def _rt_dot(terms, x, n):
    s = ZERO
    for c, e in terms:
        if n[c] != 0:
            s += _mono(e, x) * n[c]
    return s


def _rt_div(terms, x):
    s = ZERO
    for c, e in terms:
        s += _mono_d(e, x, c)
    return s


def _mono_integral(etype, e):
    """Exact integral of x^e over the reference element (rational, as Decimal)."""
    if etype == "pri":
        tri = _mono_integral("tri", e[:2])
        zi = Fraction(2, e[2] + 1) if e[2] % 2 == 0 else 0
        return tri * Decimal(zi.numerator) / Decimal(zi.denominator) if zi else Decimal(0)
    if etype in ("quad", "hex"):
        v = Fraction(1)
        for ei in e:
            v *= Fraction(2, ei + 1) if ei % 2 == 0 else 0
        return Decimal(v.numerator) / Decimal(v.denominator)
    # reference simplex = -1 + 2*(unit simplex): int x^e = 2^D int prod (2 s_i - 1)^e_i
    D = len(e)
    tot = Fraction(0)
    for ks in itertools.product(*[range(ei + 1) for ei in e]):
        c = Fraction(1)
        for ei, ki in zip(e, ks):
            c *= math.comb(ei, ki) * 2 ** ki * (-1) ** (ei - ki)
        num = 1
        for ki in ks:
            num *= math.factorial(ki)
        tot += c * Fraction(num, math.factorial(sum(ks) + D))
    tot *= 2 ** D
    return Decimal(tot.numerator) / Decimal(tot.denominator)


def _inverse(B):
    """Gauss-Jordan inverse with partial pivoting on an object array of Decimals."""
    n = B.shape[0]
    A = np.concatenate([B.copy(), np.array([[ONE if i == j else ZERO for j in range(n)]
                                             for i in range(n)], dtype=object)], axis=1)
    for c in range(n):
        piv = max(range(c, n), key=lambda r: abs(A[r, c]))
        if A[piv, c] == 0:
            raise np.linalg.LinAlgError("singular Vandermonde")
        if piv != c:
            A[[c, piv]] = A[[piv, c]]
        A[c] = A[c] / A[c, c]
        col = A[:, c].copy()
        col[c] = ZERO
        nz = [r for r in range(n) if col[r] != 0]
        if nz:
            A[nz] = A[nz] - np.outer(col[nz], A[c])
    return A[:, n:]


def _blocks(V):
    """Connected blocks (row set, column set) of the zero pattern of a square matrix."""
    n = V.shape[0]
    parent = list(range(2 * n))

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    for i in range(n):
        for j in range(n):
            if V[i, j] != 0:
                ra, rb = find(i), find(n + j)
                if ra != rb:
                    parent[ra] = rb
    groups = {}
    for i in range(n):
        groups.setdefault(find(i), [[], []])[0].append(i)
    for j in range(n):
        groups.setdefault(find(n + j), [[], []])[1].append(j)
    out = list(groups.values())
    for rows, cols in out:
        if len(rows) != len(cols):
            raise np.linalg.LinAlgError("singular flux Vandermonde (block mismatch)")
    return out


def _f64(M):
    return np.vectorize(float, otypes=[np.float64])(M)


def _dec(x):
    return Decimal(mp.nstr(x, 45, strip_zeros=False)) if not isinstance(x, int) else Decimal(x)


def _decpts(pts):
    return [tuple(_dec(c) for c in x) for x in pts]


@dataclass
class Operators:
    etype: str
    p: int
    nd: int
    nsol: int
    next: int
    nint: int
    nu: int
    nfaces: int
    nfp: int            # points of the largest face (all faces but the prism's)
    M0: np.ndarray      # N_ext x N_sol
    M12: np.ndarray     # N_u x N_sol
    M13: np.ndarray     # N_sol x N_int
    M14: np.ndarray     # N_sol x N_ext
    M15: np.ndarray     # ND.N_sol x N_int
    M16: np.ndarray     # ND.N_sol x N_ext
    P: np.ndarray       # N_int x N_u
    M19P2: np.ndarray   # N_int x ND.N_u
    w: np.ndarray       # N_sol quadrature weights  w_r = int l_r
    ext_normal: np.ndarray  # N_ext x ND reference outward unit normals
    ext_face: np.ndarray    # N_ext face id
    xsol: np.ndarray    # N_sol x ND reference coordinates
    xext: np.ndarray
    xu: np.ndarray
    cond_flux: float    # 1-norm condition of V(f), diagnostics
    face_normals: np.ndarray
    face_ptr: tuple = ()  # face f: ext points face_ptr[f] .. face_ptr[f+1]


@lru_cache(maxsize=None)
def build_operators(etype, p):
    ref = reference_element(etype, p)
    D = ref.nd
    xsol, xext, xu = _decpts(ref.xsol), _decpts(ref.xext), _decpts(ref.xu)
    nrm_ext = _decpts(ref.next_normal)
    # --- flux points: external then internal, each with its DOF normal (l.250-257)
    fpts = xext + [xu[u] for u in ref.int_u]
    fnrm = nrm_ext + [tuple(ONE if c == ref.int_dir[i] else ZERO for c in range(D))
                      for i in range(ref.nint)]
    span = rt_span(etype, p, D)
    nf = len(span)
    if nf != len(fpts):
        raise ValueError(f"RT span dim {nf} != flux points {len(fpts)}")
    Vf = np.array([[_rt_dot(terms, fpts[s], fnrm[s]) for s in range(nf)] for terms in span],
                  dtype=object)
    divpsi = np.array([[_rt_div(terms, x) for x in xsol] for terms in span], dtype=object)
    # nodal RT functions l^_r = sum_k Cf[r,k] psi_k with Cf = V(f)^-1 (l.235-237);
    # divergence table DT[r, s] = div l^_r (x_sol_s)  (l.344; reading O8)
    ns = len(xsol)
    DT = np.empty((nf, ns), dtype=object)
    cond_num = 0.0
    cond_den = 0.0
    for rows, cols in _blocks(Vf):
        B = Vf[np.ix_(rows, cols)]
        Bi = _inverse(B)             # V[rows, cols] = B  =>  Cf[cols, rows] = B^-1
        DT[cols, :] = Bi.dot(divpsi[rows, :])
        cond_num = max(cond_num, float(np.max(np.sum(np.abs(_f64(B)), axis=0))))
        cond_den = max(cond_den, float(np.max(np.sum(np.abs(_f64(Bi)), axis=0))))
    Dn = _f64(DT.T)                  # N_sol x N_f
    # --- solution basis (l.197-205)
    sspan = sol_span(etype, p, D)
    if len(sspan) != ns:
        raise ValueError("solution span / points mismatch")
    Vu = np.array([[_mono(e, x) for x in xsol] for e in sspan], dtype=object)
    Cu = _inverse(Vu)                # l_r = sum_k Cu[r,k] phi_k

    def lag(points):
        ev = np.array([[_mono(e, x) for x in points] for e in sspan], dtype=object)
        return _f64(Cu.dot(ev).T)    # [s, r] = l_r(x_s)

    M0 = lag(xext)
    M12 = lag(xu)
    ints = np.array([_mono_integral(etype, e) for e in sspan], dtype=object)
    w = _f64(Cu.dot(ints))
    M14 = Dn[:, :ref.next].copy()
    M13 = Dn[:, ref.next:].copy()
    # --- gradient operators: (M16)_{d.Nsol+s, r} = n^_{r,d} div l^_r(x_s)  (l.2869-2871)
    M16 = np.zeros((D * ns, ref.next))
    M15 = np.zeros((D * ns, ref.nint))
    for d in range(D):
        for r in range(ref.next):
            nd_ = nrm_ext[r][d]
            if nd_ != 0:
                M16[d * ns:(d + 1) * ns, r] = [float(nd_ * DT[r, s]) for s in range(ns)]
        for i in range(ref.nint):
            if ref.int_dir[i] == d:
                M15[d * ns:(d + 1) * ns, i] = M13[:, i]
    P = np.zeros((ref.nint, ref.nu))
    M19P2 = np.zeros((ref.nint, D * ref.nu))
    for i in range(ref.nint):
        P[i, ref.int_u[i]] = 1.0
        M19P2[i, ref.int_dir[i] * ref.nu + ref.int_u[i]] = 1.0
    arr = lambda pts: np.array([[float(c) for c in x] for x in pts], dtype=np.float64)
    return Operators(
        etype=etype, p=p, nd=D, nsol=ns, next=ref.next, nint=ref.nint, nu=ref.nu,
        nfaces=ref.nfaces, nfp=ref.nfp,
        M0=M0, M12=M12, M13=M13, M14=M14, M15=M15, M16=M16,
        P=P, M19P2=M19P2, w=w,
        ext_normal=arr(ref.next_normal), ext_face=np.array(ref.ext_face, dtype=np.int64),
        xsol=arr(ref.xsol), xext=arr(ref.xext), xu=arr(ref.xu),
        cond_flux=cond_num * cond_den, face_normals=arr(ref.face_normals),
        face_ptr=tuple(int(v) for v in ref.face_ptr),
    )


def rt_span_numeric(etype, p):
    """The RT span as callables (numpy, fp64) for exactness tests: list of
    (eval(x)->ND vector, div(x)->scalar)."""
    D = 2 if etype in ("quad", "tri") else 3
    span = rt_span(etype, p, D)

    def mk(terms):
        def ev(x):
            v = np.zeros(D)
            for c, e in terms:
                v[c] += np.prod([xi ** ei for xi, ei in zip(x, e)])
            return v

        def dv(x):
            s = 0.0
            for c, e in terms:
                if e[c]:
                    ee = list(e)
                    ee[c] -= 1
                    s += e[c] * np.prod([xi ** ei for xi, ei in zip(x, ee)])
            return s
        return ev, dv
    return [mk(t) for t in span]
