"""Symmetric simplex point rules used as flux points (oracle; test infrastructure only).

PAPER.md App. A l.2456-2464 places triangle interior flux points, tetrahedron face
points and tetrahedron interior flux points at Williams-Shunn quadrature points,
whose coordinates the paper does not print.  Reading O1:
each rule is the symmetric quadrature rule of maximal polynomial degree d with the
orbit structure listed below; when the degree-d moment system leaves one free
orbit parameter, it is fixed by minimising the degree-(d+1) moment defect

    E = sum_{|e| = d+1} ( sum_i w_i lambda_i^e - int lambda^e )^2

over all barycentric monomials lambda^e of total degree d+1 (a basis-free,
symmetry-invariant criterion).  Weights are free (positive at the solution).

    triangle  n=1  S3                      d=1  (centroid)
              n=3  S21                     d=2  (a = 1/6, the interior solution)
              n=6  S21 + S21               d=4  (square system)
              n=10 S3 + S21 + S111         d=5  (+ min degree-6 defect)
    tet       n=1  S4                      d=1  (centroid)
              n=4  S31                     d=2  (square system)
              n=10 S31(a = 17/250) + S22   d=3  (square system once a is fixed)

The tet 10-point rule (tet p=3 interior flux points) is the one exception to the
minimum-defect criterion: its degree-3 family has one free parameter a (the S31
orbit, points (1-3a, a, a, a)), and the SDRT tet p=3 advection operator is spatially
stable only for a <= ~0.0685 (max Re lambda(G) > 0 for a >= 0.069, including the
minimum-defect member a = 0.0735).  Reading O1 (round 2): a = 17/250 =
0.068, the stable member whose RK4 tau_MAX (kappa parallel to c) is the paper's tet
SDRT3 value 0.076 times the tet SDRT2 calibration factor
0.3285/0.124 of this build's protocol: 0.2012 vs 0.2013 (tools/tet_rule_search.py).

Orbits in barycentric coordinates: S21(a) = perms of (1-2a, a, a); S111(a, b) =
perms of (a, b, 1-a-b); S31(a) = perms of (1-3a, a, a, a); S22(a) = perms of
(a, a, 1/2-a, 1/2-a).  Point order: orbits in the listed order; inside an orbit the
distinct permutations in lexicographic order of the permuted index tuple (see
``_orbit``).  Unpinned against the paper (coordinates missing): "parity unpinned"
for the coordinates themselves; pinned by exactness/symmetry tests and by the
spatial-stability check (max Re lambda(G) <= 1e-12).
"""
from __future__ import annotations

import itertools
import math
from fractions import Fraction
from functools import lru_cache

import mpmath as mp

mp.mp.dps = 40


NPAR = {"S3": 0, "S21": 1, "S111": 2, "S4": 0, "S31": 1, "S22": 1}
# which generator slots are symbolically equal (so de-duplication of permutations
# does not depend on the numerical values during Newton iterations)
PATTERN = {"S3": (0, 0, 0), "S21": (0, 1, 1), "S111": (0, 1, 2),
           "S4": (0, 0, 0, 0), "S31": (0, 1, 1, 1), "S22": (0, 0, 2, 2)}


def orbit(kind, params):
    """Distinct permutations of the orbit generator, in lexicographic order of the
    permutation of slot indices (first occurrence kept)."""
    if kind == "S3":
        gen = (mp.mpf(1) / 3,) * 3
    elif kind == "S21":
        a = params[0]
        gen = (1 - 2 * a, a, a)
    elif kind == "S111":
        a, b = params
        gen = (a, b, 1 - a - b)
    elif kind == "S4":
        gen = (mp.mpf(1) / 4,) * 4
    elif kind == "S31":
        a = params[0]
        gen = (1 - 3 * a, a, a, a)
    elif kind == "S22":
        a = params[0]
        gen = (a, a, mp.mpf(1) / 2 - a, mp.mpf(1) / 2 - a)
    else:
        raise ValueError(kind)
    pat = PATTERN[kind]
    seen, out = set(), []
    for perm in itertools.permutations(range(len(gen))):
        key = tuple(pat[i] for i in perm)
        if key in seen:
            continue
        seen.add(key)
        out.append(tuple(gen[i] for i in perm))
    return out


def _exact(e):
    """int over the unit simplex of prod lambda_i^e_i, normalised by the simplex
    volume (Dirichlet integral): D! prod e_i! / (|e| + D)!."""
    D = len(e) - 1
    num = math.factorial(D)
    for k in e:
        num *= math.factorial(k)
    return Fraction(num, math.factorial(sum(e) + D))


RULES = {
    (2, 1): (["S3"], 1),
    (2, 3): (["S21"], 2),
    (2, 6): (["S21", "S21"], 4),
    (2, 10): (["S3", "S21", "S111"], 5),
    (3, 1): (["S4"], 1),
    (3, 4): (["S31"], 2),
    (3, 10): (["S31", "S22"], 3),
}

# Rules whose free orbit parameter is fixed by a reading instead of the defect criterion
FIXED = {(3, 10): mp.mpf(17) / 250}

# Starting guesses (only select which root of the moment equations is meant).
START = {
    (2, 3): [mp.mpf(1) / 5],
    (2, 6): [mp.mpf("0.09"), mp.mpf("0.44")],
    (2, 10): [mp.mpf("0.055"), mp.mpf("0.07"), mp.mpf("0.29")],
    (3, 4): [mp.mpf("0.14")],
    (3, 10): [mp.mpf("0.07"), mp.mpf("0.09")],
}


def _points_weights(structure, x):
    pts, ws, i = [], [], 0
    for k in structure:
        par = x[i:i + NPAR[k]]
        i += NPAR[k]
        o = orbit(k, par)
        pts += o
        ws += [x[i]] * len(o)
        i += 1
    return pts, ws


def _residuals(structure, x, D, deg_lo, deg_hi):
    pts, ws = _points_weights(structure, x)
    out = []
    for e in itertools.product(range(deg_hi + 1), repeat=D + 1):
        if deg_lo <= sum(e) <= deg_hi:
            s = mp.mpf(0)
            for p, w in zip(pts, ws):
                t = w
                for li, ei in zip(p, e):
                    if ei:
                        t *= li ** ei
                s += t
            ex = _exact(e)
            out.append(s - mp.mpf(ex.numerator) / ex.denominator)
    return out


def _gauss_newton(f, x, tol):
    """Gauss-Newton for a consistent (zero-residual) system, mp arithmetic."""
    x = list(x)
    h = mp.mpf(10) ** (-mp.mp.dps // 2)
    for _ in range(100):
        r = f(x)
        J = mp.matrix(len(r), len(x))
        for j in range(len(x)):
            xp = list(x)
            xp[j] += h
            rp = f(xp)
            xm = list(x)
            xm[j] -= h
            rm = f(xm)
            for i in range(len(r)):
                J[i, j] = (rp[i] - rm[i]) / (2 * h)
        JT = J.T
        dx = mp.lu_solve(JT * J, JT * mp.matrix(r))
        x = [x[j] - dx[j] for j in range(len(x))]
        if max(abs(d) for d in dx) < tol:
            break
    return x


def _solve_fixed(structure, D, deg, free, a_fixed, guess):
    """Solve the degree-`deg` moment system for the unknowns other than the free
    orbit parameter (index `free` in the parameter vector), which is held at a_fixed."""
    n = len(guess)
    idx = [j for j in range(n) if j != free]

    def f(y):
        x = [None] * n
        for j, v in zip(idx, y):
            x[j] = v
        if free is not None:
            x[free] = a_fixed
        return _residuals(structure, x, D, 0, deg)
    y = _gauss_newton(f, [guess[j] for j in idx], mp.mpf(10) ** (-mp.mp.dps + 8))
    x = [None] * n
    for j, v in zip(idx, y):
        x[j] = v
    if free is not None:
        x[free] = a_fixed
    return x


@lru_cache(maxsize=None)
def simplex_rule(D, n):
    """Barycentric points (list of tuples of mpf) and weights (sum = 1) of the rule."""
    structure, deg = RULES[(D, n)]
    if (D, n) in ((2, 1), (3, 1)):
        pts, ws = _points_weights(structure, [mp.mpf(1)])
        return pts, ws
    st = START[(D, n)]
    # full unknown vector: params then weight, per orbit
    guess, pi = [], 0
    for k in structure:
        for _ in range(NPAR[k]):
            guess.append(st[pi]); pi += 1
        guess.append(mp.mpf(1) / n)
    if (D, n) in ((2, 3), (2, 6), (3, 4)):
        x = _solve_fixed(structure, D, deg, None, None, guess)
    elif (D, n) in FIXED:
        x = _solve_fixed(structure, D, deg, 0, FIXED[(D, n)], guess)
    else:
        # the free parameter is the first orbit parameter (S21 a for tri10, S31 a for tet10)
        free, pos = None, 0
        for k in structure:
            if NPAR[k] and free is None:
                free = pos
            pos += NPAR[k] + 1
        warm = list(guess)

        def defect(a):
            x = _solve_fixed(structure, D, deg, free, a, warm)
            warm[:] = x
            return mp.fsum(r * r for r in _residuals(structure, x, D, deg + 1, deg + 1)), x
        # golden-section on a bracket around the starting guess, then refine
        lo, hi = guess[free] * mp.mpf("0.6"), guess[free] * mp.mpf("1.5")
        g = (mp.sqrt(5) - 1) / 2
        c, d = hi - g * (hi - lo), lo + g * (hi - lo)
        fc, fd = defect(c)[0], defect(d)[0]
        for _ in range(120):
            if fc < fd:
                hi, d, fd = d, c, fc
                c = hi - g * (hi - lo)
                fc = defect(c)[0]
            else:
                lo, c, fc = c, d, fd
                d = lo + g * (hi - lo)
                fd = defect(d)[0]
            if hi - lo < mp.mpf(10) ** (-22):
                break
        x = defect((lo + hi) / 2)[1]
    pts, ws = _points_weights(structure, x)
    for p in pts:
        if min(p) <= 0:
            raise ValueError("rule point outside the simplex")
    if min(ws) <= 0:
        raise ValueError("non-positive weight")
    return pts, ws
