"""Reference elements and point sets (oracle; test infrastructure only).

PAPER.md App. A (lines 2325-2816):
  * tensor elements [-1,1]^ND (l.2469-2471): solution points = Gauss-Legendre (GL)
    (p+1)^ND (l.2625); external flux points = GL (p+1)^(ND-1) per face (l.2618);
    internal flux points per axis d = zeros of P_p along d x GL across (reading O3,
    DESIGN.md), normal e_d, no duplication (P = I, l.2852).
  * simplices (l.2356-2464): reference triangle x,y >= -1, x+y <= 0; reference tet
    x,y,z >= -1, x+y+z <= -1 (reading O2). Edge flux points = GL (p+1) (l.2455);
    tet face points, interior unique flux points and solution points are
    Williams-Shunn rules in the paper (l.2456-2464), whose coordinates are NOT in
    the paper. Reading O1: flux points (tet faces, interior) use the
    maximal-degree symmetric quadrature rules of ``simplex_rules``; solution points
    (which do not affect the residual polynomial on affine meshes)
    use the symmetric "centroid lattice"
        lambda_k = (i_k + 1/(D+1)) / (p+1),  sum_k i_k = p,
    (barycentric; centroids of the upward sub-simplices of the degree-(p+1) uniform
    subdivision; unisolvent for P_p).  Counts match Tables A.3/A.4 (l.2791-2811).
    Supported degrees: triangles p = 1..4, tetrahedra p = 1..3.
  * internal simplex flux points: each unique point carries ND DOFs with normals
    e_0..e_{ND-1} (l.2453); order (unique index, normal index).

Ordering conventions (frozen):
  * tensor solution points lexicographic, x fastest;
  * tensor faces f = 2d + s (s=0: x_d=-1, s=1: x_d=+1); face points over the other
    axes in increasing axis order, lowest axis fastest;
  * tensor internal points: axis d major, then lexicographic (x fastest) over the
    grid {zeros(P_p) along d} x {GL across};
  * triangle edges 0:(V0,V1) y=-1, 1:(V1,V2) x+y=0, 2:(V2,V0) x=-1; edge points at
    V_a + (t+1)/2 (V_b - V_a), t ascending GL nodes;
  * tet faces 0:(V0,V1,V2) z=-1, 1:(V0,V1,V3) y=-1, 2:(V1,V2,V3) x+y+z=-1,
    3:(V0,V2,V3) x=-1; face points = simplex_rules triangle rule in face-vertex barycentrics;
  * lattice order: tri  for j: for i: (i0=m-i-j, i1=i, i2=j);
                   tet  for k: for j: for i: (i0=m-i-j-k, i1=i, i2=j, i3=k).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from functools import lru_cache

import mpmath as mp

from .simplex_rules import simplex_rule

mp.mp.dps = 40

NDIM = {"quad": 2, "tri": 2, "hex": 3, "tet": 3, "pri": 3}
NSUB = {"quad": 1, "tri": 2, "hex": 1, "tet": 6, "pri": 2}  # N_p

TRI_V = [(-1, -1), (1, -1), (-1, 1)]
TET_V = [(-1, -1, -1), (1, -1, -1), (-1, 1, -1), (-1, -1, 1)]
TRI_FACES = [(0, 1), (1, 2), (2, 0)]
TET_FACES = [(0, 1, 2), (0, 1, 3), (1, 2, 3), (0, 2, 3)]


def legendre(n, x):
    """P_n(x) and P_{n-1}(x) by the three-term recurrence."""
    p0, p1 = mp.mpf(1), x
    if n == 0:
        return p0, mp.mpf(0)
    for k in range(2, n + 1):
        p0, p1 = p1, ((2 * k - 1) * x * p1 - (k - 1) * p0) / k
    return p1, p0


@lru_cache(maxsize=None)
def gauss_legendre(n):
    """Roots of P_n (ascending) and GL weights, by Newton."""
    xs, ws = [], []
    for i in range(n):
        x = mp.cos(mp.pi * (i + mp.mpf(3) / 4) / (n + mp.mpf(1) / 2))
        for _ in range(200):
            pn, pm = legendre(n, x)
            dp = n * (x * pn - pm) / (x * x - 1)
            dx = pn / dp
            x -= dx
            if abs(dx) < mp.mpf(10) ** (-mp.mp.dps + 3):
                break
        pn, pm = legendre(n, x)
        dp = n * (x * pn - pm) / (x * x - 1)
        xs.append(x)
        ws.append(2 / ((1 - x * x) * dp * dp))
    order = sorted(range(n), key=lambda i: xs[i])
    return tuple(xs[i] for i in order), tuple(ws[i] for i in order)


def lattice(D, m):
    """Centroid lattice (reading O1): barycentric tuples, documented order."""
    out = []
    d = mp.mpf(1) / (D + 1)
    if D == 2:
        for j in range(m + 1):
            for i in range(m + 1 - j):
                idx = (m - i - j, i, j)
                out.append(tuple((mp.mpf(t) + d) / (m + 1) for t in idx))
    elif D == 3:
        for k in range(m + 1):
            for j in range(m + 1 - k):
                for i in range(m + 1 - j - k):
                    idx = (m - i - j - k, i, j, k)
                    out.append(tuple((mp.mpf(t) + d) / (m + 1) for t in idx))
    else:
        raise ValueError(D)
    return out


def bary_to_x(lam, verts):
    D = len(verts[0])
    return tuple(sum(lam[k] * verts[k][c] for k in range(len(verts))) for c in range(D))


@dataclass
class RefElement:
    etype: str
    p: int
    nd: int
    xsol: list                      # N_sol points (tuples of mpf)
    xext: list                      # N_ext points
    next_normal: list               # N_ext outward unit normals (mpf tuples)
    ext_face: list                  # face id per external point
    nfaces: int
    nfp: int                        # points per face
    xu: list                        # N_u unique internal points
    int_u: list                     # N_int: unique index of each internal point
    int_dir: list                   # N_int: axis d of the DOF normal e_d
    face_normals: list = field(default_factory=list)
    face_ptr: list = field(default_factory=list)   # face f: ext points face_ptr[f] .. face_ptr[f+1]

    @property
    def nsol(self):
        return len(self.xsol)

    @property
    def next(self):
        return len(self.xext)

    @property
    def nu(self):
        return len(self.xu)

    @property
    def nint(self):
        return len(self.int_u)

    def int_normal(self, i):
        n = [mp.mpf(0)] * self.nd
        n[self.int_dir[i]] = mp.mpf(1)
        return tuple(n)


def _tensor(etype, p):
    D = NDIM[etype]
    g, _ = gauss_legendre(p + 1)
    z, _ = gauss_legendre(p) if p >= 1 else ((), ())
    n = p + 1
    xsol = []
    if D == 2:
        for j in range(n):
            for i in range(n):
                xsol.append((g[i], g[j]))
    else:
        for k in range(n):
            for j in range(n):
                for i in range(n):
                    xsol.append((g[i], g[j], g[k]))
    xext, nrm, fid, fnorms = [], [], [], []
    for d in range(D):
        for s in range(2):
            f = 2 * d + s
            val = mp.mpf(2 * s - 1)
            nv = tuple(val if c == d else mp.mpf(0) for c in range(D))
            fnorms.append(nv)
            others = [c for c in range(D) if c != d]
            if D == 2:
                for t in range(n):
                    x = [None, None]
                    x[d] = val
                    x[others[0]] = g[t]
                    xext.append(tuple(x)); nrm.append(nv); fid.append(f)
            else:
                for tb in range(n):
                    for ta in range(n):
                        x = [None, None, None]
                        x[d] = val
                        x[others[0]] = g[ta]
                        x[others[1]] = g[tb]
                        xext.append(tuple(x)); nrm.append(nv); fid.append(f)
    xu, int_u, int_dir = [], [], []
    for d in range(D):
        axes = [z if c == d else g for c in range(D)]
        if D == 2:
            for c1 in range(len(axes[1])):
                for c0 in range(len(axes[0])):
                    int_u.append(len(xu)); int_dir.append(d)
                    xu.append((axes[0][c0], axes[1][c1]))
        else:
            for c2 in range(len(axes[2])):
                for c1 in range(len(axes[1])):
                    for c0 in range(len(axes[0])):
                        int_u.append(len(xu)); int_dir.append(d)
                        xu.append((axes[0][c0], axes[1][c1], axes[2][c2]))
    return RefElement(etype, p, D, xsol, xext, nrm, fid, 2 * D, n ** (D - 1),
                      xu, int_u, int_dir, fnorms, [f * n ** (D - 1) for f in range(2 * D + 1)])


def _simplex(etype, p):
    D = NDIM[etype]
    V = TRI_V if D == 2 else TET_V
    V = [tuple(mp.mpf(c) for c in v) for v in V]
    xsol = [bary_to_x(l, V) for l in lattice(D, p)]
    xext, nrm, fid, fnorms = [], [], [], []
    if D == 2:
        g, _ = gauss_legendre(p + 1)
        s2 = 1 / mp.sqrt(2)
        fnorms = [(mp.mpf(0), mp.mpf(-1)), (s2, s2), (mp.mpf(-1), mp.mpf(0))]
        for f, (a, b) in enumerate(TRI_FACES):
            for t in g:
                lam = (t + 1) / 2
                xext.append(tuple(V[a][c] + lam * (V[b][c] - V[a][c]) for c in range(2)))
                nrm.append(fnorms[f]); fid.append(f)
        nfp = p + 1
    else:
        s3 = 1 / mp.sqrt(3)
        z0 = mp.mpf(0)
        fnorms = [(z0, z0, mp.mpf(-1)), (z0, mp.mpf(-1), z0), (s3, s3, s3), (mp.mpf(-1), z0, z0)]
        fl, _ = simplex_rule(2, (p + 1) * (p + 2) // 2)
        for f, (a, b, c) in enumerate(TET_FACES):
            for lam in fl:
                xext.append(bary_to_x(lam, [V[a], V[b], V[c]]))
                nrm.append(fnorms[f]); fid.append(f)
        nfp = len(fl)
    nu = p * (p + 1) // 2 if D == 2 else p * (p + 1) * (p + 2) // 6
    xu = [bary_to_x(l, V) for l in simplex_rule(D, nu)[0]]
    int_u, int_dir = [], []
    for u in range(len(xu)):
        for d in range(D):
            int_u.append(u); int_dir.append(d)
    return RefElement(etype, p, D, xsol, xext, nrm, fid, D + 1, nfp, xu, int_u, int_dir, fnorms,
                      [f * nfp for f in range(D + 2)])


def _prism(p):
    """Triangular prism (App. A l.2633-2737): reference x, y >= -1, x + y <= 0,
    z in [-1, 1].  Solution points: the triangle's solution points x (p+1) GL levels in z
    (l.2731-2733).  External flux points: faces 0 (z = -1) and 1 (z = +1) carry the
    triangle rule of (p+1)(p+2)/2 points (the tet-face rule of reading O1), faces 2 (y = -1),
    3 (x + y = 0), 4 (x = -1) the (p+1)^2 GL points (edge GL x GL in z; l.2718-2720).
    Internal flux points (l.2723-2729): set 1 = the triangle's interior rule x (p+1) GL
    levels, two DOFs each (normals e_x, e_y); set 2 = the triangle-face rule x the p zeros
    of P_p in z (reading O3 as for tensor elements), one DOF (e_z).  Orders: z level
    slowest, triangle point fastest; internal points set 1 then set 2, each unique point's
    DOFs in axis order."""
    V = [tuple(mp.mpf(c) for c in v) for v in TRI_V]
    g, _ = gauss_legendre(p + 1)
    z, _ = gauss_legendre(p) if p >= 1 else ((), ())
    tri_sol = [bary_to_x(l, V) for l in lattice(2, p)]
    xsol = [(x[0], x[1], zz) for zz in g for x in tri_sol]
    s2 = 1 / mp.sqrt(2)
    z0 = mp.mpf(0)
    fnorms = [(z0, z0, mp.mpf(-1)), (z0, z0, mp.mpf(1)), (z0, mp.mpf(-1), z0), (s2, s2, z0), (mp.mpf(-1), z0, z0)]
    tface = [bary_to_x(l, V) for l in simplex_rule(2, (p + 1) * (p + 2) // 2)[0]]
    xext, nrm, fid, fptr = [], [], [], [0]
    for f, zz in ((0, mp.mpf(-1)), (1, mp.mpf(1))):
        for x in tface:
            xext.append((x[0], x[1], zz)); nrm.append(fnorms[f]); fid.append(f)
        fptr.append(len(xext))
    for f, (a, b) in zip((2, 3, 4), TRI_FACES):
        for zz in g:
            for t in g:
                lam = (t + 1) / 2
                xext.append(tuple(V[a][c] + lam * (V[b][c] - V[a][c]) for c in range(2)) + (zz,))
                nrm.append(fnorms[f]); fid.append(f)
        fptr.append(len(xext))
    tint = [bary_to_x(l, V) for l in simplex_rule(2, p * (p + 1) // 2)[0]] if p >= 1 else []
    xu, int_u, int_dir = [], [], []
    for zz in g:                       # set 1: 2-D normals
        for x in tint:
            for d in range(2):
                int_u.append(len(xu)); int_dir.append(d)
            xu.append((x[0], x[1], zz))
    for zz in z:                       # set 2: z normal
        for x in tface:
            int_u.append(len(xu)); int_dir.append(2)
            xu.append((x[0], x[1], zz))
    return RefElement("pri", p, 3, xsol, xext, nrm, fid, 5, (p + 1) ** 2, xu, int_u, int_dir, fnorms, fptr)


@lru_cache(maxsize=None)
def reference_element(etype, p):
    if p < 1 or p > 4 or (etype in ("tet", "pri") and p > 3):
        raise ValueError("unsupported degree: quad/hex/tri p in [1,4], tet/pri p in [1,3]")
    if etype in ("quad", "hex"):
        return _tensor(etype, p)
    if etype in ("tri", "tet"):
        return _simplex(etype, p)
    if etype == "pri":
        return _prism(p)
    raise ValueError(etype)
