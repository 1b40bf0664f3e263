"""Uniform periodic meshes, affine maps and face pairing (oracle; test infrastructure only).

PAPER.md §2 l.145-172 (tessellation, mapping x = M_en(x~), Jacobian J, det J, J^-1),
§3 l.497-519 (uniform meshes by sub-dividing tensor cells into N_p simplices:
N_p = 1 tensor, 2 triangles, 6 tetrahedra).  Face pairing is done the plain way:
by brute-force coordinate matching of external flux points across periodic wraps
(SPEC S:206); the face point permutation is read off the matched coordinates.

Conventions:
  * pattern (i, j[, k]) with x fastest; element id = pattern * N_p + s;
  * tri: s=0 (0,0),(1,0),(1,1); s=1 (0,0),(1,1),(0,1)  (diagonal (0,0)->(1,1));
  * tet: Kuhn split, s = index of the permutation pi of (0,1,2) in lexicographic
    order; vertices 0, e_pi0, e_pi0+e_pi1, (1,1,1); if det < 0 the 2nd and 3rd
    vertices are swapped (det J > 0 everywhere);
  * x = P0 + J (x~ - V0), J[:, k] = (P_{k+1} - P0)/2 (simplex) or diag(h/2) (tensor);
  * left/right (reading O14): the LEFT element of a face is the one whose physical
    outward unit normal has its first non-zero component (|.| > 1e-12) positive;
  * faces are listed sorted by (left element, left local face); perm[q] is the
    right element's local face-point index matching the left's local point q.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np

from .operators import build_operators

TRI_SUB = [((0, 0), (1, 0), (1, 1)), ((0, 0), (1, 1), (0, 1))]


def tet_subcells():
    out = []
    for perm in itertools.permutations(range(3)):
        e = np.eye(3)
        P = [np.zeros(3), e[perm[0]], e[perm[0]] + e[perm[1]], np.ones(3)]
        if np.linalg.det(np.array([P[1] - P[0], P[2] - P[0], P[3] - P[0]]).T) < 0:
            P[1], P[2] = P[2], P[1]
        out.append([tuple(v) for v in P])
    return out


def subcell_vertices(etype):
    if etype == "tri":
        return [list(map(np.array, s)) for s in TRI_SUB]
    if etype == "pri":
        # the triangle split extruded in z: images of the reference vertices V0, V1, V2
        # (z = -1) and of V0 at z = +1 (N_p = 2 prisms per hexahedron)
        return [[np.array(v + (0,)) for v in s] + [np.array(s[0] + (1,))] for s in TRI_SUB]
    if etype == "tet":
        return [list(map(np.array, s)) for s in tet_subcells()]
    return None


@dataclass
class Mesh:
    etype: str
    p: int
    nd: int
    N: tuple            # patterns per axis
    lo: np.ndarray
    hi: np.ndarray
    h: np.ndarray       # pattern edge per axis
    K: int              # elements
    nsub: int
    J: np.ndarray       # K x D x D
    detJ: np.ndarray    # K
    Jinv: np.ndarray    # K x D x D
    x0: np.ndarray      # K x D, image of reference vertex V0 = (-1,...,-1)
    # face list (sorted by left element, left local face)
    face_elem: np.ndarray   # F x 2 (left, right) int32
    face_lface: np.ndarray  # F x 2 int8
    face_perm: np.ndarray   # F x nfp int16
    # per element / external point
    is_left: np.ndarray     # K x nfaces bool
    nbr_elem: np.ndarray    # N_ext x K  neighbour element of each external point
    nbr_pt: np.ndarray      # N_ext x K  matching external point index in the neighbour
    periodic: tuple = ()    # per axis; False: far-field boundaries (faces with a -1 side)

    def sol_coords(self):
        """Physical coordinates of solution points, shape (N_sol, D, K) (reading O21)."""
        ops = build_operators(self.etype, self.p)
        xr = ops.xsol + 1.0  # x~ - V0
        return np.einsum("kij,sj->sik", self.J, xr) + self.x0.T[None, :, :]

    def ext_coords(self):
        ops = build_operators(self.etype, self.p)
        xr = ops.xext + 1.0
        return np.einsum("kij,sj->sik", self.J, xr) + self.x0.T[None, :, :]


def build_mesh(etype, p, N, lo, hi, periodic=None):
    """periodic[d] = 0: far-field boundaries at x_d = lo, hi: faces there
    have no partner; they are listed with -1 for the missing (exterior) side."""
    ops = build_operators(etype, p)
    D = ops.nd
    N = tuple(int(n) for n in (N if np.ndim(N) else [N] * D))
    lo = np.asarray(lo, dtype=np.float64)[:D]
    hi = np.asarray(hi, dtype=np.float64)[:D]
    h = (hi - lo) / np.array(N)
    sub = subcell_vertices(etype)
    nsub = 1 if sub is None else len(sub)
    npat = int(np.prod(N))
    K = npat * nsub
    J = np.zeros((K, D, D))
    x0 = np.zeros((K, D))
    for pat in range(npat):
        idx = []
        r = pat
        for d in range(D):
            idx.append(r % N[d])
            r //= N[d]
        origin = lo + h * np.array(idx)
        for s in range(nsub):
            e = pat * nsub + s
            if sub is None:
                J[e] = np.diag(h / 2.0)
                x0[e] = origin
            else:
                P = [origin + h * v for v in sub[s]]
                for k in range(D):
                    J[e][:, k] = (P[k + 1] - P[0]) / 2.0
                x0[e] = P[0]
    detJ = np.linalg.det(J)
    if np.any(detJ <= 0):
        raise ValueError("non-positive det J")
    Jinv = np.linalg.inv(J)
    # ---------------------------------------------------------------- face pairing
    per = np.ones(D, dtype=bool) if periodic is None else np.asarray(periodic[:D], dtype=bool)
    L = hi - lo
    xr = ops.xext + 1.0
    xe = np.einsum("kij,sj->ksi", J, xr) + x0[:, None, :]     # K x N_ext x D
    nf, nfp = ops.nfaces, ops.nfp                              # nfp: largest face
    fp = np.asarray(ops.face_ptr, dtype=np.int64)              # face f: points fp[f]..fp[f+1]
    nq = np.diff(fp)
    # face points padded to nfp (NaN beyond a face's own count: prisms mix face types)
    xe = np.stack([np.concatenate([xe[:, fp[f]:fp[f + 1]], np.full((K, nfp - nq[f], D), np.nan)], axis=1)
                   for f in range(nf)], axis=1)                # K x nf x nfp x D
    tol = 1e-9 * float(np.min(h))
    # face key: centroid wrapped into the periodic box (periodic axes only), rounded
    cen = np.nanmean(xe, axis=2)
    cen = np.where(per, np.mod(cen - lo + 0.5 * tol, L) - 0.5 * tol, cen - lo)
    key = np.round(cen / (1e-6 * float(np.min(h)))).astype(np.int64).reshape(K * nf, D)
    order = np.lexsort(key.T[::-1])
    ks = key[order]
    # group equal keys: interior faces come in pairs, far-field boundary faces alone
    partner = np.full(K * nf, -1, dtype=np.int64)
    i = 0
    while i < len(order):
        j = i + 1
        while j < len(order) and np.all(ks[j] == ks[i]):
            j += 1
        if j - i == 2:
            partner[order[i]], partner[order[i + 1]] = order[i + 1], order[i]
        elif j - i != 1:
            raise ValueError("face pairing failed: a face centroid is shared by more than 2 faces")
        i = j
    cflat = cen.reshape(K * nf, D)
    lone = np.nonzero(partner < 0)[0]
    on_ff = np.zeros(len(lone), dtype=bool)
    for d in range(D):
        if not per[d]:
            on_ff |= (np.abs(cflat[lone, d]) < tol) | (np.abs(cflat[lone, d] - L[d]) < tol)
    if not np.all(on_ff):
        raise ValueError("face pairing failed: an unpaired face is not on a far-field boundary")
    # outward physical unit normals: n = J^-T n~ / |J^-T n~|
    fn = ops.face_normals
    nphys = np.einsum("kji,fj->kfi", Jinv, fn)
    nphys /= np.linalg.norm(nphys, axis=2, keepdims=True)
    # left rule O14: first component with |.| > 1e-12 is positive
    nz = np.abs(nphys) > 1e-12
    first = np.argmax(nz, axis=2)
    is_left = np.take_along_axis(nphys, first[..., None], axis=2)[..., 0] > 0
    flat_left = is_left.reshape(K * nf)
    paired = partner >= 0
    if np.any(flat_left[paired] == flat_left[partner[paired]]):
        raise ValueError("left/right rule is not antisymmetric")
    # face point permutation by coordinate matching (mod periodic box)
    xf = xe.reshape(K * nf, nfp, D)
    pt = np.where(paired, partner, np.arange(K * nf))
    d = xf[pt][:, None, :, :] - xf[:, :, None, :]              # [face, q, q', D]
    d = d - np.where(per, L * np.round(d / L), 0.0)
    dist = np.nan_to_num(np.max(np.abs(d), axis=3), nan=np.inf)
    perm_all = np.argmin(dist, axis=2)                         # [face, q] -> q'
    valid = np.arange(nfp)[None, :] < np.tile(nq, K)[:, None]  # real points of each face
    if np.any((np.take_along_axis(dist, perm_all[..., None], axis=2)[..., 0] > tol) & valid & paired[:, None]):
        raise ValueError("face point matching failed")
    perm_all[~paired] = -1
    perm_all[~valid] = -1
    pe = np.where(paired, partner // nf, -1)
    pf = np.where(paired, partner % nf, -1)
    # per external point of each element: neighbour element and its matching point
    nbr_elem = np.full((ops.next, K), -1, dtype=np.int64)
    nbr_pt = np.full((ops.next, K), -1, dtype=np.int64)
    pe2, pf2, pa2 = pe.reshape(K, nf), pf.reshape(K, nf), perm_all.reshape(K, nf, nfp)
    for f in range(nf):
        for q in range(nq[f]):
            nbr_elem[fp[f] + q] = pe2[:, f]
            nbr_pt[fp[f] + q] = np.where(pa2[:, f, q] < 0, -1, fp[np.maximum(pf2[:, f], 0)] + pa2[:, f, q])
    # faces in (element, local face) scan order: those whose left element this is, and
    # far-field faces (exterior side -1, listed from the interior element)
    lidx = np.nonzero(flat_left | ~paired)[0]
    F = len(lidx)
    me, mf = lidx // nf, lidx % nf
    lft = flat_left[lidx]
    face_elem = np.stack([np.where(lft, me, -1), np.where(lft, pe[lidx], me)], axis=1).astype(np.int32)
    face_lface = np.stack([np.where(lft, mf, -1), np.where(lft, pf[lidx], mf)], axis=1).astype(np.int8)
    face_perm = perm_all[lidx].astype(np.int16).reshape(F, nfp)
    return Mesh(etype, p, D, N, lo, hi, h, K, nsub, J, detJ, Jinv, x0,
                face_elem, face_lface, face_perm, is_left, nbr_elem, nbr_pt, tuple(bool(x) for x in per))
