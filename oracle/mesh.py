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

    def sol_coords(self):
        """Physical coordinates of solution points, shape (N_sol, D, K) (reading O21)."""
        ops = build_operators(self.etype, self.p)
        xr = ops.xsol + 1.0  # x~ - V0
        return np.einsum("kij,sj->sik", self.J, xr) + self.x0.T[None, :, :]

    def ext_coords(self):
        ops = build_operators(self.etype, self.p)
        xr = ops.xext + 1.0
        return np.einsum("kij,sj->sik", self.J, xr) + self.x0.T[None, :, :]


def build_mesh(etype, p, N, lo, hi):
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
    L = hi - lo
    xr = ops.xext + 1.0
    xe = np.einsum("kij,sj->ksi", J, xr) + x0[:, None, :]     # K x N_ext x D
    nf, nfp = ops.nfaces, ops.nfp
    xe = xe.reshape(K, nf, nfp, D)
    tol = 1e-9 * float(np.min(h))
    # face key: centroid wrapped into the periodic box, rounded
    cen = xe.mean(axis=2)
    cen = np.mod(cen - lo + 0.5 * tol, L) - 0.5 * tol
    key = np.round(cen / (1e-6 * float(np.min(h)))).astype(np.int64).reshape(K * nf, D)
    order = np.lexsort(key.T[::-1])
    ks = key[order]
    same_next = np.all(ks[1:] == ks[:-1], axis=1)
    # every key must occur exactly twice: pairs are (order[2i], order[2i+1])
    if len(order) % 2 or not np.all(same_next[0::2]) or np.any(same_next[1::2]):
        raise ValueError("face pairing failed: a face centroid is not shared by exactly 2 faces")
    A, B = order[0::2], order[1::2]
    partner = np.empty(K * nf, dtype=np.int64)
    partner[A] = B
    partner[B] = A
    # outward physical unit normals: n = J^-T n~ / |J^-T n~|
    fn = ops.face_normals
    nphys = np.einsum("kji,fj->kfi", Jinv, fn)
    nphys /= np.linalg.norm(nphys, axis=2, keepdims=True)
    # left rule O14: first component with |.| > 1e-12 is positive
    nz = np.abs(nphys) > 1e-12
    first = np.argmax(nz, axis=2)
    is_left = np.take_along_axis(nphys, first[..., None], axis=2)[..., 0] > 0
    flat_left = is_left.reshape(K * nf)
    if np.any(flat_left == flat_left[partner]):
        raise ValueError("left/right rule is not antisymmetric")
    # face point permutation by coordinate matching (mod periodic box)
    xf = xe.reshape(K * nf, nfp, D)
    d = xf[partner][:, None, :, :] - xf[:, :, None, :]        # [face, q, q', D]
    d = d - L * np.round(d / L)
    dist = np.max(np.abs(d), axis=3)
    perm_all = np.argmin(dist, axis=2)                         # [face, q] -> q'
    if np.any(np.take_along_axis(dist, perm_all[..., None], axis=2) > tol):
        raise ValueError("face point matching failed")
    pe, pf = partner // nf, partner % nf
    nbr_elem = np.repeat(pe.reshape(K, nf), nfp, axis=1).T.copy()          # N_ext x K
    nbr_pt = (pf.reshape(K, nf, 1) * nfp + perm_all.reshape(K, nf, nfp)).reshape(K, nf * nfp).T.copy()
    lidx = np.nonzero(flat_left)[0]                                        # sorted (e, f)
    F = len(lidx)
    face_elem = np.stack([lidx // nf, pe[lidx]], axis=1).astype(np.int32)
    face_lface = np.stack([lidx % nf, pf[lidx]], axis=1).astype(np.int8)
    face_perm = perm_all[lidx].astype(np.int16).reshape(F, nfp)
    return Mesh(etype, p, D, N, lo, hi, h, K, nsub, J, detJ, Jinv, x0,
                face_elem, face_lface, face_perm, is_left, nbr_elem, nbr_pt)
