// Uniform periodic pattern meshes: sub-cell shapes, affine maps, and the
// translation-invariant face connectivity of each (shape, face), derived by exact
// integer matching of face vertex sets in a 3^D block of patterns.
// PAPER.md §2 l.145-172 (mapping, Jacobians), §3 l.497-519 (sub-division into N_p
// cells), SPEC S:206 (face point permutation by coordinate matching).
// Conventions: element id = pattern * N_p + s, pattern x fastest;
// tri s0 = (0,0),(1,0),(1,1), s1 = (0,0),(1,1),(0,1); tet = Kuhn split, shapes in
// lexicographic order of the axis permutation, vertices 0, e_a, e_a+e_b, (1,1,1),
// with vertices 1 and 2 swapped when the determinant is negative.
#include "mesh.h"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace sdrt {

typedef std::array<int, 3> I3;

static std::vector<std::vector<I3>> subcells(int etype) {
  std::vector<std::vector<I3>> out;
  if (etype == TRI) {
    out.push_back({I3{0, 0, 0}, I3{1, 0, 0}, I3{1, 1, 0}});
    out.push_back({I3{0, 0, 0}, I3{1, 1, 0}, I3{0, 1, 0}});
  } else if (etype == PRI) {
    // the triangle split extruded in z: images of the prism's reference vertices
    // V0 V1 V2 (z = -1) then V3 V4 V5 (z = +1)  (N_p = 2)
    out.push_back({I3{0, 0, 0}, I3{1, 0, 0}, I3{1, 1, 0}, I3{0, 0, 1}, I3{1, 0, 1}, I3{1, 1, 1}});
    out.push_back({I3{0, 0, 0}, I3{1, 1, 0}, I3{0, 1, 0}, I3{0, 0, 1}, I3{1, 1, 1}, I3{0, 1, 1}});
  } else if (etype == TET) {
    int perm[3] = {0, 1, 2};
    do {
      I3 e0 = {0, 0, 0}, e1 = {0, 0, 0};
      e0[perm[0]] = 1;
      e1 = e0;
      e1[perm[1]] = 1;
      std::vector<I3> P = {I3{0, 0, 0}, e0, e1, I3{1, 1, 1}};
      int a[3][3];
      for (int k = 0; k < 3; ++k)
        for (int c = 0; c < 3; ++c) a[c][k] = P[k + 1][c] - P[0][c];
      int det = a[0][0] * (a[1][1] * a[2][2] - a[1][2] * a[2][1]) -
                a[0][1] * (a[1][0] * a[2][2] - a[1][2] * a[2][0]) +
                a[0][2] * (a[1][0] * a[2][1] - a[1][1] * a[2][0]);
      if (det < 0) std::swap(P[1], P[2]);
      out.push_back(P);
    } while (std::next_permutation(perm, perm + 3));
  }
  return out;
}

// unit-cube integer corner set of a face
static std::vector<I3> face_vertices(int etype, int nd, const std::vector<I3>& P, const RefElement& r,
                                     int f) {
  std::vector<I3> v;
  if (etype_tensor(etype)) {
    int d = f / 2, side = f % 2;
    int nc = 1 << nd;
    for (int m = 0; m < nc; ++m) {
      I3 c = {0, 0, 0};
      for (int k = 0; k < nd; ++k) c[k] = (m >> k) & 1;
      if (c[d] == side) v.push_back(c);
    }
  } else {
    for (int vid : r.face_verts[f]) v.push_back(P[vid]);
  }
  std::sort(v.begin(), v.end());
  return v;
}

void Mesh::gcoords(int64_t e, int c[3]) const {
  int64_t pat = e / nsub;
  int l[3] = {0, 0, 0};
  for (int d = 0; d < nd; ++d) {
    l[d] = (int)(pat % Nloc[d]);
    pat /= Nloc[d];
  }
  for (int d = 0; d < 3; ++d) c[d] = d < nd ? l[d] + offset[d] : 0;
}

int64_t Mesh::global_id(int64_t e) const {
  int c[3];
  gcoords(e, c);
  int64_t g = 0, mul = 1;
  for (int d = 0; d < nd; ++d) {
    g += mul * c[d];
    mul *= Nglob[d];
  }
  return g * nsub + e % nsub;
}

Mesh build_mesh(int etype, int p, const int N[3], const double lo[3], const double hi[3], int rank,
                int nranks, const int pgrid[3], const int periodic[3]) {
  Mesh m;
  for (int d = 0; d < 3; ++d) m.periodic[d] = (periodic && d < etype_dim(etype)) ? (periodic[d] != 0) : 1;
  m.etype = etype;
  m.p = p;
  m.nd = etype_dim(etype);
  m.nsub = etype_nsub(etype);
  m.ref = build_reference(etype, p);
  m.rank = rank;
  m.nranks = nranks;
  int D = m.nd;
  int pg[3] = {1, 1, 1};
  if (pgrid)
    for (int d = 0; d < D; ++d) pg[d] = pgrid[d];
  int prod = 1;
  for (int d = 0; d < D; ++d) prod *= pg[d];
  if (prod != nranks || rank < 0 || rank >= nranks) throw std::invalid_argument("bad rank / pgrid");
  int rc[3] = {rank % pg[0], (rank / pg[0]) % pg[1], D == 3 ? rank / (pg[0] * pg[1]) : 0};
  for (int d = 0; d < 3; ++d) {
    m.pgrid[d] = d < D ? pg[d] : 1;
    if (d < D) {
      if (N[d] < 3) throw std::invalid_argument("N >= 3 patterns per axis required (periodic)");
      if (N[d] % pg[d]) throw std::invalid_argument("pgrid must divide N");
      if (!(hi[d] > lo[d])) throw std::invalid_argument("hi must exceed lo");
      m.Nglob[d] = N[d];
      m.Nloc[d] = N[d] / pg[d];
      m.offset[d] = rc[d] * m.Nloc[d];
      m.lo[d] = lo[d];
      m.hi[d] = hi[d];
      m.h[d] = (hi[d] - lo[d]) / N[d];
    } else {
      m.Nglob[d] = m.Nloc[d] = 1;
      m.offset[d] = 0;
      m.lo[d] = 0;
      m.hi[d] = 1;
      m.h[d] = 1;
    }
  }
  int64_t npat = 1;
  for (int d = 0; d < D; ++d) npat *= m.Nloc[d];
  m.K = npat * m.nsub;
  m.K_pad = (m.K + 31) / 32 * 32;

  const RefElement& r = m.ref;
  auto sc = subcells(etype);
  // ---- affine maps per shape: x = x0 + J (x~ - V0)
  m.J.assign(m.nsub, {});
  m.Jinv.assign(m.nsub, {});
  m.detJ.assign(m.nsub, 0.0);
  m.P0.assign(m.nsub, {0, 0, 0});
  std::vector<std::array<double, 9>> Ju(m.nsub);  // unit-cube Jacobian (h = 1)
  for (int s = 0; s < m.nsub; ++s) {
    double A[3][3] = {{0}}, Au[3][3] = {{0}};
    if (etype_tensor(etype)) {
      for (int d = 0; d < D; ++d) { A[d][d] = m.h[d] / 2; Au[d][d] = 0.5; }
    } else {
      // simplex: columns V_{k+1} - V0; prism: V1 - V0, V2 - V0, V3 - V0 (the same slots)
      for (int k = 0; k < D; ++k)
        for (int c = 0; c < D; ++c) {
          Au[c][k] = (sc[s][k + 1][c] - sc[s][0][c]) / 2.0;
          A[c][k] = Au[c][k] * m.h[c];
        }
      for (int c = 0; c < D; ++c) m.P0[s][c] = sc[s][0][c];
    }
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        m.J[s][i * 3 + j] = A[i][j];
        Ju[s][i * 3 + j] = Au[i][j];
      }
    double det, inv[3][3] = {{0}};
    if (D == 2) {
      det = A[0][0] * A[1][1] - A[0][1] * A[1][0];
      inv[0][0] = A[1][1] / det; inv[0][1] = -A[0][1] / det;
      inv[1][0] = -A[1][0] / det; inv[1][1] = A[0][0] / det;
    } else {
      det = A[0][0] * (A[1][1] * A[2][2] - A[1][2] * A[2][1]) -
            A[0][1] * (A[1][0] * A[2][2] - A[1][2] * A[2][0]) +
            A[0][2] * (A[1][0] * A[2][1] - A[1][1] * A[2][0]);
      inv[0][0] = (A[1][1] * A[2][2] - A[1][2] * A[2][1]) / det;
      inv[0][1] = (A[0][2] * A[2][1] - A[0][1] * A[2][2]) / det;
      inv[0][2] = (A[0][1] * A[1][2] - A[0][2] * A[1][1]) / det;
      inv[1][0] = (A[1][2] * A[2][0] - A[1][0] * A[2][2]) / det;
      inv[1][1] = (A[0][0] * A[2][2] - A[0][2] * A[2][0]) / det;
      inv[1][2] = (A[0][2] * A[1][0] - A[0][0] * A[1][2]) / det;
      inv[2][0] = (A[1][0] * A[2][1] - A[1][1] * A[2][0]) / det;
      inv[2][1] = (A[0][1] * A[2][0] - A[0][0] * A[2][1]) / det;
      inv[2][2] = (A[0][0] * A[1][1] - A[0][1] * A[1][0]) / det;
    }
    if (!(det > 0)) throw std::runtime_error("non-positive det J");
    m.detJ[s] = det;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) m.Jinv[s][i * 3 + j] = inv[i][j];
  }
  // ---- unit-cube positions of external flux points per shape
  auto ext_pos = [&](int s, int e) {
    std::array<double, 3> x = {0, 0, 0};
    for (int c = 0; c < D; ++c) {
      double v = m.P0[s][c];
      for (int k = 0; k < D; ++k) v += Ju[s][c * 3 + k] * (r.xext[e][k] + 1.0);
      x[c] = v;
    }
    return x;
  };
  // ---- connectivity per (shape, face) by exact vertex-set matching
  m.link.assign(m.nsub * r.nfaces, {});
  int span = 1;
  for (int d = 0; d < D; ++d) span *= 3;
  for (int s = 0; s < m.nsub; ++s)
    for (int f = 0; f < r.nfaces; ++f) {
      auto mine = face_vertices(etype, D, sc.empty() ? std::vector<I3>() : sc[s], r, f);
      int found = 0;
      FaceLink L;
      for (int oi = 0; oi < span; ++oi) {
        int o[3] = {0, 0, 0}, t = oi;
        for (int d = 0; d < D; ++d) { o[d] = t % 3 - 1; t /= 3; }
        for (int s2 = 0; s2 < m.nsub; ++s2)
          for (int f2 = 0; f2 < r.nfaces; ++f2) {
            if (o[0] == 0 && o[1] == 0 && o[2] == 0 && s2 == s && f2 == f) continue;
            auto other = face_vertices(etype, D, sc.empty() ? std::vector<I3>() : sc[s2], r, f2);
            for (auto& v : other)
              for (int d = 0; d < 3; ++d) v[d] += o[d];
            std::sort(other.begin(), other.end());
            if (other == mine) {
              ++found;
              L.off[0] = o[0]; L.off[1] = o[1]; L.off[2] = o[2];
              L.nshape = s2;
              L.nface = f2;
            }
          }
      }
      if (found != 1) throw std::runtime_error("face pairing failed");
      if ((L.off[0] != 0) + (L.off[1] != 0) + (L.off[2] != 0) > 1)
        throw std::runtime_error("internal: face neighbour differs in more than one pattern axis");
      // left rule O14 from the integer outward normal of this face
      int nrm[3] = {0, 0, 0};
      if (etype_tensor(etype)) {
        nrm[f / 2] = (f % 2) ? 1 : -1;
      } else {
        const std::vector<I3>& P = sc[s];
        const auto& fv = r.face_verts[f];
        int opp = -1;  // a vertex of the element off this face
        for (int k = 0; k < (int)P.size(); ++k)
          if (opp < 0 && std::find(fv.begin(), fv.end(), k) == fv.end()) opp = k;
        if (D == 2) {
          I3 a = P[fv[0]], b = P[fv[1]];
          nrm[0] = b[1] - a[1];
          nrm[1] = -(b[0] - a[0]);
        } else {
          I3 a = P[fv[0]], b = P[fv[1]], c = P[fv[2]];
          int u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
          int v[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
          nrm[0] = u[1] * v[2] - u[2] * v[1];
          nrm[1] = u[2] * v[0] - u[0] * v[2];
          nrm[2] = u[0] * v[1] - u[1] * v[0];
        }
        int dot = 0;
        for (int c = 0; c < D; ++c) dot += nrm[c] * (P[fv[0]][c] - P[opp][c]);
        if (dot < 0)
          for (int c = 0; c < 3; ++c) nrm[c] = -nrm[c];
      }
      L.left = 0;
      for (int c = 0; c < D; ++c)
        if (nrm[c] != 0) { L.left = nrm[c] > 0; break; }
      // face point permutation by coordinate matching (unit cube, tol 1e-9)
      const int nq = r.face_nfp(f);
      if (r.face_nfp(L.nface) != nq) throw std::runtime_error("face pairing failed: face sizes differ");
      L.perm.assign(nq, -1);
      for (int q = 0; q < nq; ++q) {
        auto x = ext_pos(s, r.face_ptr[f] + q);
        double best = 1e30;
        for (int q2 = 0; q2 < nq; ++q2) {
          auto y = ext_pos(L.nshape, r.face_ptr[L.nface] + q2);
          double dist = 0;
          for (int c = 0; c < D; ++c) dist = std::max(dist, std::fabs(y[c] + L.off[c] - x[c]));
          if (dist < best) { best = dist; L.perm[q] = q2; }
        }
        if (best > 1e-9) throw std::runtime_error("face point matching failed");
      }
      m.link[s * r.nfaces + f] = L;
    }
  for (int s = 0; s < m.nsub; ++s)
    for (int f = 0; f < r.nfaces; ++f) {
      const FaceLink& L = m.link[s * r.nfaces + f];
      if (L.left == m.link[L.nshape * r.nfaces + L.nface].left)
        throw std::runtime_error("left/right rule not antisymmetric");
    }
  // ---- metric terms per (shape, ext point): s = detJ |J^-T n~|, canonical normal
  m.sscale.assign(m.nsub * r.next, 0.0);
  m.nleft.assign(m.nsub * r.next, {0, 0, 0});
  std::vector<std::array<double, 3>> nown(m.nsub * r.nfaces);
  for (int s = 0; s < m.nsub; ++s)
    for (int f = 0; f < r.nfaces; ++f) {
      double jn[3] = {0, 0, 0}, nn = 0;
      for (int i = 0; i < D; ++i) {
        for (int j = 0; j < D; ++j) jn[i] += m.Jinv[s][j * 3 + i] * r.face_normal[f][j];
        nn += jn[i] * jn[i];
      }
      nn = std::sqrt(nn);
      for (int i = 0; i < 3; ++i) nown[s * r.nfaces + f][i] = jn[i] / nn;
      for (int q = 0; q < r.face_nfp(f); ++q) m.sscale[s * r.next + r.face_ptr[f] + q] = m.detJ[s] * nn;
    }
  for (int s = 0; s < m.nsub; ++s)
    for (int f = 0; f < r.nfaces; ++f) {
      const FaceLink& L = m.link[s * r.nfaces + f];
      auto n = L.left ? nown[s * r.nfaces + f] : nown[L.nshape * r.nfaces + L.nface];
      for (int q = 0; q < r.face_nfp(f); ++q) m.nleft[s * r.next + r.face_ptr[f] + q] = n;
    }
  build_halo(m, false);
  return m;
}

void build_halo(Mesh& m, bool force_self_halo) {
  const RefElement& r = m.ref;
  const int D = m.nd;
  m.slabs.clear();
  int64_t cur = m.K_pad;
  m.ff_row.clear();
  m.ff_col.clear();
  for (int d = 0; d < 3; ++d) {
    // ghost columns on partition axes, loopback axes and far-field (non-periodic) axes
    m.halo[d] = d < D && (m.pgrid[d] > 1 || force_self_halo || !m.periodic[d]);
    for (int side = 0; side < 2; ++side) m.gbase[d][side] = 0;
  }
  for (int d = 0; d < D; ++d) {
    if (!m.halo[d]) continue;
    int64_t tang = 1;
    for (int c = 0; c < D; ++c)
      if (c != d) tang *= m.Nloc[c];
    for (int side = 0; side < 2; ++side) {
      m.gbase[d][side] = cur;
      cur += tang * m.nsub;
    }
  }
  m.Kt = (cur + 31) / 32 * 32;
  // rank coordinates and peers
  int rc[3] = {m.rank % m.pgrid[0], (m.rank / m.pgrid[0]) % m.pgrid[1], m.rank / (m.pgrid[0] * m.pgrid[1])};
  auto rank_of = [&](const int c[3]) { return c[0] + m.pgrid[0] * (c[1] + m.pgrid[1] * c[2]); };
  for (int d = 0; d < D; ++d) {
    if (!m.halo[d]) continue;
    int oth[2], no = 0;
    for (int c = 0; c < D; ++c)
      if (c != d) oth[no++] = c;
    for (int side = 0; side < 2; ++side) {
      HaloSlab S;
      S.d = d;
      S.side = side;
      int pc[3] = {rc[0], rc[1], rc[2]};
      pc[d] += side ? 1 : -1;
      // a far-field side: the block's face lies on a non-periodic domain boundary
      const bool farfield = !m.periodic[d] && (pc[d] < 0 || pc[d] >= m.pgrid[d]);
      pc[d] = (pc[d] + m.pgrid[d]) % m.pgrid[d];
      S.peer = rank_of(pc);
      const int dir = side ? 1 : -1;
      // my boundary layer facing `side`, and my ghost slab on `side` (the peer's layer)
      const int my_layer = side ? m.Nloc[d] - 1 : 0;
      int na = no > 0 ? m.Nloc[oth[0]] : 1, nb = no > 1 ? m.Nloc[oth[1]] : 1;
      for (int tb = 0; tb < nb; ++tb)
        for (int ta = 0; ta < na; ++ta) {
          int lc[3] = {0, 0, 0};
          lc[d] = my_layer;
          if (no > 0) lc[oth[0]] = ta;
          if (no > 1) lc[oth[1]] = tb;
          int64_t lp = lc[0] + (int64_t)m.Nloc[0] * (lc[1] + (int64_t)m.Nloc[1] * lc[2]);
          int64_t tang = ta + (int64_t)na * tb;
          for (int s = 0; s < m.nsub; ++s)
            for (int f = 0; f < r.nfaces; ++f) {
              const FaceLink& L = m.link[s * r.nfaces + f];
              bool facing = L.off[d] == dir;
              for (int c = 0; c < D; ++c)
                if (c != d && L.off[c] != 0) facing = false;
              if (facing)
                for (int q = 0; q < r.face_nfp(f); ++q) {
                  S.send_row.push_back(r.face_ptr[f] + q);
                  S.send_col.push_back((int32_t)(lp * m.nsub + s));
                }
              // the peer's element across MY `side` sends its faces facing -dir;
              // store them in my ghost column for that element
              bool facing_back = L.off[d] == -dir;
              for (int c = 0; c < D; ++c)
                if (c != d && L.off[c] != 0) facing_back = false;
              if (facing_back)
                for (int q = 0; q < r.face_nfp(f); ++q) {
                  S.recv_row.push_back(r.face_ptr[f] + q);
                  S.recv_col.push_back((int32_t)(m.gbase[d][side] + tang * m.nsub + s));
                }
            }
        }
      if (farfield) {  // nothing to exchange: the ghost entries are filled with the far field
        m.ff_row.insert(m.ff_row.end(), S.recv_row.begin(), S.recv_row.end());
        m.ff_col.insert(m.ff_col.end(), S.recv_col.begin(), S.recv_col.end());
        continue;
      }
      m.slabs.push_back(S);
    }
  }
}

}  // namespace sdrt
