// C ABI: meshes and operators (host only).  See include/sdrt.h.
#include <cstring>
#include <stdexcept>

#include "capi_internal.h"

namespace sdrt {
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
}  // namespace sdrt

extern "C" {

int sdrt_abi_version(void) { return SDRT_ABI_VERSION; }
const char* sdrt_last_error(void) { return sdrt::g_err.c_str(); }

sdrt_status sdrt_mesh_create(int etype, int p, const int N[3], const double lo[3], const double hi[3],
                             const int periodic[3], int rank, int nranks, const int pgrid[3],
                             sdrt_mesh** out) {
  if (!out || !N || !lo || !hi) {
    sdrt::set_error("null argument");
    return SDRT_E_INVALID_ARG;
  }
  if (etype < 0 || etype > 4) {
    sdrt::set_error("unsupported element type");
    return SDRT_E_UNSUPPORTED;
  }
  SDRT_TRY({
    auto* m = new sdrt_mesh;
    try {
      m->m = sdrt::build_mesh(etype, p, N, lo, hi, rank, nranks, pgrid, periodic);
    } catch (...) {
      delete m;
      throw;
    }
    *out = m;
    return SDRT_OK;
  })
}

sdrt_status sdrt_mesh_info(const sdrt_mesh* mm, sdrt_mesh_info_t* out) {
  if (!mm || !out) {
    sdrt::set_error("null argument");
    return SDRT_E_INVALID_ARG;
  }
  const sdrt::Mesh& m = mm->m;
  const sdrt::RefElement& r = m.ref;
  out->etype = m.etype;
  out->p = m.p;
  out->nd = m.nd;
  out->nsol = r.nsol;
  out->next = r.next;
  out->nint = r.nint;
  out->nu = r.nu;
  out->nfaces = r.nfaces;
  out->nfp = r.nfp;
  out->nsub = m.nsub;
  for (int d = 0; d < 3; ++d) {
    out->N[d] = m.Nloc[d];
    out->Nglobal[d] = m.Nglob[d];
    out->offset[d] = m.offset[d];
  }
  out->K = m.K;
  out->K_pad = m.K_pad;
  // faces whose left element is local, plus far-field boundary faces of local elements
  int64_t nf = 0;
  for (int64_t e = 0; e < m.K; ++e) {
    int c[3];
    m.gcoords(e, c);
    for (int f = 0; f < r.nfaces; ++f) {
      const sdrt::FaceLink& L = m.link[(e % m.nsub) * r.nfaces + f];
      bool ff = false;
      for (int d = 0; d < m.nd; ++d) {
        const int cc = c[d] + L.off[d];
        if (!m.periodic[d] && (cc < 0 || cc >= m.Nglob[d])) ff = true;
      }
      nf += (L.left || ff) ? 1 : 0;
    }
  }
  out->n_faces = nf;
  out->K_trace = m.Kt;
  return SDRT_OK;
}

sdrt_status sdrt_mesh_export_maps(const sdrt_mesh* mm, int32_t* face_elem, int8_t* face_lface,
                                  int16_t* face_perm, uint8_t* is_left) {
  if (!mm) {
    sdrt::set_error("null mesh");
    return SDRT_E_INVALID_ARG;
  }
  const sdrt::Mesh& m = mm->m;
  const sdrt::RefElement& r = m.ref;
  int64_t F = 0;
  for (int64_t e = 0; e < m.K; ++e) {
    int s = (int)(e % m.nsub);
    int c[3];
    m.gcoords(e, c);
    for (int f = 0; f < r.nfaces; ++f) {
      const sdrt::FaceLink& L = m.link[s * r.nfaces + f];
      if (is_left) is_left[e * r.nfaces + f] = (uint8_t)L.left;
      bool ff = false;  // far-field boundary face: the neighbour is outside the domain
      for (int d = 0; d < m.nd; ++d) {
        const int cc = c[d] + L.off[d];
        if (!m.periodic[d] && (cc < 0 || cc >= m.Nglob[d])) ff = true;
      }
      if (!L.left && !ff) continue;
      int64_t g = 0, mul = 1;
      for (int d = 0; d < m.nd; ++d) {
        int cc = ((c[d] + L.off[d]) % m.Nglob[d] + m.Nglob[d]) % m.Nglob[d];
        g += mul * cc;
        mul *= m.Nglob[d];
      }
      const int64_t nb = ff ? -1 : g * m.nsub + L.nshape;
      const int64_t me = m.global_id(e);
      if (face_elem) {
        face_elem[2 * F] = (int32_t)(L.left ? me : -1);
        face_elem[2 * F + 1] = (int32_t)(L.left ? nb : me);
      }
      if (face_lface) {
        face_lface[2 * F] = (int8_t)(L.left ? f : -1);
        face_lface[2 * F + 1] = (int8_t)(L.left ? (ff ? -1 : L.nface) : f);
      }
      if (face_perm)  // rows of nfp (the largest face), -1 beyond this face's points
        for (int q = 0; q < r.nfp; ++q)
          face_perm[F * r.nfp + q] = (int16_t)((ff || q >= (int)L.perm.size()) ? -1 : L.perm[q]);
      ++F;
    }
  }
  return SDRT_OK;
}

sdrt_status sdrt_mesh_sol_coords(const sdrt_mesh* mm, double* x) {
  if (!mm || !x) {
    sdrt::set_error("null argument");
    return SDRT_E_INVALID_ARG;
  }
  const sdrt::Mesh& m = mm->m;
  const sdrt::RefElement& r = m.ref;
  int D = m.nd;
  for (int64_t e = 0; e < m.K; ++e) {
    int s = (int)(e % m.nsub);
    int c[3];
    m.gcoords(e, c);
    for (int q = 0; q < r.nsol; ++q)
      for (int i = 0; i < D; ++i) {
        // x = lo + h*(pattern + P0) + J (x~ + 1)
        double v = m.lo[i] + m.h[i] * (c[i] + m.P0[s][i]);
        for (int j = 0; j < D; ++j) v += m.J[s][i * 3 + j] * (r.xsol[q][j] + 1.0);
        x[((size_t)q * D + i) * m.K + e] = v;
      }
  }
  return SDRT_OK;
}

sdrt_status sdrt_mesh_detj(const sdrt_mesh* mm, double* detj) {
  if (!mm || !detj) {
    sdrt::set_error("null argument");
    return SDRT_E_INVALID_ARG;
  }
  for (int64_t e = 0; e < mm->m.K; ++e) detj[e] = mm->m.detJ[e % mm->m.nsub];
  return SDRT_OK;
}

void sdrt_mesh_destroy(sdrt_mesh* m) { delete m; }

sdrt_status sdrt_mesh_set_halo(sdrt_mesh* m, int force_self_halo) {
  if (!m) {
    sdrt::set_error("null mesh");
    return SDRT_E_INVALID_ARG;
  }
  SDRT_TRY({
    sdrt::build_halo(m->m, force_self_halo != 0);
    return SDRT_OK;
  })
}

sdrt_status sdrt_mesh_halo_lists(const sdrt_mesh* mm, int slab, int* peer, int* d, int* side, int64_t* count,
                                 int32_t* send_row, int32_t* send_col, int32_t* recv_row, int32_t* recv_col) {
  if (!mm) {
    sdrt::set_error("null mesh");
    return SDRT_E_INVALID_ARG;
  }
  const sdrt::Mesh& m = mm->m;
  if (slab < 0 || slab >= (int)m.slabs.size()) {
    if (count) *count = -1;
    if (slab == -1 && count) *count = (int64_t)m.slabs.size();
    if (slab == -1) return SDRT_OK;
    sdrt::set_error("slab index out of range");
    return SDRT_E_INVALID_ARG;
  }
  const sdrt::HaloSlab& S = m.slabs[slab];
  if (peer) *peer = S.peer;
  if (d) *d = S.d;
  if (side) *side = S.side;
  if (count) *count = (int64_t)S.send_row.size();
  for (size_t i = 0; i < S.send_row.size(); ++i) {
    if (send_row) send_row[i] = S.send_row[i];
    if (send_col) send_col[i] = S.send_col[i];
    if (recv_row) recv_row[i] = S.recv_row[i];
    if (recv_col) recv_col[i] = S.recv_col[i];
  }
  return SDRT_OK;
}

sdrt_status sdrt_mesh_neighbor(const sdrt_mesh* mm, int64_t e, int f, int64_t* col, int* face) {
  if (!mm || !col || !face) {
    sdrt::set_error("null argument");
    return SDRT_E_INVALID_ARG;
  }
  const sdrt::Mesh& m = mm->m;
  if (e < 0 || e >= m.K || f < 0 || f >= m.ref.nfaces) {
    sdrt::set_error("element / face out of range");
    return SDRT_E_INVALID_ARG;
  }
  const int s = (int)(e % m.nsub);
  const sdrt::FaceLink& L = m.link[s * m.ref.nfaces + f];
  int64_t pat = e / m.nsub;
  int c[3] = {0, 0, 0};
  for (int d = 0; d < m.nd; ++d) {
    c[d] = (int)(pat % m.Nloc[d]);
    pat /= m.Nloc[d];
  }
  *face = L.nface;
  int64_t id = 0, mul = 1;
  for (int d = 0; d < m.nd; ++d) {
    int cc = c[d] + L.off[d];
    if ((cc < 0 || cc >= m.Nloc[d]) && m.halo[d]) {
      const int a = d == 0 ? 1 : 0, b = d == 2 ? 1 : 2;
      const int64_t tang = m.nd == 2 ? c[a] : c[a] + (int64_t)m.Nloc[a] * c[b];
      *col = m.gbase[d][cc < 0 ? 0 : 1] + tang * m.nsub + L.nshape;
      return SDRT_OK;
    }
    cc = (cc + m.Nloc[d]) % m.Nloc[d];
    id += mul * cc;
    mul *= m.Nloc[d];
  }
  *col = id * m.nsub + L.nshape;
  return SDRT_OK;
}

sdrt_status sdrt_operators_build(int etype, int p, int scheme, sdrt_operators** out) {
  if (!out) {
    sdrt::set_error("null argument");
    return SDRT_E_INVALID_ARG;
  }
  if (scheme < SDRT_SCHEME_SDRT || scheme > SDRT_SCHEME_FRDG) {
    sdrt::set_error("unsupported scheme");
    return SDRT_E_UNSUPPORTED;
  }
  if (etype < 0 || etype > 4) {
    sdrt::set_error("unsupported element type");
    return SDRT_E_UNSUPPORTED;
  }
  SDRT_TRY({
    auto* o = new sdrt_operators;
    try {
      o->o = sdrt::build_operators(etype, p, scheme);
    } catch (...) {
      delete o;
      throw;
    }
    *out = o;
    return SDRT_OK;
  })
}

sdrt_status sdrt_operators_get(const sdrt_operators* oo, const char* name, double* dst, int* rows,
                               int* cols) {
  if (!oo || !name) {
    sdrt::set_error("null argument");
    return SDRT_E_INVALID_ARG;
  }
  const sdrt::Operators& o = oo->o;
  const sdrt::Mat* M = nullptr;
  std::string n(name);
  if (n == "M0") M = &o.M0;
  else if (n == "M12") M = &o.M12;
  else if (n == "M13") M = &o.M13;
  else if (n == "M14") M = &o.M14;
  else if (n == "M15") M = &o.M15;
  else if (n == "M16") M = &o.M16;
  else if (n == "P") M = &o.P;
  else if (n == "M19P2") M = &o.M19P2;
  else if (n == "Mc" && o.scheme != 0) M = &o.Mc;
  if (M) {
    if (rows) *rows = M->rows;
    if (cols) *cols = M->cols;
    if (dst) std::memcpy(dst, M->a.data(), M->a.size() * sizeof(double));
    return SDRT_OK;
  }
  const sdrt::RefElement& r = o.ref;
  if (n == "w") {
    if (rows) *rows = r.nsol;
    if (cols) *cols = 1;
    if (dst) std::memcpy(dst, o.w.data(), o.w.size() * sizeof(double));
    return SDRT_OK;
  }
  const std::vector<std::array<double, 3>>* pts = nullptr;
  if (n == "xsol") pts = &r.xsol;
  else if (n == "xext") pts = &r.xext;
  else if (n == "xu") pts = &r.xu;
  if (pts) {
    if (rows) *rows = (int)pts->size();
    if (cols) *cols = r.nd;
    if (dst)
      for (size_t i = 0; i < pts->size(); ++i)
        for (int d = 0; d < r.nd; ++d) dst[i * r.nd + d] = (*pts)[i][d];
    return SDRT_OK;
  }
  sdrt::set_error("unknown operator name");
  return SDRT_E_INVALID_ARG;
}

void sdrt_operators_destroy(sdrt_operators* o) { delete o; }

}  // extern "C"
