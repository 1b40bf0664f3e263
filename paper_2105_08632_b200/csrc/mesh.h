// Uniform periodic pattern meshes (host).  PAPER.md §2 l.145-172, §3 l.497-519.
#pragma once
#include <array>
#include <cstdint>
#include <vector>

#include "refel.h"

namespace sdrt {

// Neighbour link of local face f of sub-cell shape s (translation invariant).
struct FaceLink {
  int off[3];          // neighbour pattern offset
  int nshape, nface;   // neighbour sub-cell shape and its local face
  int left;            // 1 if this side is the LEFT element (reading O14)
  std::vector<int> perm;  // my face point q -> neighbour face point index
};

// One halo slab: the ghost layer across local face direction (d, side) of this rank's
// block.  Entries are (trace row, column) pairs of the trace arrays [N_ext][N_V][Kt];
// each entry carries N_V values.  send: rows of MY boundary elements facing the peer;
// recv: the same rows written into MY ghost columns for the peer's elements.  Both
// lists are in the canonical order (tangential pattern, sub-cell, face, point), so the
// peer's send list matches my recv list entry by entry.
struct HaloSlab {
  int d, side;      // side 0: -d direction, 1: +d direction
  int peer;         // rank owning the neighbouring block (may be this rank: periodic loopback)
  std::vector<int32_t> send_row, send_col, recv_row, recv_col;
};

struct Mesh {
  int periodic[3] = {1, 1, 1};  // 0: far-field boundaries on this axis
  // far-field ghost trace entries (trace row, ghost column): the rows of the ghost element
  // across a far-field boundary face that the boundary element reads; filled once with
  // the far-field state (sdrt_ctx_set_farfield), never exchanged
  std::vector<int32_t> ff_row, ff_col;
  int etype, p, nd, nsub;
  int Nloc[3], Nglob[3], offset[3];
  int rank, nranks, pgrid[3];
  double lo[3], hi[3], h[3];
  int64_t K, K_pad;
  RefElement ref;
  // per shape
  std::vector<std::array<double, 9>> J, Jinv;   // row-major D x D (padded to 3x3)
  std::vector<double> detJ;
  std::vector<std::array<double, 3>> P0;        // unit-cube position of the image of V0
  // per (shape, face)
  std::vector<FaceLink> link;                   // [s * nfaces + f]
  // per (shape, ext point)
  std::vector<double> sscale;                   // detJ |J^-T n~|
  std::vector<std::array<double, 3>> nleft;     // canonical (left element's) unit normal
  // halo (multi-rank / loopback): ghost columns after K_pad in the trace arrays
  int halo[3] = {0, 0, 0};                      // axis uses ghost slabs
  int64_t Kt = 0;                               // trace row stride = K_pad + ghosts (padded)
  int64_t gbase[3][2] = {{0, 0}, {0, 0}, {0, 0}};  // first ghost column of slab (d, side)
  std::vector<HaloSlab> slabs;

  int64_t pattern_of(int64_t e) const { return e / nsub; }
  // global pattern coords of local element e
  void gcoords(int64_t e, int c[3]) const;
  int64_t global_id(int64_t e) const;
};

Mesh build_mesh(int etype, int p, const int N[3], const double lo[3], const double hi[3], int rank,
                int nranks, const int pgrid[3], const int periodic[3] = nullptr);
// (Re)build the ghost layout and halo lists; force_self_halo routes periodic wraps of
// single-rank axes through the halo path as well (loopback testing on one device).
void build_halo(Mesh& m, bool force_self_halo);

}  // namespace sdrt
