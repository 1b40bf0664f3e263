// Device context: workspace plan, packed operators and geometry tables.
#pragma once
#include <cstddef>
#include <cstdint>

#include "physics.cuh"

namespace sdrt {

constexpr int MAXF = 6;      // faces per element
constexpr int MAXFP = 25;    // points per face (hex p=4)
constexpr int MAXSUB = 6;    // sub-cell shapes
constexpr int MAXEXT = 150;  // external points (hex p=4)
constexpr int RB = 8;        // rows per operator chunk

// Operator packed as row chunks of RB rows with the list of columns that carry a
// non-zero in the chunk (structural sparsity of App. B, l.2927-2932).
struct OpDev {
  int rows, cols, nchunks;
  const int* chunk_ptr;   // [nchunks+1]
  const int* col;         // [nnzcol]
  const double* val;      // [nnzcol][RB]
};

// Translation-invariant geometry of a uniform pattern mesh (fits a kernel param).
struct GeomDev {
  int nd, nsub, nfaces, nfp, next;
  int Nloc[3], Nglob[3], offset[3];
  int64_t K, Kp;
  int64_t Kt;             // trace row stride (K_pad + ghost columns)
  int halo[3];            // axis uses ghost slabs
  int64_t gbase[3][2];    // first ghost column of slab (d, side)
  double detJ[MAXSUB];
  double Jinv[MAXSUB][9];
  // per (shape, face)
  int8_t off[MAXSUB][MAXF][3];
  int8_t nshape[MAXSUB][MAXF], nface[MAXSUB][MAXF], left[MAXSUB][MAXF];
  int8_t perm[MAXSUB][MAXF][MAXFP];
  int16_t fptr[MAXF + 1];  // face f: ext points fptr[f] .. fptr[f+1] (prisms mix face sizes)
  int8_t xface[MAXEXT];    // face of each ext point
  const int* tiles;       // optional tile list (interior / boundary subsets), nullptr = all
  int ntiles;
  int osf;                // fused simplex path: one-sided flux publication (simplex.cu ks_stage_osf)
};

// per (shape, ext point) metric: s scale and canonical normal (global memory)
struct ExtMetric {
  double s, n0, n1, n2;
};

}  // namespace sdrt
