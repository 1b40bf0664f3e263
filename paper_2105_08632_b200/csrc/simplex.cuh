// Fused SDRT stage for simplex elements (tri / tet), sm_100a, fp64.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "ctx.h"
#include "physics.cuh"

namespace sdrt {

constexpr int SRB = 4;  // rows per register block of the dense operator products

// Dense App. B operator in row blocks of SRB rows with the block's non-zero columns.
struct SOp {
  int rows, cols, nblk;
  const int* ptr;      // [nblk+1]
  const int* col;      // [nnz]
  const double* val;   // [nnz][SRB]
};

struct SimplexOps {
  SOp M0;    // N_ext x N_sol
  SOp M12;   // N_u x N_sol
  SOp G;     // (N_sol*D) x (N_ext + N_u): rows (s, d), [M16 | M15 P]
  SOp M14;   // N_sol x N_ext
  SOp M13F;  // N_sol x (D N_u): M13 M19 P2, columns (d, u)
  const double* M0dense;  // N_ext x N_sol (row-major) for per-point gradient traces
};

struct SimplexBufs {
  const double* Uin;
  double* U;
  double* Us;
  double* ACC;
  double* out;
  const double* Tu;
  double* Tu_next;
  double* Tg;
  const ExtMetric* xm;  // [nsub][N_ext]
};

bool simplex_supported(int D, int P, int eq);
void simplex_launch_traces(int D, int P, int eq, const GeomDev& g, const SimplexOps& O, const double* U,
                           double* Tu, cudaStream_t st);
void simplex_launch_grad(int D, int P, int eq, const GeomDev& g, const SimplexOps& O, const PhysDev& ph,
                         const SimplexBufs& b, cudaStream_t st);
void simplex_launch_flux(int D, int P, int eq, const GeomDev& g, const SimplexOps& O, const PhysDev& ph,
                         const SimplexBufs& b, int stage, double dt, cudaStream_t st);

}  // namespace sdrt
