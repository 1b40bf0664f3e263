// Fused SDRT stage for simplex elements (tri / tet), sm_100a, fp64.
#pragma once
#include <cuda.h>  // CUtensorMap (TMA descriptors)
#include <cuda_runtime.h>

#include <cstdint>

#include "ctx.h"
#include "physics.cuh"

namespace sdrt {

// Dense App. B operator packed for the FP64 tensor-core MMA (mma.sync m8n8k4 f64):
// zero-padded to R8 = 8*mt rows and C4 = 4*kt columns, stored fragment by fragment,
// frag[(m * kt + k) * 32 + lane] = M[8 m + lane/4][4 k + lane%4], so one warp-wide
// 256-byte coalesced load fetches one A fragment.
struct SOpF {
  int rows, cols, mt, kt;
  const double* frag;
  const unsigned* kmask;  // per m-tile: bit k set if the 8x4 block (m, k) has a non-zero
};

struct SimplexOps {
  SOpF M0;    // N_ext x N_sol
  SOpF M12;   // N_u x N_sol
  SOpF G;     // (D*N_sol) x (N_ext + N_u): rows (d, s), [M16 | M15 P]; the face blocks of
              //   M16 whose normal lacks a d component are zero 8x4 blocks (skipped)
              //   FR-SDRT: (D*N_sol) x (N_ext + N_sol), [M16 | Dsol - M16 M0] on [C; U]
  SOpF M14;   // N_sol x N_ext
  SOpF M13F;  // N_sol x (D N_u): M13 M19 P2, columns (d, u)
              //   FR-SDRT: N_sol x (D N_sol), Dsol - M14 (n^ . M0), columns (d, s)
  SOpF M14F;  // [M14 | M13F]: the whole divergence on [D~; F~] (inviscid kernel B)
  int fr;     // 1: FR-SDRT (NEXT row N1), fluxes at the solution points
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
  double* Rint;          // internal-flux divergence M13 M19 P2 F~ [N_sol][N_V][Kp] (kernel A -> B)
  const ExtMetric* xm;   // [nsub][N_ext]
  double* Fexp = nullptr;  // optional (residual only): common flux F per own ext point [N_ext][N_V][Kp]
};

// TMA descriptors of [N_sol N_V rows][Kp] arrays (cached per pointer), tiles of E elements
struct SimplexTma {
  int rows = 0, E = 0;
  int64_t Kp = 0;
  const void* ptr[8] = {};
  CUtensorMap map[8];
  int next = 0;
};

bool simplex_supported(int D, int P, int eq);
// TGV diagnostics partial sums (3 per tile of 8 elements); NS only
void simplex_launch_diag(int D, int P, const GeomDev& g, const SimplexOps& O, const PhysDev& ph, SimplexTma* tma,
                         const SimplexBufs& b, const double* w, const double* Bq, int nq, double* part,
                         cudaStream_t st);
int simplex_tile_width(int D, int P, int eq);
void simplex_tma_init(SimplexTma* t, int D, int P, int eq, int64_t Kp);
void simplex_launch_traces(int D, int P, int eq, const GeomDev& g, const SimplexOps& O, SimplexTma* tma,
                           const double* U, double* Tu, cudaStream_t st);
// kernel A (viscous): gradient, published viscous traces, internal fluxes -> Rint
void simplex_launch_grad(int D, int P, int eq, const GeomDev& g, const SimplexOps& O, const PhysDev& ph,
                         SimplexTma* tma, const SimplexBufs& b, cudaStream_t st);
// kernel B: face fluxes, M14 lift (+ internal fluxes for inviscid equations), RK, traces
void simplex_launch_flux(int D, int P, int eq, const GeomDev& g, const SimplexOps& O, const PhysDev& ph,
                         SimplexTma* tma, const SimplexBufs& b, int stage, double dt, cudaStream_t st);

}  // namespace sdrt
