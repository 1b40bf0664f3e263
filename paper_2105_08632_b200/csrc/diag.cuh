// TGV ensemble-average integrands (NEXT row N4), shared by the
// tensor and simplex diagnostics kernels.
#pragma once
#include "physics.cuh"

namespace sdrt {

// E* = rho v.v, S^d : S^d and p div v at one point from the conserved variables u[NV]
// and their gradient q[j*NV + v] = d u_v / d x_j (grad v by the chain rule, reading O20),
// accumulated with weight wr
template <int D, int NV>
__device__ __forceinline__ void tgv_point(const PhysDev& ph, const double* u, const double* q, double wr,
                                          double (&acc)[3]) {
  const double rho = u[0];
  double v[D], vv = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    v[i] = u[1 + i] / rho;
    vv += v[i] * v[i];
  }
  const double pr = (ph.gamma - 1.0) * (u[D + 1] - 0.5 * rho * vv);
  double dv[D][D];  // dv[j][i] = d v_i / d x_j
#pragma unroll
  for (int j = 0; j < D; ++j)
#pragma unroll
    for (int i = 0; i < D; ++i) dv[j][i] = (q[j * NV + 1 + i] - v[i] * q[j * NV]) / rho;
  double div = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) div += dv[i][i];
  double ss = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double sij = 0.5 * (dv[j][i] + dv[i][j]) - (i == j ? div / 3.0 : 0.0);
      ss += sij * sij;
    }
  acc[0] += wr * rho * vv;
  acc[1] += wr * ss;
  acc[2] += wr * pr * div;
}

// All points of a tile of E elements: sU [NSOL][NV][E], sQ [D][NSOL][NV][E] in shared
// memory.  Bq == nullptr: the solution points with weights w[NSOL]; else the nq cubature
// points with weights w[nq] and the solution-basis values Bq[q][NSOL] (interpolation of
// u_h and of the LDG-gradient polynomial Q_h).  detj(el): the element's detJ.
template <int D, int NV, int E, int NSOL, class DetJ>
__device__ __forceinline__ void tgv_tile(const PhysDev& ph, const double* sU, const double* sQ,
                                         const double* __restrict__ w, const double* __restrict__ Bq, int nq,
                                         int64_t e0, int64_t K, DetJ detj, double (&acc)[3]) {
  const int npt = Bq ? nq : NSOL;
  for (int item = threadIdx.x; item < npt * E; item += blockDim.x) {
    const int el = item % E, pt = item / E;
    if (e0 + el >= K) continue;
    double u[NV], q[D * NV];
    if (!Bq) {
#pragma unroll
      for (int v = 0; v < NV; ++v) u[v] = sU[(pt * NV + v) * E + el];
#pragma unroll
      for (int j = 0; j < D; ++j)
#pragma unroll
        for (int v = 0; v < NV; ++v) q[j * NV + v] = sQ[((j * NSOL + pt) * NV + v) * E + el];
    } else {
#pragma unroll
      for (int k = 0; k < D * NV; ++k) q[k] = 0.0;
#pragma unroll
      for (int v = 0; v < NV; ++v) u[v] = 0.0;
      const double* bq = Bq + (int64_t)pt * NSOL;
      for (int r = 0; r < NSOL; ++r) {
        const double br = __ldg(bq + r);
#pragma unroll
        for (int v = 0; v < NV; ++v) u[v] = fma(br, sU[(r * NV + v) * E + el], u[v]);
#pragma unroll
        for (int j = 0; j < D; ++j)
#pragma unroll
          for (int v = 0; v < NV; ++v) q[j * NV + v] = fma(br, sQ[((j * NSOL + r) * NV + v) * E + el], q[j * NV + v]);
      }
    }
    tgv_point<D, NV>(ph, u, q, __ldg(w + pt) * detj(el), acc);
  }
}

}  // namespace sdrt
