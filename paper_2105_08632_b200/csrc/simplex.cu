// Fused SDRT stage for simplex elements (tri / tet) on sm_100a, fp64.
//
// Simplex operators are dense (App. B l.2855-2925, B7: all N_D components per unique
// internal point, l.2927-2932), so each App. B product is a small dense matrix applied
// to a tile of E elements held in shared memory [row][var][E] (element fastest, the ABI
// layout).  One thread computes SRB rows x all variables for one element: operator
// entries are warp-uniform reads (L1 broadcast), tile entries are bank-conflict-free.
//
//   kernel A (viscous): U_ext = M0 U, U_u = M12 U, C (l.282-291, neighbour traces),
//     Q~ = [M16 | M15 P][C; U_u] (l.2877-2880), Q = J^-T Q~ (l.299-302), and the
//     published viscous normal flux g = n_L . f^v(u, M0 Q) at the face points of the
//     side carrying LDG weight (l.330-335).
//   kernel B: the same gradient, Q_u = M18 Q (l.2897-2900), internal fluxes F~ =
//     detJ J^-1 f (l.305-311), common fluxes D~ = +/- s F (l.312-340, canonical L/R),
//     R~ = M14 D~ + M13 M19 P2 F~ (l.2919-2925), -R~/detJ, RK4 update, new traces.
// Face values are exchanged only through double-buffered traces; the own trace is
// recomputed by the same operator routine (fixed fma order), so both neighbours
// evaluate each face point's common flux from bit-identical inputs (O28).
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "simplex.cuh"

namespace sdrt {

template <int D, int P>
struct SDims {
  static constexpr int nsol = D == 2 ? (P + 1) * (P + 2) / 2 : (P + 1) * (P + 2) * (P + 3) / 6;
  static constexpr int next = D == 2 ? 3 * (P + 1) : 2 * (P + 1) * (P + 2);
  static constexpr int nu = D == 2 ? P * (P + 1) / 2 : P * (P + 1) * (P + 2) / 6;
  static constexpr int nfaces = D + 1;
  static constexpr int nfp = next / nfaces;
};

template <typename T>
__host__ __device__ constexpr T cmax(T a, T b) { return a > b ? a : b; }

template <int D, int P, int NV, bool VISC>
struct SLayout {
  using S = SDims<D, P>;
  static constexpr int U = S::nsol * NV;
  static constexpr int UE = S::next * NV;
  static constexpr int R0 = cmax(cmax(S::next * NV, VISC ? S::nu * D * NV : 0), S::nsol * NV);
  static constexpr int UU = S::nu * NV;
  static constexpr int Q = cmax(VISC ? S::nsol * D * NV : 0, S::nu * D * NV);
  static constexpr int TOTAL = U + UE + R0 + UU + Q;  // doubles per element
};

// Y[r][w][el] (+)= sum_c M[r][c] X[c][w][el], X rows c < split from X0, else X1.
// W values per row in chunks of WC; one work item = (row block, chunk, element), so
// every thread of the CTA has work even for short operators.
template <int W, int E, bool ACCUM>
__device__ __forceinline__ void sapply(const SOp& M, const double* X0, int split, const double* X1, double* Y) {
  constexpr int WC = W % 5 == 0 ? 5 : (W % 4 == 0 ? 4 : (W % 3 == 0 ? 3 : (W % 2 == 0 ? 2 : 1)));
  constexpr int NWC = W / WC;
  const int nitems = M.nblk * NWC * E;
  for (int item = threadIdx.x; item < nitems; item += blockDim.x) {
    const int el = item % E, r2 = item / E;
    const int w0 = (r2 % NWC) * WC, blk = r2 / NWC;
    double acc[SRB][WC];
#pragma unroll
    for (int k = 0; k < SRB; ++k)
#pragma unroll
      for (int w = 0; w < WC; ++w) acc[k][w] = 0.0;
    const int b = M.ptr[blk], e = M.ptr[blk + 1];
    for (int j = b; j < e; ++j) {
      const int c = __ldg(M.col + j);
      const double* xr = (c < split ? X0 + c * W * E : X1 + (c - split) * W * E) + w0 * E + el;
      double x[WC];
#pragma unroll
      for (int w = 0; w < WC; ++w) x[w] = xr[w * E];
      const double* mv = M.val + (int64_t)j * SRB;
#pragma unroll
      for (int k = 0; k < SRB; ++k) {
        const double m = __ldg(mv + k);
#pragma unroll
        for (int w = 0; w < WC; ++w) acc[k][w] = __fma_rn(m, x[w], acc[k][w]);
      }
    }
#pragma unroll
    for (int k = 0; k < SRB; ++k) {
      const int r = blk * SRB + k;
      if (r >= M.rows) break;
#pragma unroll
      for (int w = 0; w < WC; ++w) {
        double* y = Y + (r * W + w0 + w) * E + el;
        *y = ACCUM ? *y + acc[k][w] : acc[k][w];
      }
    }
  }
}

// traces to global: T[r][v][Kp] = (M0 U)[r][v] for valid elements (same fma order as sapply)
template <int NV, int E>
__device__ __forceinline__ void strace_global(const SOp& M, const double* X, double* __restrict__ T, int64_t e0,
                                              int64_t K, int64_t Kp) {
  const int nitems = M.nblk * E;
  for (int item = threadIdx.x; item < nitems; item += blockDim.x) {
    const int el = item % E, blk = item / E;
    const int64_t e = e0 + el;
    double acc[SRB][NV];
#pragma unroll
    for (int k = 0; k < SRB; ++k)
#pragma unroll
      for (int w = 0; w < NV; ++w) acc[k][w] = 0.0;
    const int b = M.ptr[blk], en = M.ptr[blk + 1];
    for (int j = b; j < en; ++j) {
      const int c = __ldg(M.col + j);
      double x[NV];
#pragma unroll
      for (int w = 0; w < NV; ++w) x[w] = X[(c * NV + w) * E + el];
      const double* mv = M.val + (int64_t)j * SRB;
#pragma unroll
      for (int k = 0; k < SRB; ++k) {
        const double m = __ldg(mv + k);
#pragma unroll
        for (int w = 0; w < NV; ++w) acc[k][w] = __fma_rn(m, x[w], acc[k][w]);
      }
    }
    if (e >= K) continue;
#pragma unroll
    for (int k = 0; k < SRB; ++k) {
      const int r = blk * SRB + k;
      if (r >= M.rows) break;
#pragma unroll
      for (int w = 0; w < NV; ++w) T[((int64_t)r * NV + w) * Kp + e] = acc[k][w];
    }
  }
}

template <int ROWS, int E>
__device__ __forceinline__ void sload(const double* __restrict__ src, double* s, int64_t e0, int64_t Kp) {
  constexpr int CH = E / 2;
  for (int idx = threadIdx.x; idx < ROWS * CH; idx += blockDim.x) {
    const int c = idx % CH, row = idx / CH;
    const double* g = src + (int64_t)row * Kp + e0 + 2 * c;
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s + row * E + 2 * c);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g));
  }
  asm volatile("cp.async.commit_group;");
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// neighbour of element e across local face f (pattern arithmetic, periodic)
__device__ __forceinline__ int snbr(const GeomDev& g, int e, int s, int f) {
  int pat = e / g.nsub;
  int c[3] = {0, 0, 0};
#pragma unroll
  for (int d = 0; d < 3; ++d)
    if (d < g.nd) {
      c[d] = (int)(pat % g.Nloc[d]);
      pat /= g.Nloc[d];
    }
  int id = 0, mul = 1;
#pragma unroll
  for (int d = 0; d < 3; ++d)
    if (d < g.nd) {
      int cc = c[d] + g.off[s][f][d];
      if ((cc < 0 || cc >= g.Nloc[d]) && g.halo[d]) {
        // ghost column: slab (d, side), tangential pattern index, neighbour sub-cell
        const int a = d == 0 ? 1 : 0, bb = d == 2 ? 1 : 2;
        const int tang = g.nd == 2 ? c[a] : c[a] + g.Nloc[a] * c[bb];
        return (int)g.gbase[d][cc < 0 ? 0 : 1] + tang * g.nsub + g.nshape[s][f];
      }
      cc = cc < 0 ? cc + g.Nloc[d] : (cc >= g.Nloc[d] ? cc - g.Nloc[d] : cc);
      id += mul * cc;
      mul *= g.Nloc[d];
    }
  return (int)(id * g.nsub + g.nshape[s][f]);
}

// C = (1/2 - b) u_L + (1/2 + b) u_R at external points into sC [next][NV][E]
template <int D, int P, int NV, int E>
__device__ __forceinline__ void common_values(const GeomDev& g, const PhysDev& ph, const double* __restrict__ Tu,
                                              const double* sUe, const int (*sNb)[E], double* sC, int64_t e0) {
  using S = SDims<D, P>;
  const double wl = 0.5 - ph.beta, wr = 0.5 + ph.beta;
  const int Kp = (int)g.Kt;  // trace row stride
  for (int item = threadIdx.x; item < S::next * E; item += blockDim.x) {
    const int el = item % E, rho = item / E;
    const int64_t e = e0 + el;
    if (e >= g.K) continue;
    const int s = sNb[D + 1][el], f = rho / S::nfp, q = rho % S::nfp;
    const int m = sNb[f][el];
    const int rho2 = g.nface[s][f] * S::nfp + g.perm[s][f][q];
    const bool left = g.left[s][f];
    double nb[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) nb[v] = Tu[(rho2 * NV + v) * Kp + m];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const double own = sUe[(rho * NV + v) * E + el];
      const double uL = left ? own : nb[v], uR = left ? nb[v] : own;
      sC[(rho * NV + v) * E + el] = wl * uL + wr * uR;
    }
  }
}

// Q = J^-T Q~ in place on sQ [nsol][D][NV][E]
template <int D, int P, int NV, int E>
__device__ __forceinline__ void metric_grad(const GeomDev& g, const int (*sNb)[E], double* sQ) {
  using S = SDims<D, P>;
  for (int item = threadIdx.x; item < S::nsol * E; item += blockDim.x) {
    const int el = item % E, sp = item / E;
    const int s = sNb[D + 1][el];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double qt[D];
#pragma unroll
      for (int d = 0; d < D; ++d) qt[d] = sQ[((sp * D + d) * NV + v) * E + el];
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) acc = fma(g.Jinv[s][j * 3 + i], qt[j], acc);
        sQ[((sp * D + i) * NV + v) * E + el] = acc;
      }
    }
  }
}

// neighbour ids sNb[f][el] and sub-cell shapes sNb[D+1][el] of a tile, once
template <int D, int E>
__device__ __forceinline__ void fill_neighbours(const GeomDev& g, int (*sNb)[E], int64_t e0) {
  for (int idx = threadIdx.x; idx < (D + 2) * E; idx += blockDim.x) {
    const int el = idx % E, f = idx / E;
    const int e = (int)e0 + el;
    const int s = e % g.nsub;
    sNb[f][el] = f == D + 1 ? s : (e < g.K ? snbr(g, e, s, f) : 0);
  }
}

// shared prologue: tile, own traces, U_u, [C, Q]
template <int D, int P, int EQ, int E>
__device__ __forceinline__ void prologue(const GeomDev& g, const SimplexOps& O, const PhysDev& ph,
                                         const double* Uin, const double* Tu, double* smem, int (*sNb)[E],
                                         int64_t e0) {
  using Ph = Phys<EQ, D>;
  using S = SDims<D, P>;
  using Ly = SLayout<D, P, Ph::NV, Ph::VISC>;
  constexpr int NV = Ph::NV;
  double* sU = smem;
  double* sUe = sU + Ly::U * E;
  double* sR0 = sUe + Ly::UE * E;
  double* sUu = sR0 + Ly::R0 * E;
  double* sQ = sUu + Ly::UU * E;
  fill_neighbours<D, E>(g, sNb, e0);
  sload<S::nsol * NV, E>(Uin, sU, e0, g.Kp);
  __syncthreads();
  sapply<NV, E, false>(O.M0, sU, 1 << 30, sU, sUe);
  sapply<NV, E, false>(O.M12, sU, 1 << 30, sU, sUu);
  __syncthreads();
  if constexpr (Ph::VISC) {
    common_values<D, P, NV, E>(g, ph, Tu, sUe, sNb, sR0, e0);
    __syncthreads();
    sapply<NV, E, false>(O.G, sR0, S::next, sUu, sQ);  // rows (s, d) -> [s][d][v]
    __syncthreads();
    metric_grad<D, P, NV, E>(g, sNb, sQ);
    __syncthreads();
  }
}

template <int D, int P, int EQ, int E>
__global__ void __launch_bounds__(256) ks_traces(GeomDev g, SimplexOps O, const double* __restrict__ U,
                                                 double* __restrict__ T) {
  constexpr int NV = Phys<EQ, D>::NV;
  extern __shared__ double smem[];
  const int64_t e0 = (int64_t)blockIdx.x * E;
  sload<SDims<D, P>::nsol * NV, E>(U, smem, e0, g.Kp);
  __syncthreads();
  strace_global<NV, E>(O.M0, smem, T, e0, g.K, g.Kt);
}

template <int D, int P, int EQ, int E>
__global__ void __launch_bounds__(256) ks_grad(GeomDev g, SimplexOps O, PhysDev ph, SimplexBufs b) {
  using Ph = Phys<EQ, D>;
  using S = SDims<D, P>;
  using Ly = SLayout<D, P, Ph::NV, Ph::VISC>;
  constexpr int NV = Ph::NV;
  extern __shared__ double smem[];
  __shared__ int sNb[D + 2][E];  // [f][el] neighbours, [D+1][el] shape
  const int64_t e0 = (int64_t)blockIdx.x * E;
  prologue<D, P, EQ, E>(g, O, ph, b.Uin, b.Tu, smem, sNb, e0);
  const double* sUe = smem + Ly::U * E;
  const double* sQ = smem + (Ly::U + Ly::UE + Ly::R0 + Ly::UU) * E;
  const bool pub_left = (0.5 + ph.beta) != 0.0, pub_right = (0.5 - ph.beta) != 0.0;
  const int Kp = (int)g.Kt;  // trace row stride
  // RP face points per item (same face): the gradient tile entries loaded for one
  // point serve RP rows of M0
  constexpr int RP = S::nfp % 2 == 0 ? 2 : 1;
  for (int item = threadIdx.x; item < (S::next / RP) * E; item += blockDim.x) {
    const int el = item % E, rho0 = (item / E) * RP;
    const int64_t e = e0 + el;
    if (e >= g.K) continue;
    const int s = sNb[D + 1][el], f = rho0 / S::nfp;
    const bool left = g.left[s][f];
    if ((left && !pub_left) || (!left && !pub_right)) continue;
    double q[RP][D * NV];
#pragma unroll
    for (int r = 0; r < RP; ++r)
#pragma unroll
      for (int k = 0; k < D * NV; ++k) q[r][k] = 0.0;
    const double* m0 = O.M0dense + rho0 * S::nsol;
#pragma unroll 2
    for (int sp = 0; sp < S::nsol; ++sp) {
      double m[RP];
#pragma unroll
      for (int r = 0; r < RP; ++r) m[r] = __ldg(m0 + r * S::nsol + sp);
#pragma unroll
      for (int k = 0; k < D * NV; ++k) {
        const double x = sQ[(sp * D * NV + k) * E + el];
#pragma unroll
        for (int r = 0; r < RP; ++r) q[r][k] = fma(m[r], x, q[r][k]);
      }
    }
#pragma unroll
    for (int r = 0; r < RP; ++r) {
      const int rho = rho0 + r;
      double u[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) u[v] = sUe[(rho * NV + v) * E + el];
      const ExtMetric mt = b.xm[s * S::next + rho];
      const double nl[3] = {mt.n0, mt.n1, mt.n2};
      double gv[NV];
      Ph::visc_dir(ph, u, q[r], nl, gv);
#pragma unroll
      for (int v = 0; v < NV; ++v) b.Tg[(rho * NV + v) * Kp + e] = gv[v];
    }
  }
}

template <int D, int P, int EQ, int E>
__global__ void __launch_bounds__(256) ks_stage(GeomDev g, SimplexOps O, PhysDev ph, SimplexBufs b, int stage,
                                                double dt) {
  using Ph = Phys<EQ, D>;
  using S = SDims<D, P>;
  using Ly = SLayout<D, P, Ph::NV, Ph::VISC>;
  constexpr int NV = Ph::NV;
  extern __shared__ double smem[];
  __shared__ int sNb[D + 2][E];  // [f][el] neighbours, [D+1][el] shape
  const int64_t e0 = (int64_t)blockIdx.x * E;
  prologue<D, P, EQ, E>(g, O, ph, b.Uin, b.Tu, smem, sNb, e0);
  double* sU = smem;
  double* sUe = sU + Ly::U * E;
  double* sR0 = sUe + Ly::UE * E;
  double* sUu = sR0 + Ly::R0 * E;
  double* sQ = sUu + Ly::UU * E;
  const int Kp = (int)g.Kt;  // trace row stride
  if constexpr (Ph::VISC) {
    // Q_u = M18 Q (M12 on each of the D*NV gradient rows), into region 0 (C is dead)
    sapply<D * NV, E, false>(O.M12, sQ, 1 << 30, sQ, sR0);
    __syncthreads();
  }
  // internal transformed fluxes for all D components (B7: simplex keeps all), into sQ
  double* sF = sQ;  // [D][nu][NV][E]
  for (int item = threadIdx.x; item < S::nu * E; item += blockDim.x) {
    const int el = item % E, u = item / E;
    const int s = sNb[D + 1][el];
    double uu[NV], qq[Ph::VISC ? D * NV : 1];
#pragma unroll
    for (int v = 0; v < NV; ++v) uu[v] = sUu[(u * NV + v) * E + el];
    if constexpr (Ph::VISC) {
#pragma unroll
      for (int k = 0; k < D * NV; ++k) qq[k] = sR0[(u * D * NV + k) * E + el];
    }
    double fo[D][NV];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      double w[D];
#pragma unroll
      for (int j = 0; j < D; ++j) w[j] = g.detJ[s] * g.Jinv[s][d * 3 + j];
      Ph::conv_dir(ph, uu, w, fo[d]);
      if constexpr (Ph::VISC) {
        double fv[NV];
        Ph::visc_dir(ph, uu, qq, w, fv);
#pragma unroll
        for (int v = 0; v < NV; ++v) fo[d][v] += fv[v];
      }
    }
#pragma unroll
    for (int d = 0; d < D; ++d)
#pragma unroll
      for (int v = 0; v < NV; ++v) sF[((d * S::nu + u) * NV + v) * E + el] = fo[d][v];
  }
  // common fluxes D~ = +/- s F at external points, in place over the own traces
  const double wl = 0.5 + ph.beta, wr = 0.5 - ph.beta;
  for (int item = threadIdx.x; item < S::next * E; item += blockDim.x) {
    const int el = item % E, rho = item / E;
    const int64_t e = e0 + el;
    if (e >= g.K) continue;
    const int s = sNb[D + 1][el], f = rho / S::nfp, q = rho % S::nfp;
    const int m = sNb[f][el];
    const int rho2 = g.nface[s][f] * S::nfp + g.perm[s][f][q];
    const bool left = g.left[s][f];
    double uo[NV], un[NV], gsum[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      un[v] = b.Tu[(rho2 * NV + v) * Kp + m];
      uo[v] = sUe[(rho * NV + v) * E + el];
      gsum[v] = 0.0;
    }
    if constexpr (Ph::VISC) {
      // g_L / g_R published by the left / right element at its own face point
      const int rL = left ? rho : rho2, rR = left ? rho2 : rho;
      const int eL = left ? (int)e : m, eR = left ? m : (int)e;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        double a = 0.0;
        if (wl != 0.0) a = wl * b.Tg[(rL * NV + v) * Kp + eL];
        if (wr != 0.0) a = fma(wr, b.Tg[(rR * NV + v) * Kp + eR], a);
        gsum[v] = a;
      }
    }
    const ExtMetric mt = b.xm[s * S::next + rho];
    const double nl[3] = {mt.n0, mt.n1, mt.n2};
    const double* uL = left ? uo : un;
    const double* uR = left ? un : uo;
    double F[NV];
    Ph::conv_common(ph, uL, uR, nl, F);
    const double sc = left ? mt.s : -mt.s;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double Fv = F[v];
      if constexpr (Ph::VISC) Fv += gsum[v] + ph.eta * (uL[v] - uR[v]);
      sUe[(rho * NV + v) * E + el] = sc * Fv;
    }
  }
  __syncthreads();
  // R~ = [M14 | M13 M19 P2] [D~; F~]  into region 0
  sapply<NV, E, false>(O.M14, sUe, 1 << 30, sUe, sR0);
  sapply<NV, E, true>(O.M13F, sF, 1 << 30, sF, sR0);
  __syncthreads();
  // -R~/detJ and the RK4 update (batched register loads)
  constexpr int TOT = S::nsol * NV * E;
  constexpr int RB_RK = 4;
  const int nth = blockDim.x;
  for (int base0 = threadIdx.x; base0 < TOT; base0 += RB_RK * nth) {
    double a0[RB_RK], a1[RB_RK];
    int64_t gi[RB_RK];
    bool ok[RB_RK];
#pragma unroll
    for (int k = 0; k < RB_RK; ++k) {
      const int idx = base0 + k * nth;
      const int el = idx % E, row = idx / E;
      ok[k] = idx < TOT && e0 + el < g.K;
      gi[k] = (int64_t)row * g.Kp + e0 + el;
      a0[k] = 0.0;
      a1[k] = 0.0;
      if (ok[k]) {
        if (stage >= 1) a0[k] = __ldcs(b.ACC + gi[k]);
        if (stage == 1 || stage == 2) a1[k] = __ldcs(b.U + gi[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < RB_RK; ++k) {
      if (!ok[k]) continue;
      const int idx = base0 + k * nth;
      const int el = idx % E;
      const int s = sNb[D + 1][el];
      const double kk = -sR0[idx] / g.detJ[s];
      double nu;
      switch (stage) {
        case -1: b.out[gi[k]] = kk; nu = 0.0; break;
        case 0: {
          const double u0 = sU[idx];
          b.ACC[gi[k]] = fma(dt / 6.0, kk, u0);
          nu = fma(0.5 * dt, kk, u0);
          b.Us[gi[k]] = nu;
        } break;
        case 1:
          b.ACC[gi[k]] = fma(dt / 3.0, kk, a0[k]);
          nu = fma(0.5 * dt, kk, a1[k]);
          b.Us[gi[k]] = nu;
          break;
        case 2:
          b.ACC[gi[k]] = fma(dt / 3.0, kk, a0[k]);
          nu = fma(dt, kk, a1[k]);
          b.Us[gi[k]] = nu;
          break;
        default:
          nu = fma(dt / 6.0, kk, a0[k]);
          b.U[gi[k]] = nu;
          break;
      }
      sU[idx] = nu;
    }
  }
  if (stage < 0) return;
  __syncthreads();
  strace_global<NV, E>(O.M0, sU, b.Tu_next, e0, g.K, g.Kt);
}

// ------------------------------------------------------------------ launchers
template <int D, int P, int EQ>
struct SCfg {
  static constexpr int E = 16;
  static constexpr int THREADS = 256;
  using Ly = SLayout<D, P, Phys<EQ, D>::NV, Phys<EQ, D>::VISC>;
  static constexpr size_t SMEM = (size_t)Ly::TOTAL * E * sizeof(double);
};

static void sset_smem(const void* k, size_t bytes) {
  if (bytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA smem attr: ") + cudaGetErrorString(e));
  }
}

template <int D, int P, int EQ>
static void srun(const GeomDev& g, const SimplexOps& O, const PhysDev& ph, const SimplexBufs& b, int stage,
                 double dt, cudaStream_t st, int which, const double* U, double* T) {
  using C = SCfg<D, P, EQ>;
  const unsigned grid = (unsigned)((g.K + C::E - 1) / C::E);
  if (which == 0) {
    if constexpr (Phys<EQ, D>::VISC) {
      auto k = ks_grad<D, P, EQ, C::E>;
      sset_smem((const void*)k, C::SMEM);
      k<<<grid, C::THREADS, C::SMEM, st>>>(g, O, ph, b);
    }
  } else if (which == 1) {
    auto k = ks_stage<D, P, EQ, C::E>;
    sset_smem((const void*)k, C::SMEM);
    k<<<grid, C::THREADS, C::SMEM, st>>>(g, O, ph, b, stage, dt);
  } else {
    auto k = ks_traces<D, P, EQ, C::E>;
    const size_t sm = (size_t)SDims<D, P>::nsol * Phys<EQ, D>::NV * C::E * sizeof(double);
    sset_smem((const void*)k, sm);
    k<<<grid, C::THREADS, sm, st>>>(g, O, U, T);
  }
}

typedef void (*SFn)(const GeomDev&, const SimplexOps&, const PhysDev&, const SimplexBufs&, int, double,
                    cudaStream_t, int, const double*, double*);

template <int D, int P>
static SFn spick_eq(int eq) {
  switch (eq) {
    case EQ_LINADV: return srun<D, P, EQ_LINADV>;
    case EQ_LINADVDIFF: return srun<D, P, EQ_LINADVDIFF>;
    case EQ_EULER: return srun<D, P, EQ_EULER>;
    case EQ_NS: return srun<D, P, EQ_NS>;
  }
  return nullptr;
}

static SFn spick(int D, int P, int eq) {
  if (D == 2) {
    switch (P) {
      case 1: return spick_eq<2, 1>(eq);
      case 2: return spick_eq<2, 2>(eq);
      case 3: return spick_eq<2, 3>(eq);
      case 4: return spick_eq<2, 4>(eq);
    }
  } else {
    switch (P) {
      case 1: return spick_eq<3, 1>(eq);
      case 2: return spick_eq<3, 2>(eq);
      case 3: return spick_eq<3, 3>(eq);
    }
  }
  return nullptr;
}

bool simplex_supported(int D, int P, int eq) { return spick(D, P, eq) != nullptr; }

void simplex_launch_traces(int D, int P, int eq, const GeomDev& g, const SimplexOps& O, const double* U,
                           double* Tu, cudaStream_t st) {
  SimplexBufs b{};
  PhysDev ph{};
  spick(D, P, eq)(g, O, ph, b, 0, 0.0, st, 2, U, Tu);
}

void simplex_launch_grad(int D, int P, int eq, const GeomDev& g, const SimplexOps& O, const PhysDev& ph,
                         const SimplexBufs& b, cudaStream_t st) {
  spick(D, P, eq)(g, O, ph, b, 0, 0.0, st, 0, nullptr, nullptr);
}

void simplex_launch_flux(int D, int P, int eq, const GeomDev& g, const SimplexOps& O, const PhysDev& ph,
                         const SimplexBufs& b, int stage, double dt, cudaStream_t st) {
  spick(D, P, eq)(g, O, ph, b, stage, dt, st, 1, nullptr, nullptr);
}

}  // namespace sdrt
