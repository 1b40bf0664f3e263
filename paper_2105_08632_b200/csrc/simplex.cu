// Fused SDRT stage for simplex elements (tri / tet) on sm_100a, fp64.
//
// Simplex operators are dense (App. B l.2855-2925, B7: all N_D components per unique
// internal point, l.2927-2932), so every App. B product is a small dense matrix times
// a tile of E elements held in shared memory as [row][var][E] (element fastest, the
// ABI layout): Y[r][n] = sum_c M[r][c] X[c][n], n = (var, element).  These products
// run on the FP64 tensor cores (mma.sync m8n8k4 f64, DMMA): operator fragments come
// from a fragment-ordered copy in global memory (L1-resident), tile fragments from
// shared memory; each output is accumulated in the fixed k order, so the same product
// on the same data gives the same bits wherever it is evaluated (the own trace
// recomputed by an element equals the trace it published, O28).
//
//   kernel A (viscous, "volume"): U_ext = M0 U, U_u = M12 U, C (l.282-291, neighbour
//     traces), Q~ = [M16 | M15 P][C; U_u] (l.2877-2880), Q = J^-T Q~ (l.299-302), the
//     published viscous normal flux g = n_L . f^v(u, M0 Q) at the face points of the
//     LDG-weighted side (l.330-335), Q_u = M18 Q (l.2897-2900), internal fluxes
//     F~ = detJ J^-1 (f^c - f^v) (l.305-311), R_int = M13 M19 P2 F~ -> HBM.
//   kernel B ("faces + update"): U_ext = M0 U, common fluxes D~ = +/- s F (l.312-340,
//     canonical L/R), R~ = R_int + M14 D~ (l.2919-2925) [inviscid: U_u, F~ and M13 F~
//     here too], -R~/detJ, RK4 update, new traces M0 U_new.
// Tiles arrive by TMA; face values are exchanged only through double-buffered traces,
// stored point-major [N_ext][K_t][N_V] (a neighbour's N_V values at one face point are
// contiguous, so the scattered neighbour gathers touch 1-2 sectors instead of N_V).
#include <cuda_runtime.h>

#include <cstring>
#include <stdexcept>
#include <string>

#include "simplex.cuh"
#include "rk.cuh"
#include "tma.cuh"
#include "diag.cuh"

namespace sdrt {

// Optional per-phase cycle accounting (build with -DSDRT_PHASE_PROF; tools only)
#ifdef SDRT_PHASE_PROF
__device__ unsigned long long g_sphase_cycles[2][16];
#define SPH_INIT long long ph_t0 = clock64();
#define SPH(kern, k)                                                           \
  if (threadIdx.x == 0) {                                                      \
    const long long ph_t1 = clock64();                                         \
    atomicAdd(&g_sphase_cycles[kern][k], (unsigned long long)(ph_t1 - ph_t0)); \
    ph_t0 = ph_t1;                                                             \
  }
#else
#define SPH_INIT
#define SPH(kern, k)
#endif

template <int D, int P>
struct SDims {
  static constexpr int nsol = D == 2 ? (P + 1) * (P + 2) / 2 : (P + 1) * (P + 2) * (P + 3) / 6;
  static constexpr int next = D == 2 ? 3 * (P + 1) : 2 * (P + 1) * (P + 2);
  static constexpr int nu = D == 2 ? P * (P + 1) / 2 : P * (P + 1) * (P + 2) / 6;
  static constexpr int nfaces = D + 1;
  static constexpr int nfp = next / nfaces;
  // k steps (columns / 4) of the packed operators
  static constexpr int kt_sol = (nsol + 3) / 4;          // M0, M12 (columns: solution points)
  static constexpr int kt_G = (next + nu + 3) / 4;       // [M16 | M15 P]
  static constexpr int kt_ext = (next + 3) / 4;          // M14
  static constexpr int kt_F = (D * nu + 3) / 4;          // M13 M19 P2
  static constexpr int kt_GF = (next + nsol + 3) / 4;    // FR-SDRT [M16 | Dsol - M16 M0]
  static constexpr int kt_FF = (D * nsol + 3) / 4;       // FR-SDRT divergence on F[s][d]
  static constexpr int kt_EF = (next + D * nu + 3) / 4;   // [M14 | M13F]
  static constexpr int kt_EFF = (next + D * nsol + 3) / 4;  // FR-SDRT [M14 | M13F]
};

template <typename T>
__host__ __device__ constexpr T cmax(T a, T b) { return a > b ? a : b; }
template <class T>
__host__ __device__ constexpr T cmin(T a, T b) { return a < b ? a : b; }

struct STileMaps {
  CUtensorMap uin, un, acc, rint;
};

// ---------------------------------------------------------------- DMMA products
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// n-tiles per warp job: one A fragment serves NGR MMAs; small groups give every warp of
// the CTA a job in the short products (n = number of 8-column tiles)
#ifndef SDRT_NGR_MODE
#define SDRT_NGR_MODE 0
#endif
#ifndef SDRT_SA_MINB
#define SDRT_SA_MINB 3
#endif
#ifndef SDRT_SB_MINB
#define SDRT_SB_MINB 4
#endif
#ifndef SDRT_SA_QCH
#define SDRT_SA_QCH 1024
#endif
// OSF kernel A: publish items compacted to the tile's left-face points (1) or all face
// points with the right-face lanes idle (0).  Measured on c5: compacted 3.78 ms vs 3.13 ms
// per kernel-A launch -- the compacted lanes walk one element's points (shared-memory
// stride N_V D E between lanes: bank conflicts on every gradient load) where the
// uncompacted lanes read consecutive elements; off
#ifndef SDRT_SA_PCOMP
#define SDRT_SA_PCOMP 0
#endif
// kernel A tiles formed in shared memory padded to a row stride of N + 4 (SLayoutA):
// removes the 2-way bank conflicts of the B-fragment loads (c5: 169 M of 519 M shared
// wavefronts), but the padded tiles need 75.8 KB per CTA (two CTAs per SM) or a
// two-chunk Q_ext (three CTAs); measured on c5 kernel A: unpadded 3.13 ms, padded at two
// CTAs / SM 3.13 ms (256 threads) / 3.63-3.66 ms (320 / 384), padded two-chunk 3.55 ms
// (unpadded two-chunk 3.65 ms): off
#ifndef SDRT_SA_PAD
#define SDRT_SA_PAD 0
#endif
#ifndef SDRT_SA_QCHP
#define SDRT_SA_QCHP 32
#endif
#ifndef SDRT_SA_NT
#define SDRT_SA_NT 256
#endif
#ifndef SDRT_SB_PF
#define SDRT_SB_PF 1
#endif
#ifndef SDRT_SB_REV
#define SDRT_SB_REV 0
#endif
#ifndef SDRT_SB_NT
#define SDRT_SB_NT 160
#endif
// kernel B: the RK update as the epilogue of the last divergence product (1) or a separate
// pass over the R~ tile after a barrier (0).  Measured: c5 kernel B 1.47 -> 1.74 ms, c2
// 16.1 -> 11.6 GDOF-stage/s with the epilogue -- the product has only N_sol/8 x 1 warp
// jobs (3 for tet p = 3), so the RK update of the tile lands on 3 of the CTA's warps: off
#ifndef SDRT_SB_EPI
#define SDRT_SB_EPI 0
#endif
// inviscid kernel B: the divergence as one [M14 | M13F] product (1) or two (0)
#ifndef SDRT_SB_ONEPRODUCT
#define SDRT_SB_ONEPRODUCT 1
#endif
#ifndef SDRT_SB_MINB_OSF
#define SDRT_SB_MINB_OSF 4
#endif
// OSF kernel B: whole shared-memory carve-out (5 CTAs / SM instead of 4); measured slower
// on c5 (B 1.49 -> 1.57 ms: the smaller L1 serves the flux gathers worse), off
#ifndef SDRT_SB_CARVE
#define SDRT_SB_CARVE 0
#endif
#ifndef SDRT_SPLIT_INTFLUX
#define SDRT_SPLIT_INTFLUX 0
#endif
#ifndef SDRT_S_E2D
#define SDRT_S_E2D 4
#endif
__host__ __device__ constexpr int ngroup(int n) {
  return SDRT_NGR_MODE == 1   ? (n % 3 == 0 && n > 5 ? 3 : (n % 2 == 0 && n > 5 ? 2 : 1))
         : SDRT_NGR_MODE == 2 ? (n <= 15 ? n : (n % 5 == 0 ? 5 : 1))
                              : (n % 5 == 0 ? 5 : (n % 4 == 0 ? 4 : (n % 3 == 0 ? 3 : (n % 2 == 0 ? 2 : 1))));
}

// One operator application Y (+)= M X over a tile: X rows c < split from X0, others
// from X1 (row stride N = W E doubles); Y rows r < M.rows.  Warp jobs = (m-tile,
// group of NGR n-tiles).  KT (k steps) is a compile-time constant: all A fragments
// of a job are requested at once (one L1/L2 round trip per job), then the MMAs run.
// XR: row stride of the X tiles (N, or N + 4 for the padded tiles of kernel A: with
// N = 40 the four k-rows a half-warp reads for a 64-bit B fragment fall on the same 8
// banks twice; a stride of 44 puts them on four disjoint bank windows)
template <int W, int E, int KT, int YS = W * E, int XR = W * E>
struct Dmm {
  static constexpr int N = W * E;
  static_assert(N % 8 == 0, "tile columns must be a multiple of 8");
  static_assert(KT <= 32, "k-step mask");
  static constexpr int NT8 = N / 8;
  static constexpr int NGR = ngroup(NT8);
  static constexpr int NG = NT8 / NGR;

  __device__ __forceinline__ static int jobs(const SOpF& M) { return M.mt * NG; }

  // Y rows at stride YS doubles (YS > N: interleaved outputs of several products)
  template <bool ACCUM>
  __device__ __forceinline__ static void job(const SOpF& M, int j, const double* X0, int split, const double* X1,
                                             double* Y) {
    const int lane = threadIdx.x & 31;
    const int m = j / NG, ng = j % NG;
    const int n0 = ng * NGR * 8 + (lane >> 2);
    const unsigned km = M.kmask ? __ldg(M.kmask + m) : 0xffffffffu;  // structurally zero blocks skipped
    const double* af = M.frag + (int64_t)m * KT * 32 + lane;
    double a[KT];
#pragma unroll
    for (int k = 0; k < KT; ++k) a[k] = (km >> k & 1u) ? __ldg(af + k * 32) : 0.0;
    double c[NGR][2];
#pragma unroll
    for (int q = 0; q < NGR; ++q) c[q][0] = c[q][1] = 0.0;
#pragma unroll
    for (int k = 0; k < KT; ++k) {
      if (!(km >> k & 1u)) continue;
      const int col = 4 * k + (lane & 3);
      const double* xr = col < split ? X0 + col * XR : X1 + (col - split) * XR;
      const bool ok = col < M.cols;
#pragma unroll
      for (int q = 0; q < NGR; ++q) {
        const double b = ok ? xr[n0 + 8 * q] : 0.0;
        dmma(c[q][0], c[q][1], a[k], b);
      }
    }
    const int r = 8 * m + (lane >> 2);
    if (r < M.rows) {
#pragma unroll
      for (int q = 0; q < NGR; ++q) {
        double2* y = reinterpret_cast<double2*>(Y + r * YS + ng * NGR * 8 + 8 * q + 2 * (lane & 3));
        if (ACCUM) {
          const double2 o = *y;
          *y = make_double2(o.x + c[q][0], o.y + c[q][1]);
        } else {
          *y = make_double2(c[q][0], c[q][1]);
        }
      }
    }
  }
};

// Y1 = M1 X1 (W1 per row, KT1 k steps) and Y2 = M2 X2 (W2, KT2) in one phase
// (independent products; M2.frag == nullptr skips the second)
template <int W1, int KT1, int W2, int KT2, int E, bool ACC1, bool ACC2, int YS1 = W1 * E, int YS2 = W2 * E>
__device__ __forceinline__ void dmm2(const SOpF& M1, const double* X1a, int s1, const double* X1b, double* Y1,
                                     const SOpF& M2, const double* X2a, int s2, const double* X2b, double* Y2) {
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int j1 = Dmm<W1, E, KT1, YS1>::jobs(M1), j2 = M2.frag ? Dmm<W2, E, KT2, YS2>::jobs(M2) : 0;
  for (int j = warp; j < j1 + j2; j += nw) {
    if (j < j1) Dmm<W1, E, KT1, YS1>::template job<ACC1>(M1, j, X1a, s1, X1b, Y1);
    else Dmm<W2, E, KT2, YS2>::template job<ACC2>(M2, j - j1, X2a, s2, X2b, Y2);
  }
}

template <int W, int KT, int E, bool ACC, int XR = W * E, int YS = W * E>
__device__ __forceinline__ void dmm1(const SOpF& M, const double* X0, int split, const double* X1, double* Y) {
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  using DM = Dmm<W, E, KT, YS, XR>;
  const int nj = DM::jobs(M);
  for (int j = warp; j < nj; j += nw) DM::template job<ACC>(M, j, X0, split, X1, Y);
}

// Y = M X (+ Yacc) with the result handed to an epilogue per lane output pair instead of
// shared memory: epi(r, n, y_n, y_n+1) for row r and the even column n (fused GEMM
// epilogue: the RK update runs on the product's registers, one barrier and the R~ tile
// round trip fewer)
template <int W, int KT, int E, bool ACC, class Epi>
__device__ __forceinline__ void dmm1_epi(const SOpF& M, const double* X0, int split, const double* X1,
                                         const double* Yacc, Epi&& epi) {
  using DM = Dmm<W, E, KT>;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int j = warp; j < DM::jobs(M); j += nw) {
    const int m = j / DM::NG, ng = j % DM::NG;
    const int n0 = ng * DM::NGR * 8 + (lane >> 2);
    const unsigned km = M.kmask ? __ldg(M.kmask + m) : 0xffffffffu;
    const double* af = M.frag + (int64_t)m * KT * 32 + lane;
    double a[KT];
#pragma unroll
    for (int k = 0; k < KT; ++k) a[k] = (km >> k & 1u) ? __ldg(af + k * 32) : 0.0;
    double c[DM::NGR][2];
#pragma unroll
    for (int q = 0; q < DM::NGR; ++q) c[q][0] = c[q][1] = 0.0;
#pragma unroll
    for (int k = 0; k < KT; ++k) {
      if (!(km >> k & 1u)) continue;
      const int col = 4 * k + (lane & 3);
      const double* xr = col < split ? X0 + col * DM::N : X1 + (col - split) * DM::N;
      const bool ok = col < M.cols;
#pragma unroll
      for (int q = 0; q < DM::NGR; ++q) dmma(c[q][0], c[q][1], a[k], ok ? xr[n0 + 8 * q] : 0.0);
    }
    const int r = 8 * m + (lane >> 2);
    if (r < M.rows) {
#pragma unroll
      for (int q = 0; q < DM::NGR; ++q) {
        const int n = ng * DM::NGR * 8 + 8 * q + 2 * (lane & 3);
        double y0 = c[q][0], y1 = c[q][1];
        if (ACC) {
          const double2 o = *reinterpret_cast<const double2*>(Yacc + r * DM::N + n);
          y0 = o.x + y0;
          y1 = o.y + y1;
        }
        epi(r, n, y0, y1);
      }
    }
  }
}

// RK update of one value (rk.cuh stage codes): kk = dU/dt, idx its tile entry, gi its
// global entry; returns the new stage value (0 for the residual-only stage -1)
__device__ __forceinline__ double rk_value(const SimplexBufs& b, int stage, double dt, double kk, int64_t gi,
                                           const double* sU, const double* sAcc, const double* sUn, int idx) {
  double nu;
  switch (stage) {
    case -1: b.out[gi] = kk; nu = 0.0; break;
    case 0: {
      const double u0 = sU[idx];
      b.ACC[gi] = fma(dt / 6.0, kk, u0);
      nu = fma(0.5 * dt, kk, u0);
      b.Us[gi] = nu;
    } break;
    case 1:
      b.ACC[gi] = fma(dt / 3.0, kk, sAcc[idx]);
      nu = fma(0.5 * dt, kk, sUn[idx]);
      b.Us[gi] = nu;
      break;
    case 2:
      b.ACC[gi] = fma(dt / 3.0, kk, sAcc[idx]);
      nu = fma(dt, kk, sUn[idx]);
      b.Us[gi] = nu;
      break;
    case 3:
      nu = fma(dt / 6.0, kk, sAcc[idx]);
      b.U[gi] = nu;
      break;
    default: {  // RK54 stage s (2N-storage, in place)
      const int s5 = stage - RK54_STAGE0;
      const double du = s5 == 0 ? dt * kk : fma(rk54_a(s5), sAcc[idx], dt * kk);
      b.ACC[gi] = du;
      nu = fma(rk54_b(s5), du, sU[idx]);
      b.U[gi] = nu;
    } break;
  }
  return nu;
}

// the same operator on the ND row blocks of a [nd][rows][W][E] tile (block stride XS
// doubles), written interleaved as Y[r][nd][W][E]: one job pool for all blocks
template <int W, int KT, int E, int ND, int XR = W * E>
__device__ __forceinline__ void dmm_blocks(const SOpF& M, const double* X, int XS, double* Y) {
  using DM = Dmm<W, E, KT, ND * W * E, XR>;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nj = DM::jobs(M);
  for (int j = warp; j < ND * nj; j += nw) {
    const int d = j / nj;
    DM::template job<false>(M, j % nj, X + d * XS, 1 << 30, X + d * XS, Y + d * W * E);
  }
}

// Y = M X with the result rows written straight from the MMA fragments to global
// memory, G[(r W + w) ld + e0 + el] (element-major ABI layout, 16-byte stores), for
// e0 + el < K.  Saves the shared-memory round trip and a barrier for final products.
template <int W, int KT, int E, bool POINT_MAJOR = false, int XR = W * E>
__device__ __forceinline__ void dmm1_global(const SOpF& M, const double* X, double* __restrict__ Gout, int64_t ld,
                                            int64_t e0, int64_t K) {
  using DM = Dmm<W, E, KT, W * E, XR>;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int j = warp; j < DM::jobs(M); j += nw) {
    const int m = j / DM::NG, ng = j % DM::NG;
    const int n0 = ng * DM::NGR * 8 + (lane >> 2);
    const double* af = M.frag + (int64_t)m * KT * 32 + lane;
    const unsigned km = M.kmask ? __ldg(M.kmask + m) : 0xffffffffu;
    double a[KT];
#pragma unroll
    for (int k = 0; k < KT; ++k) a[k] = (km >> k & 1u) ? __ldg(af + k * 32) : 0.0;
    double c[DM::NGR][2];
#pragma unroll
    for (int q = 0; q < DM::NGR; ++q) c[q][0] = c[q][1] = 0.0;
#pragma unroll
    for (int k = 0; k < KT; ++k) {
      if (!(km >> k & 1u)) continue;
      const int col = 4 * k + (lane & 3);
      const bool ok = col < M.cols;
#pragma unroll
      for (int q = 0; q < DM::NGR; ++q) dmma(c[q][0], c[q][1], a[k], ok ? X[col * XR + n0 + 8 * q] : 0.0);
    }
    const int r = 8 * m + (lane >> 2);
    if (r < M.rows) {
#pragma unroll
      for (int q = 0; q < DM::NGR; ++q) {
        const int n = ng * DM::NGR * 8 + 8 * q + 2 * (lane & 3);  // column (w, el), el even
        const int w = n / E, el = n % E;
        if constexpr (POINT_MAJOR) {  // trace layout [row][element][w]
          double* gp = Gout + ((int64_t)r * ld + e0 + el) * W + w;
          if (e0 + el < K) gp[0] = c[q][0];
          if (e0 + el + 1 < K) gp[W] = c[q][1];
        } else {  // ABI layout [row][w][element]
          double* gp = Gout + ((int64_t)r * W + w) * ld + e0 + el;
          if (e0 + el + 1 < K) *reinterpret_cast<double2*>(gp) = make_double2(c[q][0], c[q][1]);
          else if (e0 + el < K) gp[0] = c[q][0];
        }
      }
    }
  }
}

// entry M[r][c] of a fragment-packed operator
__device__ __forceinline__ double sop_at(const SOpF& M, int r, int c) {
  return __ldg(M.frag + ((int64_t)(r / 8) * M.kt + c / 4) * 32 + (r % 8) * 4 + c % 4);
}

// ---------------------------------------------------------------- tile helpers
// neighbour of element e across local face f (pattern arithmetic, periodic)
template <int D>
__device__ __forceinline__ int snbr(const GeomDev& g, int e, int s, int f) {
  // pattern coordinates in registers (no dynamically indexed local array)
  const int pat = e / g.nsub;
  const int c0 = pat % g.Nloc[0];
  const int r = pat / g.Nloc[0];
  const int c1 = D == 2 ? r : r % g.Nloc[1];
  const int c2 = D == 2 ? 0 : r / g.Nloc[1];
  int cc[3] = {c0 + g.off[s][f][0], c1 + g.off[s][f][1], D == 3 ? c2 + g.off[s][f][2] : 0};
  const int cs[3] = {c0, c1, c2};
#pragma unroll
  for (int d = 0; d < D; ++d)
    if ((cc[d] < 0 || cc[d] >= g.Nloc[d]) && g.halo[d]) {
      // ghost column: slab (d, side), tangential pattern index, neighbour sub-cell
      const int a = d == 0 ? 1 : 0, bb = d == 2 ? 1 : 2;
      const int tang = D == 2 ? cs[a] : cs[a] + g.Nloc[a] * cs[bb];
      return (int)g.gbase[d][cc[d] < 0 ? 0 : 1] + tang * g.nsub + g.nshape[s][f];
    }
#pragma unroll
  for (int d = 0; d < D; ++d) cc[d] = cc[d] < 0 ? cc[d] + g.Nloc[d] : (cc[d] >= g.Nloc[d] ? cc[d] - g.Nloc[d] : cc[d]);
  const int id = D == 2 ? cc[0] + g.Nloc[0] * cc[1] : cc[0] + g.Nloc[0] * (cc[1] + g.Nloc[1] * cc[2]);
  return id * g.nsub + g.nshape[s][f];
}

// neighbour ids sNb[f][el] and sub-cell shapes sNb[D+1][el] of a tile, once
template <int D, int E>
__device__ __forceinline__ void fill_neighbours(const GeomDev& g, int (*sNb)[E], int64_t e0) {
  for (int idx = threadIdx.x; idx < (D + 2) * E; idx += blockDim.x) {
    const int el = idx % E, f = idx / E;
    const int e = (int)e0 + el;
    const int s = e % g.nsub;
    sNb[f][el] = f == D + 1 ? s : (e < g.K ? snbr<D>(g, e, s, f) : 0);
  }
}

// C = (1/2 - b) u_L + (1/2 + b) u_R at external points into sC [next][NV][E].  Items
// (rho, el) are statically owned (item tid + k NT); NbGather::load issues every
// neighbour-trace load of this thread at the kernel start, so the gathers overlap
// the tile load and the first products.
template <int D, int P, int NV, int E, int NT>
struct NbGather {
  using S = SDims<D, P>;
  static constexpr int ITEMS = S::next * E;
  static constexpr int CI = (ITEMS + NT - 1) / NT;
  double nb[CI][NV];

  __device__ __forceinline__ void load(const GeomDev& g, const PhysDev& ph, const double* __restrict__ Tu,
                                       const int (*sNb)[E], int64_t e0) {
    const int Kp = (int)g.Kt;  // trace row stride
    const double wl = 0.5 - ph.beta, wr = 0.5 + ph.beta;
#pragma unroll
    for (int k = 0; k < CI; ++k) {
      const int item = threadIdx.x + k * NT;
      const int el = item % E, rho = item / E;
#pragma unroll
      for (int v = 0; v < NV; ++v) nb[k][v] = 0.0;
      if (item >= ITEMS || e0 + el >= g.K) continue;
      const int s = sNb[D + 1][el], f = rho / S::nfp, q = rho % S::nfp;
      // the neighbour is u_R on a face where this element is left, else u_L; a neighbour
      // whose LDG weight is 0 is not read (its trace may be stale under OSF)
      if ((g.left[s][f] ? wr : wl) == 0.0) continue;
      const int m = sNb[f][el];
      const int rho2 = g.nface[s][f] * S::nfp + g.perm[s][f][q];
#pragma unroll
      for (int v = 0; v < NV; ++v) nb[k][v] = Tu[((int64_t)rho2 * Kp + m) * NV + v];
    }
  }

  template <int CR = NV * E>  // row stride of sC
  __device__ __forceinline__ void common_values(const GeomDev& g, const PhysDev& ph, const double* sUe,
                                                const int (*sNb)[E], double* sC, int64_t e0) const {
    const double wl = 0.5 - ph.beta, wr = 0.5 + ph.beta;
#pragma unroll
    for (int k = 0; k < CI; ++k) {
      const int item = threadIdx.x + k * NT;
      const int el = item % E, rho = item / E;
      if (item >= ITEMS) break;
      if (e0 + el >= g.K) {
#pragma unroll
        for (int v = 0; v < NV; ++v) sC[rho * CR + v * E + el] = 0.0;
        continue;
      }
      const int s = sNb[D + 1][el], f = rho / S::nfp;
      const bool left = g.left[s][f];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const double own = sUe[(rho * NV + v) * E + el];
        const double uL = left ? own : nb[k][v], uR = left ? nb[k][v] : own;
        sC[rho * CR + v * E + el] = __fma_rn(wr, uR, __dmul_rn(wl, uL));  // explicit: same bits both sides
      }
    }
  }
};

// Kernel B's face gathers issued ahead (register prefetch, SDRT_SB_PF): the
// neighbour's U trace and the LDG-weighted published viscous traces g of each of the
// thread's external points, loaded before the tile wait so the latency overlaps it.
template <int D, int P, int NV, int E, int NT, bool VISC>
struct FluxGather {
  using S = SDims<D, P>;
  static constexpr int ITEMS = S::next * E;
  static constexpr int CI = (ITEMS + NT - 1) / NT;
  double un[CI][NV];
  double gs[VISC ? CI : 1][NV];

  __device__ __forceinline__ void load(const GeomDev& g, const PhysDev& ph, const double* __restrict__ Tu,
                                       const double* __restrict__ Tg, const int (*sNb)[E], int64_t e0) {
    const int Kp = (int)g.Kt;
    const double wl = 0.5 + ph.beta, wr = 0.5 - ph.beta;
#pragma unroll
    for (int k = 0; k < CI; ++k) {
      const int item = threadIdx.x + k * NT;
      const int el = item % E, rho = item / E;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        un[k][v] = 0.0;
        if constexpr (VISC) gs[k][v] = 0.0;
      }
      if (item >= ITEMS || e0 + el >= g.K) continue;
      const int s = sNb[D + 1][el], f = rho / S::nfp, q = rho % S::nfp;
      const int m = sNb[f][el];
      const int rho2 = g.nface[s][f] * S::nfp + g.perm[s][f][q];
#pragma unroll
      for (int v = 0; v < NV; ++v) un[k][v] = Tu[((int64_t)rho2 * Kp + m) * NV + v];
      if constexpr (VISC) {
        const bool left = g.left[s][f];
        const int64_t e = e0 + el;
        const int rL = left ? rho : rho2, rR = left ? rho2 : rho;
        const int64_t eL = left ? e : m, eR = left ? m : e;
        // one published side (beta = +-1/2): its raw g by a predicated load nothing
        // consumes here (weighted at use); two sides: combined now
        const bool one = (wl == 0.0) != (wr == 0.0);
        const int64_t gi = one ? (wl != 0.0 ? (int64_t)rL * Kp + eL : (int64_t)rR * Kp + eR) : 0;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          if (one) {
            gs[k][v] = Tg[gi * NV + v];
          } else {
            gs[k][v] = Phys<EQ_NS, D>::gsum_rn(wl, Tg[((int64_t)rL * Kp + eL) * NV + v], wr,
                                               Tg[((int64_t)rR * Kp + eR) * NV + v]);
          }
        }
      }
    }
  }
};

// Q = J^-T Q~ in place on sQ [D][nsol][NV][E]
template <int D, int P, int NV, int E, int QR = NV * E>  // QR: row stride of sQ
__device__ __forceinline__ void metric_grad(const GeomDev& g, const int (*sNb)[E], double* sQ) {
  using S = SDims<D, P>;
  for (int item = threadIdx.x; item < S::nsol * E; item += blockDim.x) {
    const int el = item % E, sp = item / E;
    const int s = sNb[D + 1][el];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double qt[D];
#pragma unroll
      for (int d = 0; d < D; ++d) qt[d] = sQ[(d * S::nsol + sp) * QR + v * E + el];
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) acc = fma(g.Jinv[s][j * 3 + i], qt[j], acc);
        sQ[(i * S::nsol + sp) * QR + v * E + el] = acc;
      }
    }
  }
}

// internal transformed fluxes for all D components (B7: simplices keep all) at the
// unique internal points: F~[d][u] = detJ (J^-1 (f^c - f^v))_d -> sF [D][nu][NV][E]
template <int D, int P, int EQ, int E, int UR = Phys<EQ, D>::NV * E, int FR = Phys<EQ, D>::NV * E>
__device__ __forceinline__ void internal_fluxes(const GeomDev& g, const PhysDev& ph, const int (*sNb)[E],
                                                const double* sUu, const double* sQu, double* sF, int64_t e0) {
  using Ph = Phys<EQ, D>;
  using S = SDims<D, P>;
  constexpr int NV = Ph::NV;
  constexpr int ND = SDRT_SPLIT_INTFLUX ? D : 1;  // items per point: one per direction, or all
  for (int item = threadIdx.x; item < S::nu * ND * E; item += blockDim.x) {
    const int el = item % E, r = item / E, u = r % S::nu, dsel = r / S::nu;
    if (e0 + el >= g.K) {  // padding columns: finite zeros
#pragma unroll
      for (int d = 0; d < D; ++d)
        if (ND == 1 || d == dsel)
#pragma unroll
          for (int v = 0; v < NV; ++v) sF[(d * S::nu + u) * FR + v * E + el] = 0.0;
      continue;
    }
    const int s = sNb[D + 1][el];
    double uu[NV], qq[Ph::VISC ? D * NV : 1];
#pragma unroll
    for (int v = 0; v < NV; ++v) uu[v] = sUu[u * UR + v * E + el];
    if constexpr (Ph::VISC) {
#pragma unroll
      for (int k = 0; k < D * NV; ++k) qq[k] = sQu[(u * D * NV + k) * E + el];
    }
#pragma unroll
    for (int d = 0; d < D; ++d) {
      if (ND != 1 && d != dsel) continue;
      double w[D], fo[NV];
#pragma unroll
      for (int j = 0; j < D; ++j) w[j] = g.detJ[s] * g.Jinv[s][d * 3 + j];
      Ph::conv_dir(ph, uu, w, fo);
      if constexpr (Ph::VISC) {
        double fv[NV];
        Ph::visc_dir(ph, uu, qq, w, fv);
#pragma unroll
        for (int v = 0; v < NV; ++v) fo[v] += fv[v];
      }
#pragma unroll
      for (int v = 0; v < NV; ++v) sF[(d * S::nu + u) * FR + v * E + el] = fo[v];
    }
  }
}

// ---------------------------------------------------------------- kernels
template <int D, int P, int EQ, int E>
__global__ void __launch_bounds__(256) ks_traces(GeomDev g, SimplexOps O, const __grid_constant__ STileMaps tm,
                                                 double* __restrict__ T) {
  pdl_wait();
  using S = SDims<D, P>;
  constexpr int NV = Phys<EQ, D>::NV;
  extern __shared__ __align__(128) double smem[];
  double* sU = smem;
  double* sUe = smem + S::nsol * NV * E;
  __shared__ __align__(8) uint64_t bar;
  const int64_t e0 = (int64_t)(g.tiles ? g.tiles[blockIdx.x] : (int)blockIdx.x) * E;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
    mbar_expect_tx(&bar, S::nsol * NV * E * 8);
    tma_tile<S::nsol * NV, E>(sU, &tm.uin, e0, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  dmm1_global<NV, S::kt_sol, E, true>(O.M0, sU, T, g.Kt, e0, g.K);
}

// Kernel A.  Shared-memory regions (doubles per element) by liveness:
//   X  [max(nsol NV, next D NV, D nu NV)]: U, then C, then Q_ext, then F~
//   UE [max(next NV, nu D NV)]: U_ext, then Q_u
//   UU [nu NV]: U_u
//   Q  [nsol D NV]: Q, then R_int (nsol NV)
template <int D, int P, int NV, int E>
struct SLayoutA {
  using S = SDims<D, P>;
  static constexpr int N = NV * E;  // columns (variable, element) of a tile row
  // row stride of the tiles read as DMMA B operands after being formed in shared memory
  // (C, U_u, Q, F~): N + 4 with SDRT_SA_PAD (conflict-free B fragments, see Dmm); the
  // stage-input tile U arrives by TMA and keeps N
  static constexpr int RS = SDRT_SA_PAD ? N + 4 : N;
  // Q_ext is formed and published in chunks of QCH external points (whole 8-row
  // m-tiles of M0), so region X holds one chunk (smaller with padding: 3 CTAs / SM)
  static constexpr int QCH = cmin(SDRT_SA_PAD ? SDRT_SA_QCHP : SDRT_SA_QCH, (S::next + 7) / 8 * 8);
  // region sizes in doubles per tile
  static constexpr int X = cmax(cmax(cmax(S::nsol * N, S::next * RS), QCH * D * N), D * S::nu * RS);
  static constexpr int UE = cmax(S::next * N, S::nu * D * N);
  static constexpr int UU = S::nu * RS;
  static constexpr int Q = D * S::nsol * RS;
  static constexpr int TOTAL = X + UE + UU + Q;
};

// OSF (one-sided flux publication, NS with beta = +1/2; tensor.cu publish_F): at the
// face points where this element is LEFT it evaluates the face's whole common flux
// F = Rusanov(u_L, u_R) + g_L + eta (u_L - u_R) (l.312-340) and publishes F instead of g;
// kernel B (ks_stage_osf) then applies M14 to +/- s F gathered from the two sides.
template <int D, int P, int EQ, int E, bool OSF = false>
__global__ void __launch_bounds__(SDRT_SA_NT, SDRT_SA_MINB) ks_grad(GeomDev g, SimplexOps O, PhysDev ph, SimplexBufs b,
                                               const __grid_constant__ STileMaps tm) {
  pdl_wait();
  SPH_INIT
  using Ph = Phys<EQ, D>;
  using S = SDims<D, P>;
  using Ly = SLayoutA<D, P, Ph::NV, E>;
  constexpr int NV = Ph::NV, RS = Ly::RS;
  extern __shared__ __align__(128) double smem[];
  double* sX = smem;
  double* sUe = sX + Ly::X;
  double* sUu = sUe + Ly::UE;
  double* sQ = sUu + Ly::UU;
  __shared__ int sNb[D + 2][E];  // [f][el] neighbours, [D+1][el] shape
  __shared__ __align__(8) uint64_t bar;
  const int64_t e0 = (int64_t)(g.tiles ? g.tiles[blockIdx.x] : (int)blockIdx.x) * E;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
    mbar_expect_tx(&bar, S::nsol * NV * E * 8);
    tma_tile<S::nsol * NV, E>(sX, &tm.uin, e0, &bar);
  }
  fill_neighbours<D, E>(g, sNb, e0);
  __syncthreads();
  SPH(0, 0)
  // OSF compacted publish items (SDRT_SA_PCOMP): per element slot the first item of its
  // left-face points (sPref) and each shape's left faces (sLeftF), for the publish phase
  __shared__ int sPref[E + 1];
  __shared__ signed char sLeftF[MAXSUB][4];
  if constexpr (OSF && SDRT_SA_PCOMP) {
    if (threadIdx.x < g.nsub) {
      int k = 0;
      for (int f = 0; f < S::nfaces; ++f)
        if (g.left[threadIdx.x][f]) sLeftF[threadIdx.x][k++] = (signed char)f;
    }
    if (threadIdx.x == 32) {
      int acc = 0;
      for (int el = 0; el < E; ++el) {
        sPref[el] = acc;
        if (e0 + el < g.K) {
          const int s = sNb[D + 1][el];
          for (int f = 0; f < S::nfaces; ++f) acc += g.left[s][f] ? S::nfp : 0;
        }
      }
      sPref[E] = acc;
    }
  }
  NbGather<D, P, NV, E, SDRT_SA_NT> gath;
  gath.load(g, ph, b.Tu, sNb, e0);
  mbar_wait(&bar, 0);
  // U_ext = M0 U, U_u = M12 U
  dmm2<NV, S::kt_sol, NV, S::kt_sol, E, false, false, NV * E, RS>(O.M0, sX, 1 << 30, sX, sUe, O.M12, sX, 1 << 30,
                                                                   sX, sUu);
  __syncthreads();
  SPH(0, 1)
  gath.template common_values<RS>(g, ph, sUe, sNb, sX, e0);  // C into X (U is dead)
  __syncthreads();
  SPH(0, 2)
  dmm1<NV, S::kt_G, E, false, RS, RS>(O.G, sX, S::next, sUu, sQ);  // rows (d, s) -> [d][s][v]
  __syncthreads();
  SPH(0, 3)
  metric_grad<D, P, NV, E, RS>(g, sNb, sQ);
  __syncthreads();
  SPH(0, 4)
  // gradient at the external points (M0 on each of the D NV gradient rows) into X, one
  // chunk of QCH points at a time, and g published at the chunk's points of the
  // LDG-weighted side
  const bool pub_left = (0.5 + ph.beta) != 0.0, pub_right = (0.5 - ph.beta) != 0.0;
  const int Kp = (int)g.Kt;  // trace row stride
#pragma unroll 1
  for (int r0 = 0; r0 < S::next; r0 += Ly::QCH) {
    const int nr = S::next - r0 < Ly::QCH ? S::next - r0 : Ly::QCH;
    SOpF Mc = O.M0;
    Mc.rows = nr;
    Mc.mt = (nr + 7) / 8;
    Mc.frag = O.M0.frag + (int64_t)(r0 / 8) * O.M0.kt * 32;
    if (Mc.kmask) Mc.kmask = O.M0.kmask + r0 / 8;
    if (r0 > 0) __syncthreads();  // the previous chunk's publish has read X
    // OSF: u_R of this thread's left face points (the right neighbour's published trace)
    // is pulled into L1 before the Q_ext product (no registers held across it)
    constexpr int CP = OSF ? (Ly::QCH * E + SDRT_SA_NT - 1) / SDRT_SA_NT : 1;
    auto uR_at = [&](int item) -> const double* {  // item over the chunk's (point, element)
      const int el = item % E, rho = r0 + item / E;
      if (item >= nr * E || e0 + el >= g.K) return nullptr;
      const int s = sNb[D + 1][el], f = rho / S::nfp;
      if (!g.left[s][f]) return nullptr;
      const int m = sNb[f][el];
      const int rho2 = g.nface[s][f] * S::nfp + g.perm[s][f][rho % S::nfp];
      return b.Tu + ((int64_t)rho2 * Kp + m) * NV;
    };
    if constexpr (OSF) {
#pragma unroll
      for (int k = 0; k < CP; ++k) {
        const double* a = uR_at(threadIdx.x + k * SDRT_SA_NT);
        if (a) {
          asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
          asm volatile("prefetch.global.L1 [%0];" ::"l"(a + NV - 1));
        }
      }
    }
    dmm_blocks<NV, S::kt_sol, E, D, RS>(Mc, sQ, S::nsol * RS, sX);  // Q_ext [chunk][d][v]
    __syncthreads();
  SPH(0, 5)
    auto publish = [&](int item, const double* uR) {
      const int el = item % E, rl = item / E, rho = r0 + rl;
      const int64_t e = e0 + el;
      if (e >= g.K) return;
      const int s = sNb[D + 1][el], f = rho / S::nfp;
      const bool left = g.left[s][f];
      if ((left && !pub_left) || (!left && !pub_right)) return;
      double u[NV], q[D * NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) u[v] = sUe[(rho * NV + v) * E + el];
#pragma unroll
      for (int k = 0; k < D * NV; ++k) q[k] = sX[(rl * D * NV + k) * E + el];
      const ExtMetric mt = b.xm[s * S::next + rho];
      const double nl[3] = {mt.n0, mt.n1, mt.n2};
      double gv[NV];
      Ph::visc_dir(ph, u, q, nl, gv);
      if constexpr (OSF) {  // left side: the whole common flux along n_L
        double F[NV];
        Ph::conv_common(ph, u, uR, nl, F);
        const double wl = 0.5 + ph.beta;  // = 1
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          F[v] = Ph::ldg_rn(F[v], __dmul_rn(wl, gv[v]), ph.eta, u[v], uR[v]);
          b.Tg[((int64_t)rho * Kp + e) * NV + v] = F[v];
          if (b.Fexp) b.Fexp[((int64_t)rho * NV + v) * g.Kp + e] = F[v];  // O28 export (residual only)
        }
      } else {
#pragma unroll
        for (int v = 0; v < NV; ++v) b.Tg[((int64_t)rho * Kp + e) * NV + v] = gv[v];
      }
    };
    if constexpr (OSF && SDRT_SA_PCOMP) {
      // compacted: item i -> the i-th left-face point of the tile (element slot by the
      // prefix sPref, face by the shape's left-face list): every lane carries a point
      static_assert(Ly::QCH >= S::next, "compacted publish needs one chunk");
      for (int i = threadIdx.x; i < sPref[E]; i += SDRT_SA_NT) {
        int el = 0;
#pragma unroll
        for (int j = 1; j < E; ++j) el += (i >= sPref[j]) ? 1 : 0;
        const int loc = i - sPref[el];
        const int f = sLeftF[sNb[D + 1][el]][loc / S::nfp];
        const int item = (f * S::nfp + loc % S::nfp) * E + el;
        const double* a = uR_at(item);
        double uR[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) uR[v] = a[v];
        publish(item, uR);
      }
    } else if constexpr (OSF) {
#pragma unroll
      for (int k = 0; k < CP; ++k) {
        const int item = threadIdx.x + k * SDRT_SA_NT;
        const double* a = uR_at(item);
        if (a) {
          double uR[NV];
#pragma unroll
          for (int v = 0; v < NV; ++v) uR[v] = a[v];
          publish(item, uR);
        }
      }
    } else {
      for (int item = threadIdx.x; item < nr * E; item += blockDim.x) publish(item, nullptr);
    }
  }
  __syncthreads();
  SPH(0, 6)
  dmm_blocks<NV, S::kt_sol, E, D, RS>(O.M12, sQ, S::nsol * RS, sUe);  // Q_u = M18 Q [nu][d][v] into UE
  __syncthreads();
  SPH(0, 7)
  internal_fluxes<D, P, EQ, E, RS, RS>(g, ph, sNb, sUu, sUe, sX, e0);  // F~ [D][nu][NV] into X
  __syncthreads();
  SPH(0, 8)
  dmm1_global<NV, S::kt_F, E, false, RS>(O.M13F, sX, b.Rint, g.Kp, e0, g.K);  // R_int -> HBM
  SPH(0, 9)
  SPH(0, 10)
}

// Kernel A for FR-SDRT (NEXT row N1): no internal flux points.
//   U_ext = M0 U;  C in place;  Q~ = [M16 | Dsol - M16 M0][C; U]  (gradient with the SDRT
//   correction, remark l.429-434);  Q = J^-T Q~;  Q_ext = M0 Q;  published g;  fluxes at the
//   solution points F[s][d] = detJ (J^-1 (f^c - f^v))_d (in place of Q);
//   R_int = [Dsol - M14 (n^ . M0)] F  (Eq. divergence_fr l.400-405 without the common flux).
// Regions (doubles per element): U [nsol NV] | W [next D NV] (U_ext -> C -> Q_ext) |
// Q [nsol D NV] (Q -> F).
template <int D, int P, int EQ, int E>
__global__ void __launch_bounds__(256, SDRT_SA_MINB) ks_grad_fr(GeomDev g, SimplexOps O, PhysDev ph, SimplexBufs b,
                                                               const __grid_constant__ STileMaps tm) {
  pdl_wait();
  using Ph = Phys<EQ, D>;
  using S = SDims<D, P>;
  constexpr int NV = Ph::NV;
  extern __shared__ __align__(128) double smem[];
  double* sU = smem;
  double* sW = sU + S::nsol * NV * E;
  double* sQ = sW + S::next * D * NV * E;
  __shared__ int sNb[D + 2][E];
  __shared__ __align__(8) uint64_t bar;
  const int64_t e0 = (int64_t)(g.tiles ? g.tiles[blockIdx.x] : (int)blockIdx.x) * E;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
    mbar_expect_tx(&bar, S::nsol * NV * E * 8);
    tma_tile<S::nsol * NV, E>(sU, &tm.uin, e0, &bar);
  }
  fill_neighbours<D, E>(g, sNb, e0);
  __syncthreads();
  NbGather<D, P, NV, E, 256> gath;
  gath.load(g, ph, b.Tu, sNb, e0);
  mbar_wait(&bar, 0);
  dmm1<NV, S::kt_sol, E, false>(O.M0, sU, 1 << 30, sU, sW);  // U_ext
  __syncthreads();
  gath.common_values(g, ph, sW, sNb, sW, e0);  // C in place of U_ext (same entries per item)
  __syncthreads();
  dmm1<NV, S::kt_GF, E, false>(O.G, sW, S::next, sU, sQ);  // rows (d, s) -> [d][s][v]
  __syncthreads();
  metric_grad<D, P, NV, E>(g, sNb, sQ);
  __syncthreads();
  dmm_blocks<NV, S::kt_sol, E, D>(O.M0, sQ, S::nsol * NV * E, sW);  // Q_ext [next][d][v]
  __syncthreads();
  // publish g at the face points of the LDG-weighted side (u_ext recomputed from U)
  const bool pub_left = (0.5 + ph.beta) != 0.0, pub_right = (0.5 - ph.beta) != 0.0;
  const int Kp = (int)g.Kt;
  for (int item = threadIdx.x; item < S::next * E; item += blockDim.x) {
    const int el = item % E, rho = item / E;
    const int64_t e = e0 + el;
    if (e >= g.K) continue;
    const int s = sNb[D + 1][el], f = rho / S::nfp;
    const bool left = g.left[s][f];
    if ((left && !pub_left) || (!left && !pub_right)) continue;
    double u[NV], q[D * NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) u[v] = 0.0;
    for (int sp = 0; sp < S::nsol; ++sp) {
      const double mv = sop_at(O.M0, rho, sp);
#pragma unroll
      for (int v = 0; v < NV; ++v) u[v] = fma(mv, sU[(sp * NV + v) * E + el], u[v]);
    }
#pragma unroll
    for (int k = 0; k < D * NV; ++k) q[k] = sW[(rho * D * NV + k) * E + el];
    const ExtMetric mt = b.xm[s * S::next + rho];
    const double nl[3] = {mt.n0, mt.n1, mt.n2};
    double gv[NV];
    Ph::visc_dir(ph, u, q, nl, gv);
#pragma unroll
    for (int v = 0; v < NV; ++v) b.Tg[((int64_t)rho * Kp + e) * NV + v] = gv[v];
  }
  // fluxes at the solution points, F[s][d][v] in place of Q[s][d][v] (each item reads its
  // point's gradient before writing the same entries)
  for (int item = threadIdx.x; item < S::nsol * E; item += blockDim.x) {
    const int el = item % E, sp = item / E;
    const int s = sNb[D + 1][el];
    double uu[NV], qq[D * NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) uu[v] = sU[(sp * NV + v) * E + el];
#pragma unroll
#pragma unroll
    for (int d = 0; d < D; ++d)
#pragma unroll
      for (int v = 0; v < NV; ++v) qq[d * NV + v] = sQ[((d * S::nsol + sp) * NV + v) * E + el];
    double fo[D][NV];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      double w[D], fv[NV];
#pragma unroll
      for (int j = 0; j < D; ++j) w[j] = g.detJ[s] * g.Jinv[s][d * 3 + j];
      Ph::conv_dir(ph, uu, w, fo[d]);
      Ph::visc_dir(ph, uu, qq, w, fv);
#pragma unroll
      for (int v = 0; v < NV; ++v) fo[d][v] = e0 + el < g.K ? fo[d][v] + fv[v] : 0.0;
    }
#pragma unroll
    for (int d = 0; d < D; ++d)
#pragma unroll
      for (int v = 0; v < NV; ++v) sQ[((d * S::nsol + sp) * NV + v) * E + el] = fo[d][v];
  }
  __syncthreads();
  dmm1_global<NV, S::kt_FF, E>(O.M13F, sQ, b.Rint, g.Kp, e0, g.K);  // R_int -> HBM (columns (d, s))
}

// Kernel B.  Regions (doubles per element): U [nsol NV] (stage input), R [nsol NV]
// (R_int, accumulated), UN, ACC [nsol NV] (RK registers), UE [next NV] (own traces,
// then D~, then the new traces); inviscid: UU [nu NV], F [D nu NV].
template <int D, int P, int NV, bool INT>
struct SLayoutB {
  using S = SDims<D, P>;
  static constexpr int U = S::nsol * NV;
  static constexpr int UE = S::next * NV;
  static constexpr int UU = INT ? S::nu * NV : 0;
  static constexpr int F = INT ? D * (S::nsol > S::nu ? S::nsol : S::nu) * NV : 0;  // SDRT or FR
  static constexpr int TOTAL = 4 * U + UE + UU + F;
};

template <int D, int P, int EQ, int E, bool FEXP = false>
__global__ void __launch_bounds__(SDRT_SB_NT, SDRT_SB_MINB) ks_stage(GeomDev g, SimplexOps O, PhysDev ph, SimplexBufs b, int stage,
                                                double dt, const __grid_constant__ STileMaps tm) {
  pdl_wait();
  SPH_INIT
  using Ph = Phys<EQ, D>;
  using S = SDims<D, P>;
  constexpr bool INT = !Ph::VISC;  // internal fluxes evaluated here (inviscid only)
  using Ly = SLayoutB<D, P, Ph::NV, INT>;
  constexpr int NV = Ph::NV;
  extern __shared__ __align__(128) double smem[];
  double* sU = smem;
  double* sR = sU + Ly::U * E;
  double* sUn = sR + Ly::U * E;
  double* sAcc = sUn + Ly::U * E;
  double* sUe = sAcc + Ly::U * E;
  double* sUu = sUe + Ly::UE * E;
  double* sF = sUu + Ly::UU * E;
  __shared__ int sNb[D + 2][E];
  __shared__ __align__(8) uint64_t bar[2];
  const int64_t e0 = (int64_t)(g.tiles ? g.tiles[blockIdx.x] : (int)blockIdx.x) * E;
  constexpr unsigned TB = S::nsol * NV * E * 8;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
    mbar_expect_tx(&bar[0], TB);
    tma_tile<S::nsol * NV, E>(sU, &tm.uin, e0, &bar[0]);
    const unsigned later = (INT ? 0 : TB) + (stage_reads_un(stage) ? TB : 0) + (stage_reads_acc(stage) ? TB : 0);
    mbar_expect_tx(&bar[1], later);
    if constexpr (!INT) tma_tile<S::nsol * NV, E>(sR, &tm.rint, e0, &bar[1]);
    if (stage_reads_un(stage)) tma_tile<S::nsol * NV, E>(sUn, &tm.un, e0, &bar[1]);
    if (stage_reads_acc(stage)) tma_tile<S::nsol * NV, E>(sAcc, &tm.acc, e0, &bar[1]);
  }
  fill_neighbours<D, E>(g, sNb, e0);
  __syncthreads();
  SPH(1, 0)
#if SDRT_SB_PF
  FluxGather<D, P, NV, E, SDRT_SB_NT, Ph::VISC> fg;
  fg.load(g, ph, b.Tu, b.Tg, sNb, e0);
#endif
  mbar_wait(&bar[0], 0);
  // own traces (and, inviscid, U_u)
  const SOpF none{0, 0, 0, 0, nullptr, nullptr};
  dmm2<NV, S::kt_sol, NV, S::kt_sol, E, false, false>(O.M0, sU, 1 << 30, sU, sUe, (INT && !O.fr) ? O.M12 : none, sU,
                                                        1 << 30, sU, sUu);
  __syncthreads();
  SPH(1, 1)
  // common fluxes D~ = +/- s F at external points, in place over the own traces
  const double wl = 0.5 + ph.beta, wr = 0.5 - ph.beta;
  const int Kp = (int)g.Kt;  // trace row stride
  auto face_flux = [&](int item, const double* unp, const double* gsp) {
    const int el = item % E, rho = item / E;
    const int64_t e = e0 + el;
    if (e >= g.K) {
#pragma unroll
      for (int v = 0; v < NV; ++v) sUe[(rho * NV + v) * E + el] = 0.0;
      return;
    }
    const int s = sNb[D + 1][el], f = rho / S::nfp, q = rho % S::nfp;
    const int m = sNb[f][el];
    const bool left = g.left[s][f];
    double uo[NV], un[NV], gsum[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      uo[v] = sUe[(rho * NV + v) * E + el];
      gsum[v] = 0.0;
    }
    if (unp) {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        un[v] = unp[v];
        if constexpr (Ph::VISC) gsum[v] = gsp[v];
      }
    } else {
      const int rho2 = g.nface[s][f] * S::nfp + g.perm[s][f][q];
#pragma unroll
      for (int v = 0; v < NV; ++v) un[v] = b.Tu[((int64_t)rho2 * Kp + m) * NV + v];
      if constexpr (Ph::VISC) {
        // g_L / g_R published by the left / right element at its own face point
        const int rL = left ? rho : rho2, rR = left ? rho2 : rho;
        const int eL = left ? (int)e : m, eR = left ? m : (int)e;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          double a = 0.0;
          if (wl != 0.0) a = __dmul_rn(wl, b.Tg[((int64_t)rL * Kp + eL) * NV + v]);
          if (wr != 0.0) a = __fma_rn(wr, b.Tg[((int64_t)rR * Kp + eR) * NV + v], a);
          gsum[v] = a;
        }
      }
    }
    const ExtMetric mt = b.xm[s * S::next + rho];
    const double nl[3] = {mt.n0, mt.n1, mt.n2};
    double uL[NV], uR[NV];  // by value: a runtime pointer select would put uo/un in local memory
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      uL[v] = left ? uo[v] : un[v];
      uR[v] = left ? un[v] : uo[v];
    }
    double F[NV];
    Ph::conv_common(ph, uL, uR, nl, F);
    const double sc = left ? mt.s : -mt.s;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double Fv = F[v];
      if constexpr (Ph::VISC) Fv = Ph::ldg_rn(Fv, gsum[v], ph.eta, uL[v], uR[v]);
      sUe[(rho * NV + v) * E + el] = sc * Fv;
      if (FEXP) b.Fexp[((int64_t)rho * NV + v) * g.Kp + e] = Fv;  // O28 export (residual only)
    }
  };
#if SDRT_SB_PF
#pragma unroll
  for (int k = 0; k < fg.CI; ++k) {
    const int item = threadIdx.x + k * SDRT_SB_NT;
    double gk[NV];
    {
      const double wl = 0.5 + ph.beta, wr = 0.5 - ph.beta;
      const double w1 = (wl == 0.0) != (wr == 0.0) ? (wl != 0.0 ? wl : wr) : 1.0;
#pragma unroll
      for (int v = 0; v < NV; ++v) gk[v] = Ph::VISC ? __dmul_rn(w1, fg.gs[Ph::VISC ? k : 0][v]) : 0.0;
    }
    if (item < S::next * E) face_flux(item, fg.un[k], gk);
  }
#else
  for (int item = threadIdx.x; item < S::next * E; item += blockDim.x) face_flux(item, nullptr, nullptr);
#endif
  if constexpr (INT) {
    if (O.fr) {  // FR-SDRT: fluxes at the solution points, F[s][d][v]
      for (int item = threadIdx.x; item < S::nsol * E; item += blockDim.x) {
        const int el = item % E, sp = item / E;
        const int s = sNb[D + 1][el];
        double uu[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) uu[v] = sU[(sp * NV + v) * E + el];
#pragma unroll
        for (int d = 0; d < D; ++d) {
          double w[D], fo[NV];
#pragma unroll
          for (int j = 0; j < D; ++j) w[j] = g.detJ[s] * g.Jinv[s][d * 3 + j];
          Ph::conv_dir(ph, uu, w, fo);
#pragma unroll
          for (int v = 0; v < NV; ++v) sF[((d * S::nsol + sp) * NV + v) * E + el] = e0 + el < g.K ? fo[v] : 0.0;
        }
      }
    } else {
      internal_fluxes<D, P, EQ, E>(g, ph, sNb, sUu, nullptr, sF, e0);
    }
  }
  mbar_wait(&bar[1], 0);  // R_int and the RK registers have landed
  __syncthreads();
  SPH(1, 2)
#if SDRT_SB_EPI && SDRT_SB_ONEPRODUCT
  // R~ = [M14 | M13F][D~; F~] (inviscid) or R_int + M14 D~, -R~/detJ and the RK update
  // as the product's epilogue (l.2919-2925, l.347-350)
  auto rk_epi = [&](int r, int n, double y0, double y1) {
    const int v = n / E, el = n % E;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int idx = (r * NV + v) * E + el + h;
      const int64_t e = e0 + el + h;
      if (e >= g.K) {
        sU[idx] = 0.0;
        continue;
      }
      const double kk = -(h ? y1 : y0) / g.detJ[sNb[D + 1][el + h]];
      sU[idx] = rk_value(b, stage, dt, kk, (int64_t)(r * NV + v) * g.Kp + e, sU, sAcc, sUn, idx);
    }
  };
  if constexpr (INT) {
    if (O.fr) dmm1_epi<NV, S::kt_EFF, E, false>(O.M14F, sUe, S::next, sF, nullptr, rk_epi);
    else dmm1_epi<NV, S::kt_EF, E, false>(O.M14F, sUe, S::next, sF, nullptr, rk_epi);
  } else {
    dmm1_epi<NV, S::kt_ext, E, true>(O.M14, sUe, 1 << 30, sUe, sR, rk_epi);
  }
  SPH(1, 4)
#else
  // R~ = R_int + M14 D~ [+ M13 M19 P2 F~]
  if constexpr (INT) {
#if SDRT_SB_ONEPRODUCT
    // one product [M14 | M13F] on [D~; F~] (no intermediate barrier or accumulate pass)
    if (O.fr) dmm1<NV, S::kt_EFF, E, false>(O.M14F, sUe, S::next, sF, sR);
    else dmm1<NV, S::kt_EF, E, false>(O.M14F, sUe, S::next, sF, sR);
  SPH(1, 3)
#else
    dmm1<NV, S::kt_ext, E, false>(O.M14, sUe, 1 << 30, sUe, sR);
    __syncthreads();
  SPH(1, 3)
    if (O.fr) dmm1<NV, S::kt_FF, E, true>(O.M13F, sF, 1 << 30, sF, sR);
    else dmm1<NV, S::kt_F, E, true>(O.M13F, sF, 1 << 30, sF, sR);
#endif
  } else {
    dmm1<NV, S::kt_ext, E, true>(O.M14, sUe, 1 << 30, sUe, sR);
  }
  __syncthreads();
  SPH(1, 4)
  // -R~/detJ and the RK4 update (registers from shared memory), new state into sU
  for (int idx = threadIdx.x; idx < S::nsol * NV * E; idx += blockDim.x) {
    const int el = idx % E, row = idx / E;
    const int64_t e = e0 + el;
    if (e >= g.K) {
      sU[idx] = 0.0;
      continue;
    }
    const int64_t gi = (int64_t)row * g.Kp + e;
    const int s = sNb[D + 1][el];
    const double kk = -sR[idx] / g.detJ[s];
    double nu;
    switch (stage) {
      case -1: b.out[gi] = kk; nu = 0.0; break;
      case 0: {
        const double u0 = sU[idx];
        b.ACC[gi] = fma(dt / 6.0, kk, u0);
        nu = fma(0.5 * dt, kk, u0);
        b.Us[gi] = nu;
      } break;
      case 1:
        b.ACC[gi] = fma(dt / 3.0, kk, sAcc[idx]);
        nu = fma(0.5 * dt, kk, sUn[idx]);
        b.Us[gi] = nu;
        break;
      case 2:
        b.ACC[gi] = fma(dt / 3.0, kk, sAcc[idx]);
        nu = fma(dt, kk, sUn[idx]);
        b.Us[gi] = nu;
        break;
      case 3:
        nu = fma(dt / 6.0, kk, sAcc[idx]);
        b.U[gi] = nu;
        break;
      default: {  // RK54 stage s (2N-storage, in place)
        const int s5 = stage - RK54_STAGE0;
        const double du = s5 == 0 ? dt * kk : fma(rk54_a(s5), sAcc[idx], dt * kk);
        b.ACC[gi] = du;
        nu = fma(rk54_b(s5), du, sU[idx]);
        b.U[gi] = nu;
      } break;
    }
    sU[idx] = nu;
  }
#endif
  if (stage < 0) return;
  __syncthreads();
  SPH(1, 5)
  dmm1_global<NV, S::kt_sol, E, true>(O.M0, sU, b.Tu_next, g.Kt, e0, g.K);  // traces of the new state
  SPH(1, 6)
  SPH(1, 7)
}

// Kernel B with one-sided flux publication (OSF, NS with beta = +1/2): the common flux
// of every face point was evaluated once by the face's left element (ks_grad<OSF>) and
// published in T_g; here D~ = +s F (own left faces) / -s F (right faces, gathered from
// the left neighbour), R~ = R_int + M14 D~ (l.2919-2925), -R~/detJ, RK update, and the
// traces of the new state at the faces where this element is RIGHT (the only ones
// kernel A reads with beta = 1/2).  The stage input is read only where the RK formula
// needs it (RK4 stage 0, RK54).
template <int D, int P, int EQ, int E, bool FEXP = false>
__global__ void __launch_bounds__(SDRT_SB_NT, SDRT_SB_MINB_OSF) ks_stage_osf(GeomDev g, SimplexOps O, PhysDev ph,
                                                                    SimplexBufs b, int stage, double dt,
                                                                    const __grid_constant__ STileMaps tm) {
  pdl_wait();
  using Ph = Phys<EQ, D>;
  using S = SDims<D, P>;
  using Ly = SLayoutB<D, P, Ph::NV, false>;
  constexpr int NV = Ph::NV, NT = SDRT_SB_NT;
  extern __shared__ __align__(128) double smem[];
  double* sU = smem;
  double* sR = sU + Ly::U * E;
  double* sUn = sR + Ly::U * E;
  double* sAcc = sUn + Ly::U * E;
  double* sD = sAcc + Ly::U * E;  // D~ [next][NV][E]
  __shared__ int sNb[D + 2][E];
  __shared__ __align__(8) uint64_t bar;
  // SDRT_SB_REV: reverse tile order (kernel A's last-written tiles first, see tensor.cu SDRT_TB_REV)
  const int bx = SDRT_SB_REV ? (int)(gridDim.x - 1 - blockIdx.x) : (int)blockIdx.x;
  const int64_t e0 = (int64_t)(g.tiles ? g.tiles[bx] : bx) * E;
  const bool need_in = stage == 0 || stage >= RK54_STAGE0;
  constexpr unsigned TB = S::nsol * NV * E * 8;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
    mbar_expect_tx(&bar, TB * (1 + (need_in ? 1 : 0) + (stage_reads_un(stage) ? 1 : 0) + (stage_reads_acc(stage) ? 1 : 0)));
    tma_tile<S::nsol * NV, E>(sR, &tm.rint, e0, &bar);
    if (need_in) tma_tile<S::nsol * NV, E>(sU, &tm.uin, e0, &bar);
    if (stage_reads_un(stage)) tma_tile<S::nsol * NV, E>(sUn, &tm.un, e0, &bar);
    if (stage_reads_acc(stage)) tma_tile<S::nsol * NV, E>(sAcc, &tm.acc, e0, &bar);
  }
  fill_neighbours<D, E>(g, sNb, e0);
  __syncthreads();
  // the published F of each of this thread's face points (own for left faces, the left
  // neighbour's otherwise), requested before the tile wait
  constexpr int ITEMS = S::next * E, CI = (ITEMS + NT - 1) / NT;
  const int Kp = (int)g.Kt;
  double Fv[CI][NV];
#pragma unroll
  for (int k = 0; k < CI; ++k) {
    const int item = threadIdx.x + k * NT;
    const int el = item % E, rho = item / E;
#pragma unroll
    for (int v = 0; v < NV; ++v) Fv[k][v] = 0.0;
    if (item >= ITEMS || e0 + el >= g.K) continue;
    const int s = sNb[D + 1][el], f = rho / S::nfp;
    int64_t at;
    if (g.left[s][f]) {
      at = (int64_t)rho * Kp + e0 + el;
    } else {
      const int rho2 = g.nface[s][f] * S::nfp + g.perm[s][f][rho % S::nfp];
      at = (int64_t)rho2 * Kp + sNb[f][el];
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) Fv[k][v] = b.Tg[at * NV + v];
  }
#pragma unroll
  for (int k = 0; k < CI; ++k) {
    const int item = threadIdx.x + k * NT;
    const int el = item % E, rho = item / E;
    if (item >= ITEMS) continue;
    const int64_t e = e0 + el;
    double sc = 0.0;
    if (e < g.K) {
      const int s = sNb[D + 1][el], f = rho / S::nfp;
      const ExtMetric mt = b.xm[s * S::next + rho];
      sc = g.left[s][f] ? mt.s : -mt.s;
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      sD[(rho * NV + v) * E + el] = sc * Fv[k][v];
      if (FEXP && e < g.K) b.Fexp[((int64_t)rho * NV + v) * g.Kp + e] = Fv[k][v];  // O28 export (residual only)
    }
  }
  mbar_wait(&bar, 0);
  __syncthreads();
#if SDRT_SB_EPI
  // R~ = R_int + M14 D~ with the RK update as the product's epilogue (l.2919-2925, l.347-350)
  dmm1_epi<NV, S::kt_ext, E, true>(O.M14, sD, 1 << 30, sD, sR, [&](int r, int n, double y0, double y1) {
    const int v = n / E, el = n % E;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int idx = (r * NV + v) * E + el + h;
      const int64_t e = e0 + el + h;
      if (e >= g.K) {
        sU[idx] = 0.0;
        continue;
      }
      const double kk = -(h ? y1 : y0) / g.detJ[sNb[D + 1][el + h]];
      sU[idx] = rk_value(b, stage, dt, kk, (int64_t)(r * NV + v) * g.Kp + e, sU, sAcc, sUn, idx);
    }
  });
#else
  dmm1<NV, S::kt_ext, E, true>(O.M14, sD, 1 << 30, sD, sR);  // R~ = R_int + M14 D~
  __syncthreads();
  for (int idx = threadIdx.x; idx < S::nsol * NV * E; idx += NT) {
    const int el = idx % E, row = idx / E;
    const int64_t e = e0 + el;
    if (e >= g.K) {
      sU[idx] = 0.0;
      continue;
    }
    const int64_t gi = (int64_t)row * g.Kp + e;
    const int s = sNb[D + 1][el];
    const double kk = -sR[idx] / g.detJ[s];
    double nu;
    switch (stage) {
      case -1: b.out[gi] = kk; nu = 0.0; break;
      case 0: {
        const double u0 = sU[idx];
        b.ACC[gi] = fma(dt / 6.0, kk, u0);
        nu = fma(0.5 * dt, kk, u0);
        b.Us[gi] = nu;
      } break;
      case 1:
        b.ACC[gi] = fma(dt / 3.0, kk, sAcc[idx]);
        nu = fma(0.5 * dt, kk, sUn[idx]);
        b.Us[gi] = nu;
        break;
      case 2:
        b.ACC[gi] = fma(dt / 3.0, kk, sAcc[idx]);
        nu = fma(dt, kk, sUn[idx]);
        b.Us[gi] = nu;
        break;
      case 3:
        nu = fma(dt / 6.0, kk, sAcc[idx]);
        b.U[gi] = nu;
        break;
      default: {  // RK54 stage s (2N-storage, in place)
        const int s5 = stage - RK54_STAGE0;
        const double du = s5 == 0 ? dt * kk : fma(rk54_a(s5), sAcc[idx], dt * kk);
        b.ACC[gi] = du;
        nu = fma(rk54_b(s5), du, sU[idx]);
        b.U[gi] = nu;
      } break;
    }
    sU[idx] = nu;
  }
#endif
  if (stage < 0) return;
  __syncthreads();
  // traces of the new state M0 U at the right-side faces only (point-major)
  using DM = Dmm<NV, E, S::kt_sol>;
  const int warp = threadIdx.x >> 5, nw = NT >> 5, lane = threadIdx.x & 31;
  for (int j = warp; j < DM::jobs(O.M0); j += nw) {
    const int m = j / DM::NG, ng = j % DM::NG;
    const int n0 = ng * DM::NGR * 8 + (lane >> 2);
    const double* af = O.M0.frag + (int64_t)m * S::kt_sol * 32 + lane;
    const unsigned km = O.M0.kmask ? __ldg(O.M0.kmask + m) : 0xffffffffu;
    double a[S::kt_sol];
#pragma unroll
    for (int k = 0; k < S::kt_sol; ++k) a[k] = (km >> k & 1u) ? __ldg(af + k * 32) : 0.0;
    double c[DM::NGR][2];
#pragma unroll
    for (int q = 0; q < DM::NGR; ++q) c[q][0] = c[q][1] = 0.0;
#pragma unroll
    for (int k = 0; k < S::kt_sol; ++k) {
      if (!(km >> k & 1u)) continue;
      const int col = 4 * k + (lane & 3);
      const bool ok = col < O.M0.cols;
#pragma unroll
      for (int q = 0; q < DM::NGR; ++q) dmma(c[q][0], c[q][1], a[k], ok ? sU[col * DM::N + n0 + 8 * q] : 0.0);
    }
    const int r = 8 * m + (lane >> 2);
    if (r < O.M0.rows) {
      const int f = r / S::nfp;
#pragma unroll
      for (int q = 0; q < DM::NGR; ++q) {
        const int n = ng * DM::NGR * 8 + 8 * q + 2 * (lane & 3);  // column (w, el), el even
        const int w = n / E, el = n % E;
        double* gp = b.Tu_next + ((int64_t)r * g.Kt + e0 + el) * NV + w;
        if (e0 + el < g.K && !g.left[sNb[D + 1][el]][f]) gp[0] = c[q][0];
        if (e0 + el + 1 < g.K && !g.left[sNb[D + 1][el + 1]][f]) gp[NV] = c[q][1];
      }
    }
  }
}

// TGV diagnostics (NEXT row N4): per tile the solution-point
// quadrature sums (w_r detJ_s) of E* = rho v.v, S^d : S^d and p div v, grad v from the
// LDG gradient (the prologue of kernel A) by the chain rule (reading O20).
template <int D, int P, int EQ, int E>
__global__ void __launch_bounds__(256) ks_diag(GeomDev g, SimplexOps O, PhysDev ph, SimplexBufs b, const double* w,
                                               const double* Bq, int nq, double* part,
                                               const __grid_constant__ STileMaps tm) {
  using Ph = Phys<EQ, D>;
  using S = SDims<D, P>;
  constexpr int NV = Ph::NV, NT = 256;
  extern __shared__ __align__(128) double smem[];
  double* sU = smem;
  double* sUe = sU + S::nsol * NV * E;
  double* sUu = sUe + S::next * NV * E;
  double* sC = sUu + S::nu * NV * E;
  double* sQ = sC + S::next * NV * E;
  __shared__ double red[3 * NT];
  __shared__ int sNb[D + 2][E];
  __shared__ __align__(8) uint64_t bar;
  const int64_t e0 = (int64_t)blockIdx.x * E;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
    mbar_expect_tx(&bar, S::nsol * NV * E * 8);
    tma_tile<S::nsol * NV, E>(sU, &tm.uin, e0, &bar);
  }
  fill_neighbours<D, E>(g, sNb, e0);
  __syncthreads();
  NbGather<D, P, NV, E, NT> gath;
  gath.load(g, ph, b.Tu, sNb, e0);
  mbar_wait(&bar, 0);
  dmm2<NV, S::kt_sol, NV, S::kt_sol, E, false, false>(O.M0, sU, 1 << 30, sU, sUe, O.M12, sU, 1 << 30, sU, sUu);
  __syncthreads();
  gath.common_values(g, ph, sUe, sNb, sC, e0);
  __syncthreads();
  dmm1<NV, S::kt_G, E, false>(O.G, sC, S::next, sUu, sQ);  // rows (d, s) -> [d][s][v]
  __syncthreads();
  metric_grad<D, P, NV, E>(g, sNb, sQ);
  __syncthreads();
  double acc[3] = {0.0, 0.0, 0.0};
  if constexpr (NV == D + 2)
    tgv_tile<D, NV, E, S::nsol>(ph, sU, sQ, w, Bq, nq, e0, g.K, [&](int el) { return g.detJ[sNb[D + 1][el]]; }, acc);
#pragma unroll
  for (int k = 0; k < 3; ++k) red[k * NT + threadIdx.x] = acc[k];
  __syncthreads();
  for (int h = NT / 2; h > 0; h >>= 1) {
    if (threadIdx.x < h)
#pragma unroll
      for (int k = 0; k < 3; ++k) red[k * NT + threadIdx.x] += red[k * NT + threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < 3; ++k) part[3 * blockIdx.x + k] = red[k * NT];
}

// ------------------------------------------------------------------ launchers
template <int D, int P, int EQ>
struct SCfg {
  static constexpr int NV = Phys<EQ, D>::NV;
  static constexpr bool VISC = Phys<EQ, D>::VISC;
  // tile width: MMA rows hold NV E (a multiple of 8) columns; 2-D systems (N_V = 4) may
  // take 4-element tiles (SDRT_S_E2D): twice the CTAs for the small latency-bound meshes
  static constexpr int E = (D == 2 && (NV * SDRT_S_E2D) % 8 == 0) ? SDRT_S_E2D : 8;
  static constexpr int THREADS = 256;
  static constexpr size_t SMEM_A = (size_t)SLayoutA<D, P, NV, E>::TOTAL * sizeof(double);
  static constexpr size_t SMEM_B = (size_t)SLayoutB<D, P, NV, !VISC>::TOTAL * E * sizeof(double);
  static constexpr size_t SMEM_T = (size_t)(SDims<D, P>::nsol + SDims<D, P>::next) * NV * E * sizeof(double);
};

// carve: request the whole 228 KB shared-memory carve-out (kernels whose operator
// fragments fit the remaining L1; the default carve-out stops short of 5 x 38 KB CTAs)
static void sset_smem(const void* k, size_t bytes, bool carve = false) {
  if (bytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA smem attr: ") + cudaGetErrorString(e));
  }
  if (carve) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA carveout attr: ") + cudaGetErrorString(e));
  }
}

static STileMaps smaps(SimplexTma* t, const SimplexBufs& b, const double* uin, bool full) {
  STileMaps m;
  std::memset(&m, 0, sizeof(m));
  m.uin = cached_tile_map(t, uin);
  if (full) {
    if (b.U) m.un = cached_tile_map(t, b.U);
    if (b.ACC) m.acc = cached_tile_map(t, b.ACC);
    if (b.Rint) m.rint = cached_tile_map(t, b.Rint);
  }
  return m;
}

template <int D, int P, int EQ>
static void srun(const GeomDev& g, const SimplexOps& O, const PhysDev& ph, SimplexTma* tma, const SimplexBufs& b,
                 int stage, double dt, cudaStream_t st, int which, const double* U, double* T) {
  using C = SCfg<D, P, EQ>;
  const unsigned grid = g.tiles ? (unsigned)g.ntiles : (unsigned)((g.K + C::E - 1) / C::E);
  if (grid == 0) return;
  if (which == 0) {
    if constexpr (Phys<EQ, D>::VISC) {
      if (O.fr) {
        auto k = ks_grad_fr<D, P, EQ, C::E>;
        const size_t sm = (size_t)(SDims<D, P>::nsol * (1 + D) + SDims<D, P>::next * D) * C::NV * C::E * sizeof(double);
        sset_smem((const void*)k, sm);
        CUDA_LAUNCH_OK(launch_pdl(k, grid, 256, sm, st, g, O, ph, b, smaps(tma, b, b.Uin, false)));
      } else {
        auto k = ks_grad<D, P, EQ, C::E>;
        if constexpr (EQ == EQ_NS)
          if (g.osf) k = ks_grad<D, P, EQ, C::E, true>;
        sset_smem((const void*)k, C::SMEM_A);
        CUDA_LAUNCH_OK(launch_pdl(k, grid, SDRT_SA_NT, C::SMEM_A, st, g, O, ph, b, smaps(tma, b, b.Uin, false)));
      }
    }
  } else if (which == 1) {
    if constexpr (EQ == EQ_NS) {
      if (g.osf && !O.fr) {
        auto k = b.Fexp ? ks_stage_osf<D, P, EQ, C::E, true> : ks_stage_osf<D, P, EQ, C::E>;
        sset_smem((const void*)k, C::SMEM_B, SDRT_SB_CARVE != 0);
        CUDA_LAUNCH_OK(launch_pdl(k, grid, SDRT_SB_NT, C::SMEM_B, st, g, O, ph, b, stage, dt, smaps(tma, b, b.Uin, true)));
        return;
      }
    }
    auto k = b.Fexp ? ks_stage<D, P, EQ, C::E, true> : ks_stage<D, P, EQ, C::E>;
    sset_smem((const void*)k, C::SMEM_B);
    CUDA_LAUNCH_OK(launch_pdl(k, grid, SDRT_SB_NT, C::SMEM_B, st, g, O, ph, b, stage, dt, smaps(tma, b, b.Uin, true)));
  } else {
    auto k = ks_traces<D, P, EQ, C::E>;
    sset_smem((const void*)k, C::SMEM_T);
    CUDA_LAUNCH_OK(launch_pdl(k, grid, C::THREADS, C::SMEM_T, st, g, O, smaps(tma, b, U, false), T));
  }
}

template <int D, int P, int EQ>
static void stma(SimplexTma* t, int64_t Kp) {
  using C = SCfg<D, P, EQ>;
  t->rows = SDims<D, P>::nsol * C::NV;
  t->E = C::E;
  t->Kp = Kp;
  for (int i = 0; i < 8; ++i) t->ptr[i] = nullptr;
  t->next = 0;
}

typedef void (*SFn)(const GeomDev&, const SimplexOps&, const PhysDev&, SimplexTma*, const SimplexBufs&, int, double,
                    cudaStream_t, int, const double*, double*);
typedef void (*STmaFn)(SimplexTma*, int64_t);

template <int D, int P>
static SFn spick_eq(int eq, STmaFn* m) {
  switch (eq) {
    case EQ_LINADV: *m = stma<D, P, EQ_LINADV>; return srun<D, P, EQ_LINADV>;
    case EQ_LINADVDIFF: *m = stma<D, P, EQ_LINADVDIFF>; return srun<D, P, EQ_LINADVDIFF>;
    case EQ_EULER: *m = stma<D, P, EQ_EULER>; return srun<D, P, EQ_EULER>;
    case EQ_NS: *m = stma<D, P, EQ_NS>; return srun<D, P, EQ_NS>;
  }
  return nullptr;
}

static SFn spick(int D, int P, int eq, STmaFn* m) {
  *m = nullptr;
  if (D == 2) {
    switch (P) {
      case 1: return spick_eq<2, 1>(eq, m);
      case 2: return spick_eq<2, 2>(eq, m);
      case 3: return spick_eq<2, 3>(eq, m);
      case 4: return spick_eq<2, 4>(eq, m);
    }
  } else {
    switch (P) {
      case 1: return spick_eq<3, 1>(eq, m);
      case 2: return spick_eq<3, 2>(eq, m);
      case 3: return spick_eq<3, 3>(eq, m);
    }
  }
  return nullptr;
}

int simplex_tile_width(int D, int P, int eq) {
  (void)P;
  const int nv = (eq == EQ_LINADV || eq == EQ_LINADVDIFF) ? 1 : D + 2;
  return (D == 2 && (nv * SDRT_S_E2D) % 8 == 0) ? SDRT_S_E2D : 8;  // SCfg<...>::E
}

void simplex_launch_diag(int D, int P, const GeomDev& g, const SimplexOps& O, const PhysDev& ph, SimplexTma* tma,
                         const SimplexBufs& b, const double* w, const double* Bq, int nq, double* part,
                         cudaStream_t st) {
  if (D != 3 || P < 1 || P > 3) throw std::runtime_error("unsupported: TGV diagnostics need a 3-D NS context");
  auto launch = [&](auto kern, size_t per_el) {
    const size_t sm = per_el * 8 * sizeof(double);
    sset_smem((const void*)kern, sm);
    const unsigned grid = (unsigned)((g.K + 7) / 8);
    kern<<<grid, 256, sm, st>>>(g, O, ph, b, w, Bq, nq, part, smaps(tma, b, b.Uin, false));
  };
  // regions per element: U, U_ext, U_u, C, Q  (N_V = 5)
  auto per_el = [](int nsol, int next, int nu) { return (size_t)(4 * nsol + 2 * next + nu) * 5; };
  if (P == 1) launch(ks_diag<3, 1, EQ_NS, 8>, per_el(SDims<3, 1>::nsol, SDims<3, 1>::next, SDims<3, 1>::nu));
  else if (P == 2) launch(ks_diag<3, 2, EQ_NS, 8>, per_el(SDims<3, 2>::nsol, SDims<3, 2>::next, SDims<3, 2>::nu));
  else launch(ks_diag<3, 3, EQ_NS, 8>, per_el(SDims<3, 3>::nsol, SDims<3, 3>::next, SDims<3, 3>::nu));
}

bool simplex_supported(int D, int P, int eq) {
  STmaFn m;
  return spick(D, P, eq, &m) != nullptr;
}

void simplex_tma_init(SimplexTma* t, int D, int P, int eq, int64_t Kp) {
  STmaFn m;
  spick(D, P, eq, &m);
  m(t, Kp);
}

void simplex_launch_traces(int D, int P, int eq, const GeomDev& g, const SimplexOps& O, SimplexTma* tma,
                           const double* U, double* Tu, cudaStream_t st) {
  SimplexBufs b{};
  PhysDev ph{};
  STmaFn m;
  spick(D, P, eq, &m)(g, O, ph, tma, b, 0, 0.0, st, 2, U, Tu);
}

void simplex_launch_grad(int D, int P, int eq, const GeomDev& g, const SimplexOps& O, const PhysDev& ph,
                         SimplexTma* tma, const SimplexBufs& b, cudaStream_t st) {
  STmaFn m;
  spick(D, P, eq, &m)(g, O, ph, tma, b, 0, 0.0, st, 0, nullptr, nullptr);
}

void simplex_launch_flux(int D, int P, int eq, const GeomDev& g, const SimplexOps& O, const PhysDev& ph,
                         SimplexTma* tma, const SimplexBufs& b, int stage, double dt, cudaStream_t st) {
  STmaFn m;
  spick(D, P, eq, &m)(g, O, ph, tma, b, stage, dt, st, 1, nullptr, nullptr);
}

#ifdef SDRT_PHASE_PROF
void simplex_phase_cycles(unsigned long long* out, bool reset) {
  cudaMemcpyFromSymbol(out, g_sphase_cycles, sizeof(g_sphase_cycles));
  if (reset) {
    static unsigned long long z[2][16] = {};
    cudaMemcpyToSymbol(g_sphase_cycles, z, sizeof(z));
  }
}
#endif

}  // namespace sdrt

#ifdef SDRT_PHASE_PROF
extern "C" void sdrt_debug_sphase_cycles(unsigned long long* out, int reset) {
  sdrt::simplex_phase_cycles(out, reset != 0);
}
#endif
