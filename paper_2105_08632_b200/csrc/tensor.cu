// Fused SDRT stage for tensor-product elements (quad / hex) on sm_100a, fp64.
//
// The App. B operators of tensor elements factor into 1D line operators along the
// GL-aligned flux lines (App. A l.2618-2625; B7 structural sparsity
// l.2927-2932: one normal component per unique internal point), so a stage is
// evaluated line by line with the whole element tile resident in shared memory:
//
//   kernel A (viscous only): U, neighbour U traces -> common value C (l.282-291) ->
//     gradient Q~ = M16 C + M15 U_int along lines (l.295-298), Q = J^-T Q~ (l.299-302)
//     -> viscous normal flux g = n_L . f^v(u, q) at face points, published as a trace
//     (the common viscous flux (1/2+b) g_L + (1/2-b) g_R + eta (u_L - u_R), l.330-335,
//     needs only these N_V numbers per face point, not the D N_V gradient)
//   kernel B: U, traces -> [gradient again] -> per line: internal transformed flux
//     (l.305-311, one component per point), common flux at both ends (Rusanov l.324-328
//     + LDG), divergence R~ = M14 D~ + M13 F~ (l.2919-2925) accumulated per direction
//     -> dU/dt = -R~/detJ (l.347-350) -> RK4 register update -> traces of the new state.
//
// Tile: E consecutive elements per CTA, shared memory [point][var][E] (element
// fastest, matching the ABI layout so global loads/stores are row segments of E
// doubles).  Face values are exchanged only through traces [N_ext][N_V][K_pad]
// written by the previous stage (double-buffered), so each face point's common flux
// is evaluated by both neighbours from bit-identical inputs (explicit fma chains for
// the trace interpolation, published g read back by both sides) and D~_R = -D~_L
// bitwise (O28).
#include <cuda_runtime.h>

#include <cstring>
#include <stdexcept>
#include <type_traits>
#include <string>

#include "tensor.cuh"
#include "rk.cuh"
#include "tma.cuh"
#include "diag.cuh"

// kernel A internal fluxes on element pairs (16-byte shared-memory loads): 0 never,
// 1 always, 2 for scalar equations only (measured: c3 43.7 -> 41.6 us; NS spills)
#ifndef SDRT_TA_PAIR
#define SDRT_TA_PAIR 2
#endif
// kernel A internal fluxes and published g by DMMA line interpolation (NS, E = 8);
// parity-green but measured slower on c4 (253 -> 314 us: only 16 of 32 lanes carry
// physics after the mma, and the fragments cost registers), so off by default
#ifndef SDRT_TA_DMMA
#define SDRT_TA_DMMA 0
#endif
// kernel A gradient on element pairs (GradNb2), same modes (measured: c3 41.6 -> 40.2 us,
// c4 253 -> 256 us)
#ifndef SDRT_TA_GPAIR
#define SDRT_TA_GPAIR 2
#endif
// kernel A internal-flux items ordered (a, t, el) with a compile-time point index per
// warp-uniform branch (SDRT_TA_AUNI = 1) or (t, a, el) with a runtime index (0)
#ifndef SDRT_TA_AUNI
#define SDRT_TA_AUNI 0
#endif
// sum-factorised diagnostics: elements per pass for p <= 3 (38.4 KB of shared memory per
// element at p = 3; p = 4 takes one element per pass)
#ifndef SDRT_DIAG_G
#define SDRT_DIAG_G 1
#endif
// OSF kernel B: R_int and u_n read from global memory in the update (1) or staged by TMA (0).
// Measured on c4: 147 us (direct, three CTAs per SM) vs 97 us (TMA, two): the TMA tiles are
// requested at the CTA start and land while the flux gather runs; off
#ifndef SDRT_TB_DIRECT
#define SDRT_TB_DIRECT 0
#endif
// kernel A gradient through the composite per-axis operator Line1D::Gq (GradNb): 1 on, 0 the
// step-by-step form (own traces, common values, U_int, then Dfl)
#ifndef SDRT_TA_GQ
#define SDRT_TA_GQ 1
#endif
// kernel A internal fluxes and published g by register-blocked line items (visc_line):
// 0 off (per-point items), 1 on
// line items on the one-sided publication path (NS), instead of per-point visc_internal
// and publish_F items: 0 off; 1 one item per d-line for its internal points (visc_sline;
// measured on c4: kernel A 252 vs 242 us, phase imbalance against the publish items and
// spills); 2 (default) two half-line items per d-line, the second carrying the published
// end (visc_hline; c4 kernel A 242 -> 220 us, 31.8 -> 34.1 GDOF-stage/s)
#ifndef SDRT_TA_SLINE
#define SDRT_TA_SLINE 2
#endif
#ifndef SDRT_TA_LINE
#define SDRT_TA_LINE 1
#endif
// half-line items (hex p = 3, N_V odd, 8-element tiles): row-pair swizzle of the gradient
// tile sQ.  A warp's four x-lines (t = y + 4 z, y = 0..3) start 4 points = 20 rows of 64 B
// apart: all in the same half of the 128-byte bank window (2-way conflict on every load of
// direction 0).  Row r of point s is stored at r ^ ((s >> 2) & 1): adjacent y rows swap
// halves, conflict-free in all three directions, no extra shared memory.  Bitwise the
// unswizzled kernel (layout only).
#ifndef SDRT_TA_QSWZ
#define SDRT_TA_QSWZ 0
#endif
// half-line items: which warps take which half of the lines.  0: warps 0-3 the first
// halves, 4-7 the second; 1: the half is bit 1 of the warp index, so the two warps of a
// CTA that share a scheduler (w, w + 4) run the same code (instruction-cache reuse)
#ifndef SDRT_TA_HMAP
#define SDRT_TA_HMAP 0
#endif
// one-sided publication kernel A, divergence: the partial sums of R_int over the directions
// accumulated by a global read-modify-write of the owning thread (0) or by
// red.global.add.f64 onto the first direction's store (1, default: no load, no prefetch
// registers, 126 -> 121 registers; the directions are separated by CTA barriers and each
// address belongs to one CTA, so the sum order is fixed: deterministic; each direction's
// fma chain is rounded before it is added, fl(R + fl(chain)), instead of one chain through
// R, so not bitwise mode 0).  Measured on c4: kernel A 220 -> 203 us, 34.2 -> 36.15
// GDOF-stage/s.
#ifndef SDRT_TA_DRED
#define SDRT_TA_DRED 1
#endif
// half-line items: 1 = software-pipelined component loads (the next needed component's n
// shared-memory loads are issued before the current component's interpolation sums)
#ifndef SDRT_TA_HPIPE
#define SDRT_TA_HPIPE 0
#endif
// one-sided publication kernel A as a persistent kernel (kt_grad_p: MINB CTAs per SM, each
// walking tiles blockIdx.x, + gridDim.x, ...): the next tile's stage input (TMA), neighbour
// indices and neighbour traces are requested during the current tile's last divergence
// phase, when the state and gradient tiles are dead, instead of at the next CTA's start
// (the tile + neighbour-load latency is ~15 % of a one-tile CTA's life).  Same per-tile
// arithmetic (bitwise the one-tile kernel).
#ifndef SDRT_TA_PERSIST
#define SDRT_TA_PERSIST 0
#endif
// half-line items: warp-pair barriers.  Warps w and w + 4 hold the two halves of the same
// four d-lines x 8 elements in every direction; with the divergence items of those lines
// given to the same 64 threads, the flux -> divergence -> next flux hand-offs through the
// internal-flux buffer are pair-local, so the direction loop synchronises on named
// barriers of 64 threads (bar.sync 1 + pair) and the pairs drift apart (flux work of one
// overlaps the divergence stores of another).  One CTA-wide barrier stays after the last
// flux phase: a point's R_int entry is written by different pairs in different
// directions, and the RED order of directions 1 and 2 (and the store before them) must be
// fixed.  Same arithmetic per item and the same order per address (bitwise mode 0).
#ifndef SDRT_TA_PAIRB
#define SDRT_TA_PAIRB 0
#endif
// kernel B walks the tiles in reverse launch order (CTA i takes tile grid - 1 - i): kernel
// A runs first tile -> last, so kernel B starts on the tiles whose R_int and published
// fluxes kernel A wrote last (still in the 126 MB L2) and ends on the first tiles, which
// the next stage's kernel A reads first.  Tile order only: bitwise.  1 (default): the
// one-sided publication kernel B only (c4, working set >> L2: 36.1 -> 36.5 GDOF-stage/s);
// 2: the two-sided kernel B as well (measured slower on the L2-resident c3: 35.0 -> 34.5).
#ifndef SDRT_TB_REV
#define SDRT_TB_REV 1
#endif
// one-sided kernel B: TMA loads with an L2 evict-first policy for R_int (1: read once, dead
// afterwards) and also for the RK registers u_n and ACC (2: next read a whole stage later)
#ifndef SDRT_TB_EF
#define SDRT_TB_EF 0
#endif

namespace sdrt {

// swizzled sQ (SDRT_TA_QSWZ): offset (in doubles) added to the linear address of the i-th
// load (point lb + i ls) of component v along d-line t; v, i compile-time at the call sites
template <int d, int E>
struct QSwz {
  int f;
  __device__ __forceinline__ explicit QSwz(int t) {
    if constexpr (d == 0) f = (t & 1) * E;                      // s = y & 1, row parity (v + i) & 1
    else if constexpr (d == 1) f = (t & 1) ? -E : E;            // s = i & 1, row parity (x + v) & 1
    else f = ((t >> 2) & 1) ? ((t & 1) ? -E : E) : 0;           // s = y & 1, row parity (x + v) & 1
  }
  __device__ __forceinline__ int off(int v, int i) const {
    if constexpr (d == 0) return ((v + i) & 1) ? -f : f;
    else if constexpr (d == 1) return (i & 1) ? ((v & 1) ? -f : f) : 0;
    else return (v & 1) ? -f : f;
  }
};

// Optional per-phase cycle accounting (build with -DSDRT_PHASE_PROF; tools only):
// thread 0 of every CTA adds the clock64() time of each phase after its barrier.
#ifdef SDRT_PHASE_PROF
__device__ unsigned long long g_phase_cycles[2][16];
#define PH_INIT long long ph_t0 = clock64();
#define PH(kern, k)                                                           \
  if (threadIdx.x == 0) {                                                     \
    const long long ph_t1 = clock64();                                        \
    atomicAdd(&g_phase_cycles[kern][k], (unsigned long long)(ph_t1 - ph_t0)); \
    ph_t0 = ph_t1;                                                            \
  }
#else
#define PH_INIT
#define PH(kern, k)
#endif

template <int D, int P>
struct TDims {
  static constexpr int n = P + 1;
  static constexpr int NL = D == 2 ? n : n * n;  // lines per direction (= points per face)
  static constexpr int NS = D == 2 ? n * n : n * n * n;
  static constexpr int NEXT = 2 * D * NL;
};

// first point index and point stride of line t along direction d
template <int D, int P>
__device__ __forceinline__ int lbase(int d, int t) {
  constexpr int n = P + 1;
  if constexpr (D == 2) return d == 0 ? n * t : t;
  return d == 0 ? n * t : (d == 1 ? (t % n) + n * n * (t / n) : t);
}
template <int D, int P>
__device__ __forceinline__ int lstr(int d) {
  constexpr int n = P + 1;
  return d == 0 ? 1 : (d == 1 ? n : n * n);
}

// neighbour element along axis d (delta = -1 / +1), periodic pattern grid, N_p = 1.
// 32-bit arithmetic (K < 2^31); evaluated once per tile element (fill_nbrs).
template <int D>
__device__ __forceinline__ int tnbr(const TensorGeom& g, int e, int d, int delta) {
  // pattern coordinates in registers (no dynamically indexed local array)
  const int c0 = e % g.N[0];
  const int r = e / g.N[0];
  const int c1 = D == 2 ? r : r % g.N[1];
  const int c2 = D == 2 ? 0 : r / g.N[1];
  const int Nd = d == 0 ? g.N[0] : (d == 1 ? g.N[1] : g.N[2]);
  int v = (d == 0 ? c0 : (d == 1 ? c1 : c2)) + delta;
  const bool hal = d == 0 ? g.halo[0] != 0 : (d == 1 ? g.halo[1] != 0 : g.halo[2] != 0);
  if ((v < 0 || v >= Nd) && hal) {
    // ghost column of the neighbouring rank's element: slab (d, side), tangential index
    const int ca = d == 0 ? c1 : c0, cb = d == 2 ? c1 : c2;
    const int na = d == 0 ? g.N[1] : g.N[0];
    const int tang = D == 2 ? ca : ca + na * cb;
    return (int)g.gbase[d][v < 0 ? 0 : 1] + tang;
  }
  v = v < 0 ? v + Nd : (v >= Nd ? v - Nd : v);
  if (d == 0) return v + g.N[0] * (c1 + g.N[1] * c2);
  if (d == 1) return c0 + g.N[0] * (v + g.N[1] * c2);
  return c0 + g.N[0] * (c1 + g.N[1] * v);
}

// neighbour ids of a tile's elements: sNb[2d + side][el] (side 0: x_d - 1, 1: x_d + 1)
template <int D, int E>
__device__ __forceinline__ void fill_nbrs(const TensorGeom& g, int (*sNb)[E], int64_t e0) {
  for (int idx = threadIdx.x; idx < 2 * D * E; idx += blockDim.x) {
    const int el = idx % E, k = idx / E;
    const int e = (int)e0 + el;
    sNb[k][el] = e < g.K ? tnbr<D>(g, e, k / 2, (k % 2) ? 1 : -1) : 0;
  }
}

// value at a line end: explicit fma chain in fixed order (bit-identical wherever used)
template <int n>
__device__ __forceinline__ double interp_end(const double (&Iend)[TMAXP + 1], const double* u) {
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < n; ++i) acc = __fma_rn(Iend[i], u[i], acc);
  return acc;
}

// ---- TMA (cp.async.bulk.tensor) + mbarrier helpers ------------------------------
struct TileMaps {
  CUtensorMap uin, un, acc, rv;  // stage input, u_n, RK accumulator, R_int
};

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Tile load [row][E] <- src[row][e0 .. e0+E): 16-byte cp.async (LDGSTS), all in
// flight at once.  Rows have K_pad >= e0 + E columns (ABI), so no guards are needed;
// padding columns are loaded but never used.
template <int D, int P, int NV, int E>
__device__ __forceinline__ void load_tile(const double* __restrict__ src, double* sU, int64_t e0, int64_t K,
                                          int64_t Kp) {
  constexpr int NS = TDims<D, P>::NS;
  constexpr int CH = E / 2;  // 16-byte chunks per row
  (void)K;
  for (int idx = threadIdx.x; idx < NS * NV * CH; idx += blockDim.x) {
    const int c = idx % CH, row = idx / CH;
    const double* g = src + (int64_t)row * Kp + e0 + 2 * c;
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sU + row * E + 2 * c);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g));
  }
  asm volatile("cp.async.commit_group;");
}

__device__ __forceinline__ void wait_tile() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// L2 prefetch of the rows [N_ext][N_V] of a trace array seen by a tile's face
// neighbours (and optionally of the tile itself)
template <int D, int P, int NV, int E>
__device__ __forceinline__ void prefetch_traces(const TensorGeom& g, const int (*sNb)[E], const double* __restrict__ T,
                                                int64_t e0, bool own) {
  using Tm = TDims<D, P>;
  constexpr int NL = Tm::NL;
  for (int item = threadIdx.x; item < 2 * D * NL * NV; item += blockDim.x) {
    const int v = item % NV, ext = item / NV;
    const int face = ext / NL, d = face / 2, side = face % 2;
    // the neighbour across face (d, side) reads its opposite face (d, 1-side)
    const int ext_n = (2 * d + 1 - side) * NL + ext % NL;
    const int m = sNb[face][0];
    prefetch_l2(T + ((int64_t)ext_n * NV + v) * g.Kt + m);
    if (own) prefetch_l2(T + ((int64_t)ext * NV + v) * g.Kt + e0);
  }
}

template <int D, int P, int NV, int E>
__device__ __forceinline__ void prefetch_rows(const double* __restrict__ A, int64_t e0, int64_t Kp) {
  constexpr int NS = TDims<D, P>::NS;
  for (int row = threadIdx.x; row < NS * NV; row += blockDim.x) prefetch_l2(A + (int64_t)row * Kp + e0);
}

// Phase: gradient along lines -> sQ[d][s][v][E] = (2/h_d) (M16 C + M15 U_int)
// (l.282-302).  One work item = (direction, line, variable, element), statically
// mapped: thread tid owns items tid + k THREADS.  The neighbour traces of all its items
// are loaded into registers first (GradNb::load, issued before the tile wait), so their
// latency overlaps the tile load.
template <int D, int P, int EQ, int E, int THREADS, int NI = P>
struct GradNb {
  using T = TDims<D, P>;
  static constexpr int NV = Phys<EQ, D>::NV;
  static constexpr int ITEMS = D * T::NL * NV * E;
  static constexpr int CI = (ITEMS + THREADS - 1) / THREADS;
  double nb[CI][2];

  __device__ __forceinline__ void load(const TensorGeom& g, const PhysDev& ph, const double* __restrict__ Tu,
                                       const int (*sNb)[E], int64_t e0) {
    constexpr int NL = T::NL;
    const int Kt = (int)g.Kt;
    const double wl = 0.5 - ph.beta, wr = 0.5 + ph.beta;
#pragma unroll
    for (int k = 0; k < CI; ++k) {
      const int item = threadIdx.x + k * THREADS;
      nb[k][0] = nb[k][1] = 0.0;
      if (item < ITEMS) {
        const int el = item % E, r = item / E, v = r % NV, r2 = r / NV, t = r2 % NL, d = r2 / NL;
        if (e0 + el < g.K) {  // a neighbour whose LDG weight is 0 is not read (may be stale)
          if (wl != 0.0) nb[k][0] = Tu[(((2 * d + 1) * NL + t) * NV + v) * Kt + sNb[2 * d][el]];
          if (wr != 0.0) nb[k][1] = Tu[(((2 * d + 0) * NL + t) * NV + v) * Kt + sNb[2 * d + 1][el]];
        }
      }
    }
  }

  // sNbR (OSF): the right neighbours' traces nb[.][1] are also stored to sNbR[d][t][v][el]
  // for publish_F (the same (d, t, v, el) entries)
  template <bool SWZ = false>
  __device__ __forceinline__ void compute(const TensorGeom& g, const Line1D& L, const PhysDev& ph, const double* sU,
                                          double* sQ, int64_t e0, double* sNbR = nullptr) const {
    constexpr int n = T::n, NL = T::NL, NS = T::NS;
    static_assert(!SWZ || SDRT_TA_GQ != 0, "swizzled sQ: composite-operator gradient only");
    const double wl = 0.5 - ph.beta, wr = 0.5 + ph.beta;
#pragma unroll
    for (int k = 0; k < CI; ++k) {
      const int item = threadIdx.x + k * THREADS;
      if (item >= ITEMS) break;
      const int el = item % E, r = item / E, v = r % NV, r2 = r / NV, t = r2 % NL, d = r2 / NL;
      if (e0 + el >= g.K) continue;
      if (sNbR) sNbR[item] = nb[k][1];
      const int lb = lbase<D, P>(d, t), ls = lstr<D, P>(d);
      double u[n];
#pragma unroll
      for (int i = 0; i < n; ++i) u[i] = sU[((lb + i * ls) * NV + v) * E + el];
#if SDRT_TA_GQ
      // composite operator (Line1D::Gq); d is warp-uniform (items are d-major), so the
      // branches select compile-time coefficient sets
      auto gq = [&](auto dc) {
        constexpr int dd = decltype(dc)::value;
#pragma unroll
        for (int i = 0; i < n; ++i) {
          double q = L.H0[dd][i] * nb[k][0];
          q = fma(L.H1[dd][i], nb[k][1], q);
#pragma unroll
          for (int j = 0; j < n; ++j) q = fma(L.Gq[dd][i][j], u[j], q);
          if constexpr (SWZ) {  // SDRT_TA_QSWZ: row r of point s at r ^ ((s >> 2) & 1)
            const int pt = lb + i * ls, row = (dd * NS + pt) * NV + v;
            sQ[(row ^ ((pt >> 2) & 1)) * E + el] = q;
          } else {
            sQ[((dd * NS + (lb + i * ls)) * NV + v) * E + el] = q;
          }
        }
      };
      if (d == 0) gq(std::integral_constant<int, 0>{});
      else if (d == 1) gq(std::integral_constant<int, 1>{});
      else if constexpr (D == 3) gq(std::integral_constant<int, 2>{});
      continue;
#endif
      // common values at both ends (own trace recomputed bit-identically, neighbour read)
      const double own0 = interp_end<n>(L.Iend[0], u), own1 = interp_end<n>(L.Iend[1], u);
      // face x_d = -1: this element is RIGHT; face x_d = +1: this element is LEFT
      const double c0 = wl != 0.0 ? wl * nb[k][0] + wr * own0 : own0;
      const double c1 = wr != 0.0 ? wl * own1 + wr * nb[k][1] : own1;
      double ui[NI];
#pragma unroll
      for (int a = 0; a < NI; ++a) {
        if constexpr (NI == n) {  // FR: the flux points are the solution points (Iint = I)
          ui[a] = u[a];
        } else {
          double s = 0.0;
#pragma unroll
          for (int i = 0; i < n; ++i) s = fma(L.Iint[a][i], u[i], s);
          ui[a] = s;
        }
      }
      const double jd = g.jinv[d];
#pragma unroll
      for (int i = 0; i < n; ++i) {
        double q = L.Dfl[i][0] * c0;
#pragma unroll
        for (int a = 0; a < NI; ++a) q = fma(L.Dfl[i][a + 1], ui[a], q);
        q = fma(L.Dfl[i][NI + 1], c1, q);
        sQ[((d * NS + (lb + i * ls)) * NV + v) * E + el] = jd * q;
      }
    }
  }
};

// GradNb on element pairs (el0, el0 + 1): 16-byte shared-memory loads and stores, the
// same arithmetic per element (SDRT_TA_GPAIR)
template <int D, int P, int EQ, int E, int THREADS, int NI = P>
struct GradNb2 {
  using T = TDims<D, P>;
  static constexpr int NV = Phys<EQ, D>::NV;
  static constexpr int E2 = E / 2;
  static constexpr int ITEMS = D * T::NL * NV * E2;
  static constexpr int CI = (ITEMS + THREADS - 1) / THREADS;
  double nb[CI][2][2];  // [item][element of the pair][face side]

  __device__ __forceinline__ void load(const TensorGeom& g, const PhysDev& ph, const double* __restrict__ Tu,
                                       const int (*sNb)[E], int64_t e0) {
    constexpr int NL = T::NL;
    const int Kt = (int)g.Kt;
    const double wl = 0.5 - ph.beta, wr = 0.5 + ph.beta;
#pragma unroll
    for (int k = 0; k < CI; ++k) {
      const int item = threadIdx.x + k * THREADS;
#pragma unroll
      for (int h = 0; h < 2; ++h) nb[k][h][0] = nb[k][h][1] = 0.0;
      if (item < ITEMS) {
        const int el0 = 2 * (item % E2), r = item / E2, v = r % NV, r2 = r / NV, t = r2 % NL, d = r2 / NL;
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (e0 + el0 + h < g.K) {
            if (wl != 0.0) nb[k][h][0] = Tu[(((2 * d + 1) * NL + t) * NV + v) * Kt + sNb[2 * d][el0 + h]];
            if (wr != 0.0) nb[k][h][1] = Tu[(((2 * d + 0) * NL + t) * NV + v) * Kt + sNb[2 * d + 1][el0 + h]];
          }
      }
    }
  }

  __device__ __forceinline__ void compute(const TensorGeom& g, const Line1D& L, const PhysDev& ph, const double* sU,
                                          double* sQ, int64_t e0, double* = nullptr) const {
    constexpr int n = T::n, NL = T::NL, NS = T::NS;
    const double wl = 0.5 - ph.beta, wr = 0.5 + ph.beta;
#pragma unroll
    for (int k = 0; k < CI; ++k) {
      const int item = threadIdx.x + k * THREADS;
      if (item >= ITEMS) break;
      const int el0 = 2 * (item % E2), r = item / E2, v = r % NV, r2 = r / NV, t = r2 % NL, d = r2 / NL;
      const int lb = lbase<D, P>(d, t), ls = lstr<D, P>(d);
      double u[2][n];
#pragma unroll
      for (int i = 0; i < n; ++i) {
        const double2 x = *reinterpret_cast<const double2*>(sU + ((lb + i * ls) * NV + v) * E + el0);
        u[0][i] = x.x;
        u[1][i] = x.y;
      }
#if SDRT_TA_GQ
      // composite operator (Line1D::Gq), d warp-uniform (items d-major): compile-time
      // coefficient sets per branch
      auto gq2 = [&](auto dc) {
        constexpr int dd = decltype(dc)::value;
#pragma unroll
        for (int i = 0; i < n; ++i) {
          double q0 = L.H0[dd][i] * nb[k][0][0], q1 = L.H0[dd][i] * nb[k][1][0];
          q0 = fma(L.H1[dd][i], nb[k][0][1], q0);
          q1 = fma(L.H1[dd][i], nb[k][1][1], q1);
#pragma unroll
          for (int j = 0; j < n; ++j) {
            q0 = fma(L.Gq[dd][i][j], u[0][j], q0);
            q1 = fma(L.Gq[dd][i][j], u[1][j], q1);
          }
          *reinterpret_cast<double2*>(sQ + ((dd * NS + (lb + i * ls)) * NV + v) * E + el0) = make_double2(q0, q1);
        }
      };
      if (d == 0) gq2(std::integral_constant<int, 0>{});
      else if (d == 1) gq2(std::integral_constant<int, 1>{});
      else if constexpr (D == 3) gq2(std::integral_constant<int, 2>{});
      continue;
#endif
      const double jd = g.jinv[d];
      double q2[2][n];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double own0 = interp_end<n>(L.Iend[0], u[h]), own1 = interp_end<n>(L.Iend[1], u[h]);
        const double c0 = wl != 0.0 ? wl * nb[k][h][0] + wr * own0 : own0;
        const double c1 = wr != 0.0 ? wl * own1 + wr * nb[k][h][1] : own1;
        double ui[NI];
#pragma unroll
        for (int a = 0; a < NI; ++a) {
          if constexpr (NI == n) {
            ui[a] = u[h][a];
          } else {
            double s = 0.0;
#pragma unroll
            for (int i = 0; i < n; ++i) s = fma(L.Iint[a][i], u[h][i], s);
            ui[a] = s;
          }
        }
#pragma unroll
        for (int i = 0; i < n; ++i) {
          double q = L.Dfl[i][0] * c0;
#pragma unroll
          for (int a = 0; a < NI; ++a) q = fma(L.Dfl[i][a + 1], ui[a], q);
          q = fma(L.Dfl[i][NI + 1], c1, q);
          q2[h][i] = jd * q;
        }
      }
#pragma unroll
      for (int i = 0; i < n; ++i)
        *reinterpret_cast<double2*>(sQ + ((d * NS + (lb + i * ls)) * NV + v) * E + el0) = make_double2(q2[0][i], q2[1][i]);
    }
  }
};

// traces of a state held in shared memory -> T[N_ext][N_V][Kt]
template <int D, int P, int NV, int E>
__device__ __forceinline__ void write_traces(const TensorGeom& g, const Line1D& L, const double* sU,
                                             double* __restrict__ T, int64_t e0) {
  using Tm = TDims<D, P>;
  constexpr int n = Tm::n, NL = Tm::NL;
  for (int item = threadIdx.x; item < 2 * D * NL * NV * E; item += blockDim.x) {
    const int el = item % E, r = item / E, v = r % NV, r2 = r / NV, t = r2 % NL, face = r2 / NL;
    const int64_t e = e0 + el;
    if (e >= g.K) continue;
    const int d = face / 2, side = face % 2;
    const int lb = lbase<D, P>(d, t), ls = lstr<D, P>(d);
    double u[n];
#pragma unroll
    for (int i = 0; i < n; ++i) u[i] = sU[((lb + i * ls) * NV + v) * E + el];
    T[((int64_t)(face * NL + t) * NV + v) * g.Kt + e] = interp_end<n>(L.Iend[side], u);
  }
}

template <int D, int P, int EQ, int E>
__global__ void __launch_bounds__(256) kt_traces(TensorGeom g, Line1D L, const __grid_constant__ TileMaps tm,
                                                 double* __restrict__ T) {
  pdl_wait();
  constexpr int NV = Phys<EQ, D>::NV;
  constexpr int ROWS = TDims<D, P>::NS * NV;
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t bar;
  const int64_t e0 = (int64_t)(g.tiles ? g.tiles[blockIdx.x] : (int)blockIdx.x) * E;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
    mbar_expect_tx(&bar, ROWS * E * 8);
    tma_tile<ROWS, E>(smem, &tm.uin, e0, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  write_traces<D, P, NV, E>(g, L, smem, T, e0);
}

// kernel A keeps two internal-flux buffers when both fit two CTAs per SM
// (OSF adds the [D][NL][NV][E] face buffer; two CTAs of <= 112.9 KB fit per SM)
__host__ __device__ constexpr bool tensor_a_dbuf(int D, int NS, int NL, int NV, int E, int NI, bool osf = false) {
  return (size_t)(NS * NV * E * (1 + D) + 2 * NL * NI * NV * E + (osf ? D * NL * NV * E : 0)) * sizeof(double) <=
         112 * 1024;
}

// Kernel A phase helpers -----------------------------------------------------------
// publish g = n_L . f^v(u, q) at the face point (d, side, t) of element slot el
template <int D, int P, int EQ, int E, int d>
__device__ __forceinline__ void publish_g(const TensorGeom& g, const Line1D& L, const PhysDev& ph, const double* sU,
                                          const double* sQ, double* __restrict__ Tg, int64_t e0, int side, int t,
                                          int el) {
  using Ph = Phys<EQ, D>;
  using T = TDims<D, P>;
  constexpr int NV = Ph::NV, n = T::n, NL = T::NL, NS = T::NS;
  const int64_t e = e0 + el;
  if (e >= g.K) return;
  const int ext = (2 * d + side) * NL + t;
  const int lb = lbase<D, P>(d, t), ls = lstr<D, P>(d);
  double u[NV], q[D * NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double ul[n];
#pragma unroll
    for (int i = 0; i < n; ++i) ul[i] = sU[((lb + i * ls) * NV + v) * E + el];
    u[v] = interp_end<n>(L.Iend[side], ul);
#pragma unroll
    for (int dd = 0; dd < D; ++dd) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < n; ++i) s = fma(L.Iend[side][i], sQ[((dd * NS + (lb + i * ls)) * NV + v) * E + el], s);
      q[dd * NV + v] = s;
    }
  }
  double gv[NV];
  Ph::template visc_axis<d>(ph, u, q, 1.0, gv);  // canonical (left) normal +e_d
#pragma unroll
  for (int v = 0; v < NV; ++v) Tg[((int64_t)ext * NV + v) * g.Kt + e] = gv[v];
}

// One-sided flux publication (OSF; beta = +1/2, the TGV settings of c4/c5, O15): with
// LDG weights (1/2 + b, 1/2 - b) = (1, 0) the common viscous flux of a face is the LEFT
// element's g alone (l.330-335), and the common value is the RIGHT element's trace
// (l.282-291), so the left element holds every input of the face's whole common flux
// F = Rusanov(u_L, u_R) + g_L + eta (u_L - u_R) (l.312-340) once it has its gradient:
// kernel A evaluates F ONCE per face at its x_d = +1 ends (this element LEFT; u_R = the
// right neighbour's published trace), publishes it in the g slot of T_g, and adds the
// face's M14 term to R_int; kernel B only reads the left neighbours' F for its x_d = -1
// faces.  Both sides apply the same stored number: D~_R = -D~_L bitwise (O28).
template <int D, int P, int EQ, int E, int d>
// sP [NL][NV][E] of direction d: on entry the right neighbours' x_d = -1 traces (stored by
// GradNb), on exit sface F (read by the divergence of direction d)
__device__ __forceinline__ void publish_F(const TensorGeom& g, const Line1D& L, const PhysDev& ph, const double* sU,
                                          const double* sQ, const TensorBufs& b, double* sP, int64_t e0, int t,
                                          int el) {
  using Ph = Phys<EQ, D>;
  using T = TDims<D, P>;
  constexpr int NV = Ph::NV, n = T::n, NL = T::NL, NS = T::NS;
  const int64_t e = e0 + el;
  if (e >= g.K) return;
  const int ext = (2 * d + 1) * NL + t;  // own x_d = +1 end
  double uR[NV];  // the right neighbour's x_d = -1 trace
#pragma unroll
  for (int v = 0; v < NV; ++v) uR[v] = sP[(t * NV + v) * E + el];
  const int lb = lbase<D, P>(d, t), ls = lstr<D, P>(d);
  double u[NV], q[D * NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double ul[n];
#pragma unroll
    for (int i = 0; i < n; ++i) ul[i] = sU[((lb + i * ls) * NV + v) * E + el];
    u[v] = interp_end<n>(L.Iend[1], ul);
#pragma unroll
    for (int dd = 0; dd < D; ++dd) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < n; ++i) s = fma(L.Iend[1][i], sQ[((dd * NS + (lb + i * ls)) * NV + v) * E + el], s);
      q[dd * NV + v] = s;
    }
  }
  double gv[NV], F[NV];
  Ph::template visc_axis<d>(ph, u, q, 1.0, gv);  // canonical (left) normal +e_d
  Ph::template conv_common_axis<d>(ph, u, uR, F);
  const double wl = 0.5 + ph.beta;  // = 1
  const double sface = g.sface[d];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    F[v] = Ph::ldg_rn(F[v], __dmul_rn(wl, gv[v]), ph.eta, u[v], uR[v]);
    b.Tg[((int64_t)ext * NV + v) * g.Kt + e] = F[v];
    sP[(t * NV + v) * E + el] = sface * F[v];
  }
  if (b.Fexp) {  // O28 export (residual only): F at the own ext point
#pragma unroll
    for (int v = 0; v < NV; ++v) b.Fexp[((int64_t)ext * NV + v) * g.Kp + e] = F[v];
  }
}

// internal transformed flux F~ = detJ (J^-1 (f^c - f^v))_d at internal point a of d-line t
// (one normal component, B7; l.305-311) -> sF[t][a][v][el]
template <int D, int P, int EQ, int E, int d, int NI, int AC = -1>
__device__ __forceinline__ void visc_internal(const TensorGeom& g, const Line1D& L, const PhysDev& ph,
                                              const double* sU, const double* sQ, double* sF, int t, int a_, int el) {
  const int a = AC >= 0 ? AC : a_;  // AC: internal point index known at compile time
  using Ph = Phys<EQ, D>;
  using T = TDims<D, P>;
  constexpr int NV = Ph::NV, n = T::n, NS = T::NS;
  const int lb = lbase<D, P>(d, t), ls = lstr<D, P>(d);
  double ua[NV], qa[D * NV];
  if constexpr (NI == n) {  // FR: the flux points are the solution points (Iint = I)
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      ua[v] = sU[((lb + a * ls) * NV + v) * E + el];
#pragma unroll
      for (int dd = 0; dd < D; ++dd) qa[dd * NV + v] = sQ[((dd * NS + (lb + a * ls)) * NV + v) * E + el];
    }
  } else {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < n; ++i) s = fma(L.Iint[a][i], sU[((lb + i * ls) * NV + v) * E + el], s);
      ua[v] = s;
#pragma unroll
      for (int dd = 0; dd < D; ++dd) {
        double s2 = 0.0;
#pragma unroll
        for (int i = 0; i < n; ++i) s2 = fma(L.Iint[a][i], sQ[((dd * NS + (lb + i * ls)) * NV + v) * E + el], s2);
        qa[dd * NV + v] = s2;
      }
    }
  }
  double fc[NV], fv[NV];
  const double wf = g.detJ * g.jinv[d];
  Ph::template conv_axis<d>(ph, ua, wf, fc);
  Ph::template visc_axis<d>(ph, ua, qa, wf, fv);
#pragma unroll
  for (int v = 0; v < NV; ++v) sF[((t * NI + a) * NV + v) * E + el] = fc[v] + fv[v];
}

// Streamed line item (SDRT_TA_SLINE, one-sided flux publication path): one item = all NI
// internal flux points of one d-line t of one element.  Each component the axis physics
// reads (u_v; q[d][.]; q[j][0], q[j][1+d], q[j][1+j] for j != d) is loaded from shared
// memory ONCE (n values) and interpolated to the NI points from registers, instead of
// once per point (visc_internal: NI x the loads).  A compiler memory fence after each
// component keeps the next component's loads from being hoisted (at most n loads in
// flight), so the NI points' inputs (NI x 16 values) plus the physics fit the 128
// registers of two 256-thread CTAs per SM.  The interpolation sums are the same fma
// chains as visc_internal's (bitwise the per-point items).
template <int D, int P, int EQ, int E, int d, int NI>
__device__ __forceinline__ void visc_sline(const TensorGeom& g, const Line1D& L, const PhysDev& ph, const double* sU,
                                           const double* sQ, double* sF, int t, int el) {
  using Ph = Phys<EQ, D>;
  using T = TDims<D, P>;
  constexpr int NV = Ph::NV, n = T::n, NS = T::NS;
  static_assert(NI < n, "streamed line items: SDRT internal points only");
  const int lb = lbase<D, P>(d, t), ls = lstr<D, P>(d);
  double ua[NI][NV], qa[NI][D * NV];
#pragma unroll
  for (int c = 0; c < NV + D * NV; ++c) {
    const int dd = c < NV ? -1 : (c - NV) / NV, v = c < NV ? c : (c - NV) % NV;
    if (dd >= 0 && !(dd == d || v == 0 || v == 1 + d || v == 1 + dd)) {
#pragma unroll
      for (int a = 0; a < NI; ++a) qa[a][dd * NV + v] = 0.0;  // not read by visc_axis<d>
      continue;
    }
    const double* base = dd < 0 ? sU + (lb * NV + v) * E + el : sQ + ((dd * NS + lb) * NV + v) * E + el;
    double x[n];
#pragma unroll
    for (int i = 0; i < n; ++i) x[i] = base[i * ls * NV * E];
#pragma unroll
    for (int a = 0; a < NI; ++a) {
      double s2 = 0.0;
#pragma unroll
      for (int i = 0; i < n; ++i) s2 = fma(L.Iint[a][i], x[i], s2);
      if (dd < 0) ua[a][v] = s2;
      else qa[a][dd * NV + v] = s2;
    }
    asm volatile("" ::: "memory");
  }
  const double wf = g.detJ * g.jinv[d];
#pragma unroll
  for (int a = 0; a < NI; ++a) {
    double fc[NV], fv[NV];
    Ph::template conv_axis<d>(ph, ua[a], wf, fc);
    Ph::template visc_axis<d>(ph, ua[a], qa[a], wf, fv);
#pragma unroll
    for (int v = 0; v < NV; ++v) sF[((t * NI + a) * NV + v) * E + el] = fc[v] + fv[v];
    asm volatile("" ::: "memory");
  }
}

// Half-line items (SDRT_TA_SLINE = 2, one-sided flux publication): the outputs of a d-line
// -- its NI internal flux points and its published x_d = +1 end -- split over TWO items of
// (almost) equal work: H = 0 the first ceil(NI/2) internal points, H = 1 the others plus
// the end (publish_F's common flux).  Each item loads every component it needs once and
// interpolates it to its two outputs from registers (half the loads of per-point items,
// 2 x 16 live inputs).  Same arithmetic as visc_internal / publish_F (bitwise).
template <int D, int P, int EQ, int E, int d, int NI, int H, bool SWZ = false>
__device__ __forceinline__ void visc_hline(const TensorGeom& g, const Line1D& L, const PhysDev& ph, const double* sU,
                                           const double* sQ, double* sF, const TensorBufs& b, double* sP,
                                           int64_t e0, int t, int el) {
  using Ph = Phys<EQ, D>;
  using T = TDims<D, P>;
  constexpr int NV = Ph::NV, n = T::n, NS = T::NS, NL = T::NL;
  static_assert(NI < n, "half-line items: SDRT internal points only");
  constexpr int A0 = H == 0 ? 0 : (NI + 1) / 2;           // first internal point
  constexpr int NA = H == 0 ? (NI + 1) / 2 : NI - A0;     // internal points of this item
  constexpr int NO = NA + H;                              // + the published end (H = 1)
  const int lb = lbase<D, P>(d, t), ls = lstr<D, P>(d);
  static_assert(!SWZ || (D == 3 && n == 4 && (NV & 1) == 1 && E == 8), "swizzled sQ: hex p = 3, odd N_V, 8-element tiles");
  const QSwz<d, E> qz(t);
  double uo[NO][NV], qo[NO][D * NV];
  constexpr int NC = NV + D * NV;
  // component c = (dd, v): dd = -1 the state, else the gradient along dd; needed by visc_axis<d>?
  auto needed = [](int c) {
    const int dd = c < NV ? -1 : (c - NV) / NV, v = c < NV ? c : (c - NV) % NV;
    return dd < 0 || dd == d || v == 0 || v == 1 + d || v == 1 + dd;
  };
  auto ld = [&](int c, double (&x)[n]) {  // the n line values of component c
    const int dd = c < NV ? -1 : (c - NV) / NV, v = c < NV ? c : (c - NV) % NV;
    const double* base = dd < 0 ? sU + (lb * NV + v) * E + el : sQ + ((dd * NS + lb) * NV + v) * E + el;
    if constexpr (SWZ) {
#pragma unroll
      for (int i = 0; i < n; ++i) x[i] = base[i * ls * NV * E + (dd < 0 ? 0 : qz.off(v, i))];
    } else {
#pragma unroll
      for (int i = 0; i < n; ++i) x[i] = base[i * ls * NV * E];
    }
  };
  double x[n], xn[n];
  if constexpr (SDRT_TA_HPIPE != 0) ld(0, x);
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int dd = c < NV ? -1 : (c - NV) / NV, v = c < NV ? c : (c - NV) % NV;
    if (!needed(c)) {
#pragma unroll
      for (int o = 0; o < NO; ++o) qo[o][dd * NV + v] = 0.0;  // not read by visc_axis<d>
      continue;
    }
    if constexpr (SDRT_TA_HPIPE != 0) {  // the next needed component's loads before this one's sums
      int c2 = c + 1;
      while (c2 < NC && !needed(c2)) ++c2;
      if (c2 < NC) ld(c2, xn);
    } else {
      ld(c, x);
    }
#pragma unroll
    for (int o = 0; o < NO; ++o) {
      double s2;
      if (o < NA) {
        s2 = 0.0;
#pragma unroll
        for (int i = 0; i < n; ++i) s2 = fma(L.Iint[A0 + o][i], x[i], s2);
      } else if (dd < 0) {
        s2 = interp_end<n>(L.Iend[1], x);
      } else {
        s2 = 0.0;
#pragma unroll
        for (int i = 0; i < n; ++i) s2 = fma(L.Iend[1][i], x[i], s2);
      }
      if (dd < 0) uo[o][v] = s2;
      else qo[o][dd * NV + v] = s2;
    }
    if constexpr (SDRT_TA_HPIPE != 0) {
#pragma unroll
      for (int i = 0; i < n; ++i) x[i] = xn[i];
    }
    asm volatile("" ::: "memory");
  }
  const double wf = g.detJ * g.jinv[d];
#pragma unroll
  for (int o = 0; o < NA; ++o) {
    double fc[NV], fv[NV];
    Ph::template conv_axis<d>(ph, uo[o], wf, fc);
    Ph::template visc_axis<d>(ph, uo[o], qo[o], wf, fv);
#pragma unroll
    for (int v = 0; v < NV; ++v) sF[((t * NI + A0 + o) * NV + v) * E + el] = fc[v] + fv[v];
  }
  if constexpr (H == 1) {  // the x_d = +1 end: publish_F
    const int64_t e = e0 + el;
    if (e >= g.K) return;
    const int ext = (2 * d + 1) * NL + t;
    double* p1 = sP + d * NL * NV * E;
    double uR[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) uR[v] = p1[(t * NV + v) * E + el];
    double gv[NV], F[NV];
    Ph::template visc_axis<d>(ph, uo[NA], qo[NA], 1.0, gv);
    Ph::template conv_common_axis<d>(ph, uo[NA], uR, F);
    const double wl = 0.5 + ph.beta;
    const double sface = g.sface[d];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      F[v] = Ph::ldg_rn(F[v], __dmul_rn(wl, gv[v]), ph.eta, uo[NA][v], uR[v]);
      b.Tg[((int64_t)ext * NV + v) * g.Kt + e] = F[v];
      p1[(t * NV + v) * E + el] = sface * F[v];
    }
    if (b.Fexp) {
#pragma unroll
      for (int v = 0; v < NV; ++v) b.Fexp[((int64_t)ext * NV + v) * g.Kp + e] = F[v];
    }
  }
}

// visc_internal for the element pair (el0, el0 + 1): 16-byte shared-memory loads
// (SDRT_TA_PAIR), the physics evaluated per element
template <int D, int P, int EQ, int E, int d, int NI>
__device__ __forceinline__ void visc_internal2(const TensorGeom& g, const Line1D& L, const PhysDev& ph,
                                               const double* sU, const double* sQ, double* sF, int t, int a,
                                               int el0) {
  using Ph = Phys<EQ, D>;
  using T = TDims<D, P>;
  constexpr int NV = Ph::NV, n = T::n, NS = T::NS;
  const int lb = lbase<D, P>(d, t), ls = lstr<D, P>(d);
  auto ld2 = [&](const double* base, int idx) { return *reinterpret_cast<const double2*>(base + idx * E + el0); };
  double2 ua[NV], qa[D * NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    if constexpr (NI == n) {
      ua[v] = ld2(sU, (lb + a * ls) * NV + v);
#pragma unroll
      for (int dd = 0; dd < D; ++dd) qa[dd * NV + v] = ld2(sQ, (dd * NS + (lb + a * ls)) * NV + v);
    } else {
      double2 s = make_double2(0.0, 0.0);
#pragma unroll
      for (int i = 0; i < n; ++i) {
        const double2 x = ld2(sU, (lb + i * ls) * NV + v);
        s.x = fma(L.Iint[a][i], x.x, s.x);
        s.y = fma(L.Iint[a][i], x.y, s.y);
      }
      ua[v] = s;
#pragma unroll
      for (int dd = 0; dd < D; ++dd) {
        double2 s2 = make_double2(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < n; ++i) {
          const double2 x = ld2(sQ, (dd * NS + (lb + i * ls)) * NV + v);
          s2.x = fma(L.Iint[a][i], x.x, s2.x);
          s2.y = fma(L.Iint[a][i], x.y, s2.y);
        }
        qa[dd * NV + v] = s2;
      }
    }
  }
  const double wf = g.detJ * g.jinv[d];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    double u1[NV], q1[D * NV], fc[NV], fv[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) u1[v] = h ? ua[v].y : ua[v].x;
#pragma unroll
    for (int k = 0; k < D * NV; ++k) q1[k] = h ? qa[k].y : qa[k].x;
    Ph::template conv_axis<d>(ph, u1, wf, fc);
    Ph::template visc_axis<d>(ph, u1, q1, wf, fv);
#pragma unroll
    for (int v = 0; v < NV; ++v) sF[((t * NI + a) * NV + v) * E + el0 + h] = fc[v] + fv[v];
  }
}

// Register-blocked line item (SDRT_TA_LINE): one item = one d-line t of one element.
// The outputs of the line -- its NI internal flux points and the published end(s) --
// are produced in passes of LGRP outputs: per pass, every component the axis physics
// reads (u and the gradient entries; the others are dead code) is loaded from shared
// memory once and interpolated to the pass's outputs from registers (the line
// operators are kernel parameters: constant-bank DFMA operands), so one shared-memory
// load feeds LGRP DFMAs instead of one, with LGRP x (N_V + D N_V) accumulators live.
// Outputs: internal transformed fluxes F~ = detJ J^-1 (f^c - f^v) -> sF[t][a][v][el],
// published viscous normal flux g = n_L . f^v at the end(s) -> Tg (PAPER.md l.305-311,
// l.330-335; B7 l.2927-2932).
// scalar equations (N_V = 1): all outputs of a line in one pass
#ifndef SDRT_TA_LGRP
#define SDRT_TA_LGRP 4
#endif
// systems (N_V > 1, the NS registers): line items on/off, outputs per pass, and whether
// each pass is its own item (SDRT_TA_LSPLIT_SYS = 1).  Measured on c4 (hex p=3 NS, kernel
// A per launch): per-point items 251 us; line items with 128-thread CTAs (254 registers,
// 8 warps / SM) 253 us; one item per 2-output pass at 256 threads (spills) 291 us;
// per-output passes 337 us.  The NS line items need ~2x the registers, which halves the
// resident warps and cancels the 40 % cut in shared-memory wavefronts; off for systems.
#ifndef SDRT_TA_LINE_SYS
#define SDRT_TA_LINE_SYS 0
#endif
#ifndef SDRT_TA_LGRP_SYS
#define SDRT_TA_LGRP_SYS 2
#endif
#ifndef SDRT_TA_LSPLIT_SYS
#define SDRT_TA_LSPLIT_SYS 1
#endif
// PUB: published ends, bit 0 = the x_d = -1 end (side 0), bit 1 = the x_d = +1 end
// G: outputs per pass; SPLIT: the line's passes are separate items (gsel = this item's)
template <int D, int P, int EQ, int E, int d, int NI, int PUB, int G, bool SPLIT>
__device__ __forceinline__ void visc_line(const TensorGeom& g, const Line1D& L, const PhysDev& ph, const double* sU,
                                          const double* sQ, double* sF, double* __restrict__ Tg, int64_t e0, int t,
                                          int el, int gsel) {
  using Ph = Phys<EQ, D>;
  using T = TDims<D, P>;
  constexpr int NV = Ph::NV, n = T::n, NS = T::NS, NL = T::NL;
  constexpr int NC = NV + D * NV;  // components: u_v, then q[dd][v]
  constexpr int NO = NI + (PUB & 1) + (PUB >> 1 & 1);
  const int lb = lbase<D, P>(d, t), ls = lstr<D, P>(d);
  const double wf = g.detJ * g.jinv[d];
  const int64_t e = e0 + el;
#pragma unroll
  for (int g0 = 0; g0 < NO; g0 += G) {
    if (SPLIT && g0 != gsel * G) continue;
    double o[G][NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double* base = c < NV ? sU + (lb * NV + c) * E + el : sQ + (((c / NV - 1) * NS + lb) * NV + c % NV) * E + el;
      double x[n];
#pragma unroll
      for (int i = 0; i < n; ++i) x[i] = base[i * ls * NV * E];
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const int k = g0 + j;
        if (k >= NO) break;
        if (k < NI) {
          if constexpr (NI == n) {  // FR: the flux points are the solution points (Iint = I)
            o[j][c] = x[k];
          } else {
            double s = L.Iint[k][0] * x[0];
#pragma unroll
            for (int i = 1; i < n; ++i) s = fma(L.Iint[k][i], x[i], s);
            o[j][c] = s;
          }
        } else {
          const int side = PUB == 3 ? k - NI : (PUB == 2 ? 1 : 0);
          o[j][c] = interp_end<n>(L.Iend[side], x);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const int k = g0 + j;
      if (k >= NO) break;
      if (k < NI) {
        double fc[NV], fv[NV];
        Ph::template conv_axis<d>(ph, o[j], wf, fc);
        Ph::template visc_axis<d>(ph, o[j], o[j] + NV, wf, fv);
#pragma unroll
        for (int v = 0; v < NV; ++v) sF[((t * NI + k) * NV + v) * E + el] = fc[v] + fv[v];
      } else if (e < g.K) {
        const int side = PUB == 3 ? k - NI : (PUB == 2 ? 1 : 0);
        double gv[NV];
        Ph::template visc_axis<d>(ph, o[j], o[j] + NV, 1.0, gv);  // canonical (left) normal +e_d
        const int ext = (2 * d + side) * NL + t;
#pragma unroll
        for (int v = 0; v < NV; ++v) Tg[((int64_t)ext * NV + v) * g.Kt + e] = gv[v];
      }
    }
  }
}

// FP64 tensor-core (DMMA m8n8k4) form of a d-line's interpolations (SDRT_TA_DMMA):
// one warp per line t, the 8 x 4 operator [Iint (NI rows); Iend (2 rows); 0] applied to
// every needed component (u_v and the gradient entries, the line's points as k, the 8
// tile elements as columns).  Lane (r = lane / 4, elements 2 (lane % 4) + {0, 1}) then
// holds all components at point r of its two elements: r < NI internal flux point ->
// F~ into sF; r = NI + side (published side) -> g = n_L . f^v into Tg.  The mma is a pure
// asm statement, so products whose outputs the axis physics never reads are removed.
__device__ __forceinline__ void dmma_pure(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

template <int D, int P, int EQ, int E, int d, int NI>
__device__ __forceinline__ void visc_line_dmma(const TensorGeom& g, const Line1D& L, const PhysDev& ph,
                                               const double* sU, const double* sQ, double* sF,
                                               double* __restrict__ Tg, int64_t e0, int t, bool pub0, bool pub1) {
  static_assert(E == 8, "one 8-column tile per line");
  using Ph = Phys<EQ, D>;
  using T = TDims<D, P>;
  constexpr int NV = Ph::NV, n = T::n, NS = T::NS, NL = T::NL, KT = (n + 3) / 4;
  static_assert(NI + 2 <= 8, "operator rows");
  const int lane = threadIdx.x & 31;
  const int r = lane >> 2, kc = lane & 3, col = lane >> 2;
  const int lb = lbase<D, P>(d, t), ls = lstr<D, P>(d);
  double a[KT];
#pragma unroll
  for (int k = 0; k < KT; ++k) {
    const int i = 4 * k + kc;
    double v = 0.0;
    if (i < n) {
      if (r < NI) v = (NI == n) ? (r == i ? 1.0 : 0.0) : L.Iint[r][i];
      else if (r == NI) v = L.Iend[0][i];
      else if (r == NI + 1) v = L.Iend[1][i];
    }
    a[k] = v;
  }
  auto line = [&](const double* base) {  // base: the component's point-0 row at element 0
    double c0 = 0.0, c1 = 0.0;
#pragma unroll
    for (int k = 0; k < KT; ++k) {
      const int i = 4 * k + kc;
      const double b = i < n ? base[(i * ls) * NV * E + col] : 0.0;
      dmma_pure(c0, c1, a[k], b);
    }
    return make_double2(c0, c1);
  };
  double2 cu[NV], cq[D * NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) cu[v] = line(sU + (lb * NV + v) * E);
#pragma unroll
  for (int dd = 0; dd < D; ++dd)
#pragma unroll
    for (int v = 0; v < NV; ++v) cq[dd * NV + v] = line(sQ + ((dd * NS + lb) * NV + v) * E);
  const bool inner = r < NI;
  const int side = r - NI;
  const bool pub = (side == 0 && pub0) || (side == 1 && pub1);
  if (!inner && !pub) return;
  const double wf = g.detJ * g.jinv[d];
  const double wd = inner ? wf : 1.0;  // canonical (left) normal +e_d for the published g
  const int ext = (2 * d + (side > 0 ? 1 : 0)) * NL + t;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int el = 2 * kc + h;
    double u[NV], q[D * NV], fc[NV], fv[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) u[v] = h ? cu[v].y : cu[v].x;
#pragma unroll
    for (int k = 0; k < D * NV; ++k) q[k] = h ? cq[k].y : cq[k].x;
    Ph::template visc_axis<d>(ph, u, q, wd, fv);
    if (inner) {
      Ph::template conv_axis<d>(ph, u, wf, fc);
#pragma unroll
      for (int v = 0; v < NV; ++v) sF[((t * NI + r) * NV + v) * E + el] = fc[v] + fv[v];
    } else if (e0 + el < g.K) {
#pragma unroll
      for (int v = 0; v < NV; ++v) Tg[((int64_t)ext * NV + v) * g.Kt + e0 + el] = fv[v];
    }
  }
}

// Kernel A (viscous equations) = the element-local "volume" work: gradient, published
// viscous normal-flux traces, and the internal-flux part of the divergence
// R_int = M13 M19 P2 F~ (convective + viscous, l.305-311, l.2919-2925) -> b.Rv
// [N_sol][N_V][Kp]; kernel B adds the face part M14 D~.
// Phases after the gradient: [publish g + F_v(d=0)] [div(0) + F_v(1)] [div(1) + F_v(2)]
// [div(2)], with the internal-flux buffer double-buffered so each phase has work for
// every thread.
// Kernel A body for the tile starting at element e0 (kt_grad: one tile per CTA; kt_fused:
// the A jobs of the persistent schedule).  bar: the CTA's TMA mbarrier, already
// initialised when init == false; par: the phase parity this use waits for.
// PERS (kt_grad_p): the tile's TMA, neighbour indices and neighbour traces (gnp) were
// requested by the caller / the previous tile; this tile requests those of tile e0n
// (-1: none) into sNbN during its last divergence phase
template <int D, int P, int EQ, int E, int NT, int NI, bool OSF, bool PERS = false>
__device__ __forceinline__ void grad_tile(const TensorGeom& g, const Line1D& L, const PhysDev& ph, const TensorBufs& b,
                                          const TileMaps& tm, int64_t e0, int (*sNb)[E], uint64_t* barp, bool init,
                                          unsigned par, GradNb<D, P, EQ, E, NT, NI>* gnp = nullptr, int64_t e0n = -1,
                                          int (*sNbN)[E] = nullptr) {
  PH_INIT
  using Ph = Phys<EQ, D>;
  using T = TDims<D, P>;
  constexpr int NV = Ph::NV, NL = T::NL, NS = T::NS;
  constexpr int NFB = NL * NI * NV * E;  // one internal-flux buffer
  constexpr bool DBUF = tensor_a_dbuf(D, NS, NL, NV, E, NI, OSF);
  // half-line items on a swizzled gradient tile (see SDRT_TA_QSWZ)
  constexpr bool QSWZ = SDRT_TA_QSWZ != 0 && SDRT_TA_GQ != 0 && OSF && SDRT_TA_SLINE == 2 && NV > 1 && NI < T::n &&
                        D == 3 && T::n == 4 && (NV & 1) == 1 && E == 8 && SDRT_TA_GPAIR != 1;
  extern __shared__ __align__(128) double smem[];
  double* sU = smem;
  double* sQ = smem + NS * NV * E;
  double* sF = sQ + D * NS * NV * E;  // 2 x [NL][P][NV][E]
  // OSF: [D][NL][NV][E], the right neighbours' traces, then sface F at the x_d = +1 ends
  double* sP = sF + (DBUF ? 2 : 1) * NFB;
  if constexpr (PERS) {
    static_assert(OSF && !DBUF && Ph::NV > 1, "persistent kernel A: the one-sided publication path");
    mbar_wait(barp, par);
    __syncthreads();
  PH(0, 1)
    if constexpr (QSWZ) gnp->template compute<true>(g, L, ph, sU, sQ, e0, sP);
    else gnp->compute(g, L, ph, sU, sQ, e0, sP);
  } else {
  if (threadIdx.x == 0) {  // the stage-input tile by TMA
    if (init) {
      mbar_init(barp, 1);
      mbar_fence_init();
    }
    mbar_expect_tx(barp, NS * NV * E * 8);
    tma_tile<NS * NV, E>(sU, &tm.uin, e0, barp);
  }
  fill_nbrs<D, E>(g, sNb, e0);
  __syncthreads();
  PH(0, 0)
  {
    constexpr bool GPAIR = SDRT_TA_GPAIR == 1 || (SDRT_TA_GPAIR == 2 && Ph::NV == 1);
    std::conditional_t<GPAIR, GradNb2<D, P, EQ, E, NT, NI>, GradNb<D, P, EQ, E, NT, NI>> gn;
    gn.load(g, ph, b.Tu, sNb, e0);
    mbar_wait(barp, par);
    __syncthreads();
  PH(0, 1)
    if constexpr (QSWZ) gn.template compute<true>(g, L, ph, sU, sQ, e0, OSF ? sP : nullptr);
    else gn.compute(g, L, ph, sU, sQ, e0, OSF ? sP : nullptr);
  }
  }
  __syncthreads();
  PH(0, 2)
  // publish on the sides that carry LDG weight: side 1 (left) if 1/2 + beta != 0,
  // side 0 (right) if 1/2 - beta != 0
  const bool pub1 = (0.5 + ph.beta) != 0.0, pub0 = (0.5 - ph.beta) != 0.0;
  const int nsides = (pub0 ? 1 : 0) + (pub1 ? 1 : 0);
  const int npub = nsides * NL * E;  // published ends per direction (in that direction's phase)
  constexpr int NFI = NL * NI * E;   // internal-flux items per direction
  constexpr int NDI = NL * NV * E;  // divergence items per direction
#pragma unroll 1
  for (int ph_ = 0; ph_ <= D; ++ph_) {
    // phase ph_: fluxes of direction ph_ (buffer ph_&1) [+ publish g in phase 0], then
    // the divergence of direction ph_-1 (buffer (ph_-1)&1) whose partial sums were
    // requested from L2 before the flux work
    const int dd = ph_ - 1;
    // LINE mode with fewer line items than threads (NL E < NT): threads 0 .. NL E - 1
    // run one line item each, the others all divergence items (so the heavy line work
    // never holds the divergence prefetch registers)
    constexpr bool LINE = (NV > 1 ? SDRT_TA_LINE_SYS : SDRT_TA_LINE) != 0 && SDRT_TA_DMMA == 0;
    constexpr int LG = NV > 1 ? SDRT_TA_LGRP_SYS : SDRT_TA_LGRP;   // outputs per pass
    constexpr bool LSP = NV > 1 && SDRT_TA_LSPLIT_SYS != 0;          // one item per pass
    constexpr int NGRP = LSP ? (NI + 2 + LG - 1) / LG : 1;
    constexpr int NLI = NL * E * NGRP;  // line items per direction
    constexpr bool LSPLIT = LINE && NLI < NT;
    constexpr int NDT = LSPLIT ? NT - NLI : NT;  // threads running divergence items
    constexpr int CD = (NDI + NDT - 1) / NDT;
    const bool divthr = !LSPLIT || (int)threadIdx.x >= NLI;
    const int dtid = LSPLIT ? (int)threadIdx.x - NLI : (int)threadIdx.x;
    // partial sums of R_int requested before the flux work (not in LSPLIT mode: there
    // the divergence threads do no flux work, and the prefetch registers would be live
    // across the line items in the register allocation)
    constexpr bool DRED = SDRT_TA_DRED == 2 || (SDRT_TA_DRED == 1 && OSF);  // 2: every kernel-A path
    double prev[(LSPLIT || DRED) ? 1 : CD][(LSPLIT || DRED) ? 1 : P + 1];
    if (!LSPLIT && !DRED && ph_ >= 2 && divthr) {
#pragma unroll
      for (int k = 0; k < CD; ++k) {
        const int item = dtid + k * NDT;
        const int el = item % E, r = item / E, v = r % NV, t = r / NV;
        if (item < NDI && e0 + el < g.K) {
          const int lb = lbase<D, P>(dd, t), ls = lstr<D, P>(dd);
          const double* src = b.Rv + (int64_t)(lb * NV + v) * g.Kp + e0 + el;
#pragma unroll
          for (int i = 0; i <= P; ++i) prev[k][i] = src[(int64_t)i * ls * NV * g.Kp];
        }
      }
    }
    constexpr bool LDMMA = SDRT_TA_DMMA != 0 && E == 8 && Ph::VISC && NV > 1;
    static_assert(!OSF || (!LDMMA && !LINE), "OSF runs on the per-point kernel-A items");
    constexpr bool SLINE = OSF && SDRT_TA_SLINE == 1 && NV > 1 && NI < T::n;
    constexpr bool HLINE = OSF && SDRT_TA_SLINE == 2 && NV > 1 && NI < T::n;  // publishes in its items
    const int nA = (ph_ < D && !LDMMA && !LINE && !HLINE) ? npub : 0;
    constexpr bool PAIR = SDRT_TA_PAIR == 1 || (SDRT_TA_PAIR == 2 && NV == 1);
    const int nB = (ph_ < D && !LDMMA && !LINE) ? (HLINE ? 2 * NL * E : SLINE ? NL * E : (PAIR ? NFI / 2 : NFI)) : 0;
    // divergence of direction ph_-1 from buffer (ph_-1)&1 (single buffer when two do
    // not fit two CTAs per SM: then it runs before this phase's fluxes overwrite it)
    constexpr bool PAIRB = SDRT_TA_PAIRB != 0 && HLINE && !PERS && !DBUF && NT == 256 && NL * E == 128;
    const int pair = (threadIdx.x >> 5) & 3;  // PAIRB: warps pair, pair + 4
    auto phase_sync = [&](bool cta) {
      if constexpr (PAIRB) {
        if (!cta) {
          asm volatile("bar.sync %0, 64;" ::"r"(1 + pair) : "memory");
          return;
        }
      }
      __syncthreads();
    };
    auto divergence = [&]() {
      const double* f0 = sF + (DBUF ? (dd & 1) * NFB : 0);
      if (!divthr) return;
#pragma unroll
      for (int k = 0; k < CD; ++k) {
        int item = dtid + k * NDT;
        int el = item % E, r = item / E, v = r % NV, t = r / NV;
        if constexpr (PAIRB) {  // the pair's own four lines: 4 NV E items over its 64 threads
          const int j = ((int)(threadIdx.x >> 7) * 32 + (int)(threadIdx.x & 31)) + k * 64;
          el = j % E, v = (j / E) % NV, t = 4 * pair + j / (E * NV);
          item = j < 4 * NV * E ? 0 : NDI;
        }
        if (item >= NDI || e0 + el >= g.K) continue;
        const int lb = lbase<D, P>(dd, t), ls = lstr<D, P>(dd);
        double f[NI];
#pragma unroll
        for (int a = 0; a < NI; ++a) f[a] = f0[((t * NI + a) * NV + v) * E + el];
        double fp = 0.0;  // OSF: the x_d = +1 face term (M14) joins R_int
        if constexpr (OSF) fp = sP[((dd * NL + t) * NV + v) * E + el];
        double* dst = b.Rv + (int64_t)(lb * NV + v) * g.Kp + e0 + el;
#pragma unroll
        for (int i = 0; i <= P; ++i) {
          double acc = 0.0;
          if constexpr (DRED) {
          } else if constexpr (LSPLIT) {
            if (ph_ >= 2) acc = dst[(int64_t)i * ls * NV * g.Kp];
          } else if (ph_ >= 2) {
            acc = prev[k][i];
          }
#pragma unroll
          for (int a = 0; a < NI; ++a) acc = fma(L.Dfl[i][a + 1], f[a], acc);
          if constexpr (OSF) acc = fma(L.Dfl[i][NI + 1], fp, acc);
          if constexpr (DRED) {
            if (ph_ >= 2) {
              asm volatile("red.global.add.f64 [%0], %1;" ::"l"(dst + (int64_t)i * ls * NV * g.Kp), "d"(acc) : "memory");
              continue;
            }
          }
          dst[(int64_t)i * ls * NV * g.Kp] = acc;
        }
      }
    };
    if constexpr (PERS) {
      // last phase: the state and gradient tiles are dead (every thread fenced its reads
      // against the async proxy before the barrier that ended phase D - 1)
      if (ph_ == D && e0n >= 0) {
        if (threadIdx.x == 0) {
          mbar_expect_tx(barp, NS * NV * E * 8);
          tma_tile<NS * NV, E>(sU, &tm.uin, e0n, barp);
        }
        fill_nbrs<D, E>(g, sNbN, e0n);
        __syncthreads();
        gnp->load(g, ph, b.Tu, sNbN, e0n);
      }
    }
    if constexpr (!DBUF) {
      if (ph_ >= 1) divergence();
      phase_sync(false);
    }
    if constexpr (LDMMA) {
      if (ph_ < D) {
        double* f1 = sF + (DBUF ? (ph_ & 1) * NFB : 0);
        const int warp = threadIdx.x >> 5, nw = NT >> 5;
        for (int t = warp; t < NL; t += nw) {
          if (ph_ == 0) visc_line_dmma<D, P, EQ, E, 0, NI>(g, L, ph, sU, sQ, f1, b.Tg, e0, t, pub0, pub1);
          else if (ph_ == 1) visc_line_dmma<D, P, EQ, E, 1, NI>(g, L, ph, sU, sQ, f1, b.Tg, e0, t, pub0, pub1);
          else if constexpr (D == 3) visc_line_dmma<D, P, EQ, E, 2, NI>(g, L, ph, sU, sQ, f1, b.Tg, e0, t, pub0, pub1);
        }
      }
    }
    if constexpr (LINE) {
      const int pubm = (pub0 ? 1 : 0) | (pub1 ? 2 : 0);
      // items: (line, element[, pass]); LSP: one item per pass of LG outputs (more
      // items, each loading the line once) instead of one per line
      auto line_d = [&](auto dc, int t, int el, double* f1, int gs) {
        constexpr int d = decltype(dc)::value;
        switch (pubm) {  // block-uniform: one instantiation per published-side set
          case 2: visc_line<D, P, EQ, E, d, NI, 2, LG, LSP>(g, L, ph, sU, sQ, f1, b.Tg, e0, t, el, gs); break;
          case 1: visc_line<D, P, EQ, E, d, NI, 1, LG, LSP>(g, L, ph, sU, sQ, f1, b.Tg, e0, t, el, gs); break;
          default: visc_line<D, P, EQ, E, d, NI, 3, LG, LSP>(g, L, ph, sU, sQ, f1, b.Tg, e0, t, el, gs); break;
        }
      };
      for (int it = threadIdx.x; it < (ph_ < D ? NLI : 0); it += LSPLIT ? NLI : NT) {
        const int el = it % E, t = (it / E) % NL, gs = it / (E * NL);
        double* f1 = sF + (DBUF ? (ph_ & 1) * NFB : 0);
        if (ph_ == 0) line_d(std::integral_constant<int, 0>{}, t, el, f1, gs);
        else if (ph_ == 1) line_d(std::integral_constant<int, 1>{}, t, el, f1, gs);
        else if constexpr (D == 3) line_d(std::integral_constant<int, 2>{}, t, el, f1, gs);
      }
    }
    for (int item = threadIdx.x; item < nA + nB; item += blockDim.x) {
      if (item < nA) {  // published ends of direction ph_
        const int el = item % E, r = item / E;
        const int t = r % NL, k = r / NL;
        const int side = (nsides == 2) ? k : (pub1 ? 1 : 0);
        if constexpr (OSF) {
          double* p1 = sP + ph_ * NL * NV * E;
          if (ph_ == 0) publish_F<D, P, EQ, E, 0>(g, L, ph, sU, sQ, b, p1, e0, t, el);
          else if (ph_ == 1) publish_F<D, P, EQ, E, 1>(g, L, ph, sU, sQ, b, p1, e0, t, el);
          else if constexpr (D == 3) publish_F<D, P, EQ, E, 2>(g, L, ph, sU, sQ, b, p1, e0, t, el);
        } else {
          if (ph_ == 0) publish_g<D, P, EQ, E, 0>(g, L, ph, sU, sQ, b.Tg, e0, side, t, el);
          else if (ph_ == 1) publish_g<D, P, EQ, E, 1>(g, L, ph, sU, sQ, b.Tg, e0, side, t, el);
          else if constexpr (D == 3) publish_g<D, P, EQ, E, 2>(g, L, ph, sU, sQ, b.Tg, e0, side, t, el);
        }
      } else if constexpr (HLINE) {
        // items 0 .. 2 NL E - 1 (no separate publish items): half h = first / second half of
        // each line, warp-uniform (NL E is a multiple of 32)
        int el = item % E, t = (item / E) % NL, h = item / (NL * E);
        if constexpr (SDRT_TA_HMAP != 0 && NL * E == 128 && NT == 256) {
          // warps w and w + 4 (one scheduler) run the same half: h = bit 1 of the warp index
          const int w = item >> 5, lane = item & 31;
          h = (w >> 1) & 1;
          t = 4 * ((w & 1) + 2 * (w >> 2)) + (lane >> 3);
          el = lane & 7;
        }
        double* f1 = sF + (DBUF ? (ph_ & 1) * NFB : 0);
        auto run = [&](auto dc) {
          constexpr int d = decltype(dc)::value;
          if (h == 0) visc_hline<D, P, EQ, E, d, NI, 0, QSWZ>(g, L, ph, sU, sQ, f1, b, sP, e0, t, el);
          else visc_hline<D, P, EQ, E, d, NI, 1, QSWZ>(g, L, ph, sU, sQ, f1, b, sP, e0, t, el);
        };
        if (ph_ == 0) run(std::integral_constant<int, 0>{});
        else if (ph_ == 1) run(std::integral_constant<int, 1>{});
        else if constexpr (D == 3) run(std::integral_constant<int, 2>{});
      } else if constexpr (SLINE) {
        const int i2 = item - nA, el = i2 % E, t = i2 / E;
        double* f1 = sF + (DBUF ? (ph_ & 1) * NFB : 0);
        if (ph_ == 0) visc_sline<D, P, EQ, E, 0, NI>(g, L, ph, sU, sQ, f1, t, el);
        else if (ph_ == 1) visc_sline<D, P, EQ, E, 1, NI>(g, L, ph, sU, sQ, f1, t, el);
        else if constexpr (D == 3) visc_sline<D, P, EQ, E, 2, NI>(g, L, ph, sU, sQ, f1, t, el);
      } else if constexpr (PAIR) {
        constexpr int E2 = E / 2;
        const int i2 = item - nA, el = 2 * (i2 % E2), r = i2 / E2, a = r % NI, t = r / NI;
        double* f1 = sF + (DBUF ? (ph_ & 1) * NFB : 0);
        if (ph_ == 0) visc_internal2<D, P, EQ, E, 0, NI>(g, L, ph, sU, sQ, f1, t, a, el);
        else if (ph_ == 1) visc_internal2<D, P, EQ, E, 1, NI>(g, L, ph, sU, sQ, f1, t, a, el);
        else if constexpr (D == 3) visc_internal2<D, P, EQ, E, 2, NI>(g, L, ph, sU, sQ, f1, t, a, el);
      } else if constexpr (SDRT_TA_AUNI != 0 && NI <= 4) {
        // items (a, t, el), a slowest: a is warp-uniform (NL E is a multiple of 32), so the
        // branches give each internal point its own compile-time coefficient set
        const int i2 = item - nA, el = i2 % E, r = i2 / E, t = r % NL, a = r / NL;
        double* f1 = sF + (DBUF ? (ph_ & 1) * NFB : 0);
        auto run = [&](auto dc, auto ac) {
          constexpr int d = decltype(dc)::value, A = decltype(ac)::value;
          if constexpr (A < NI) visc_internal<D, P, EQ, E, d, NI, A>(g, L, ph, sU, sQ, f1, t, A, el);
        };
        auto by_a = [&](auto dc) {
          if (a == 0) run(dc, std::integral_constant<int, 0>{});
          else if (a == 1) run(dc, std::integral_constant<int, 1>{});
          else if (a == 2) run(dc, std::integral_constant<int, 2>{});
          else run(dc, std::integral_constant<int, 3>{});
        };
        if (ph_ == 0) by_a(std::integral_constant<int, 0>{});
        else if (ph_ == 1) by_a(std::integral_constant<int, 1>{});
        else if constexpr (D == 3) by_a(std::integral_constant<int, 2>{});
      } else {
        const int i2 = item - nA, el = i2 % E, r = i2 / E, a = r % NI, t = r / NI;
        double* f1 = sF + (DBUF ? (ph_ & 1) * NFB : 0);
        if (ph_ == 0) visc_internal<D, P, EQ, E, 0, NI>(g, L, ph, sU, sQ, f1, t, a, el);
        else if (ph_ == 1) visc_internal<D, P, EQ, E, 1, NI>(g, L, ph, sU, sQ, f1, t, a, el);
        else if constexpr (D == 3) visc_internal<D, P, EQ, E, 2, NI>(g, L, ph, sU, sQ, f1, t, a, el);
      }
    }
    if constexpr (DBUF) {
      if (ph_ >= 1) divergence();
    }
    if constexpr (PERS) {
      if (ph_ == D - 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    phase_sync(ph_ == D - 1);
  PH(0, 3 + ph_)
  }
}

template <int D, int P, int EQ, int E, int NT, int MINB, int NI, bool OSF = false>
__global__ void __launch_bounds__(NT, MINB) kt_grad(TensorGeom g, Line1D L, PhysDev ph, TensorBufs b,
                                                    const __grid_constant__ TileMaps tm) {
  pdl_wait();
  __shared__ int sNb[2 * D][E];
  __shared__ __align__(8) uint64_t bar;
  const int64_t e0 = (int64_t)(g.tiles ? g.tiles[blockIdx.x] : (int)blockIdx.x) * E;
  grad_tile<D, P, EQ, E, NT, NI, OSF>(g, L, ph, b, tm, e0, sNb, &bar, true, 0);
}

// Persistent one-sided-publication kernel A (SDRT_TA_PERSIST): see the macro's comment
template <int D, int P, int EQ, int E, int NT, int MINB, int NI>
__global__ void __launch_bounds__(NT, MINB) kt_grad_p(TensorGeom g, Line1D L, PhysDev ph, TensorBufs b,
                                                      const __grid_constant__ TileMaps tm, int ntiles) {
  pdl_wait();
  using T = TDims<D, P>;
  constexpr int NV = Phys<EQ, D>::NV;
  __shared__ int sNb[2][2 * D][E];
  __shared__ __align__(8) uint64_t bar;
  extern __shared__ __align__(128) double smem[];
  auto tile_e0 = [&](int t) { return (int64_t)(g.tiles ? g.tiles[t] : t) * E; };
  int tile = blockIdx.x;
  if (tile >= ntiles) return;
  int64_t e0 = tile_e0(tile);
  GradNb<D, P, EQ, E, NT, NI> gn;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
    mbar_expect_tx(&bar, T::NS * NV * E * 8);
    tma_tile<T::NS * NV, E>(smem, &tm.uin, e0, &bar);
  }
  fill_nbrs<D, E>(g, sNb[0], e0);
  __syncthreads();
  gn.load(g, ph, b.Tu, sNb[0], e0);
  unsigned par = 0;
  int buf = 0;
#pragma unroll 1
  for (; tile < ntiles; tile += gridDim.x) {
    const int next = tile + (int)gridDim.x;
    const int64_t e0n = next < ntiles ? tile_e0(next) : -1;
    grad_tile<D, P, EQ, E, NT, NI, true, true>(g, L, ph, b, tm, e0, sNb[buf], &bar, false, par, &gn, e0n, sNb[buf ^ 1]);
    par ^= 1u;
    buf ^= 1;
    e0 = e0n;
  }
}

// Kernel B: common fluxes at the line ends (Rusanov / upwind + the published viscous
// traces + LDG jump, l.312-340), the face part of the divergence M14 D~ (l.2919-2925),
// [inviscid equations: also the internal fluxes and M13 F~, which kernel A does
// otherwise], R~ = sum + R_int, -R~/detJ, RK4 update, new traces.
template <int D, int P, int EQ, int E, int NT, int MINB, int NI, bool FEXP = false>
__global__ void __launch_bounds__(NT, MINB) kt_stage(TensorGeom g, Line1D L, PhysDev ph, TensorBufs b, int stage,
                                                   double dt, const __grid_constant__ TileMaps tm) {
  pdl_wait();
  PH_INIT
  using Ph = Phys<EQ, D>;
  using T = TDims<D, P>;
  constexpr int NV = Ph::NV, n = T::n, NL = T::NL, NS = T::NS;
  constexpr bool INT = !Ph::VISC;     // internal fluxes evaluated here (inviscid only)
  constexpr int NF = INT ? NI + 2 : 2;  // flux-line slots per line held in sF
  extern __shared__ __align__(128) double smem[];
  // regions allocated per stage (the launcher sizes dynamic smem the same way):
  // sU, sR, sF always; u_n for stages 1, 2; ACC for stages 1..3
  double* sU = smem;
  double* sR = smem + NS * NV * E;    // R~ accumulator, starts as R_int (kernel A)
  double* sF = sR + NS * NV * E;      // [NL][NF][NV][E] flux-line values of one direction
  double* sAcc = sF + NL * NF * NV * E;                             // RK accumulator / RK54 dU
  double* sUn = sAcc + (stage_reads_acc(stage) ? NS * NV * E : 0);  // RK register u_n (RK4 stages 1, 2)
  __shared__ int sNb[2 * D][E];
  __shared__ __align__(8) uint64_t bar[2];
  const int bx = SDRT_TB_REV == 2 ? (int)(gridDim.x - 1 - blockIdx.x) : (int)blockIdx.x;
  const int64_t e0 = (int64_t)(g.tiles ? g.tiles[bx] : bx) * E;
  // every element-local input of the tile is requested up front by TMA: the stage
  // input (barrier 0), then R_int and the RK registers (barrier 1), waited for only
  // where they are used
  constexpr unsigned TB = NS * NV * E * 8;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
    mbar_expect_tx(&bar[0], TB);
    tma_tile<NS * NV, E>(sU, &tm.uin, e0, &bar[0]);
    const unsigned later = (Ph::VISC ? TB : 0) + (stage_reads_un(stage) ? TB : 0) + (stage_reads_acc(stage) ? TB : 0);
    mbar_expect_tx(&bar[1], later);
    if constexpr (Ph::VISC) tma_tile<NS * NV, E>(sR, &tm.rv, e0, &bar[1]);
    if (stage_reads_un(stage)) tma_tile<NS * NV, E>(sUn, &tm.un, e0, &bar[1]);
    if (stage_reads_acc(stage)) tma_tile<NS * NV, E>(sAcc, &tm.acc, e0, &bar[1]);
  }
  fill_nbrs<D, E>(g, sNb, e0);
  __syncthreads();
  PH(1, 0)
  const double wl = 0.5 + ph.beta, wr = 0.5 - ph.beta;
  const int Kt = (int)g.Kt;  // trace row stride
  // one direction of the flux-line work; instantiated per direction (compile-time d
  // removes the structural zeros of the normal e_d from the physics)
  // End items (t, side, el) of every direction are statically owned (item tid + k NT):
  // the traces they need (neighbour U trace, published viscous traces) for direction
  // d+1 are requested while direction d finishes, and for d = 0 before the tile wait,
  // so their latency overlaps other work.  Raw values only; combined at use.
  constexpr int NEI = 2 * NL * E, CE = (NEI + NT - 1) / NT;
  double un[CE][NV], tga[CE][NV], tgb[CE][NV];
  auto load_dir = [&](auto dc) {
    constexpr int d = decltype(dc)::value;
#pragma unroll
    for (int k = 0; k < CE; ++k) {
      const int item = threadIdx.x + k * NT;
      const int el = item % E, r = item / E, side = r % 2, t = r / 2;
      const int64_t e = e0 + el;
      if (item >= NEI) break;
      const int m = sNb[2 * d + side][el];
      // canonical (left, right) = (x_d- element, x_d+ element)
      const int xL = (2 * d + 1) * NL + t, xR = (2 * d) * NL + t;  // left's +face, right's -face
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        un[k][v] = b.Tu[((side ? xR : xL) * NV + v) * Kt + m];
        if constexpr (Ph::VISC) {
          // predicated loads into zeroed registers: nothing consumes them here
          const int eL = side ? (int)e : m, eR = side ? m : (int)e;
          tga[k][v] = 0.0;
          tgb[k][v] = 0.0;
          if (wl != 0.0) tga[k][v] = b.Tg[(xL * NV + v) * Kt + eL];
          if (wr != 0.0) tgb[k][v] = b.Tg[(xR * NV + v) * Kt + eR];
        }
      }
    }
  };
  auto direction = [&](auto dc) {
    constexpr int d = decltype(dc)::value;
    const double wf = g.detJ * g.jinv[d];  // transformed-flux weight detJ (J^-1)_dd
    const double sface = g.sface[d];
    for (int item = threadIdx.x; item < (INT ? NL * NI * E : 0); item += blockDim.x) {
      const int el = item % E, r = item / E, a = r % NI, t = r / NI;
      const int lb = lbase<D, P>(d, t), ls = lstr<D, P>(d);
      double ua[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        if constexpr (NI == n) {  // FR: solution points
          ua[v] = sU[((lb + a * ls) * NV + v) * E + el];
        } else {
          double s = 0.0;
#pragma unroll
          for (int i = 0; i < n; ++i) s = fma(L.Iint[a][i], sU[((lb + i * ls) * NV + v) * E + el], s);
          ua[v] = s;
        }
      }
      double f[NV];
      Ph::template conv_axis<d>(ph, ua, wf, f);
#pragma unroll
      for (int v = 0; v < NV; ++v) sF[((t * NF + a + 1) * NV + v) * E + el] = f[v];
    }
#pragma unroll
    for (int k = 0; k < CE; ++k) {
      const int item = threadIdx.x + k * NT;
      if (item >= NEI) break;
      const int el = item % E, r = item / E, side = r % 2, t = r / 2;
      const int lb = lbase<D, P>(d, t), ls = lstr<D, P>(d);
      double uo[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        double ul[n];
#pragma unroll
        for (int i = 0; i < n; ++i) ul[i] = sU[((lb + i * ls) * NV + v) * E + el];
        uo[v] = interp_end<n>(L.Iend[side], ul);
      }
      double uL[NV], uR[NV];  // by value (no runtime pointer select into register arrays)
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        uL[v] = side ? uo[v] : un[k][v];
        uR[v] = side ? un[k][v] : uo[v];
      }
      double F[NV];
      Ph::template conv_common_axis<d>(ph, uL, uR, F);
      if constexpr (Ph::VISC) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          double gsum = 0.0;
          if (wl != 0.0) gsum = __dmul_rn(wl, tga[k][v]);
          if (wr != 0.0) gsum = __fma_rn(wr, tgb[k][v], gsum);
          F[v] = Ph::ldg_rn(F[v], gsum, ph.eta, uL[v], uR[v]);
        }
      }
      const int kf = side ? NF - 1 : 0;
#pragma unroll
      for (int v = 0; v < NV; ++v) sF[((t * NF + kf) * NV + v) * E + el] = sface * F[v];
      if (FEXP && e0 + el < g.K) {  // O28 export (residual only): F at the own ext point (2d + side, t)
#pragma unroll
        for (int v = 0; v < NV; ++v) b.Fexp[((int64_t)((2 * d + side) * NL + t) * NV + v) * g.Kp + e0 + el] = F[v];
      }
    }
    if constexpr (d + 1 < D) load_dir(std::integral_constant<int, d + 1>{});
    if (d == 0) mbar_wait(&bar[1], 0);  // R_int and the RK registers have landed
    __syncthreads();
  PH(1, 2)
    // divergence along the lines: R_i += sum_k L_k'(g_i) Fline_k (M14 at the ends with
    // the sign of the outward normal folded into L_0', M13 inside when INT)
    for (int item = threadIdx.x; item < NL * NV * E; item += blockDim.x) {
      const int el = item % E, r = item / E, v = r % NV, t = r / NV;
      const int lb = lbase<D, P>(d, t), ls = lstr<D, P>(d);
      double f[NF];
#pragma unroll
      for (int k = 0; k < NF; ++k) f[k] = sF[((t * NF + k) * NV + v) * E + el];
#pragma unroll
      for (int i = 0; i < n; ++i) {
        double* dst = sR + ((lb + i * ls) * NV + v) * E + el;
        double acc = (d == 0 && INT) ? 0.0 : *dst;
        if constexpr (INT) {
#pragma unroll
          for (int k = 0; k < NF; ++k) acc = fma(L.Dfl[i][k], f[k], acc);
        } else {
          acc = fma(L.Dfl[i][0], f[0], acc);
          acc = fma(L.Dfl[i][NI + 1], f[1], acc);
        }
        *dst = acc;
      }
    }
    __syncthreads();
  PH(1, 3)
  };
  load_dir(std::integral_constant<int, 0>{});
  mbar_wait(&bar[0], 0);
  __syncthreads();
  PH(1, 1)
  direction(std::integral_constant<int, 0>{});
  direction(std::integral_constant<int, 1>{});
  if constexpr (D == 3) direction(std::integral_constant<int, 2>{});
  // dU/dt = -R~/detJ (R~ includes R_int), RK4 (3-register form) along x-lines: one item = (x-line,
  // variable, element) holds the line's new values in registers, writes them to sU and
  // the registers, and publishes the two x-face traces from the same registers.
  const double idet = 1.0 / g.detJ;
  for (int item = threadIdx.x; item < NL * NV * E; item += NT) {
    const int el = item % E, r = item / E, v = r % NV, t = r / NV;
    const int64_t e = e0 + el;
    if (e >= g.K) continue;
    const int p0 = n * t;  // x-line t: points n t .. n t + n - 1
    double un[n];
#pragma unroll
    for (int i = 0; i < n; ++i) {
      const int idx = ((p0 + i) * NV + v) * E + el;
      const int64_t gi = (int64_t)((p0 + i) * NV + v) * g.Kp + e;
      const double kk = -sR[idx] * idet;
      double nu;
      switch (stage) {
        case -1:
          b.out[gi] = kk;
          nu = 0.0;
          break;
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
      un[i] = nu;
      sU[idx] = nu;
    }
    if (stage >= 0) {
      b.Tu_next[((int64_t)(0 * NL + t) * NV + v) * g.Kt + e] = interp_end<n>(L.Iend[0], un);
      b.Tu_next[((int64_t)(1 * NL + t) * NV + v) * g.Kt + e] = interp_end<n>(L.Iend[1], un);
    }
  }
  if (stage < 0) return;
  __syncthreads();
  PH(1, 4)
  // traces of the new state on the faces normal to y (and z): both ends per item
  for (int item = threadIdx.x; item < (D - 1) * NL * NV * E; item += blockDim.x) {
    const int el = item % E, r = item / E, v = r % NV, r2 = r / NV, t = r2 % NL, d = 1 + r2 / NL;
    const int64_t e = e0 + el;
    if (e >= g.K) continue;
    const int lb = lbase<D, P>(d, t), ls = lstr<D, P>(d);
    double u[n];
#pragma unroll
    for (int i = 0; i < n; ++i) u[i] = sU[((lb + i * ls) * NV + v) * E + el];
    b.Tu_next[((int64_t)((2 * d) * NL + t) * NV + v) * g.Kt + e] = interp_end<n>(L.Iend[0], u);
    b.Tu_next[((int64_t)((2 * d + 1) * NL + t) * NV + v) * g.Kt + e] = interp_end<n>(L.Iend[1], u);
  }
  PH(1, 15)
}

// Kernel B with one-sided flux publication (OSF, see publish_F): R_int already holds the
// internal fluxes and the x_d = +1 faces (kernel A), so per tile this kernel gathers
// the left neighbours' published F of its D x_d = -1 faces, completes
// R~ = R_int + sum_d M14_(d,-) D~ in the RK update (l.2919-2925, l.347-350), and publishes
// the x_d = -1 traces of the new state (the only traces kernel A reads with beta = 1/2).
// The stage input is not read except where the RK formula needs it (RK4 stage 0, RK54).
// Kernel B (OSF) body for the tile starting at element e0 (kt_stage_osf: one tile per
// CTA; kt_fused: the B jobs of the persistent schedule); bar / init / par as grad_tile.
template <int D, int P, int EQ, int E, int NT, bool FEXP>
__device__ __forceinline__ void stage_osf_tile(const TensorGeom& g, const Line1D& L, const PhysDev& ph,
                                               const TensorBufs& b, int stage, double dt, const TileMaps& tm,
                                               int64_t e0, int (*sNb)[E], uint64_t* barp, bool init, unsigned par) {
  using Ph = Phys<EQ, D>;
  using T = TDims<D, P>;
  constexpr int NV = Ph::NV, n = T::n, NL = T::NL, NS = T::NS;
  extern __shared__ __align__(128) double smem[];
  const bool need_in = stage == 0 || stage >= RK54_STAGE0;
  // SDRT_TB_DIRECT: R_int and u_n are read straight from global memory in the update (one
  // read per value, coalesced rows of E elements) instead of being staged by TMA, so the
  // CTA needs 55 KB of shared memory instead of 95 KB (3 CTAs per SM in every stage)
  constexpr bool DIRECT = SDRT_TB_DIRECT != 0;
  double* sR = smem;                                  // R_int (kernel A); unused if DIRECT
  double* sF = sR + (DIRECT ? 0 : NS * NV * E);       // [D][NL][NV][E] left neighbours' F (x_d = -1 faces)
  double* sU = sF + D * NL * NV * E;    // new state (stage input first where the RK formula reads it)
  double* sAcc = sU + NS * NV * E;
  double* sUn = sAcc + (stage_reads_acc(stage) ? NS * NV * E : 0);
  constexpr unsigned TB = NS * NV * E * 8;
  uint64_t& bar = *barp;
  if (threadIdx.x == 0) {
    if (init) {
      mbar_init(&bar, 1);
      mbar_fence_init();
    }
    const unsigned bytes = TB * ((DIRECT ? 0 : 1) + (need_in ? 1 : 0) + (!DIRECT && stage_reads_un(stage) ? 1 : 0) +
                                 (stage_reads_acc(stage) ? 1 : 0));
    mbar_expect_tx(&bar, bytes);
    constexpr bool EF = SDRT_TB_EF != 0;  // read-once streams: L2 evict-first
    if (!DIRECT) tma_tile<NS * NV, E, EF>(sR, &tm.rv, e0, &bar);
    if (need_in) tma_tile<NS * NV, E>(sU, &tm.uin, e0, &bar);
    if (!DIRECT && stage_reads_un(stage)) tma_tile<NS * NV, E, (SDRT_TB_EF > 1)>(sUn, &tm.un, e0, &bar);
    if (stage_reads_acc(stage)) tma_tile<NS * NV, E, (SDRT_TB_EF > 1)>(sAcc, &tm.acc, e0, &bar);
  }
  fill_nbrs<D, E>(g, sNb, e0);
  __syncthreads();
  // gather F of the x_d = -1 faces: the left neighbour's x_d = +1 ext point, 8-byte
  // cp.async straight into shared memory (element fastest: runs of consecutive columns)
  for (int item = threadIdx.x; item < D * NL * NV * E; item += NT) {
    const int el = item % E, r = item / E, v = r % NV, r2 = r / NV, t = r2 % NL, d = r2 / NL;
    const int64_t m = e0 + el < g.K ? sNb[2 * d][el] : 0;
    const double* src = b.Tg + ((int64_t)((2 * d + 1) * NL + t) * NV + v) * g.Kt + m;
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sF + item);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(src));
  }
  asm volatile("cp.async.commit_group;");
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  mbar_wait(&bar, par);
  __syncthreads();
  if constexpr (FEXP) {  // O28 export (residual only): F at the own x_d = -1 ext points
    for (int item = threadIdx.x; item < D * NL * NV * E; item += NT) {
      const int el = item % E, r = item / E, v = r % NV, r2 = r / NV, t = r2 % NL, d = r2 / NL;
      if (e0 + el < g.K) b.Fexp[((int64_t)((2 * d) * NL + t) * NV + v) * g.Kp + e0 + el] = sF[item];
    }
  }
  // R~ = R_int + the x_d = -1 face terms (sface_d Dfl[.][0] F), dU/dt = -R~/detJ, RK update
  // along x-lines (item = x-line t, variable, element); x = -1 trace from registers
  const double idet = 1.0 / g.detJ;
  for (int item = threadIdx.x; item < NL * NV * E; item += NT) {
    const int el = item % E, r = item / E, v = r % NV, t = r / NV;
    const int64_t e = e0 + el;
    if (e >= g.K) continue;
    const int j = t % n, k = D == 3 ? t / n : 0;  // y (and z) position of x-line t
    auto F = [&](int d, int tl) { return sF[((d * NL + tl) * NV + v) * E + el]; };
    const double fx = g.sface[0] * F(0, t);
    // y-line through (i, j[, k]): index i + n k, position j; z-line: index i + n j, position k
    double cy = 0.0, cz = 0.0;
#pragma unroll
    for (int q = 0; q < n; ++q) {
      if (q == j) cy = L.Dfl[q][0] * g.sface[1];
      if (D == 3 && q == k) cz = L.Dfl[q][0] * g.sface[2];
    }
    const int p0 = n * t;
    double un[n];
#pragma unroll
    for (int i = 0; i < n; ++i) {
      const int idx = ((p0 + i) * NV + v) * E + el;
      const int64_t gi = (int64_t)((p0 + i) * NV + v) * g.Kp + e;
      double R = fma(L.Dfl[i][0], fx, DIRECT ? b.Rv[gi] : sR[idx]);
      R = fma(cy, F(1, D == 3 ? i + n * k : i), R);
      if constexpr (D == 3) R = fma(cz, F(2, i + n * j), R);
      const double kk = -R * idet;
      double nu;
      switch (stage) {
        case -1:
          b.out[gi] = kk;
          nu = 0.0;
          break;
        case 0: {
          const double u0 = sU[idx];
          b.ACC[gi] = fma(dt / 6.0, kk, u0);
          nu = fma(0.5 * dt, kk, u0);
          b.Us[gi] = nu;
        } break;
        case 1:
          b.ACC[gi] = fma(dt / 3.0, kk, sAcc[idx]);
          nu = fma(0.5 * dt, kk, DIRECT ? b.U[gi] : sUn[idx]);
          b.Us[gi] = nu;
          break;
        case 2:
          b.ACC[gi] = fma(dt / 3.0, kk, sAcc[idx]);
          nu = fma(dt, kk, DIRECT ? b.U[gi] : sUn[idx]);
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
      un[i] = nu;
      sU[idx] = nu;
    }
    if (stage >= 0) b.Tu_next[((int64_t)(0 * NL + t) * NV + v) * g.Kt + e] = interp_end<n>(L.Iend[0], un);
  }
  if (stage < 0) return;
  __syncthreads();
  // x_d = -1 traces of the new state on the faces normal to y (and z)
  for (int item = threadIdx.x; item < (D - 1) * NL * NV * E; item += NT) {
    const int el = item % E, r = item / E, v = r % NV, r2 = r / NV, t = r2 % NL, d = 1 + r2 / NL;
    const int64_t e = e0 + el;
    if (e >= g.K) continue;
    const int lb = lbase<D, P>(d, t), ls = lstr<D, P>(d);
    double u[n];
#pragma unroll
    for (int i = 0; i < n; ++i) u[i] = sU[((lb + i * ls) * NV + v) * E + el];
    b.Tu_next[((int64_t)((2 * d) * NL + t) * NV + v) * g.Kt + e] = interp_end<n>(L.Iend[0], u);
  }
}

template <int D, int P, int EQ, int E, int NT, int MINB, bool FEXP = false>
__global__ void __launch_bounds__(NT, MINB) kt_stage_osf(TensorGeom g, Line1D L, PhysDev ph, TensorBufs b, int stage,
                                                       double dt, const __grid_constant__ TileMaps tm) {
  pdl_wait();
  __shared__ int sNb[2 * D][E];
  __shared__ __align__(8) uint64_t bar;
  const int bx = SDRT_TB_REV != 0 ? (int)(gridDim.x - 1 - blockIdx.x) : (int)blockIdx.x;
  const int64_t e0 = (int64_t)(g.tiles ? g.tiles[bx] : bx) * E;
  stage_osf_tile<D, P, EQ, E, NT, FEXP>(g, L, ph, b, stage, dt, tm, e0, sNb, &bar, true, 0);
}

// Fused RK stage: kernel A and kernel B (OSF) of one stage as the jobs of ONE persistent
// launch (FuseSched, tensor.cuh).  A job = grad_tile on one tile, then a release of the
// tile's flag; B job = acquire the flags of the tiles it reads (its own R_int and the
// published common fluxes of its x_d = -1 neighbours), then stage_osf_tile.  Jobs are taken
// in list order from an atomic ticket, and every dependency of a B job is an A job earlier
// in the list, so a waiting CTA only waits for A jobs that running CTAs already hold (A
// jobs never wait): no deadlock whatever the number of resident CTAs.  Per element the
// arithmetic is exactly kernel A's and kernel B's, so the stage is bitwise the two-kernel
// one; R_int is read back a few hundred tiles after it was written (L2, not HBM), and the
// B jobs' HBM streams overlap the A jobs' shared-memory-bound work on the same SMs.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// SDRT_FUSE_NOINLINE: the two job bodies as separate (non-inlined) functions, each with its
// own register allocation (the inlined pair spills ~100 bytes at 128 registers)
#ifndef SDRT_FUSE_NOINLINE
#define SDRT_FUSE_NOINLINE 0
#endif
template <int D, int P, int EQ, int E, int NT, int NI>
__device__ __noinline__ void grad_job(const TensorGeom& g, const Line1D& L, const PhysDev& ph, const TensorBufs& b,
                                      const TileMaps& tm, int64_t e0, int (*sNb)[E], uint64_t* barp, unsigned par) {
  grad_tile<D, P, EQ, E, NT, NI, true>(g, L, ph, b, tm, e0, sNb, barp, false, par);
}
template <int D, int P, int EQ, int E, int NT>
__device__ __noinline__ void stage_job(const TensorGeom& g, const Line1D& L, const PhysDev& ph, const TensorBufs& b,
                                       int stage, double dt, const TileMaps& tm, int64_t e0, int (*sNb)[E],
                                       uint64_t* barp, unsigned par) {
  stage_osf_tile<D, P, EQ, E, NT, false>(g, L, ph, b, stage, dt, tm, e0, sNb, barp, false, par);
}

template <int D, int P, int EQ, int E, int NT, int MINB, int NI>
__global__ void __launch_bounds__(NT, MINB) kt_fused(TensorGeom g, Line1D L, PhysDev ph, TensorBufs b, int stage,
                                                     double dt, const __grid_constant__ TileMaps tm, FuseSched fs) {
  pdl_wait();
  __shared__ int sNb[2 * D][E];
  __shared__ __align__(8) uint64_t barA, barB;
  // loop state in shared memory (nothing held in registers across a job body: the A body
  // uses all 128)
  __shared__ int sJob;
  __shared__ unsigned sEpoch, sPar[2];
  if (threadIdx.x == 0) {
    mbar_init(&barA, 1);
    mbar_init(&barB, 1);
    mbar_fence_init();
    // this launch's epoch: one more than the last launch's (ctr[2] advances when the last
    // CTA of a launch exits, after every CTA has read it), so a CUDA-graph replay works too
    sEpoch = (unsigned)ld_acquire_u32((const unsigned*)fs.ctr + 2) + 1u;
    sPar[0] = sPar[1] = 0;
  }
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) sJob = atomicAdd(fs.ctr, 1);
    __syncthreads();
    if (sJob >= fs.njobs) break;
    const int code = fs.jobs[sJob];
    if ((code & 1) == 0) {
      grad_tile<D, P, EQ, E, NT, NI, true>(g, L, ph, b, tm, (int64_t)(code >> 1) * E, sNb, &barA, false, sPar[0]);
      // this thread's R_int / published-flux stores before the B job's TMA reads of them
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        st_release_u32(fs.flags + (fs.jobs[sJob] >> 1), sEpoch);
        sPar[0] ^= 1u;
      }
    } else {
      if (threadIdx.x == 0) {
        const int* dl = fs.deps + (int64_t)(code >> 1) * FUSE_DEPS;
        for (int k = 0; k < FUSE_DEPS; ++k) {
          const int t = dl[k];
          if (t < 0) break;
          while ((int)(ld_acquire_u32(fs.flags + t) - sEpoch) < 0) __nanosleep(100);
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      __syncthreads();
      stage_osf_tile<D, P, EQ, E, NT, false>(g, L, ph, b, stage, dt, tm, (int64_t)(code >> 1) * E, sNb, &barB, false,
                                             sPar[1]);
      __syncthreads();
      if (threadIdx.x == 0) sPar[1] ^= 1u;
    }
    // this job's shared-memory accesses before the next job's TMA writes into the buffers
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(fs.ctr + 1, 1) == (int)gridDim.x - 1) {  // last CTA: reset for the next launch
      fs.ctr[0] = 0;
      fs.ctr[1] = 0;
      __threadfence();
      atomicAdd(fs.ctr + 2, 1);
    }
  }
}

// TGV diagnostics (NEXT row N4): per tile the solution-point
// quadrature sums of E* = rho v.v, S^d : S^d and p div v, with grad v from the LDG
// gradient (GradNb) by the chain rule (reading O20).  part[3 tile + k] (fixed-order
// block reduction: deterministic).
template <int NT>
__device__ __forceinline__ void block_sum3(double (&a)[3], double* red, double* out) {
#pragma unroll
  for (int k = 0; k < 3; ++k) red[k * NT + threadIdx.x] = a[k];
  __syncthreads();
  for (int h = NT / 2; h > 0; h >>= 1) {
    if (threadIdx.x < h)
#pragma unroll
      for (int k = 0; k < 3; ++k) red[k * NT + threadIdx.x] += red[k * NT + threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < 3; ++k) out[k] = red[k * NT];
}

// Degree-10 cubature of one element (tensor, 3-D) applied sum-factorised through the 1D
// factor B1 [nq][n] of Bq = B1 (x) B1 (x) B1 (x fastest; refel.cpp cubature_interp_1d):
// per component c (u_v, then q[j][v]), Y1 = B1 along x, Y2 = B1 along y (shared memory),
// then every cubature point contracts along z and evaluates the integrands -- the same
// polynomial values as the dense Bq rows, 3 (nq n^3 + ...) instead of
// nq^3 n^3 multiply-adds per component.  Returns nothing; accumulates into acc.
template <int D, int P, int NV, int E, int NT, int G>
__device__ __forceinline__ void tgv_element_sf(const PhysDev& ph, const double* sU, const double* sQ,
                                               const double* sB1, int nq, const double* __restrict__ w,
                                               double detj, int el0, int ng, double* sY1, double* sY2,
                                               double (&acc)[3]) {
  // G element slots el0 .. el0 + ng - 1 at a time (element slot fastest in every item)
  constexpr int n = P + 1, NS = n * n * n, NC = NV + D * NV;
  auto X = [&](int c, int s, int el) {  // component c at solution point s of element el
    return c < NV ? sU[(s * NV + c) * E + el] : sQ[(((c - NV) / NV * NS + s) * NV + (c - NV) % NV) * E + el];
  };
  // Y1[c][rz][ry][qx][g] = sum_rx B1[qx][rx] X_c(rx, ry, rz)
  for (int it = threadIdx.x; it < NC * n * n * nq * G; it += NT) {
    const int gi = it % G, r0 = it / G, qx = r0 % nq, r = r0 / nq, ry = r % n, r2 = r / n, rz = r2 % n, c = r2 / n;
    if (gi >= ng) continue;
    double a = 0.0;
#pragma unroll
    for (int rx = 0; rx < n; ++rx) a = fma(sB1[qx * n + rx], X(c, rx + n * (ry + n * rz), el0 + gi), a);
    sY1[it] = a;
  }
  __syncthreads();
  // Y2[c][rz][qy][qx][g] = sum_ry B1[qy][ry] Y1[c][rz][ry][qx][g]
  for (int it = threadIdx.x; it < NC * n * nq * nq * G; it += NT) {
    const int gi = it % G, r0 = it / G, qx = r0 % nq, r = r0 / nq, qy = r % nq, r2 = r / nq, rz = r2 % n, c = r2 / n;
    if (gi >= ng) continue;
    double a = 0.0;
#pragma unroll
    for (int ry = 0; ry < n; ++ry) a = fma(sB1[qy * n + ry], sY1[(((c * n + rz) * n + ry) * nq + qx) * G + gi], a);
    sY2[it] = a;
  }
  __syncthreads();
  // every cubature point (qx, qy, qz) of every element: contract along z, then the integrands
  for (int it = threadIdx.x; it < nq * nq * nq * G; it += NT) {
    const int gi = it % G, q = it / G, qx = q % nq, qy = (q / nq) % nq, qz = q / (nq * nq);
    if (gi >= ng) continue;
    double v[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      double a = 0.0;
#pragma unroll
      for (int rz = 0; rz < n; ++rz) a = fma(sB1[qz * n + rz], sY2[((((c * n + rz) * nq + qy) * nq + qx)) * G + gi], a);
      v[c] = a;
    }
    tgv_point<D, NV>(ph, v, v + NV, __ldg(w + q) * detj, acc);
  }
}

template <int D, int P, int EQ, int E, int NT, int NI>
__global__ void __launch_bounds__(NT) kt_diag(TensorGeom g, Line1D L, PhysDev ph, TensorBufs b, const double* w,
                                              const double* Bq, int nq, double* part,
                                              const __grid_constant__ TileMaps tm, const double* B1, int nq1) {
  using Ph = Phys<EQ, D>;
  using T = TDims<D, P>;
  constexpr int NV = Ph::NV, NS = T::NS;
  extern __shared__ __align__(128) double smem[];
  double* sU = smem;
  double* sQ = smem + NS * NV * E;
  __shared__ double red[3 * NT];
  __shared__ int sNb[2 * D][E];
  __shared__ __align__(8) uint64_t bar;
  const int64_t e0 = (int64_t)blockIdx.x * E;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
    mbar_expect_tx(&bar, NS * NV * E * 8);
    tma_tile<NS * NV, E>(sU, &tm.uin, e0, &bar);
  }
  fill_nbrs<D, E>(g, sNb, e0);
  __syncthreads();
  {
    GradNb<D, P, EQ, E, NT, NI> gn;
    gn.load(g, ph, b.Tu, sNb, e0);
    mbar_wait(&bar, 0);
    __syncthreads();
    gn.compute(g, L, ph, sU, sQ, e0);
  }
  __syncthreads();
  double acc[3] = {0.0, 0.0, 0.0};
  if constexpr (NV == D + 2 && D == 3) {
    if (B1) {  // sum-factorised cubature, one element at a time
      __shared__ double sB1[64];
      for (int i = threadIdx.x; i < nq1 * (P + 1); i += NT) sB1[i] = B1[i];
      constexpr int G = P >= 4 ? 1 : SDRT_DIAG_G;  // elements per pass (shared-memory bound)
      double* sY1 = sQ + D * NS * NV * E;
      double* sY2 = sY1 + (NV + D * NV) * (P + 1) * (P + 1) * 6 * G;
      __syncthreads();
      for (int el = 0; el < E; el += G) {
        if (e0 + el >= g.K) break;
        const int ng = (int)(g.K - (e0 + el) < G ? g.K - (e0 + el) : G);
        tgv_element_sf<D, P, NV, E, NT, G>(ph, sU, sQ, sB1, nq1, w, g.detJ, el, ng, sY1, sY2, acc);
      }
    } else {
      tgv_tile<D, NV, E, NS>(ph, sU, sQ, w, Bq, nq, e0, g.K, [&](int) { return g.detJ; }, acc);
    }
  } else if constexpr (NV == D + 2) {
    tgv_tile<D, NV, E, NS>(ph, sU, sQ, w, Bq, nq, e0, g.K, [&](int) { return g.detJ; }, acc);
  }
  block_sum3<NT>(acc, red, part + 3 * blockIdx.x);
}

// ------------------------------------------------------------------ launchers
template <int D, int P, int EQ>
struct TCfg {
  static constexpr int NV = Phys<EQ, D>::NV;
  static constexpr bool VISC = Phys<EQ, D>::VISC;
  static constexpr int NL = TDims<D, P>::NL;
  static constexpr int NS = TDims<D, P>::NS;
  // tiles: kernel A (viscous volume work) and kernel B (faces + update) take E elements
  // per CTA of NT threads; small tiles keep several CTAs resident per SM so their
  // load / compute / store phases interleave
  static constexpr int E = NV > 1 ? 8 : (D == 3 ? 16 : 32);  // kernel B and traces
  static constexpr int EA = E;
#ifndef SDRT_TB_NT
#define SDRT_TB_NT 320
#endif
  static constexpr int NTB = SDRT_TB_NT;
#ifndef SDRT_TA_NT
#define SDRT_TA_NT 256
#endif
// systems (N_V > 1): 128-thread CTAs so the register-blocked line items (SDRT_TA_LINE,
// LGRP outputs per pass) get up to 255 registers at two CTAs per SM
#ifndef SDRT_TA_NT_SYS
#define SDRT_TA_NT_SYS 256
#endif
  static constexpr int NTA = NV > 1 ? SDRT_TA_NT_SYS : SDRT_TA_NT;
#ifndef SDRT_TB_MINB
#define SDRT_TB_MINB 2
#endif
  static constexpr int MINB_B = SDRT_TB_MINB;
  static constexpr int MINB_A = 2;
  static constexpr int THREADS = 256;
  static constexpr size_t TILE = (size_t)NS * NV * E * sizeof(double);
  static constexpr size_t TILEA = (size_t)NS * NV * EA * sizeof(double);
  // kernel A: tile, gradient, two internal-flux buffers of NI points per line (NI = p
  // for SDRT, p+1 solution points for FR)
  static constexpr size_t smem_a(int ni, bool osf = false) {
    return TILEA * (1 + D) + (tensor_a_dbuf(D, NS, NL, NV, EA, ni, osf) ? 2 : 1) * (size_t)NL * ni * NV * EA * sizeof(double) +
           (osf ? (size_t)D * NL * NV * EA * sizeof(double) : 0);
  }
  // kernel B, one-sided flux publication: R_int, the x_d = -1 face fluxes, the state tile
  // (stage input where read) and the RK registers the stage reads
  static size_t smem_b_osf(int stage) {
    if (SDRT_TB_DIRECT) return TILE + (size_t)D * NL * NV * E * sizeof(double) + (stage_reads_acc(stage) ? TILE : 0);
    return TILE * 2 + (size_t)D * NL * NV * E * sizeof(double) + (stage_reads_acc(stage) ? TILE : 0) +
           (stage_reads_un(stage) ? TILE : 0);
  }
  // kernel B: sU, sR, flux-line slots, + the RK registers the stage reads (ACC: stages
  // 1..3, u_n: stages 1, 2)
  static constexpr size_t smem_b0(int ni) {
    return TILE * 2 + (size_t)NL * (VISC ? 2 : ni + 2) * NV * E * sizeof(double);
  }
  static size_t smem_b(int stage, int ni) {
    return smem_b0(ni) + (stage_reads_acc(stage) ? TILE : 0) + (stage_reads_un(stage) ? TILE : 0);
  }
  static constexpr size_t SMEM_T = TILE;
};

template <int D, int P, int EQ>
static void set_smem(const void* k, size_t bytes) {
  if (bytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    // CTAs above ~98 KB: the whole 228 KB carve-out, so that two fit per SM (the default
    // carve-out stops near 200 KB; measured: OSF kernel A at 112.6 KB ran 1 CTA / SM)
    if (e == cudaSuccess && bytes > 98 * 1024)
      e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA smem attr: ") + cudaGetErrorString(e));
  }
}

static const CUtensorMap& tma_map(TensorTma* t, const void* ptr) { return cached_tile_map(t, ptr); }

static TileMaps maps_for(TensorTma* t, const TensorBufs& b, bool full) {
  TileMaps m;
  std::memset(&m, 0, sizeof(m));
  m.uin = tma_map(t, b.Uin);
  if (full) {
    if (b.U) m.un = tma_map(t, b.U);
    if (b.ACC) m.acc = tma_map(t, b.ACC);
    if (b.Rv) m.rv = tma_map(t, b.Rv);
  }
  return m;
}

// dynamic shared memory of the fused stage kernel: the larger of kernel A's (OSF) and
// kernel B's (OSF, any stage) layouts
template <int D, int P, int EQ>
static size_t fuse_smem() {
  using C = TCfg<D, P, EQ>;
  size_t sm = C::smem_a(P, true);
  for (int s : {0, 1, 2, 3, RK54_STAGE0, RK54_STAGE0 + 1})
    if (C::smem_b_osf(s) > sm) sm = C::smem_b_osf(s);
  return sm;
}

template <int D, int P, int EQ, int NI>
static void run_stage_ni(const TensorGeom& g, const Line1D& L, const PhysDev& ph, TensorTma* tma,
                         const TensorBufs& b, int stage, double dt, cudaStream_t st, int which) {
  using C = TCfg<D, P, EQ>;
  if (which == 0) {
    if constexpr (Phys<EQ, D>::VISC) {
      const unsigned grid = g.tiles ? (unsigned)g.ntiles : (unsigned)((g.K + C::EA - 1) / C::EA);
      if (grid == 0) return;
      if constexpr (EQ == EQ_NS) {
        if (g.osf) {
#if SDRT_TA_PERSIST
          if constexpr (!tensor_a_dbuf(D, TDims<D, P>::NS, TDims<D, P>::NL, Phys<EQ, D>::NV, C::EA, NI, true)) {
            auto kp = kt_grad_p<D, P, EQ, C::EA, C::NTA, C::MINB_A, NI>;
            set_smem<D, P, EQ>((const void*)kp, C::smem_a(NI, true));
            static int cap = 0;  // resident CTAs of this device
            if (cap == 0) {
              int nb = 0, dev = 0, nsm = 0;
              cudaGetDevice(&dev);
              cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kp, C::NTA, C::smem_a(NI, true));
              cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
              cap = nb * nsm > 0 ? nb * nsm : 1;
            }
            const unsigned gp = grid < (unsigned)cap ? grid : (unsigned)cap;
            CUDA_LAUNCH_OK(launch_pdl(kp, gp, C::NTA, C::smem_a(NI, true), st, g, L, ph, b, maps_for(tma, b, false), (int)grid));
            return;
          }
#endif
          auto ka = kt_grad<D, P, EQ, C::EA, C::NTA, C::MINB_A, NI, true>;
          set_smem<D, P, EQ>((const void*)ka, C::smem_a(NI, true));
          CUDA_LAUNCH_OK(launch_pdl(ka, grid, C::NTA, C::smem_a(NI, true), st, g, L, ph, b, maps_for(tma, b, false)));
          return;
        }
      }
      auto ka = kt_grad<D, P, EQ, C::EA, C::NTA, C::MINB_A, NI>;
      set_smem<D, P, EQ>((const void*)ka, C::smem_a(NI));
      CUDA_LAUNCH_OK(launch_pdl(ka, grid, C::NTA, C::smem_a(NI), st, g, L, ph, b, maps_for(tma, b, false)));
    }
  } else {
    const unsigned grid = g.tiles ? (unsigned)g.ntiles : (unsigned)((g.K + C::E - 1) / C::E);
    if (grid == 0) return;
    if constexpr (EQ == EQ_NS) {
      if (g.osf) {
        constexpr int MB = SDRT_TB_DIRECT ? 3 : C::MINB_B;
        auto kb = b.Fexp ? kt_stage_osf<D, P, EQ, C::E, C::NTB, MB, true> : kt_stage_osf<D, P, EQ, C::E, C::NTB, MB>;
        set_smem<D, P, EQ>((const void*)kb, C::smem_b_osf(2));
        CUDA_LAUNCH_OK(launch_pdl(kb, grid, C::NTB, C::smem_b_osf(stage), st, g, L, ph, b, stage, dt, maps_for(tma, b, true)));
        return;
      }
    }
    auto kb = b.Fexp ? kt_stage<D, P, EQ, C::E, C::NTB, C::MINB_B, NI, true> : kt_stage<D, P, EQ, C::E, C::NTB, C::MINB_B, NI>;
    set_smem<D, P, EQ>((const void*)kb, C::smem_b(2, NI));
    CUDA_LAUNCH_OK(launch_pdl(kb, grid, C::NTB, C::smem_b(stage, NI), st, g, L, ph, b, stage, dt, maps_for(tma, b, true)));
  }
}

// SDRT: P internal flux points per line; FR (L.fr): the P+1 solution points
template <int D, int P, int EQ>
static void run_stage(const TensorGeom& g, const Line1D& L, const PhysDev& ph, TensorTma* tma, const TensorBufs& b,
                      int stage, double dt, cudaStream_t st, int which) {
  if (L.fr) run_stage_ni<D, P, EQ, P + 1>(g, L, ph, tma, b, stage, dt, st, which);
  else run_stage_ni<D, P, EQ, P>(g, L, ph, tma, b, stage, dt, st, which);
}

template <int D, int P, int EQ>
static void run_traces(const TensorGeom& g, const Line1D& L, TensorTma* tma, const double* U, double* Tu,
                       cudaStream_t st) {
  using C = TCfg<D, P, EQ>;
  const unsigned grid = (unsigned)((g.K + C::E - 1) / C::E);
  auto k = kt_traces<D, P, EQ, C::E>;
  set_smem<D, P, EQ>((const void*)k, C::SMEM_T);
  TensorBufs b{};
  b.Uin = U;
  CUDA_LAUNCH_OK(launch_pdl(k, grid, C::THREADS, C::SMEM_T, st, g, L, maps_for(tma, b, false), Tu));
}

template <int D, int P, int EQ>
static void run_diag(const TensorGeom& g, const Line1D& L, const PhysDev& ph, TensorTma* tma, const TensorBufs& b,
                     const double* w, const double* Bq, int nq, double* part, cudaStream_t st, const double* B1,
                     int nq1) {
  using C = TCfg<D, P, EQ>;
  const unsigned grid = (unsigned)((g.K + C::E - 1) / C::E);
  auto k = L.fr ? kt_diag<D, P, EQ, C::E, 256, P + 1> : kt_diag<D, P, EQ, C::E, 256, P>;
  if (B1 && nq1 > 6) B1 = nullptr;  // the shared-memory buffers are sized for degree <= 10
  constexpr int NC = C::NV + D * C::NV, n = P + 1;
  constexpr int G = P >= 4 ? 1 : SDRT_DIAG_G;
  const size_t sm = C::TILE * (1 + D) + (size_t)NC * n * 6 * (n + 6) * G * sizeof(double);
  set_smem<D, P, EQ>((const void*)k, sm);
  k<<<grid, 256, sm, st>>>(g, L, ph, b, w, Bq, nq, part, maps_for(tma, b, false), B1, nq1);
}

template <int D, int P, int EQ>
static void init_tma(TensorTma* t, int64_t Kp) {
  using C = TCfg<D, P, EQ>;
  t->rows = C::NS * C::NV;
  t->E = C::E;
  t->Kp = Kp;
  for (int i = 0; i < 8; ++i) t->ptr[i] = nullptr;
  t->next = 0;
}

typedef void (*StageFn)(const TensorGeom&, const Line1D&, const PhysDev&, TensorTma*, const TensorBufs&, int, double,
                        cudaStream_t, int);
typedef void (*TraceFn)(const TensorGeom&, const Line1D&, TensorTma*, const double*, double*, cudaStream_t);
typedef void (*TmaFn)(TensorTma*, int64_t);

template <int D, int P>
static void pick(int eq, StageFn* s, TraceFn* t, TmaFn* m) {
  switch (eq) {
    case EQ_LINADV: *s = run_stage<D, P, EQ_LINADV>; *t = run_traces<D, P, EQ_LINADV>; *m = init_tma<D, P, EQ_LINADV>; break;
    case EQ_LINADVDIFF:
      *s = run_stage<D, P, EQ_LINADVDIFF>;
      *t = run_traces<D, P, EQ_LINADVDIFF>;
      *m = init_tma<D, P, EQ_LINADVDIFF>;
      break;
    case EQ_EULER: *s = run_stage<D, P, EQ_EULER>; *t = run_traces<D, P, EQ_EULER>; *m = init_tma<D, P, EQ_EULER>; break;
    default: *s = run_stage<D, P, EQ_NS>; *t = run_traces<D, P, EQ_NS>; *m = init_tma<D, P, EQ_NS>; break;
  }
}

static void pick_all(int D, int P, int eq, StageFn* s, TraceFn* t, TmaFn* m) {
  *s = nullptr;
  *t = nullptr;
  *m = nullptr;
  if (D == 2) {
    switch (P) {
      case 1: pick<2, 1>(eq, s, t, m); break;
      case 2: pick<2, 2>(eq, s, t, m); break;
      case 3: pick<2, 3>(eq, s, t, m); break;
      case 4: pick<2, 4>(eq, s, t, m); break;
    }
  } else {
    switch (P) {
      case 1: pick<3, 1>(eq, s, t, m); break;
      case 2: pick<3, 2>(eq, s, t, m); break;
      case 3: pick<3, 3>(eq, s, t, m); break;
      case 4: pick<3, 4>(eq, s, t, m); break;
    }
  }
}

template <int D, int P>
static int twidth(int eq) {
  switch (eq) {
    case EQ_LINADV: return TCfg<D, P, EQ_LINADV>::E;
    case EQ_LINADVDIFF: return TCfg<D, P, EQ_LINADVDIFF>::E;
    case EQ_EULER: return TCfg<D, P, EQ_EULER>::E;
    default: return TCfg<D, P, EQ_NS>::E;
  }
}

int tensor_tile_width(int D, int P, int eq) {
  if (D == 2) return P == 1 ? twidth<2, 1>(eq) : P == 2 ? twidth<2, 2>(eq) : P == 3 ? twidth<2, 3>(eq) : twidth<2, 4>(eq);
  return P == 1 ? twidth<3, 1>(eq) : P == 2 ? twidth<3, 2>(eq) : P == 3 ? twidth<3, 3>(eq) : twidth<3, 4>(eq);
}

bool tensor_supported(int D, int P, int eq) {
  StageFn s;
  TraceFn t;
  TmaFn m;
  if (eq < 0 || eq > 3) return false;
  pick_all(D, P, eq, &s, &t, &m);
  return s != nullptr;
}

void tensor_tma_init(TensorTma* tma, int D, int P, int eq, int64_t Kp) {
  StageFn s;
  TraceFn t;
  TmaFn m;
  pick_all(D, P, eq, &s, &t, &m);
  m(tma, Kp);
}

void tensor_launch_grad(int D, int P, int eq, const TensorGeom& g, const Line1D& L, const PhysDev& ph,
                        TensorTma* tma, const TensorBufs& b, cudaStream_t st) {
  StageFn s;
  TraceFn t;
  TmaFn m;
  pick_all(D, P, eq, &s, &t, &m);
  s(g, L, ph, tma, b, 0, 0.0, st, 0);
}

void tensor_launch_flux(int D, int P, int eq, const TensorGeom& g, const Line1D& L, const PhysDev& ph,
                        TensorTma* tma, const TensorBufs& b, int stage, double dt, cudaStream_t st) {
  StageFn s;
  TraceFn t;
  TmaFn m;
  pick_all(D, P, eq, &s, &t, &m);
  s(g, L, ph, tma, b, stage, dt, st, 1);
}

template <int D, int P, int EQ>
static int fuse_ctas_t() {
  if constexpr (EQ == EQ_NS) {
    using C = TCfg<D, P, EQ>;
    auto k = kt_fused<D, P, EQ, C::EA, C::NTA, C::MINB_A, P>;
    const size_t sm = fuse_smem<D, P, EQ>();
    set_smem<D, P, EQ>((const void*)k, sm);
    int nb = 0, dev = 0, nsm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, C::NTA, sm) != cudaSuccess) return 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    return nb * nsm;
  }
  return 0;
}

template <int D, int P, int EQ>
static void run_fused_t(const TensorGeom& g, const Line1D& L, const PhysDev& ph, TensorTma* tma, const TensorBufs& b,
                        int stage, double dt, const FuseSched& fs, cudaStream_t st) {
  if constexpr (EQ == EQ_NS) {
    using C = TCfg<D, P, EQ>;
    static const int nctas = fuse_ctas_t<D, P, EQ>();
    if (nctas <= 0) throw std::runtime_error("internal: fused stage kernel has no resident CTA");
    auto k = kt_fused<D, P, EQ, C::EA, C::NTA, C::MINB_A, P>;
    CUDA_LAUNCH_OK(launch_pdl(k, (unsigned)nctas, C::NTA, fuse_smem<D, P, EQ>(), st, g, L, ph, b, stage, dt,
                              maps_for(tma, b, true), fs));
  } else {
    throw std::runtime_error("internal: fused stage kernel is NS-only");
  }
}

int tensor_fuse_ctas(int D, int P, int eq) {
  if (eq != EQ_NS) return 0;
  if (D == 2) return P == 1 ? fuse_ctas_t<2, 1, EQ_NS>() : P == 2 ? fuse_ctas_t<2, 2, EQ_NS>() : P == 3 ? fuse_ctas_t<2, 3, EQ_NS>() : fuse_ctas_t<2, 4, EQ_NS>();
  return P == 1 ? fuse_ctas_t<3, 1, EQ_NS>() : P == 2 ? fuse_ctas_t<3, 2, EQ_NS>() : P == 3 ? fuse_ctas_t<3, 3, EQ_NS>() : fuse_ctas_t<3, 4, EQ_NS>();
}

void tensor_launch_fused(int D, int P, int eq, const TensorGeom& g, const Line1D& L, const PhysDev& ph,
                         TensorTma* tma, const TensorBufs& b, int stage, double dt, const FuseSched& fs,
                         cudaStream_t st) {
  if (eq != EQ_NS || L.fr || g.tiles || b.Fexp || stage < 0) throw std::runtime_error("internal: fused stage misuse");
  if (D == 2) {
    switch (P) {
      case 1: run_fused_t<2, 1, EQ_NS>(g, L, ph, tma, b, stage, dt, fs, st); break;
      case 2: run_fused_t<2, 2, EQ_NS>(g, L, ph, tma, b, stage, dt, fs, st); break;
      case 3: run_fused_t<2, 3, EQ_NS>(g, L, ph, tma, b, stage, dt, fs, st); break;
      default: run_fused_t<2, 4, EQ_NS>(g, L, ph, tma, b, stage, dt, fs, st); break;
    }
  } else {
    switch (P) {
      case 1: run_fused_t<3, 1, EQ_NS>(g, L, ph, tma, b, stage, dt, fs, st); break;
      case 2: run_fused_t<3, 2, EQ_NS>(g, L, ph, tma, b, stage, dt, fs, st); break;
      case 3: run_fused_t<3, 3, EQ_NS>(g, L, ph, tma, b, stage, dt, fs, st); break;
      default: run_fused_t<3, 4, EQ_NS>(g, L, ph, tma, b, stage, dt, fs, st); break;
    }
  }
}

// Job list of the fused stage on a periodic single-rank pattern mesh (element order x
// fastest, tiles of E consecutive elements): deps[t] = t and the tiles holding the x_d - 1
// neighbours of t's elements; B(t) is placed after A(min(max deps[t] + lag, ntiles - 1)).
bool tensor_fuse_plan(int D, const int N[3], int64_t K, int E, int lag, std::vector<int>* jobs,
                      std::vector<int>* deps) {
  const int64_t nt = (K + E - 1) / E;
  deps->assign((size_t)nt * FUSE_DEPS, -1);
  std::vector<std::vector<int>> after((size_t)nt);
  for (int64_t t = 0; t < nt; ++t) {
    int* dl = deps->data() + t * FUSE_DEPS;
    int nd = 0;
    int64_t last = t;
    auto add = [&](int64_t u) {
      for (int k = 0; k < nd; ++k)
        if (dl[k] == (int)u) return true;
      if (nd == FUSE_DEPS) return false;
      dl[nd++] = (int)u;
      last = u > last ? u : last;
      return true;
    };
    add(t);
    for (int64_t e = t * E; e < (t + 1) * E && e < K; ++e) {
      const int64_t c[3] = {e % N[0], (e / N[0]) % N[1], D == 3 ? e / ((int64_t)N[0] * N[1]) : 0};
      for (int d = 0; d < D; ++d) {
        int64_t cc[3] = {c[0], c[1], c[2]};
        cc[d] = (cc[d] + N[d] - 1) % N[d];
        const int64_t m = cc[0] + (int64_t)N[0] * (cc[1] + (int64_t)N[1] * cc[2]);
        if (!add(m / E)) return false;
      }
    }
    const int64_t at = last + lag < nt - 1 ? last + lag : nt - 1;
    after[(size_t)at].push_back((int)t);
  }
  jobs->clear();
  for (int64_t a = 0; a < nt; ++a) {
    jobs->push_back((int)(a * 2));
    for (int t : after[(size_t)a]) jobs->push_back(t * 2 + 1);
  }
  return true;
}

void tensor_launch_diag(int D, int P, const TensorGeom& g, const Line1D& L, const PhysDev& ph, TensorTma* tma,
                        const TensorBufs& b, const double* w, const double* Bq, int nq, double* part,
                        cudaStream_t st, const double* B1, int nq1) {
  if (D != 3) throw std::runtime_error("unsupported: TGV diagnostics need a 3-D NS context");
  switch (P) {
    case 1: run_diag<3, 1, EQ_NS>(g, L, ph, tma, b, w, Bq, nq, part, st, B1, nq1); break;
    case 2: run_diag<3, 2, EQ_NS>(g, L, ph, tma, b, w, Bq, nq, part, st, B1, nq1); break;
    case 3: run_diag<3, 3, EQ_NS>(g, L, ph, tma, b, w, Bq, nq, part, st, B1, nq1); break;
    default: run_diag<3, 4, EQ_NS>(g, L, ph, tma, b, w, Bq, nq, part, st, B1, nq1); break;
  }
}

void tensor_launch_traces(int D, int P, int eq, const TensorGeom& g, const Line1D& L, TensorTma* tma,
                          const double* U, double* Tu, cudaStream_t st) {
  StageFn s;
  TraceFn t;
  TmaFn m;
  pick_all(D, P, eq, &s, &t, &m);
  t(g, L, tma, U, Tu, st);
}

#ifdef SDRT_PHASE_PROF
void tensor_phase_cycles(unsigned long long* out, bool reset) {
  cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(g_phase_cycles));
  if (reset) {
    static unsigned long long z[2][16] = {};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  }
}
#endif

}  // namespace sdrt

#ifdef SDRT_PHASE_PROF
// tools-only accessor of the profiling build (libsdrt_prof.so); not part of include/sdrt.h
extern "C" void sdrt_debug_phase_cycles(unsigned long long* out, int reset) {
  sdrt::tensor_phase_cycles(out, reset != 0);
}
#endif
