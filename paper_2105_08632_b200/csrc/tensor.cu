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

#include <stdexcept>
#include <string>

#include "tensor.cuh"

namespace sdrt {

template <int D, int P>
struct TDims {
  static constexpr int n = P + 1;
  static constexpr int NL = D == 2 ? n : n * n;  // lines per direction (= points per face)
  static constexpr int NS = D == 2 ? n * n : n * n * n;
  static constexpr int NEXT = 2 * D * NL;
};

template <int D, int P>
__device__ __forceinline__ int sidx(int d, int t, int i) {
  constexpr int n = P + 1;
  if constexpr (D == 2) {
    return d == 0 ? i + n * t : t + n * i;
  } else {
    const int ta = t % n, tb = t / n;
    return d == 0 ? i + n * (ta + n * tb) : (d == 1 ? ta + n * (i + n * tb) : ta + n * (tb + n * i));
  }
}

// neighbour element along axis d (delta = -1 / +1), periodic pattern grid, N_p = 1
template <int D>
__device__ __forceinline__ int64_t tnbr(const TensorGeom& g, int64_t e, int d, int delta) {
  int c[3];
  int64_t r = e;
  c[0] = (int)(r % g.N[0]);
  r /= g.N[0];
  c[1] = (int)(r % g.N[1]);
  r /= g.N[1];
  c[2] = (int)r;
  int v = c[d] + delta;
  if ((v < 0 || v >= g.N[d]) && g.halo[d]) {
    // ghost column of the neighbouring rank's element: slab (d, side), tangential index
    const int a = d == 0 ? 1 : 0, bb = d == 2 ? 1 : 2;
    const int64_t tang = D == 2 ? c[a] : c[a] + (int64_t)g.N[a] * c[bb];
    return g.gbase[d][v < 0 ? 0 : 1] + tang;
  }
  v = v < 0 ? v + g.N[d] : (v >= g.N[d] ? v - g.N[d] : v);
  c[d] = v;
  return (int64_t)c[0] + (int64_t)g.N[0] * (c[1] + (int64_t)g.N[1] * c[2]);
}

// value at a line end: explicit fma chain in fixed order (bit-identical wherever used)
template <int n>
__device__ __forceinline__ double interp_end(const double (&Iend)[TMAXP + 1], const double* u) {
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < n; ++i) acc = __fma_rn(Iend[i], u[i], acc);
  return acc;
}

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
__device__ __forceinline__ void prefetch_traces(const TensorGeom& g, const double* __restrict__ T, int64_t e0,
                                                bool own) {
  using Tm = TDims<D, P>;
  constexpr int NL = Tm::NL;
  for (int item = threadIdx.x; item < 2 * D * NL * NV; item += blockDim.x) {
    const int v = item % NV, ext = item / NV;
    const int face = ext / NL, d = face / 2, side = face % 2;
    // the neighbour across face (d, side) reads its opposite face (d, 1-side)
    const int ext_n = (2 * d + 1 - side) * NL + ext % NL;
    const int64_t m = tnbr<D>(g, e0, d, side ? 1 : -1);
    prefetch_l2(T + ((int64_t)ext_n * NV + v) * g.Kt + m);
    if (own) prefetch_l2(T + ((int64_t)ext * NV + v) * g.Kt + e0);
  }
}

template <int D, int P, int NV, int E>
__device__ __forceinline__ void prefetch_rows(const double* __restrict__ A, int64_t e0, int64_t Kp) {
  constexpr int NS = TDims<D, P>::NS;
  for (int row = threadIdx.x; row < NS * NV; row += blockDim.x) prefetch_l2(A + (int64_t)row * Kp + e0);
}

// gradient along lines -> sQ[d][s][v][E] = (2/h_d) (M16 C + M15 U_int)   (l.295-302)
template <int D, int P, int EQ, int E>
__device__ __forceinline__ void gradient_lines(const TensorGeom& g, const Line1D& L, const PhysDev& ph,
                                               const double* __restrict__ Tu, const double* sU, double* sQ,
                                               int64_t e0) {
  using T = TDims<D, P>;
  constexpr int n = T::n, NL = T::NL, NS = T::NS;
  constexpr int NV = Phys<EQ, D>::NV;
  const double wl = 0.5 - ph.beta, wr = 0.5 + ph.beta;
#pragma unroll
  for (int d = 0; d < D; ++d)
  for (int item = threadIdx.x; item < NL * E; item += blockDim.x) {
    const int el = item % E, t = item / E;
    const int64_t e = e0 + el;
    if (e >= g.K) continue;
    const int64_t mlo = tnbr<D>(g, e, d, -1), mhi = tnbr<D>(g, e, d, +1);
    // neighbour traces for all variables first (loads in flight together)
    double nbl[NV], nbh[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      nbl[v] = Tu[((int64_t)((2 * d + 1) * NL + t) * NV + v) * g.Kt + mlo];
      nbh[v] = Tu[((int64_t)((2 * d + 0) * NL + t) * NV + v) * g.Kt + mhi];
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double u[n];
#pragma unroll
      for (int i = 0; i < n; ++i) u[i] = sU[(sidx<D, P>(d, t, i) * NV + v) * E + el];
      // common values at both ends (own trace recomputed bit-identically, neighbour read)
      const double own0 = interp_end<n>(L.Iend[0], u), own1 = interp_end<n>(L.Iend[1], u);
      const double nb0 = nbl[v];
      const double nb1 = nbh[v];
      const double c0 = wl * nb0 + wr * own0;   // face x_d = -1: this element is RIGHT
      const double c1 = wl * own1 + wr * nb1;   // face x_d = +1: this element is LEFT
      double ui[P];
#pragma unroll
      for (int a = 0; a < P; ++a) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < n; ++i) s = fma(L.Iint[a][i], u[i], s);
        ui[a] = s;
      }
#pragma unroll
      for (int i = 0; i < n; ++i) {
        double q = L.Dfl[i][0] * c0;
#pragma unroll
        for (int a = 0; a < P; ++a) q = fma(L.Dfl[i][a + 1], ui[a], q);
        q = fma(L.Dfl[i][P + 1], c1, q);
        sQ[((d * NS + sidx<D, P>(d, t, i)) * NV + v) * E + el] = g.jinv[d] * q;
      }
    }
  }
}

// traces of a state held in shared memory -> T[N_ext][N_V][Kp]
template <int D, int P, int NV, int E>
__device__ __forceinline__ void write_traces(const TensorGeom& g, const Line1D& L, const double* sU,
                                             double* __restrict__ T, int64_t e0) {
  using Tm = TDims<D, P>;
  constexpr int n = Tm::n, NL = Tm::NL, NEXT = Tm::NEXT;
  (void)NEXT;
#pragma unroll
  for (int face = 0; face < 2 * D; ++face) {
    const int d = face / 2, side = face % 2;
    for (int item = threadIdx.x; item < NL * NV * E; item += blockDim.x) {
      const int el = item % E, r = item / E, v = r % NV, t = r / NV;
      const int64_t e = e0 + el;
      if (e >= g.K) continue;
      const int ext = face * NL + t;
      double u[n];
#pragma unroll
      for (int i = 0; i < n; ++i) u[i] = sU[(sidx<D, P>(d, t, i) * NV + v) * E + el];
      T[((int64_t)ext * NV + v) * g.Kt + e] = interp_end<n>(L.Iend[side], u);
    }
  }
}

template <int D, int P, int EQ, int E>
__global__ void __launch_bounds__(256) kt_traces(TensorGeom g, Line1D L, const double* __restrict__ U,
                                                 double* __restrict__ T) {
  constexpr int NV = Phys<EQ, D>::NV;
  extern __shared__ double smem[];
  const int64_t e0 = (int64_t)blockIdx.x * E;
  load_tile<D, P, NV, E>(U, smem, e0, g.K, g.Kp);
  wait_tile();
  __syncthreads();
  write_traces<D, P, NV, E>(g, L, smem, T, e0);
}

// kernel A: gradient + published viscous normal-flux traces
template <int D, int P, int EQ, int E>
__global__ void __launch_bounds__(256) kt_grad(TensorGeom g, Line1D L, PhysDev ph, TensorBufs b) {
  using Ph = Phys<EQ, D>;
  using T = TDims<D, P>;
  constexpr int NV = Ph::NV, n = T::n, NL = T::NL, NS = T::NS;
  extern __shared__ double smem[];
  double* sU = smem;
  double* sQ = smem + NS * NV * E;
  const int64_t e0 = (int64_t)blockIdx.x * E;
  load_tile<D, P, NV, E>(b.Uin, sU, e0, g.K, g.Kp);
  prefetch_traces<D, P, NV, E>(g, b.Tu, e0, false);
  wait_tile();
  __syncthreads();
  gradient_lines<D, P, EQ, E>(g, L, ph, b.Tu, sU, sQ, e0);
  __syncthreads();
  // publish g at face points of the sides that carry weight: side 1 (left) if
  // 1/2 + beta != 0, side 0 (right) if 1/2 - beta != 0
  const bool pub1 = (0.5 + ph.beta) != 0.0, pub0 = (0.5 - ph.beta) != 0.0;
#pragma unroll
  for (int face = 0; face < 2 * D; ++face)
  for (int item = threadIdx.x; item < NL * E; item += blockDim.x) {
    const int el = item % E, t = item / E;
    const int d = face / 2, side = face % 2, ext = face * NL + t;
    if ((side == 1 && !pub1) || (side == 0 && !pub0)) continue;
    const int64_t e = e0 + el;
    if (e >= g.K) continue;
    double u[NV], q[D * NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double ul[n];
#pragma unroll
      for (int i = 0; i < n; ++i) ul[i] = sU[(sidx<D, P>(d, t, i) * NV + v) * E + el];
      u[v] = interp_end<n>(L.Iend[side], ul);
#pragma unroll
      for (int dd = 0; dd < D; ++dd) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < n; ++i) s = fma(L.Iend[side][i], sQ[((dd * NS + sidx<D, P>(d, t, i)) * NV + v) * E + el], s);
        q[dd * NV + v] = s;
      }
    }
    double nL[D];
#pragma unroll
    for (int k = 0; k < D; ++k) nL[k] = (k == d) ? 1.0 : 0.0;  // canonical (left) normal +e_d
    double gv[NV];
    Ph::visc_dir(ph, u, q, nL, gv);
#pragma unroll
    for (int v = 0; v < NV; ++v) b.Tg[((int64_t)ext * NV + v) * g.Kt + e] = gv[v];
  }
}

// kernel B: fluxes, divergence, RK update, new traces
template <int D, int P, int EQ, int E>
__global__ void __launch_bounds__(256) kt_stage(TensorGeom g, Line1D L, PhysDev ph, TensorBufs b, int stage,
                                                double dt) {
  using Ph = Phys<EQ, D>;
  using T = TDims<D, P>;
  constexpr int NV = Ph::NV, n = T::n, NL = T::NL, NS = T::NS;
  extern __shared__ double smem[];
  double* sU = smem;
  double* sR = smem + NS * NV * E;
  double* sQ = sR + NS * NV * E;
  const int64_t e0 = (int64_t)blockIdx.x * E;
  load_tile<D, P, NV, E>(b.Uin, sU, e0, g.K, g.Kp);
  // warm L2 with everything this tile reads later: neighbour traces, published
  // viscous traces, RK registers (their latency is otherwise exposed mid-kernel)
  prefetch_traces<D, P, NV, E>(g, b.Tu, e0, false);
  if constexpr (Ph::VISC) prefetch_traces<D, P, NV, E>(g, b.Tg, e0, true);
  if (stage == 1 || stage == 2) prefetch_rows<D, P, NV, E>(b.U, e0, g.Kp);
  if (stage >= 1) prefetch_rows<D, P, NV, E>(b.ACC, e0, g.Kp);
  wait_tile();
  __syncthreads();
  if constexpr (Ph::VISC) {
    gradient_lines<D, P, EQ, E>(g, L, ph, b.Tu, sU, sQ, e0);
    __syncthreads();
  }
  const double wl = 0.5 + ph.beta, wr = 0.5 - ph.beta;
  // neighbour element ids of the tile, once: sNb[2d + side][el]
  __shared__ int sNb[2 * D][E];
  for (int idx = threadIdx.x; idx < 2 * D * E; idx += blockDim.x) {
    const int el = idx % E, k = idx / E;
    const int64_t e = e0 + el;
    sNb[k][el] = e < g.K ? (int)tnbr<D>(g, e, k / 2, (k % 2) ? 1 : -1) : 0;
  }
  __syncthreads();
  const int Kp = (int)g.Kt;  // trace row stride
  // one code copy for all directions (runtime d): keeps the kernel inside the I-cache
#pragma unroll 1
  for (int d = 0; d < D; ++d) {
    const double wf = g.detJ * g.jinv[d];  // transformed-flux weight detJ (J^-1)_dd
    const int str = (d == 0 ? 1 : (d == 1 ? n : n * n)) * NV * E;  // point stride along the line
    for (int item = threadIdx.x; item < NL * E; item += blockDim.x) {
      const int el = item % E, t = item / E;
      const int e = (int)(e0 + el);
      if (e >= g.K) continue;
      const int base = d == 0 ? n * t : (d == 1 ? (D == 2 ? t : (t % n) + n * n * (t / n)) : t);
      const double* pu = sU + base * NV * E + el;
      const double* pq = sQ + base * NV * E + el;
      double* pr = sR + base * NV * E + el;
      // issue the line-end global loads first (consumed after the internal points)
      const int mlo = sNb[2 * d][el], mhi = sNb[2 * d + 1][el];
      const int xL = (2 * d + 1) * NL + t, xR = (2 * d) * NL + t;  // left's +face, right's -face
      double un0[NV], un1[NV], gs0[NV], gs1[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        un0[v] = b.Tu[(xL * NV + v) * Kp + mlo];   // left neighbour's trace (I am right)
        un1[v] = b.Tu[(xR * NV + v) * Kp + mhi];   // right neighbour's trace (I am left)
        if constexpr (Ph::VISC) {
          const double* tg = b.Tg;
          double a0 = 0.0, a1 = 0.0;
          if (wl != 0.0) {
            a0 = wl * tg[(xL * NV + v) * Kp + mlo];
            a1 = wl * tg[(xL * NV + v) * Kp + e];
          }
          if (wr != 0.0) {
            a0 = fma(wr, tg[(xR * NV + v) * Kp + e], a0);
            a1 = fma(wr, tg[(xR * NV + v) * Kp + mhi], a1);
          }
          gs0[v] = a0;
          gs1[v] = a1;
        }
      }
      double r[n][NV];
#pragma unroll
      for (int i = 0; i < n; ++i)
#pragma unroll
        for (int v = 0; v < NV; ++v) r[i][v] = d == 0 ? 0.0 : pr[i * str + v * E];
      // both ends: common flux with canonical (left, right) = (x_d- element, x_d+ element)
      double nL[D];
#pragma unroll
      for (int k = 0; k < D; ++k) nL[k] = (k == d) ? 1.0 : 0.0;
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        double uo[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          double ul[n];
#pragma unroll
          for (int i = 0; i < n; ++i) ul[i] = pu[i * str + v * E];
          uo[v] = interp_end<n>(L.Iend[side], ul);
        }
        const double* uL = side ? uo : un0;
        const double* uR = side ? un1 : uo;
        double F[NV];
        Ph::conv_common(ph, uL, uR, nL, F);
        if constexpr (Ph::VISC) {
#pragma unroll
          for (int v = 0; v < NV; ++v) F[v] += (side ? gs1[v] : gs0[v]) + ph.eta * (uL[v] - uR[v]);
        }
        const double sD = side ? g.sface[d] : -g.sface[d];
        // M14 column of this end: -L_0' (x_d = -1), +L_{p+1}' (x_d = +1)
#pragma unroll
        for (int i = 0; i < n; ++i) {
          const double m14 = side ? L.Dfl[i][P + 1] : -L.Dfl[i][0];
#pragma unroll
          for (int v = 0; v < NV; ++v) r[i][v] = fma(m14, sD * F[v], r[i][v]);
        }
      }
      // internal flux points along the line (normal e_d): F~ = detJ (J^-1 f)_d
      // (not unrolled: bounds the live range to one point)
#pragma unroll 1
      for (int a = 0; a < P; ++a) {
        double ua[NV], qa[Ph::VISC ? D * NV : 1], w[D], f[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          double sacc = 0.0;
#pragma unroll
          for (int i = 0; i < n; ++i) sacc = fma(L.Iint[a][i], pu[i * str + v * E], sacc);
          ua[v] = sacc;
        }
        if constexpr (Ph::VISC) {
#pragma unroll
          for (int dd = 0; dd < D; ++dd)
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              double sacc = 0.0;
#pragma unroll
              for (int i = 0; i < n; ++i) sacc = fma(L.Iint[a][i], pq[dd * NS * NV * E + i * str + v * E], sacc);
              qa[dd * NV + v] = sacc;
            }
        }
#pragma unroll
        for (int k = 0; k < D; ++k) w[k] = (k == d) ? wf : 0.0;
        Ph::conv_dir(ph, ua, w, f);
        if constexpr (Ph::VISC) {
          double fv[NV];
          Ph::visc_dir(ph, ua, qa, w, fv);
#pragma unroll
          for (int v = 0; v < NV; ++v) f[v] += fv[v];
        }
#pragma unroll
        for (int i = 0; i < n; ++i)
#pragma unroll
          for (int v = 0; v < NV; ++v) r[i][v] = fma(L.Dfl[i][a + 1], f[v], r[i][v]);
      }
#pragma unroll
      for (int i = 0; i < n; ++i)
#pragma unroll
        for (int v = 0; v < NV; ++v) pr[i * str + v * E] = r[i][v];
    }
    __syncthreads();
  }
  // dU/dt = -R~/detJ, RK4 (3-register form), new state into sU.  Rows are processed in
  // batches of RB_RK per thread with all global loads of a batch issued before use.
  const double idet = 1.0 / g.detJ;
  constexpr int TOT = NS * NV * E;
  constexpr int RB_RK = 5;
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
      const double kk = -sR[idx] * idet;
      double nu;
      switch (stage) {
        case -1:
          b.out[gi[k]] = kk;
          nu = 0.0;
          break;
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
  write_traces<D, P, NV, E>(g, L, sU, b.Tu_next, e0);
}

// ------------------------------------------------------------------ launchers
template <int D, int P, int EQ>
struct TCfg {
  static constexpr int NV = Phys<EQ, D>::NV;
  static constexpr int E = NV > 1 ? 8 : (D == 3 ? 16 : 32);
  static constexpr int NL = TDims<D, P>::NL;
  static constexpr int THREADS = ((NL * E + 31) / 32) * 32 > 256 ? 256 : ((NL * E + 31) / 32) * 32;
  static constexpr size_t TILE = (size_t)TDims<D, P>::NS * NV * E * sizeof(double);
  static constexpr size_t SMEM_A = TILE * (1 + D);
  static constexpr size_t SMEM_B = TILE * (2 + (Phys<EQ, D>::VISC ? D : 0));
  static constexpr size_t SMEM_T = TILE;
};

template <int D, int P, int EQ>
static void set_smem(const void* k, size_t bytes) {
  if (bytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA smem attr: ") + cudaGetErrorString(e));
  }
}

template <int D, int P, int EQ>
static void run_stage(const TensorGeom& g, const Line1D& L, const PhysDev& ph, const TensorBufs& b, int stage,
                      double dt, cudaStream_t st, int which) {
  using C = TCfg<D, P, EQ>;
  const unsigned grid = (unsigned)((g.K + C::E - 1) / C::E);
  if (which == 0) {
    if constexpr (Phys<EQ, D>::VISC) {
      auto ka = kt_grad<D, P, EQ, C::E>;
      set_smem<D, P, EQ>((const void*)ka, C::SMEM_A);
      ka<<<grid, C::THREADS, C::SMEM_A, st>>>(g, L, ph, b);
    }
  } else {
    auto kb = kt_stage<D, P, EQ, C::E>;
    set_smem<D, P, EQ>((const void*)kb, C::SMEM_B);
    kb<<<grid, C::THREADS, C::SMEM_B, st>>>(g, L, ph, b, stage, dt);
  }
}

template <int D, int P, int EQ>
static void run_traces(const TensorGeom& g, const Line1D& L, const double* U, double* Tu, cudaStream_t st) {
  using C = TCfg<D, P, EQ>;
  const unsigned grid = (unsigned)((g.K + C::E - 1) / C::E);
  auto k = kt_traces<D, P, EQ, C::E>;
  set_smem<D, P, EQ>((const void*)k, C::SMEM_T);
  k<<<grid, C::THREADS, C::SMEM_T, st>>>(g, L, U, Tu);
}

typedef void (*StageFn)(const TensorGeom&, const Line1D&, const PhysDev&, const TensorBufs&, int, double,
                        cudaStream_t, int);
typedef void (*TraceFn)(const TensorGeom&, const Line1D&, const double*, double*, cudaStream_t);

template <int D, int P>
static void pick(int eq, StageFn* s, TraceFn* t) {
  switch (eq) {
    case EQ_LINADV: *s = run_stage<D, P, EQ_LINADV>; *t = run_traces<D, P, EQ_LINADV>; break;
    case EQ_LINADVDIFF: *s = run_stage<D, P, EQ_LINADVDIFF>; *t = run_traces<D, P, EQ_LINADVDIFF>; break;
    case EQ_EULER: *s = run_stage<D, P, EQ_EULER>; *t = run_traces<D, P, EQ_EULER>; break;
    default: *s = run_stage<D, P, EQ_NS>; *t = run_traces<D, P, EQ_NS>; break;
  }
}

static void pick_all(int D, int P, int eq, StageFn* s, TraceFn* t) {
  *s = nullptr;
  *t = nullptr;
  if (D == 2) {
    switch (P) {
      case 1: pick<2, 1>(eq, s, t); break;
      case 2: pick<2, 2>(eq, s, t); break;
      case 3: pick<2, 3>(eq, s, t); break;
      case 4: pick<2, 4>(eq, s, t); break;
    }
  } else {
    switch (P) {
      case 1: pick<3, 1>(eq, s, t); break;
      case 2: pick<3, 2>(eq, s, t); break;
      case 3: pick<3, 3>(eq, s, t); break;
      case 4: pick<3, 4>(eq, s, t); break;
    }
  }
}

bool tensor_supported(int D, int P, int eq) {
  StageFn s;
  TraceFn t;
  if (eq < 0 || eq > 3) return false;
  pick_all(D, P, eq, &s, &t);
  return s != nullptr;
}

void tensor_launch_grad(int D, int P, int eq, const TensorGeom& g, const Line1D& L, const PhysDev& ph,
                        const TensorBufs& b, cudaStream_t st) {
  StageFn s;
  TraceFn t;
  pick_all(D, P, eq, &s, &t);
  s(g, L, ph, b, 0, 0.0, st, 0);
}

void tensor_launch_flux(int D, int P, int eq, const TensorGeom& g, const Line1D& L, const PhysDev& ph,
                        const TensorBufs& b, int stage, double dt, cudaStream_t st) {
  StageFn s;
  TraceFn t;
  pick_all(D, P, eq, &s, &t);
  s(g, L, ph, b, stage, dt, st, 1);
}

void tensor_launch_traces(int D, int P, int eq, const TensorGeom& g, const Line1D& L, const double* U,
                          double* Tu, cudaStream_t st) {
  StageFn s;
  TraceFn t;
  pick_all(D, P, eq, &s, &t);
  t(g, L, U, Tu, st);
}

}  // namespace sdrt
