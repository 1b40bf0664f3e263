// SDRT residual + classical RK4 on sm_100a (fp64) and the device-side C ABI.
//
// Residual per stage, §2.1 l.268-350 in App. B matrix form l.2855-2925:
//   U_ext = M0 U, U_u = M12 U                                   (interp kernels)
//   [viscous] C = (1/2-b) u_L + (1/2+b) u_R at face points      (k_common_value)
//             Q~ = [M16 | M15 P] [C; U_u], Q = J^-T Q~           (apply + k_metric_grad)
//             Q_ext = M5 Q, Q_u = M18 Q                          (apply on [s][d][v][n])
//   F~_u = detJ J^-1 f(U_u, Q_u)                                (k_int_flux)
//   D~ = +/- s F(u_L, u_R, q_L, q_R, n_L), once per face point   (k_face_flux, canonical L/R)
//   R~ = [M14 | M13 M19 P2] [D~; F~_u]                           (apply)
//   dU/dt = -R~/detJ, fused with the RK4 register update        (k_rk)
// Layouts (element fastest, K_pad columns):  U, R [N_sol][N_V][Kp];  U_ext [N_ext][N_V][Kp];
// Xg = [C; U_u] [(N_ext+N_u)][N_V][Kp];  Q [N_sol][D][N_V][Kp];  Q_ext [N_ext][D][N_V][Kp];
// Q_u [N_u][D][N_V][Kp];  Xd = [D~; F~_u] [(N_ext + D N_u)][N_V][Kp].
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "capi_internal.h"
// TGV diagnostics on tensor elements: the degree-10 cubature interpolation applied
// sum-factorised through its 1D factor (1) or as the dense N_q x N_sol matrix (0)
#ifndef SDRT_DIAG_SF
#define SDRT_DIAG_SF 1
#endif
#include "comm.h"
#include "ctx.h"
#include "tensor.cuh"
#include "simplex.cuh"
#include "rk.cuh"

namespace sdrt {

#define CUDA_OK(x)                                                                        \
  do {                                                                                    \
    cudaError_t err_ = (x);                                                               \
    if (err_ != cudaSuccess)                                                              \
      throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(err_) + " at " \
                               #x);                                                       \
  } while (0)

// ------------------------------------------------------------------------ kernels
// Y[r][j] = sum_c M[r][c] X[c][j]  for j in [0, W)  (one row chunk per blockIdx.y)
__global__ void __launch_bounds__(256) k_apply(OpDev M, const double* __restrict__ X,
                                               double* __restrict__ Y, int64_t W) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int ch = blockIdx.y;
  if (j >= W) return;
  double acc[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) acc[r] = 0.0;
  const int b = M.chunk_ptr[ch], e = M.chunk_ptr[ch + 1];
  for (int k = b; k < e; ++k) {
    const double x = X[(int64_t)__ldg(M.col + k) * W + j];
    const double* v = M.val + (int64_t)k * RB;
#pragma unroll
    for (int r = 0; r < RB; ++r) acc[r] = fma(__ldg(v + r), x, acc[r]);
  }
  const int r0 = ch * RB;
#pragma unroll
  for (int r = 0; r < RB; ++r)
    if (r0 + r < M.rows) Y[(int64_t)(r0 + r) * W + j] = acc[r];
}

// neighbour of local element n across local face f: element id and its face
__device__ __forceinline__ int64_t nbr_elem(const GeomDev& g, int64_t n, int s, int f) {
  int64_t pat = n / g.nsub;
  int c[3] = {0, 0, 0};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    if (d < g.nd) {
      c[d] = (int)(pat % g.Nloc[d]);
      pat /= g.Nloc[d];
    }
  }
  int64_t id = 0, mul = 1;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    if (d < g.nd) {
      int cc = c[d] + g.off[s][f][d];
      if (cc < 0) cc += g.Nloc[d];
      if (cc >= g.Nloc[d]) cc -= g.Nloc[d];
      id += mul * cc;
      mul *= g.Nloc[d];
    }
  }
  return id * g.nsub + g.nshape[s][f];
}

// C at external points: (1/2-b) u_L + (1/2+b) u_R, written into Xg rows [0, N_ext)
template <int NV>
__global__ void __launch_bounds__(256) k_common_value(GeomDev g, PhysDev ph, const double* __restrict__ Uext,
                                                      double* __restrict__ Xg) {
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int e = blockIdx.y;
  if (n >= g.K) return;
  const int s = (int)(n % g.nsub);
  const int f = g.xface[e], q = e - g.fptr[f];
  const int64_t m = nbr_elem(g, n, s, f);
  const int e2 = g.fptr[g.nface[s][f]] + g.perm[s][f][q];
  const bool left = g.left[s][f];
  const double wl = 0.5 - ph.beta, wr = 0.5 + ph.beta;
#pragma unroll
  for (int a = 0; a < NV; ++a) {
    const double mine = Uext[((int64_t)e * NV + a) * g.Kp + n];
    const double other = Uext[((int64_t)e2 * NV + a) * g.Kp + m];
    const double uL = left ? mine : other, uR = left ? other : mine;
    Xg[((int64_t)e * NV + a) * g.Kp + n] = wl * uL + wr * uR;
  }
}

// Q = J^-T Q~ in place on [s][d][v][n]
template <int D, int NV>
__global__ void __launch_bounds__(256) k_metric_grad(GeomDev g, double* __restrict__ Q, int nsol) {
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int sp = blockIdx.y;
  if (n >= g.K) return;
  const int s = (int)(n % g.nsub);
#pragma unroll
  for (int a = 0; a < NV; ++a) {
    double qt[D];
#pragma unroll
    for (int d = 0; d < D; ++d) qt[d] = Q[(((int64_t)sp * D + d) * NV + a) * g.Kp + n];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double v = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) v = fma(g.Jinv[s][j * 3 + i], qt[j], v);
      Q[(((int64_t)sp * D + i) * NV + a) * g.Kp + n] = v;
    }
  }
}

// F~_u[d][u] = (detJ J^-1 f(u, q))_d  into Xd rows [N_ext + d N_u + u]
template <int EQ, int D>
__global__ void __launch_bounds__(256) k_int_flux(GeomDev g, PhysDev ph, const double* __restrict__ Uu,
                                                  const double* __restrict__ Qu, double* __restrict__ Xd,
                                                  int nu, int next) {
  using P = Phys<EQ, D>;
  constexpr int NV = P::NV;
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int u = blockIdx.y;
  if (n >= g.K) return;
  const int s = (int)(n % g.nsub);
  double uu[NV], qq[D * NV];
#pragma unroll
  for (int a = 0; a < NV; ++a) uu[a] = Uu[((int64_t)u * NV + a) * g.Kp + n];
  if constexpr (P::VISC) {
#pragma unroll
    for (int d = 0; d < D; ++d)
#pragma unroll
      for (int a = 0; a < NV; ++a) qq[d * NV + a] = Qu[(((int64_t)u * D + d) * NV + a) * g.Kp + n];
  }
#pragma unroll
  for (int d = 0; d < D; ++d) {
    double w[D];
#pragma unroll
    for (int j = 0; j < D; ++j) w[j] = g.detJ[s] * g.Jinv[s][d * 3 + j];
    double f[NV];
    P::conv_dir(ph, uu, w, f);
    if constexpr (P::VISC) {
      double fv[NV];
      P::visc_dir(ph, uu, qq, w, fv);
#pragma unroll
      for (int a = 0; a < NV; ++a) f[a] += fv[a];
    }
#pragma unroll
    for (int a = 0; a < NV; ++a) Xd[(((int64_t)next + d * nu + u) * NV + a) * g.Kp + n] = f[a];
  }
}

// D~ at external points: common flux with canonical (left, right) order
template <int EQ, int D>
__global__ void __launch_bounds__(256) k_face_flux(GeomDev g, PhysDev ph, const ExtMetric* __restrict__ xm,
                                                   const double* __restrict__ Uext,
                                                   const double* __restrict__ Qext, double* __restrict__ Xd,
                                                   double* __restrict__ Fexp) {
  using P = Phys<EQ, D>;
  constexpr int NV = P::NV;
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int e = blockIdx.y;
  if (n >= g.K) return;
  const int s = (int)(n % g.nsub);
  const int f = g.xface[e], q = e - g.fptr[f];
  const int64_t m = nbr_elem(g, n, s, f);
  const int e2 = g.fptr[g.nface[s][f]] + g.perm[s][f][q];
  const bool left = g.left[s][f];
  double um[NV], uo[NV], qm[D * NV], qo[D * NV];
#pragma unroll
  for (int a = 0; a < NV; ++a) {
    um[a] = Uext[((int64_t)e * NV + a) * g.Kp + n];
    uo[a] = Uext[((int64_t)e2 * NV + a) * g.Kp + m];
  }
  if constexpr (P::VISC) {
#pragma unroll
    for (int d = 0; d < D; ++d)
#pragma unroll
      for (int a = 0; a < NV; ++a) {
        qm[d * NV + a] = Qext[(((int64_t)e * D + d) * NV + a) * g.Kp + n];
        qo[d * NV + a] = Qext[(((int64_t)e2 * D + d) * NV + a) * g.Kp + m];
      }
  }
  const ExtMetric mt = xm[s * g.next + e];
  const double nl[3] = {mt.n0, mt.n1, mt.n2};
  double F[NV];
  if (left) P::common_flux(ph, um, uo, qm, qo, nl, F);
  else P::common_flux(ph, uo, um, qo, qm, nl, F);
  const double sc = left ? mt.s : -mt.s;
#pragma unroll
  for (int a = 0; a < NV; ++a) Xd[((int64_t)e * NV + a) * g.Kp + n] = sc * F[a];
  if (Fexp)  // O28 export: the common flux this element applies at its ext point e
#pragma unroll
    for (int a = 0; a < NV; ++a) Fexp[((int64_t)e * NV + a) * g.Kp + n] = F[a];
}

// k = -R~/detJ ; mode 0: out = k ; RK4 stage update otherwise (3-register form):
//  stage 0: ACC = U + dt/6 k, Us = U + dt/2 k     stage 1: ACC += dt/3 k, Us = U + dt/2 k
//  stage 2: ACC += dt/3 k, Us = U + dt k           stage 3: U = ACC + dt/6 k
__global__ void __launch_bounds__(256) k_rk(GeomDev g, const double* __restrict__ R, int rows, int stage,
                                            double dt, double* __restrict__ out, double* __restrict__ U,
                                            double* __restrict__ Us, double* __restrict__ ACC) {
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  if (n >= g.K || r >= rows) return;
  const int s = (int)(n % g.nsub);
  const int64_t i = (int64_t)r * g.Kp + n;
  const double k = -R[i] / g.detJ[s];
  switch (stage) {
    case -1: out[i] = k; break;
    case 0: {
      const double u = U[i];
      ACC[i] = fma(dt / 6.0, k, u);
      Us[i] = fma(0.5 * dt, k, u);
    } break;
    case 1: {
      ACC[i] = fma(dt / 3.0, k, ACC[i]);
      Us[i] = fma(0.5 * dt, k, U[i]);
    } break;
    case 2: {
      ACC[i] = fma(dt / 3.0, k, ACC[i]);
      Us[i] = fma(dt, k, U[i]);
    } break;
    default: U[i] = fma(dt / 6.0, k, ACC[i]); break;
  }
}

// divergence check: first element with a non-finite value (or rho/p <= 0)
template <int EQ, int D>
__global__ void k_check(GeomDev g, PhysDev ph, const double* __restrict__ U, int nsol,
                        unsigned long long* bad) {
  using P = Phys<EQ, D>;
  constexpr int NV = P::NV;
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= g.K) return;
  for (int sp = 0; sp < nsol; ++sp) {
    double u[NV];
    bool ok = true;
    for (int a = 0; a < NV; ++a) {
      u[a] = U[((int64_t)sp * NV + a) * g.Kp + n];
      ok = ok && isfinite(u[a]);
    }
    if constexpr (NV > 1) {
      double kin = 0.0;
      for (int d = 0; d < D; ++d) kin += u[1 + d] * u[1 + d];
      const double p = (ph.gamma - 1.0) * (u[D + 1] - 0.5 * kin / u[0]);
      ok = ok && u[0] > 0.0 && p > 0.0;
    }
    if (!ok) {
      atomicMin(bad, (unsigned long long)n);
      return;
    }
  }
}

// halo: pack / unpack trace entries (row, col) x N_V  <->  contiguous buffer
// trace element (point row, variable v, column col): [row][v][Kt] (tensor path) or
// point-major [row][Kt][v] (simplex path)
__device__ __forceinline__ int64_t trace_at(int64_t row, int v, int64_t col, int64_t Kt, int NV, bool pm) {
  return pm ? (row * Kt + col) * NV + v : (row * NV + v) * Kt + col;
}

__global__ void k_halo_pack(const double* __restrict__ T, int64_t Kt, int NV, const int32_t* __restrict__ row,
                            const int32_t* __restrict__ col, int64_t n, double* __restrict__ buf, bool pm) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * NV) return;
  const int64_t k = idx / NV;
  const int v = (int)(idx % NV);
  buf[idx] = T[trace_at(row[k], v, col[k], Kt, NV, pm)];
}

__global__ void k_halo_unpack(double* __restrict__ T, int64_t Kt, int NV, const int32_t* __restrict__ row,
                              const int32_t* __restrict__ col, int64_t n, const double* __restrict__ buf, bool pm) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * NV) return;
  const int64_t k = idx / NV;
  const int v = (int)(idx % NV);
  T[trace_at(row[k], v, col[k], Kt, NV, pm)] = buf[idx];
}

// far-field ghost entries (boundaries with the limiting values of the
// initial field): the U traces of the ghost element = the far-field state, its published
// viscous normal flux = 0 (f^v of a constant state)
__global__ void k_ff_fill(double* __restrict__ Tu0, double* __restrict__ Tu1, double* __restrict__ Tg, int64_t Kt,
                          int NV, const int32_t* __restrict__ row, const int32_t* __restrict__ col, int64_t n,
                          const double* __restrict__ state, bool pm) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * NV) return;
  const int64_t k = idx / NV;
  const int v = (int)(idx % NV);
  const int64_t at = trace_at(row[k], v, col[k], Kt, NV, pm);
  Tu0[at] = state[v];
  Tu1[at] = state[v];
  if (Tg) Tg[at] = 0.0;
}

// sum of the per-tile diagnostics partials in a fixed order (one block), scaled:
// out = { <rho v.v>, 2 mu <S:S>, -<p div v> }
__global__ void k_diag_final(const double* __restrict__ part, int64_t ntile, double inv_vol, double mu,
                             double* __restrict__ out) {
  __shared__ double red[3][256];
  double a[3] = {0.0, 0.0, 0.0};
  for (int64_t t = threadIdx.x; t < ntile; t += 256)
    for (int k = 0; k < 3; ++k) a[k] += part[3 * t + k];
  for (int k = 0; k < 3; ++k) red[k][threadIdx.x] = a[k];
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if ((int)threadIdx.x < h)
      for (int k = 0; k < 3; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = red[0][0] * inv_vol;
    out[1] = 2.0 * mu * red[1][0] * inv_vol;
    out[2] = -red[2][0] * inv_vol;
  }
}

// ------------------------------------------------------------------------ host side
struct OpHost {
  std::vector<int> ptr, col;
  std::vector<double> val;
  int rows, cols, nchunks;
};

static OpHost pack(const Mat& M) {
  OpHost o;
  o.rows = M.rows;
  o.cols = M.cols;
  o.nchunks = (M.rows + RB - 1) / RB;
  o.ptr.push_back(0);
  for (int ch = 0; ch < o.nchunks; ++ch) {
    for (int c = 0; c < M.cols; ++c) {
      bool nz = false;
      for (int r = ch * RB; r < std::min(M.rows, (ch + 1) * RB); ++r) nz = nz || M(r, c) != 0.0;
      if (!nz) continue;
      o.col.push_back(c);
      for (int r = ch * RB; r < (ch + 1) * RB; ++r) o.val.push_back(r < M.rows ? M(r, c) : 0.0);
    }
    o.ptr.push_back((int)o.col.size());
  }
  return o;
}

static size_t align256(size_t x) { return (x + 255) / 256 * 256; }

struct Plan {
  size_t off_uext, off_xg, off_q, off_qext, off_qu, off_xd, off_r, off_us, off_acc, off_ops, off_xm,
      off_bad, off_tu0, off_tu1, off_tg, off_sops, off_halo, halo_entries, off_ff, off_tiles, off_diag, off_cub,
      off_fuse, total;
  size_t ops_bytes;
};

static void build_ops(const Operators& O, int D, Mat ops[5]) {
  const RefElement& r = O.ref;
  int ns = r.nsol;
  ops[0] = O.M0;
  ops[1] = O.M12;
  // gradient G[(s,d)][ [C (next) ; U_u (nu)] ]
  Mat G(ns * D, r.next + r.nu);
  for (int s = 0; s < ns; ++s)
    for (int d = 0; d < D; ++d) {
      for (int e = 0; e < r.next; ++e) G(s * D + d, e) = O.M16(d * ns + s, e);
      for (int i = 0; i < r.nint; ++i) {
        double v = O.M15(d * ns + s, i);
        if (v != 0.0) G(s * D + d, r.next + r.int_u[i]) += v;
      }
    }
  ops[2] = G;
  // divergence Dv[s][ [D~ (next) ; F~_u (D nu, [d][u])] ]
  Mat Dv(ns, r.next + D * r.nu);
  for (int s = 0; s < ns; ++s) {
    for (int e = 0; e < r.next; ++e) Dv(s, e) = O.M14(s, e);
    for (int i = 0; i < r.nint; ++i) {
      double v = O.M13(s, i);
      if (v != 0.0) Dv(s, r.next + r.int_dir[i] * r.nu + r.int_u[i]) += v;
    }
  }
  ops[3] = Dv;
}

}  // namespace sdrt

using namespace sdrt;

enum KTag { T_M0 = 0, T_M12, T_CV, T_GRAD, T_METRIC, T_QEXT, T_QU, T_IFLUX, T_FFLUX, T_DIV, T_RK,
            T_TRACE, T_FA, T_FB, T_STRACE, T_SA, T_SB, T_FAB, T_NTAGS };
static const char* KTAG_NAMES[T_NTAGS] = {"interp_ext(M0)", "interp_int(M12)", "common_value", "gradient(M16|M15P)",
                                          "metric_grad", "grad_interp_ext(M5)", "grad_interp_int(M18)",
                                          "int_flux", "face_flux", "divergence(M14|M13M19P2)", "rk_update",
                                          "tensor_traces", "tensor_grad(A)", "tensor_stage(B)",
                                          "simplex_traces", "simplex_grad(A)", "simplex_stage(B)",
                                          "tensor_fused(A+B)"};

struct sdrt_ctx {
  bool timing = false;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
  std::vector<cudaEvent_t> pool;
  size_t pool_used = 0;
  GeomDev g;
  PhysDev ph;
  int eq, nd, nv, nsol, next, nu, nint;
  bool visc;
  double *Uext, *Xg, *Q, *Qext, *Qu, *Xd, *R, *Us, *ACC;
  ExtMetric* xm;
  unsigned long long* bad;
  OpDev op[4];
  int64_t launches = 0;
  // fused tensor-product path
  bool fused = false;
  int etype = 0, p = 0;
  TensorGeom tg;
  Line1D line;
  TensorTma tma;
  // interior / boundary tile lists (multi-rank overlap): tiles of tile_w elements
  int tile_w = 0, n_int = 0, n_bnd = 0;
  double* d_part = nullptr;  // diagnostics partial sums
  double* d_w = nullptr;     // solution-point quadrature weights w_r (App. B reading of l.2052)
  double diag_vol = 0.0;     // sum_e detJ_e sum_r w_r
  double* d_cub = nullptr;   // cubature of the diagnostics: B [ncub][nsol], then weights [ncub]
  int ncub = 0;              // 0: solution-point quadrature
  int nq1 = 0;               // tensor elements: cubature points per axis (1D factor stored after w)
  int cub_cap = 0;           // points reserved (the degree-10 rule)
  const int* d_tiles = nullptr;  // [n_int interior tiles][n_bnd boundary tiles]
  double* Tu[2] = {nullptr, nullptr};
  double* Tg = nullptr;
  int cur = 0;
  // fused simplex path
  bool sfused = false;
  SimplexOps sops;
  SimplexTma stma;
  // halo exchange
  bool needs_halo = false, loopback = false;
  int nslab = 0;
  int slab_peer[6], slab_d[6], slab_side[6];
  int64_t slab_off[7];        // entry offsets of each slab in the send/recv lists
  int32_t *h_srow = nullptr, *h_scol = nullptr, *h_rrow = nullptr, *h_rcol = nullptr;
  double* h_stage = nullptr;  // loopback staging buffer
  double* h_send = nullptr;   // NCCL exchange buffers (workspace)
  double* h_recv = nullptr;
  NcclComm* comm = nullptr;   // sdrt_ctx_attach_comm: the library exchanges through NCCL
  int64_t ff_n = 0;           // far-field ghost entries
  int32_t *ff_row = nullptr, *ff_col = nullptr;
  double* ff_state = nullptr;
  bool ff_pending = false;    // far-field entries not yet filled (sdrt_ctx_set_farfield)
  int rank = 0, nranks = 1;
  bool auto_halo = false;     // library performs the (loopback) exchange itself
  double* Fexp = nullptr;     // sdrt_face_flux: per-ext-point common flux export (residual only)
  // slab-pipelined stages (fused tensor path, one-sided flux publication, single rank):
  // the mesh is cut into `slabs` z-ranges; kernel A of slab k and kernel B of other
  // slabs run concurrently on two streams, ordered by per-slab events (fused_steps_slabs)
  int slabs = 0;
  // fused RK stage (tensor.cu kt_fused): kernel A + kernel B in one persistent launch
  bool fuse = false;
  FuseSched fsd{};
  int slab_tile[17] = {};     // first tile of slab k (slab_tile[slabs] = number of tiles)
  const int* d_iota = nullptr;  // tile ids 0 .. ntiles-1 (slab k = d_iota + slab_tile[k])
  cudaStream_t sA = nullptr, sB = nullptr;
  cudaEvent_t evA[16] = {}, evB[16] = {}, evStart = nullptr, evEnd = nullptr;
  // CUDA-graph replay of K-step runs (sdrt_ctx_set_graph): the launch sequence of one
  // sdrt_rk_step / sdrt_rk54_step call, captured on the library's own stream gst and
  // replayed while (U, dt, nsteps, integrator, trace buffer) repeat
  // default off: measured slower than the direct PDL launches on every config (c1 0.106 ->
  // 0.055, c2 18.2 -> 9.3, c3 33.4 -> 26.9 GDOF-stage/s: the programmatic overlap of
  // consecutive stage kernels is worth more than the saved launch calls)
  int graph_mode = 0;         // -1 auto (on below GRAPH_AUTO_DOF), 0 off, 1 on
  int64_t dof = 0;
  cudaStream_t gst = nullptr;
  cudaEvent_t gev[2] = {nullptr, nullptr};
  struct GraphEntry {  // one per starting trace buffer (an odd stage count flips it)
    cudaGraphExec_t exec = nullptr;
    double* U = nullptr;
    double dt = 0.0;
    int nsteps = -1, kind = -1, cur1 = 0;
    int64_t launches = 0;
  } gent[2];
};

// Dense operator in DMMA fragment order (simplex.cuh SOpF): rows padded to 8, columns
// to 4, frag[(m * kt + k) * 32 + lane] = M[8 m + lane / 4][4 k + lane % 4].
struct OpHostF {
  std::vector<double> frag;
  std::vector<unsigned> kmask;  // per m-tile, bit k: block (m, k) has a non-zero
  int rows, cols, mt, kt;
};

static OpHostF pack_frag(const Mat& M) {
  OpHostF o;
  o.rows = M.rows;
  o.cols = M.cols;
  o.mt = (M.rows + 7) / 8;
  o.kt = (M.cols + 3) / 4;
  if (o.kt > 32) throw std::runtime_error("internal: operator too wide for the k-step mask");
  o.frag.assign((size_t)o.mt * o.kt * 32, 0.0);
  o.kmask.assign(o.mt, 0u);
  for (int m = 0; m < o.mt; ++m)
    for (int k = 0; k < o.kt; ++k)
      for (int lane = 0; lane < 32; ++lane) {
        const int r = 8 * m + lane / 4, c = 4 * k + lane % 4;
        if (r < M.rows && c < M.cols) {
          o.frag[((size_t)m * o.kt + k) * 32 + lane] = M(r, c);
          if (M(r, c) != 0.0) o.kmask[m] |= 1u << k;
        }
      }
  return o;
}

// simplex operators: M0, M12, G = [M16 | M15 P] rows (s,d), M14, M13 M19 P2 (cols (d,u))
static void simplex_pack(const Operators& O, int D, std::vector<OpHostF>* out) {
  const RefElement& r = O.ref;
  int ns = r.nsol;
  Mat G(ns * D, r.next + r.nu);  // rows (d, s)
  for (int s2 = 0; s2 < ns; ++s2)
    for (int d = 0; d < D; ++d) {
      for (int e = 0; e < r.next; ++e) G(d * ns + s2, e) = O.M16(d * ns + s2, e);
      for (int i = 0; i < r.nint; ++i) {
        double v = O.M15(d * ns + s2, i);
        if (v != 0.0) G(d * ns + s2, r.next + r.int_u[i]) += v;
      }
    }
  Mat M13F(ns, D * r.nu);
  for (int s2 = 0; s2 < ns; ++s2)
    for (int i = 0; i < r.nint; ++i) {
      double v = O.M13(s2, i);
      if (v != 0.0) M13F(s2, r.int_dir[i] * r.nu + r.int_u[i]) += v;
    }
  if (O.scheme != 0) {
    // FR (l.400-413, gradient remark l.429-434): with Mc = div g (FR-SDRT: M14, FR-DG: the
    // DG lifting) and Mc_d = Mc n^_d, the gradient [Mc_d | Dsol_d - Mc_d M0] on [C; U] with
    // rows (d, s); the divergence Dsol - Mc (n^ . M0) on the solution-point fluxes F[d][s]
    // (columns (d, s)); the face lift Mc (kernel B)
    G = Mat(ns * D, r.next + ns);
    M13F = Mat(ns, ns * D);
    for (int s2 = 0; s2 < ns; ++s2)
      for (int d = 0; d < D; ++d) {
        for (int e = 0; e < r.next; ++e) G(d * ns + s2, e) = O.Mc(s2, e) * r.ext_normal[e][d];
        for (int q = 0; q < ns; ++q) {
          double gc = O.Dsol[d](s2, q), dv = O.Dsol[d](s2, q);
          for (int e = 0; e < r.next; ++e) {
            gc -= O.Mc(s2, e) * r.ext_normal[e][d] * O.M0(e, q);
            dv -= O.Mc(s2, e) * r.ext_normal[e][d] * O.M0(e, q);
          }
          G(d * ns + s2, r.next + q) = gc;
          M13F(s2, d * ns + q) = dv;
        }
      }
  }
  out->clear();
  out->push_back(pack_frag(O.M0));
  out->push_back(pack_frag(O.M12));
  out->push_back(pack_frag(G));
  out->push_back(pack_frag(O.scheme != 0 ? O.Mc : O.M14));
  out->push_back(pack_frag(M13F));
  // [M14 | M13 M19 P2] on [D~; F~] (inviscid kernel B: the whole divergence in one product)
  const Mat& Mf = O.scheme != 0 ? O.Mc : O.M14;
  Mat MF(ns, r.next + M13F.cols);
  for (int s2 = 0; s2 < ns; ++s2) {
    for (int e = 0; e < r.next; ++e) MF(s2, e) = Mf(s2, e);
    for (int j = 0; j < M13F.cols; ++j) MF(s2, r.next + j) = M13F(s2, j);
  }
  out->push_back(pack_frag(MF));
}

static int nvars(int eq, int D) { return (eq == SDRT_EQ_LINADV || eq == SDRT_EQ_LINADVDIFF) ? 1 : D + 2; }

// points of the diagnostics cubature exact to `degree` (refel.cpp cubature_interp)
static int cub_points(int etype, int D, int degree) {
  const int n = etype_tensor(etype) ? degree / 2 + 1 : (degree + D - 1) / 2 + 1;
  return D == 2 ? n * n : n * n * n;
}

// Which path a context runs: the fused tensor / simplex element kernels, or the generic
// operator path (unsupported element-degree-equation combinations, or the
// SDRT_FORCE_GENERIC=1 cross-check hook).  Decided before the workspace is planned so
// each path reserves only its own buffers.
enum PathKind { PATH_GENERIC = 0, PATH_TENSOR = 1, PATH_SIMPLEX = 2 };
static PathKind choose_path(const Mesh& m, const sdrt_physics* ph) {
  const char* fg = getenv("SDRT_FORCE_GENERIC");
  if (fg && fg[0] == '1') return PATH_GENERIC;
  if (etype_tensor(m.etype)) return tensor_supported(m.nd, m.p, ph->eq) ? PATH_TENSOR : PATH_GENERIC;
  if (m.etype == TRI || m.etype == TET) return simplex_supported(m.nd, m.p, ph->eq) ? PATH_SIMPLEX : PATH_GENERIC;
  return PATH_GENERIC;  // prisms
}

static Plan make_plan(const Mesh& m, const Operators& O, const sdrt_physics* ph, std::vector<OpHost>* packed) {
  const RefElement& r = O.ref;
  int D = m.nd, NV = nvars(ph->eq, D);
  bool visc = ph->eq == SDRT_EQ_LINADVDIFF || ph->eq == SDRT_EQ_NS;
  const bool gen = choose_path(m, ph) == PATH_GENERIC;
  size_t col = (size_t)NV * m.K_pad * sizeof(double);
  Plan p;
  size_t o = 0;
  // generic-path intermediates (Appendix-B products in HBM); none on the fused paths
  p.off_uext = o; o += gen ? align256(r.next * col) : 0;
  p.off_xg = o; o += gen ? align256((r.next + r.nu) * col) : 0;
  p.off_q = o; o += gen && visc ? align256((size_t)r.nsol * D * col) : 0;
  p.off_qext = o; o += gen && visc ? align256((size_t)r.next * D * col) : 0;
  p.off_qu = o; o += gen && visc ? align256((size_t)r.nu * D * col) : 0;
  p.off_xd = o; o += gen ? align256((r.next + (size_t)D * r.nu) * col) : 0;
  // R~ (generic) / R_int (fused, viscous), the RK stage register and accumulator
  p.off_r = o; o += align256((size_t)r.nsol * col);
  p.off_us = o; o += align256((size_t)r.nsol * col);
  p.off_acc = o; o += align256((size_t)r.nsol * col);
  Mat ops[5];
  build_ops(O, D, ops);
  size_t ob = 0;
  std::vector<OpHost> pk;
  for (int i = 0; i < (gen ? 4 : 0); ++i) {
    pk.push_back(pack(ops[i]));
    ob += align256(pk.back().ptr.size() * sizeof(int)) + align256(pk.back().col.size() * sizeof(int) + 4) +
          align256(pk.back().val.size() * sizeof(double) + 8);
  }
  p.off_ops = o; o += ob;
  p.ops_bytes = ob;
  p.off_xm = o; o += align256((size_t)m.nsub * r.next * sizeof(ExtMetric));
  p.off_bad = o; o += 256;
  size_t tb = gen ? 0 : align256((size_t)r.next * NV * m.Kt * sizeof(double));  // fused: trace arrays
  p.off_tu0 = o; o += tb;
  p.off_tu1 = o; o += tb;
  p.off_tg = o; o += tb;
  p.off_sops = o;
  if (choose_path(m, ph) == PATH_SIMPLEX) {
    std::vector<OpHostF> s4;
    simplex_pack(O, D, &s4);
    for (auto& h : s4) o += align256(h.frag.size() * sizeof(double)) + align256(h.kmask.size() * sizeof(unsigned) + 4);
  }
  // halo lists: send (row, col) and recv (row, col) int32 for all slabs, + a loopback
  // staging buffer of the same number of values, + the send / recv buffers of the
  // library's own NCCL exchange (sdrt_ctx_attach_comm)
  size_t ent = 0;
  for (const HaloSlab& S : m.slabs) ent += S.send_row.size();
  p.halo_entries = ent;
  p.off_halo = o;
  o += align256(ent * 4 * sizeof(int32_t)) + 3 * align256(ent * NV * sizeof(double));
  // far-field ghost entries (row, col) int32 + the far-field state
  p.off_ff = o;
  o += align256(m.ff_row.size() * 2 * sizeof(int32_t)) + 256;
  // interior / boundary tile lists of the fused paths (tiles of >= 4 elements)
  p.off_tiles = o;
  o += align256(((size_t)m.K / 4 + 2) * sizeof(int32_t));
  // TGV diagnostics: per-tile partial sums (3 per tile of >= 8 elements) + weights w
  p.off_diag = o;
  o += align256((3 * ((size_t)m.K / 8 + 2) + r.nsol + 8) * sizeof(double));
  // degree-10 cubature of the diagnostics (l.2075): interpolation matrix + weights
  p.off_cub = o;
  o += align256(((size_t)cub_points(r.etype, r.nd, 10) * (r.nsol + 1) + 64) * sizeof(double));  // + 1D factor
  // fused RK stage (tensor path, tiles of >= 8 elements): job list (2 per tile),
  // dependency table (FUSE_DEPS per tile), per-tile flags, 4 counters
  p.off_fuse = o;
  if (etype_tensor(m.etype) && ph->eq == EQ_NS) o += align256((((size_t)m.K / 8 + 2) * (3 + FUSE_DEPS) + 4) * sizeof(int32_t));
  p.total = o;
  if (packed) *packed = pk;
  return p;
}

// Diagnostics rule: degree 0 = the solution points (weights w), else the cubature exact
// to `degree` (refel.cpp cubature_interp) uploaded into the reserved area (synchronous).
static void set_diag_rule(sdrt_ctx* c, int etype, int degree) {
  if (degree == 0) {
    c->ncub = 0;
    return;
  }
  std::vector<double> w;
  Mat B;
  cubature_interp(etype, c->p, degree, w, B);
  if ((int)w.size() > c->cub_cap || B.cols != c->nsol) throw std::runtime_error("cubature larger than reserved");
  CUDA_OK(cudaMemcpy(c->d_cub, B.a.data(), B.a.size() * sizeof(double), cudaMemcpyHostToDevice));
  CUDA_OK(cudaMemcpy(c->d_cub + B.a.size(), w.data(), w.size() * sizeof(double), cudaMemcpyHostToDevice));
  c->ncub = (int)w.size();
  c->nq1 = 0;
  if (etype_tensor(etype)) {  // the 1D factor, after the weights (sum-factorised application)
    std::vector<double> B1;
    cubature_interp_1d(c->p, degree, B1);
    if (B1.size() > 64) throw std::runtime_error("cubature 1D factor larger than reserved");
    CUDA_OK(cudaMemcpy(c->d_cub + B.a.size() + w.size(), B1.data(), B1.size() * sizeof(double),
                       cudaMemcpyHostToDevice));
    c->nq1 = degree / 2 + 1;
  }
}

extern "C" {

size_t sdrt_ctx_workspace_bytes(const sdrt_mesh* m, const sdrt_operators* o, const sdrt_physics* ph) {
  if (!m || !o || !ph) return 0;
  try {
    return make_plan(m->m, o->o, ph, nullptr).total;
  } catch (...) {
    return 0;
  }
}

sdrt_status sdrt_ctx_create(const sdrt_mesh* mm, const sdrt_operators* oo, const sdrt_physics* ph, void* d_ws,
                            size_t ws_bytes, void* stream, sdrt_ctx** out) {
  if (!mm || !oo || !ph || !out || !d_ws) {
    set_error("null argument");
    return SDRT_E_INVALID_ARG;
  }
  const Mesh& m = mm->m;
  const Operators& O = oo->o;
  if (m.etype != O.ref.etype || m.p != O.ref.p) {
    set_error("mesh and operators disagree on element type / degree");
    return SDRT_E_INVALID_ARG;
  }
  if (ph->eq < 0 || ph->eq > 3) {
    set_error("unknown equation");
    return SDRT_E_INVALID_ARG;
  }
  if (m.slabs.size() > 0 && !((etype_tensor(m.etype) || m.etype == TRI || m.etype == TET))) {
    set_error("halo exchange needs the fused paths");
    return SDRT_E_UNSUPPORTED;
  }
  SDRT_TRY({
    std::vector<OpHost> pk;
    Plan p = make_plan(m, O, ph, &pk);
    if (ws_bytes < p.total || ((uintptr_t)d_ws % 256)) {
      set_error("workspace too small or not 256-byte aligned");
      return SDRT_E_WORKSPACE;
    }
    cudaStream_t st = (cudaStream_t)stream;
    char* base = (char*)d_ws;
    auto* c = new sdrt_ctx;
    const RefElement& r = O.ref;
    c->eq = ph->eq;
    c->nd = m.nd;
    c->nv = nvars(ph->eq, m.nd);
    c->nsol = r.nsol;
    c->dof = (int64_t)m.K * r.nsol * c->nv;
    c->next = r.next;
    c->nu = r.nu;
    c->nint = r.nint;
    c->visc = ph->eq == SDRT_EQ_LINADVDIFF || ph->eq == SDRT_EQ_NS;
    c->Uext = (double*)(base + p.off_uext);
    c->Xg = (double*)(base + p.off_xg);
    c->Q = (double*)(base + p.off_q);
    c->Qext = (double*)(base + p.off_qext);
    c->Qu = (double*)(base + p.off_qu);
    c->Xd = (double*)(base + p.off_xd);
    c->R = (double*)(base + p.off_r);
    c->Us = (double*)(base + p.off_us);
    c->ACC = (double*)(base + p.off_acc);
    c->xm = (ExtMetric*)(base + p.off_xm);
    c->bad = (unsigned long long*)(base + p.off_bad);
    // operators (generic path)
    size_t o = p.off_ops;
    for (int i = 0; i < (int)pk.size(); ++i) {
      OpHost& h = pk[i];
      int* dptr = (int*)(base + o);
      CUDA_OK(cudaMemcpyAsync(dptr, h.ptr.data(), h.ptr.size() * sizeof(int), cudaMemcpyHostToDevice, st));
      o += align256(h.ptr.size() * sizeof(int));
      int* dcol = (int*)(base + o);
      if (!h.col.empty())
        CUDA_OK(cudaMemcpyAsync(dcol, h.col.data(), h.col.size() * sizeof(int), cudaMemcpyHostToDevice, st));
      o += align256(h.col.size() * sizeof(int) + 4);
      double* dval = (double*)(base + o);
      if (!h.val.empty())
        CUDA_OK(cudaMemcpyAsync(dval, h.val.data(), h.val.size() * sizeof(double), cudaMemcpyHostToDevice, st));
      o += align256(h.val.size() * sizeof(double) + 8);
      c->op[i] = OpDev{h.rows, h.cols, h.nchunks, dptr, dcol, dval};
    }
    // geometry
    GeomDev& g = c->g;
    std::memset(&g, 0, sizeof(g));
    g.nd = m.nd;
    g.nsub = m.nsub;
    g.nfaces = r.nfaces;
    g.nfp = r.nfp;
    g.next = r.next;
    for (int d = 0; d < 3; ++d) {
      g.Nloc[d] = m.Nloc[d];
      g.Nglob[d] = m.Nglob[d];
      g.offset[d] = m.offset[d];
    }
    g.K = m.K;
    g.Kp = m.K_pad;
    for (int f = 0; f <= r.nfaces; ++f) g.fptr[f] = (int16_t)r.face_ptr[f];
    for (int e = 0; e < r.next; ++e) g.xface[e] = (int8_t)r.ext_face[e];
    for (int s = 0; s < m.nsub; ++s) {
      g.detJ[s] = m.detJ[s];
      for (int k = 0; k < 9; ++k) g.Jinv[s][k] = m.Jinv[s][k];
      for (int f = 0; f < r.nfaces; ++f) {
        const FaceLink& L = m.link[s * r.nfaces + f];
        for (int d = 0; d < 3; ++d) g.off[s][f][d] = (int8_t)L.off[d];
        g.nshape[s][f] = (int8_t)L.nshape;
        g.nface[s][f] = (int8_t)L.nface;
        g.left[s][f] = (int8_t)L.left;
        for (int q = 0; q < (int)L.perm.size(); ++q) g.perm[s][f][q] = (int8_t)L.perm[q];
      }
    }
    g.Kt = m.Kt;
    for (int d = 0; d < 3; ++d) {
      g.halo[d] = m.halo[d];
      g.gbase[d][0] = m.gbase[d][0];
      g.gbase[d][1] = m.gbase[d][1];
    }
    // halo plan
    c->nslab = (int)m.slabs.size();
    c->needs_halo = c->nslab > 0;
    c->loopback = c->needs_halo;
    c->auto_halo = false;
    c->rank = m.rank;
    c->nranks = m.nranks;
    {
      int64_t ofs = 0;
      std::vector<int32_t> lists;
      std::vector<int32_t> sr, sc, rr, rcol;
      for (int i = 0; i < c->nslab; ++i) {
        const HaloSlab& S = m.slabs[i];
        c->slab_peer[i] = S.peer;
        c->slab_d[i] = S.d;
        c->slab_side[i] = S.side;
        c->slab_off[i] = ofs;
        if (S.peer != m.rank) c->loopback = false;
        if (S.send_row.size() != S.recv_row.size()) throw std::runtime_error("internal: halo list sizes differ");
        sr.insert(sr.end(), S.send_row.begin(), S.send_row.end());
        sc.insert(sc.end(), S.send_col.begin(), S.send_col.end());
        rr.insert(rr.end(), S.recv_row.begin(), S.recv_row.end());
        rcol.insert(rcol.end(), S.recv_col.begin(), S.recv_col.end());
        ofs += (int64_t)S.send_row.size();
      }
      c->slab_off[c->nslab] = ofs;
      c->auto_halo = c->loopback;
      if (ofs > 0) {
        int32_t* hl = (int32_t*)(base + p.off_halo);
        c->h_srow = hl;
        c->h_scol = hl + ofs;
        c->h_rrow = hl + 2 * ofs;
        c->h_rcol = hl + 3 * ofs;
        CUDA_OK(cudaMemcpyAsync(c->h_srow, sr.data(), ofs * 4, cudaMemcpyHostToDevice, st));
        CUDA_OK(cudaMemcpyAsync(c->h_scol, sc.data(), ofs * 4, cudaMemcpyHostToDevice, st));
        CUDA_OK(cudaMemcpyAsync(c->h_rrow, rr.data(), ofs * 4, cudaMemcpyHostToDevice, st));
        CUDA_OK(cudaMemcpyAsync(c->h_rcol, rcol.data(), ofs * 4, cudaMemcpyHostToDevice, st));
        c->h_stage = (double*)(base + p.off_halo + align256(ofs * 4 * sizeof(int32_t)));
        c->h_send = (double*)((char*)c->h_stage + align256(ofs * c->nv * sizeof(double)));
        c->h_recv = (double*)((char*)c->h_send + align256(ofs * c->nv * sizeof(double)));
        CUDA_OK(cudaStreamSynchronize(st));
      }
    }
    c->ff_n = (int64_t)m.ff_row.size();
    if (c->ff_n > 0) {
      c->ff_row = (int32_t*)(base + p.off_ff);
      c->ff_col = c->ff_row + c->ff_n;
      c->ff_state = (double*)(base + p.off_ff + align256(c->ff_n * 2 * sizeof(int32_t)));
      CUDA_OK(cudaMemcpyAsync(c->ff_row, m.ff_row.data(), c->ff_n * 4, cudaMemcpyHostToDevice, st));
      CUDA_OK(cudaMemcpyAsync(c->ff_col, m.ff_col.data(), c->ff_n * 4, cudaMemcpyHostToDevice, st));
      c->ff_pending = true;
    }
    std::vector<ExtMetric> xm(m.nsub * r.next);
    for (int i = 0; i < m.nsub * r.next; ++i)
      xm[i] = ExtMetric{m.sscale[i], m.nleft[i][0], m.nleft[i][1], m.nleft[i][2]};
    CUDA_OK(cudaMemcpyAsync(c->xm, xm.data(), xm.size() * sizeof(ExtMetric), cudaMemcpyHostToDevice, st));
    // zero the intermediate buffers (padding columns stay finite)
    CUDA_OK(cudaMemsetAsync(base, 0, p.off_ops, st));
    c->ph = PhysDev{{ph->c[0], ph->c[1], ph->c[2]}, ph->mu, ph->gamma, ph->Pr, ph->beta, ph->eta,
                    ph->mu * ph->gamma / ((ph->gamma - 1.0) * ph->Pr)};
    // fused tensor-product path (default for quad/hex; SDRT_FORCE_GENERIC=1 selects the
    // generic operator path, a test hook for cross-checking the two)
    c->etype = m.etype;
    c->p = m.p;
    const PathKind path = choose_path(m, ph);
    c->fused = path == PATH_TENSOR;
    if (c->fused && (int64_t)r.next * c->nv * m.Kt >= (int64_t(1) << 31)) {
      // the tensor kernels index trace arrays [N_ext][N_V][K_t] in 32-bit arithmetic
      delete c;
      set_error("unsupported: mesh too large for the fused tensor kernels (N_ext N_V K_trace >= 2^31; "
                "hex p=3 Navier-Stokes: K < 4.4e6 elements per rank)");
      return SDRT_E_UNSUPPORTED;
    }
    if (c->fused) {
      TensorGeom& t = c->tg;
      std::memset(&t, 0, sizeof(t));
      for (int d = 0; d < 3; ++d) t.N[d] = m.Nloc[d];
      t.K = m.K;
      t.Kp = m.K_pad;
      t.Kt = m.Kt;
      for (int d = 0; d < 3; ++d) {
        t.halo[d] = m.halo[d];
        t.gbase[d][0] = m.gbase[d][0];
        t.gbase[d][1] = m.gbase[d][1];
      }
      t.detJ = m.detJ[0];
      {
        // one-sided flux publication (tensor.cu publish_F): NS with beta = +1/2 (the
        // left element holds every input of a face's common flux) on meshes without
        // far-field ghosts (a ghost is never a kernel-A element); SDRT_OSF=0 disables it
        const char* ev = std::getenv("SDRT_OSF");
        t.osf = ph->eq == EQ_NS && ph->beta == 0.5 && m.ff_row.empty() && !(ev && ev[0] == '0');
      }
      for (int d = 0; d < 3; ++d) {
        t.jinv[d] = d < m.nd ? m.Jinv[0][d * 3 + d] : 0.0;
        t.sface[d] = d < m.nd ? m.detJ[0] * t.jinv[d] : 0.0;
      }
      for (int f = 0; f < r.nfaces; ++f)
        for (int q = 0; q < r.nfp; ++q)
          if (m.link[f].perm[q] != q) throw std::runtime_error("internal: tensor face permutation not identity");
      Line1D& L = c->line;
      std::memset(&L, 0, sizeof(L));
      int n = m.p + 1;
      if (O.scheme == 0) {
        for (int i = 0; i < n; ++i) {
          L.Iend[0][i] = O.M0(0 * r.nfp + 0, i);
          L.Iend[1][i] = O.M0(1 * r.nfp + 0, i);
          for (int a = 0; a < m.p; ++a) L.Iint[a][i] = O.M12(a, i);
          L.Dfl[i][0] = -O.M14(i, 0 * r.nfp + 0);
          L.Dfl[i][m.p + 1] = O.M14(i, 1 * r.nfp + 0);
          for (int a = 0; a < m.p; ++a) L.Dfl[i][a + 1] = O.M13(i, a);
        }
      } else {
        // FR on the first x-line: the "internal points" are the n solution points
        // (Iint = I); end coefficients -div g of the x = -1 face and div g of x = +1
        // (signs as the SDRT M14 columns); interior coefficients Dsol - end x Iend
        L.fr = 1;
        for (int i = 0; i < n; ++i) {
          L.Iend[0][i] = O.M0(0 * r.nfp + 0, i);
          L.Iend[1][i] = O.M0(1 * r.nfp + 0, i);
          L.Iint[i][i] = 1.0;
        }
        for (int i = 0; i < n; ++i) {
          const double e0 = -O.Mc(i, 0 * r.nfp + 0), e1 = O.Mc(i, 1 * r.nfp + 0);
          L.Dfl[i][0] = e0;
          L.Dfl[i][n + 1] = e1;
          for (int j = 0; j < n; ++j) L.Dfl[i][j + 1] = O.Dsol[0](i, j) - e0 * L.Iend[0][j] - e1 * L.Iend[1][j];
        }
      }
      {
        // composite gradient operator per axis (tensor.cuh Line1D::Gq), long double
        const int NI = L.fr ? n : m.p;
        const long double wl = 0.5L - (long double)ph->beta, wr = 0.5L + (long double)ph->beta;
        for (int d = 0; d < m.nd; ++d) {
          const long double jd = t.jinv[d];
          for (int i = 0; i < n; ++i) {
            for (int j = 0; j < n; ++j) {
              long double a = (long double)L.Dfl[i][0] * wr * L.Iend[0][j] + (long double)L.Dfl[i][NI + 1] * wl * L.Iend[1][j];
              for (int k = 0; k < NI; ++k) a += (long double)L.Dfl[i][k + 1] * L.Iint[k][j];
              L.Gq[d][i][j] = (double)(jd * a);
            }
            L.H0[d][i] = (double)(jd * L.Dfl[i][0] * wl);
            L.H1[d][i] = (double)(jd * L.Dfl[i][NI + 1] * wr);
          }
        }
      }
      tensor_tma_init(&c->tma, m.nd, m.p, ph->eq, m.K_pad);
      c->Tu[0] = (double*)(base + p.off_tu0);
      c->Tu[1] = (double*)(base + p.off_tu1);
      c->Tg = (double*)(base + p.off_tg);
    }
    c->sfused = path == PATH_SIMPLEX;
    if (O.scheme != 0 && !c->fused && !c->sfused) {
      delete c;
      set_error("unsupported: FR schemes run on the fused element kernels");
      return SDRT_E_UNSUPPORTED;
    }
    c->sops.fr = O.scheme != 0;
    if ((m.slabs.size() > 0 || !m.ff_row.empty()) && !c->fused && !c->sfused) {
      delete c;
      set_error("unsupported: halo exchange and far-field boundaries are implemented for the fused paths only");
      return SDRT_E_UNSUPPORTED;
    }
    if (c->sfused) {
      std::vector<OpHostF> s4;
      simplex_pack(O, m.nd, &s4);
      size_t so = p.off_sops;
      SOpF* dst[6] = {&c->sops.M0, &c->sops.M12, &c->sops.G, &c->sops.M14, &c->sops.M13F, &c->sops.M14F};
      for (int i = 0; i < 6; ++i) {
        OpHostF& h = s4[i];
        double* dval = (double*)(base + so);
        CUDA_OK(cudaMemcpyAsync(dval, h.frag.data(), h.frag.size() * sizeof(double), cudaMemcpyHostToDevice, st));
        so += align256(h.frag.size() * sizeof(double));
        unsigned* dmask = (unsigned*)(base + so);
        CUDA_OK(cudaMemcpyAsync(dmask, h.kmask.data(), h.kmask.size() * sizeof(unsigned), cudaMemcpyHostToDevice, st));
        so += align256(h.kmask.size() * sizeof(unsigned) + 4);
        const unsigned full = h.kt >= 32 ? ~0u : (1u << h.kt) - 1u;
        bool dense = true;
        for (unsigned mk : h.kmask) dense = dense && mk == full;
        *dst[i] = SOpF{h.rows, h.cols, h.mt, h.kt, dval, dense ? nullptr : dmask};  // dense: no mask reads
      }
      {
        // one-sided flux publication (simplex.cu ks_stage_osf): as for the tensor path
        const char* ev = std::getenv("SDRT_OSF");
        c->g.osf = ph->eq == EQ_NS && ph->beta == 0.5 && m.ff_row.empty() && O.scheme == 0 && !(ev && ev[0] == '0');
      }
      simplex_tma_init(&c->stma, m.nd, m.p, ph->eq, m.K_pad);
      c->Tu[0] = (double*)(base + p.off_tu0);
      c->Tu[1] = (double*)(base + p.off_tu1);
      c->Tg = (double*)(base + p.off_tg);
      CUDA_OK(cudaStreamSynchronize(st));
    }
    // diagnostics buffers: weights w and the quadrature volume
    c->d_w = (double*)(base + p.off_diag);
    c->d_part = c->d_w + ((r.nsol + 7) / 8) * 8;
    CUDA_OK(cudaMemcpyAsync(c->d_w, O.w.data(), r.nsol * sizeof(double), cudaMemcpyHostToDevice, st));
    {
      double sw = 0.0, sd = 0.0;
      for (int i = 0; i < r.nsol; ++i) sw += O.w[i];
      for (int64_t e = 0; e < m.K; ++e) sd += m.detJ[e % m.nsub];
      c->diag_vol = sw * sd;
    }
    c->d_cub = (double*)(base + p.off_cub);
    c->cub_cap = cub_points(r.etype, r.nd, 10);
    CUDA_OK(cudaStreamSynchronize(st));
    if (r.etype != PRI) set_diag_rule(c, r.etype, 10);  // diagnostics run on the fused paths (no prisms)
    // interior / boundary tile lists for the overlapped multi-rank stage:
    // a tile is interior if none of its elements lies in a pattern layer next to a
    // partition face (ghost neighbours only occur there)
    if ((c->fused || c->sfused) && (m.halo[0] || m.halo[1] || m.halo[2])) {
      c->tile_w = c->fused ? tensor_tile_width(m.nd, m.p, ph->eq) : simplex_tile_width(m.nd, m.p, ph->eq);
      const int ntile = (int)((m.K + c->tile_w - 1) / c->tile_w);
      std::vector<int> inner, bnd;
      for (int tl = 0; tl < ntile; ++tl) {
        bool b = false;
        for (int j = 0; j < c->tile_w && !b; ++j) {
          const int64_t e = (int64_t)tl * c->tile_w + j;
          if (e >= m.K) break;
          int64_t pat = e / m.nsub;
          for (int d = 0; d < m.nd; ++d) {
            const int cd = (int)(pat % m.Nloc[d]);
            pat /= m.Nloc[d];
            if (m.halo[d] && (cd == 0 || cd == m.Nloc[d] - 1)) b = true;
          }
        }
        (b ? bnd : inner).push_back(tl);
      }
      c->n_int = (int)inner.size();
      c->n_bnd = (int)bnd.size();
      inner.insert(inner.end(), bnd.begin(), bnd.end());
      int* dt = (int*)(base + p.off_tiles);
      if (!inner.empty())
        CUDA_OK(cudaMemcpyAsync(dt, inner.data(), inner.size() * sizeof(int), cudaMemcpyHostToDevice, st));
      c->d_tiles = dt;
    }
    // slab pipeline (fused_steps_slabs): 3-D fused tensor path with one-sided flux
    // publication on one rank; slab k = whole z-planes [z_k, z_k+1) (every neighbour across
    // an x or y face lies in the same slab, across a z face in slab k +- 1 mod S);
    // SDRT_SLABS = S (4..16; default 0 = off: measured on c4, S = 4 / 8 / 16 give 27.4 / 24.9 /
    // 24.1 GDOF-stage/s against 31.9 single-stream -- kernel A already fills every SM
    // (two CTAs), the concurrent B CTAs displace it, and the 2S launches and events per
    // stage add their own gaps)
    if (c->fused && c->tg.osf && m.nd == 3 && !(m.halo[0] || m.halo[1] || m.halo[2])) {
      const char* ev = std::getenv("SDRT_SLABS");
      int S = ev ? std::atoi(ev) : 0;
      const int E = tensor_tile_width(m.nd, m.p, ph->eq);
      const int64_t plane = (int64_t)m.Nloc[0] * m.Nloc[1] * m.nsub;
      if (S > m.Nloc[2]) S = m.Nloc[2];
      if (S >= 4 && S <= 16 && plane % E == 0) {
        const int64_t tpp = plane / E;  // tiles per z-plane
        const int ntile = (int)(tpp * m.Nloc[2]);
        std::vector<int> iota(ntile);
        for (int i = 0; i < ntile; ++i) iota[i] = i;
        int* di = (int*)(base + p.off_tiles);
        CUDA_OK(cudaMemcpyAsync(di, iota.data(), iota.size() * sizeof(int), cudaMemcpyHostToDevice, st));
        CUDA_OK(cudaStreamSynchronize(st));
        c->d_iota = di;
        c->slabs = S;
        for (int k = 0; k <= S; ++k) c->slab_tile[k] = (int)(tpp * ((int64_t)m.Nloc[2] * k / S));
        CUDA_OK(cudaStreamCreateWithFlags(&c->sA, cudaStreamNonBlocking));
        CUDA_OK(cudaStreamCreateWithFlags(&c->sB, cudaStreamNonBlocking));
        for (int k = 0; k < S; ++k) {
          CUDA_OK(cudaEventCreateWithFlags(&c->evA[k], cudaEventDisableTiming));
          CUDA_OK(cudaEventCreateWithFlags(&c->evB[k], cudaEventDisableTiming));
        }
        CUDA_OK(cudaEventCreateWithFlags(&c->evStart, cudaEventDisableTiming));
        CUDA_OK(cudaEventCreateWithFlags(&c->evEnd, cudaEventDisableTiming));
      }
    }
    // fused RK stage (kt_fused): 3-D fused tensor NS path with one-sided flux publication
    // on one periodic rank, SDRT operators; SDRT_FUSE=1 enables it, SDRT_FUSE_LAG = the lag
    // in tiles between a B job's last dependency and its place in the job list (default
    // 2 x the resident CTAs)
    if (c->fused && c->tg.osf && !c->line.fr && !(m.halo[0] || m.halo[1] || m.halo[2]) && c->slabs == 0) {
      const char* ev = std::getenv("SDRT_FUSE");
      const int E = tensor_tile_width(m.nd, m.p, ph->eq);
      const int nctas = (ev && ev[0] == '1' && E >= 8) ? tensor_fuse_ctas(m.nd, m.p, ph->eq) : 0;
      if (nctas > 0) {
        const char* el = std::getenv("SDRT_FUSE_LAG");
        const int lag = el ? std::atoi(el) : 2 * nctas;
        std::vector<int> jobs, deps;
        if (tensor_fuse_plan(m.nd, m.Nloc, m.K, E, lag, &jobs, &deps)) {
          const int64_t nt = (m.K + E - 1) / E;
          int* fb = (int*)(base + p.off_fuse);
          CUDA_OK(cudaMemcpyAsync(fb, jobs.data(), jobs.size() * sizeof(int), cudaMemcpyHostToDevice, st));
          CUDA_OK(cudaMemcpyAsync(fb + 2 * nt, deps.data(), deps.size() * sizeof(int), cudaMemcpyHostToDevice, st));
          int* ctr = fb + 2 * nt + FUSE_DEPS * nt;
          CUDA_OK(cudaMemsetAsync(ctr, 0, (4 + nt) * sizeof(int), st));
          c->fsd.jobs = fb;
          c->fsd.deps = fb + 2 * nt;
          c->fsd.ctr = ctr;
          c->fsd.flags = (unsigned*)(ctr + 4);
          c->fsd.njobs = (int)jobs.size();
          c->fuse = true;
          CUDA_OK(cudaStreamSynchronize(st));
        }
      }
    }
    CUDA_OK(cudaStreamSynchronize(st));  // host vectors go out of scope
    *out = c;
    return SDRT_OK;
  })
}

void sdrt_ctx_destroy(sdrt_ctx* c) {
  if (!c) return;
  for (auto& ge : c->gent)
    if (ge.exec) cudaGraphExecDestroy(ge.exec);
  if (c->gst) {
    cudaEventDestroy(c->gev[0]);
    cudaEventDestroy(c->gev[1]);
    cudaStreamDestroy(c->gst);
  }
  for (auto e : c->pool) cudaEventDestroy(e);
  if (c->slabs > 0) {
    for (int k = 0; k < c->slabs; ++k) {
      cudaEventDestroy(c->evA[k]);
      cudaEventDestroy(c->evB[k]);
    }
    cudaEventDestroy(c->evStart);
    cudaEventDestroy(c->evEnd);
    cudaStreamDestroy(c->sA);
    cudaStreamDestroy(c->sB);
  }
  if (c->comm) nccl_comm_destroy(c->comm);
  delete c;
}

sdrt_status sdrt_ctx_set_graph(sdrt_ctx* c, int mode) {
  if (!c || mode < -1 || mode > 1) {
    set_error("invalid argument: mode -1 (auto), 0 (off) or 1 (on)");
    return SDRT_E_INVALID_ARG;
  }
  c->graph_mode = mode;
  return SDRT_OK;
}

sdrt_status sdrt_ctx_set_timing(sdrt_ctx* c, int enable) {
  if (!c) {
    set_error("null ctx");
    return SDRT_E_INVALID_ARG;
  }
  c->timing = enable != 0;
  c->ev.clear();
  c->pool_used = 0;
  return SDRT_OK;
}

sdrt_status sdrt_ctx_kernel_times(sdrt_ctx* c, int max_tags, char* names, double* ms, int64_t* counts,
                                  int* ntags) {
  if (!c || !ms || !counts || !ntags) {
    set_error("null argument");
    return SDRT_E_INVALID_ARG;
  }
  SDRT_TRY({
    for (auto& e : c->ev) CUDA_OK(cudaEventSynchronize(e.second.second));
    int n = std::min(max_tags, (int)T_NTAGS);
    for (int t = 0; t < n; ++t) {
      ms[t] = 0.0;
      counts[t] = 0;
      if (names) {
        std::strncpy(names + 64 * t, KTAG_NAMES[t], 63);
        names[64 * t + 63] = 0;
      }
    }
    for (auto& e : c->ev) {
      float v = 0.f;
      CUDA_OK(cudaEventElapsedTime(&v, e.second.first, e.second.second));
      if (e.first < n) {
        ms[e.first] += v;
        counts[e.first] += 1;
      }
    }
    *ntags = n;
    c->ev.clear();
    c->pool_used = 0;
    return SDRT_OK;
  })
}
int64_t sdrt_ctx_last_launches(const sdrt_ctx* c) { return c ? c->launches : -1; }

}  // extern "C"

namespace sdrt {

static cudaEvent_t get_event(sdrt_ctx* c) {
  if (c->pool_used == c->pool.size()) {
    cudaEvent_t e;
    CUDA_OK(cudaEventCreate(&e));
    c->pool.push_back(e);
  }
  return c->pool[c->pool_used++];
}

// RAII marker: records a start/stop event pair around one launch when timing is on
struct Mark {
  sdrt_ctx* c;
  cudaStream_t st;
  int tag;
  cudaEvent_t a = nullptr;
  Mark(sdrt_ctx* c_, cudaStream_t st_, int tag_) : c(c_), st(st_), tag(tag_) {
    if (c->timing) {
      a = get_event(c);
      CUDA_OK(cudaEventRecord(a, st));
    }
    c->launches++;
  }
  ~Mark() {
    if (c->timing) {
      cudaEvent_t b = get_event(c);
      cudaEventRecord(b, st);
      c->ev.push_back({tag, {a, b}});
    }
  }
};

static void apply(sdrt_ctx* c, int tag, const OpDev& M, const double* X, double* Y, int64_t W, cudaStream_t st) {
  dim3 grid((unsigned)((W + 255) / 256), (unsigned)M.nchunks);
  Mark mk(c, st, tag);
  k_apply<<<grid, 256, 0, st>>>(M, X, Y, W);
}

template <int EQ, int D>
static void residual_impl(sdrt_ctx* c, const double* U, int stage, double dt, double* out, double* Ubase,
                          cudaStream_t st) {
  constexpr int NV = Phys<EQ, D>::NV;
  const GeomDev& g = c->g;
  const int64_t W = (int64_t)NV * g.Kp;
  const unsigned gx = (unsigned)((g.K + 255) / 256);
  apply(c, T_M0, c->op[0], U, c->Uext, W, st);                                  // U_ext = M0 U
  apply(c, T_M12, c->op[1], U, c->Xg + (size_t)c->next * W, W, st);             // U_u = M12 U
  if constexpr (Phys<EQ, D>::VISC) {
    {
      Mark mk(c, st, T_CV);
      k_common_value<NV><<<dim3(gx, c->next), 256, 0, st>>>(g, c->ph, c->Uext, c->Xg);
    }
    apply(c, T_GRAD, c->op[2], c->Xg, c->Q, W, st);                             // Q~ = G [C; U_u]
    {
      Mark mk(c, st, T_METRIC);
      k_metric_grad<D, NV><<<dim3(gx, c->nsol), 256, 0, st>>>(g, c->Q, c->nsol);
    }
    apply(c, T_QEXT, c->op[0], c->Q, c->Qext, (int64_t)D * W, st);              // Q_ext = M5 Q
    apply(c, T_QU, c->op[1], c->Q, c->Qu, (int64_t)D * W, st);                  // Q_u = M18 Q
  }
  {
    Mark mk(c, st, T_IFLUX);
    k_int_flux<EQ, D><<<dim3(gx, c->nu), 256, 0, st>>>(g, c->ph, c->Xg + (size_t)c->next * W, c->Qu, c->Xd,
                                                        c->nu, c->next);
  }
  {
    Mark mk(c, st, T_FFLUX);
    k_face_flux<EQ, D><<<dim3(gx, c->next), 256, 0, st>>>(g, c->ph, c->xm, c->Uext, c->Qext, c->Xd,
                                                                             c->Fexp);
  }
  apply(c, T_DIV, c->op[3], c->Xd, c->R, W, st);                                 // R~ = Dv [D~; F~_u]
  {
    Mark mk(c, st, T_RK);
    k_rk<<<dim3(gx, c->nsol * NV), 256, 0, st>>>(g, c->R, c->nsol * NV, stage, dt, out, Ubase, c->Us, c->ACC);
  }
}

template <int EQ, int D>
static bool check_impl(sdrt_ctx* c, const double* U, cudaStream_t st, int64_t* bad_elem) {
  unsigned long long init = ~0ull, host = 0;
  CUDA_OK(cudaMemcpyAsync(c->bad, &init, sizeof(init), cudaMemcpyHostToDevice, st));
  k_check<EQ, D><<<(unsigned)((c->g.K + 255) / 256), 256, 0, st>>>(c->g, c->ph, U, c->nsol, c->bad);
  CUDA_OK(cudaMemcpyAsync(&host, c->bad, sizeof(host), cudaMemcpyDeviceToHost, st));
  CUDA_OK(cudaStreamSynchronize(st));
  *bad_elem = host == ~0ull ? -1 : (int64_t)host;
  return host == ~0ull;
}

static double* trace_buf(sdrt_ctx* c, int which) { return which == 0 ? c->Tu[c->cur] : c->Tg; }

static void halo_pack(sdrt_ctx* c, int which, double* buf, cudaStream_t st) {
  const int64_t n = c->slab_off[c->nslab];
  if (n == 0) return;
  const int64_t tot = n * c->nv;
  k_halo_pack<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(trace_buf(c, which), c->g.Kt, c->nv, c->h_srow,
                                                              c->h_scol, n, buf, c->sfused);
  c->launches++;
}

static void halo_unpack(sdrt_ctx* c, int which, const double* buf, cudaStream_t st) {
  const int64_t n = c->slab_off[c->nslab];
  if (n == 0) return;
  const int64_t tot = n * c->nv;
  k_halo_unpack<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(trace_buf(c, which), c->g.Kt, c->nv, c->h_rrow,
                                                                c->h_rcol, n, buf, c->sfused);
  c->launches++;
}

// loopback: every slab's peer is this rank; slab (d, s) receives what slab (d, 1-s) sent
static void halo_loopback(sdrt_ctx* c, int which, cudaStream_t st) {
  if (!c->needs_halo) return;
  halo_pack(c, which, c->h_stage, st);
  for (int i = 0; i < c->nslab; ++i) {
    int j = -1;
    for (int k = 0; k < c->nslab; ++k)
      if (c->slab_d[k] == c->slab_d[i] && c->slab_side[k] == 1 - c->slab_side[i]) j = k;
    const int64_t n = c->slab_off[i + 1] - c->slab_off[i];
    if (n != c->slab_off[j + 1] - c->slab_off[j]) throw std::runtime_error("internal: loopback slab sizes");
    const int64_t tot = n * c->nv;
    k_halo_unpack<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
        trace_buf(c, which), c->g.Kt, c->nv, c->h_rrow + c->slab_off[i], c->h_rcol + c->slab_off[i], n,
        c->h_stage + c->slab_off[j] * c->nv, c->sfused);
    c->launches++;
  }
}

static void fused_traces(sdrt_ctx* c, const double* U, cudaStream_t st) {
  {
    Mark mk(c, st, T_TRACE);
    tensor_launch_traces(c->nd, c->p, c->eq, c->tg, c->line, &c->tma, U, c->Tu[c->cur], st);
  }
  if (c->auto_halo) halo_loopback(c, 0, st);
}

static void fused_stage(sdrt_ctx* c, const double* Uin, double* U, int stage, double dt, double* out,
                        cudaStream_t st) {
  TensorBufs b;
  b.Uin = Uin;
  b.U = U;
  b.Us = c->Us;
  b.ACC = c->ACC;
  b.out = out;
  b.Tu = c->Tu[c->cur];
  b.Tu_next = c->Tu[c->cur ^ 1];
  b.Tg = c->Tg;
  b.Rv = c->R;
  b.Fexp = stage < 0 ? c->Fexp : nullptr;
  if (c->fuse && stage >= 0 && !c->auto_halo) {
    {
      Mark mk(c, st, T_FAB);
      tensor_launch_fused(c->nd, c->p, c->eq, c->tg, c->line, c->ph, &c->tma, b, stage, dt, c->fsd, st);
    }
    c->cur ^= 1;
    return;
  }
  if (c->visc) {
    {
      Mark mk(c, st, T_FA);
      tensor_launch_grad(c->nd, c->p, c->eq, c->tg, c->line, c->ph, &c->tma, b, st);
    }
    if (c->auto_halo) halo_loopback(c, 1, st);
  }
  {
    Mark mk(c, st, T_FB);
    tensor_launch_flux(c->nd, c->p, c->eq, c->tg, c->line, c->ph, &c->tma, b, stage, dt, st);
  }
  if (stage >= 0) {
    c->cur ^= 1;
    if (c->auto_halo) halo_loopback(c, 0, st);
  }
}

// Slab-pipelined RK stages (fused tensor path, one-sided flux publication, one rank).
// Per stage, kernel A of slab k runs on stream sA and kernel B of slab k on stream sB;
// the dependencies of one stage on the previous are exactly
//   A(s, k) after B(s-1, k) and B(s-1, k+1)   (its stage input, its +z neighbours' traces)
//   B(s, k) after A(s, k) and A(s, k-1)       (R_int, its -z neighbours' common fluxes)
// (indices mod S; the same per-element arithmetic as fused_stage, so the result is bitwise
// the unsplit one).  Stream order supplies the lower slab of each pair, one event the
// other: A(s, k) waits for evB[k+1] (evB[S-1] for the last slab), B(s, k) for evA[k]
// (evA[S-1] for slab 0, whose -z neighbours are the last slab).  The write-after-read
// hazards on the double-buffered traces, R_int and the published fluxes are covered by
// the same chain for S >= 4.  While slab k's B streams from HBM, later
// slabs' A (compute-bound) run on the other SMs.
static void fused_steps_slabs(sdrt_ctx* c, double* U, double dt, int nsteps, const int* stages, int nst,
                              cudaStream_t st) {
  const int S = c->slabs;
  CUDA_OK(cudaEventRecord(c->evStart, st));
  CUDA_OK(cudaStreamWaitEvent(c->sA, c->evStart, 0));
  CUDA_OK(cudaStreamWaitEvent(c->sB, c->evStart, 0));
  bool first = true;
  for (int step = 0; step < nsteps; ++step) {
    for (int si = 0; si < nst; ++si) {
      const int stage = stages[si];
      TensorBufs b;
      b.Uin = (stage == 0 || stage >= RK54_STAGE0) ? U : c->Us;
      b.U = U;
      b.Us = c->Us;
      b.ACC = c->ACC;
      b.out = nullptr;
      b.Tu = c->Tu[c->cur];
      b.Tu_next = c->Tu[c->cur ^ 1];
      b.Tg = c->Tg;
      b.Rv = c->R;
      b.Fexp = nullptr;
      for (int k = 0; k < S; ++k) {
        if (!first) CUDA_OK(cudaStreamWaitEvent(c->sA, c->evB[k + 1 < S ? k + 1 : S - 1], 0));
        TensorGeom tgp = c->tg;
        tgp.tiles = c->d_iota + c->slab_tile[k];
        tgp.ntiles = c->slab_tile[k + 1] - c->slab_tile[k];
        {
          Mark mk(c, c->sA, T_FA);
          tensor_launch_grad(c->nd, c->p, c->eq, tgp, c->line, c->ph, &c->tma, b, c->sA);
        }
        CUDA_OK(cudaEventRecord(c->evA[k], c->sA));
      }
      for (int k = 0; k < S; ++k) {
        CUDA_OK(cudaStreamWaitEvent(c->sB, c->evA[k == 0 ? S - 1 : k], 0));
        TensorGeom tgp = c->tg;
        tgp.tiles = c->d_iota + c->slab_tile[k];
        tgp.ntiles = c->slab_tile[k + 1] - c->slab_tile[k];
        {
          Mark mk(c, c->sB, T_FB);
          tensor_launch_flux(c->nd, c->p, c->eq, tgp, c->line, c->ph, &c->tma, b, stage, dt, c->sB);
        }
        CUDA_OK(cudaEventRecord(c->evB[k], c->sB));
      }
      c->cur ^= 1;
      first = false;
    }
  }
  CUDA_OK(cudaEventRecord(c->evEnd, c->sB));
  CUDA_OK(cudaStreamWaitEvent(st, c->evEnd, 0));
}

// Replay of a K-step run as one CUDA graph (latency-bound small meshes: hundreds of
// few-microsecond launches per call).  The run's launch sequence is captured once on the
// library stream gst (joined to the caller's stream by events, so capture works whatever
// stream the caller passes, including the legacy default stream) and replayed while the
// call repeats with the same state pointer, dt, step count, integrator and trace buffer;
// the graph holds exactly the kernels a direct call launches (PDL edges included).
constexpr int64_t GRAPH_AUTO_DOF = int64_t(1) << 22;

template <class F>
static bool graph_run(sdrt_ctx* c, int kind, double* U, double dt, int nsteps, cudaStream_t st, F&& enqueue) {
  const bool on = c->graph_mode == 1 || (c->graph_mode == -1 && c->dof < GRAPH_AUTO_DOF);
  if (!on || c->timing || c->comm || c->slabs > 0 || nsteps <= 0) return false;
  if (!c->gst) {
    CUDA_OK(cudaStreamCreateWithFlags(&c->gst, cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreateWithFlags(&c->gev[0], cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&c->gev[1], cudaEventDisableTiming));
  }
  sdrt_ctx::GraphEntry& ge = c->gent[c->cur & 1];
  const bool hit = ge.exec && ge.U == U && ge.dt == dt && ge.nsteps == nsteps && ge.kind == kind;
  CUDA_OK(cudaEventRecord(c->gev[0], st));
  CUDA_OK(cudaStreamWaitEvent(c->gst, c->gev[0], 0));
  if (!hit) {
    if (ge.exec) {
      CUDA_OK(cudaGraphExecDestroy(ge.exec));
      ge.exec = nullptr;
    }
    const int cur0 = c->cur;
    c->launches = 0;
    cudaGraph_t graph = nullptr;
    CUDA_OK(cudaStreamBeginCapture(c->gst, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue(c->gst);
    } catch (...) {
      cudaStreamEndCapture(c->gst, &graph);
      if (graph) cudaGraphDestroy(graph);
      c->cur = cur0;
      throw;
    }
    CUDA_OK(cudaStreamEndCapture(c->gst, &graph));
    const cudaError_t e = cudaGraphInstantiate(&ge.exec, graph, 0);
    cudaGraphDestroy(graph);
    CUDA_OK(e);
    ge.U = U;
    ge.dt = dt;
    ge.nsteps = nsteps;
    ge.kind = kind;
    ge.cur1 = c->cur;
    ge.launches = c->launches;
    c->cur = cur0;
  }
  CUDA_OK(cudaGraphLaunch(ge.exec, c->gst));
  c->cur = ge.cur1;
  c->launches = ge.launches;
  CUDA_OK(cudaEventRecord(c->gev[1], c->gst));
  CUDA_OK(cudaStreamWaitEvent(st, c->gev[1], 0));
  return true;
}

static void sfused_traces(sdrt_ctx* c, const double* U, cudaStream_t st) {
  {
    Mark mk(c, st, T_STRACE);
    simplex_launch_traces(c->nd, c->p, c->eq, c->g, c->sops, &c->stma, U, c->Tu[c->cur], st);
  }
  if (c->auto_halo) halo_loopback(c, 0, st);
}

static void sfused_stage(sdrt_ctx* c, const double* Uin, double* U, int stage, double dt, double* out,
                         cudaStream_t st) {
  SimplexBufs b;
  b.Uin = Uin;
  b.U = U;
  b.Us = c->Us;
  b.ACC = c->ACC;
  b.out = out;
  b.Tu = c->Tu[c->cur];
  b.Tu_next = c->Tu[c->cur ^ 1];
  b.Tg = c->Tg;
  b.Rint = c->R;
  b.xm = c->xm;
  b.Fexp = stage < 0 ? c->Fexp : nullptr;
  if (c->visc) {
    {
      Mark mk(c, st, T_SA);
      simplex_launch_grad(c->nd, c->p, c->eq, c->g, c->sops, c->ph, &c->stma, b, st);
    }
    if (c->auto_halo) halo_loopback(c, 1, st);
  }
  {
    Mark mk(c, st, T_SB);
    simplex_launch_flux(c->nd, c->p, c->eq, c->g, c->sops, c->ph, &c->stma, b, stage, dt, st);
  }
  if (stage >= 0) {
    c->cur ^= 1;
    if (c->auto_halo) halo_loopback(c, 0, st);
  }
}

// library-internal multi-rank stepping over NCCL (defined at the end of this file)
static void comm_steps(sdrt_ctx* c, double* U, double dt, int nsteps, const int* stages, int nstages, cudaStream_t st);
static void comm_residual(sdrt_ctx* c, const double* U, double* out, cudaStream_t st);
static bool comm_check(sdrt_ctx* c, const double* U, cudaStream_t st, int64_t* bad_elem);

typedef void (*ResFn)(sdrt_ctx*, const double*, int, double, double*, double*, cudaStream_t);
typedef bool (*ChkFn)(sdrt_ctx*, const double*, cudaStream_t, int64_t*);

static ResFn pick_res(int eq, int D) {
#define CASE(E, DD) \
  if (eq == E && D == DD) return residual_impl<E, DD>;
  CASE(0, 2) CASE(0, 3) CASE(1, 2) CASE(1, 3) CASE(2, 2) CASE(2, 3) CASE(3, 2) CASE(3, 3)
#undef CASE
  return nullptr;
}
static ChkFn pick_chk(int eq, int D) {
#define CASE(E, DD) \
  if (eq == E && D == DD) return check_impl<E, DD>;
  CASE(0, 2) CASE(0, 3) CASE(1, 2) CASE(1, 3) CASE(2, 2) CASE(2, 3) CASE(3, 2) CASE(3, 3)
#undef CASE
  return nullptr;
}

}  // namespace sdrt

extern "C" {

sdrt_status sdrt_residual(sdrt_ctx* c, const double* d_U, double* d_dUdt, void* stream) {
  if (!c || !d_U || !d_dUdt) {
    set_error("null argument");
    return SDRT_E_INVALID_ARG;
  }
  SDRT_TRY({
    c->launches = 0;
    cudaStream_t st = (cudaStream_t)stream;
    if (c->ff_pending) {
      set_error("far-field boundaries not set: call sdrt_ctx_set_farfield first");
      return SDRT_E_INVALID_ARG;
    }
    if (c->comm) {
      comm_residual(c, d_U, d_dUdt, st);
      CUDA_OK(cudaGetLastError());
      return SDRT_OK;
    }
    if (c->needs_halo && !c->auto_halo) {
      set_error("unsupported: multi-rank context without a communicator; call sdrt_ctx_attach_comm, or use "
                "the staged API (sdrt_stage_*) with sdrt_halo_pack/unpack");
      return SDRT_E_UNSUPPORTED;
    }
    if (c->fused) {
      fused_traces(c, d_U, st);
      fused_stage(c, d_U, nullptr, -1, 0.0, d_dUdt, st);
    } else if (c->sfused) {
      sfused_traces(c, d_U, st);
      sfused_stage(c, d_U, nullptr, -1, 0.0, d_dUdt, st);
    } else {
      pick_res(c->eq, c->nd)(c, d_U, -1, 0.0, d_dUdt, nullptr, st);
    }
    CUDA_OK(cudaGetLastError());
    return SDRT_OK;
  })
}

sdrt_status sdrt_face_flux(sdrt_ctx* c, const double* d_U, double* d_dUdt, double* d_F, void* stream) {
  if (!c || !d_F) {
    set_error("null argument");
    return SDRT_E_INVALID_ARG;
  }
  c->Fexp = d_F;
  const sdrt_status st = sdrt_residual(c, d_U, d_dUdt, stream);
  c->Fexp = nullptr;
  return st;
}

sdrt_status sdrt_rk_step(sdrt_ctx* c, double* d_U, double dt, int nsteps, int check_every, void* stream) {
  if (!c || !d_U || nsteps < 0) {
    set_error("invalid argument");
    return SDRT_E_INVALID_ARG;
  }
  SDRT_TRY({
    c->launches = 0;
    cudaStream_t st = (cudaStream_t)stream;
    if (c->ff_pending) {
      set_error("far-field boundaries not set: call sdrt_ctx_set_farfield first");
      return SDRT_E_INVALID_ARG;
    }
    if (c->comm) {
      static const int rk4[4] = {0, 1, 2, 3};
      for (int done = 0; done < nsteps;) {
        const int n = check_every > 0 ? std::min(check_every, nsteps - done) : nsteps - done;
        comm_steps(c, d_U, dt, n, rk4, 4, st);
        done += n;
        int64_t bad;
        if (check_every > 0 && !comm_check(c, d_U, st, &bad)) {
          char buf[200];
          snprintf(buf, sizeof buf, "diverged after step %d: %s", done,
                   bad >= 0 ? ("element " + std::to_string(bad) + " of this rank non-finite or non-physical").c_str()
                            : "non-finite or non-physical state on another rank");
          set_error(buf);
          return SDRT_E_DIVERGED;
        }
      }
      CUDA_OK(cudaGetLastError());
      return SDRT_OK;
    }
    if (c->needs_halo && !c->auto_halo) {
      set_error("unsupported: multi-rank context without a communicator; call sdrt_ctx_attach_comm, or use "
                "the staged API (sdrt_stage_*) with sdrt_halo_pack/unpack");
      return SDRT_E_UNSUPPORTED;
    }
    ResFn res = pick_res(c->eq, c->nd);
    if (check_every <= 0 &&
        graph_run(c, 4, d_U, dt, nsteps, st, [&](cudaStream_t gs) {
          if (c->fused) fused_traces(c, d_U, gs);
          if (c->sfused) sfused_traces(c, d_U, gs);
          for (int step = 0; step < nsteps; ++step)
            for (int s = 0; s < 4; ++s) {
              if (c->fused) fused_stage(c, s == 0 ? d_U : c->Us, d_U, s, dt, nullptr, gs);
              else if (c->sfused) sfused_stage(c, s == 0 ? d_U : c->Us, d_U, s, dt, nullptr, gs);
              else res(c, s == 0 ? d_U : c->Us, s, dt, nullptr, d_U, gs);
            }
        })) {
      CUDA_OK(cudaGetLastError());
      return SDRT_OK;
    }
    if (c->fused && nsteps > 0) fused_traces(c, d_U, st);
    if (c->sfused && nsteps > 0) sfused_traces(c, d_U, st);
    if (c->slabs > 0 && nsteps > 0) {
      static const int rk4[4] = {0, 1, 2, 3};
      for (int done = 0; done < nsteps;) {
        const int n = check_every > 0 ? std::min(check_every, nsteps - done) : nsteps - done;
        fused_steps_slabs(c, d_U, dt, n, rk4, 4, st);
        done += n;
        CUDA_OK(cudaGetLastError());
        int64_t bad;
        if (check_every > 0 && !pick_chk(c->eq, c->nd)(c, d_U, st, &bad)) {
          char buf[160];
          snprintf(buf, sizeof buf, "diverged: element %lld non-finite or non-physical after step %d",
                   (long long)bad, done);
          set_error(buf);
          return SDRT_E_DIVERGED;
        }
      }
      return SDRT_OK;
    }
    for (int step = 0; step < nsteps; ++step) {
      for (int s = 0; s < 4; ++s) {
        if (c->fused) fused_stage(c, s == 0 ? d_U : c->Us, d_U, s, dt, nullptr, st);
        else if (c->sfused) sfused_stage(c, s == 0 ? d_U : c->Us, d_U, s, dt, nullptr, st);
        else res(c, s == 0 ? d_U : c->Us, s, dt, nullptr, d_U, st);
      }
      CUDA_OK(cudaGetLastError());
      if (check_every > 0 && (step + 1) % check_every == 0) {
        int64_t bad;
        if (!pick_chk(c->eq, c->nd)(c, d_U, st, &bad)) {
          char buf[160];
          snprintf(buf, sizeof buf, "diverged: element %lld non-finite or non-physical after step %d",
                   (long long)bad, step + 1);
          set_error(buf);
          return SDRT_E_DIVERGED;
        }
      }
    }
    return SDRT_OK;
  })
}

sdrt_status sdrt_rk54_step(sdrt_ctx* c, double* d_U, double dt, int nsteps, int check_every, void* stream) {
  if (!c || !d_U || nsteps < 0) {
    set_error("invalid argument");
    return SDRT_E_INVALID_ARG;
  }
  if (!c->fused && !c->sfused) {
    set_error("unsupported: RK54 needs a fused path (tensor or simplex kernels)");
    return SDRT_E_UNSUPPORTED;
  }
  SDRT_TRY({
    c->launches = 0;
    cudaStream_t st = (cudaStream_t)stream;
    if (c->ff_pending) {
      set_error("far-field boundaries not set: call sdrt_ctx_set_farfield first");
      return SDRT_E_INVALID_ARG;
    }
    if (c->comm) {
      static const int rk54[5] = {RK54_STAGE0, RK54_STAGE0 + 1, RK54_STAGE0 + 2, RK54_STAGE0 + 3, RK54_STAGE0 + 4};
      for (int done = 0; done < nsteps;) {
        const int n = check_every > 0 ? std::min(check_every, nsteps - done) : nsteps - done;
        comm_steps(c, d_U, dt, n, rk54, 5, st);
        done += n;
        int64_t bad;
        if (check_every > 0 && !comm_check(c, d_U, st, &bad)) {
          set_error("diverged after step " + std::to_string(done) + " (RK54, multi-rank)");
          return SDRT_E_DIVERGED;
        }
      }
      CUDA_OK(cudaGetLastError());
      return SDRT_OK;
    }
    if (c->needs_halo && !c->auto_halo) {
      set_error("unsupported: multi-rank context without a communicator; call sdrt_ctx_attach_comm, or use "
                "the staged API (sdrt_stage_*) with sdrt_halo_pack/unpack");
      return SDRT_E_UNSUPPORTED;
    }
    if (check_every <= 0 &&
        graph_run(c, 5, d_U, dt, nsteps, st, [&](cudaStream_t gs) {
          if (c->fused) fused_traces(c, d_U, gs);
          if (c->sfused) sfused_traces(c, d_U, gs);
          for (int step = 0; step < nsteps; ++step)
            for (int s = 0; s < 5; ++s) {
              if (c->fused) fused_stage(c, d_U, d_U, RK54_STAGE0 + s, dt, nullptr, gs);
              else sfused_stage(c, d_U, d_U, RK54_STAGE0 + s, dt, nullptr, gs);
            }
        })) {
      CUDA_OK(cudaGetLastError());
      return SDRT_OK;
    }
    if (c->fused && nsteps > 0) fused_traces(c, d_U, st);
    if (c->sfused && nsteps > 0) sfused_traces(c, d_U, st);
    if (c->slabs > 0 && nsteps > 0) {
      static const int rk54[5] = {RK54_STAGE0, RK54_STAGE0 + 1, RK54_STAGE0 + 2, RK54_STAGE0 + 3, RK54_STAGE0 + 4};
      for (int done = 0; done < nsteps;) {
        const int n = check_every > 0 ? std::min(check_every, nsteps - done) : nsteps - done;
        fused_steps_slabs(c, d_U, dt, n, rk54, 5, st);
        done += n;
        CUDA_OK(cudaGetLastError());
        int64_t bad;
        if (check_every > 0 && !pick_chk(c->eq, c->nd)(c, d_U, st, &bad)) {
          set_error("diverged after step " + std::to_string(done) + " (RK54)");
          return SDRT_E_DIVERGED;
        }
      }
      return SDRT_OK;
    }
    for (int step = 0; step < nsteps; ++step) {
      for (int s = 0; s < 5; ++s) {
        if (c->fused) fused_stage(c, d_U, d_U, RK54_STAGE0 + s, dt, nullptr, st);
        else sfused_stage(c, d_U, d_U, RK54_STAGE0 + s, dt, nullptr, st);
      }
      CUDA_OK(cudaGetLastError());
      if (check_every > 0 && (step + 1) % check_every == 0) {
        int64_t bad;
        if (!pick_chk(c->eq, c->nd)(c, d_U, st, &bad)) {
          char buf[160];
          snprintf(buf, sizeof buf, "diverged: element %lld non-finite or non-physical after step %d",
                   (long long)bad, step + 1);
          set_error(buf);
          return SDRT_E_DIVERGED;
        }
      }
    }
    return SDRT_OK;
  })
}

sdrt_status sdrt_diagnostics_rule(sdrt_ctx* c, int degree) {
  if (!c || degree < 0 || degree > 10) {
    set_error("invalid argument: degree must be 0 (solution points) or 1..10");
    return SDRT_E_INVALID_ARG;
  }
  SDRT_TRY({
    set_diag_rule(c, c->etype, degree);
    return SDRT_OK;
  })
}

sdrt_status sdrt_diagnostics(sdrt_ctx* c, const double* d_U, double* d_out, void* stream) {
  if (!c || !d_U || !d_out) {
    set_error("invalid argument");
    return SDRT_E_INVALID_ARG;
  }
  if (c->eq != SDRT_EQ_NS || c->nd != 3 || (!c->fused && !c->sfused) || c->needs_halo) {
    set_error("unsupported: TGV diagnostics need a single-rank 3-D Navier-Stokes context on a fused path");
    return SDRT_E_UNSUPPORTED;
  }
  SDRT_TRY({
    cudaStream_t st = (cudaStream_t)stream;
    c->launches = 0;
    int64_t ntile;
    if (c->fused) {
      fused_traces(c, d_U, st);
      TensorBufs b{};
      b.Uin = d_U;
      b.Tu = c->Tu[c->cur];
      tensor_launch_diag(c->nd, c->p, c->tg, c->line, c->ph, &c->tma, b, c->ncub ? c->d_cub + (size_t)c->ncub * c->nsol : c->d_w,
                         c->ncub ? c->d_cub : nullptr, c->ncub, c->d_part, st,
                         c->ncub && c->nq1 && SDRT_DIAG_SF ? c->d_cub + (size_t)c->ncub * (c->nsol + 1) : nullptr,
                         c->nq1);
      ntile = (c->g.K + tensor_tile_width(c->nd, c->p, c->eq) - 1) / tensor_tile_width(c->nd, c->p, c->eq);
    } else {
      sfused_traces(c, d_U, st);
      SimplexBufs b{};
      b.Uin = d_U;
      b.Tu = c->Tu[c->cur];
      simplex_launch_diag(c->nd, c->p, c->g, c->sops, c->ph, &c->stma, b,
                          c->ncub ? c->d_cub + (size_t)c->ncub * c->nsol : c->d_w, c->ncub ? c->d_cub : nullptr, c->ncub,
                          c->d_part, st);
      ntile = (c->g.K + 7) / 8;
    }
    k_diag_final<<<1, 256, 0, st>>>(c->d_part, ntile, 1.0 / c->diag_vol, c->ph.mu, d_out);
    c->launches += 2;
    CUDA_OK(cudaGetLastError());
    return SDRT_OK;
  })
}

sdrt_status sdrt_halo_info(const sdrt_ctx* c, int* nslab, int* peer, int* d, int* side, int64_t* offset) {
  if (!c || !nslab) {
    set_error("null argument");
    return SDRT_E_INVALID_ARG;
  }
  *nslab = c->nslab;
  for (int i = 0; i < c->nslab; ++i) {
    if (peer) peer[i] = c->slab_peer[i];
    if (d) d[i] = c->slab_d[i];
    if (side) side[i] = c->slab_side[i];
  }
  if (offset)
    for (int i = 0; i <= c->nslab; ++i) offset[i] = c->slab_off[i] * c->nv;
  return SDRT_OK;
}

sdrt_status sdrt_halo_pack(sdrt_ctx* c, int which, double* d_send, void* stream) {
  if (!c || (which != 0 && which != 1) || (!d_send && c->needs_halo)) {
    set_error("invalid argument");
    return SDRT_E_INVALID_ARG;
  }
  SDRT_TRY({
    halo_pack(c, which, d_send, (cudaStream_t)stream);
    CUDA_OK(cudaGetLastError());
    return SDRT_OK;
  })
}

sdrt_status sdrt_halo_unpack(sdrt_ctx* c, int which, const double* d_recv, void* stream) {
  if (!c || (which != 0 && which != 1) || (!d_recv && c->needs_halo)) {
    set_error("invalid argument");
    return SDRT_E_INVALID_ARG;
  }
  SDRT_TRY({
    halo_unpack(c, which, d_recv, (cudaStream_t)stream);
    CUDA_OK(cudaGetLastError());
    return SDRT_OK;
  })
}

sdrt_status sdrt_stage_traces(sdrt_ctx* c, const double* d_U, void* stream) {
  if (!c || !d_U || (!c->fused && !c->sfused)) {
    set_error("invalid argument (staged API needs a fused path)");
    return SDRT_E_INVALID_ARG;
  }
  SDRT_TRY({
    c->launches = 0;
    bool ah = c->auto_halo;
    c->auto_halo = false;
    if (c->fused) fused_traces(c, d_U, (cudaStream_t)stream);
    else sfused_traces(c, d_U, (cudaStream_t)stream);
    c->auto_halo = ah;
    CUDA_OK(cudaGetLastError());
    return SDRT_OK;
  })
}

sdrt_status sdrt_stage_grad(sdrt_ctx* c, double* d_U, int stage, void* stream) {
  return sdrt_stage_grad_part(c, d_U, stage, 0, stream);
}

sdrt_status sdrt_stage_flux(sdrt_ctx* c, double* d_U, int stage, double dt, double* d_out, void* stream) {
  return sdrt_stage_flux_part(c, d_U, stage, dt, d_out, 0, stream);
}

}  // extern "C"

// stage codes accepted by the staged API (rk.cuh): -1, RK4 0..3, RK54 10..14
static bool stage_valid(int stage) {
  return (stage >= -1 && stage <= 3) || (stage >= RK54_STAGE0 && stage < RK54_STAGE0 + 5);
}

// geometry restricted to a tile subset: part 0 = all tiles, 1 = interior, 2 = boundary
static bool part_geom(sdrt_ctx* c, int part, TensorGeom* tg, GeomDev* g) {
  *tg = c->tg;
  *g = c->g;
  if (part == 0) return true;
  if (!c->d_tiles) {  // no partition faces: everything is interior
    if (part == 2) return false;
    return true;
  }
  const int* list = part == 1 ? c->d_tiles : c->d_tiles + c->n_int;
  const int n = part == 1 ? c->n_int : c->n_bnd;
  tg->tiles = g->tiles = list;
  tg->ntiles = g->ntiles = n;
  return n > 0;
}

extern "C" {

sdrt_status sdrt_stage_grad_part(sdrt_ctx* c, double* d_U, int stage, int part, void* stream) {
  if (!c || !d_U || !stage_valid(stage) || part < 0 || part > 2 || (!c->fused && !c->sfused)) {
    set_error("invalid argument");
    return SDRT_E_INVALID_ARG;
  }
  if (!c->visc) return SDRT_OK;
  SDRT_TRY({
    cudaStream_t st = (cudaStream_t)stream;
    const double* Uin = (stage <= 0 || stage >= RK54_STAGE0) ? d_U : c->Us;
    TensorGeom tgp;
    GeomDev gp;
    if (!part_geom(c, part, &tgp, &gp)) return SDRT_OK;
    if (c->fused) {
      TensorBufs b{};
      b.Uin = Uin;
      b.Tu = c->Tu[c->cur];
      b.Tg = c->Tg;
      b.Rv = c->R;
      Mark mk(c, st, T_FA);
      tensor_launch_grad(c->nd, c->p, c->eq, tgp, c->line, c->ph, &c->tma, b, st);
    } else {
      SimplexBufs b{};
      b.Uin = Uin;
      b.Tu = c->Tu[c->cur];
      b.Tg = c->Tg;
      b.Rint = c->R;
      b.xm = c->xm;
      Mark mk(c, st, T_SA);
      simplex_launch_grad(c->nd, c->p, c->eq, gp, c->sops, c->ph, &c->stma, b, st);
    }
    CUDA_OK(cudaGetLastError());
    return SDRT_OK;
  })
}

sdrt_status sdrt_stage_flux_part(sdrt_ctx* c, double* d_U, int stage, double dt, double* d_out, int part,
                                 void* stream) {
  if (!c || !d_U || !stage_valid(stage) || (stage == -1 && !d_out) || part < 0 || part > 2 ||
      (!c->fused && !c->sfused)) {
    set_error("invalid argument");
    return SDRT_E_INVALID_ARG;
  }
  SDRT_TRY({
    cudaStream_t st = (cudaStream_t)stream;
    const double* Uin = (stage <= 0 || stage >= RK54_STAGE0) ? d_U : c->Us;
    TensorGeom tgp;
    GeomDev gp;
    const bool any = part_geom(c, part, &tgp, &gp);
    // the trace double buffer flips once per stage: after the whole mesh (part 0) or
    // after the boundary part (part 2) of the overlapped sequence interior -> boundary
    const bool flip = stage >= 0 && part != 1;
    if (!any) {
      if (flip) c->cur ^= 1;
      return SDRT_OK;
    }
    if (c->fused) {
      TensorBufs b;
      b.Uin = Uin;
      b.U = d_U;
      b.Us = c->Us;
      b.ACC = c->ACC;
      b.out = d_out;
      b.Tu = c->Tu[c->cur];
      b.Tu_next = c->Tu[c->cur ^ 1];
      b.Tg = c->Tg;
      b.Rv = c->R;
      Mark mk(c, st, T_FB);
      tensor_launch_flux(c->nd, c->p, c->eq, tgp, c->line, c->ph, &c->tma, b, stage, dt, st);
    } else {
      SimplexBufs b;
      b.Uin = Uin;
      b.U = d_U;
      b.Us = c->Us;
      b.ACC = c->ACC;
      b.out = d_out;
      b.Tu = c->Tu[c->cur];
      b.Tu_next = c->Tu[c->cur ^ 1];
      b.Tg = c->Tg;
      b.Rint = c->R;
      b.xm = c->xm;
      Mark mk(c, st, T_SB);
      simplex_launch_flux(c->nd, c->p, c->eq, gp, c->sops, c->ph, &c->stma, b, stage, dt, st);
    }
    if (flip) c->cur ^= 1;
    CUDA_OK(cudaGetLastError());
    return SDRT_OK;
  })
}

}  // extern "C"

// ------------------------------------------------------------------------------------
// Multi-rank stepping inside the library: the U traces after the
// trace-producing kernel and, for viscous equations, the published viscous traces after
// kernel A are packed on the compute stream, exchanged by grouped ncclSend / ncclRecv
// on the library's comm stream (ordered by events), and unpacked into the ghost trace
// columns.  While an exchange is in flight the interior tiles (no ghost reads) run;
// the boundary tiles run after the unpack.  Per-element arithmetic is that of the
// single-rank kernels, so the partitioned result equals the single-rank one.
namespace sdrt {

static void check_status(sdrt_status s) {
  if (s != SDRT_OK) throw std::runtime_error(sdrt_last_error());
}

// pack `which` (0: U traces, 1: viscous traces) and post the exchange on the comm stream
static void comm_start(sdrt_ctx* c, int which, cudaStream_t st) {
  if (c->nslab == 0) return;
  halo_pack(c, which, c->h_send, st);
  NcclComm* cm = c->comm;
  CUDA_OK(cudaEventRecord(nccl_comm_event(cm, 0), st));
  CUDA_OK(cudaStreamWaitEvent(nccl_comm_stream(cm), nccl_comm_event(cm, 0), 0));
  const double* sb[6];
  double* rb[6];
  int64_t ns[6], nr[6];
  int ps[6], pr[6];
  for (int i = 0; i < c->nslab; ++i) {
    int j = -1;  // the slab that receives what the peer of slab i's opposite side sends
    for (int k = 0; k < c->nslab; ++k)
      if (c->slab_d[k] == c->slab_d[i] && c->slab_side[k] == 1 - c->slab_side[i]) j = k;
    if (j < 0) throw std::runtime_error("internal: halo slab without its opposite");
    // what I send from slab (d, side) lands in the peer's slab (d, 1-side); what I
    // receive in slab (d, 1-side) the peer there sent from its slab (d, side).  Every
    // rank posts in slab order, so NCCL's in-order matching per peer pair pairs them.
    sb[i] = c->h_send + c->slab_off[i] * c->nv;
    ns[i] = (c->slab_off[i + 1] - c->slab_off[i]) * c->nv;
    ps[i] = c->slab_peer[i];
    rb[i] = c->h_recv + c->slab_off[j] * c->nv;
    nr[i] = (c->slab_off[j + 1] - c->slab_off[j]) * c->nv;
    pr[i] = c->slab_peer[j];
  }
  nccl_exchange(cm, c->nslab, sb, ns, ps, rb, nr, pr);
  CUDA_OK(cudaEventRecord(nccl_comm_event(cm, 1), nccl_comm_stream(cm)));
}

// make the compute stream wait for the exchange and unpack into the ghost columns
static void comm_finish(sdrt_ctx* c, int which, cudaStream_t st) {
  if (c->nslab == 0) return;
  CUDA_OK(cudaStreamWaitEvent(st, nccl_comm_event(c->comm, 1), 0));
  halo_unpack(c, which, c->h_recv, st);
}

static void comm_steps(sdrt_ctx* c, double* U, double dt, int nsteps, const int* stages, int nstages,
                       cudaStream_t st) {
  if (nsteps <= 0) return;
  const bool ah = c->auto_halo;
  c->auto_halo = false;  // the staged calls must not run the loopback kernels
  const int64_t l0 = c->launches;
  check_status(sdrt_stage_traces(c, U, st));
  c->launches += l0;
  comm_start(c, 0, st);
  for (int step = 0; step < nsteps; ++step)
    for (int k = 0; k < nstages; ++k) {
      const int s = stages[k];
      if (c->visc) {
        check_status(sdrt_stage_grad_part(c, U, s, 1, st));  // interior || U-trace exchange
        comm_finish(c, 0, st);
        check_status(sdrt_stage_grad_part(c, U, s, 2, st));
        comm_start(c, 1, st);
        check_status(sdrt_stage_flux_part(c, U, s, dt, nullptr, 1, st));  // interior || g exchange
        comm_finish(c, 1, st);
      } else {
        check_status(sdrt_stage_flux_part(c, U, s, dt, nullptr, 1, st));
        comm_finish(c, 0, st);
      }
      check_status(sdrt_stage_flux_part(c, U, s, dt, nullptr, 2, st));
      comm_start(c, 0, st);  // traces of the new stage input
    }
  comm_finish(c, 0, st);
  c->auto_halo = ah;
}

static void comm_residual(sdrt_ctx* c, const double* U, double* out, cudaStream_t st) {
  const bool ah = c->auto_halo;
  c->auto_halo = false;
  double* Um = const_cast<double*>(U);  // stage -1 reads U only
  check_status(sdrt_stage_traces(c, U, st));
  comm_start(c, 0, st);
  comm_finish(c, 0, st);
  if (c->visc) {
    check_status(sdrt_stage_grad(c, Um, -1, st));
    comm_start(c, 1, st);
    comm_finish(c, 1, st);
  }
  check_status(sdrt_stage_flux(c, Um, -1, 0.0, out, st));
  c->auto_halo = ah;
}

// divergence check over all ranks: every rank learns whether any rank went bad
static bool comm_check(sdrt_ctx* c, const double* U, cudaStream_t st, int64_t* bad_elem) {
  int64_t local = -1;
  const bool ok = pick_chk(c->eq, c->nd)(c, U, st, &local);
  unsigned long long flag = ok ? ~0ull : 0ull, host = 0;
  CUDA_OK(cudaMemcpyAsync(c->bad + 1, &flag, sizeof(flag), cudaMemcpyHostToDevice, st));
  nccl_allreduce_min_u64(c->comm, c->bad + 1, st);
  CUDA_OK(cudaMemcpyAsync(&host, c->bad + 1, sizeof(host), cudaMemcpyDeviceToHost, st));
  CUDA_OK(cudaStreamSynchronize(st));
  *bad_elem = ok ? -1 : local;
  return host == ~0ull;
}

}  // namespace sdrt

extern "C" {

sdrt_status sdrt_comm_unique_id(uint8_t id[128]) {
  if (!id) {
    set_error("null argument");
    return SDRT_E_INVALID_ARG;
  }
  try {
    nccl_unique_id(id);
    return SDRT_OK;
  } catch (const std::exception& e) {
    set_error(e.what());
    return SDRT_E_NCCL;
  }
}

sdrt_status sdrt_ctx_attach_comm(sdrt_ctx* c, const uint8_t id[128], int rank, int nranks) {
  if (!c || !id || nranks < 1 || rank < 0 || rank >= nranks) {
    set_error("invalid argument");
    return SDRT_E_INVALID_ARG;
  }
  if (rank != c->rank || nranks != c->nranks) {
    set_error("communicator rank / size differ from the mesh partition's (sdrt_mesh_create rank, nranks)");
    return SDRT_E_INVALID_ARG;
  }
  if (!c->needs_halo || (!c->fused && !c->sfused)) {
    set_error("unsupported: the context has no halo slabs (single-rank mesh without sdrt_mesh_set_halo) or "
              "no fused path");
    return SDRT_E_UNSUPPORTED;
  }
  if (c->comm) {
    nccl_comm_destroy(c->comm);
    c->comm = nullptr;
  }
  try {
    c->comm = nccl_comm_create(id, rank, nranks);
    return SDRT_OK;
  } catch (const std::exception& e) {
    set_error(e.what());
    return SDRT_E_NCCL;
  }
}

}  // extern "C"

extern "C" sdrt_status sdrt_ctx_set_farfield(sdrt_ctx* c, const double* state, void* stream) {
  if (!c || !state) {
    set_error("null argument");
    return SDRT_E_INVALID_ARG;
  }
  if (c->ff_n == 0) {
    set_error("the mesh has no far-field boundaries (all axes periodic)");
    return SDRT_E_INVALID_ARG;
  }
  SDRT_TRY({
    cudaStream_t st = (cudaStream_t)stream;
    CUDA_OK(cudaMemcpyAsync(c->ff_state, state, c->nv * sizeof(double), cudaMemcpyHostToDevice, st));
    const int64_t tot = c->ff_n * c->nv;
    k_ff_fill<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(c->Tu[0], c->Tu[1], c->visc ? c->Tg : nullptr, c->g.Kt,
                                                             c->nv, c->ff_row, c->ff_col, c->ff_n, c->ff_state,
                                                             c->sfused);
    CUDA_OK(cudaGetLastError());
    CUDA_OK(cudaStreamSynchronize(st));  // the host state buffer may go away
    c->ff_pending = false;
    return SDRT_OK;
  })
}
