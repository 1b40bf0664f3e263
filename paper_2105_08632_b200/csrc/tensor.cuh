// Fused sum-factorised SDRT stage for tensor-product elements (quad/hex), sm_100a.
#pragma once
#include <cuda.h>  // CUtensorMap (TMA descriptors)
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "physics.cuh"

namespace sdrt {

constexpr int TMAXP = 4;  // max degree of the fused tensor path

// 1D line operators, extracted on the host from the App. B matrices (so the fused
// path applies exactly the operators the generic path does):
//   Iend[s][i] = ell_i(-1 / +1)              (M0 restricted to one line)
//   Iint[a][i] = ell_i(zeta_a)               (M12 restricted to one line)
//   Dfl[i][f]  = L_f'(g_i), f over the flux line {-1, zeta_1..zeta_p, +1}
//                (M13 columns are Dfl[.][1..p]; M14 = -Dfl[.][0] (x=-1), +Dfl[.][p+1] (x=+1);
//                 M16 = n . M14 = Dfl[.][0] / Dfl[.][p+1] for both ends)
//   FR schemes (Line1D::fr = 1): the "internal points" are the p+1
//   solution points (Iint = I), Dfl[.][1..p+1] = Dsol - Dfl[.][0] Iend[0] - Dfl[.][p+2]
//   Iend[1] (discontinuous-flux derivative minus its end values times the correction
//   derivatives), Dfl[.][0] / Dfl[.][p+2] = the correction derivatives -g_L', g_R'
//   (FR-SDRT: the SDRT end values; FR-DG: Radau).
//   Gq[d][i][j], H0[d][i], H1[d][i]: the gradient along axis d at solution point i of a
//   line (l.282-302) as ONE composite operator on the line's solution values and the two
//   neighbour traces: (2/h_d) Dfl . [C_-; Iint u; C_+] with C_- = wl nb_- + wr Iend0 u,
//   C_+ = wl Iend1 u + wr nb_+ (wl = 1/2 - beta, wr = 1/2 + beta), i.e.
//   q_i = sum_j Gq[d][i][j] u_j + H0[d][i] nb_- + H1[d][i] nb_+ (built on the host from the
//   operators above, beta and J^-T; the same linear map in fewer operations).
struct Line1D {
  double Iend[2][TMAXP + 1];
  double Iint[TMAXP + 1][TMAXP + 1];
  double Dfl[TMAXP + 1][TMAXP + 3];
  double Gq[3][TMAXP + 1][TMAXP + 1];
  double H0[3][TMAXP + 1], H1[3][TMAXP + 1];
  int fr;  // 0: SDRT (p internal flux points), 1: FR (p+1 solution points)
};

struct TensorGeom {
  int N[3];           // local patterns per axis
  int64_t K, Kp;
  int64_t Kt;         // trace row stride (K_pad + ghost columns)
  int halo[3];        // axis d exchanges through ghost slabs (multi-rank / loopback)
  int64_t gbase[3][2];  // first ghost column of slab (d, side)
  double jinv[3];     // 2 / h_d  (J^-T = diag)
  double detJ;        // prod h_d / 2
  double sface[3];    // detJ * 2 / h_d  (= detJ |J^-T n~| on faces normal to d)
  const int* tiles;   // optional tile list (interior / boundary subsets), nullptr = all tiles
  int ntiles;
  int osf;            // one-sided flux publication (NS, beta = 1/2, no far-field axis): kernel A
                      // publishes the whole common flux of its x_d = +1 faces (tensor.cu publish_F)
};
int tensor_tile_width(int D, int P, int eq);

struct TensorBufs {
  const double* Uin;  // stage input (U or Us)
  double* U;          // u_n register (ABI state)
  double* Us;         // stage register
  double* ACC;        // RK accumulator
  double* out;        // residual output (stage == -1)
  const double* Tu;   // traces of the stage input  [N_ext][N_V][Kp]
  double* Tu_next;    // traces of the stage output
  double* Tg;         // published viscous normal-flux traces [N_ext][N_V][Kp] (OSF: the common flux F)
  double* Rv;         // viscous internal-flux divergence M13 F~_v [N_sol][N_V][Kp] (kernel A -> B)
  double* Fexp = nullptr;  // optional (residual only): common flux F per own ext point [N_ext][N_V][Kp]
};

// TMA descriptors of the element-major state-like arrays [N_sol N_V rows][Kp] seen by
// the fused kernels: 2-D tiles of E elements x box_rows rows land in shared memory in
// the kernels' own [row][E] layout.  Encoded on the host per array pointer (cached).
struct TensorTma {
  int rows = 0, E = 0;
  int64_t Kp = 0;
  const void* ptr[8] = {};
  CUtensorMap map[8];
  int next = 0;
};
void tensor_tma_init(TensorTma* t, int D, int P, int eq, int64_t Kp);

// Launchers (tensor.cu).  stage: -1 residual, 0..3 RK4 stages.
void tensor_launch_traces(int D, int P, int eq, const TensorGeom& g, const Line1D& L, TensorTma* tma,
                          const double* U, double* Tu, cudaStream_t st);
// kernel A (viscous equations only): gradient + published viscous normal-flux traces
void tensor_launch_grad(int D, int P, int eq, const TensorGeom& g, const Line1D& L, const PhysDev& ph,
                        TensorTma* tma, const TensorBufs& b, cudaStream_t st);
// kernel B: fluxes, divergence, RK update, new traces
void tensor_launch_flux(int D, int P, int eq, const TensorGeom& g, const Line1D& L, const PhysDev& ph,
                        TensorTma* tma, const TensorBufs& b, int stage, double dt, cudaStream_t st);
bool tensor_supported(int D, int P, int eq);

// Fused RK stage (kernel A + kernel B in ONE persistent launch; one-sided flux
// publication, one rank, periodic, SDRT; tensor.cu kt_fused).  CTAs take jobs in the
// order of a host-built list: every tile's A job in tile order, and each tile's B job
// after the A jobs of the tiles it reads (its own R_int, its left neighbours' published
// fluxes) plus a lag, so a B job rarely waits and reads R_int back from L2.
constexpr int FUSE_DEPS = 8;  // max tiles a B job depends on
struct FuseSched {
  const int* jobs;   // [njobs] tile << 1 | (1: B job)
  const int* deps;   // [ntiles][FUSE_DEPS] tiles whose A job the tile's B job reads (-1: none)
  int* ctr;          // [4]: next job, CTAs done, launch epoch (zeroed once)
  unsigned* flags;   // [ntiles]: epoch of the tile's last finished A job (zeroed once)
  int njobs;
};
// job list + dependency table (false: a tile depends on more than FUSE_DEPS tiles)
bool tensor_fuse_plan(int D, const int N[3], int64_t K, int E, int lag, std::vector<int>* jobs,
                      std::vector<int>* deps);
// whether the fused stage kernel exists for (D, P, eq) and its persistent grid size
int tensor_fuse_ctas(int D, int P, int eq);
void tensor_launch_fused(int D, int P, int eq, const TensorGeom& g, const Line1D& L, const PhysDev& ph,
                         TensorTma* tma, const TensorBufs& b, int stage, double dt, const FuseSched& fs,
                         cudaStream_t st);
// TGV diagnostics partial sums (3 per tile: rho v.v, S^d:S^d, p div v, solution-point
// weighted); NS only
// B1 (optional, with Bq): the nq1 x (P+1) 1D factor of Bq = B1 (x) B1 (x) B1, applied
// sum-factorised (3 contractions of 4 x 6 instead of the dense 216 x 64 per component)
void tensor_launch_diag(int D, int P, const TensorGeom& g, const Line1D& L, const PhysDev& ph, TensorTma* tma,
                        const TensorBufs& b, const double* w, const double* Bq, int nq, double* part,
                        cudaStream_t st, const double* B1 = nullptr, int nq1 = 0);

}  // namespace sdrt
