/*
 * sdrt.h — C ABI of the B200-native SDRT residual / RK4 library (libsdrt.so).
 *
 * Spectral Difference Raviart-Thomas (SDRT), arXiv 2105.08632:
 *   semi-discrete residual dU/dt = -J^-1 (div~ f~)  ....... §2.1, l.268-350
 *   matrix form R~ = M14 D~ + M13 M19 P2 F~ ................ App. B, l.2828-2925
 *   explicit Runge-Kutta (classical RK4) ................... l.351, l.1124
 *
 * Conventions
 *   - All entry points return sdrt_status (0 = OK). On failure sdrt_last_error()
 *     returns a thread-local message. No exception crosses the ABI.
 *   - Opaque handles are library-owned host objects freed by their _destroy.
 *   - ALL device memory is caller-owned (plain device pointers). The library never
 *     calls cudaMalloc: the context lives in one caller-provided workspace of
 *     sdrt_ctx_workspace_bytes() bytes (256-byte aligned).
 *   - Streams are cudaStream_t passed as void*. Calls enqueue asynchronously.
 *   - State layout (every fp64 state-like array): row-major [row][alpha*K_pad + n]
 *     = [N_sol][N_V][K_pad], point-major, then variable, element fastest. This is
 *     App. B's state matrix U^(u) (N_sol x N_V|Omega_e|, l.2835-2843). Columns
 *     n >= K (padding) are ignored on input and left unspecified on output.
 *   - Element order: pattern (i,j[,k]) x fastest, then subcell s; id = pattern*N_p+s
 *     (DESIGN.md "Mesh"); reference point orders: DESIGN.md "Ordering".
 */
#ifndef SDRT_H
#define SDRT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDRT_ABI_VERSION 1

typedef enum {
  SDRT_OK = 0,
  SDRT_E_INVALID_ARG = -1,
  SDRT_E_UNSUPPORTED = -2,
  SDRT_E_ILL_CONDITIONED = -3,
  SDRT_E_CUDA = -4,
  SDRT_E_NCCL = -5,
  SDRT_E_WORKSPACE = -6,
  SDRT_E_DIVERGED = -7,
  SDRT_E_INTERNAL = -8
} sdrt_status;

/* element types (App. A); N_p = 1, 2, 1, 6, 2 sub-cells per pattern (l.499).
 * Prisms (NEXT row N3, l.2633-2737; p <= 3, SDRT scheme) mix triangular and
 * quadrilateral faces: faces 0, 1 (z = -1, +1) carry (p+1)(p+2)/2 points, faces 2-4
 * (p+1)^2; nfp reports the largest face and face_perm rows are padded with -1; they
 * run on the generic operator path (no fused prism kernels). */
typedef enum { SDRT_QUAD = 0, SDRT_TRI = 1, SDRT_HEX = 2, SDRT_TET = 3, SDRT_PRI = 4 } sdrt_etype;
/* schemes: SDRT (the path); FR-SDRT and FR-DG flux reconstruction on the same data
 * (NEXT row N1): no internal flux points, solution-point fluxes
 * with the SDRT (FR-SDRT) or DG (FR-DG: Radau on tensor elements, DG lifting on
 * simplices) corrections */
typedef enum { SDRT_SCHEME_SDRT = 0, SDRT_SCHEME_FRSDRT = 1, SDRT_SCHEME_FRDG = 2 } sdrt_scheme;
/* equations: linear advection, linear advection-diffusion (l.1658), Euler
 * (l.1909-1935), compressible Navier-Stokes (l.2012-2030) */
typedef enum { SDRT_EQ_LINADV = 0, SDRT_EQ_LINADVDIFF = 1, SDRT_EQ_EULER = 2, SDRT_EQ_NS = 3 } sdrt_eq;

typedef struct {
  int eq;          /* sdrt_eq */
  double c[3];     /* advection velocity (linear equations) */
  double mu;       /* diffusivity (lin.) / dynamic viscosity (NS) */
  double gamma;    /* ratio of specific heats (Euler/NS) */
  double Pr;       /* Prandtl number (NS) */
  double beta;     /* LDG common-value parameter, Eq. common_var_for_grad l.290 */
  double eta;      /* LDG penalty, l.332-334 */
} sdrt_physics;

typedef struct sdrt_mesh sdrt_mesh;
typedef struct sdrt_operators sdrt_operators;
typedef struct sdrt_ctx sdrt_ctx;

typedef struct {
  int etype, p, nd;
  int nsol, next, nint, nu, nfaces, nfp;
  int nsub;            /* N_p */
  int N[3];            /* local patterns per axis (this rank) */
  int Nglobal[3];      /* global patterns per axis */
  int offset[3];       /* first global pattern index of this rank */
  int64_t K;           /* local elements */
  int64_t K_pad;       /* K rounded up to a multiple of 32 */
  int64_t n_faces;     /* local face count (faces whose left element is local) */
  int64_t K_trace;     /* row stride of the internal trace arrays (K_pad + ghost columns) */
} sdrt_mesh_info_t;

int sdrt_abi_version(void);
const char* sdrt_last_error(void);

/* Uniform mesh of N[0] x N[1] (x N[2]) patterns on the box [lo, hi], each pattern
 * split into N_p sub-cells. periodic[d] = 1: periodic axis;
 * 0: far-field boundaries at x_d = lo[d] and hi[d] (the paper's vortex, PAPER.md l.1952:
 * "the limiting values of the initial conditions ... at boundaries with constant x"):
 * the boundary faces' exterior state is a constant far-field state set with
 * sdrt_ctx_set_farfield (fused element paths only).  periodic = NULL: all periodic.
 * N[d] >= 3.
 * Multi-rank: the pattern grid is block-partitioned by pgrid (pgrid[d] divides
 * N[d]); rank r owns block (r % pg0, (r / pg0) % pg1, r / (pg0 pg1)).
 * Single rank: rank = 0, nranks = 1, pgrid = NULL.
 * Errors: SDRT_E_INVALID_ARG (bad sizes), SDRT_E_UNSUPPORTED (etype/p). */
sdrt_status sdrt_mesh_create(int etype, int p, const int N[3], const double lo[3], const double hi[3],
                             const int periodic[3], int rank, int nranks, const int pgrid[3],
                             sdrt_mesh** out);
sdrt_status sdrt_mesh_info(const sdrt_mesh* m, sdrt_mesh_info_t* out);
/* Face list of the (local) mesh, faces sorted by (left element, left local face)
 * (reading O14: left = element whose outward unit normal has its first non-zero
 * component positive).  face_elem[F][2] = (left, right) element ids (global ids
 * for multi-rank), face_lface[F][2] local face ids, face_perm[F][nfp] = right's
 * local face-point index matching the left's point q, is_left[K][nfaces].
 * Any pointer may be NULL. Host memory, caller-owned. */
sdrt_status sdrt_mesh_export_maps(const sdrt_mesh* m, int32_t* face_elem, int8_t* face_lface,
                                  int16_t* face_perm, uint8_t* is_left);
/* Physical coordinates of the solution points: x[N_sol][D][K] (host). */
sdrt_status sdrt_mesh_sol_coords(const sdrt_mesh* m, double* x);
/* Per-element det J (host, [K]), used for conservation sums. */
sdrt_status sdrt_mesh_detj(const sdrt_mesh* m, double* detj);
void sdrt_mesh_destroy(sdrt_mesh* m);
/* Halo (multi-rank element partition).  Trace arrays carry ghost columns
 * after K_pad for the neighbouring ranks' boundary elements; one exchange moves, per
 * slab (axis d, side), the face-point traces of this rank's boundary elements facing the
 * peer.  force_self_halo = 1 routes periodic wraps of single-rank axes through the same
 * path (loopback; the library then exchanges by itself).  Call before sdrt_ctx_create. */
sdrt_status sdrt_mesh_set_halo(sdrt_mesh* m, int force_self_halo);
/* slab = -1: *count = number of slabs.  Otherwise the slab's peer rank, axis, side,
 * entry count and (trace row, column) lists in the canonical order (any pointer may be
 * NULL; host arrays of *count int32).  The peer's send list for its opposite slab
 * matches this rank's recv list entry by entry. */
sdrt_status sdrt_mesh_halo_lists(const sdrt_mesh* m, int slab, int* peer, int* d, int* side, int64_t* count,
                                 int32_t* send_row, int32_t* send_col, int32_t* recv_row, int32_t* recv_col);
/* Trace column the kernels read for the neighbour of local element e across local face
 * f (a local element id, or a ghost column >= K_pad), and the neighbour's local face. */
sdrt_status sdrt_mesh_neighbor(const sdrt_mesh* m, int64_t e, int f, int64_t* col, int* face);

/* Appendix-B operators for (etype, p), built in __float128 and rounded once.
 * Errors: SDRT_E_UNSUPPORTED, SDRT_E_ILL_CONDITIONED (cond(V^f) > 1e12). */
sdrt_status sdrt_operators_build(int etype, int p, int scheme, sdrt_operators** out);
/* name in {"M0","M12","M13","M14","M15","M16","P","M19P2","w","xsol","xext","xu"}, and for
 * the FR schemes "Mc" (N_sol x N_ext, div g_nu at the solution points: M14 for FR-SDRT,
 * l.407-413; FR-DG: Radau g_DG on tensor elements, the DG lifting M^-1 L on simplices,
 * l.371-373). dst == NULL queries the shape. Row-major doubles, host memory.
 * Errors: SDRT_E_INVALID_ARG for an unknown name. */
sdrt_status sdrt_operators_get(const sdrt_operators* o, const char* name, double* dst, int* rows,
                               int* cols);
void sdrt_operators_destroy(sdrt_operators* o);

/* Device workspace size for a context (bytes). */
size_t sdrt_ctx_workspace_bytes(const sdrt_mesh* m, const sdrt_operators* o, const sdrt_physics* ph);
/* Create a context over caller-owned device workspace d_ws (>= the size above).
 * Uploads operators and geometry tables on `stream`. The mesh and operators may be
 * destroyed afterwards. Errors: SDRT_E_WORKSPACE, SDRT_E_CUDA, SDRT_E_INVALID_ARG. */
sdrt_status sdrt_ctx_create(const sdrt_mesh* m, const sdrt_operators* o, const sdrt_physics* ph,
                            void* d_ws, size_t ws_bytes, void* stream, sdrt_ctx** out);
/* dU/dt = -J^-1 R~ for the device state d_U -> d_dUdt (both [N_sol][N_V][K_pad]). */
sdrt_status sdrt_residual(sdrt_ctx* c, const double* d_U, double* d_dUdt, void* stream);
/* Conservation check (reading O28): the residual of d_U as sdrt_residual, and in d_F
 * ([N_ext][N_V][K_pad], device, caller-owned) the common normal flux F (Rusanov /
 * upwind + LDG, along the LEFT element's unit normal, before the
 * metric scale s) that each element applied at each of its external points: the left
 * side applies D~ = +s F, the right side D~ = -s F of the same value, so for every
 * face point F(left, q) == F(right, perm[q]) bit for bit.  Single-rank contexts (as
 * sdrt_residual).  Errors: SDRT_E_INVALID_ARG for null pointers. */
sdrt_status sdrt_face_flux(sdrt_ctx* c, const double* d_U, double* d_dUdt, double* d_F, void* stream);
/* nsteps classical RK4 steps of size dt, in place on d_U. check_every > 0 syncs the
 * stream every check_every steps and returns SDRT_E_DIVERGED (message names the
 * first non-finite / non-physical element and step) if the state went bad. */
sdrt_status sdrt_rk_step(sdrt_ctx* c, double* d_U, double dt, int nsteps, int check_every, void* stream);
/* nsteps steps of RK54 (five stages, two registers, fourth order; PAPER.md l.1120,
 * l.1200, stability polynomial l.1124; Carpenter & Kennedy 2N-storage coefficients),
 * in place on d_U; the context's RK accumulator holds the second register.  Fused
 * element paths only (SDRT_E_UNSUPPORTED otherwise).  check_every as sdrt_rk_step. */
sdrt_status sdrt_rk54_step(sdrt_ctx* c, double* d_U, double dt, int nsteps, int check_every, void* stream);
/* Taylor-Green-vortex diagnostics of the device state d_U:
 * d_out (3 device doubles) = { <E*> = <rho v.v>, eps2 = 2 mu <S^d : S^d>,
 * eps3 = -<p div v> } with rho_inf = v_inf = L = t_c = 1.  Ensemble averages by the
 * context's rule (sdrt_diagnostics_rule): by default the paper's degree-10 quadrature
 * (l.2075) of the solution polynomial u_h and of the LDG-gradient polynomial Q_h
 * (l.295-302), grad v by the chain rule (DESIGN.md readings).  eps1 = -d<E*>/dt is left
 * to the caller.  Single-rank 3-D NS contexts on a fused path; SDRT_E_UNSUPPORTED
 * otherwise.  Enqueued on stream. */
sdrt_status sdrt_diagnostics(sdrt_ctx* c, const double* d_U, double* d_out, void* stream);
/* Quadrature of sdrt_diagnostics: degree 1..10 = a rule exact to that degree on the
 * reference element (Gauss-Legendre products on quad/hex, collapsed Gauss-Legendre
 * products on tri/tet; default 10), 0 = the solution points with weights w_r = int l_r.
 * Synchronous host->device upload.  SDRT_E_INVALID_ARG outside 0..10. */
sdrt_status sdrt_diagnostics_rule(sdrt_ctx* c, int degree);
/* CUDA-graph replay of K-step runs (the run is PAPER.md's explicit RK stepping, l.351,
 * l.1120): with mode 1 (or -1: on for meshes below 2^22 DOF; the default is 0, off, because
 * the direct launches with programmatic dependent launch measured faster on every config)
 * sdrt_rk_step / sdrt_rk54_step with check_every <= 0 capture their launch
 * sequence once into a CUDA graph on a library-owned stream and replay it while the call
 * repeats with the same d_U, dt, nsteps and integrator; results are bitwise those of the
 * direct launches.  0 disables.  The graph is ordered after prior work on `stream` and
 * later work on `stream` after it (events).  Not used with timing, a communicator or the
 * slab schedule.  SDRT_E_INVALID_ARG for other modes. */
sdrt_status sdrt_ctx_set_graph(sdrt_ctx* c, int mode);
/* Per-kernel device timing (CUDA events recorded on the launching stream around each
 * kernel) for measurement: enable, run, then read per-kernel totals.  names receives
 * max_tags NUL-terminated strings of 64 bytes each (may be NULL); ms/counts get the
 * summed device milliseconds and launch counts per kernel; *ntags the count used.
 * Reading synchronises on the recorded events and resets the accumulators. */
sdrt_status sdrt_ctx_set_timing(sdrt_ctx* c, int enable);
sdrt_status sdrt_ctx_kernel_times(sdrt_ctx* c, int max_tags, char* names, double* ms, int64_t* counts,
                                  int* ntags);
/* Staged stage API for multi-rank runs (caller performs the halo exchange between calls):
 *   sdrt_stage_traces(U)                       traces of U          -> exchange which=0
 *   for stage s in 0..3:
 *     sdrt_stage_grad(U, s)   (viscous only)   viscous traces       -> exchange which=1
 *     sdrt_stage_flux(U, s, dt, NULL)          RK stage, new traces -> exchange which=0
 * stage = -1 with d_out computes dU/dt into d_out instead (residual).  The stage input
 * is U for s <= 0 and the internal stage register otherwise.  RK54 stages are
 * stage = 10 + s, s = 0..4 (stage input U, updated in place). */
sdrt_status sdrt_stage_traces(sdrt_ctx* c, const double* d_U, void* stream);
sdrt_status sdrt_stage_grad(sdrt_ctx* c, double* d_U, int stage, void* stream);
sdrt_status sdrt_stage_flux(sdrt_ctx* c, double* d_U, int stage, double dt, double* d_out, void* stream);
/* Overlap variants: the same stage on a subset of the element tiles,
 * part = 0 all, 1 interior tiles (no element in a pattern layer next to a partition
 * face: they read no ghost values), 2 boundary tiles.  A stage split as
 *   grad(1) || [exchange 0 in flight], grad(2), flux(1) || [exchange 1], flux(2)
 * gives results identical to part 0 (every element is in exactly one part; the
 * trace double buffer flips after part 2).  Without partition faces every tile is
 * interior and part 2 is empty.  Errors: SDRT_E_INVALID_ARG for part outside 0..2. */
sdrt_status sdrt_stage_grad_part(sdrt_ctx* c, double* d_U, int stage, int part, void* stream);
sdrt_status sdrt_stage_flux_part(sdrt_ctx* c, double* d_U, int stage, double dt, double* d_out, int part,
                                 void* stream);
/* Halo buffers: *nslab slabs; peer/d/side per slab (arrays of 6), offset[nslab+1] =
 * value offsets of each slab's segment in the contiguous send / recv buffers (doubles).
 * pack copies this rank's outgoing traces (which = 0: U traces of the current stage
 * input, 1: published viscous traces) into d_send; unpack scatters d_recv, where
 * segment i holds what the peer of slab i sent from its opposite slab, into the ghost
 * columns.  Device buffers, caller-owned. */
sdrt_status sdrt_halo_info(const sdrt_ctx* c, int* nslab, int* peer, int* d, int* side, int64_t* offset);
sdrt_status sdrt_halo_pack(sdrt_ctx* c, int which, double* d_send, void* stream);
sdrt_status sdrt_halo_unpack(sdrt_ctx* c, int which, const double* d_recv, void* stream);
/* Far-field boundaries (NEXT row N4): state[N_V] (host, conserved
 * variables) is the exterior state of every far-field boundary face.  The common
 * flux there is the interior one of l.312-340 with u_ext = state and, for viscous
 * equations, a zero exterior gradient (the viscous flux of a constant state), the
 * left/right roles by reading O14.  Must be called once before sdrt_residual /
 * sdrt_rk_step on a context whose mesh has a non-periodic axis (SDRT_E_INVALID_ARG
 * from those otherwise); synchronous.  SDRT_E_INVALID_ARG if the mesh is periodic. */
sdrt_status sdrt_ctx_set_farfield(sdrt_ctx* c, const double* state, void* stream);
/* NCCL inside the library.  Rank 0 calls sdrt_comm_unique_id and
 * broadcasts the 128 bytes to the other ranks (e.g. with torch.distributed); every rank
 * then calls sdrt_ctx_attach_comm on its context (collective: all ranks of the
 * partition, one GPU each, current device selected).  From then on sdrt_residual,
 * sdrt_rk_step and sdrt_rk54_step run the whole multi-rank stage inside the library:
 * the face traces of each partition face are packed, exchanged by grouped
 * ncclSend/ncclRecv on the library's comm stream (ordered against the caller's stream
 * by events) and unpacked into ghost columns, overlapped with the interior tiles; a
 * check_every > 0 divergence check is all-reduced so every rank returns
 * SDRT_E_DIVERGED together.  The partitioned result equals the single-rank one element
 * by element.  rank / nranks must be those the mesh was created with.  A single-rank
 * mesh with sdrt_mesh_set_halo(m, 1) exchanges its periodic faces through NCCL with
 * itself (nranks = 1).  NCCL is loaded at run time (libnccl.so.2; the process's copy
 * if one is loaded).  Errors: SDRT_E_NCCL (NCCL missing or failing), SDRT_E_INVALID_ARG,
 * SDRT_E_UNSUPPORTED (no halo slabs / no fused path).  The communicator is destroyed
 * with the context. */
sdrt_status sdrt_comm_unique_id(uint8_t id[128]);
sdrt_status sdrt_ctx_attach_comm(sdrt_ctx* c, const uint8_t id[128], int rank, int nranks);
/* Number of kernel launches enqueued by the last sdrt_residual / sdrt_rk_step call. */
int64_t sdrt_ctx_last_launches(const sdrt_ctx* c);
void sdrt_ctx_destroy(sdrt_ctx* c);

#ifdef __cplusplus
}
#endif
#endif /* SDRT_H */
