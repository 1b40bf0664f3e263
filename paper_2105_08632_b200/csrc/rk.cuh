// Time-integrator stage codes of the fused kernels' epilogue (kernel B).
//   stage -1      : residual only, dU/dt written to `out`
//   stage 0..3    : classical RK4, 3 registers (U = u_n, Us = stage input, ACC)
//   stage 10..14  : RK54 stage s = stage - 10 (five stages, two registers, fourth order,
//                   Carpenter & Kennedy, stability polynomial
//                   l.1124), 2N-storage: dU <- A_s dU + dt k;  U <- U + B_s dU; the stage
//                   input is U itself and ACC holds dU.
#pragma once

namespace sdrt {

constexpr int RK54_STAGE0 = 10;

__host__ __device__ constexpr double rk54_a(int s) {
  return s == 0 ? 0.0
       : s == 1 ? -567301805773.0 / 1357537059087.0
       : s == 2 ? -2404267990393.0 / 2016746695238.0
       : s == 3 ? -3550918686646.0 / 2091501179385.0
                : -1275806237668.0 / 842570457699.0;
}
__host__ __device__ constexpr double rk54_b(int s) {
  return s == 0 ? 1432997174477.0 / 9575080441755.0
       : s == 1 ? 5161836677717.0 / 13612068292357.0
       : s == 2 ? 1720146321549.0 / 2090206949498.0
       : s == 3 ? 3134564353537.0 / 4481467310338.0
                : 2277821191437.0 / 14882151754819.0;
}

// which RK registers a stage reads (besides the stage input)
__host__ __device__ constexpr bool stage_reads_acc(int stage) {
  return stage >= RK54_STAGE0 ? stage > RK54_STAGE0 : stage >= 1;
}
__host__ __device__ constexpr bool stage_reads_un(int stage) { return stage == 1 || stage == 2; }

}  // namespace sdrt
