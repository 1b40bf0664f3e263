// Pointwise physics on the device (fp64).
//   linear advection-diffusion f = c u - mu grad u
//   upwind Lax-Friedrichs                                    Eq. flux_advection l.491-496
//   Euler: f = (rho v, rho v v + p I, (rho E + p) v), rho E = p/(g-1) + rho v.v/2   l.1909-1935
//   NS viscous: (0, -tau, -(mu c_p/Pr) grad T - tau.v)       l.2012-2030
//     (mu c_p/Pr) grad T = mu g/((g-1) Pr) grad(p/rho)       reading O18
//     primitive gradients from conserved-variable gradients  reading O20
//   Rusanov: n.(fL+fR)/2 + phi/2 (uL-uR), phi = max(|vL.n|+aL, |vR.n|+aR)  l.324-328, O13
//   LDG: C = (1/2-b) uL + (1/2+b) uR                         l.282-291
//        Fv = n.[(1/2+b) fvL + (1/2-b) fvR] + eta (uL - uR)  l.330-335, O10
#pragma once

namespace sdrt {

enum { EQ_LINADV = 0, EQ_LINADVDIFF = 1, EQ_EULER = 2, EQ_NS = 3 };

struct PhysDev {
  double c[3];
  double mu, gamma, Pr, beta, eta;
  double kappa;  // mu gamma / ((gamma - 1) Pr), formed once on the host (same IEEE ops)
};

template <int EQ, int D>
struct Phys {
  static constexpr int NV = (EQ == EQ_LINADV || EQ == EQ_LINADVDIFF) ? 1 : D + 2;
  static constexpr bool VISC = (EQ == EQ_LINADVDIFF || EQ == EQ_NS);

  // convective flux component along direction vector w: sum_d w_d f_d(u)
  static __device__ __forceinline__ void conv_dir(const PhysDev& ph, const double* u, const double* w,
                                                  double* out) {
    if constexpr (NV == 1) {
      double cw = 0.0;
#pragma unroll
      for (int d = 0; d < D; ++d) cw += ph.c[d] * w[d];
      out[0] = cw * u[0];
    } else {
      const double rho = u[0];
      const double ir = 1.0 / rho;
      double v[D], vv = 0.0, vw = 0.0;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        v[d] = u[1 + d] * ir;
        vv += v[d] * u[1 + d];
        vw += v[d] * w[d];
      }
      const double p = (ph.gamma - 1.0) * (u[D + 1] - 0.5 * vv);
      out[0] = rho * vw;
#pragma unroll
      for (int i = 0; i < D; ++i) out[1 + i] = u[1 + i] * vw + p * w[i];
      out[D + 1] = (u[D + 1] + p) * vw;
    }
  }

  // viscous flux component along w: sum_d w_d fv_d(u, q), q[d*NV + a] = d u_a / d x_d
  static __device__ __forceinline__ void visc_dir(const PhysDev& ph, const double* u, const double* q,
                                                  const double* w, double* out) {
    if constexpr (EQ == EQ_LINADVDIFF) {
      double s = 0.0;
#pragma unroll
      for (int d = 0; d < D; ++d) s += w[d] * q[d];
      out[0] = -ph.mu * s;
    } else if constexpr (EQ == EQ_NS) {
      const double g = ph.gamma;
      const double rho = u[0];
      const double ir = 1.0 / rho;
      double v[D], vv = 0.0;
#pragma unroll
      for (int i = 0; i < D; ++i) {
        v[i] = u[1 + i] * ir;
        vv += v[i] * v[i];
      }
      const double p = (g - 1.0) * (u[D + 1] - 0.5 * rho * vv);
      // grad v: dv[i][d] = (d(rho v_i)/dx_d - v_i d rho/dx_d) / rho
      double dv[D][D];
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int d = 0; d < D; ++d) dv[i][d] = (q[d * NV + 1 + i] - v[i] * q[d * NV]) * ir;
      double div = 0.0;
#pragma unroll
      for (int i = 0; i < D; ++i) div += dv[i][i];
      const double kappa = ph.kappa;
      // tau_{id} w_d, heat flux . w
      out[0] = 0.0;
      double tw[D];
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double s = 0.0;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          double tau = ph.mu * (dv[i][d] + dv[d][i] - (i == d ? (2.0 / 3.0) * div : 0.0));
          s += tau * w[d];
        }
        tw[i] = s;
        out[1 + i] = -s;
      }
      double hw = 0.0;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        double vdv = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) vdv += v[i] * dv[i][d];
        const double dp = (g - 1.0) * (q[d * NV + D + 1] - 0.5 * vv * q[d * NV] - rho * vdv);
        const double dT = (dp - p * ir * q[d * NV]) * ir;
        hw += dT * w[d];
      }
      double tv = 0.0;
#pragma unroll
      for (int i = 0; i < D; ++i) tv += tw[i] * v[i];
      out[D + 1] = -kappa * hw - tv;
    } else {
#pragma unroll
      for (int a = 0; a < NV; ++a) out[a] = 0.0;
    }
  }

  // Axis-aligned forms for w = wd e_D0 (tensor elements: B7's single normal component,
  // l.2927-2932): the same fluxes touching only the entries that component needs (for NS
  // the gradient entries d rho, d(rho v_D0), d(rho v_j) / dx_j of the tangential axes
  // and all entries along D0), so unused gradient interpolations are dead code.
  template <int D0>
  static __device__ __forceinline__ void conv_axis(const PhysDev& ph, const double* u, double wd, double* out) {
    if constexpr (NV == 1) {
      out[0] = ph.c[D0] * wd * u[0];
    } else {
      const double rho = u[0];
      const double ir = 1.0 / rho;
      double vv = 0.0;
#pragma unroll
      for (int d = 0; d < D; ++d) vv += u[1 + d] * ir * u[1 + d];
      const double vw = u[1 + D0] * ir * wd;
      const double p = (ph.gamma - 1.0) * (u[D + 1] - 0.5 * vv);
      out[0] = rho * vw;
#pragma unroll
      for (int i = 0; i < D; ++i) out[1 + i] = i == D0 ? u[1 + i] * vw + p * wd : u[1 + i] * vw;
      out[D + 1] = (u[D + 1] + p) * vw;
    }
  }

  template <int D0>
  static __device__ __forceinline__ void visc_axis(const PhysDev& ph, const double* u, const double* q, double wd,
                                                   double* out) {
    if constexpr (EQ == EQ_LINADVDIFF) {
      out[0] = -ph.mu * (wd * q[D0]);
    } else if constexpr (EQ == EQ_NS) {
      const double g = ph.gamma;
      const double rho = u[0];
      const double ir = 1.0 / rho;
      double v[D], vv = 0.0;
#pragma unroll
      for (int i = 0; i < D; ++i) {
        v[i] = u[1 + i] * ir;
        vv += v[i] * v[i];
      }
      const double p = (g - 1.0) * (u[D + 1] - 0.5 * rho * vv);
      // dvn[i] = d v_i / dx_D0, dvt[j] = d v_D0 / dx_j, div from d v_j / dx_j
      double dvn[D], dvt[D], div = 0.0;
#pragma unroll
      for (int i = 0; i < D; ++i) dvn[i] = (q[D0 * NV + 1 + i] - v[i] * q[D0 * NV]) * ir;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        dvt[j] = j == D0 ? dvn[D0] : (q[j * NV + 1 + D0] - v[D0] * q[j * NV]) * ir;
        div += j == D0 ? dvn[D0] : (q[j * NV + 1 + j] - v[j] * q[j * NV]) * ir;
      }
      const double kappa = ph.kappa;
      out[0] = 0.0;
      double tv = 0.0;
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const double tau = ph.mu * (dvn[i] + dvt[i] - (i == D0 ? (2.0 / 3.0) * div : 0.0));
        const double s = tau * wd;
        out[1 + i] = -s;
        tv += s * v[i];
      }
      double vdv = 0.0;
#pragma unroll
      for (int i = 0; i < D; ++i) vdv += v[i] * dvn[i];
      const double dp = (g - 1.0) * (q[D0 * NV + D + 1] - 0.5 * vv * q[D0 * NV] - rho * vdv);
      const double dT = (dp - p * ir * q[D0 * NV]) * ir;
      out[D + 1] = -kappa * (dT * wd) - tv;
    } else {
#pragma unroll
      for (int a = 0; a < NV; ++a) out[a] = 0.0;
    }
  }

  // ---- common fluxes with explicitly rounded arithmetic (reading O28) ----------------
  // The fused kernels evaluate a face point's common flux on BOTH sides of the face,
  // from bit-identical inputs, in whichever inlined copy of the face code owns each
  // side's item.  With free FMA contraction the compiler may fuse different products
  // in different copies (measured: 1-ulp differences on tets with eta != 0), so every
  // operation of the common flux is an explicit IEEE op (__dmul_rn / __dadd_rn /
  // __fma_rn, IEEE division and sqrt): the same inputs give the same bits everywhere.
  static __device__ __forceinline__ double dot_rn(const double* a, const double* b) {
    double s = __dmul_rn(a[0], b[0]);
#pragma unroll
    for (int d = 1; d < D; ++d) s = __fma_rn(a[d], b[d], s);
    return s;
  }
  // Euler flux along n plus the Rusanov wave speed |v.n| + a of one state
  static __device__ __forceinline__ double euler_dir_rn(const PhysDev& ph, const double* u, const double* n,
                                                        double* f) {
    const double ir = 1.0 / u[0];
    const double vn = __dmul_rn(dot_rn(u + 1, n), ir);
    const double vv = __dmul_rn(dot_rn(u + 1, u + 1), ir);                          // rho |v|^2
    const double p = __dmul_rn(ph.gamma - 1.0, __fma_rn(-0.5, vv, u[D + 1]));
    f[0] = __dmul_rn(u[0], vn);
#pragma unroll
    for (int i = 0; i < D; ++i) f[1 + i] = __fma_rn(p, n[i], __dmul_rn(u[1 + i], vn));
    f[D + 1] = __dmul_rn(__dadd_rn(u[D + 1], p), vn);
    return __dadd_rn(fabs(vn), sqrt(__dmul_rn(__dmul_rn(ph.gamma, p), ir)));
  }

  // convective common flux (upwind LF for linear, Rusanov otherwise) along n
  static __device__ __forceinline__ void conv_common(const PhysDev& ph, const double* uL, const double* uR,
                                                     const double* n, double* F) {
    if constexpr (NV == 1) {
      const double cn = dot_rn(ph.c, n);
      F[0] = __fma_rn(__dmul_rn(0.5, fabs(cn)), __dsub_rn(uL[0], uR[0]),
                      __dmul_rn(__dmul_rn(0.5, cn), __dadd_rn(uL[0], uR[0])));
    } else {
      double fL[NV], fR[NV];
      const double sL = euler_dir_rn(ph, uL, n, fL), sR = euler_dir_rn(ph, uR, n, fR);
      const double hphi = __dmul_rn(0.5, fmax(sL, sR));
#pragma unroll
      for (int a = 0; a < NV; ++a)
        F[a] = __fma_rn(hphi, __dsub_rn(uL[a], uR[a]), __dmul_rn(0.5, __dadd_rn(fL[a], fR[a])));
    }
  }

  // Euler flux along +e_D0 and the Rusanov wave speed (explicitly rounded, no
  // structural zeros of the normal)
  template <int D0>
  static __device__ __forceinline__ double euler_axis_rn(const PhysDev& ph, const double* u, double* f) {
    const double ir = 1.0 / u[0];
    const double vn = __dmul_rn(u[1 + D0], ir);
    const double vv = __dmul_rn(dot_rn(u + 1, u + 1), ir);
    const double p = __dmul_rn(ph.gamma - 1.0, __fma_rn(-0.5, vv, u[D + 1]));
    f[0] = u[1 + D0];
#pragma unroll
    for (int i = 0; i < D; ++i) f[1 + i] = i == D0 ? __fma_rn(u[1 + i], vn, p) : __dmul_rn(u[1 + i], vn);
    f[D + 1] = __dmul_rn(__dadd_rn(u[D + 1], p), vn);
    return __dadd_rn(fabs(vn), sqrt(__dmul_rn(__dmul_rn(ph.gamma, p), ir)));
  }

  // conv_common along the axis normal +e_D0 (tensor faces): the same Rusanov flux
  template <int D0>
  static __device__ __forceinline__ void conv_common_axis(const PhysDev& ph, const double* uL, const double* uR,
                                                          double* F) {
    if constexpr (NV == 1) {
      const double cn = ph.c[D0];
      F[0] = __fma_rn(__dmul_rn(0.5, fabs(cn)), __dsub_rn(uL[0], uR[0]),
                      __dmul_rn(__dmul_rn(0.5, cn), __dadd_rn(uL[0], uR[0])));
    } else {
      double fL[NV], fR[NV];
      const double sL = euler_axis_rn<D0>(ph, uL, fL), sR = euler_axis_rn<D0>(ph, uR, fR);
      const double hphi = __dmul_rn(0.5, fmax(sL, sR));
#pragma unroll
      for (int a = 0; a < NV; ++a)
        F[a] = __fma_rn(hphi, __dsub_rn(uL[a], uR[a]), __dmul_rn(0.5, __dadd_rn(fL[a], fR[a])));
    }
  }

  // LDG part of the common flux (l.330-335, O10) from the LDG-weighted published
  // viscous normal flux gsum = (1/2+b) g_L + (1/2-b) g_R: F + gsum + eta (u_L - u_R)
  static __device__ __forceinline__ double ldg_rn(double F, double gsum, double eta, double uL, double uR) {
    return __dadd_rn(F, __fma_rn(eta, __dsub_rn(uL, uR), gsum));
  }
  static __device__ __forceinline__ double gsum_rn(double wl, double gL, double wr, double gR) {
    return __fma_rn(wr, gR, __dmul_rn(wl, gL));
  }

  // common normal flux along nL (left element's unit normal)
  static __device__ __forceinline__ void common_flux(const PhysDev& ph, const double* uL, const double* uR,
                                                     const double* qL, const double* qR, const double* n,
                                                     double* F) {
    if constexpr (NV == 1) {
      double cn = 0.0;
#pragma unroll
      for (int d = 0; d < D; ++d) cn += ph.c[d] * n[d];
      F[0] = 0.5 * cn * (uL[0] + uR[0]) + 0.5 * fabs(cn) * (uL[0] - uR[0]);
    } else {
      double fL[NV], fR[NV];
      conv_dir(ph, uL, n, fL);
      conv_dir(ph, uR, n, fR);
      double sL = 0.0, sR = 0.0;
      {
        const double irL = 1.0 / uL[0], irR = 1.0 / uR[0];
        double vnL = 0.0, vnR = 0.0, vvL = 0.0, vvR = 0.0;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          vnL += uL[1 + d] * n[d];
          vnR += uR[1 + d] * n[d];
          vvL += uL[1 + d] * uL[1 + d];
          vvR += uR[1 + d] * uR[1 + d];
        }
        vnL *= irL;
        vnR *= irR;
        const double pL = (ph.gamma - 1.0) * (uL[D + 1] - 0.5 * vvL * irL);
        const double pR = (ph.gamma - 1.0) * (uR[D + 1] - 0.5 * vvR * irR);
        sL = fabs(vnL) + sqrt(ph.gamma * pL * irL);
        sR = fabs(vnR) + sqrt(ph.gamma * pR * irR);
      }
      const double phi = fmax(sL, sR);
#pragma unroll
      for (int a = 0; a < NV; ++a) F[a] = 0.5 * (fL[a] + fR[a]) + 0.5 * phi * (uL[a] - uR[a]);
    }
    if constexpr (VISC) {
      double gL[NV], gR[NV];
      visc_dir(ph, uL, qL, n, gL);
      visc_dir(ph, uR, qR, n, gR);
      const double wl = 0.5 + ph.beta, wr = 0.5 - ph.beta;
#pragma unroll
      for (int a = 0; a < NV; ++a) F[a] += wl * gL[a] + wr * gR[a] + ph.eta * (uL[a] - uR[a]);
    }
  }
};

}  // namespace sdrt
