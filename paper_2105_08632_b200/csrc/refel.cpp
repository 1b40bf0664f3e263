// Reference elements and Appendix-B operators, built once on the host in
// __float128 and rounded once to fp64.
//
// PAPER.md citations:
//   reference elements, spans, point layouts ....... App. A, l.2325-2816
//   solution / flux Vandermonde, nodal bases ........ §2.1 l.192-248
//   M0, M12, M13, M14, M15, M16, P, M19.P2 .......... App. B l.2845-2925
// Readings: O1 (simplex flux points = maximal-degree symmetric
// quadrature rules, solution points = centroid lattice), O2 (tet x+y+z <= -1),
// O3 (tensor internal points at zeros of P_p), O5 (any basis of the span).
//
// Construction route (deliberately different from the oracle's):
//   tensor elements: closed-form products of 1D Lagrange polynomials on the GL
//     nodes and on the flux line {-1, zeros(P_p), +1} (the RT nodal basis of
//     Q_{p+1,p,..} factorises; Huynh link l.388);
//   simplices: flux Vandermonde over shifted monomials xi = (x+1)/2 (RT_p is
//     affine invariant), Gauss-Jordan in __float128.
#include "refel.h"

#include <quadmath.h>

#include <algorithm>
#include <cmath>
#include <functional>
#include <map>
#include <stdexcept>

namespace sdrt {

typedef __float128 qd;
typedef std::array<qd, 3> P3;

static qd qabs(qd x) { return x < 0 ? -x : x; }

// ------------------------------------------------------------------ Gauss-Legendre
static void legendre_pair(int n, qd x, qd& pn, qd& pm) {
  qd p0 = 1, p1 = x;
  if (n == 0) { pn = 1; pm = 0; return; }
  for (int k = 2; k <= n; ++k) {
    qd p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
    p0 = p1;
    p1 = p2;
  }
  pn = p1;
  pm = p0;
}

// Roots of P_n ascending (Newton from Chebyshev-like guesses) and weights.
static void gauss_legendre(int n, std::vector<qd>& x, std::vector<qd>& w) {
  x.assign(n, 0);
  w.assign(n, 0);
  for (int i = 0; i < n; ++i) {
    qd r = cos(M_PI * (i + 0.75) / (n + 0.5));
    for (int it = 0; it < 100; ++it) {
      qd pn, pm;
      legendre_pair(n, r, pn, pm);
      qd dp = n * (r * pn - pm) / (r * r - 1);
      qd dx = pn / dp;
      r -= dx;
      if (qabs(dx) < 1e-33Q) break;
    }
    qd pn, pm;
    legendre_pair(n, r, pn, pm);
    qd dp = n * (r * pn - pm) / (r * r - 1);
    x[i] = r;
    w[i] = 2 / ((1 - r * r) * dp * dp);
  }
  std::vector<int> idx(n);
  for (int i = 0; i < n; ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](int a, int b) { return x[a] < x[b]; });
  std::vector<qd> xs(n), ws(n);
  for (int i = 0; i < n; ++i) { xs[i] = x[idx[i]]; ws[i] = w[idx[i]]; }
  x = xs;
  w = ws;
}

// ------------------------------------------------------------------ small dense LA
// Solve A X = B (A n x n, B n x m) in place by Gauss-Jordan with partial pivoting.
static void gj_solve(std::vector<qd>& A, int n, std::vector<qd>& B, int m) {
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (qabs(A[(size_t)r * n + c]) > qabs(A[(size_t)piv * n + c])) piv = r;
    if (A[(size_t)piv * n + c] == 0) throw std::runtime_error("singular Vandermonde matrix");
    if (piv != c) {
      for (int k = 0; k < n; ++k) std::swap(A[(size_t)c * n + k], A[(size_t)piv * n + k]);
      for (int k = 0; k < m; ++k) std::swap(B[(size_t)c * m + k], B[(size_t)piv * m + k]);
    }
    qd inv = 1 / A[(size_t)c * n + c];
    for (int k = 0; k < n; ++k) A[(size_t)c * n + k] *= inv;
    for (int k = 0; k < m; ++k) B[(size_t)c * m + k] *= inv;
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      qd f = A[(size_t)r * n + c];
      if (f == 0) continue;
      for (int k = 0; k < n; ++k) A[(size_t)r * n + k] -= f * A[(size_t)c * n + k];
      for (int k = 0; k < m; ++k) B[(size_t)r * m + k] -= f * B[(size_t)c * m + k];
    }
  }
}

// ------------------------------------------------------------------ simplex rules
// Reading O1.  Orbits in barycentric coordinates; point order = distinct
// permutations of the generator in lexicographic order of the slot permutation.
enum Orbit { S3, S21, S111, S4, S31, S22 };
static int npar(Orbit o) { return o == S21 || o == S31 || o == S22 ? 1 : (o == S111 ? 2 : 0); }

static std::vector<std::vector<qd>> orbit_points(Orbit o, const qd* par) {
  std::vector<qd> gen;
  std::vector<int> pat;
  switch (o) {
    case S3: gen = {1 / (qd)3, 1 / (qd)3, 1 / (qd)3}; pat = {0, 0, 0}; break;
    case S21: gen = {1 - 2 * par[0], par[0], par[0]}; pat = {0, 1, 1}; break;
    case S111: gen = {par[0], par[1], 1 - par[0] - par[1]}; pat = {0, 1, 2}; break;
    case S4: gen = {0.25Q, 0.25Q, 0.25Q, 0.25Q}; pat = {0, 0, 0, 0}; break;
    case S31: gen = {1 - 3 * par[0], par[0], par[0], par[0]}; pat = {0, 1, 1, 1}; break;
    case S22: gen = {par[0], par[0], 0.5Q - par[0], 0.5Q - par[0]}; pat = {0, 0, 2, 2}; break;
  }
  int n = (int)gen.size();
  std::vector<int> perm(n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  std::vector<std::vector<int>> seen;
  std::vector<std::vector<qd>> out;
  do {
    std::vector<int> key(n);
    for (int i = 0; i < n; ++i) key[i] = pat[perm[i]];
    if (std::find(seen.begin(), seen.end(), key) != seen.end()) continue;
    seen.push_back(key);
    std::vector<qd> pt(n);
    for (int i = 0; i < n; ++i) pt[i] = gen[perm[i]];
    out.push_back(pt);
  } while (std::next_permutation(perm.begin(), perm.end()));
  return out;
}

struct RuleSpec {
  std::vector<Orbit> orbits;
  int degree;
  std::vector<double> start;  // starting orbit parameters (select the root)
  bool minimise;              // one free parameter fixed by min next-degree defect
  double fixed_num = 0, fixed_den = 0;  // or: first orbit parameter held at num/den
};

static RuleSpec rule_spec(int D, int n) {
  if (D == 2 && n == 1) return {{S3}, 1, {}, false};
  if (D == 2 && n == 3) return {{S21}, 2, {0.2}, false};
  if (D == 2 && n == 6) return {{S21, S21}, 4, {0.09, 0.44}, false};
  if (D == 2 && n == 10) return {{S3, S21, S111}, 5, {0.055, 0.07, 0.29}, true};
  if (D == 3 && n == 1) return {{S4}, 1, {}, false};
  if (D == 3 && n == 4) return {{S31}, 2, {0.14}, false};
  // tet p=3 interior: the S31 parameter is fixed at 17/250 (reading O1, round 2: the
  // degree-3 family is spatially unstable for a >= 0.069; a = 0.068 reproduces the
  // paper's tet SDRT3 RK4 tau_MAX, under the SDRT2 calibration)
  if (D == 3 && n == 10) return {{S31, S22}, 3, {0.07, 0.09}, false, 17, 250};
  throw std::runtime_error("no simplex rule of this size (supported: tri p<=4, tet p<=3)");
}

// Dirichlet integral over the unit simplex normalised by its volume.
static qd dirichlet(const std::vector<int>& e) {
  int D = (int)e.size() - 1;
  qd num = 1;
  for (int k = 2; k <= D; ++k) num *= k;
  int tot = D;
  for (int v : e) {
    for (int k = 2; k <= v; ++k) num *= k;
    tot += v;
  }
  qd den = 1;
  for (int k = 2; k <= tot; ++k) den *= k;
  return num / den;
}

static void exps_eq(int nb, int deg, std::vector<std::vector<int>>& out) {
  std::vector<int> e(nb, 0);
  std::function<void(int, int)> rec = [&](int i, int rem) {
    if (i == nb - 1) { e[i] = rem; out.push_back(e); return; }
    for (int k = rem; k >= 0; --k) { e[i] = k; rec(i + 1, rem - k); }
  };
  rec(0, deg);
}

struct RuleSolver {
  int D;
  RuleSpec spec;
  std::vector<std::vector<int>> eq_lo, eq_next;  // monomials deg <= d, and == d+1
  int nunk;

  RuleSolver(int D_, int n) : D(D_), spec(rule_spec(D_, n)) {
    for (int d = 0; d <= spec.degree; ++d) exps_eq(D + 1, d, eq_lo);
    exps_eq(D + 1, spec.degree + 1, eq_next);
    nunk = 0;
    for (auto o : spec.orbits) nunk += npar(o) + 1;
  }
  void unpack(const std::vector<qd>& x, std::vector<std::vector<qd>>& pts, std::vector<qd>& ws) const {
    pts.clear();
    ws.clear();
    int i = 0;
    for (auto o : spec.orbits) {
      auto op = orbit_points(o, &x[i]);
      i += npar(o);
      for (auto& p : op) { pts.push_back(p); ws.push_back(x[i]); }
      i += 1;
    }
  }
  std::vector<qd> residual(const std::vector<qd>& x, const std::vector<std::vector<int>>& eqs) const {
    std::vector<std::vector<qd>> pts;
    std::vector<qd> ws;
    unpack(x, pts, ws);
    std::vector<qd> r(eqs.size());
    for (size_t k = 0; k < eqs.size(); ++k) {
      qd s = 0;
      for (size_t q = 0; q < pts.size(); ++q) {
        qd t = ws[q];
        for (int c = 0; c <= D; ++c)
          for (int m = 0; m < eqs[k][c]; ++m) t *= pts[q][c];
        s += t;
      }
      r[k] = s - dirichlet(eqs[k]);
    }
    return r;
  }
  // Gauss-Newton on the degree-d equations over the unknowns except `fixed` (-1: none).
  void solve(std::vector<qd>& x, int fixed) const {
    std::vector<int> free_idx;
    for (int j = 0; j < nunk; ++j)
      if (j != fixed) free_idx.push_back(j);
    int nf = (int)free_idx.size();
    for (int it = 0; it < 60; ++it) {
      std::vector<qd> r = residual(x, eq_lo);
      int m = (int)r.size();
      std::vector<qd> J((size_t)m * nf);
      const qd h = 1e-14Q;
      for (int j = 0; j < nf; ++j) {
        std::vector<qd> xp = x, xm = x;
        xp[free_idx[j]] += h;
        xm[free_idx[j]] -= h;
        std::vector<qd> rp = residual(xp, eq_lo), rm = residual(xm, eq_lo);
        for (int i = 0; i < m; ++i) J[(size_t)i * nf + j] = (rp[i] - rm[i]) / (2 * h);
      }
      std::vector<qd> A((size_t)nf * nf, 0), b(nf, 0);
      for (int a = 0; a < nf; ++a) {
        for (int c = 0; c < nf; ++c) {
          qd s = 0;
          for (int i = 0; i < m; ++i) s += J[(size_t)i * nf + a] * J[(size_t)i * nf + c];
          A[(size_t)a * nf + c] = s;
        }
        qd s = 0;
        for (int i = 0; i < m; ++i) s += J[(size_t)i * nf + a] * r[i];
        b[a] = s;
      }
      gj_solve(A, nf, b, 1);
      qd mx = 0;
      for (int j = 0; j < nf; ++j) {
        x[free_idx[j]] -= b[j];
        mx = std::max(mx, qabs(b[j]));
      }
      if (mx < 1e-30Q) break;
    }
  }
  qd defect(std::vector<qd>& x, int fixed, qd a) const {
    x[fixed] = a;
    solve(x, fixed);
    std::vector<qd> r = residual(x, eq_next);
    qd s = 0;
    for (auto v : r) s += v * v;
    return s;
  }
};

// Barycentric points of the rule (n points in D dims).
static std::vector<std::vector<qd>> simplex_rule(int D, int n) {
  RuleSolver S(D, n);
  std::vector<qd> x;
  int si = 0, first_par = -1;
  for (auto o : S.spec.orbits) {
    for (int k = 0; k < npar(o); ++k) {
      if (first_par < 0) first_par = (int)x.size();
      x.push_back((qd)S.spec.start[si++]);
    }
    x.push_back(1 / (qd)n);
  }
  if (S.nunk == 1) {  // centroid
    x[0] = 1;
  } else if (S.spec.fixed_den > 0) {
    x[first_par] = (qd)S.spec.fixed_num / (qd)S.spec.fixed_den;
    S.solve(x, first_par);
  } else if (!S.spec.minimise) {
    S.solve(x, -1);
  } else {
    // golden section, then secant on the derivative of the defect
    qd a0 = x[first_par], lo = a0 * 0.6Q, hi = a0 * 1.5Q;
    const qd g = (sqrtq(5.0Q) - 1) / 2;
    std::vector<qd> xc = x, xd = x;
    qd c = hi - g * (hi - lo), d = lo + g * (hi - lo);
    qd fc = S.defect(xc, first_par, c), fd = S.defect(xd, first_par, d);
    for (int it = 0; it < 80 && hi - lo > 1e-9Q; ++it) {
      if (fc < fd) {
        hi = d; d = c; fd = fc; xd = xc;
        c = hi - g * (hi - lo);
        fc = S.defect(xc, first_par, c);
      } else {
        lo = c; c = d; fc = fd; xc = xd;
        d = lo + g * (hi - lo);
        fd = S.defect(xd, first_par, d);
      }
    }
    qd a = (lo + hi) / 2;
    std::vector<qd> xw = xc;
    auto dE = [&](qd t) {
      const qd h = 1e-11Q;
      std::vector<qd> x1 = xw, x2 = xw;
      qd e1 = S.defect(x1, first_par, t + h), e2 = S.defect(x2, first_par, t - h);
      return (e1 - e2) / (2 * h);
    };
    qd a1 = a * (1 + 1e-7Q), f0 = dE(a), f1 = dE(a1);
    for (int it = 0; it < 40; ++it) {
      if (f1 == f0) break;
      qd a2 = a1 - f1 * (a1 - a) / (f1 - f0);
      a = a1; f0 = f1; a1 = a2; f1 = dE(a1);
      if (qabs(a1 - a) < 1e-28Q) break;
    }
    x = xw;
    S.defect(x, first_par, a1);
  }
  std::vector<std::vector<qd>> pts;
  std::vector<qd> ws;
  S.unpack(x, pts, ws);
  for (auto& p : pts)
    for (auto v : p)
      if (!(v > 0)) throw std::runtime_error("simplex rule point outside the element");
  for (auto w : ws)
    if (!(w > 0)) throw std::runtime_error("simplex rule weight not positive");
  return pts;
}

// Centroid lattice (solution points of simplices), documented order.
static std::vector<std::vector<qd>> centroid_lattice(int D, int m) {
  std::vector<std::vector<qd>> out;
  qd del = 1 / (qd)(D + 1);
  if (D == 2) {
    for (int j = 0; j <= m; ++j)
      for (int i = 0; i <= m - j; ++i)
        out.push_back({(m - i - j + del) / (m + 1), (i + del) / (m + 1), (j + del) / (m + 1)});
  } else {
    for (int k = 0; k <= m; ++k)
      for (int j = 0; j <= m - k; ++j)
        for (int i = 0; i <= m - j - k; ++i)
          out.push_back({(m - i - j - k + del) / (m + 1), (i + del) / (m + 1), (j + del) / (m + 1),
                         (k + del) / (m + 1)});
  }
  return out;
}

static const int TRI_V[3][2] = {{-1, -1}, {1, -1}, {-1, 1}};
static const int TET_V[4][3] = {{-1, -1, -1}, {1, -1, -1}, {-1, 1, -1}, {-1, -1, 1}};
static const int TRI_F[3][2] = {{0, 1}, {1, 2}, {2, 0}};
static const int TET_F[4][3] = {{0, 1, 2}, {0, 1, 3}, {1, 2, 3}, {0, 2, 3}};

void simplex_ref_vertices(int etype, std::vector<std::array<double, 3>>& V) {
  V.clear();
  if (etype == TRI)
    for (auto& v : TRI_V) V.push_back({(double)v[0], (double)v[1], 0.0});
  else
    for (auto& v : TET_V) V.push_back({(double)v[0], (double)v[1], (double)v[2]});
}

// ------------------------------------------------------------------ reference element (qd)
struct RefQ {
  RefElement r;
  std::vector<P3> xsol, xext, xu, next_n;
};

static P3 bary(const std::vector<qd>& lam, const std::vector<P3>& verts) {
  P3 x = {0, 0, 0};
  for (size_t k = 0; k < verts.size(); ++k)
    for (int c = 0; c < 3; ++c) x[c] += lam[k] * verts[k][c];
  return x;
}

static std::array<double, 3> to_d(const P3& x) { return {(double)x[0], (double)x[1], (double)x[2]}; }

// Prism reference vertices (x, y >= -1, x + y <= 0, z in [-1, 1]) and faces:
// 0 z = -1, 1 z = +1 (triangles), 2 y = -1, 3 x + y = 0, 4 x = -1 (quadrilaterals)
static const int PRI_F[5][4] = {{0, 1, 2, -1}, {3, 4, 5, -1}, {0, 1, 4, 3}, {1, 2, 5, 4}, {2, 0, 3, 5}};

static RefQ build_ref_q(int etype, int p) {
  if (p < 1 || p > 4 || ((etype == TET || etype == PRI) && p > 3))
    throw std::runtime_error("unsupported degree: quad/hex/tri p in [1,4], tet/pri p in [1,3]");
  RefQ R;
  RefElement& r = R.r;
  r.etype = etype;
  r.p = p;
  r.nd = etype_dim(etype);
  int D = r.nd;
  if (etype == PRI) {
    // PAPER.md App. A l.2633-2737: triangle solution points x (p+1) GL levels; the
    // triangle faces carry the tet-face triangle rule, the quadrilateral faces edge GL x
    // GL; internal set 1 = triangle interior rule x (p+1) GL levels (normals e_x, e_y),
    // set 2 = triangle-face rule x the p zeros of P_p (normal e_z).  z slowest.
    std::vector<qd> g, gw, z, zw;
    gauss_legendre(p + 1, g, gw);
    gauss_legendre(p, z, zw);
    std::vector<P3> V;
    for (auto& v : TRI_V) V.push_back({(qd)v[0], (qd)v[1], 0});
    std::vector<P3> tsol, tface, tint;
    for (auto& lam : centroid_lattice(2, p)) tsol.push_back(bary(lam, V));
    for (auto& lam : simplex_rule(2, (p + 1) * (p + 2) / 2)) tface.push_back(bary(lam, V));
    for (auto& lam : simplex_rule(2, p * (p + 1) / 2)) tint.push_back(bary(lam, V));
    for (auto zz : g)
      for (auto& x : tsol) R.xsol.push_back({x[0], x[1], zz});
    const qd s2 = 1 / sqrtq(2.0Q);
    P3 fn[5] = {{0, 0, -1}, {0, 0, 1}, {0, -1, 0}, {s2, s2, 0}, {-1, 0, 0}};
    r.nfaces = 5;
    r.nfp = (p + 1) * (p + 1);
    r.face_ptr.push_back(0);
    for (int f = 0; f < 5; ++f) {
      r.face_normal.push_back(to_d(fn[f]));
      std::vector<int> fv;
      for (int k = 0; k < 4; ++k)
        if (PRI_F[f][k] >= 0) fv.push_back(PRI_F[f][k]);
      r.face_verts.push_back(fv);
      if (f < 2) {
        for (auto& x : tface) {
          R.xext.push_back({x[0], x[1], f == 0 ? (qd)-1 : (qd)1});
          R.next_n.push_back(fn[f]);
          r.ext_face.push_back(f);
        }
      } else {
        const P3 &A = V[TRI_F[f - 2][0]], &B = V[TRI_F[f - 2][1]];
        for (auto zz : g)
          for (int t = 0; t <= p; ++t) {
            qd lam = (g[t] + 1) / 2;
            R.xext.push_back({A[0] + lam * (B[0] - A[0]), A[1] + lam * (B[1] - A[1]), zz});
            R.next_n.push_back(fn[f]);
            r.ext_face.push_back(f);
          }
      }
      r.face_ptr.push_back((int)R.xext.size());
    }
    for (auto zz : g)
      for (auto& x : tint) {
        for (int d = 0; d < 2; ++d) {
          r.int_u.push_back((int)R.xu.size());
          r.int_dir.push_back(d);
        }
        R.xu.push_back({x[0], x[1], zz});
      }
    for (auto zz : z)
      for (auto& x : tface) {
        r.int_u.push_back((int)R.xu.size());
        r.int_dir.push_back(2);
        R.xu.push_back({x[0], x[1], zz});
      }
  } else if (etype_tensor(etype)) {
    std::vector<qd> g, gw, z, zw;
    gauss_legendre(p + 1, g, gw);
    gauss_legendre(p, z, zw);
    int n = p + 1;
    if (D == 2) {
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) R.xsol.push_back({g[i], g[j], 0});
    } else {
      for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j)
          for (int i = 0; i < n; ++i) R.xsol.push_back({g[i], g[j], g[k]});
    }
    r.nfaces = 2 * D;
    r.nfp = D == 2 ? n : n * n;
    for (int d = 0; d < D; ++d)
      for (int s = 0; s < 2; ++s) {
        int f = 2 * d + s;
        qd val = 2 * s - 1;
        P3 nv = {0, 0, 0};
        nv[d] = val;
        r.face_normal.push_back(to_d(nv));
        int o[2], no = 0;
        for (int c = 0; c < D; ++c)
          if (c != d) o[no++] = c;
        if (D == 2) {
          for (int t = 0; t < n; ++t) {
            P3 x = {0, 0, 0};
            x[d] = val;
            x[o[0]] = g[t];
            R.xext.push_back(x); R.next_n.push_back(nv); r.ext_face.push_back(f);
          }
        } else {
          for (int tb = 0; tb < n; ++tb)
            for (int ta = 0; ta < n; ++ta) {
              P3 x = {0, 0, 0};
              x[d] = val;
              x[o[0]] = g[ta];
              x[o[1]] = g[tb];
              R.xext.push_back(x); R.next_n.push_back(nv); r.ext_face.push_back(f);
            }
        }
      }
    for (int d = 0; d < D; ++d) {
      const std::vector<qd>* ax[3];
      for (int c = 0; c < 3; ++c) ax[c] = (c == d) ? &z : &g;
      int n2 = D == 3 ? (int)ax[2]->size() : 1;
      for (int c2 = 0; c2 < n2; ++c2)
        for (int c1 = 0; c1 < (int)ax[1]->size(); ++c1)
          for (int c0 = 0; c0 < (int)ax[0]->size(); ++c0) {
            r.int_u.push_back((int)R.xu.size());
            r.int_dir.push_back(d);
            R.xu.push_back({(*ax[0])[c0], (*ax[1])[c1], D == 3 ? (*ax[2])[c2] : (qd)0});
          }
    }
  } else {
    std::vector<P3> V;
    if (D == 2)
      for (auto& v : TRI_V) V.push_back({(qd)v[0], (qd)v[1], 0});
    else
      for (auto& v : TET_V) V.push_back({(qd)v[0], (qd)v[1], (qd)v[2]});
    for (auto& lam : centroid_lattice(D, p)) R.xsol.push_back(bary(lam, V));
    if (D == 2) {
      std::vector<qd> g, gw;
      gauss_legendre(p + 1, g, gw);
      qd s2 = 1 / sqrtq(2.0Q);
      P3 fn[3] = {{0, -1, 0}, {s2, s2, 0}, {-1, 0, 0}};
      r.nfaces = 3;
      r.nfp = p + 1;
      for (int f = 0; f < 3; ++f) {
        r.face_normal.push_back(to_d(fn[f]));
        r.face_verts.push_back({TRI_F[f][0], TRI_F[f][1]});
        for (int t = 0; t <= p; ++t) {
          qd lam = (g[t] + 1) / 2;
          const P3 &A = V[TRI_F[f][0]], &B = V[TRI_F[f][1]];
          R.xext.push_back({A[0] + lam * (B[0] - A[0]), A[1] + lam * (B[1] - A[1]), 0});
          R.next_n.push_back(fn[f]);
          r.ext_face.push_back(f);
        }
      }
    } else {
      qd s3 = 1 / sqrtq(3.0Q);
      P3 fn[4] = {{0, 0, -1}, {0, -1, 0}, {s3, s3, s3}, {-1, 0, 0}};
      auto fl = simplex_rule(2, (p + 1) * (p + 2) / 2);
      r.nfaces = 4;
      r.nfp = (int)fl.size();
      for (int f = 0; f < 4; ++f) {
        r.face_normal.push_back(to_d(fn[f]));
        r.face_verts.push_back({TET_F[f][0], TET_F[f][1], TET_F[f][2]});
        std::vector<P3> fv = {V[TET_F[f][0]], V[TET_F[f][1]], V[TET_F[f][2]]};
        for (auto& lam : fl) {
          R.xext.push_back(bary(lam, fv));
          R.next_n.push_back(fn[f]);
          r.ext_face.push_back(f);
        }
      }
    }
    int nu = D == 2 ? p * (p + 1) / 2 : p * (p + 1) * (p + 2) / 6;
    for (auto& lam : simplex_rule(D, nu)) R.xu.push_back(bary(lam, V));
    for (int u = 0; u < (int)R.xu.size(); ++u)
      for (int d = 0; d < D; ++d) {
        r.int_u.push_back(u);
        r.int_dir.push_back(d);
      }
  }
  if (r.face_ptr.empty())
    for (int f = 0; f <= r.nfaces; ++f) r.face_ptr.push_back(f * r.nfp);
  r.nsol = (int)R.xsol.size();
  r.next = (int)R.xext.size();
  r.nu = (int)R.xu.size();
  r.nint = (int)r.int_u.size();
  for (auto& x : R.xsol) r.xsol.push_back(to_d(x));
  for (auto& x : R.xext) r.xext.push_back(to_d(x));
  for (auto& x : R.xu) r.xu.push_back(to_d(x));
  for (auto& x : R.next_n) r.ext_normal.push_back(to_d(x));
  return R;
}

RefElement build_reference(int etype, int p) { return build_ref_q(etype, p).r; }

// ------------------------------------------------------------------ operators
static qd lag(const std::vector<qd>& nd, int j, qd x) {
  qd v = 1;
  for (size_t k = 0; k < nd.size(); ++k)
    if ((int)k != j) v *= (x - nd[k]) / (nd[j] - nd[k]);
  return v;
}
static qd lag_d(const std::vector<qd>& nd, int j, qd x) {
  qd s = 0;
  for (size_t m = 0; m < nd.size(); ++m) {
    if ((int)m == j) continue;
    qd t = 1 / (nd[j] - nd[m]);
    for (size_t k = 0; k < nd.size(); ++k)
      if ((int)k != j && k != m) t *= (x - nd[k]) / (nd[j] - nd[k]);
    s += t;
  }
  return s;
}

static void finish_gradient_ops(Operators& O) {
  const RefElement& r = O.ref;
  int D = r.nd, ns = r.nsol;
  O.M16 = Mat(D * ns, r.next);
  O.M15 = Mat(D * ns, r.nint);
  for (int d = 0; d < D; ++d) {
    for (int e = 0; e < r.next; ++e) {
      double nd = r.ext_normal[e][d];
      if (nd != 0.0)
        for (int s = 0; s < ns; ++s) O.M16(d * ns + s, e) = nd * O.M14(s, e);
    }
    for (int i = 0; i < r.nint; ++i)
      if (r.int_dir[i] == d)
        for (int s = 0; s < ns; ++s) O.M15(d * ns + s, i) = O.M13(s, i);
  }
  O.P = Mat(r.nint, r.nu);
  O.M19P2 = Mat(r.nint, D * r.nu);
  for (int i = 0; i < r.nint; ++i) {
    O.P(i, r.int_u[i]) = 1.0;
    O.M19P2(i, r.int_dir[i] * r.nu + r.int_u[i]) = 1.0;
  }
}

static Operators tensor_operators(int etype, int p) {
  RefQ R = build_ref_q(etype, p);
  Operators O;
  O.ref = R.r;
  const RefElement& r = O.ref;
  int D = r.nd, n = p + 1, ns = r.nsol;
  std::vector<qd> g, gw, z, zw;
  gauss_legendre(n, g, gw);
  gauss_legendre(p, z, zw);
  std::vector<qd> fl;  // flux line {-1, zeros(P_p), +1}
  fl.push_back(-1);
  for (auto v : z) fl.push_back(v);
  fl.push_back(1);
  auto sidx = [&](int s, int c) { int t = s; for (int k = 0; k < c; ++k) t /= n; return t % n; };
  O.M0 = Mat(r.next, ns);
  O.M14 = Mat(ns, r.next);
  for (int e = 0; e < r.next; ++e) {
    int f = r.ext_face[e], d = f / 2, side = f % 2;
    qd xd = side ? 1 : -1;
    for (int s = 0; s < ns; ++s) {
      bool tang = true;
      for (int c = 0; c < D; ++c)
        if (c != d && qabs(R.xext[e][c] - g[sidx(s, c)]) > 1e-25Q) tang = false;
      if (!tang) continue;
      O.M0(e, s) = (double)lag(g, sidx(s, d), xd);
      // RT nodal function of this DOF: n_d * L_end(x_d) * prod ell; div = n_d L_end'(x_d)
      int endk = side ? p + 1 : 0;
      O.M14(s, e) = (double)((side ? 1 : -1) * lag_d(fl, endk, g[sidx(s, d)]));
    }
  }
  O.M12 = Mat(r.nu, ns);
  O.M13 = Mat(ns, r.nint);
  for (int i = 0; i < r.nint; ++i) {
    int d = r.int_dir[i], u = r.int_u[i];
    int a = -1;
    for (int k = 0; k < p; ++k)
      if (qabs(R.xu[u][d] - z[k]) < 1e-25Q) a = k;
    for (int s = 0; s < ns; ++s) {
      bool tang = true;
      for (int c = 0; c < D; ++c)
        if (c != d && qabs(R.xu[u][c] - g[sidx(s, c)]) > 1e-25Q) tang = false;
      if (!tang) continue;
      O.M12(u, s) = (double)lag(g, sidx(s, d), z[a]);
      O.M13(s, i) = (double)lag_d(fl, a + 1, g[sidx(s, d)]);
    }
  }
  O.w.assign(ns, 0.0);
  for (int s = 0; s < ns; ++s) {
    qd w = 1;
    for (int c = 0; c < D; ++c) w *= gw[sidx(s, c)];
    O.w[s] = (double)w;
  }
  O.cond_flux = 0.0;
  finish_gradient_ops(O);
  // FR data: solution-basis derivatives along each axis (1D Lagrange on the GL nodes)
  // and the FR-DG correction divergence (Radau polynomials of degree p+1 along the
  // face normal: g_L = (-1)^{p+1}/2 (P_{p+1} - P_p), g_R(x) = g_L(-x))
  O.Dsol.assign(D, Mat(ns, ns));
  for (int d = 0; d < D; ++d)
    for (int s = 0; s < ns; ++s)
      for (int q = 0; q < ns; ++q) {
        bool tang = true;
        for (int c = 0; c < D; ++c)
          if (c != d && sidx(s, c) != sidx(q, c)) tang = false;
        if (tang) O.Dsol[d](s, q) = (double)lag_d(g, sidx(q, d), g[sidx(s, d)]);
      }
  auto legd = [](int n, qd x) {  // P_n'(x) for |x| < 1
    qd pn, pm;
    legendre_pair(n, x, pn, pm);
    return n == 0 ? (qd)0 : (qd)n * (x * pn - pm) / (x * x - 1);
  };
  const qd sg = (p + 1) % 2 ? -1 : 1;  // (-1)^{p+1}
  O.Mc = Mat(ns, r.next);
  for (int e = 0; e < r.next; ++e) {
    int f = r.ext_face[e], d = f / 2, side = f % 2;
    for (int s = 0; s < ns; ++s) {
      bool tang = true;
      for (int c = 0; c < D; ++c)
        if (c != d && qabs(R.xext[e][c] - g[sidx(s, c)]) > 1e-25Q) tang = false;
      if (!tang) continue;
      const qd xi = g[sidx(s, d)];
      if (side == 0) O.Mc(s, e) = (double)(-(sg / 2) * (legd(p + 1, xi) - legd(p, xi)));     // div(-e_d g_L)
      else O.Mc(s, e) = (double)(-(sg / 2) * (legd(p + 1, -xi) - legd(p, -xi)));            // div(+e_d g_R)
    }
  }
  return O;
}

// monomials in xi = (x+1)/2
static qd mono(const std::vector<int>& e, const P3& x) {
  qd v = 1;
  for (size_t c = 0; c < e.size(); ++c) {
    qd xi = (x[c] + 1) / 2;
    for (int k = 0; k < e[c]; ++k) v *= xi;
  }
  return v;
}
// d/dx_c of the xi-monomial = (1/2) d/dxi_c
static qd mono_dx(const std::vector<int>& e, const P3& x, int c) {
  if (e[c] == 0) return 0;
  std::vector<int> ee = e;
  ee[c] -= 1;
  return (qd)e[c] * mono(ee, x) / 2;
}

static void exps_total(int D, int p, std::vector<std::vector<int>>& out) {
  for (int d = 0; d <= p; ++d) {
    std::vector<std::vector<int>> t;
    exps_eq(D, d, t);
    for (auto& e : t) out.push_back(e);
  }
}

// Quadrature on the unit m-simplex {t >= 0, sum t <= 1} (m = 1, 2, 3) by the collapsed
// (Duffy) product of nq-point Gauss-Legendre rules: exact for degree <= 2 nq - m.
static void unit_simplex_rule(int m, int nq, std::vector<std::array<qd, 3>>& pts, std::vector<qd>& wts) {
  std::vector<qd> g, gw;
  gauss_legendre(nq, g, gw);
  pts.clear();
  wts.clear();
  for (int i = 0; i < nq; ++i) {
    const qd a = (g[i] + 1) / 2, wa = gw[i] / 2;
    if (m == 1) {
      pts.push_back({a, 0, 0});
      wts.push_back(wa);
      continue;
    }
    for (int j = 0; j < nq; ++j) {
      const qd b = (g[j] + 1) / 2, wb = gw[j] / 2;
      if (m == 2) {
        pts.push_back({a, (1 - a) * b, 0});
        wts.push_back(wa * wb * (1 - a));
        continue;
      }
      for (int k = 0; k < nq; ++k) {
        const qd c = (g[k] + 1) / 2, wc = gw[k] / 2;
        pts.push_back({a, (1 - a) * b, (1 - a) * (1 - b) * c});
        wts.push_back(wa * wb * wc * (1 - a) * (1 - a) * (1 - b));
      }
    }
  }
}

// FR-DG correction on simplices (l.371-373: the correction functions that recover nodal
// DG): the DG lifting Mc = M^-1 L with M_rs = int l_r l_s over the reference simplex and
// L_{r nu} = int_{face(nu)} l_r ell_nu dS~, ell_nu the degree-p Lagrange basis of the
// face's flux points in the face parameters; integrals by collapsed Gauss rules.
// Y: solution basis coefficients (l_r = sum_k Y[k][r] mono(Ptot[k], x)).
static Mat simplex_dg_lift(const RefQ& R, const std::vector<qd>& Y, const std::vector<std::vector<int>>& Ptot) {
  const RefElement& r = R.r;
  const int D = r.nd, ns = r.nsol, nq = r.p + 3;
  std::vector<P3> V;
  if (D == 2)
    for (auto& v : TRI_V) V.push_back({(qd)v[0], (qd)v[1], 0});
  else
    for (auto& v : TET_V) V.push_back({(qd)v[0], (qd)v[1], (qd)v[2]});
  auto lval = [&](const P3& x, std::vector<qd>& out) {
    out.assign(ns, 0);
    for (int k = 0; k < ns; ++k) {
      const qd m = mono(Ptot[k], x);
      for (int rr = 0; rr < ns; ++rr) out[rr] += Y[(size_t)k * ns + rr] * m;
    }
  };
  auto affine = [&](const std::vector<P3>& verts, const std::array<qd, 3>& t) {
    P3 x = verts[0];
    for (size_t i = 1; i < verts.size(); ++i)
      for (int c = 0; c < 3; ++c) x[c] += t[i - 1] * (verts[i][c] - verts[0][c]);
    return x;
  };
  std::vector<std::array<qd, 3>> pts;
  std::vector<qd> wts, lv;
  // mass matrix (|det J| of the unit-simplex map: 4 tri, 8 tet)
  std::vector<qd> M((size_t)ns * ns, 0);
  unit_simplex_rule(D, nq, pts, wts);
  const qd vdet = D == 2 ? 4 : 8;
  for (size_t q = 0; q < pts.size(); ++q) {
    lval(affine(V, pts[q]), lv);
    for (int a = 0; a < ns; ++a)
      for (int b = 0; b < ns; ++b) M[(size_t)a * ns + b] += wts[q] * vdet * lv[a] * lv[b];
  }
  // face lifts
  std::vector<qd> L((size_t)ns * r.next, 0);
  std::vector<std::vector<int>> fsp;
  exps_total(D - 1, r.p, fsp);
  const int nfp = (int)fsp.size();
  unit_simplex_rule(D - 1, nq, pts, wts);
  for (int f = 0; f < r.nfaces; ++f) {
    std::vector<P3> fv;
    for (int k = 0; k < D; ++k) fv.push_back(V[D == 2 ? TRI_F[f][k] : TET_F[f][k]]);
    // Gram matrix of the edge vectors, face measure scale sqrt(det G)
    qd G[2][2] = {{0, 0}, {0, 0}};
    for (int a = 0; a < D - 1; ++a)
      for (int b = 0; b < D - 1; ++b)
        for (int c = 0; c < 3; ++c) G[a][b] += (fv[a + 1][c] - fv[0][c]) * (fv[b + 1][c] - fv[0][c]);
    const qd gdet = D == 2 ? G[0][0] : G[0][0] * G[1][1] - G[0][1] * G[1][0];
    const qd scale = sqrtq(gdet);
    std::vector<int> nus;
    for (int nu = 0; nu < r.next; ++nu)
      if (r.ext_face[nu] == f) nus.push_back(nu);
    if ((int)nus.size() != nfp) throw std::runtime_error("face point count != dim P_p(face)");
    // face parameters of the face points: G t = T^T (x - x0)
    std::vector<std::array<qd, 3>> tf;
    for (int nu : nus) {
      qd rhs[2] = {0, 0};
      for (int a = 0; a < D - 1; ++a)
        for (int c = 0; c < 3; ++c) rhs[a] += (fv[a + 1][c] - fv[0][c]) * (R.xext[nu][c] - fv[0][c]);
      if (D == 2) tf.push_back({rhs[0] / G[0][0], 0, 0});
      else
        tf.push_back({(rhs[0] * G[1][1] - G[0][1] * rhs[1]) / gdet, (G[0][0] * rhs[1] - G[1][0] * rhs[0]) / gdet, 0});
    }
    auto tmono = [&](const std::vector<int>& e, const std::array<qd, 3>& t) {
      qd v = 1;
      for (size_t c = 0; c < e.size(); ++c)
        for (int k = 0; k < e[c]; ++k) v *= t[c];
      return v;
    };
    // face Lagrange basis: B = V^T (B[j][i] = t_j^e_i), Z = B^-1, ell_j = sum_i Z[i][j] t^e_i
    std::vector<qd> B((size_t)nfp * nfp), Z((size_t)nfp * nfp, 0);
    for (int j = 0; j < nfp; ++j)
      for (int i = 0; i < nfp; ++i) B[(size_t)j * nfp + i] = tmono(fsp[i], tf[j]);
    for (int i = 0; i < nfp; ++i) Z[(size_t)i * nfp + i] = 1;
    gj_solve(B, nfp, Z, nfp);
    for (size_t q = 0; q < pts.size(); ++q) {
      lval(affine(fv, pts[q]), lv);
      std::vector<qd> tm(nfp);
      for (int i = 0; i < nfp; ++i) tm[i] = tmono(fsp[i], pts[q]);
      for (int j = 0; j < nfp; ++j) {
        qd ell = 0;
        for (int i = 0; i < nfp; ++i) ell += Z[(size_t)i * nfp + j] * tm[i];
        const qd w = wts[q] * scale * ell;
        for (int a = 0; a < ns; ++a) L[(size_t)a * r.next + nus[j]] += w * lv[a];
      }
    }
  }
  gj_solve(M, ns, L, r.next);  // L <- M^-1 L
  Mat Mc(ns, r.next);
  for (int a = 0; a < ns; ++a)
    for (int nu = 0; nu < r.next; ++nu) Mc(a, nu) = (double)L[(size_t)a * r.next + nu];
  return Mc;
}

static Operators simplex_operators(int etype, int p) {
  RefQ R = build_ref_q(etype, p);
  Operators O;
  O.ref = R.r;
  const RefElement& r = O.ref;
  int D = r.nd, ns = r.nsol;
  // RT span: simplex P_p^D (+) xi Pbar_p(xi) (App. A l.2364; affine invariant);
  // prism [P_p(xi0, xi1)^2 (+) (xi0, xi1) Pbar_p(xi0, xi1)] P_p(xi2) x P_p(xi0, xi1) P_{p+1}(xi2)
  // (l.2640-2642; invariant under the affine x -> xi); solution span P_p (simplex) or
  // P_p(xi0, xi1) P_p(xi2) (prism, l.2731-2733)
  struct VT { std::vector<std::pair<int, std::vector<int>>> terms; };
  std::vector<VT> span;
  std::vector<std::vector<int>> Ptot, Phom;
  if (etype == PRI) {
    std::vector<std::vector<int>> T2, H2;
    exps_total(2, p, T2);
    exps_eq(2, p, H2);
    for (int c = 0; c <= p; ++c)
      for (auto& e : T2) Ptot.push_back({e[0], e[1], c});
    for (int c = 0; c <= p; ++c) {
      for (int k = 0; k < 2; ++k)
        for (auto& e : T2) span.push_back({{{k, {e[0], e[1], c}}}});
      for (auto& e : H2) span.push_back({{{0, {e[0] + 1, e[1], c}}, {1, {e[0], e[1] + 1, c}}}});
    }
    for (int c = 0; c <= p + 1; ++c)
      for (auto& e : T2) span.push_back({{{2, {e[0], e[1], c}}}});
  } else {
    exps_total(D, p, Ptot);
    exps_eq(D, p, Phom);
    for (int c = 0; c < D; ++c)
      for (auto& e : Ptot) span.push_back({{{c, e}}});
    for (auto& e : Phom) {
      VT v;
      for (int c = 0; c < D; ++c) {
        auto ee = e;
        ee[c] += 1;
        v.terms.push_back({c, ee});
      }
      span.push_back(v);
    }
  }
  int nf = (int)span.size();
  if (nf != r.next + r.nint) throw std::runtime_error("RT span dimension mismatch");
  std::vector<P3> fx;
  std::vector<P3> fn;
  for (int e = 0; e < r.next; ++e) { fx.push_back(R.xext[e]); fn.push_back(R.next_n[e]); }
  for (int i = 0; i < r.nint; ++i) {
    fx.push_back(R.xu[r.int_u[i]]);
    P3 nv = {0, 0, 0};
    nv[r.int_dir[i]] = 1;
    fn.push_back(nv);
  }
  // flux Vandermonde V[k][s] = psi_k(x_s).n_s ; nodal functions C = V^-1 (C V = I)
  // We need DT = C * divpsi (nf x ns): solve V^T C^T = I  ->  C = (V^T)^-1 ... use
  // C V = I  <=>  V^T C^T = I; then DT = C divpsi  <=>  V^T ... solve V^T Y = ? .
  // Simplest: form A = V^T (n x n), solve A X = I for X = C^T, then DT = X^T divpsi.
  std::vector<qd> A((size_t)nf * nf), X((size_t)nf * nf, 0);
  for (int k = 0; k < nf; ++k)
    for (int s = 0; s < nf; ++s) {
      qd v = 0;
      for (auto& t : span[k].terms)
        if (fn[s][t.first] != 0) v += mono(t.second, fx[s]) * fn[s][t.first];
      A[(size_t)s * nf + k] = v;  // A = V^T
    }
  double vnorm = 0;
  {
    std::vector<double> colsum(nf, 0.0);
    for (int s = 0; s < nf; ++s)
      for (int k = 0; k < nf; ++k) colsum[k] += std::fabs((double)A[(size_t)s * nf + k]);
    for (double v : colsum) vnorm = std::max(vnorm, v);
  }
  for (int i = 0; i < nf; ++i) X[(size_t)i * nf + i] = 1;
  gj_solve(A, nf, X, nf);  // X = (V^T)^-1 = C^T
  double inorm = 0;
  {
    std::vector<double> colsum(nf, 0.0);
    for (int i = 0; i < nf; ++i)
      for (int j = 0; j < nf; ++j) colsum[j] += std::fabs((double)X[(size_t)i * nf + j]);
    for (double v : colsum) inorm = std::max(inorm, v);
  }
  O.cond_flux = vnorm * inorm;
  if (O.cond_flux > 1e12) throw std::runtime_error("flux Vandermonde ill-conditioned (> 1e12)");
  // divergence of nodal function r at solution point s: sum_k C[r][k] div psi_k(x_s),
  // C[r][k] = X[k][r]
  std::vector<qd> divpsi((size_t)nf * ns);
  for (int k = 0; k < nf; ++k)
    for (int s = 0; s < ns; ++s) {
      qd v = 0;
      for (auto& t : span[k].terms) v += mono_dx(t.second, R.xsol[s], t.first);
      divpsi[(size_t)k * ns + s] = v;
    }
  O.M14 = Mat(ns, r.next);
  O.M13 = Mat(ns, r.nint);
  for (int rr = 0; rr < nf; ++rr)
    for (int s = 0; s < ns; ++s) {
      qd v = 0;
      for (int k = 0; k < nf; ++k) v += X[(size_t)k * nf + rr] * divpsi[(size_t)k * ns + s];
      if (rr < r.next) O.M14(s, rr) = (double)v;
      else O.M13(s, rr - r.next) = (double)v;
    }
  // solution basis P_p in xi monomials
  int nb = (int)Ptot.size();
  if (nb != ns) throw std::runtime_error("solution span mismatch");
  std::vector<qd> B((size_t)ns * ns), Y((size_t)ns * ns, 0);
  for (int k = 0; k < ns; ++k)
    for (int s = 0; s < ns; ++s) B[(size_t)s * ns + k] = mono(Ptot[k], R.xsol[s]);  // B = Vu^T
  for (int i = 0; i < ns; ++i) Y[(size_t)i * ns + i] = 1;
  gj_solve(B, ns, Y, ns);  // Y = (Vu^T)^-1 ; l_r = sum_k Y[k][r] phi_k
  auto interp = [&](const std::vector<P3>& pts, Mat& M) {
    M = Mat((int)pts.size(), ns);
    for (size_t q = 0; q < pts.size(); ++q)
      for (int rr = 0; rr < ns; ++rr) {
        qd v = 0;
        for (int k = 0; k < ns; ++k) v += Y[(size_t)k * ns + rr] * mono(Ptot[k], pts[q]);
        M((int)q, rr) = (double)v;
      }
  };
  interp(R.xext, O.M0);
  interp(R.xu, O.M12);
  // FR data: solution-basis derivatives and the FR-DG correction (DG lifting)
  O.Dsol.assign(D, Mat(ns, ns));
  for (int d = 0; d < D; ++d)
    for (int s = 0; s < ns; ++s)
      for (int rr = 0; rr < ns; ++rr) {
        qd v = 0;
        for (int k = 0; k < ns; ++k) v += Y[(size_t)k * ns + rr] * mono_dx(Ptot[k], R.xsol[s], d);
        O.Dsol[d](s, rr) = (double)v;
      }
  // weights: int over the reference simplex of xi^e = 2^D prod e_i! / (|e|+D)!; prism:
  // the triangle's 4 e0! e1! / (e0+e1+2)! times int_{-1}^{1} xi2^e2 dz = 2 / (e2 + 1)
  O.w.assign(ns, 0.0);
  const int DS = etype == PRI ? 2 : D;  // simplex factor dimension
  for (int rr = 0; rr < ns; ++rr) {
    qd v = 0;
    for (int k = 0; k < ns; ++k) {
      const auto& e = Ptot[k];
      qd num = 1;
      int tot = DS;
      for (int c = 0; c < DS; ++c) {
        for (int m = 2; m <= e[c]; ++m) num *= m;
        tot += e[c];
      }
      qd den = 1;
      for (int m = 2; m <= tot; ++m) den *= m;
      qd val = num / den * (DS == 2 ? 4 : 8);
      if (etype == PRI) val *= (qd)2 / (e[2] + 1);
      v += Y[(size_t)k * ns + rr] * val;
    }
    O.w[rr] = (double)v;
  }
  if (etype != PRI) O.Mc = simplex_dg_lift(R, Y, Ptot);
  finish_gradient_ops(O);
  return O;
}

// Degree-`degree` cubature of the reference element (TGV ensemble averages, l.2075) and
// the solution-basis interpolation B(q, r) = l_r(x_q).  Tensor: Gauss-Legendre products
// with degree/2 + 1 points per axis; simplex: collapsed (Duffy) Gauss-Legendre products
// with (degree + D - 1)/2 + 1 points per direction, mapped affinely (|det| 4 tri, 8 tet).
// 1D factor of the tensor-element cubature interpolation: B1[q][t] = l_t(g_q), the
// degree-p Lagrange basis on the p+1 Gauss-Legendre solution points at the degree/2+1
// Gauss-Legendre cubature points, so that cubature_interp's B = B1 (x) B1 (x) B1 (x
// fastest); row-major nq x (p+1)
void cubature_interp_1d(int p, int degree, std::vector<double>& B1) {
  std::vector<qd> g, gw, gs, gsw;
  gauss_legendre(degree / 2 + 1, g, gw);
  gauss_legendre(p + 1, gs, gsw);
  B1.assign(g.size() * (p + 1), 0.0);
  for (size_t q = 0; q < g.size(); ++q)
    for (int t = 0; t <= p; ++t) B1[q * (p + 1) + t] = (double)lag(gs, t, g[q]);
}

void cubature_interp(int etype, int p, int degree, std::vector<double>& w, Mat& B) {
  if (etype == PRI) throw std::runtime_error("unsupported: diagnostics cubature on prisms");
  RefQ R = build_ref_q(etype, p);
  const RefElement& r = R.r;
  const int D = r.nd, ns = r.nsol;
  std::vector<P3> xq;
  std::vector<qd> wq;
  if (etype_tensor(etype)) {
    std::vector<qd> g, gw;
    gauss_legendre(degree / 2 + 1, g, gw);
    const int nq = (int)g.size();
    const int tot = D == 2 ? nq * nq : nq * nq * nq;
    for (int q = 0; q < tot; ++q) {
      const int i = q % nq, j = (q / nq) % nq, k = q / (nq * nq);
      xq.push_back({g[i], g[j], D == 3 ? g[k] : (qd)0});
      wq.push_back(gw[i] * gw[j] * (D == 3 ? gw[k] : (qd)1));
    }
    std::vector<qd> gs, gsw;
    gauss_legendre(p + 1, gs, gsw);
    const int n = p + 1;
    B = Mat((int)xq.size(), ns);
    for (size_t q = 0; q < xq.size(); ++q)
      for (int s = 0; s < ns; ++s) {
        qd v = 1;
        int t = s;
        for (int c = 0; c < D; ++c, t /= n) v *= lag(gs, t % n, xq[q][c]);
        B((int)q, s) = (double)v;
      }
  } else {
    std::vector<std::array<qd, 3>> tp;
    unit_simplex_rule(D, (degree + D - 1) / 2 + 1, tp, wq);
    std::vector<P3> V;
    if (D == 2)
      for (auto& v : TRI_V) V.push_back({(qd)v[0], (qd)v[1], 0});
    else
      for (auto& v : TET_V) V.push_back({(qd)v[0], (qd)v[1], (qd)v[2]});
    for (size_t q = 0; q < tp.size(); ++q) {
      P3 x = V[0];
      for (int i = 0; i < D; ++i)
        for (int c = 0; c < 3; ++c) x[c] += tp[q][i] * (V[i + 1][c] - V[0][c]);
      xq.push_back(x);
      wq[q] *= D == 2 ? 4 : 8;
    }
    std::vector<std::vector<int>> Ptot;
    exps_total(D, p, Ptot);
    std::vector<qd> A((size_t)ns * ns), Y((size_t)ns * ns, 0);
    for (int k = 0; k < ns; ++k)
      for (int s = 0; s < ns; ++s) A[(size_t)s * ns + k] = mono(Ptot[k], R.xsol[s]);
    for (int i = 0; i < ns; ++i) Y[(size_t)i * ns + i] = 1;
    gj_solve(A, ns, Y, ns);  // l_r = sum_k Y[k][r] phi_k
    B = Mat((int)xq.size(), ns);
    for (size_t q = 0; q < xq.size(); ++q)
      for (int rr = 0; rr < ns; ++rr) {
        qd v = 0;
        for (int k = 0; k < ns; ++k) v += Y[(size_t)k * ns + rr] * mono(Ptot[k], xq[q]);
        B((int)q, rr) = (double)v;
      }
  }
  w.assign(wq.size(), 0.0);
  for (size_t q = 0; q < wq.size(); ++q) w[q] = (double)wq[q];
}

Operators build_operators(int etype, int p, int scheme) {
  Operators O;
  if (etype_tensor(etype)) O = tensor_operators(etype, p);
  else if (etype == TRI || etype == TET || etype == PRI) O = simplex_operators(etype, p);
  else throw std::runtime_error("unknown element type");
  if (scheme < 0 || scheme > 2) throw std::runtime_error("unsupported scheme");
  if (etype == PRI && scheme != 0) throw std::runtime_error("unsupported: FR schemes on prisms");
  O.scheme = scheme;
  if (scheme == 1) O.Mc = O.M14;  // FR-SDRT: div g_nu = div psi_nu (l.407-413)
  return O;
}

}  // namespace sdrt
