// Reference elements, point sets and Appendix-B operators (host, quad precision).
// Product-side construction; shares no code with oracle/.
#pragma once
#include <array>
#include <string>
#include <vector>

namespace sdrt {

enum EType { QUAD = 0, TRI = 1, HEX = 2, TET = 3, PRI = 4 };

inline int etype_dim(int et) { return (et == QUAD || et == TRI) ? 2 : 3; }
inline int etype_nsub(int et) { return (et == TRI || et == PRI) ? 2 : (et == TET ? 6 : 1); }
inline bool etype_tensor(int et) { return et == QUAD || et == HEX; }

// Dense row-major double matrix.
struct Mat {
  int rows = 0, cols = 0;
  std::vector<double> a;
  Mat() {}
  Mat(int r, int c) : rows(r), cols(c), a((size_t)r * c, 0.0) {}
  double& operator()(int i, int j) { return a[(size_t)i * cols + j]; }
  double operator()(int i, int j) const { return a[(size_t)i * cols + j]; }
};

struct RefElement {
  int etype, p, nd;
  int nsol, next, nint, nu, nfaces, nfp;
  std::vector<std::array<double, 3>> xsol, xext, xu;  // reference coordinates (rounded)
  std::vector<std::array<double, 3>> ext_normal;       // outward unit normals per ext point
  std::vector<int> ext_face;                            // face id per ext point
  std::vector<int> int_u, int_dir;                      // per internal point
  std::vector<std::array<double, 3>> face_normal;       // per face
  std::vector<std::vector<int>> face_verts;             // reference vertex ids per face (simplex, prism)
  std::vector<int> face_ptr;                            // face f: ext points face_ptr[f] .. face_ptr[f+1]
  int face_nfp(int f) const { return face_ptr[f + 1] - face_ptr[f]; }
};

struct Operators {
  RefElement ref;
  Mat M0, M12, M13, M14, M15, M16, P, M19P2;
  std::vector<double> w;  // int of the solution nodal basis over the reference element
  double cond_flux = 0.0;
  // flux reconstruction (NEXT row N1): scheme 0 SDRT, 1 FR-SDRT,
  // 2 FR-DG; Dsol[d](s, r) = d l_r / d x~_d (x~_s); Mc(s, nu) = div g_nu (x~_s)
  int scheme = 0;
  std::vector<Mat> Dsol;
  Mat Mc;
};

// Build; throws std::runtime_error with a message on failure.
RefElement build_reference(int etype, int p);
Operators build_operators(int etype, int p, int scheme = 0);

// Cubature exact to `degree` on the reference element (weights w) and the solution-basis
// interpolation B(q, r) = l_r(x_q) (TGV diagnostics, l.2075).
void cubature_interp(int etype, int p, int degree, std::vector<double>& w, Mat& B);
void cubature_interp_1d(int p, int degree, std::vector<double>& B1);

// Reference vertices of the simplices (x~ of vertex k), used by mesh code.
void simplex_ref_vertices(int etype, std::vector<std::array<double, 3>>& V);

}  // namespace sdrt
