// Element stiffness of the Q4 (plane stress) / Hex8 (isotropic) element by
// 2-point Gauss quadrature -- the reference's element_stiffness (mesh.py:254):
// KE = sum_q w_q detJ B_q^T D B_q, symmetrised.  Local dof = local_node*ndim + c,
// local nodes counter-clockwise (bottom face then top face in 3D).
#pragma once
#include <cmath>
#include <vector>

namespace tmg {

inline void constitutive_matrix(int ndim, double E, double nu, double* D /*6x6 or 3x3*/) {
  if (ndim == 2) {
    const double c = E / (1.0 - nu * nu);
    const double v[9] = {c, c * nu, 0, c * nu, c, 0, 0, 0, c * (1.0 - nu) / 2.0};
    for (int i = 0; i < 9; ++i) D[i] = v[i];
    return;
  }
  const double lam = E * nu / ((1 + nu) * (1 - 2 * nu));
  const double mu = E / (2 * (1 + nu));
  for (int i = 0; i < 36; ++i) D[i] = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) D[i * 6 + j] = lam;
  for (int i = 0; i < 3; ++i) D[i * 6 + i] += 2 * mu;
  for (int i = 3; i < 6; ++i) D[i * 6 + i] = mu;
}

// Returns the (nd x nd) row-major matrix, nd = ndim * 2^ndim.
inline std::vector<double> element_stiffness(int ndim, const double* h, double E, double nu) {
  const int nn = 1 << ndim, nd = ndim * nn, ns = ndim == 2 ? 3 : 6;
  const double sgn[3][8] = {{-1, 1, 1, -1, -1, 1, 1, -1},
                            {-1, -1, 1, 1, -1, -1, 1, 1},
                            {-1, -1, -1, -1, 1, 1, 1, 1}};
  double D[36];
  constitutive_matrix(ndim, E, nu, D);
  double detJ = 1.0;
  for (int d = 0; d < ndim; ++d) detJ *= h[d] / 2.0;
  const double g = 1.0 / std::sqrt(3.0);
  std::vector<double> ke(nd * nd, 0.0), B(ns * nd), DB(ns * nd);
  const int npts = 1 << ndim;
  for (int q = 0; q < npts; ++q) {
    // point order: first axis slowest (matches the nested loops of mesh.py:239-250)
    double xi[3];
    for (int d = 0; d < ndim; ++d) xi[d] = ((q >> (ndim - 1 - d)) & 1) ? g : -g;
    double grad[3][8];
    for (int a = 0; a < nn; ++a) {
      for (int d = 0; d < ndim; ++d) {
        double v = sgn[d][a] * (ndim == 2 ? 0.25 : 0.125);
        for (int e = 0; e < ndim; ++e)
          if (e != d) v *= (1 + sgn[e][a] * xi[e]);
        grad[d][a] = v / (h[d] / 2.0);
      }
    }
    for (int i = 0; i < ns * nd; ++i) B[i] = 0.0;
    for (int a = 0; a < nn; ++a) {
      if (ndim == 2) {
        B[0 * nd + 2 * a] = grad[0][a];
        B[1 * nd + 2 * a + 1] = grad[1][a];
        B[2 * nd + 2 * a] = grad[1][a];
        B[2 * nd + 2 * a + 1] = grad[0][a];
      } else {
        B[0 * nd + 3 * a] = grad[0][a];
        B[1 * nd + 3 * a + 1] = grad[1][a];
        B[2 * nd + 3 * a + 2] = grad[2][a];
        B[3 * nd + 3 * a] = grad[1][a];
        B[3 * nd + 3 * a + 1] = grad[0][a];
        B[4 * nd + 3 * a + 1] = grad[2][a];
        B[4 * nd + 3 * a + 2] = grad[1][a];
        B[5 * nd + 3 * a] = grad[2][a];
        B[5 * nd + 3 * a + 2] = grad[0][a];
      }
    }
    for (int s = 0; s < ns; ++s)
      for (int j = 0; j < nd; ++j) {
        double acc = 0.0;
        for (int t = 0; t < ns; ++t) acc += D[s * ns + t] * B[t * nd + j];
        DB[s * nd + j] = acc;
      }
    for (int i = 0; i < nd; ++i)
      for (int j = 0; j < nd; ++j) {
        double acc = 0.0;
        for (int s = 0; s < ns; ++s) acc += B[s * nd + i] * DB[s * nd + j];
        ke[i * nd + j] += detJ * acc;
      }
  }
  std::vector<double> sym(nd * nd);
  for (int i = 0; i < nd; ++i)
    for (int j = 0; j < nd; ++j) sym[i * nd + j] = 0.5 * (ke[i * nd + j] + ke[j * nd + i]);
  return sym;
}

}  // namespace tmg
