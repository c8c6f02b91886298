// Hex8 matrix-free operator in the reflection-character (Hadamard) basis,
// element-centric, streamed along z.  The default 3D level-0 path
// (FineOp<3>::STREAM): every kernel that applies K(rho) on a 3D level 0
// (k_apply, k_residual, k_jacobi, k_cheb, k_cg_pq, k_apply_sym, k_bjacobi)
// calls fine3_rows(op, src, epi).
//
// Why: the node-gather form of K u (mesh.py:327, element matrix KE 24 x 24)
// costs 576 FMA per node, which makes the operator FP64-bound on B200 at ~4x
// its HBM time.  The unit-modulus KE of an axis-aligned box element is
// invariant under the three mirror reflections of the box (a reflection of axis
// a flips the sign of displacement component a).  In the basis of the 8
// characters of that reflection group -- per component the 2x2x2 Hadamard
// transform of the 8 corner values, u^[s] = sum_a (-1)^{popcount(s&a)} u[a] --
// KE becomes block diagonal with 45 nonzeros (ν > 0; 33 for ν = 0), the s = 0
// (mean) character decoupled entirely (rigid translations):
//     KE u = T^T (KE^ (T u)),   KE^ = T KE T^T / 64,   T^T T = 8 I.
// One element then costs a forward transform, 45 FMA and an inverse transform.
// The transforms factor per axis and are shared along z: the x-y transform of
// an element's top face is the next element's bottom face, and the two
// elements' contributions to a node plane are summed in x-y-character space
// before one inverse.  ~175 FP64 operations per element instead of 576.
//
// Mapping: a CTA is a TX x TY column of threads over an x-y node patch that
// overlaps its neighbours by one node; thread (tx,ty) owns the element column
// whose lowest corner is node (i0+tx, j0+ty) and walks a z chunk.  Per step
// (one element layer, ONE barrier) the source values and free-dof masks of the
// next node plane, (TX+1) x (TY+1), are staged in shared memory once (4-deep
// ring: the row's own value is read again two steps later); each element's
// corner contributions reach the neighbouring node columns through warp
// shuffles (x: a warp is one row of TX = 32 columns) and a double-buffered
// shared row (y).  Nodes with tx, ty >= 1 are complete and handed to the
// epilogue: epi(node, i, j, k, out, self), out = row of Z K Z + I_fixed
// applied to the source, self = the (unmasked) source value.
//
// Numerics: the same operator as the node gather up to fp64 rounding (the
// character-space coefficients are formed from the reference KE on the host and
// the entries outside the 45-term pattern are verified to vanish).
#pragma once

namespace tmg {
namespace f3h {
#ifndef TMG_F3H_TY
#define TMG_F3H_TY 8
#endif
constexpr int TX = 32, TY = TMG_F3H_TY, NT = TX * TY;
constexpr int SX = TX + 1, SY = TY + 1, NS = SX * SY;   // staged node columns of a plane
constexpr int NLD = (NS + NT - 1) / NT;                  // staged loads per thread
constexpr int NZ = 45;
// (row, col) of the nonzeros of KE^ in the (character s, component c) -> 3 s + c
// numbering; rows and columns of s = 0 vanish.  Character bits: x = 1, y = 2, z = 4.
#define TMG_F3H_NZ_R 3, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 11, 12, 12, 13, 13, 14, 14, \
                     14, 15, 15, 16, 16, 16, 17, 17, 18, 18, 18, 19, 19, 20, 20, 21, 22, 23
#define TMG_F3H_NZ_C 3, 7, 14, 4, 6, 5, 12, 4, 6, 3, 7, 14, 8, 13, 9, 20, 10, 17, 11, 16, 18, 5, 12, 8, 13, 3, 7, \
                     14, 15, 19, 11, 16, 18, 10, 17, 11, 16, 18, 15, 19, 9, 20, 21, 22, 23
__host__ __device__ constexpr int nz_row(int z) {
  constexpr unsigned char R[NZ] = {TMG_F3H_NZ_R};
  return R[z];
}
__host__ __device__ constexpr int nz_col(int z) {
  constexpr unsigned char C[NZ] = {TMG_F3H_NZ_C};
  return C[z];
}
// the 45 nonzeros grouped by character block chi (members (s, c) with
// s = chi ^ axis(c)): member rows 3 s + c, and per (row member, column member)
// the index into the 45 coefficients (-1: structural zero)
#define TMG_F3H_MEM 3, 7, 14, 0, 10, 17, 9, 1, 20, 6, 4, 23, 15, 19, 2, 12, 22, 5, 21, 13, 8, 18, 16, 11
#define TMG_F3H_KID                                                                                                \
  0, 1, 2, 9, 10, 11, 25, 26, 27, -1, -1, -1, -1, 16, 17, -1, 33, 34, 14, -1, 15, -1, -1, -1, 40, -1, 41, 8, 7, -1, \
      4, 3, -1, -1, -1, 44, 28, 29, -1, 38, 39, -1, -1, -1, -1, 22, -1, 21, -1, 43, -1, 6, -1, 5, 42, -1, -1, -1,   \
      24, 23, -1, 13, 12, 37, 36, 35, 32, 31, 30, 20, 19, 18
__host__ __device__ constexpr int blk_member(int chi, int i) {
  constexpr signed char Mm[24] = {TMG_F3H_MEM};
  return Mm[chi * 3 + i];
}
__host__ __device__ constexpr int blk_coef(int chi, int i, int j) {
  constexpr signed char K[72] = {TMG_F3H_KID};
  return K[(chi * 3 + i) * 3 + j];
}
constexpr int NB = 4;            // staged-plane buffers (the row's own value is read two steps on)
constexpr int U_PLANE = 3 * NS;  // doubles per staged plane (component-major)
constexpr int X_PLANE = 3 * NT;  // per thread: contributions to the node one row up
constexpr size_t SMEM_BYTES = sizeof(double) * (NB * U_PLANE + 2 * X_PLANE) + NB * NS;

// KE (reference corner numbering, mesh.py:73) -> the 45 character-space
// coefficients; returns the largest |entry| outside the pattern relative to the
// largest inside (the caller requires ~rounding).
inline double hat_coefficients(const double* ke, double* keh) {
  static const int m_of_a[8] = {0, 1, 3, 2, 4, 5, 7, 6};  // corner bits (x + 2y + 4z) -> local corner
  double T[24][24] = {};
  for (int s = 0; s < 8; ++s)
    for (int a = 0; a < 8; ++a) {
      const double sg = (__builtin_popcount(s & a) & 1) ? -1.0 : 1.0;
      for (int c = 0; c < 3; ++c) T[s * 3 + c][m_of_a[a] * 3 + c] = sg;
    }
  static double TK[24][24], H[24][24];
  for (int i = 0; i < 24; ++i)
    for (int j = 0; j < 24; ++j) {
      double v = 0.0;
      for (int q = 0; q < 24; ++q) v += T[i][q] * ke[q * 24 + j];
      TK[i][j] = v;
    }
  for (int i = 0; i < 24; ++i)
    for (int j = 0; j < 24; ++j) {
      double v = 0.0;
      for (int q = 0; q < 24; ++q) v += TK[i][q] * T[j][q];
      H[i][j] = v / 64.0;
    }
  bool in[24][24] = {};
  double mx = 0.0;
  for (int z = 0; z < NZ; ++z) {
    const int r = nz_row(z), c = nz_col(z);
    in[r][c] = true;
    keh[z] = 0.5 * (H[r][c] + H[c][r]);  // exactly symmetric
    mx = std::max(mx, std::fabs(keh[z]));
  }
  double off = 0.0;
  for (int i = 0; i < 24; ++i)
    for (int j = 0; j < 24; ++j)
      if (!in[i][j]) off = std::max(off, std::fabs(H[i][j]));
  return mx > 0.0 ? off / mx : 1.0;
}

#ifndef TMG_F3H_OCC
#define TMG_F3H_OCC 2  // CTAs per SM the z-chunking is sized for
#endif
// grid: x-y tiles of (TX-1) x (TY-1) output columns; z chunks chosen so the
// whole grid fills the SMs in as few, as full waves as possible (per-CTA cost ~
// chunk length + 2 warm-up layers)
inline dim3 grid(const Lat& L) {
  const int gx = (L.nn[0] + TX - 2) / (TX - 1), gy = (L.nn[1] + TY - 2) / (TY - 1);
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const long long slots = (long long)sms * TMG_F3H_OCC;
  const int nz = L.nn[2];
  int best = 1;
  double best_cost = 1e300;
  for (int nch = 1; nch <= nz; ++nch) {
    const int zc = (nz + nch - 1) / nch;
    const int used = (nz + zc - 1) / zc;  // chunks actually non-empty
    const long long ctas = (long long)gx * gy * used;
    const double waves = std::ceil((double)ctas / (double)slots);
    const double cost = waves * (zc + 2.5);
    if (cost < best_cost - 1e-9) { best_cost = cost; best = used; }
  }
  return dim3(gx, gy, best);
}
}  // namespace f3h

template <class Src, class Epi>
__device__ __forceinline__ void fine3h_rows(const FineOp<3>& op, const Src& src, Epi&& epi) {
  using namespace f3h;
  extern __shared__ __align__(16) double f3h_sm[];
  double* U = f3h_sm;                                                    // [NB][3][NS] source (unmasked)
  double* X = U + NB * U_PLANE;                                          // [2][3][NT] row-up contributions
  unsigned char* M = reinterpret_cast<unsigned char*>(X + 2 * X_PLANE);  // [NB][NS] free-dof masks
  const int t = threadIdx.x, tx = t % TX, ty = t / TX;
  const int nn0 = op.L.nn[0], nn1 = op.L.nn[1], nn2 = op.L.nn[2];
  const int ne0 = op.ne[0], ne1 = op.ne[1], ne2 = op.ne[2];
  const int i0 = (int)blockIdx.x * (TX - 1) - 1, j0 = (int)blockIdx.y * (TY - 1) - 1;
  const int zc = (nn2 + gridDim.z - 1) / gridDim.z;
  const int z0 = (int)blockIdx.z * zc, z1 = min(nn2, z0 + zc);
  if (z0 >= z1) return;  // (whole CTA)
  const long long plane = (long long)nn0 * nn1;
  // staged loads of this thread: plane-local node ids (or -1 outside the lattice)
  int ld_node[NLD];
#pragma unroll
  for (int u = 0; u < NLD; ++u) {
    const int st = t + u * NT;
    const int gi = i0 + st % SX, gj = j0 + st / SX;
    ld_node[u] = (st < NS && gi >= 0 && gi < nn0 && gj >= 0 && gj < nn1) ? gi + nn0 * gj : -1;
  }
  const int gi = i0 + tx, gj = j0 + ty;
  const bool el_ok = gi >= 0 && gi < ne0 && gj >= 0 && gj < ne1;
  const long long el2d = el_ok ? gi + (long long)ne0 * gj : 0;
  const bool out_ok = tx >= 1 && ty >= 1 && gi < nn0 && gj < nn1;
  const int own_st = tx + SX * ty;

  // carried between steps: the x-y character transform of the bottom face of
  // this element column (Fb), the top-corner contributions of the last element
  // layer to the current plane (Gp, character space), and the own node's
  // partial sum (own + left column) of the plane awaiting output (W0)
  double Fb[4][3], Gp[4][3], W0[3];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int c = 0; c < 3; ++c) Fb[q][c] = Gp[q][c] = 0.0;
#pragma unroll
  for (int c = 0; c < 3; ++c) W0[c] = 0.0;

  // step k: stage node plane k+1, output plane k-1, element layer k
  for (int k = z0 - 2; k <= z1; ++k) {
    const int pz = k + 1;  // plane staged this step
    double Ek = 0.0;
    if (k >= z0 - 1 && k < z1 && k >= 0 && k < ne2 && el_ok) Ek = __ldg(op.E + el2d + (long long)ne0 * ne1 * k);
    if (k < z1) {
      const bool pin = pz >= 0 && pz < nn2;
      double* Ub = U + (pz & (NB - 1)) * U_PLANE;
      unsigned char* Mb = M + (pz & (NB - 1)) * NS;
#pragma unroll
      for (int u = 0; u < NLD; ++u) {
        const int st = t + u * NT;
        if (st < NS) {
          double v[3] = {0.0, 0.0, 0.0};
          unsigned mk = 0u;
          if (pin && ld_node[u] >= 0) {
            const int node = (int)(ld_node[u] + plane * pz);
            src.load(node, 0, 0, 0, v);
            mk = __ldg(op.mask + node);
          }
#pragma unroll
          for (int c = 0; c < 3; ++c) Ub[c * NS + st] = v[c];
          Mb[st] = (unsigned char)mk;
        }
      }
    }
    __syncthreads();
    // plane k-1 complete: own + left column (W0) + the row below (X)
    if (k - 1 >= z0 && out_ok) {
      const int pk = k - 1;
      const double* Xb = X + (pk & 1) * X_PLANE;
      const double* Us = U + (pk & (NB - 1)) * U_PLANE;
      const unsigned mk = M[(pk & (NB - 1)) * NS + own_st];
      double out[3], self[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        self[c] = Us[c * NS + own_st];
        const double acc = W0[c] + Xb[c * NT + t - TX];
        out[c] = ((mk >> c) & 1u) ? acc : self[c];
      }
      epi((int)(gi + (long long)nn0 * gj + plane * pk), gi, gj, pk, out, self);
    }
    if (k >= z1) break;
    // top face (plane k+1) of the element column: masked corners, x-y transform
    double Ft[4][3];
    {
      const double* Ub = U + (pz & (NB - 1)) * U_PLANE;
      const unsigned char* Mb = M + (pz & (NB - 1)) * NS;
      const int sts[4] = {own_st, own_st + 1, own_st + SX, own_st + SX + 1};
      double v[4][3];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const unsigned mk = Mb[sts[a]];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double x = Ub[c * NS + sts[a]];
          v[a][c] = ((mk >> c) & 1u) ? x : 0.0;
        }
      }
      // F[qx + 2 qy] = sum over corners (x, y) of (-1)^(qx x + qy y) v[x + 2y]
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double a0 = v[0][c] + v[1][c], a1 = v[0][c] - v[1][c];
        const double a2 = v[2][c] + v[3][c], a3 = v[2][c] - v[3][c];
        Ft[0][c] = a0 + a2;
        Ft[1][c] = a1 + a3;
        Ft[2][c] = a0 - a2;
        Ft[3][c] = a1 - a3;
      }
    }
    if (k >= z0 - 1) {
      // element layer k (zero when outside the mesh: Ek = 0), one character
      // block at a time: member (s = q + 4 qz, c) has u^ = E (Fb[q] +- Ft[q]);
      // its output y^ goes to the bottom plane (+) and the top plane (+-)
      double T[4][3];
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int c = 0; c < 3; ++c) T[q][c] = 0.0;
#pragma unroll
      for (int chi = 0; chi < 8; ++chi) {
        double uh[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const int m = blk_member(chi, j), sj = m / 3, cj = m % 3, q = sj & 3;
          uh[j] = (sj & 4) ? Ek * (Fb[q][cj] - Ft[q][cj]) : Ek * (Fb[q][cj] + Ft[q][cj]);
        }
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const int m = blk_member(chi, i), si = m / 3, ci = m % 3, q = si & 3;
          if (si == 0) continue;  // the mean character: zero row
          double y = 0.0;
          bool any = false;
#pragma unroll
          for (int j = 0; j < 3; ++j)
            if (blk_coef(chi, i, j) >= 0) {
              y = any ? fma(op.keh[blk_coef(chi, i, j)], uh[j], y) : op.keh[blk_coef(chi, i, j)] * uh[j];
              any = true;
            }
          if (!any) continue;
          Gp[q][ci] += y;  // bottom corners (z = 0): plane k, joins the last layer's top part
          T[q][ci] = (si & 4) ? T[q][ci] - y : T[q][ci] + y;
        }
      }
      // x-y inverse of plane k's character sums -> corner (x, y) contributions
      double Wc[4][3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double b0 = Gp[0][c] + Gp[2][c], b2 = Gp[0][c] - Gp[2][c];
        const double b1 = Gp[1][c] + Gp[3][c], b3 = Gp[1][c] - Gp[3][c];
        Wc[0][c] = b0 + b1;  // corner (0,0): own node
        Wc[1][c] = b0 - b1;  // corner (1,0): node (i+1, j)
        Wc[2][c] = b2 + b3;  // corner (0,1): node (i, j+1)
        Wc[3][c] = b2 - b3;  // corner (1,1): node (i+1, j+1)
      }
      // x neighbours are lanes of the same warp (TX == 32): the left column's
      // (1,0) corner joins the own node, its (1,1) corner the node one row up,
      // which the row above reads through shared memory after the next barrier
      double* Xw = X + (k & 1) * X_PLANE;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        W0[c] = Wc[0][c] + __shfl_up_sync(0xffffffffu, Wc[1][c], 1);
        Xw[c * NT + t] = Wc[2][c] + __shfl_up_sync(0xffffffffu, Wc[3][c], 1);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int c = 0; c < 3; ++c) Gp[q][c] = T[q][c];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int c = 0; c < 3; ++c) Fb[q][c] = Ft[q][c];
  }
}

}  // namespace tmg
