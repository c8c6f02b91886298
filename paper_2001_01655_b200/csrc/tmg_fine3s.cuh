// Hex8 matrix-free operator, character basis (see tmg_fine3h.cuh for the
// algebra: KE = T^T KE^ T with the 45-term KE^), element columns streamed along
// z -- the register-prefetch variant: no producer warp, no raw rings.
//
// Mapping: a CTA is TY warps; warp ty is one row of 32 node columns, thread
// (tx, ty) owns node column (i0+tx, j0+ty) AND the element column whose lowest
// corner that node is.  Per plane every thread loads the source vectors of its
// own node straight from global memory (one step ahead, into registers),
// finishes them (src.finish: e.g. D^-1 r + beta p), and publishes the masked
// value in a double-buffered shared plane; the element's other three corners of
// the plane are its neighbours' values (shared memory, one CTA barrier per
// step).  Corner contributions return to the nodes through warp shuffles (x) and
// a double-buffered shared row (y).  With HALO the node row above the last warp
// row is loaded and finished by warp 0 in a second pass, so all TY warps own an
// element row: TY x 31 element columns complete 30 x (TY-1) node columns per
// plane.  Without HALO the last warp row only feeds nodes (30 x (TY-2) outputs).
//
// Shared memory is ~45 KB at TY = 8 (two or more CTAs per SM, independent
// barriers); occupancy is set by registers (TMG_F3S_MINB CTAs per SM).
#pragma once

namespace tmg {
namespace f3s {
#ifndef TMG_F3S_TY
#define TMG_F3S_TY 8
#endif
#ifndef TMG_F3S_HALO
#define TMG_F3S_HALO 1
#endif
#ifndef TMG_F3S_MINB
#define TMG_F3S_MINB 2
#endif
constexpr int TX = 32, TY = TMG_F3S_TY, NT = TX * TY;
constexpr bool HALO = TMG_F3S_HALO != 0;
constexpr int NR = TY + (HALO ? 1 : 0);   // node rows of a staged plane
constexpr int OX = TX - 2, OY = NR - 2;   // complete node columns per tile
constexpr int UROW = NR * TX + 8;         // doubles per component of a staged plane (+ pad: the x+1 read of the last node)
constexpr int NSELF = 3;                  // private ring of finished (unmasked) own values
// shared-memory layout (doubles, then bytes)
constexpr size_t OFF_U = 0;                                  // [2][3][UROW] masked source planes
constexpr size_t OFF_X = OFF_U + sizeof(double) * 2 * 3 * UROW;   // [2][3][NT] contributions to the node one row up
constexpr size_t OFF_S = OFF_X + sizeof(double) * 2 * 3 * NT;     // [NSELF][3][NT] own unmasked source
constexpr size_t OFF_M = OFF_S + sizeof(double) * NSELF * 3 * NT; // [NSELF][NT] own free-dof masks
constexpr size_t SMEM_BYTES = OFF_M + (size_t)NSELF * NT;

// grid: x-y tiles of OX x OY complete node columns; z chunks so that the grid
// fills the SMs (x MINB) in as few, as full waves as possible (per-CTA cost ~
// chunk length + 2 warm-up layers)
inline dim3 grid(const Lat& L) {
  const int gx = (L.nn[0] + OX - 1) / OX, gy = (L.nn[1] + OY - 1) / OY;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const long long slots = (long long)sms * TMG_F3S_MINB;
  const int nz = L.nn[2];
  int best = 1;
  double best_cost = 1e300;
  for (int nch = 1; nch <= nz; ++nch) {
    const int zc = (nz + nch - 1) / nch;
    const int used = (nz + zc - 1) / zc;
    const long long ctas = (long long)gx * gy * used;
    const double waves = std::ceil((double)ctas / (double)slots);
    const double cost = waves * (zc + 2.5);
    if (cost < best_cost - 1e-9) { best_cost = cost; best = used; }
  }
  return dim3(gx, gy, best);
}
}  // namespace f3s

template <class Src, class Epi>
__device__ __forceinline__ void fine3s_rows(const FineOp<3>& op, const Src& src, const f3h::EpiIn& ein, Epi&& epi) {
  using namespace f3s;
  using f3h::blk_coef;
  using f3h::blk_member;
  constexpr int NV = Src::NV;
  extern __shared__ __align__(16) unsigned char f3s_raw[];
  double* U = reinterpret_cast<double*>(f3s_raw + OFF_U);
  double* X = reinterpret_cast<double*>(f3s_raw + OFF_X);
  double* Sf = reinterpret_cast<double*>(f3s_raw + OFF_S);
  unsigned char* Mk = f3s_raw + OFF_M;
  const int t = threadIdx.x, tx = t % TX, ty = t / TX;
  const int nn0 = op.L.nn[0], nn1 = op.L.nn[1], nn2 = op.L.nn[2];
  const int ne0 = op.ne[0], ne1 = op.ne[1], ne2 = op.ne[2];
  const long long plane = (long long)nn0 * nn1, eplane = (long long)ne0 * ne1;
  const int i0 = (int)blockIdx.x * OX - 1, j0 = (int)blockIdx.y * OY - 1;
  const int zc = (nn2 + gridDim.z - 1) / gridDim.z;
  const int z0 = (int)blockIdx.z * zc, z1 = min(nn2, z0 + zc);
  if (z0 >= z1) return;  // (whole CTA)
  const int gi = i0 + tx, gj = j0 + ty;
  const bool node_ok = gi >= 0 && gi < nn0 && gj >= 0 && gj < nn1;
  const bool el_ok = tx < TX - 1 && ty < NR - 1 && gi >= 0 && gi < ne0 && gj >= 0 && gj < ne1;
  const bool out_ok = tx >= 1 && tx < TX - 1 && ty >= 1 && ty < NR - 1 && gi < nn0 && gj < nn1;
  const long long own2d = node_ok ? gi + (long long)nn0 * gj : 0;
  const long long own_el2d = el_ok ? gi + (long long)ne0 * gj : 0;
  // the halo node row (HALO): node (i0+tx, j0+NR-1), finished by warp 0
  const int gjh = j0 + NR - 1;
  const bool halo_ok = HALO && ty == 0 && gi >= 0 && gi < nn0 && gjh < nn1;
  const long long halo2d = halo_ok ? gi + (long long)nn0 * gjh : 0;
  if (t < 8) {  // the pad words are read (never used: their element has E = 0) -- keep them finite
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int c = 0; c < 3; ++c) U[(s * 3 + c) * UROW + NR * TX + t] = 0.0;
  }

  // raw source values of a node of plane p (zeros outside the lattice)
  auto load_raw = [&](int p, bool ok, long long n2d, double (*raw)[3], unsigned& mk) {
    const bool in = ok && p >= 0 && p < nn2;
    const long long node = n2d + plane * p;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const double* vp = src.vec(v);
#pragma unroll
      for (int c = 0; c < 3; ++c) raw[v][c] = (in && vp) ? __ldg(vp + 3 * node + c) : 0.0;
    }
    mk = in ? (unsigned)__ldg(op.mask + node) : 0u;
  };
  // finish a node of plane p into the staged plane (row r of the tile) and, for
  // the own node, the private self / mask ring slot ss
  auto finish = [&](int p, bool ok, const double (*raw)[3], unsigned mk, int r, int ss, bool own) {
    const bool in = ok && p >= 0 && p < nn2;
    double out[3] = {0.0, 0.0, 0.0};
    if (in) src.finish(raw, out);
    double* Ub = U + (p & 1) * 3 * UROW + r * TX + tx;
#pragma unroll
    for (int c = 0; c < 3; ++c) Ub[c * UROW] = ((mk >> c) & 1u) ? out[c] : 0.0;
    if (own) {
#pragma unroll
      for (int c = 0; c < 3; ++c) Sf[(ss * 3 + c) * NT + t] = out[c];
      Mk[ss * NT + t] = (unsigned char)mk;
    }
  };
  auto load_epi = [&](int pk, double (*e)[3]) {
    const bool ok = out_ok && pk >= z0 && pk < z1;
    const long long node = own2d + plane * pk;
#pragma unroll
    for (int v = 0; v < f3h::NVE; ++v)
#pragma unroll
      for (int c = 0; c < 3; ++c) e[v][c] = (ok && ein.v[v]) ? __ldg(ein.v[v] + 3 * node + c) : 0.0;
  };
  auto load_E = [&](int k) { return (el_ok && k >= 0 && k < ne2) ? __ldg(op.E + k * eplane + own_el2d) : 0.0; };
  // x-y transform of the element column's face in plane p
  auto face = [&](int p, double (*F)[3]) {
    const double* Ub = U + (p & 1) * 3 * UROW + ty * TX + tx;
    constexpr int off[4] = {0, 1, TX, TX + 1};
    double v[4][3];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) v[a][c] = Ub[c * UROW + off[a]];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double a0 = v[0][c] + v[1][c], a1 = v[0][c] - v[1][c];
      const double a2 = v[2][c] + v[3][c], a3 = v[2][c] - v[3][c];
      F[0][c] = a0 + a2;
      F[1][c] = a1 + a3;
      F[2][c] = a0 - a2;
      F[3][c] = a1 - a3;
    }
  };
  double epre[f3h::NVE][3], W0[3] = {0.0, 0.0, 0.0};
  // plane pk complete: own + left column (W0) + the row below (X); epilogue
  auto output = [&](int pk, int ss) {
    if (!(pk >= z0 && pk < z1 && out_ok)) return;
    const double* Xb = X + (pk & 1) * 3 * NT + t - TX;
    const unsigned mk = Mk[ss * NT + t];
    double out[3], self[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      self[c] = Sf[(ss * 3 + c) * NT + t];
      const double acc = W0[c] + Xb[c * NT];
      out[c] = ((mk >> c) & 1u) ? acc : self[c];
    }
    epi((int)(own2d + plane * pk), gi, gj, pk, out, self, epre);
  };
  // element layer k: bottom face Fb, top face Ft (computed here), the bottom
  // plane's character sums G (completed here), the next plane's T (produced here)
  auto layer = [&](int k, double Ek, const double (*Fb)[3], double (*Ft)[3], double (*G)[3], double (*T)[3]) {
    face(k + 1, Ft);
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
        G[q][ci] += y;
        T[q][ci] = (si & 4) ? T[q][ci] - y : T[q][ci] + y;
      }
    }
    double Wc[4][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double b0 = G[0][c] + G[2][c], b2 = G[0][c] - G[2][c];
      const double b1 = G[1][c] + G[3][c], b3 = G[1][c] - G[3][c];
      Wc[0][c] = b0 + b1;  // corner (0,0): own node
      Wc[1][c] = b0 - b1;  // corner (1,0): node (i+1, j)
      Wc[2][c] = b2 + b3;  // corner (0,1): node (i, j+1)
      Wc[3][c] = b2 - b3;  // corner (1,1): node (i+1, j+1)
    }
    double* Xw = X + (k & 1) * 3 * NT + t;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      W0[c] = Wc[0][c] + __shfl_up_sync(0xffffffffu, Wc[1][c], 1);
      Xw[c * NT] = Wc[2][c] + __shfl_up_sync(0xffffffffu, Wc[3][c], 1);
    }
  };

  // ---- prologue: planes z0-1 and z0 staged, plane z0+1 in flight ----
  double raw[NV][3], rawh[HALO ? NV : 1][3];
  unsigned mkr = 0u, mkh = 0u;
  int sp = 0;  // self-ring slot of the next plane to finish
  auto stage = [&](int p) {  // finish plane p from the registers, then load plane p + 1
    finish(p, node_ok, raw, mkr, ty, sp, true);
    load_raw(p + 1, node_ok && p + 1 <= z1, own2d, raw, mkr);
    if (HALO && ty == 0) {
      finish(p, halo_ok, rawh, mkh, NR - 1, 0, false);
      load_raw(p + 1, halo_ok && p + 1 <= z1, halo2d, rawh, mkh);
    }
    sp = sp + 1 == NSELF ? 0 : sp + 1;
  };
  load_raw(z0 - 1, node_ok, own2d, raw, mkr);
  if (HALO && ty == 0) load_raw(z0 - 1, halo_ok, halo2d, rawh, mkh);
  stage(z0 - 1);
  stage(z0);
  double Enext = load_E(z0 - 1);
  double F0[4][3], F1[4][3], G0[4][3], G1[4][3];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int c = 0; c < 3; ++c) G0[q][c] = 0.0;
  __syncthreads();
  face(z0 - 1, F0);
  // self-ring slot of the plane output next (plane z0 - 1 sits in slot 0, never output)
  int so = 0;
  int k = z0 - 1;
  // step k: [barrier] output plane k-1, prefetch, stage plane k+2, layer k
#define TMG_F3S_STEP(Fb, Ft, Ga, Gb)                                   \
  {                                                                     \
    __syncthreads();                                                    \
    output(k - 1, so);                                                  \
    so = (k - 1 >= z0 - 1) ? (so + 1 == NSELF ? 0 : so + 1) : so;       \
    const double Ek = Enext;                                            \
    Enext = load_E(k + 1);                                              \
    load_epi(k, epre);                                                  \
    if (k + 2 <= z1) stage(k + 2);                                      \
    layer(k, Ek, Fb, Ft, Ga, Gb);                                       \
    ++k;                                                                \
  }
  for (; k + 1 < z1;) {
    TMG_F3S_STEP(F0, F1, G0, G1)
    TMG_F3S_STEP(F1, F0, G1, G0)
  }
  if (k < z1) TMG_F3S_STEP(F0, F1, G0, G1)
#undef TMG_F3S_STEP
  __syncthreads();
  output(k - 1, so);  // plane z1-1
  __syncthreads();    // (the kernels' reductions follow with every thread)
}

}  // namespace tmg
