// Hex8 matrix-free operator, character basis, z-streamed (tmg_fine3h.cuh) with
// every row of 32 element columns served by a PAIR of consumer warps: the eight
// 3x3 character blocks of KE^ split into two halves that touch disjoint halves
// of the x-y character sums -- warp half h owns the pairs m = chi & 3 in
// {2h, 2h+1}, i.e. for component c the face characters q in
// {qb, qb+1}, qb = 2 (h ^ (c == 1)).  Each thread then carries 6 + 6 + 6 + 6
// doubles of face / accumulator state instead of 12 + 12 + 12 + 12, the kernel
// fits 16 consumer warps (+ the TMA producer warp) per SM at <= 120 registers,
// and the two halves of a step (FP64 blocks vs staging / epilogue traffic) overlap
// on the SM's schedulers.
//   A warps (h = 0): half the blocks, the own-row corners (0,0), (1,0) of the
//     inverse transform -> the node's own value W0, output + epilogue.
//   B warps (h = 1): the other half, the corners (0,1), (1,1) -> the row-up
//     contributions X, and the staging (`finish`) of the producer's raw planes.
// The halves meet once per step: each publishes the 6 partial sums
// (G_qb + G_qb+1, G_qb - G_qb+1 per component) in shared memory, one named
// barrier per warp pair, and completes its corners from both.
// Numerics: the same sums as tmg_fine3h.cuh, associated identically per corner.
#pragma once

namespace tmg {
namespace f3p {
using namespace f3h;
constexpr int NCP = 2 * NT;          // consumer threads (16 warps)
constexpr int NTHP = NCP + 32 * NPROD;  // + the producer warps
constexpr size_t OFF_Z = al128(f3h::SMEM_BYTES);                 // [2 (half)][6][NT] partial sums
constexpr size_t SMEM_BYTES_P = OFF_Z + sizeof(double) * 2 * 6 * NT;
static_assert(SMEM_BYTES_P <= 227 * 1024 - 2048, "f3p shared memory");
__host__ __device__ constexpr int qbase(int h, int c) { return 2 * (h ^ (c == 1 ? 1 : 0)); }
}  // namespace f3p

template <int H, class Src, class Epi>
__device__ __forceinline__ void fine3p_consumer(const FineOp<3>& op, const Src& src, const f3h::EpiIn& ein, Epi&& epi,
                                                unsigned char* smem, int tb, int i0, int j0, int z0, int z1, int R) {
  using namespace f3p;
  unsigned long long* raw_full = reinterpret_cast<unsigned long long*>(smem + OFF_BAR);
  unsigned long long* raw_free = raw_full + NSR;
  double* SR = reinterpret_cast<double*>(smem + OFF_SRAW);
  unsigned char* MR = smem + OFF_MRAW;
  double* U = reinterpret_cast<double*>(smem + OFF_U);
  double* S = reinterpret_cast<double*>(smem + OFF_S);
  unsigned char* M = smem + OFF_M;
  double* X = reinterpret_cast<double*>(smem + OFF_X);
  double* Z = reinterpret_cast<double*>(smem + OFF_Z);
  const int nn0 = op.L.nn[0], nn1 = op.L.nn[1], nn2 = op.L.nn[2];
  const int ne0 = op.ne[0], ne1 = op.ne[1], ne2 = op.ne[2];
  const long long plane = (long long)nn0 * nn1, eplane = (long long)ne0 * ne1;
  const int t = tb;  // index of the thread among its half's 256 (tx + 32 ty)
  const int tx = t % TX, ty = t / TX;
  const int gi = i0 + tx, gj = j0 + ty;
  const bool el_ok = gi >= 0 && gi < ne0 && gj >= 0 && gj < ne1;
  const bool out_ok = tx >= 1 && ty >= 1 && gi < nn0 && gj < nn1;
  const int own_st = tx + SX * ty;
  const long long own_node2d = gi + (long long)nn0 * gj;
  const long long own_el2d = el_ok ? gi + (long long)ne0 * gj : 0;
  const int nlo = max(i0, 0);

  // ---- B warps: staging of the raw planes (identical to tmg_fine3h.cuh) ----
  const int pl_par = (int)(plane & 1), pl_m16 = (int)(plane & 15);
  int fin_st[NFIN], fin_off[NFIN], fin_mrow[NFIN], fin_par[NFIN][NVS], fin_m16[NFIN];
  bool fin_in[NFIN];
  if (H == 1) {
#pragma unroll
    for (int u = 0; u < NFIN; ++u) {
      const int st = t + u * NT;
      const int sx = st % SX, sy = st / SX;
      const int gx = i0 + sx, gy = j0 + sy;
      fin_st[u] = st;
      fin_in[u] = st < NS && gx >= 0 && gx < nn0 && gy >= 0 && gy < nn1;
      const long long rowoff = (long long)gy * nn0 + nlo;
      fin_off[u] = sy * ROWD + 3 * (gx - nlo);
      fin_mrow[u] = sy * MROW + (gx - nlo);
#pragma unroll
      for (int v = 0; v < NVS; ++v) {
        const double* vp = v < Src::NV ? src.vec(v) : nullptr;
        fin_par[u][v] = vp ? (int)((((unsigned long long)vp >> 3) + (unsigned long long)(3 * rowoff)) & 1ull) : 0;
      }
      fin_m16[u] = (int)(((unsigned long long)op.mask + (unsigned long long)rowoff) & 15ull);
    }
  }
  // (the ring positions of the next plane to stage are carried from plane to plane:
  // no division by the ring depths or multiplication by the plane size per step)
  static_assert((NU & (NU - 1)) == 0, "finished-plane ring depth: a power of two");
  int f_s3 = 0, f_su = 0, f_p = z0 - 1;
  unsigned f_ph = 0u;
  int f_pm16 = ((z0 - 1) * pl_m16) & 15;
  auto finish = [&](int) {
    const int p = f_p, s3 = f_s3, su = f_su;
    mbar_wait(raw_full + s3, f_ph);
    const bool pin = p >= 0 && p < nn2;
    const int ppar = p & pl_par, pm16 = f_pm16;
    ++f_p;
    f_pm16 = (f_pm16 + pl_m16) & 15;
    f_su = (f_su + 1) & (NU - 1);
    if (++f_s3 == NSR) {
      f_s3 = 0;
      f_ph ^= 1u;
    }
#pragma unroll
    for (int u = 0; u < NFIN; ++u) {
      if (u > 0 && fin_st[u] >= NS) break;
      double out[3] = {0.0, 0.0, 0.0};
      unsigned mk = 0u;
      if (pin && fin_in[u]) {
        double raw[NVS][3];
#pragma unroll
        for (int v = 0; v < NVS; ++v) {
          const double* rb = SR + (s3 * NVS + v) * SY * ROWD + fin_off[u] + (fin_par[u][v] ^ ppar);
#pragma unroll
          for (int c = 0; c < 3; ++c) raw[v][c] = (v < Src::NV && src.vec(v)) ? rb[c] : 0.0;
        }
        src.finish(raw, out);
        mk = MR[s3 * SY * MROW + fin_mrow[u] + ((fin_m16[u] + pm16) & 15)];
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        U[su * U_PLANE + c * NS + fin_st[u]] = ((mk >> c) & 1u) ? out[c] : 0.0;
        S[su * U_PLANE + c * NS + fin_st[u]] = out[c];
      }
      M[su * NS + fin_st[u]] = (unsigned char)mk;
    }
    __syncwarp();
    if ((t & 31) == 0) mbar_arrive(raw_free + s3);
  };

  // ---- A warps: epilogue inputs, output ----
  long long node_k = own_node2d + plane * (z0 - 1);  // the own node in plane k (advanced with k)
  const double* Ep = op.E + own_el2d + eplane * (z0 + 1);  // the own element in layer k + 2
  auto load_epi = [&](int pk, double (*e)[3]) {
    const bool ok = out_ok && pk >= z0 && pk < z1;
    const int node = (int)node_k;  // (pk == k; node ids fit an int, as in the epilogues)
#pragma unroll
    for (int v = 0; v < NVE; ++v) {
      const double* ev = ein.v[v] + 3ll * node;  // (32 x 32 -> 64-bit multiply-add: one instruction)
#pragma unroll
      for (int c = 0; c < 3; ++c) e[v][c] = (ok && ein.v[v]) ? __ldg(ev + c) : 0.0;
    }
  };
  auto load_E = [&](int k) {
    return (el_ok && k >= 0 && k < ne2 && k < z1) ? __ldg(op.E + k * eplane + own_el2d) : 0.0;
  };
  auto load_E2 = [&](int k2) {  // layer k2 = k + 2 through the running pointer
    return (el_ok && k2 >= 0 && k2 < ne2 && k2 < z1) ? __ldg(Ep) : 0.0;
  };
  double epre[NVE][3], W0[3] = {0.0, 0.0, 0.0};
  auto output = [&](int k) {
    const int pk = k - 1;
    if (!(pk >= z0 && pk < z1 && out_ok)) return;
    const int su = (int)((unsigned)(pk - z0 + 1) & (unsigned)(NU - 1));
    const double* Xb = X + (pk & 1) * X_PLANE + t - TX;
    const double* Us = S + su * U_PLANE + own_st;
    const unsigned mk = M[su * NS + own_st];
    double out[3], self[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      self[c] = Us[c * NS];
      const double acc = W0[c] + Xb[c * NC];
      out[c] = ((mk >> c) & 1u) ? acc : self[c];
    }
    epi((int)(node_k - plane), gi, gj, pk, out, self, epre);  // (pk == k - 1)
  };

  // ---- both halves: the owned characters of a face, a layer ----
  // F[c][e]: character q = qbase(H, c) + e of component c
  auto face = [&](int su, double (*F)[2]) {
    const double* Ub = U + su * U_PLANE + own_st;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double v0 = Ub[c * NS], v1 = Ub[c * NS + 1], v2 = Ub[c * NS + SX], v3 = Ub[c * NS + SX + 1];
      const double a0 = v0 + v1, a1 = v0 - v1, a2 = v2 + v3, a3 = v2 - v3;
      if (qbase(H, c) == 0) {
        F[c][0] = a0 + a2;
        F[c][1] = a1 + a3;
      } else {
        F[c][0] = a0 - a2;
        F[c][1] = a1 - a3;
      }
    }
  };
  // layer k: bottom characters Fb, top Ft (computed here); G: the bottom plane's
  // sums (completed here), T: the next plane's (produced here)
  auto layer = [&](int k, double Ek, const double (*Fb)[2], double (*Ft)[2], double (*G)[2], double (*T)[2]) {
    face((int)((unsigned)(k + 2 - z0) & (unsigned)(NU - 1)), Ft);
    bool tset[3][2] = {};
#pragma unroll
    for (int chi = 0; chi < 8; ++chi) {
      if (((chi >> 1) & 1) != H) continue;  // the other half's block
      double uh[3];
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int m = blk_member(chi, j), sj = m / 3, cj = m % 3, e = (sj & 3) - qbase(H, cj);
        uh[j] = (sj & 4) ? Fb[cj][e] - Ft[cj][e] : Fb[cj][e] + Ft[cj][e];
      }
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int m = blk_member(chi, i), si = m / 3, ci = m % 3, e = (si & 3) - qbase(H, ci);
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
        G[ci][e] = fma(Ek, y, G[ci][e]);
        if (tset[ci][e]) T[ci][e] = fma((si & 4) ? -Ek : Ek, y, T[ci][e]);
        else T[ci][e] = ((si & 4) ? -Ek : Ek) * y;
        tset[ci][e] = true;
      }
    }
    // partial inverse: per component the sum and difference of the two owned
    // characters; the partner warp holds the other two
    double* Zw = Z + (H * 6) * NT + t;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      Zw[(2 * c) * NT] = G[c][0] + G[c][1];
      Zw[(2 * c + 1) * NT] = G[c][0] - G[c][1];
    }
    asm volatile("bar.sync %0, 64;" ::"r"(2 + ty) : "memory");  // the two warps of this row
    const double* Zo = Z + ((1 - H) * 6) * NT + t;
    // s01 / d01: sum / difference of characters 0, 1; s23 / d23: of 2, 3
    double keep[3], pass[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double own_s = G[c][0] + G[c][1], own_d = G[c][0] - G[c][1];
      const double oth_s = Zo[(2 * c) * NT], oth_d = Zo[(2 * c + 1) * NT];
      const bool own01 = qbase(H, c) == 0;
      const double s01 = own01 ? own_s : oth_s, s23 = own01 ? oth_s : own_s;
      const double d01 = own01 ? own_d : oth_d, d23 = own01 ? oth_d : own_d;
      // (with b0 = G0 + G2, b1 = G1 + G3, b2 = G0 - G2, b3 = G1 - G3 of tmg_fine3h.cuh:
      //  corner (0,0) = b0 + b1, (1,0) = b0 - b1, (0,1) = b2 + b3, (1,1) = b2 - b3)
      if (H == 0) {
        keep[c] = s01 + s23;  // corner (0,0): own node
        pass[c] = d01 + d23;  // corner (1,0): node (i+1, j)
      } else {
        keep[c] = s01 - s23;  // corner (0,1): node (i, j+1)
        pass[c] = d01 - d23;  // corner (1,1): node (i+1, j+1)
      }
    }
    if (H == 0) {
#pragma unroll
      for (int c = 0; c < 3; ++c) W0[c] = keep[c] + __shfl_up_sync(0xffffffffu, pass[c], 1);
    } else {
      double* Xw = X + (k & 1) * X_PLANE + t;
#pragma unroll
      for (int c = 0; c < 3; ++c) Xw[c * NC] = keep[c] + __shfl_up_sync(0xffffffffu, pass[c], 1);
    }
  };

  double F0[3][2], F1[3][2], G0[3][2], G1[3][2];
#pragma unroll
  for (int c = 0; c < 3; ++c) G0[c][0] = G0[c][1] = 0.0;
  if (H == 1) finish(0);  // plane z0-1
  double Enext = load_E(z0 - 1), Enext2 = load_E(z0);
  asm volatile("bar.sync 1, %0;" ::"n"(NCP) : "memory");
  if (H == 1) finish(1);
  face(0, F0);
  int k = z0 - 1;
  // step k: [barrier] A: output plane k-1, prefetch; B: stage plane k+2; both: layer k
#define TMG_F3P_STEP(Fb, Ft, Ga, Gb)                                          \
  {                                                                            \
    asm volatile("bar.sync 1, %0;" ::"n"(NCP) : "memory");                     \
    if (H == 0) output(k);                                                     \
    const double Ek = Enext;                                                   \
    Enext = Enext2;                                                            \
    Enext2 = load_E2(k + 2);                                                   \
    if (H == 0) load_epi(k, epre);                                             \
    if (H == 1 && k + 3 - z0 <= R) finish(k + 3 - z0);                         \
    layer(k, Ek, Fb, Ft, Ga, Gb);                                              \
    ++k;                                                                       \
    node_k += plane;                                                           \
    Ep += eplane;                                                              \
  }
  for (; k + 1 < z1;) {
    TMG_F3P_STEP(F0, F1, G0, G1)
    TMG_F3P_STEP(F1, F0, G1, G0)
  }
  if (k < z1) TMG_F3P_STEP(F0, F1, G0, G1)
#undef TMG_F3P_STEP
  asm volatile("bar.sync 1, %0;" ::"n"(NCP) : "memory");
  if (H == 0) output(k);  // plane z1-1
}

template <class Src, class Epi>
__device__ __forceinline__ void fine3p_rows(const FineOp<3>& op, const Src& src, const f3h::EpiIn& ein, Epi&& epi) {
  using namespace f3p;
  static_assert(Src::NV <= NVS, "source vectors");
  extern __shared__ __align__(128) unsigned char f3p_raw[];
  unsigned long long* raw_full = reinterpret_cast<unsigned long long*>(f3p_raw + OFF_BAR);
  unsigned long long* raw_free = raw_full + NSR;
  const int t = threadIdx.x;
  const int nn0 = op.L.nn[0], nn2 = op.L.nn[2];
  const int i0 = (int)blockIdx.x * (TX - 1) - 1, j0 = (int)blockIdx.y * (TY - 1) - 1;
  const int zc = (nn2 + gridDim.z - 1) / gridDim.z;
  const int z0 = (int)blockIdx.z * zc, z1 = min(nn2, z0 + zc);
  if (z0 >= z1) return;  // (whole CTA)
  const int R = z1 - z0 + 1;
  const int nlo = max(i0, 0), ncnt = min(i0 + SX, nn0) - nlo;
  if (t == 0) {
    for (int b = 0; b < NSR; ++b) {
      mbar_init(raw_full + b, 1);
      mbar_init(raw_free + b, NT / 32);  // one arrival per staging (B) warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (t >= NCP) {
    produce<Src>(op, src, reinterpret_cast<double*>(f3p_raw + OFF_SRAW), f3p_raw + OFF_MRAW, raw_full, raw_free,
                 (t - NCP) & 31, z0, R, j0, nlo, ncnt, (t - NCP) >> 5, NPROD);
  } else {
    const int w = t >> 5, h = w & 1;                 // warp pair (row) w / 2, half h
    const int tb = (t & 31) + 32 * (w >> 1);         // tx + 32 ty
    if (h == 0) fine3p_consumer<0>(op, src, ein, static_cast<Epi&&>(epi), f3p_raw, tb, i0, j0, z0, z1, R);
    else fine3p_consumer<1>(op, src, ein, static_cast<Epi&&>(epi), f3p_raw, tb, i0, j0, z0, z1, R);
  }
  __syncthreads();  // (the kernels' reductions follow with every thread)
}

}  // namespace tmg
