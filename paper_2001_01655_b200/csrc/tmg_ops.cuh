// Level operators of the geometric hierarchy and the node-parallel kernels that
// apply them.  Two operator kinds share one interface:
//
//  * FineOp<DIM>:   the level-0 stiffness K(rho) kept matrix-free -- element moduli
//    (8 B/element) and the unit-modulus element matrix KE.  KE travels BY VALUE in
//    the kernel parameters, so every KE coefficient is a constant-bank operand of
//    the DFMA (no shared-memory or L1 traffic for it).  A row of K is gathered
//    node-centrically from the 2^DIM elements around the node, so the product is
//    assembled atomic-free with no colouring pass.  The symmetric Dirichlet
//    elimination of mesh.py:313 (Z K Z + I_fixed) is applied on the fly from a
//    per-node free-dof bitmask.
//  * StencilOp<DIM>: a Galerkin coarse operator P^T A P of a geometric level.  On a
//    structured grid with bilinear/trilinear P it is exactly a 3^DIM-point nodal
//    stencil of DIM x DIM blocks, stored structure-of-arrays
//    A[(slot*DIM*DIM + a*DIM + b) * n_nodes + node] so that a warp reads 32
//    consecutive doubles per (slot, a, b).  Out-of-domain slots hold zeros, so all
//    coefficient loads are unconditional (full memory-level parallelism).  No index
//    arrays are stored.
//
// Node kernels use a 2D/3D launch (32x8 / 32x4x2 threads): one thread per node,
// x fastest, coordinates straight from blockIdx/threadIdx (no index division).
#pragma once
#include "tmg_common.cuh"

namespace tmg {

// local corner numbering of mesh.py:73-102
__host__ __device__ constexpr int corner_of(int dx, int dy, int dz) { return (dy ? 3 - dx : dx) + 4 * dz; }
__host__ __device__ constexpr int corner_x(int m) { return ((m & 3) == 1 || (m & 3) == 2) ? 1 : 0; }
__host__ __device__ constexpr int corner_y(int m) { return (m & 3) >= 2 ? 1 : 0; }
__host__ __device__ constexpr int corner_z(int m) { return m >> 2; }

template <int DIM>
struct Slots {  // 3^DIM stencil neighbourhood, slot = (dx+1) + 3(dy+1) + 9(dz+1)
  static constexpr int NS = DIM == 2 ? 9 : 27;
  __host__ __device__ static constexpr int dx(int s) { return s % 3 - 1; }
  __host__ __device__ static constexpr int dy(int s) { return (s / 3) % 3 - 1; }
  __host__ __device__ static constexpr int dz(int s) { return DIM == 3 ? s / 9 - 1 : 0; }
  __host__ __device__ static constexpr int of(int x, int y, int z) {
    return (x + 1) + 3 * (y + 1) + (DIM == 3 ? 9 * (z + 1) : 0);
  }
};

// Register fence: the values must be materialised here.  Placed after a batch of
// loads it stops the scheduler from sinking each load next to its first use
// (which serialises L2 round trips on the thread-starved coarse levels).
// (multi-operand asm statements: one operand per statement does not hold the
// batch together, eight do -- verified on the SASS with cuobjdump.)
template <int N>
__device__ __forceinline__ void reg_fence(double* v) {
#pragma unroll
  for (int t = 0; t + 8 <= N; t += 8)
    asm volatile("" : "+d"(v[t]), "+d"(v[t + 1]), "+d"(v[t + 2]), "+d"(v[t + 3]), "+d"(v[t + 4]), "+d"(v[t + 5]),
                 "+d"(v[t + 6]), "+d"(v[t + 7]));
#pragma unroll
  for (int t = N - N % 8; t < N; ++t) asm volatile("" : "+d"(v[t]));
}
__device__ __forceinline__ double ldv(const double* p) { return __ldg(p); }
__device__ __forceinline__ double2 ldv2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }

template <int DIM>
__device__ __forceinline__ void load_node(const double* __restrict__ v, int node, double out[DIM]) {
  if (DIM == 2) {
    const double2 t = ldv2(v + 2 * node);
    out[0] = t.x;
    out[1] = t.y;
  } else {
#pragma unroll
    for (int c = 0; c < DIM; ++c) out[c] = ldv(v + node * DIM + c);
  }
}
template <int DIM>
__device__ __forceinline__ void store_node(double* __restrict__ v, int node, const double in[DIM]) {
  if (DIM == 2) {
    reinterpret_cast<double2*>(v)[node] = make_double2(in[0], in[1]);
  } else {
#pragma unroll
    for (int c = 0; c < DIM; ++c) v[node * DIM + c] = in[c];
  }
}

// ----------------------------------------------------------------------------
// geometric transfers (multigrid.py:288-315): 1D hat interpolation per axis,
// Kronecker product with x fastest, identity on axes with one element.
// ----------------------------------------------------------------------------
struct Coarsening {
  Lat F, C;  // fine / coarse node lattices
  int co[3]; // 1 if the axis is coarsened (fine element count > 1)
};

// fine candidates of coarse index I on one axis: up to 3 (index, weight)
__device__ __forceinline__ int fine_of_coarse(int I, int co, int nf, int idx[3], double w[3]) {
  if (!co) { idx[0] = I; w[0] = 1.0; return 1; }
  int c = 0;
  const int base = 2 * I;
  if (base - 1 >= 0 && base - 1 < nf) { idx[c] = base - 1; w[c] = 0.5; ++c; }
  if (base < nf) { idx[c] = base; w[c] = 1.0; ++c; }
  if (base + 1 < nf) { idx[c] = base + 1; w[c] = 0.5; ++c; }
  return c;
}
// the same as three fixed slots: valid candidates first, in order, then
// (clamped index, weight 0) fillers
__device__ __forceinline__ void fine_of_coarse3(int I, int co, int nf, int idx[3], double w[3]) {
  const int c = fine_of_coarse(I, co, nf, idx, w);
#pragma unroll
  for (int q = 0; q < 3; ++q)
    if (q >= c) { idx[q] = idx[0]; w[q] = 0.0; }
}
// coarse parents of fine index i on one axis: up to 2 (index, weight)
__device__ __forceinline__ int coarse_of_fine(int i, int co, int idx[2], double w[2]) {
  if (!co) { idx[0] = i; w[0] = 1.0; return 1; }
  if ((i & 1) == 0) { idx[0] = i >> 1; w[0] = 1.0; return 1; }
  idx[0] = (i - 1) >> 1; idx[1] = (i + 1) >> 1; w[0] = w[1] = 0.5;
  return 2;
}
// (P e)(fine node i,j,k), branch-light: parents clamp to the same node with weight 0.
template <int DIM>
__device__ __forceinline__ void prolong_at(const Coarsening& T, const double* __restrict__ e, int i, int j, int k,
                                           double out[DIM]) {
  int ix[2], iy[2], iz[2];
  double wx[2], wy[2], wz[2];
  const int nx = coarse_of_fine(i, T.co[0], ix, wx);
  const int ny = coarse_of_fine(j, T.co[1], iy, wy);
  int nz = 1;
  if (DIM == 3) nz = coarse_of_fine(k, T.co[2], iz, wz);
  else { iz[0] = 0; wz[0] = 1.0; }
#pragma unroll
  for (int c = 0; c < DIM; ++c) out[c] = 0.0;
  for (int c2 = 0; c2 < nz; ++c2)
    for (int b = 0; b < ny; ++b)
      for (int a = 0; a < nx; ++a) {
        const double ww = wx[a] * wy[b] * wz[c2];
        double v[DIM];
        load_node<DIM>(e, T.C.id(ix[a], iy[b], iz[c2]), v);
#pragma unroll
        for (int c = 0; c < DIM; ++c) out[c] += ww * v[c];
      }
}

// ----------------------------------------------------------------------------
// vector sources: value of the vector being multiplied at (node, i, j, k)
// ----------------------------------------------------------------------------
// DIRECT: the source is a pointwise combination of vectors, cheap enough to be
// evaluated per neighbour (2D FineOp direct path); ProlongSrc is not.
// The DIRECT sources also expose the vectors they read (NV, vec(v); nullptr =
// not read) and finish(raw, out) on staged copies raw[v][c] -- the streamed 3D
// operator (tmg_fine3h.cuh) moves the vectors with TMA and finishes them in
// shared memory.  finish() performs load()'s arithmetic in load()'s order.
template <int DIM>
struct VecSrc {
  static constexpr bool DIRECT = true;
  static constexpr int NV = 1;
  const double* __restrict__ v;
  __device__ void load(int node, int, int, int, double out[DIM]) const { load_node<DIM>(v, node, out); }
  __device__ const double* vec(int) const { return v; }
  __device__ void finish(const double (*raw)[DIM], double out[DIM]) const {
#pragma unroll
    for (int c = 0; c < DIM; ++c) out[c] = raw[0][c];
  }
};
template <int DIM>
struct ScaledSrc {  // s .* v
  static constexpr bool DIRECT = true;
  const double* __restrict__ v;
  const double* __restrict__ s;
  static constexpr int NV = 2;
  __device__ void load(int node, int, int, int, double out[DIM]) const {
    double a[DIM], b[DIM];
    load_node<DIM>(v, node, a);
    load_node<DIM>(s, node, b);
#pragma unroll
    for (int c = 0; c < DIM; ++c) out[c] = a[c] * b[c];
  }
  __device__ const double* vec(int i) const { return i == 0 ? v : s; }
  __device__ void finish(const double (*raw)[DIM], double out[DIM]) const {
#pragma unroll
    for (int c = 0; c < DIM; ++c) out[c] = raw[0][c] * raw[1][c];
  }
};
template <int DIM>
struct AxpySrc {  // z + beta * p  (beta == 0 -> z; never touches p then)
  static constexpr bool DIRECT = true;
  const double* __restrict__ z;
  const double* __restrict__ p;
  double beta;
  static constexpr int NV = 2;
  __device__ void load(int node, int, int, int, double out[DIM]) const {
    load_node<DIM>(z, node, out);
    if (beta != 0.0) {
      double q[DIM];
      load_node<DIM>(p, node, q);
#pragma unroll
      for (int c = 0; c < DIM; ++c) out[c] += beta * q[c];
    }
  }
  __device__ const double* vec(int i) const { return i == 0 ? z : (beta != 0.0 ? p : nullptr); }
  __device__ void finish(const double (*raw)[DIM], double out[DIM]) const {
#pragma unroll
    for (int c = 0; c < DIM; ++c) out[c] = raw[0][c];
    if (beta != 0.0) {
#pragma unroll
      for (int c = 0; c < DIM; ++c) out[c] += beta * raw[1][c];
    }
  }
};
template <int DIM>
struct ChebSrc {  // dinv .* r + beta * p  (dinv == nullptr: r + beta * p)
  static constexpr bool DIRECT = true;
  const double* __restrict__ r;
  const double* __restrict__ p;
  const double* __restrict__ dinv;
  double beta;
  static constexpr int NV = 3;
  __device__ const double* vec(int i) const { return i == 0 ? r : (i == 1 ? dinv : (beta != 0.0 ? p : nullptr)); }
  __device__ void finish(const double (*raw)[DIM], double out[DIM]) const {
    if (dinv) {
#pragma unroll
      for (int c = 0; c < DIM; ++c) out[c] = raw[1][c] * raw[0][c];
    } else {
#pragma unroll
      for (int c = 0; c < DIM; ++c) out[c] = raw[0][c];
    }
    if (beta != 0.0) {
#pragma unroll
      for (int c = 0; c < DIM; ++c) out[c] += beta * raw[2][c];
    }
  }
  __device__ void load(int node, int, int, int, double out[DIM]) const {
    double a[DIM], d[DIM];
    load_node<DIM>(r, node, a);
    if (dinv) {
      load_node<DIM>(dinv, node, d);
#pragma unroll
      for (int c = 0; c < DIM; ++c) out[c] = d[c] * a[c];
    } else {
#pragma unroll
      for (int c = 0; c < DIM; ++c) out[c] = a[c];
    }
    if (beta != 0.0) {
      double q[DIM];
      load_node<DIM>(p, node, q);
#pragma unroll
      for (int c = 0; c < DIM; ++c) out[c] += beta * q[c];
    }
  }
};
template <int DIM>
struct ProlongSrc {  // x + P e (coarse-grid correction evaluated on the fly)
  static constexpr bool DIRECT = false;
  const double* __restrict__ x;
  const double* __restrict__ e;
  Coarsening T;
  __device__ void load(int node, int i, int j, int k, double out[DIM]) const {
    double pe[DIM];
    load_node<DIM>(x, node, out);
    prolong_at<DIM>(T, e, i, j, k, pe);
#pragma unroll
    for (int c = 0; c < DIM; ++c) out[c] += pe[c];
  }
};

// ----------------------------------------------------------------------------
// FineOp
// ----------------------------------------------------------------------------
template <int DIM>
struct FineOp {
  static constexpr int NN = 1 << DIM, NE = DIM * NN, DD = DIM * DIM;
  Lat L;
  int ne[3];
  const double* __restrict__ E;
  const uint8_t* __restrict__ mask;  // bit c set -> dof c of the node is free
  double ke[NE * NE];                // kernel-parameter constant bank
  double keh[DIM == 3 ? 45 : 1];     // 3D: KE in the reflection-character basis (tmg_fine3h.cuh)

  __device__ int elem_id(int ex, int ey, int ez) const { return ex + ne[0] * (ey + ne[1] * ez); }

  // Shared-memory tile of one node block (node_block<DIM>: BX x BY x BZ) plus a
  // one-node halo: the source vector (unmasked), the free-dof masks and the
  // moduli of the (BX+1)(BY+1)(BZ+1) elements touching the tile.  Every value is
  // read from L2/HBM once per block instead of once per neighbouring thread.
// 3D level-0 variant: the paired-warp stream (tmg_fine3p.cuh) unless another is asked for
#if !defined(TMG_F3P) && !defined(TMG_F3H) && !defined(TMG_F3S) && !defined(TMG_FINE3_TILE)
#define TMG_F3P 1
#endif
#ifndef TMG_F3_BX
#define TMG_F3_BX 16
#define TMG_F3_BY 4
#define TMG_F3_BZ 4
#endif
  // 3D tile 16x4x4 (648 staged nodes / 425 elements per 256 rows; 32x4x2: 816 /
  // 495).  Measured config-4 sweep / residual: 16x4x4 145 / 103 us, 16x8x2 151 /
  // 106, 32x2x4 157 / 110, 32x4x2 157 / 111, 8x8x4 173 / 125.
#ifndef TMG_F2_BX
#define TMG_F2_BX 32
#define TMG_F2_BY 8
#endif
  static constexpr int BX = DIM == 2 ? TMG_F2_BX : TMG_F3_BX, BY = DIM == 2 ? TMG_F2_BY : TMG_F3_BY,
                       BZ = DIM == 2 ? 1 : TMG_F3_BZ;
  static_assert(BX * BY * BZ == TPB, "FineOp tile must have TPB threads");
  static constexpr int HX = BX + 2, HY = BY + 2, HZ = DIM == 2 ? 1 : BZ + 2;
  static constexpr int EX = BX + 1, EY = BY + 1, EZ = DIM == 2 ? 1 : BZ + 1;
  static constexpr int NH = HX * HY * HZ, NEL = EX * EY * EZ;
  static constexpr size_t SMEM_BYTES = sizeof(double) * (NH * DIM + NEL) + NH;
  // resident blocks per SM the register budget is sized for (2D: 48 regs, 3D: 80)
#ifndef TMG_F3_MINB
#define TMG_F3_MINB 3  // 3D: 80 registers, 3 CTAs per SM (measured best of 2/3/4)
#endif
#ifndef TMG_F2_MINB
#define TMG_F2_MINB 5  // 2D: 48 registers, 5 CTAs per SM (measured: sweep 5.82 -> 5.45 us vs 4 / 6 CTAs)
#endif
  // 3D rows are streamed (STREAM: one launch shape for every 3D level-0 kernel):
  // by default the element-centric character-basis operator of tmg_fine3h.cuh
  // (~175 FP64 operations per element instead of 576, TMA-fed, warp
  // specialised); -DTMG_F3S selects the register-prefetch variant of tmg_fine3s.cuh (measured slower), -DTMG_FINE3_TILE the node-per-thread tile below
  // (row()), kept as the measured A/B baseline.
#ifdef TMG_FINE3_TILE
  static constexpr bool STREAM = false;
#else
  static constexpr bool STREAM = DIM == 3;
#endif
#ifndef TMG_F3H_MINB
#define TMG_F3H_MINB 1
#endif
#ifndef TMG_F3H_TY
#define TMG_F3H_TY 8  // consumer warps of the 3D stream (rows of 32 element columns)
#endif
#if defined(TMG_FINE3_TILE)
  static constexpr int MINB = DIM == 2 ? TMG_F2_MINB : TMG_F3_MINB;
  static constexpr int THREADS = TPB;
#elif defined(TMG_F3P)
#ifndef TMG_F3H_NPROD
#define TMG_F3H_NPROD 3
#endif
  static constexpr int MINB = DIM == 2 ? TMG_F2_MINB : 1;  // 3D: one CTA per SM (tmg_fine3p.cuh)
  static constexpr int THREADS = DIM == 2 ? TPB : 64 * TMG_F3H_TY + 32 * TMG_F3H_NPROD;  // 3D: a warp pair per row + the TMA producer warps
#elif !defined(TMG_F3S)
  static constexpr int MINB = DIM == 2 ? TMG_F2_MINB : TMG_F3H_MINB;  // 3D: one CTA per SM (tmg_fine3h.cuh)
#ifndef TMG_F3H_NPROD
#define TMG_F3H_NPROD 3
#endif
  static constexpr int THREADS = DIM == 2 ? TPB : 32 * TMG_F3H_TY + 32 * TMG_F3H_NPROD;  // 3D: consumer warps + the TMA producer warp(s)
#else
#ifndef TMG_F3S_TY
#define TMG_F3S_TY 8
#endif
#ifndef TMG_F3S_MINB
#define TMG_F3S_MINB 2
#endif
  static constexpr int MINB = DIM == 2 ? TMG_F2_MINB : TMG_F3S_MINB;  // 3D: tmg_fine3s.cuh
  static constexpr int THREADS = DIM == 2 ? TPB : 32 * TMG_F3S_TY;
#endif

  // out = (Z K Z + I_fixed) row block of node (i,j,k) applied to src.  Called by
  // ALL threads of the block (it stages the tile and synchronises); only threads
  // with `active` compute.
  // 2D direct path (compile with -DTMG_FINE_DIRECT=1): each thread loads its 3x3
  // node neighbourhood, 2x2 element moduli and masks straight from L1/L2 -- no
  // tile, no barrier.  10 % faster than the tile in the stand-alone prototype
  // (tools/proto/fine2d.cu) but 4 % slower inside the library (64-register cap
  // of the 4-blocks/SM budget), so the tile stays the default.
  template <class Src>
  __device__ void row_direct(int node, int i, int j, const Src& src, double out[DIM], double self[DIM]) const {
    double xv[9][DIM];
    unsigned mk[9];
    double ev[4];
#pragma unroll
    for (int s2 = 0; s2 < 9; ++s2) {
      const int ii = i + s2 % 3 - 1, jj = j + s2 / 3 - 1;
      const bool in = ii >= 0 && ii < L.nn[0] && jj >= 0 && jj < L.nn[1];
      const int m = in ? L.id(ii, jj, 0) : node;
      src.load(m, ii, jj, 0, xv[s2]);
      mk[s2] = in ? (unsigned)__ldg(mask + m) : 0u;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int ex = i - 1 + (e & 1), ey = j - 1 + (e >> 1);
      const bool in = ex >= 0 && ex < ne[0] && ey >= 0 && ey < ne[1];
      ev[e] = in ? __ldg(E + elem_id(in ? ex : 0, in ? ey : 0, 0)) : 0.0;
    }
#pragma unroll
    for (int d = 0; d < DIM; ++d) self[d] = xv[4][d];
#pragma unroll
    for (int s2 = 0; s2 < 9; ++s2)
#pragma unroll
      for (int d = 0; d < DIM; ++d)
        if (!((mk[s2] >> d) & 1u)) xv[s2][d] = 0.0;
    double acc[DIM];
#pragma unroll
    for (int c = 0; c < DIM; ++c) acc[c] = 0.0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int ex = e & 1, ey = e >> 1;  // element (i-1+ex, j-1+ey)
      const int ln = corner_of(1 - ex, 1 - ey, 0);
      double t[DIM];
#pragma unroll
      for (int c = 0; c < DIM; ++c) t[c] = 0.0;
#pragma unroll
      for (int m = 0; m < NN; ++m) {
        const int s2 = Slots<DIM>::of(ex - 1 + corner_x(m), ey - 1 + corner_y(m), 0);
#pragma unroll
        for (int c = 0; c < DIM; ++c)
#pragma unroll
          for (int d = 0; d < DIM; ++d) t[c] += ke[(ln * DIM + c) * NE + m * DIM + d] * xv[s2][d];
      }
#pragma unroll
      for (int c = 0; c < DIM; ++c) acc[c] += ev[e] * t[c];
    }
#pragma unroll
    for (int c = 0; c < DIM; ++c) out[c] = ((mk[4] >> c) & 1u) ? acc[c] : self[c];
  }

  template <class Src>
  __device__ void row(bool active, int node, int i, int j, int k, const Src& src, double out[DIM],
                      double self[DIM]) const {
#ifndef TMG_FINE_DIRECT  // measured in the library: tile 5.8 us vs direct 6.1 us per sweep
#define TMG_FINE_DIRECT 0
#endif
    if constexpr (TMG_FINE_DIRECT && DIM == 2 && Src::DIRECT) {
      if (active) row_direct(node, i, j, src, out, self);
      return;
    }
    extern __shared__ double tmg_sm[];
    double* xs = tmg_sm;
    double* es = xs + NH * DIM;
    unsigned char* ms = reinterpret_cast<unsigned char*>(es + NEL);
    const int i0 = blockIdx.x * BX - 1, j0 = blockIdx.y * BY - 1, k0 = DIM == 3 ? (int)blockIdx.z * BZ - 1 : 0;
    // All loads of the tile are issued before the first shared store (the loops
    // below are unrolled over the <= PH / PE passes of the TPB threads), so a
    // block pays one global round trip for its tile, not one per pass.
    const int t0 = lin_tid();
    constexpr int PH = (NH + TPB - 1) / TPB, PE = (NEL + TPB - 1) / TPB;
    double v[PH][DIM];
    unsigned mk[PH];
    double ev[PE];
#pragma unroll
    for (int u = 0; u < PH; ++u) {
      const int t = t0 + u * TPB;
      const int hx = t % HX, hy = (t / HX) % HY, hz = t / (HX * HY);
      const int gi = i0 + hx, gj = j0 + hy, gk = DIM == 3 ? k0 + hz : 0;
      mk[u] = 0u;
      if (t < NH && L.inside(gi, gj, gk)) {
        const int m = L.id(gi, gj, gk);
        src.load(m, gi, gj, gk, v[u]);
        mk[u] = __ldg(mask + m);
      } else {
#pragma unroll
        for (int d = 0; d < DIM; ++d) v[u][d] = 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < PE; ++u) {
      const int t = t0 + u * TPB;
      const int ex = t % EX, ey = (t / EX) % EY, ez = t / (EX * EY);
      const int gi = i0 + ex, gj = j0 + ey, gk = DIM == 3 ? k0 + ez : 0;
      const bool ok = t < NEL && gi >= 0 && gi < ne[0] && gj >= 0 && gj < ne[1] &&
                      (DIM == 2 || (gk >= 0 && gk < ne[2]));
      ev[u] = ok ? __ldg(E + elem_id(gi, gj, gk)) : 0.0;
    }
    // 3D: the tile holds masked values (each staged value is read by up to 27
    // threads; masking once here removes 81 selects per row), the row's own
    // unmasked value and mask come straight from global memory
    constexpr bool PREMASK = DIM == 3;
    unsigned self_mk = 0u;
    if (PREMASK && active) {
      src.load(node, i, j, k, self);
      self_mk = __ldg(mask + node);
    }
#pragma unroll
    for (int u = 0; u < PH; ++u) {
      const int t = t0 + u * TPB;
      if (t < NH) {
#pragma unroll
        for (int d = 0; d < DIM; ++d) xs[t * DIM + d] = (!PREMASK || ((mk[u] >> d) & 1u)) ? v[u][d] : 0.0;
        if (!PREMASK) ms[t] = (unsigned char)mk[u];
      }
    }
#pragma unroll
    for (int u = 0; u < PE; ++u) {
      const int t = t0 + u * TPB;
      if (t < NEL) es[t] = ev[u];
    }
    __syncthreads();
    if (!active) return;
    const int tx = threadIdx.x, ty = threadIdx.y, tz = DIM == 3 ? threadIdx.z : 0;
    constexpr int NS = Slots<DIM>::NS;
    double xv[NS][DIM];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int h = (tx + 1 + Slots<DIM>::dx(s)) + HX * ((ty + 1 + Slots<DIM>::dy(s)) + HY * (tz + (DIM == 3 ? 1 : 0) +
                                                                                                Slots<DIM>::dz(s)));
      if constexpr (PREMASK) {
#pragma unroll
        for (int d = 0; d < DIM; ++d) xv[s][d] = xs[h * DIM + d];
      } else {
        const unsigned mk = ms[h];
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
          const double v = xs[h * DIM + d];
          if (s == NS / 2) self[d] = v;
          xv[s][d] = ((mk >> d) & 1u) ? v : 0.0;
        }
      }
    }
    double acc[DIM];
#pragma unroll
    for (int c = 0; c < DIM; ++c) acc[c] = 0.0;
#pragma unroll
    for (int ez = 0; ez < (DIM == 3 ? 2 : 1); ++ez)
#pragma unroll
      for (int ey = 0; ey < 2; ++ey)
#pragma unroll
        for (int ex = 0; ex < 2; ++ex) {
          const double Ee = es[(tx + ex) + EX * ((ty + ey) + EY * (tz + ez))];
          const int ln = corner_of(1 - ex, 1 - ey, DIM == 3 ? 1 - ez : 0);
          double t[DIM];
#pragma unroll
          for (int c = 0; c < DIM; ++c) t[c] = 0.0;
#pragma unroll
          for (int m = 0; m < NN; ++m) {
            const int s = Slots<DIM>::of(ex - 1 + corner_x(m), ey - 1 + corner_y(m),
                                         DIM == 3 ? ez - 1 + corner_z(m) : 0);
#pragma unroll
            for (int c = 0; c < DIM; ++c)
#pragma unroll
              for (int d = 0; d < DIM; ++d) t[c] += ke[(ln * DIM + c) * NE + m * DIM + d] * xv[s][d];
          }
#pragma unroll
          for (int c = 0; c < DIM; ++c) acc[c] += Ee * t[c];
        }
    const unsigned mn = PREMASK ? self_mk : ms[(tx + 1) + HX * ((ty + 1) + HY * (tz + (DIM == 3 ? 1 : 0)))];
#pragma unroll
    for (int c = 0; c < DIM; ++c) out[c] = ((mn >> c) & 1u) ? acc[c] : self[c];
  }

  // block (i -> j) of Z K Z + I_fixed, i and j lattice neighbours (|i-j|_inf <= 1)
  __device__ void block(int i0, int i1, int i2, int j0, int j1, int j2, double blk[DD]) const {
#pragma unroll
    for (int t = 0; t < DD; ++t) blk[t] = 0.0;
    const int lo0 = max(max(i0, j0) - 1, 0), hi0 = min(min(i0, j0), ne[0] - 1);
    const int lo1 = max(max(i1, j1) - 1, 0), hi1 = min(min(i1, j1), ne[1] - 1);
    const int lo2 = DIM == 3 ? max(max(i2, j2) - 1, 0) : 0;
    const int hi2 = DIM == 3 ? min(min(i2, j2), ne[2] - 1) : 0;
    for (int ez = lo2; ez <= hi2; ++ez)
      for (int ey = lo1; ey <= hi1; ++ey)
        for (int ex = lo0; ex <= hi0; ++ex) {
          const double Ee = E[elem_id(ex, ey, ez)];
          const int li = corner_of(i0 - ex, i1 - ey, DIM == 3 ? i2 - ez : 0);
          const int lj = corner_of(j0 - ex, j1 - ey, DIM == 3 ? j2 - ez : 0);
#pragma unroll
          for (int a = 0; a < DIM; ++a)
#pragma unroll
            for (int b = 0; b < DIM; ++b) blk[a * DIM + b] += Ee * ke[(li * DIM + a) * NE + lj * DIM + b];
        }
    const unsigned mi = mask[L.id(i0, i1, i2)], mj = mask[L.id(j0, j1, j2)];
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int b = 0; b < DIM; ++b)
        if (!(((mi >> a) & 1u) && ((mj >> b) & 1u))) blk[a * DIM + b] = 0.0;
    if (i0 == j0 && i1 == j1 && i2 == j2) {
#pragma unroll
      for (int a = 0; a < DIM; ++a)
        if (!((mi >> a) & 1u)) blk[a * DIM + a] = 1.0;
    }
  }
};

}  // namespace tmg
#include "tmg_fine3h.cuh"
#include "tmg_fine3s.cuh"
#include "tmg_fine3p.cuh"
namespace tmg {
// the streamed 3D row path (FineOp<3>::STREAM): character-basis elements, the
// epilogue's input vectors staged by the producer warp (ein)
template <class Src, class Epi>
__device__ __forceinline__ void fine3_rows(const FineOp<3>& op, const Src& src, const f3h::EpiIn& ein, Epi&& epi) {
#if defined(TMG_F3P)
  fine3p_rows(op, src, ein, static_cast<Epi&&>(epi));
#elif !defined(TMG_F3S)
  fine3h_rows(op, src, ein, static_cast<Epi&&>(epi));
#else
  fine3s_rows(op, src, ein, static_cast<Epi&&>(epi));
#endif
}
#if defined(TMG_F3P)
inline dim3 fine3_grid(const Lat& L) { return f3h::grid(L); }
constexpr int fine3_threads() { return f3p::NTHP; }
constexpr size_t fine3_smem() { return f3p::SMEM_BYTES_P; }
#elif !defined(TMG_F3S)
inline dim3 fine3_grid(const Lat& L) { return f3h::grid(L); }
constexpr int fine3_threads() { return f3h::NTH; }
constexpr size_t fine3_smem() { return f3h::SMEM_BYTES; }
#else
inline dim3 fine3_grid(const Lat& L) { return f3s::grid(L); }
constexpr int fine3_threads() { return f3s::NT; }
constexpr size_t fine3_smem() { return f3s::SMEM_BYTES; }
#endif

// ----------------------------------------------------------------------------
// StencilOp
// ----------------------------------------------------------------------------
template <int DIM>
struct StencilOp {
  // 2D: a Galerkin operator is symmetric, so only the centre and the "upper"
  // slots (s >= C0, offsets lexicographically >= 0) are stored, A[(h*DD + q)*n +
  // node] with h = s - C0; a lower slot of node i is the transposed upper block of
  // its neighbour, read at the neighbour's index (unit-stride across a warp):
  // 5 of 9 blocks per node (config-1 GMG PCG iteration -2.5 %).  3D keeps all 27
  // slots (C0 = 0): the mirrored loads of 13 slots push the batched, fully
  // unrolled row past its register budget (measured 84 -> 98-216 us per config-4
  // level-1 sweep in every variant tried).
#ifndef TMG_ST_SYM3
#define TMG_ST_SYM3 0
#endif
  static constexpr int NS = Slots<DIM>::NS, DD = DIM * DIM, C0 = (DIM == 2 || TMG_ST_SYM3) ? NS / 2 : 0,
                       NH = NS - C0;
  Lat L;
  const double* __restrict__ A;
  // block of slot s at node (i, j, k) into av; a lower slot whose neighbour is
  // outside the lattice reads the node's own (finite) storage: the caller zeroes
  // the block (block()) or the neighbour's value (row()) then
  __device__ __forceinline__ bool slot_block(int s, int node, int i, int j, int k, double av[DD]) const {
    const int n = (int)L.n;
    if (s >= C0) {
#pragma unroll
      for (int q = 0; q < DD; ++q) av[q] = ldv(A + ((s - C0) * DD + q) * n + node);
      return true;
    }
    const int ii = i + Slots<DIM>::dx(s), jj = j + Slots<DIM>::dy(s), kk = k + Slots<DIM>::dz(s);
    const bool in = L.inside(ii, jj, DIM == 3 ? kk : 0);
    const int nb = in ? L.id(ii, jj, DIM == 3 ? kk : 0) : node;
    const int h = (NS - 1 - s) - C0;
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int b = 0; b < DIM; ++b) av[a * DIM + b] = ldv(A + (h * DD + b * DIM + a) * n + nb);
    return in;
  }

  // Loads are issued in batches of G slots (all coefficient and vector loads of a
  // batch before any arithmetic) so a thread has G*(DD+DIM) loads in flight --
  // coarse levels have too few threads to hide L2 latency by occupancy alone.
  static constexpr size_t SMEM_BYTES = 0;
  static constexpr int BX = 32, BY = DIM == 2 ? 8 : 4, BZ = DIM == 2 ? 1 : 2;  // = node_block<DIM>()
#ifndef TMG_ST_MINB
#define TMG_ST_MINB 2  // 3D stencil rows: 128 instead of 254 registers (config-3 PCG 370.8 -> 355.7 us/iter; 3 / 4: slower)
#endif
  static constexpr int MINB = TMG_ST_MINB;  // large register budget: batched loads in flight
  static constexpr int THREADS = TPB;
  static constexpr bool STREAM = false;
  // 3D symmetric storage (TMG_ST_SYM3): the centre block and, pair by pair, the
  // upper block A_h(i) with x at node i + off and the transposed upper block of
  // the node below, A_h(i - off)^T, with x at node i - off.  Every stored block is
  // read by two rows (its owner's and the row of the node it couples to, one to
  // nn0*nn1 nodes later): HBM sees 14 of the 27 blocks per node, the second
  // read is an L2 hit.  GP pairs of loads (2 x 9 coefficients + 2 x 3 vector
  // entries each) are in flight per batch.
  template <class Src>
  __device__ __forceinline__ void row_sym3(int node, int i, int j, int k, const Src& src, double out[3],
                                           double self[3]) const {
    const int n = (int)L.n;
    double acc[3];
    {
      double xv[3], av[9];
      src.load(node, i, j, k, xv);
#pragma unroll
      for (int q = 0; q < 9; ++q) av[q] = ldv(A + q * n + node);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        self[a] = xv[a];
        acc[a] = av[a * 3] * xv[0] + av[a * 3 + 1] * xv[1] + av[a * 3 + 2] * xv[2];
      }
    }
    constexpr int GP = 2, NP = NS / 2;  // 13 pairs
#pragma unroll
    for (int h0 = 1; h0 <= NP; h0 += GP) {
      double au[GP][9], al[GP][9], xu[GP][3], xl[GP][3];
#pragma unroll
      for (int g = 0; g < GP; ++g) {
        const int h = h0 + g;
        if (h > NP) {
#pragma unroll
          for (int q = 0; q < 9; ++q) au[g][q] = al[g][q] = 0.0;
#pragma unroll
          for (int d = 0; d < 3; ++d) xu[g][d] = xl[g][d] = 0.0;
          continue;
        }
        const int s = C0 + h, dx = Slots<3>::dx(s), dy = Slots<3>::dy(s), dz = Slots<3>::dz(s);
        // upper neighbour (clamped: the stored block is zero when it is off the lattice)
        const int iu = min(max(i + dx, 0), L.nn[0] - 1), ju = min(max(j + dy, 0), L.nn[1] - 1),
                  ku = min(max(k + dz, 0), L.nn[2] - 1);
        src.load(L.id(iu, ju, ku), iu, ju, ku, xu[g]);
#pragma unroll
        for (int q = 0; q < 9; ++q) au[g][q] = ldv(A + (h * 9 + q) * n + node);
        // lower neighbour: its upper block, transposed
        const int il = i - dx, jl = j - dy, kl = k - dz;
        const bool in = L.inside(il, jl, kl);
        const int nb = in ? L.id(il, jl, kl) : node;
        src.load(nb, in ? il : i, in ? jl : j, in ? kl : k, xl[g]);
        if (!in) {
#pragma unroll
          for (int d = 0; d < 3; ++d) xl[g][d] = 0.0;
        }
#pragma unroll
        for (int q = 0; q < 9; ++q) al[g][q] = ldv(A + (h * 9 + q) * n + nb);
      }
      reg_fence<GP * 9>(&au[0][0]);
      reg_fence<GP * 9>(&al[0][0]);
      reg_fence<GP * 3>(&xu[0][0]);
      reg_fence<GP * 3>(&xl[0][0]);
#pragma unroll
      for (int g = 0; g < GP; ++g)
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) acc[a] += au[g][a * 3 + b] * xu[g][b] + al[g][b * 3 + a] * xl[g][b];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) out[c] = acc[c];
  }

  template <class Src>
  __device__ void row(bool active, int node, int i, int j, int k, const Src& src, double out[DIM],
                      double self[DIM]) const {
    if (!active) return;
    if constexpr (DIM == 3 && C0 > 0) {
      row_sym3(node, i, j, k, src, out, self);
      return;
    }
    constexpr int G = DIM == 2 ? 9 : 3;
    double acc[DIM];
#pragma unroll
    for (int c = 0; c < DIM; ++c) acc[c] = 0.0;
#pragma unroll
    for (int s0 = 0; s0 < NS; s0 += G) {
      double xv[G][DIM], av[G][DD];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int s = s0 + g;
        const int ii = min(max(i + Slots<DIM>::dx(s), 0), L.nn[0] - 1);
        const int jj = min(max(j + Slots<DIM>::dy(s), 0), L.nn[1] - 1);
        const int kk = DIM == 3 ? min(max(k + Slots<DIM>::dz(s), 0), L.nn[2] - 1) : 0;
        src.load(L.id(ii, jj, kk), ii, jj, kk, xv[g]);  // clamped; upper-slot coefficients are 0 there
        if (!slot_block(s, node, i, j, k, av[g])) {      // lower slot off the lattice: no contribution
#pragma unroll
          for (int d = 0; d < DIM; ++d) xv[g][d] = 0.0;
        }
      }
      reg_fence<G * DIM>(&xv[0][0]);
      reg_fence<G * DD>(&av[0][0]);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (s0 + g == NS / 2) {
#pragma unroll
          for (int d = 0; d < DIM; ++d) self[d] = xv[g][d];
        }
#pragma unroll
        for (int a = 0; a < DIM; ++a)
#pragma unroll
          for (int b = 0; b < DIM; ++b) acc[a] += av[g][a * DIM + b] * xv[g][b];
      }
    }
#pragma unroll
    for (int c = 0; c < DIM; ++c) out[c] = acc[c];
  }

  __device__ void block(int i0, int i1, int i2, int j0, int j1, int j2, double blk[DD]) const {
    const int s = Slots<DIM>::of(j0 - i0, j1 - i1, DIM == 3 ? j2 - i2 : 0);
    if (!slot_block(s, L.id(i0, i1, i2), i0, i1, i2, blk))
#pragma unroll
      for (int t = 0; t < DD; ++t) blk[t] = 0.0;
  }
};

// launch geometry of the row kernels below: streamed operators (FineOp<3>)
// launch one CTA per 16x16 node column and z-chunk, the others one thread per node
template <int DIM, class Op>
inline dim3 row_grid(const Lat& L) {
  if constexpr (Op::STREAM) return fine3_grid(L);
  else return dim3((L.nn[0] + Op::BX - 1) / Op::BX, (L.nn[1] + Op::BY - 1) / Op::BY, (L.nn[2] + Op::BZ - 1) / Op::BZ);
}
template <int DIM, class Op>
inline dim3 row_block() {
  if constexpr (Op::STREAM) return dim3(fine3_threads(), 1, 1);
  else return dim3(Op::BX, Op::BY, Op::BZ);
}
template <class Op>
constexpr size_t row_smem() {
  if constexpr (Op::STREAM) return fine3_smem();
  else return Op::SMEM_BYTES;
}
#define TMG_ROW_OP_LAUNCH_L(Lat_, op_) \
  row_grid<DIM, decltype(op_)>(Lat_), row_block<DIM, decltype(op_)>(), row_smem<decltype(op_)>()

// ----------------------------------------------------------------------------
// generic node-parallel kernels (2D/3D launch: node_grid / node_block)
// ----------------------------------------------------------------------------
#define TMG_NODE_IDX                                                                   \
  const int ci = blockIdx.x * blockDim.x + threadIdx.x;                                \
  const int cj = blockIdx.y * blockDim.y + threadIdx.y;                                \
  const int ck = blockIdx.z * blockDim.z + threadIdx.z;                                \
  const bool active = ci < op.L.nn[0] && cj < op.L.nn[1] && ck < op.L.nn[2];           \
  const int node = active ? op.L.id(ci, cj, ck) : 0;

// y = A x
template <int DIM, class Op>
__global__ void __launch_bounds__(Op::THREADS, Op::MINB) k_apply(const __grid_constant__ Op op, const double* __restrict__ x,
                                               double* __restrict__ y) {
  TMG_PDL_ENTRY;
  if constexpr (Op::STREAM) {
    fine3_rows(op, VecSrc<DIM>{x}, f3h::EpiIn{{nullptr, nullptr}},
               [&](int node, int, int, int, const double* out, const double*, const double (*)[3]) {
                 store_node<DIM>(y, node, out);
               });
  } else {
    TMG_NODE_IDX
    double out[DIM], self[DIM];
    op.row(active, node, ci, cj, ck, VecSrc<DIM>{x}, out, self);
    if (!active) return;
    store_node<DIM>(y, node, out);
  }
}

// y = ds .* A (ds .* v)   (Lanczos on D^-1/2 A D^-1/2)
template <int DIM, class Op>
__global__ void __launch_bounds__(Op::THREADS, Op::MINB) k_apply_sym(const __grid_constant__ Op op, const double* __restrict__ v,
                                                   const double* __restrict__ ds, double* __restrict__ y) {
  TMG_PDL_ENTRY;
  if constexpr (Op::STREAM) {
    fine3_rows(op, ScaledSrc<DIM>{v, ds}, f3h::EpiIn{{ds, nullptr}},
               [&](int node, int, int, int, const double* o, const double*, const double (*e)[3]) {
                 double out[DIM];
#pragma unroll
                 for (int c = 0; c < DIM; ++c) out[c] = o[c] * e[0][c];
                 store_node<DIM>(y, node, out);
               });
  } else {
    TMG_NODE_IDX
    double out[DIM], self[DIM], d[DIM];
    op.row(active, node, ci, cj, ck, ScaledSrc<DIM>{v, ds}, out, self);
    if (!active) return;
    load_node<DIM>(ds, node, d);
#pragma unroll
    for (int c = 0; c < DIM; ++c) out[c] *= d[c];
    store_node<DIM>(y, node, out);
  }
}

// r = b - A x
template <int DIM, class Op>
__global__ void __launch_bounds__(Op::THREADS, Op::MINB) k_residual(const __grid_constant__ Op op, const double* __restrict__ x,
                                                  const double* __restrict__ b, double* __restrict__ r) {
  TMG_PDL_ENTRY;
  if constexpr (Op::STREAM) {
    fine3_rows(op, VecSrc<DIM>{x}, f3h::EpiIn{{b, nullptr}},
               [&](int node, int, int, int, const double* o, const double*, const double (*e)[3]) {
                 double bb[DIM];
#pragma unroll
                 for (int c = 0; c < DIM; ++c) bb[c] = e[0][c] - o[c];
                 store_node<DIM>(r, node, bb);
               });
  } else {
    TMG_NODE_IDX
    double out[DIM], self[DIM], bb[DIM];
    load_node<DIM>(b, node, bb);  // in flight while the tile is staged
    op.row(active, node, ci, cj, ck, VecSrc<DIM>{x}, out, self);
    if (!active) return;
#pragma unroll
    for (int c = 0; c < DIM; ++c) out[c] = bb[c] - out[c];
    store_node<DIM>(r, node, out);
  }
}

// xo = xs + w D^-1 (b - A xs)   (weighted Jacobi sweep, multigrid.py:57) where xs is
// the source vector (x, or x + P e when the coarse correction is fused in).
// DOT: also reduce sum(xo . b) into red (the PCG r.z of the last level-0 sweep).
template <int DIM, class Op, class Src, bool DOT>
__device__ __forceinline__ void jacobi_body(const Op& op, const Src& src, const double* __restrict__ b,
                                            const double* __restrict__ dinv, const double* __restrict__ wp,
                                            double* __restrict__ xo, const Red& red) {
  TMG_NODE_IDX
  double v = 0.0;
  double out[DIM], self[DIM], bb[DIM], d[DIM];
  load_node<DIM>(b, node, bb);  // epilogue operands in flight while the tile is staged
  load_node<DIM>(dinv, node, d);
  const double w = *wp;
  op.row(active, node, ci, cj, ck, src, out, self);
  if (active) {
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
      out[c] = self[c] + w * (d[c] * (bb[c] - out[c]));
      if (DOT) v += out[c] * bb[c];
    }
    store_node<DIM>(xo, node, out);
  }
  if (DOT) grid_reduce(v, red);
}

template <int DIM, class Op, bool DOT>
__global__ void __launch_bounds__(Op::THREADS, Op::MINB) k_jacobi(const __grid_constant__ Op op, const double* __restrict__ x,
                                                const double* __restrict__ b, const double* __restrict__ dinv,
                                                const double* __restrict__ wp, double* __restrict__ xo, Red red) {
  TMG_PDL_ENTRY;
  if constexpr (Op::STREAM) {
    const double w = *wp;
    double v = 0.0;
    fine3_rows(op, VecSrc<DIM>{x}, f3h::EpiIn{{b, dinv}},
               [&](int node, int, int, int, const double* o, const double* self, const double (*e)[3]) {
                 double out[DIM];
#pragma unroll
                 for (int c = 0; c < DIM; ++c) {
                   out[c] = self[c] + w * (e[1][c] * (e[0][c] - o[c]));
                   if (DOT) v += out[c] * e[0][c];
                 }
                 store_node<DIM>(xo, node, out);
               });
    if (DOT) grid_reduce(v, red);
  } else {
    jacobi_body<DIM, Op, VecSrc<DIM>, DOT>(op, VecSrc<DIM>{x}, b, dinv, wp, xo, red);
  }
}

// first post-smoothing sweep with the coarse-grid correction fused in:
// xs = x + P e evaluated on the fly, xo = xs + w D^-1 (b - A xs)
template <int DIM, class Op, bool DOT>
__global__ void __launch_bounds__(Op::THREADS, Op::MINB) k_prolong_jacobi(const __grid_constant__ Op op, const double* __restrict__ x,
                                                        const double* __restrict__ e, Coarsening T,
                                                        const double* __restrict__ b, const double* __restrict__ dinv,
                                                        const double* __restrict__ wp, double* __restrict__ xo,
                                                        Red red) {
  TMG_PDL_ENTRY;
  jacobi_body<DIM, Op, ProlongSrc<DIM>, DOT>(op, ProlongSrc<DIM>{x, e, T}, b, dinv, wp, xo, red);
}

// xo = x + w B^-1 (b - A x), B the nodal diagonal blocks (multigrid.py:90)
template <int DIM, class Op>
__global__ void __launch_bounds__(Op::THREADS, Op::MINB) k_bjacobi(const __grid_constant__ Op op, const double* __restrict__ x,
                                                 const double* __restrict__ b, const double* __restrict__ binv,
                                                 const double* __restrict__ wp, double* __restrict__ xo) {
  TMG_PDL_ENTRY;
  if constexpr (Op::STREAM) {
    const double w = *wp;
    fine3_rows(op, VecSrc<DIM>{x}, f3h::EpiIn{{b, nullptr}},
               [&](int node, int, int, int, const double* o, const double* self, const double (*e)[3]) {
      double r[DIM], out[DIM];
#pragma unroll
      for (int c = 0; c < DIM; ++c) r[c] = e[0][c] - o[c];
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < DIM; ++c) s += binv[node * DIM * DIM + a * DIM + c] * r[c];
        out[a] = self[a] + w * s;
      }
      store_node<DIM>(xo, node, out);
    });
    return;
  }
  TMG_NODE_IDX
  double out[DIM], self[DIM], r[DIM];
  op.row(active, node, ci, cj, ck, VecSrc<DIM>{x}, out, self);
  if (!active) return;
  const double w = *wp;
  load_node<DIM>(b, node, r);
#pragma unroll
  for (int c = 0; c < DIM; ++c) r[c] -= out[c];
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < DIM; ++c) s += binv[node * DIM * DIM + a * DIM + c] * r[c];
    out[a] = self[a] + w * s;
  }
  store_node<DIM>(xo, node, out);
}

// One Chebyshev step (multigrid.py:131 recurrence):
//   p' = z + beta p ; x += alpha p' ; r' = r - alpha A p'
// with z = D^-1 r (zs = r, Jacobi-Chebyshev) or z = SOR solve of r (zs = z, dinv = nullptr).
template <int DIM, class Op>
__global__ void __launch_bounds__(Op::THREADS, Op::MINB) k_cheb(const __grid_constant__ Op op, const double* __restrict__ r,
                                              const double* __restrict__ zs, const double* __restrict__ p, const double* __restrict__ dinv,
                                              const double* __restrict__ coef, int step, int x_zero,
                                              double* __restrict__ x, double* __restrict__ po,
                                              double* __restrict__ ro) {
  TMG_PDL_ENTRY;
  if constexpr (Op::STREAM) {
    const double alpha = coef[2 * step], beta = step == 0 ? 0.0 : coef[2 * step + 1];
    fine3_rows(op, ChebSrc<DIM>{zs, p, dinv, beta}, f3h::EpiIn{{r, x_zero ? nullptr : x}},
               [&](int node, int, int, int, const double* o, const double* pv, const double (*e)[3]) {
      double rr[DIM], xv[DIM];
#pragma unroll
      for (int c = 0; c < DIM; ++c) {
        rr[c] = e[0][c];
        xv[c] = x_zero ? 0.0 : e[1][c];
      }
#pragma unroll
      for (int c = 0; c < DIM; ++c) {
        xv[c] += alpha * pv[c];
        rr[c] -= alpha * o[c];
      }
      if (po) store_node<DIM>(po, node, pv);
      store_node<DIM>(x, node, xv);
      if (ro) store_node<DIM>(ro, node, rr);
    });
    return;
  }
  TMG_NODE_IDX
  const double alpha = coef[2 * step], beta = step == 0 ? 0.0 : coef[2 * step + 1];
  double out[DIM], pv[DIM], rr[DIM], xv[DIM];
  op.row(active, node, ci, cj, ck, ChebSrc<DIM>{zs, p, dinv, beta}, out, pv);
  if (!active) return;
  load_node<DIM>(r, node, rr);
  if (x_zero) {
#pragma unroll
    for (int c = 0; c < DIM; ++c) xv[c] = 0.0;
  } else {
    load_node<DIM>(x, node, xv);
  }
#pragma unroll
  for (int c = 0; c < DIM; ++c) {
    xv[c] += alpha * pv[c];
    rr[c] -= alpha * out[c];
  }
  if (po) store_node<DIM>(po, node, pv);  // nullptr: last step of a pass, p' is never read
  store_node<DIM>(x, node, xv);
  if (ro) store_node<DIM>(ro, node, rr);  // nullptr: last step of a pass, r' is never read
}

// diagonal / nodal block inverses of a level operator
template <int DIM, class Op>
__global__ void __launch_bounds__(TPB, 1) k_diag(const __grid_constant__ Op op, double* __restrict__ diag,
                                              double* __restrict__ binv, unsigned* __restrict__ bad) {
  TMG_PDL_ENTRY;
  TMG_NODE_IDX
  if (!active) return;
  double blk[DIM * DIM];
  op.block(ci, cj, ck, ci, cj, ck, blk);
#pragma unroll
  for (int c = 0; c < DIM; ++c) {
    diag[node * DIM + c] = blk[c * DIM + c];
    if (blk[c * DIM + c] == 0.0) atomicOr(bad, 1u);
  }
  if (binv) {
    double inv[DIM * DIM];
    double det;
    if (DIM == 2) {
      det = blk[0] * blk[3] - blk[1] * blk[2];
      inv[0] = blk[3] / det; inv[1] = -blk[1] / det; inv[2] = -blk[2] / det; inv[3] = blk[0] / det;
    } else {
      const double* m = blk;
      const double c00 = m[4] * m[8] - m[5] * m[7], c01 = m[5] * m[6] - m[3] * m[8], c02 = m[3] * m[7] - m[4] * m[6];
      det = m[0] * c00 + m[1] * c01 + m[2] * c02;
      inv[0] = c00 / det; inv[1] = (m[2] * m[7] - m[1] * m[8]) / det; inv[2] = (m[1] * m[5] - m[2] * m[4]) / det;
      inv[3] = c01 / det; inv[4] = (m[0] * m[8] - m[2] * m[6]) / det; inv[5] = (m[2] * m[3] - m[0] * m[5]) / det;
      inv[6] = c02 / det; inv[7] = (m[1] * m[6] - m[0] * m[7]) / det; inv[8] = (m[0] * m[4] - m[1] * m[3]) / det;
    }
    if (!(fabs(det) >= 1e-300)) atomicOr(bad, 2u);
#pragma unroll
    for (int t = 0; t < DIM * DIM; ++t) binv[node * DIM * DIM + t] = inv[t];
  }
}

// dense row-major copy of a level operator (small coarsest levels only)
template <int DIM, class Op>
__global__ void __launch_bounds__(TPB, 1) k_to_dense(const __grid_constant__ Op op, double* __restrict__ Ad) {
  TMG_PDL_ENTRY;
  TMG_NODE_IDX
  if (!active) return;
  const long long n = op.L.n * DIM;
  for (int s = 0; s < Slots<DIM>::NS; ++s) {
    const int ii = ci + Slots<DIM>::dx(s), jj = cj + Slots<DIM>::dy(s), kk = ck + Slots<DIM>::dz(s);
    if (!op.L.inside(ii, jj, kk)) continue;
    double blk[DIM * DIM];
    op.block(ci, cj, ck, ii, jj, kk, blk);
    const long long m = op.L.id(ii, jj, kk);
    for (int a = 0; a < DIM; ++a)
      for (int b = 0; b < DIM; ++b) Ad[((long long)node * DIM + a) * n + m * DIM + b] = blk[a * DIM + b];
  }
}

// bc = P^T r ; optionally the first (zero-start) Jacobi sweep of the coarse level:
// xc = w * dinvc .* bc  (fused so the coarse level starts with one kernel fewer)
template <int DIM>
__global__ void __launch_bounds__(TPB, 1) k_restrict(Coarsening T, const double* __restrict__ r, double* __restrict__ bc,
                                                  const double* __restrict__ dinvc, const double* __restrict__ wp,
                                                  double* __restrict__ xc) {
  TMG_PDL_ENTRY;
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  const int J = blockIdx.y * blockDim.y + threadIdx.y;
  const int K = blockIdx.z * blockDim.z + threadIdx.z;
  if (!(I < T.C.nn[0] && J < T.C.nn[1] && K < T.C.nn[2])) return;
  const int node = T.C.id(I, J, K);
  // fixed 3^DIM gather (invalid candidates clamped, weight 0): every load is
  // issued at once instead of one data-dependent loop trip at a time; the
  // valid terms are summed in the same order, and the zero-weight ones add
  // exact zeros, so the result is bit-identical
  int ix[3], iy[3], iz[3];
  double wx[3], wy[3], wz[3];
  fine_of_coarse3(I, T.co[0], T.F.nn[0], ix, wx);
  fine_of_coarse3(J, T.co[1], T.F.nn[1], iy, wy);
  if (DIM == 3) fine_of_coarse3(K, T.co[2], T.F.nn[2], iz, wz);
  else { iz[0] = iz[1] = iz[2] = 0; wz[0] = 1.0; wz[1] = wz[2] = 0.0; }
  double acc[DIM];
#pragma unroll
  for (int c = 0; c < DIM; ++c) acc[c] = 0.0;
#pragma unroll
  for (int c2 = 0; c2 < (DIM == 3 ? 3 : 1); ++c2)
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double ww = wx[a] * wy[b] * wz[c2];
        double v[DIM];
        load_node<DIM>(r, T.F.id(ix[a], iy[b], iz[c2]), v);
#pragma unroll
        for (int c = 0; c < DIM; ++c) acc[c] += ww * v[c];
      }
  store_node<DIM>(bc, node, acc);
  if (xc) {
    const double w = *wp;
    double d[DIM];
    load_node<DIM>(dinvc, node, d);
#pragma unroll
    for (int c = 0; c < DIM; ++c) d[c] = w * d[c] * acc[c];
    store_node<DIM>(xc, node, d);
  }
}

// x += P e
template <int DIM>
__global__ void __launch_bounds__(TPB, 1) k_prolong_add(Coarsening T, const double* __restrict__ e, double* __restrict__ x) {
  TMG_PDL_ENTRY;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  const int k = blockIdx.z * blockDim.z + threadIdx.z;
  if (!(i < T.F.nn[0] && j < T.F.nn[1] && k < T.F.nn[2])) return;
  const int node = T.F.id(i, j, k);
  double pe[DIM], xv[DIM];
  prolong_at<DIM>(T, e, i, j, k, pe);
  load_node<DIM>(x, node, xv);
#pragma unroll
  for (int c = 0; c < DIM; ++c) xv[c] += pe[c];
  store_node<DIM>(x, node, xv);
}

// Galerkin product A_c = P^T A P into stencil storage; one thread per
// (coarse node, stencil slot).  The fine operator is read through its block()
// provider, so level 0 is never assembled.
template <int DIM, class Op>
__global__ void __launch_bounds__(TPB, 1) k_rap(const __grid_constant__ Op op, Coarsening T, double* __restrict__ Ac) {
  TMG_PDL_ENTRY;
  constexpr int DD = DIM * DIM, C0 = StencilOp<DIM>::C0, NH = StencilOp<DIM>::NH;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= T.C.n * NH) return;  // the stored slots of StencilOp
  const int s = C0 + (int)(t / T.C.n);
  const long long node = t - (long long)(s - C0) * T.C.n;
  int I0, I1, I2;
  T.C.ijk(node, I0, I1, I2);
  const int J0 = I0 + Slots<DIM>::dx(s), J1 = I1 + Slots<DIM>::dy(s), J2 = I2 + Slots<DIM>::dz(s);
  double acc[DD];
#pragma unroll
  for (int q = 0; q < DD; ++q) acc[q] = 0.0;
  if (T.C.inside(J0, J1, J2)) {
    int fi[3][3], fj[3][3], ni[3], nj[3];
    double wi[3][3], wj[3][3];
    const int Iv[3] = {I0, I1, I2}, Jv[3] = {J0, J1, J2};
    for (int d = 0; d < 3; ++d) {
      if (d < DIM) {
        ni[d] = fine_of_coarse(Iv[d], T.co[d], T.F.nn[d], fi[d], wi[d]);
        nj[d] = fine_of_coarse(Jv[d], T.co[d], T.F.nn[d], fj[d], wj[d]);
      } else {
        ni[d] = nj[d] = 1; fi[d][0] = fj[d][0] = 0; wi[d][0] = wj[d][0] = 1.0;
      }
    }
    double blk[DD];
    for (int a2 = 0; a2 < ni[2]; ++a2)
      for (int a1 = 0; a1 < ni[1]; ++a1)
        for (int a0 = 0; a0 < ni[0]; ++a0) {
          const double wa = wi[0][a0] * wi[1][a1] * wi[2][a2];
          for (int b2 = 0; b2 < nj[2]; ++b2) {
            if (abs(fj[2][b2] - fi[2][a2]) > 1) continue;
            for (int b1 = 0; b1 < nj[1]; ++b1) {
              if (abs(fj[1][b1] - fi[1][a1]) > 1) continue;
              for (int b0 = 0; b0 < nj[0]; ++b0) {
                if (abs(fj[0][b0] - fi[0][a0]) > 1) continue;
                const double ww = wa * wj[0][b0] * wj[1][b1] * wj[2][b2];
                op.block(fi[0][a0], fi[1][a1], fi[2][a2], fj[0][b0], fj[1][b1], fj[2][b2], blk);
#pragma unroll
                for (int q = 0; q < DD; ++q) acc[q] += ww * blk[q];
              }
            }
          }
        }
  }
#pragma unroll
  for (int q = 0; q < DD; ++q) Ac[((s - C0) * DD + q) * T.C.n + node] = acc[q];
}

}  // namespace tmg
