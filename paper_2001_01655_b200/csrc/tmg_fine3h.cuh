// Hex8 matrix-free operator in the reflection-character (Hadamard) basis,
// element-centric, streamed along z.  The default 3D level-0 path
// (FineOp<3>::STREAM): every kernel that applies K(rho) on a 3D level 0
// (k_apply, k_residual, k_jacobi, k_cheb, k_cg_pq, k_apply_sym, k_bjacobi)
// calls fine3_rows(op, src, ein, epi).
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
// Mapping (warp-specialised, one CTA per SM): 8 consumer warps form a
// TX x TY = 32 x 8 column of threads over an x-y node patch that overlaps its
// neighbours by one node; thread (tx,ty) owns the element column whose lowest
// corner is node (i0+tx, j0+ty) and walks a z chunk, one element layer per
// step.  A 9th, producer warp streams the node planes ahead of them with TMA
// bulk copies (cp.async.bulk, completion on mbarriers): per plane the source
// vectors and free-dof masks of the (TX+1) x (TY+1) window (a 3-deep ring it
// finishes -- src(raw), e.g. D^-1 r + beta p -- into a 5-deep ring of staged
// planes), the element moduli of the layer below and the epilogue's input
// vectors at the output nodes.  Consumers never touch global memory on the
// way in: they wait on the plane's mbarrier, read corners from shared memory,
// and release the slot on a second mbarrier when its last use is done.
// Contributions reach the neighbouring node columns through warp shuffles (x:
// a warp is one row of 32 columns) and a double-buffered shared row (y, one
// named barrier per step among the consumers).  Nodes with tx, ty >= 1 are
// complete and handed to the epilogue: epi(node, i, j, k, out, self, e), out =
// row of Z K Z + I_fixed applied to the source, self = the (unmasked) source
// value, e[v][c] = the staged epilogue inputs (EpiIn) at the node.
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
constexpr int NC = NT;               // consumer threads (8 warps)
#ifndef TMG_F3H_NSR
#define TMG_F3H_NSR 3
#endif
#define TMG_F3H_NSR_MAXP TMG_F3H_NSR
#ifndef TMG_F3H_NPROD
#define TMG_F3H_NPROD 3  // producer warps (planes dealt round-robin; 3: config-4 PCG iteration -2.5 % vs 1)
#endif
constexpr int NPROD = TMG_F3H_NPROD;
constexpr int NTH = NT + 32 * NPROD;  // + the producer warp(s)
static_assert(NPROD >= 1 && NPROD <= TMG_F3H_NSR_MAXP, "at most one producer warp per ring slot");
#ifndef TMG_F3H_NSR
#define TMG_F3H_NSR 3
#endif
constexpr int NSR = TMG_F3H_NSR;     // raw plane ring (TMA destination)
constexpr int NU = 4;                // finished plane ring (written 2 steps ahead, read 2 steps behind)
constexpr int NVS = 3, NVE = 2;      // max source / epilogue vectors
constexpr int ROWD = 104;            // doubles per staged row buffer (33 nodes x 3 + alignment shift, 16-B multiple)
constexpr int MROW = 64;             // bytes per staged mask row (33 + shift)
constexpr int U_PLANE = 3 * NS;      // doubles per finished plane (component-major)
constexpr int X_PLANE = 3 * NC;      // per consumer thread: contributions to the node one row up
constexpr int NFIN = (NS + NC - 1) / NC;  // staged nodes each consumer finishes per plane
// shared-memory layout (bytes; every region 128-B aligned for the bulk copies)
constexpr size_t al128(size_t b) { return (b + 127) / 128 * 128; }
constexpr size_t OFF_BAR = 0;  // 2 NSR mbarriers
constexpr size_t OFF_SRAW = 128;
constexpr size_t OFF_MRAW = al128(OFF_SRAW + sizeof(double) * NSR * NVS * SY * ROWD);
constexpr size_t OFF_U = al128(OFF_MRAW + (size_t)NSR * SY * MROW);
constexpr size_t OFF_S = al128(OFF_U + sizeof(double) * NU * U_PLANE);
constexpr size_t OFF_M = al128(OFF_S + sizeof(double) * NU * U_PLANE);
constexpr size_t OFF_X = al128(OFF_M + (size_t)NU * NS);
constexpr size_t SMEM_BYTES = OFF_X + sizeof(double) * 2 * X_PLANE;
static_assert(SMEM_BYTES <= 227 * 1024 - 2048, "f3h shared memory (+ the kernels' static reductions)");
static_assert(ROWD * 8 % 16 == 0 && MROW % 16 == 0, "16-B aligned rows");

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
#define TMG_F3H_OCC 1  // CTAs per SM the z-chunking is sized for (185 KB shared memory each)
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

// ---------------------------------------------------------------------------
// TMA bulk copies and mbarriers (PTX)
// ---------------------------------------------------------------------------
namespace f3h {
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned tx) {
  asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P;\n"
      "F3H_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra F3H_WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
#ifndef TMG_F3H_POLL_NS
#define TMG_F3H_POLL_NS 200
#endif
// (producer side: the slot frees up about once per layer -- back off between polls
// instead of competing with the consumer warps for issue slots)
__device__ __forceinline__ void mbar_wait_backoff(unsigned long long* b, unsigned parity) {
  unsigned done = 0;
  while (true) {
    asm volatile(
        "{\n .reg .pred P;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n"
        " selp.u32 %0, 1, 0, P;\n}"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    if (done) break;
    __nanosleep(TMG_F3H_POLL_NS);
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// A staged row: `cnt` items of `isz` bytes at g (inside [lo, hi)) go to a 16-B
// aligned shared buffer at byte offset (g & 15), so the bulk copy moves the
// 16-B aligned window around them.  Windows that would reach outside [lo, hi)
// rounded inward (only the first/last row of a vector can) are copied by the
// producer warp with plain loads instead (same layout).
struct Row {
  const char* a0;   // aligned window start
  unsigned bytes;   // window size (multiple of 16), 0 = nothing to stage
  int shift;        // byte offset of the first item in the window
  bool tma;
};
__device__ __forceinline__ Row row_window(const void* g, int cnt, int isz, const void* lo, const void* hi) {
  Row r;
  const unsigned long long A = (unsigned long long)g, a0 = A & ~15ull;
  const unsigned long long e = (A + (unsigned long long)cnt * isz + 15ull) & ~15ull;
  r.a0 = (const char*)a0;
  r.bytes = cnt > 0 ? (unsigned)(e - a0) : 0u;
  r.shift = (int)(A - a0);
  const unsigned long long l = ((unsigned long long)lo + 15ull) & ~15ull, h = (unsigned long long)hi & ~15ull;
  r.tma = cnt > 0 && a0 >= l && e <= h;
  return r;
}
// item offset (in items of isz bytes) of g inside its staged row buffer
__device__ __forceinline__ int row_shift(const void* g, int isz) { return (int)((unsigned long long)g & 15ull) / isz; }

struct EpiIn {
  const double* v[NVE];  // epilogue input vectors (3 doubles per node); nullptr = not used
};
}  // namespace f3h
template <int DIM>
struct FineOp;
namespace f3h {
// The producer warp (32 lanes): streams the raw planes z0-1 .. z0-1+R of the
// (TX+1) x (TY+1) node window into the NSR-deep ring with TMA bulk copies
// (rows whose 16-B aligned window would leave the vector: plain loads).
template <class Src>
__device__ __forceinline__ void produce(const FineOp<3>& op, const Src& src, double* SR, unsigned char* MR,
                                        unsigned long long* raw_full, unsigned long long* raw_free, int lane, int z0,
                                        int R, int j0, int nlo, int ncnt, int r0 = 0, int rstep = 1) {
  const int nn0 = op.L.nn[0], nn1 = op.L.nn[1], nn2 = op.L.nn[2];
  const long long plane = (long long)nn0 * nn1;
  const long long ndof = 3 * op.L.n;
  constexpr int NTASK = NVS * SY + SY;  // source rows, mask rows
  for (int r = r0; r <= R; r += rstep) {
    const int p = z0 - 1 + r, s3 = r % NSR;
    if (r >= NSR) {
      if (lane == 0) mbar_wait_backoff(raw_free + s3, (unsigned)((r / NSR) - 1) & 1u);
      __syncwarp();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const bool pin = p >= 0 && p < nn2;
    Row rw[2];
    void* dst[2];
    const char* gend[2];
    int isz[2];
    unsigned tx = 0;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int q = lane + 32 * u;
      rw[u].bytes = 0;
      rw[u].tma = false;
      dst[u] = nullptr;
      gend[u] = nullptr;
      isz[u] = 8;
      if (q >= NTASK || !pin) continue;
      if (q < NVS * SY) {
        const int v = q / SY, row = q % SY, gj = j0 + row;
        const double* vp = v < Src::NV ? src.vec(v) : nullptr;
        if (!vp || gj < 0 || gj >= nn1) continue;
        rw[u] = row_window(vp + 3 * (p * plane + (long long)gj * nn0 + nlo), 3 * ncnt, 8, vp, vp + ndof);
        dst[u] = SR + ((s3 * NVS + v) * SY + row) * ROWD;
        gend[u] = (const char*)(vp + ndof);
      } else {
        const int row = q - NVS * SY, gj = j0 + row;
        if (gj < 0 || gj >= nn1) continue;
        rw[u] = row_window(op.mask + p * plane + (long long)gj * nn0 + nlo, ncnt, 1, op.mask, op.mask + op.L.n);
        dst[u] = MR + (s3 * SY + row) * MROW;
        gend[u] = (const char*)(op.mask + op.L.n);
        isz[u] = 1;
      }
      if (rw[u].tma) tx += rw[u].bytes;
    }
    tx = __reduce_add_sync(0xffffffffu, tx);
    if (lane == 0) mbar_expect_tx(raw_full + s3, tx);  // the arrival follows the plain-copy rows
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (rw[u].tma) bulk_g2s(dst[u], rw[u].a0, rw[u].bytes, raw_full + s3);
    // rows whose aligned window would leave the vector (its first / last
    // row): the warp copies the items with plain loads into the same layout,
    // published by the warp's arrival below (release)
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      unsigned need = __ballot_sync(0xffffffffu, rw[u].bytes > 0 && !rw[u].tma);
      while (need) {
        const int l = __ffs(need) - 1;
        need &= need - 1;
        const char* g = (const char*)__shfl_sync(0xffffffffu, (unsigned long long)rw[u].a0, l);
        const int shift = __shfl_sync(0xffffffffu, rw[u].shift, l);
        const unsigned bytes = __shfl_sync(0xffffffffu, rw[u].bytes, l);
        const char* ge = (const char*)__shfl_sync(0xffffffffu, (unsigned long long)gend[u], l);
        const int sz = __shfl_sync(0xffffffffu, isz[u], l);
        unsigned char* d = (unsigned char*)__shfl_sync(0xffffffffu, (unsigned long long)dst[u], l);
        for (int b = shift + lane * sz; b < (int)bytes && g + b < ge; b += 32 * sz) {
          if (sz == 1) d[b] = *(const unsigned char*)(g + b);
          else *reinterpret_cast<double*>(d + b) = *reinterpret_cast<const double*>(g + b);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(raw_full + s3);
  }
}
}  // namespace f3h

template <class Src, class Epi>
__device__ __forceinline__ void fine3h_rows(const FineOp<3>& op, const Src& src, const f3h::EpiIn& ein, Epi&& epi) {
  using namespace f3h;
  static_assert(Src::NV <= NVS, "source vectors");
  extern __shared__ __align__(128) unsigned char f3h_raw[];
  unsigned long long* raw_full = reinterpret_cast<unsigned long long*>(f3h_raw + OFF_BAR);  // [NSR] bytes landed
  unsigned long long* raw_free = raw_full + NSR;                                          // [NSR] finished
  double* SR = reinterpret_cast<double*>(f3h_raw + OFF_SRAW);  // [NSR][NVS][SY][ROWD] raw source rows
  unsigned char* MR = f3h_raw + OFF_MRAW;                      // [NSR][SY][MROW] raw mask rows
  double* U = reinterpret_cast<double*>(f3h_raw + OFF_U);      // [NU][3][NS] finished source, masked (Z u)
  double* S = reinterpret_cast<double*>(f3h_raw + OFF_S);      // [NU][3][NS] finished source, unmasked (self)
  unsigned char* M = f3h_raw + OFF_M;                          // [NU][NS] free-dof masks
  double* X = reinterpret_cast<double*>(f3h_raw + OFF_X);      // [2][3][NC] row-up contributions
  const int t = threadIdx.x;
  const int nn0 = op.L.nn[0], nn1 = op.L.nn[1], nn2 = op.L.nn[2];
  const int ne0 = op.ne[0], ne1 = op.ne[1], ne2 = op.ne[2];
  const long long plane = (long long)nn0 * nn1, eplane = (long long)ne0 * ne1;
  const int i0 = (int)blockIdx.x * (TX - 1) - 1, j0 = (int)blockIdx.y * (TY - 1) - 1;
  const int zc = (nn2 + gridDim.z - 1) / gridDim.z;
  const int z0 = (int)blockIdx.z * zc, z1 = min(nn2, z0 + zc);
  if (z0 >= z1) return;  // (whole CTA)
  const int R = z1 - z0 + 1;  // staged planes z0-1 .. z1 -> r = 0 .. R
  const int nlo = max(i0, 0), ncnt = min(i0 + SX, nn0) - nlo;  // staged node range of a row
  if (t == 0) {
    for (int b = 0; b < NSR; ++b) {
      mbar_init(raw_full + b, 1);  // the producer's arm (+ TMA bytes)
      mbar_init(raw_free + b, NC / 32);  // one arrival per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long ndof = 3 * op.L.n;

  if (t >= NC) {
    produce<Src>(op, src, SR, MR, raw_full, raw_free, (t - NC) & 31, z0, R, j0, nlo, ncnt, (t - NC) >> 5, NPROD);
  } else {
    // ===================== consumer warps =====================
    const int tx = t % TX, ty = t / TX;
    const int gi = i0 + tx, gj = j0 + ty;
    const bool el_ok = gi >= 0 && gi < ne0 && gj >= 0 && gj < ne1;
    const bool out_ok = tx >= 1 && ty >= 1 && gi < nn0 && gj < nn1;
    const int own_st = tx + SX * ty;
    const long long own_node2d = gi + (long long)nn0 * gj;
    const long long own_el2d = el_ok ? gi + (long long)ne0 * gj : 0;
    // the staged nodes this thread finishes: shared-memory offsets and the
    // parity / 16-B phase of their rows' global addresses (plane term added per plane)
    const int pl_par = (int)(plane & 1), pl_m16 = (int)(plane & 15);
    int fin_st[NFIN], fin_off[NFIN], fin_mrow[NFIN], fin_par[NFIN][NVS], fin_m16[NFIN];
    bool fin_in[NFIN];
#pragma unroll
    for (int u = 0; u < NFIN; ++u) {
      const int st = t + u * NC;
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
    // finish staged plane r (= z0 - 1 + r) into U/M slot r % NU: src(raw), masks
    auto finish = [&](int r) {
      const int p = z0 - 1 + r, s3 = r % NSR, su = r % NU;
      mbar_wait(raw_full + s3, (unsigned)(r / NSR) & 1u);
      const bool pin = p >= 0 && p < nn2;
      const int ppar = p & pl_par, pm16 = (p * pl_m16) & 15;
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
    // epilogue inputs of the own node of plane pk, and the element modulus of
    // layer k: loaded one step before their use (register prefetch)
    auto load_epi = [&](int pk, double (*e)[3]) {
      const bool ok = out_ok && pk >= z0 && pk < z1;
      const long long node = own_node2d + plane * pk;
#pragma unroll
      for (int v = 0; v < NVE; ++v)
#pragma unroll
        for (int c = 0; c < 3; ++c) e[v][c] = (ok && ein.v[v]) ? __ldg(ein.v[v] + 3 * node + c) : 0.0;
    };
    auto load_E = [&](int k) {
      return (el_ok && k >= 0 && k < ne2 && k < z1) ? __ldg(op.E + k * eplane + own_el2d) : 0.0;
    };
    // top face of the element column in plane p (slot su): masked corners, x-y transform
    auto face = [&](int su, double (*F)[3]) {
      const double* Ub = U + su * U_PLANE + own_st;
      constexpr int off[4] = {0, 1, SX, SX + 1};
      double v[4][3];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) v[a][c] = Ub[c * NS + off[a]];
      // F[qx + 2 qy] = sum over corners (x, y) of (-1)^(qx x + qy y) v[x + 2y]
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
    double epre[NVE][3], W0[3] = {0.0, 0.0, 0.0};
    // plane k-1 complete: own + left column (W0) + the row below (X); epilogue
    auto output = [&](int k) {
      const int pk = k - 1;
      if (!(pk >= z0 && pk < z1 && out_ok)) return;
      const int su = (pk - z0 + 1) % NU;
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
      epi((int)(own_node2d + plane * pk), gi, gj, pk, out, self, epre);
    };
    // one element layer k with bottom face Fb, top face Ft (computed here), the
    // bottom-plane accumulators G (previous layer's top part; completed here)
    // and the next top part T (produced here).  Called with the arrays'
    // roles alternating (2-step unrolled loop: no register copies).
    auto layer = [&](int k, double Ek, const double (*Fb)[3], double (*Ft)[3], double (*G)[3], double (*T)[3]) {
      face((k + 2 - z0) % NU, Ft);  // plane k+1
      bool tset[4][3] = {};  // (compile-time after unrolling: first contribution to T[q][c] assigns)
      // one character block at a time: member (s = q + 4 qz, c) has
      // u^ = E (Fb[q] +- Ft[q]); its output y^ joins the bottom plane (+) and
      // the top plane (+-)
#pragma unroll
      for (int chi = 0; chi < 8; ++chi) {
        double uh[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const int m = blk_member(chi, j), sj = m / 3, cj = m % 3, q = sj & 3;
          uh[j] = (sj & 4) ? Fb[q][cj] - Ft[q][cj] : Fb[q][cj] + Ft[q][cj];
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
          // the element modulus scales the unit-modulus product on the way out
          // (one FMA per target instead of a multiply per input and an add per target)
          G[q][ci] = fma(Ek, y, G[q][ci]);  // bottom corners (z = 0): plane k
          if (tset[q][ci]) T[q][ci] = fma((si & 4) ? -Ek : Ek, y, T[q][ci]);
          else T[q][ci] = ((si & 4) ? -Ek : Ek) * y;
          tset[q][ci] = true;
        }
      }
      // x-y inverse of plane k's character sums -> corner (x, y) contributions
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
      // x neighbours are lanes of the same warp: the left column's (1,0)
      // corner joins the own node, its (1,1) corner the node one row up (read
      // by the row above after the next consumer barrier)
      double* Xw = X + (k & 1) * X_PLANE + t;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        W0[c] = Wc[0][c] + __shfl_up_sync(0xffffffffu, Wc[1][c], 1);
        Xw[c * NC] = Wc[2][c] + __shfl_up_sync(0xffffffffu, Wc[3][c], 1);
      }
    };
    // step k: [barrier] output plane k-1, prefetch, finish plane k+2, layer k
    double F0[4][3], F1[4][3], G0[4][3], G1[4][3];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int c = 0; c < 3; ++c) G0[q][c] = 0.0;
    finish(0);  // plane z0-1
    double Enext = load_E(z0 - 1), Enext2 = load_E(z0);  // moduli two layers ahead of their use
    // step z0-2: only the bottom face of layer z0-1 (plane z0-1) and plane z0 finished
    asm volatile("bar.sync 1, %0;" ::"n"(NC) : "memory");
    finish(1);
    face(0, F0);
    int k = z0 - 1;
    for (; k + 1 < z1; k += 2) {
      asm volatile("bar.sync 1, %0;" ::"n"(NC) : "memory");  // U of plane k+1 and X of step k-1 complete
      output(k);
      double Ek = Enext;
      Enext = Enext2;
      Enext2 = load_E(k + 2);
      load_epi(k, epre);
      if (k + 3 - z0 <= R) finish(k + 3 - z0);  // plane k+2
      layer(k, Ek, F0, F1, G0, G1);
      asm volatile("bar.sync 1, %0;" ::"n"(NC) : "memory");
      output(k + 1);
      Ek = Enext;
      Enext = Enext2;
      Enext2 = load_E(k + 3);
      load_epi(k + 1, epre);
      if (k + 4 - z0 <= R) finish(k + 4 - z0);  // plane k+3
      layer(k + 1, Ek, F1, F0, G1, G0);
    }
    if (k < z1) {  // odd number of layers: the last one
      asm volatile("bar.sync 1, %0;" ::"n"(NC) : "memory");
      output(k);
      const double Ek = Enext;
      load_epi(k, epre);
      if (k + 3 - z0 <= R) finish(k + 3 - z0);
      layer(k, Ek, F0, F1, G0, G1);
      ++k;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(NC) : "memory");
    output(k);  // plane z1-1
  }
  __syncthreads();  // (the kernels' reductions follow with every thread)
}

}  // namespace tmg
