// Block-sparse (BSR) operators for the algebraic levels of the hierarchy:
// SA-AMG coarse operators (nvec x nvec blocks), prolongations P (bs x nvec) and
// restrictions P^T (nvec x bs).  Column indices are sorted within each block row
// (the reference's scipy CSR matrices are canonical, multigrid.py:262), blocks are
// row-major.  Row kernels give each block row a group of 2^gshift lanes; the R
// outputs of a row stay in registers.
#pragma once
#include <algorithm>

#include "tmg_ops.cuh"

#ifndef TMG_BSR_MINB
#define TMG_BSR_MINB 4  // min CTAs per SM of the square BSR row kernels (64 registers; measured 1/4/6/8)
#endif
#ifndef TMG_BSR_XFER_MINB
// min CTAs per SM of the transfer kernels (P, P^T): 6 for the 2D level-0 2x3 /
// 3x2 blocks (config 2 AMG iteration 660 -> 642 us), 4 otherwise (the 3x3 and
// the 3D 3x6 / 6x6 transfers are slower at 6)
#define TMG_BSR_XFER_MINB ((R * C == 6) ? 6 : 4)
#endif

namespace tmg {

struct Bsr {
  int nrows = 0, ncols = 0;  // block rows / block columns
  int R = 1, C = 1;          // block shape
  long long nnzb = 0;
  DevBuf<int> rowptr, col;
  DevBuf<double> val;
  // 3x3 blocks padded to 10 doubles (16-byte aligned, 128-bit loads) for the
  // V-cycle row kernels; made once the hierarchy is built (pad_blocks)
  DevBuf<double> vpad;
  long long scalar_nnz() const { return nnzb * R * C; }
};

template <int R, int C>
struct BsrView {
  const int* __restrict__ rowptr;
  const int* __restrict__ col;
  const double* __restrict__ val;
  int nrows;
  int gshift;  // 2^gshift lanes cooperate on one block row (row kernels below)
  const double* __restrict__ vpad;  // R*C odd: padded copy (stride R*C+1) or nullptr
};
// Lanes per block row: the largest power of two <= half the mean blocks per row
// (<= 32).  The coarse Galerkin levels carry 15-60 blocks per row, where one
// thread per row is a serial latency chain; the fine-level P (3 blocks per row)
// keeps 1-2 lanes.  Runtime value: the xor-butterfly below never leaves its
// aligned group, so no template instantiation per group size is needed.
inline int bsr_gshift(int nrows, long long nnzb) {
  const double avg = nrows > 0 ? double(nnzb) / nrows : 1.0;
  int g = 0;
  while (g < 5 && double(2 << g) <= avg) ++g;
  return g;
}
template <int R, int C>
inline BsrView<R, C> view(const Bsr& m) {
  return BsrView<R, C>{m.rowptr.get(), m.col.get(), m.val.get(), m.nrows, bsr_gshift(m.nrows, m.nnzb), m.vpad.get()};
}
// grid of a row kernel on m (threads = rows << gshift)
inline unsigned bsr_grid(const Bsr& m) {
  const long long t = (long long)m.nrows << bsr_gshift(m.nrows, m.nnzb);
  return (unsigned)std::max<long long>(1, (t + TPB - 1) / TPB);
}

// Row handled by this thread's lane group, and the lane within the group.
template <int R, int C>
__device__ __forceinline__ int bsr_row_id(const BsrView<R, C>& A, int& lane) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  lane = (int)(t & ((1 << A.gshift) - 1));
  return (int)(t >> A.gshift);
}

// y_row = sum_j A_rj x_j (row of R outputs), lanes of a group stride over the
// row's blocks and combine with an xor butterfly: every lane of the group ends
// with the full sums.  Must be reached by all lanes of the warp (rows past the
// end contribute zeros).
template <int R, int C>
__device__ __forceinline__ void bsr_row(const BsrView<R, C>& A, int row, int lane, const double* __restrict__ x,
                                        double out[R]) {
#pragma unroll
  for (int a = 0; a < R; ++a) out[a] = 0.0;
  if (row < A.nrows) {
    const int e = A.rowptr[row + 1];
    for (int p = A.rowptr[row] + lane; p < e; p += (1 << A.gshift)) {
      const int j = A.col[p];
      double xv[C];
#pragma unroll
      for (int b = 0; b < C; ++b) {
        if constexpr (C % 2 == 0) {  // 16-byte aligned node values
          if (b % 2 == 0) {
            const double2 t2 = __ldg(reinterpret_cast<const double2*>(x + (long long)j * C + b));
            xv[b] = t2.x;
            xv[b + 1] = t2.y;
          }
        } else {
          xv[b] = __ldg(x + (long long)j * C + b);
        }
      }
      const double* blk = A.val + (long long)p * R * C;
      if constexpr ((R * C) % 2 == 0) {  // 16-byte aligned blocks: 128-bit loads
        double bv[R * C];
#pragma unroll
        for (int q = 0; q < R * C / 2; ++q) {
          const double2 t2 = __ldg(reinterpret_cast<const double2*>(blk) + q);
          bv[2 * q] = t2.x;
          bv[2 * q + 1] = t2.y;
        }
#pragma unroll
        for (int a = 0; a < R; ++a)
#pragma unroll
          for (int b = 0; b < C; ++b) out[a] += bv[a * C + b] * xv[b];
      } else if (A.vpad) {  // padded odd blocks: stride R*C+1 doubles, 16-byte aligned
        constexpr int S2 = (R * C + 1) / 2;
        double bv[2 * S2];
        const double2* b2 = reinterpret_cast<const double2*>(A.vpad + (long long)p * (R * C + 1));
#pragma unroll
        for (int q = 0; q < S2; ++q) {
          const double2 t2 = __ldg(b2 + q);
          bv[2 * q] = t2.x;
          bv[2 * q + 1] = t2.y;
        }
#pragma unroll
        for (int a = 0; a < R; ++a)
#pragma unroll
          for (int b = 0; b < C; ++b) out[a] += bv[a * C + b] * xv[b];
      } else {
#pragma unroll
        for (int a = 0; a < R; ++a)
#pragma unroll
          for (int b = 0; b < C; ++b) out[a] += __ldg(blk + a * C + b) * xv[b];
      }
    }
  }
  for (int off = (1 << A.gshift) >> 1; off > 0; off >>= 1)
#pragma unroll
    for (int a = 0; a < R; ++a) out[a] += __shfl_xor_sync(0xffffffffu, out[a], off);
}

// y = A x (+ y if accumulate)
template <int R, int C>
__global__ void __launch_bounds__(TPB, TMG_BSR_XFER_MINB) k_bsr_apply(BsrView<R, C> A, const double* __restrict__ x,
                                                   double* __restrict__ y, int accumulate) {
  TMG_PDL_ENTRY;
  int lane;
  const int row = bsr_row_id(A, lane);
  double out[R];
  bsr_row<R, C>(A, row, lane, x, out);
  if (row >= A.nrows || lane != 0) return;
#pragma unroll
  for (int a = 0; a < R; ++a) {
    const long long i = (long long)row * R + a;
    y[i] = accumulate ? y[i] + out[a] : out[a];
  }
}

// bc = P^T r as a BSR product with the stored transpose; optional fused first
// zero-start Jacobi sweep of the coarse level, xc = w dinvc .* bc
template <int R, int C>
__global__ void __launch_bounds__(TPB, TMG_BSR_XFER_MINB) k_bsr_restrict(BsrView<R, C> Pt, const double* __restrict__ r,
                                                      double* __restrict__ bc, const double* __restrict__ dinvc,
                                                      const double* __restrict__ wp, double* __restrict__ xc) {
  TMG_PDL_ENTRY;
  int lane;
  const int row = bsr_row_id(Pt, lane);
  double out[R];
  bsr_row<R, C>(Pt, row, lane, r, out);
  if (row >= Pt.nrows || lane != 0) return;
  const double w = xc ? *wp : 0.0;
#pragma unroll
  for (int a = 0; a < R; ++a) {
    const long long i = (long long)row * R + a;
    bc[i] = out[a];
    if (xc) xc[i] = w * dinvc[i] * out[a];
  }
}

// r = b - A x
template <int R>
__global__ void __launch_bounds__(TPB, TMG_BSR_MINB) k_bsr_residual(BsrView<R, R> A, const double* __restrict__ x,
                                                      const double* __restrict__ b, double* __restrict__ r) {
  TMG_PDL_ENTRY;
  int lane;
  const int row = bsr_row_id(A, lane);
  double out[R];
  bsr_row<R, R>(A, row, lane, x, out);
  if (row >= A.nrows || lane != 0) return;
#pragma unroll
  for (int a = 0; a < R; ++a) {
    const long long i = (long long)row * R + a;
    r[i] = b[i] - out[a];
  }
}

// xo = x + w D^-1 (b - A x); DOT: reduce xo.b
template <int R, bool DOT>
__global__ void __launch_bounds__(TPB, TMG_BSR_MINB) k_bsr_jacobi(BsrView<R, R> A, const double* __restrict__ x,
                                                    const double* __restrict__ b, const double* __restrict__ dinv,
                                                    const double* __restrict__ wp, double* __restrict__ xo, Red red) {
  TMG_PDL_ENTRY;
  int lane;
  const int row = bsr_row_id(A, lane);
  double out[R];
  bsr_row<R, R>(A, row, lane, x, out);
  double v = 0.0;
  if (row < A.nrows && lane == 0) {
    const double w = *wp;
#pragma unroll
    for (int a = 0; a < R; ++a) {
      const long long i = (long long)row * R + a;
      const double xn = x[i] + w * (dinv[i] * (b[i] - out[a]));
      xo[i] = xn;
      if (DOT) v += xn * b[i];
    }
  }
  if (DOT) grid_reduce(v, red);
}

// One Chebyshev step on a BSR level: p' = D^-1 r + beta p; x += alpha p'; r' = r - alpha A p'
// (p' of neighbours is needed, so p' is produced by k_bsr_cheb_p first).
__global__ void k_bsr_cheb_p(const double* __restrict__ r, const double* __restrict__ p,
                             const double* __restrict__ dinv, const double* __restrict__ coef, int step,
                             double* __restrict__ po, long long n) {
  TMG_PDL_ENTRY;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double beta = step == 0 ? 0.0 : coef[2 * step + 1];
  const double z = dinv ? dinv[i] * r[i] : r[i];  // dinv == nullptr: r holds the SOR solve z
  po[i] = beta == 0.0 ? z : z + beta * p[i];
}
// The last step of a Chebyshev pass whose residual r' nobody reads: only
// x += alpha p' with p' = D^-1 r + beta p remains -- a vector update, no
// operator application (any level storage; same arithmetic as the full step).
// bdot != nullptr: also reduce sum(x' . bdot) into red (the PCG r.z when this is
// the last kernel of the level-0 V-cycle; grid <= the reduction's partial slots).
__global__ void k_cheb_x_only(const double* __restrict__ r, const double* __restrict__ p,
                              const double* __restrict__ dinv, const double* __restrict__ coef, int step, int x_zero,
                              double* __restrict__ x, long long n, const double* __restrict__ bdot, Red red) {
  TMG_PDL_ENTRY;
  const double alpha = coef[2 * step], beta = step == 0 ? 0.0 : coef[2 * step + 1];
  const long long stride = (long long)gridDim.x * blockDim.x;
  double v = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    const double z = dinv ? dinv[i] * r[i] : r[i];
    const double pv = beta == 0.0 ? z : z + beta * p[i];
    const double x0 = x_zero ? 0.0 : x[i];
    const double xn = x0 + alpha * pv;
    x[i] = xn;
    if (bdot) v += xn * bdot[i];
  }
  if (bdot) grid_reduce(v, red);
}
template <int R>
__global__ void __launch_bounds__(TPB, TMG_BSR_MINB) k_bsr_cheb(BsrView<R, R> A, const double* __restrict__ r,
                                                  const double* __restrict__ pn, const double* __restrict__ coef,
                                                  int step, int x_zero, double* __restrict__ x,
                                                  double* __restrict__ ro) {
  TMG_PDL_ENTRY;
  int lane;
  const int row = bsr_row_id(A, lane);
  const double alpha = coef[2 * step];
  double out[R];
  bsr_row<R, R>(A, row, lane, pn, out);
  if (row >= A.nrows || lane != 0) return;
#pragma unroll
  for (int a = 0; a < R; ++a) {
    const long long i = (long long)row * R + a;
    x[i] = (x_zero ? 0.0 : x[i]) + alpha * pn[i];
    if (ro) ro[i] = r[i] - alpha * out[a];
  }
}

// y = ds .* A (ds .* v)
template <int R>
__global__ void __launch_bounds__(TPB, TMG_BSR_MINB) k_bsr_apply_sym(BsrView<R, R> A, const double* __restrict__ v,
                                                       const double* __restrict__ ds, double* __restrict__ tmp,
                                                       double* __restrict__ y) {
  TMG_PDL_ENTRY;
  int lane;
  const int row = bsr_row_id(A, lane);
  double out[R];
  bsr_row<R, R>(A, row, lane, tmp, out);
  if (row >= A.nrows || lane != 0) return;
#pragma unroll
  for (int a = 0; a < R; ++a) {
    const long long i = (long long)row * R + a;
    y[i] = ds[i] * out[a];
  }
}
__global__ void k_vmul(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ y, long long n) {
  TMG_PDL_ENTRY;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) y[i] = a[i] * b[i];
}

// scalar diagonal of a square BSR
template <int R>
__global__ void k_bsr_diag(BsrView<R, R> A, double* __restrict__ d, unsigned* __restrict__ bad) {
  TMG_PDL_ENTRY;
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= A.nrows) return;
  double dv[R];
#pragma unroll
  for (int a = 0; a < R; ++a) dv[a] = 0.0;
  for (int p = A.rowptr[row]; p < A.rowptr[row + 1]; ++p)
    if (A.col[p] == row) {
#pragma unroll
      for (int a = 0; a < R; ++a) dv[a] = A.val[(long long)p * R * R + a * R + a];
    }
#pragma unroll
  for (int a = 0; a < R; ++a) {
    d[(long long)row * R + a] = dv[a];
    if (dv[a] == 0.0) atomicOr(bad, 1u);
  }
}

// dense row-major copy of a square BSR (coarsest level)
template <int R>
__global__ void k_bsr_to_dense(BsrView<R, R> A, double* __restrict__ Ad, long long n) {
  TMG_PDL_ENTRY;
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= A.nrows) return;
  for (int p = A.rowptr[row]; p < A.rowptr[row + 1]; ++p) {
    const int j = A.col[p];
    for (int a = 0; a < R; ++a)
      for (int b = 0; b < R; ++b)
        Ad[((long long)row * R + a) * n + (long long)j * R + b] = A.val[(long long)p * R * R + a * R + b];
  }
}

__global__ void k_bsr_pad(const double* __restrict__ val, long long nnzb, int rc, double* __restrict__ vp) {
  TMG_PDL_ENTRY;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= nnzb * (rc + 1)) return;
  const long long p = i / (rc + 1);
  const int q = (int)(i - p * (rc + 1));
  vp[i] = q < rc ? val[p * rc + q] : 0.0;
}
// padded V-cycle copy of an odd-block-size BSR (no-op otherwise)
inline void bsr_pad_blocks(Bsr& m, cudaStream_t s) {
  const int rc = m.R * m.C;
  if (rc % 2 == 0 || m.nnzb == 0 || m.vpad.get()) return;
  m.vpad.alloc(m.nnzb * (rc + 1), s);
  launch(k_bsr_pad, grid_for(m.nnzb * (rc + 1)), TPB, 0, s, (const double*)m.val.get(), m.nnzb, rc, m.vpad.get());
  note_launch();
}

// Dispatch helpers over the block shapes used by SA-AMG (dpn in {2,3}, nvec in {3,6}).
#define TMG_BSR_SQUARE_DISPATCH(Rv, ...)                        \
  switch (Rv) {                                                 \
    case 1: { constexpr int RR = 1; __VA_ARGS__; } break;        \
    case 2: { constexpr int RR = 2; __VA_ARGS__; } break;        \
    case 3: { constexpr int RR = 3; __VA_ARGS__; } break;        \
    case 6: { constexpr int RR = 6; __VA_ARGS__; } break;        \
    default: throw Error(-1, "unsupported BSR block size");     \
  }
#define TMG_BSR_RECT_DISPATCH(Rv, Cv, ...)                                              \
  if (Rv == 2 && Cv == 3) { constexpr int RR = 2, CC = 3; __VA_ARGS__; }                \
  else if (Rv == 3 && Cv == 2) { constexpr int RR = 3, CC = 2; __VA_ARGS__; }           \
  else if (Rv == 3 && Cv == 6) { constexpr int RR = 3, CC = 6; __VA_ARGS__; }           \
  else if (Rv == 6 && Cv == 3) { constexpr int RR = 6, CC = 3; __VA_ARGS__; }           \
  else if (Rv == 3 && Cv == 3) { constexpr int RR = 3, CC = 3; __VA_ARGS__; }           \
  else if (Rv == 6 && Cv == 6) { constexpr int RR = 6, CC = 6; __VA_ARGS__; }           \
  else if (Rv == 2 && Cv == 2) { constexpr int RR = 2, CC = 2; __VA_ARGS__; }           \
  else if (Rv == 1 && Cv == 3) { constexpr int RR = 1, CC = 3; __VA_ARGS__; }           \
  else if (Rv == 3 && Cv == 1) { constexpr int RR = 3, CC = 1; __VA_ARGS__; }           \
  else if (Rv == 1 && Cv == 6) { constexpr int RR = 1, CC = 6; __VA_ARGS__; }           \
  else if (Rv == 6 && Cv == 1) { constexpr int RR = 6, CC = 1; __VA_ARGS__; }           \
  else if (Rv == 1 && Cv == 1) { constexpr int RR = 1, CC = 1; __VA_ARGS__; }           \
  else throw Error(-1, "unsupported BSR block shape");

}  // namespace tmg
