// Coarsest-level direct solve (reference: splu of the coarsest operator,
// multigrid.py:256-258): blocked right-looking Cholesky A = L L^T on the FP64
// tensor pipe, then the explicit inverse A^-1 = L^-T L^-1 formed from the factor
// (every V-cycle applies it as one bandwidth-bound GEMV, tmg_dense.cuh).
//
// All the O(n^3) work runs in one DMMA (mma.sync m8n8k4 .f64) tile GEMM,
//   C[i0:i0+64, j0:j0+64] = beta C + alpha op(A) op(B)   (K streamed in 32-chunks),
// used for the panel solve L21 = A21 L11^-T, the trailing update
// A22 -= L21 L21^T (lower tiles only), the block rows of Y = L^-1 and the
// Gram product Y^T Y.  The NB x NB diagonal blocks are factorised and inverted
// in shared memory by one CTA (k_chol_diag).  Flops: n^3/3 (factor) + ~2n^3/3
// (L^-1, dense block rows) + n^3/3 (Y^T Y, lower tiles) vs the n^3 of the
// Gauss-Jordan inverse it replaces (TMG_COARSE=gj keeps that path for A/B).
#pragma once
#include "tmg_common.cuh"

namespace tmg {

constexpr int CH_NB = 64;   // factor block
constexpr int GT_M = 64;    // GEMM output tile (GT_M x GT_M per CTA, 8 warps)
constexpr int GT_K = 32;    // K chunk staged in shared memory

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// C (M x N, row-major ldc) = beta * C + alpha * op(A) op(B) over k in [0, K).
// op(A)[i][k] = TA ? A[k*lda + i] : A[i*lda + k];  op(B)[k][j] = TB ? B[j*ldb + k] : B[k*ldb + j].
// lower: only tiles with tile_i >= tile_j (symmetric outputs / trailing updates).
// kmin: first k of the sum -- 0, or i0 (1) / j0 (2) of the tile when the
// operand below it is known to vanish (triangular factors).
// Fragments (PTX m8n8k4 .f64 row.col): lane l = 4g + t holds A[g][t], B[t][g]
// and C[g][2t..2t+1] of its 8x8 tile; warp w owns a 16 x 32 sub-tile.
// Batched (blockIdx.z = q): operands advance by sA / sB / sC doubles per batch
// entry and entry q has Mq = min(M, Mtot - q * dM) rows (dM = 0: every entry M).
struct GemmBatch {
  long long sA = 0, sB = 0, sC = 0;
  int Mtot = 0, dM = 0;
  int k_is_m = 0;  // 1: the contraction length of entry q is Mq too (A operand Mq x Mq)
};
template <bool TA, bool TB>
__global__ void __launch_bounds__(256) k_dgemm_tile(int M, int N, int K, double alpha, const double* __restrict__ A,
                                                    long long lda, const double* __restrict__ B, long long ldb,
                                                    double beta, double* __restrict__ C, long long ldc, int lower,
                                                    int kmin, GemmBatch bt) {
  TMG_PDL_ENTRY;
  if (lower && blockIdx.y < blockIdx.x) return;
  if (gridDim.z > 1 || bt.dM) {
    const long long q = blockIdx.z;
    A += q * bt.sA;
    B += q * bt.sB;
    C += q * bt.sC;
    if (bt.dM) M = min(M, bt.Mtot - (int)q * bt.dM);
    if (bt.k_is_m) K = M;
    if ((int)(blockIdx.y * GT_M) >= M) return;  // (whole CTA)
  }
  __shared__ double As[GT_K][GT_M + 4];  // As[kk][ii] = op(A)[i0+ii][k0+kk]
  __shared__ double Bs[GT_K][GT_M + 4];  // Bs[kk][jj] = op(B)[k0+kk][j0+jj]
  const int i0 = blockIdx.y * GT_M, j0 = blockIdx.x * GT_M;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int r0 = (warp >> 1) * 16, c0 = (warp & 1) * 32;
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int kstart = kmin == 1 ? (int)(blockIdx.y * GT_M) : (kmin == 2 ? (int)(blockIdx.x * GT_M) : 0);
  for (int k0 = kstart; k0 < K; k0 += GT_K) {
    __syncthreads();
    for (int t = threadIdx.x; t < GT_K * GT_M; t += blockDim.x) {
      // coalesced global reads: the contiguous index runs fastest
      int kk, ii;
      if (TA) { kk = t / GT_M; ii = t % GT_M; } else { ii = t / GT_K; kk = t % GT_K; }
      const int gi = i0 + ii, gk = k0 + kk;
      As[kk][ii] = (gi < M && gk < K) ? (TA ? A[(long long)gk * lda + gi] : A[(long long)gi * lda + gk]) : 0.0;
      int kb, jj;
      if (TB) { jj = t / GT_K; kb = t % GT_K; } else { kb = t / GT_M; jj = t % GT_M; }
      const int gj = j0 + jj, gkb = k0 + kb;
      Bs[kb][jj] = (gj < N && gkb < K) ? (TB ? B[(long long)gj * ldb + gkb] : B[(long long)gkb * ldb + gj]) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < GT_K; c += 4) {
      double av[2], bv[4];
#pragma unroll
      for (int a = 0; a < 2; ++a) av[a] = As[c + tq][r0 + a * 8 + g];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = Bs[c + tq][c0 + b * 8 + g];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma884(acc[a][b], av[a], bv[b]);
    }
  }
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int gi = i0 + r0 + a * 8 + g;
    if (gi >= M) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int gj = j0 + c0 + b * 8 + 2 * tq + e;
        if (gj >= N) continue;
        double* dst = C + (long long)gi * ldc + gj;
        *dst = (beta == 0.0 ? 0.0 : beta * *dst) + alpha * acc[a][b][e];
      }
  }
}

// Diagonal block k0 (kb <= CH_NB): L11 = chol(A11), written back into A's lower
// triangle, and Dinv = L11^-1 (lower) for the panel solve and the inverse.  One
// CTA of 1024 threads (16 per row), ONE barrier per elimination step: step p reads the pivot d = S[p][p] and
// the still unscaled column p, updates the trailing lower triangle with
// S[i][j] -= S[i][p] S[j][p] / d (the scaling by sqrt(d) is applied to all columns
// at the end: L[i][p] = S[i][p] / sqrt(d_p)) and eliminates column p from the
// rows below it in Y (Y starts as the identity and ends as the inverse of the
// unit-lower factor, rescaled at the end as well).
__global__ void __launch_bounds__(1024) k_chol_diag(double* __restrict__ A, long long n, int k0, int kb,
                                                   double* __restrict__ Dinv, unsigned* __restrict__ bad) {
  TMG_PDL_ENTRY;
  extern __shared__ double chol_sm[];  // S[CH_NB][CH_NB + 1], Y[CH_NB][CH_NB + 1]
  double (*S)[CH_NB + 1] = reinterpret_cast<double (*)[CH_NB + 1]>(chol_sm);
  double (*Y)[CH_NB + 1] = reinterpret_cast<double (*)[CH_NB + 1]>(chol_sm + CH_NB * (CH_NB + 1));
  const int t = threadIdx.x;
  for (int q = t; q < kb * kb; q += blockDim.x) {
    const int i = q / kb, j = q % kb;
    S[i][j] = i >= j ? A[(long long)(k0 + i) * n + k0 + j] : 0.0;
    Y[i][j] = i == j ? 1.0 : 0.0;
  }
  // thread -> (row i, column group): 16 threads per row, columns j = g, g + 16, ...
  const int ri = t >> 4, g = t & 15;
  for (int p = 0; p < kb; ++p) {
    __syncthreads();
    const double d = S[p][p];
    if (t == 0 && !(d > 0.0)) atomicOr(bad, 1u);
    if (ri > p && ri < kb) {
      const double m = S[ri][p] / (d > 0.0 ? d : 1.0);  // multiplier of row p for row ri (unit-lower L)
      for (int j = p + 1 + g; j <= ri; j += 16) S[ri][j] -= m * S[j][p];
      // unit-lower inverse: Yrow_ri -= m * Yrow_p (columns <= p are the nonzeros of row p)
      for (int j = g; j <= p; j += 16) Y[ri][j] -= m * Y[p][j];
    }
  }
  __syncthreads();
  // A11 = Lu D Lu^T (Lu unit lower = S[i][j] / S[j][j], D = pivots) -> L = Lu sqrt(D),
  // L^-1 = sqrt(D)^-1 Lu^-1
  for (int q = t; q < kb * kb; q += blockDim.x) {
    const int i = q / kb, j = q % kb;
    const double dj = S[j][j] > 0.0 ? S[j][j] : 1.0, di = S[i][i] > 0.0 ? S[i][i] : 1.0;
    if (i > j) A[(long long)(k0 + i) * n + k0 + j] = S[i][j] / sqrt(dj);
    else if (i == j) A[(long long)(k0 + i) * n + k0 + j] = sqrt(dj);
    Dinv[(long long)i * CH_NB + j] = i >= j ? Y[i][j] / sqrt(di) : 0.0;
  }
}

// Y's diagonal block rows start as the NB x NB inverses (Y_kk = Dinv_k)
__global__ void k_chol_put_diag(double* __restrict__ Yb, long long n, int k0, int kb, const double* __restrict__ Dinv) {
  TMG_PDL_ENTRY;
  for (int q = threadIdx.x + blockIdx.x * blockDim.x; q < kb * kb; q += blockDim.x * gridDim.x) {
    const int i = q / kb, j = q % kb;
    Yb[(long long)(k0 + i) * n + k0 + j] = Dinv[(long long)i * CH_NB + j];
  }
}

// mirror the lower triangle into the upper one (the inverse is symmetric; the
// GEMV apply reads full rows)
__global__ void k_sym_from_lower(double* __restrict__ A, long long n) {
  TMG_PDL_ENTRY;
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= n * n) return;
  const long long i = q / n, j = q % n;
  if (j > i) A[q] = A[j * n + i];
}

// Dense SPD coarse inverse via Cholesky (setup; stream-ordered, no host sync).
// A: the coarse matrix in (row-major n x n), its inverse out; bad |= 1 on a
// non-positive pivot.
inline dim3 gemm_tiles(long long m, long long nn) {
  return dim3((unsigned)((nn + GT_M - 1) / GT_M), (unsigned)((m + GT_M - 1) / GT_M));
}
inline void cholesky_inverse(double* a, long long n, unsigned* bad, cudaStream_t s) {
  const int nb = (int)((n + CH_NB - 1) / CH_NB);
  DevBuf<double> Dinv, Y, P;
  Dinv.alloc((size_t)nb * CH_NB * CH_NB, s);
  Y.alloc((size_t)n * n, s);
  P.alloc((size_t)n * n, s);  // panel scratch (factor), T = L_BA Y_AA (inverse)
  const GemmBatch one{};
  // 1. A = L L^T (L in A's lower triangle); Dinv_k = L_kk^-1
  for (int k = 0; k < nb; ++k) {
    const int k0 = k * CH_NB, kb = (int)std::min<long long>(CH_NB, n - k0), k1 = k0 + kb;
    double* Dk = Dinv.get() + (size_t)k * CH_NB * CH_NB;
    launch(k_chol_diag, 1, 1024, 2 * CH_NB * (CH_NB + 1) * sizeof(double), s, a, n, k0, kb, Dk, bad);
    note_launch();
    const long long m = n - k1;
    if (m <= 0) continue;
    // L21 = A21 L11^-T into the scratch, copied over A21
    launch(k_dgemm_tile<false, true>, gemm_tiles(m, kb), 256, 0, s, (int)m, kb, kb, 1.0,
           (const double*)(a + k1 * n + k0), n, (const double*)Dk, (long long)CH_NB, 0.0, P.get(), (long long)CH_NB, 0, 0,
           one);
    TMG_CUDA(cudaMemcpy2DAsync(a + k1 * n + k0, n * sizeof(double), P.get(), CH_NB * sizeof(double),
                               kb * sizeof(double), m, cudaMemcpyDeviceToDevice, s));
    // A22 -= L21 L21^T (lower tiles)
    launch(k_dgemm_tile<false, true>, gemm_tiles(m, m), 256, 0, s, (int)m, (int)m, kb, -1.0,
           (const double*)(a + k1 * n + k0), n, (const double*)(a + k1 * n + k0), n, 1.0, a + k1 * n + k1, n, 1, 0, one);
    note_launch(2);
  }
  // 2. Y = L^-1 by recursive doubling.  The diagonal NB blocks are Dinv_k; at
  // block size b every pair of adjacent diagonal blocks A = [2qb, 2qb + b),
  // B = [2qb + b, 2qb + 2b) (cut at n) gets its off-diagonal block
  //     Y_BA = - Y_BB (L_BA Y_AA)
  // from two GEMMs batched over the pairs q (blockIdx.z): ~2 log2(n / NB)
  // launches of many tiles instead of 2 n / NB launches of few.
  Y.zero(s);
  for (int i = 0; i < nb; ++i) {
    const int i0 = i * CH_NB, ib = (int)std::min<long long>(CH_NB, n - i0);
    launch(k_chol_put_diag, 16, 256, 0, s, Y.get(), n, i0, ib, (const double*)(Dinv.get() + (size_t)i * CH_NB * CH_NB));
  }
  note_launch(nb);
  for (long long bsz = CH_NB; bsz < n; bsz *= 2) {
    const int pairs = (int)((n - bsz + 2 * bsz - 1) / (2 * bsz));  // pairs whose B block is non-empty
    if (pairs <= 0) break;
    GemmBatch bt;
    bt.sA = bt.sB = bt.sC = 2 * bsz * (n + 1);  // next pair: 2b rows and 2b columns further
    bt.Mtot = (int)(n - bsz);                   // rows below the first A block ...
    bt.dM = (int)(2 * bsz);                     // ... consumed 2b per pair: Mq = min(b, n - b - 2qb)
    dim3 g = gemm_tiles(bsz, bsz);
    g.z = (unsigned)pairs;
    // T_BA = L_BA Y_AA   (Y_AA lower triangular: k from the tile's j0)
    launch(k_dgemm_tile<false, false>, g, 256, 0, s, (int)bsz, (int)bsz, (int)bsz, 1.0, (const double*)(a + bsz * n), n,
           (const double*)Y.get(), n, 0.0, P.get() + bsz * n, n, 0, 2, bt);
    // Y_BA = - Y_BB T_BA   (the contraction runs over the rows of B: Mq of them)
    bt.k_is_m = 1;
    launch(k_dgemm_tile<false, false>, g, 256, 0, s, (int)bsz, (int)bsz, (int)bsz, -1.0,
           (const double*)(Y.get() + bsz * (n + 1)), n, (const double*)(P.get() + bsz * n), n, 0.0, Y.get() + bsz * n, n,
           0, 0, bt);
    note_launch(2);
  }
  // 3. A^-1 = Y^T Y (lower tiles; Y lower triangular: k from the tile's i0), mirrored
  launch(k_dgemm_tile<true, false>, gemm_tiles(n, n), 256, 0, s, (int)n, (int)n, (int)n, 1.0, (const double*)Y.get(),
         n, (const double*)Y.get(), n, 0.0, a, n, 1, 1, one);
  launch(k_sym_from_lower, grid_for(n * n), TPB, 0, s, a, n);
  note_launch(2);
  TMG_CUDA(cudaGetLastError());
}

}  // namespace tmg
