// Right-preconditioned restarted (F)GMRES on the device (reference krylov.py:48
// _gmres_core, the default Krylov method of the reference's SolverHarness).
//
// Vectors live in HBM: the Krylov basis V ((m+1) x n, row per vector) and, for
// the flexible variant, Z (m x n).  Per Arnoldi step the device runs the
// preconditioner (one V-cycle), w = K z, and the orthogonalisation; the host
// receives the new Hessenberg column (j+2 scalars) and applies the Givens
// rotations in the reference's order and arithmetic, so the convergence test
// |g[j+1]| <= tol and the least-squares solve are the reference's own.
//
// Orthogonalisation: classical Gram-Schmidt applied twice (CGS2) instead of the
// reference's modified Gram-Schmidt.  Both produce the same Hessenberg matrix
// in exact arithmetic and CGS2 is at least as stable as MGS; it needs 2 passes
// over V per pass instead of j+1 dependent dot/axpy pairs (2(j+1) kernels),
// which is what makes a 200-vector restart affordable on the device.
#pragma once
#include <cmath>
#include <vector>

#include "tmg_gmg.cuh"
#include "tmg_kern.cuh"

namespace tmg {

constexpr double GMRES_BREAKDOWN_TOL = 1e-14;  // krylov.py:13
constexpr int MDOT_CHUNK = 256 * 8;            // elements per block in the multi-dot

// partials[blk * nv + i] = sum over the block's chunk of V_i . w
__global__ void __launch_bounds__(256) k_mdot(const double* __restrict__ V, long long n, int nv,
                                              const double* __restrict__ w, double* __restrict__ partials) {
  TMG_PDL_ENTRY;
  __shared__ double ws[8];
  const long long base = blockIdx.x * (long long)MDOT_CHUNK;
  double wv[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const long long e = base + threadIdx.x + 256LL * u;
    wv[u] = e < n ? w[e] : 0.0;
  }
  for (int i = 0; i < nv; ++i) {
    const double* v = V + (long long)i * n;
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const long long e = base + threadIdx.x + 256LL * u;
      if (e < n) s += v[e] * wv[u];
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) t += ws[k];
      partials[(long long)blockIdx.x * nv + i] = t;
    }
    __syncthreads();
  }
}

// h[i] = sum_blk partials[blk * nv + i] (fixed order: deterministic); hacc[i] += h[i]
__global__ void __launch_bounds__(256) k_mdot_finish(const double* __restrict__ partials, int nblk, int nv,
                                                     double* __restrict__ h, double* __restrict__ hacc) {
  TMG_PDL_ENTRY;
  const int i = blockIdx.x;
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) s += partials[(long long)b * nv + i];
  s = block_sum(s);
  if (threadIdx.x == 0) {
    h[i] = s;
    if (hacc) hacc[i] += s;
  }
}

// w -= sum_i h[i] V_i
__global__ void k_mv_sub(const double* __restrict__ V, long long n, int nv, const double* __restrict__ h,
                         double* __restrict__ w) {
  TMG_PDL_ENTRY;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= n) return;
  double s = 0.0;
  for (int i = 0; i < nv; ++i) s += h[i] * V[(long long)i * n + e];
  w[e] -= s;
}

// out = sum_i y[i] V_i (+ out if accumulate)
__global__ void k_lincomb(const double* __restrict__ V, long long n, int nv, const double* __restrict__ y,
                          double* __restrict__ out, int accumulate) {
  TMG_PDL_ENTRY;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= n) return;
  double s = 0.0;
  for (int i = 0; i < nv; ++i) s += y[i] * V[(long long)i * n + e];
  out[e] = accumulate ? out[e] + s : s;
}

// y = x * (1 / *nrm)  (the reference divides: V[j+1] = w / H[j+1, j])
__global__ void k_div_by(const double* __restrict__ x, const double* __restrict__ nrm, double* __restrict__ y,
                         long long n) {
  TMG_PDL_ENTRY;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e < n) y[e] = x[e] / *nrm;
}
__global__ void k_axpy_inplace(const double* __restrict__ z, double* __restrict__ x, long long n) {
  TMG_PDL_ENTRY;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e < n) x[e] += z[e];
}
__global__ void k_sqrt_inplace(double* v) {
  TMG_PDL_ENTRY;
  *v = sqrt(*v);
}

struct GmresResult {
  int iterations = 0, converged = 0;
  double ms = 0;
  std::vector<double> hist;
};

template <int DIM>
GmresResult gmres_solve(const Operator& K, Hierarchy* H, const double* b_dev, double* x_dev, bool use_x0,
                        double rtol, int maxit, int restart, bool flexible, cudaStream_t s) {
  TMG_REQUIRE(rtol > 0.0 && rtol < 1.0, "rtol must be in (0, 1)");
  TMG_REQUIRE(restart >= 1, "restart must be >= 1");
  TMG_REQUIRE(maxit >= 0, "max_iterations must be >= 0");
  const long long n = K.ndof;
  const int mcap = std::max(1, std::min(restart, std::max(maxit, 1)));
  const unsigned gv = red_grid(n), ge = grid_for(n);
  const int nblk = (int)((n + MDOT_CHUNK - 1) / MDOT_CHUNK);
  auto op0 = K.template fine<DIM>();
  DevBuf<double> V, Z, w, r, z, t, partials, h, hacc, y, scal;
  V.alloc((size_t)(mcap + 1) * n, s);
  if (flexible) Z.alloc((size_t)mcap * n, s);
  w.alloc(n, s); r.alloc(n, s); z.alloc(n, s); t.alloc(n, s);
  partials.alloc((size_t)nblk * (mcap + 1), s);
  h.alloc(mcap + 1, s); hacc.alloc(mcap + 1, s); y.alloc(mcap + 1, s);
  scal.alloc(4, s);
  RedSlot red;
  red.alloc(gv, s);
  cudaEvent_t e0, e1;
  TMG_CUDA(cudaEventCreate(&e0));
  TMG_CUDA(cudaEventCreate(&e1));
  TMG_CUDA(cudaEventRecord(e0, s));

  auto apply_K = [&](const double* in, double* out) {
    launch(k_apply<DIM, decltype(op0)>, TMG_ROW_OP_LAUNCH_L(K.L, op0), s, op0,
           in, out);
    note_launch();
  };
  auto precond = [&](const double* in, double* out) {
    if (H) {
      vcycle<DIM>(*H, 0, in, out, s);
    } else {
      TMG_CUDA(cudaMemcpyAsync(out, in, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
  };
  auto norm_to = [&](const double* v, double* dst_dev) {  // dst_dev = ||v||
    Red rd = red.red();
    rd.result = dst_dev;
    launch(k_dot, gv, TPB, 0, s, v, v, n, rd);
    launch(k_sqrt_inplace, 1, 1, 0, s, dst_dev);
    note_launch(2);
  };
  auto fetch = [&](const double* dev, double* host, int cnt) {
    TMG_CUDA(cudaMemcpyAsync(host, dev, cnt * sizeof(double), cudaMemcpyDeviceToHost, s));
    TMG_CUDA(cudaStreamSynchronize(s));
  };
  auto residual = [&]() {  // r = b - K x
    launch(k_residual<DIM, decltype(op0)>, TMG_ROW_OP_LAUNCH_L(K.L, op0), s,
           op0, (const double*)x_dev, b_dev, r.get());
    note_launch();
  };

  if (!use_x0) TMG_CUDA(cudaMemsetAsync(x_dev, 0, n * sizeof(double), s));
  residual();
  double sc[2];
  norm_to(r.get(), scal.get());
  norm_to(b_dev, scal.get() + 1);
  fetch(scal.get(), sc, 2);
  GmresResult res;
  res.hist.push_back(sc[0]);
  const double tol = rtol * sc[1];
  if (sc[0] <= tol) {
    res.converged = 1;
  } else {
    int total = 0;
    bool broke_down = false;
    std::vector<double> Hm, cs, sn, g, col, yv;
    double beta = sc[0];
    while (total < maxit && !broke_down) {
      if (beta <= tol) break;
      const int m = std::min(restart, maxit - total);
      Hm.assign((size_t)(m + 1) * m, 0.0);
      cs.assign(m, 0.0);
      sn.assign(m, 0.0);
      g.assign(m + 1, 0.0);
      g[0] = beta;
      // V[0] = r / beta
      TMG_CUDA(cudaMemcpyAsync(scal.get() + 2, &beta, sizeof(double), cudaMemcpyHostToDevice, s));
      launch(k_div_by, ge, TPB, 0, s, (const double*)r.get(), (const double*)(scal.get() + 2), V.get(), n);
      note_launch();
      int j_used = 0;
      for (int j = 0; j < m; ++j) {
        double* Vj = V.get() + (long long)j * n;
        double* zj = flexible ? Z.get() + (long long)j * n : z.get();
        precond(Vj, zj);
        apply_K(zj, w.get());
        // CGS2: h = V^T w ; w -= V h ; twice.  hacc accumulates H[0..j, j].
        TMG_CUDA(cudaMemsetAsync(hacc.get(), 0, (j + 1) * sizeof(double), s));
        for (int pass = 0; pass < 2; ++pass) {
          launch(k_mdot, (unsigned)nblk, 256, 0, s, (const double*)V.get(), n, j + 1, (const double*)w.get(),
                 partials.get());
          launch(k_mdot_finish, (unsigned)(j + 1), 256, 0, s, (const double*)partials.get(), nblk, j + 1, h.get(),
                 hacc.get());
          launch(k_mv_sub, ge, TPB, 0, s, (const double*)V.get(), n, j + 1, (const double*)h.get(), w.get());
          note_launch(3);
        }
        norm_to(w.get(), hacc.get() + j + 1);
        col.resize(j + 2);
        fetch(hacc.get(), col.data(), j + 2);
        for (int i = 0; i <= j + 1; ++i) Hm[(size_t)i * m + j] = col[i];
        const double hjj1 = Hm[(size_t)(j + 1) * m + j];
        const bool breakdown = hjj1 < GMRES_BREAKDOWN_TOL;
        if (!breakdown) {
          launch(k_div_by, ge, TPB, 0, s, (const double*)w.get(), (const double*)(hacc.get() + j + 1),
                 V.get() + (long long)(j + 1) * n, n);
          note_launch();
        }
        // Givens rotations exactly as krylov.py:97-108
        for (int i = 0; i < j; ++i) {
          const double hij = Hm[(size_t)i * m + j], hi1j = Hm[(size_t)(i + 1) * m + j];
          const double tt = cs[i] * hij + sn[i] * hi1j;
          Hm[(size_t)(i + 1) * m + j] = -sn[i] * hij + cs[i] * hi1j;
          Hm[(size_t)i * m + j] = tt;
        }
        const double hjj = Hm[(size_t)j * m + j], hj1 = Hm[(size_t)(j + 1) * m + j];
        const double denom = std::hypot(hjj, hj1);
        cs[j] = denom != 0.0 ? hjj / denom : 1.0;
        sn[j] = denom != 0.0 ? hj1 / denom : 0.0;
        Hm[(size_t)j * m + j] = denom;
        Hm[(size_t)(j + 1) * m + j] = 0.0;
        g[j + 1] = -sn[j] * g[j];
        g[j] = cs[j] * g[j];
        total += 1;
        j_used = j + 1;
        res.hist.push_back(std::fabs(g[j + 1]));
        if (std::fabs(g[j + 1]) <= tol || breakdown || total >= maxit) {
          broke_down = breakdown;
          break;
        }
      }
      if (j_used > 0) {
        // back substitution on triu(H[:j_used, :j_used]) y = g[:j_used]
        yv.assign(j_used, 0.0);
        for (int i = j_used - 1; i >= 0; --i) {
          double acc = g[i];
          for (int k2 = i + 1; k2 < j_used; ++k2) acc -= Hm[(size_t)i * m + k2] * yv[k2];
          yv[i] = acc / Hm[(size_t)i * m + i];
        }
        TMG_CUDA(cudaMemcpyAsync(y.get(), yv.data(), j_used * sizeof(double), cudaMemcpyHostToDevice, s));
        if (flexible) {
          launch(k_lincomb, ge, TPB, 0, s, (const double*)Z.get(), n, j_used, (const double*)y.get(), x_dev, 1);
          note_launch();
        } else {
          launch(k_lincomb, ge, TPB, 0, s, (const double*)V.get(), n, j_used, (const double*)y.get(), t.get(), 0);
          note_launch();
          precond(t.get(), z.get());
          launch(k_axpy_inplace, ge, TPB, 0, s, (const double*)z.get(), x_dev, n);
          note_launch();
        }
      }
      residual();
      norm_to(r.get(), scal.get());
      fetch(scal.get(), sc, 1);
      beta = sc[0];
      res.hist.back() = beta;
      if (beta <= tol) break;
    }
    res.iterations = total;
    residual();
    norm_to(r.get(), scal.get());
    fetch(scal.get(), sc, 1);
    res.converged = sc[0] <= tol;
  }
  TMG_CUDA(cudaEventRecord(e1, s));
  TMG_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  TMG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  res.ms = ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return res;
}

}  // namespace tmg
