// Geometric multigrid hierarchy (reference multigrid.py:200-336) on the device:
// level 0 is the matrix-free FineOp, coarser levels are Galerkin stencils built by
// k_rap, the coarsest is inverted densely.  The V-cycle (multigrid.py:231) is an
// enqueue-only host routine, so it can be captured into a CUDA graph.
//
// Kernel fusion in the weighted-Jacobi V-cycle (same arithmetic as Alg. 1):
//   * the zero-start first pre-sweep x = w D^-1 b of a coarse level is written by
//     the restriction kernel that produces b (k_restrict), and for level 0 by the
//     PCG update kernel that produces r;
//   * the coarse-grid correction x += P e is evaluated on the fly inside the first
//     post-smoothing sweep (k_prolong_jacobi);
//   * the last level-0 sweep also reduces r.z for PCG.
#pragma once
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <memory>

#include "tmg_dense.cuh"
#include "tmg_ke.h"
#include "tmg_ops.cuh"

namespace tmg {

enum SmootherKind { SM_JACOBI = 0, SM_BLOCK_JACOBI = 1, SM_CHEBYSHEV = 2 };

struct SmootherCfg {
  int kind = SM_JACOBI;
  double weight = 0.5;
  int degree = 2;
  int lanczos_steps = 10;
  uint64_t seed = 0;
  double safeguard = 0.0;  // >0: Jacobi weight capped at safeguard / lambda_hat (Lanczos)
};

// ----------------------------------------------------------------------------
// small vector kernels
// ----------------------------------------------------------------------------
// Reduction kernels run on a small grid (RED_BLOCKS) with 4 independent loads in
// flight per thread, so the last-block combine reads few partials.
constexpr unsigned RED_BLOCKS = 296;  // 2 per SM
inline unsigned red_grid(long long n) { return std::min<unsigned>(grid_for(n), RED_BLOCKS); }

__global__ void __launch_bounds__(TPB) k_dot(const double* __restrict__ a, const double* __restrict__ b, long long n,
                                             Red red) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    const double a0 = __ldg(a + i), a1 = __ldg(a + i + stride), a2 = __ldg(a + i + 2 * stride),
                 a3 = __ldg(a + i + 3 * stride);
    const double b0 = __ldg(b + i), b1 = __ldg(b + i + stride), b2 = __ldg(b + i + 2 * stride),
                 b3 = __ldg(b + i + 3 * stride);
    s0 += a0 * b0; s1 += a1 * b1; s2 += a2 * b2; s3 += a3 * b3;
  }
  for (; i < n; i += stride) s0 += a[i] * b[i];
  grid_reduce((s0 + s1) + (s2 + s3), red);
}
__global__ void k_scale_vec(const double* __restrict__ b, const double* __restrict__ d, const double* __restrict__ wp,
                            double* __restrict__ x, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) x[i] = *wp * (d[i] * b[i]);
}
template <int DIM>
__global__ void k_bscale_vec(const double* __restrict__ b, const double* __restrict__ binv, const double* __restrict__ wp,
                             double* __restrict__ x, long long nnodes) {
  const long long node = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (node >= nnodes) return;
  const double w = *wp;
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < DIM; ++c) s += binv[node * DIM * DIM + a * DIM + c] * b[node * DIM + c];
    x[node * DIM + a] = w * s;
  }
}
__global__ void k_recip(const double* __restrict__ d, double* __restrict__ dinv, double* __restrict__ dsq, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  dinv[i] = 1.0 / d[i];
  if (dsq) dsq[i] = sqrt(1.0 / d[i]);
}
// splitmix64 start vector, bit-identical to oracle.splitmix_uniform
__global__ void k_splitmix(double* __restrict__ v, long long n, unsigned long long seed) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long G = 0x9E3779B97F4A7C15ULL;
  unsigned long long z = seed * G + (unsigned long long)(i + 1) * G;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z = z ^ (z >> 31);
  v[i] = (double)(z >> 11) * 0x1.0p-53 * 2.0 - 1.0;
}
__global__ void k_div_sqrt(double* __restrict__ v, const double* __restrict__ s2, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) v[i] = v[i] / sqrt(*s2);
}
// w -= a v + b vprev  (b from beta2 slot j-1 or 0)
__global__ void k_lz_orth(double* __restrict__ w, const double* __restrict__ v, const double* __restrict__ vp,
                          const double* __restrict__ alpha, const double* __restrict__ beta2, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double a = *alpha;
  const double b = beta2 ? sqrt(*beta2) : 0.0;
  w[i] = b != 0.0 ? w[i] - a * v[i] - b * vp[i] : w[i] - a * v[i];
}
__global__ void k_lz_next(double* __restrict__ v, double* __restrict__ vp, const double* __restrict__ w,
                          const double* __restrict__ beta2, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  vp[i] = v[i];
  v[i] = w[i] / sqrt(*beta2);
}
// Largest eigenvalue of the Lanczos tridiagonal by Sturm bisection, then the
// Chebyshev step coefficients on [0.1, 1.1] * lambda (multigrid.py:129-149).
// With wout: the safeguarded Jacobi weight min(w0, sg / lambda) instead.
__global__ void k_lz_finish(const double* __restrict__ alpha, const double* __restrict__ beta2, int steps,
                            int degree, double* __restrict__ coef, double* __restrict__ lmax_out, double w0,
                            double sg, double* __restrict__ wout) {
  int m = steps;
  for (int j = 0; j < steps; ++j)
    if (!(sqrt(beta2[j]) > 1e-300)) { m = j + 1; break; }
  double lo = 1e300, hi = -1e300;
  for (int j = 0; j < m; ++j) {
    const double bl = j > 0 ? sqrt(beta2[j - 1]) : 0.0, br = j < m - 1 ? sqrt(beta2[j]) : 0.0;
    lo = fmin(lo, alpha[j] - bl - br);
    hi = fmax(hi, alpha[j] + bl + br);
  }
  for (int it = 0; it < 200; ++it) {  // count of eigenvalues < x via LDL^T pivots
    const double x = 0.5 * (lo + hi);
    if (x == lo || x == hi) break;
    int cnt = 0;
    double q = 1.0;
    for (int j = 0; j < m; ++j) {
      const double b2 = j > 0 ? beta2[j - 1] : 0.0;
      q = (alpha[j] - x) - (j > 0 ? b2 / q : 0.0);
      if (q == 0.0) q = -1e-300;
      if (q < 0.0) ++cnt;
    }
    if (cnt == m) hi = x; else lo = x;
  }
  const double lam = hi;
  *lmax_out = lam;
  if (wout) *wout = fmin(w0, sg / lam);
  if (!coef) return;
  const double a = 0.1 * lam, b = 1.1 * lam, theta = 0.5 * (b + a), delta = 0.5 * (b - a);
  double al = 0.0, be = 0.0;
  for (int i = 0; i < degree; ++i) {
    if (i == 0) { al = 1.0 / theta; be = 0.0; }
    else { be = (delta * al / 2.0) * (delta * al / 2.0); al = 1.0 / (theta - be / al); }
    coef[2 * i] = al;
    coef[2 * i + 1] = be;
  }
}

// ----------------------------------------------------------------------------
// the stiffness operator K(rho) (mesh.py:327)
// ----------------------------------------------------------------------------
struct Operator {
  int dim = 2;
  Lat L{};
  int ne[3] = {1, 1, 1};
  double h[3] = {1, 1, 1};
  double nu = 0.3;
  long long nelem = 0, ndof = 0;
  DevBuf<double> E, ke;
  DevBuf<uint8_t> mask;
  std::vector<double> ke_host;
  template <int DIM>
  FineOp<DIM> fine() const {
    FineOp<DIM> o;
    o.L = L;
    for (int d = 0; d < 3; ++d) o.ne[d] = ne[d];
    o.E = E.get();
    o.mask = mask.get();
    std::memcpy(o.ke, ke_host.data(), sizeof(o.ke));
    return o;
  }
};

// ----------------------------------------------------------------------------
// levels
// ----------------------------------------------------------------------------
struct Level {
  bool fine = false;  // level operator is the matrix-free FineOp
  Lat L{};
  long long ndof = 0;
  const Operator* op = nullptr;  // for fine levels
  DevBuf<double> A;              // stencil storage (coarse geometric levels)
  DevBuf<double> diag, dinv, dsq, binv;
  DevBuf<double> b, x, xt, r, rt, p, pt;
  Coarsening T{};  // to the next level
  DevBuf<double> coef, lmax;  // Chebyshev
  DevBuf<double> wdev;        // Jacobi weight used by the kernels (safeguarded)
};

struct Hierarchy {
  int dim = 2;
  int n_pre = 1, n_post = 1;
  SmootherCfg sm;
  std::vector<std::unique_ptr<Level>> lv;
  DenseInverse coarse;
  std::vector<int> provenance;
  RedSlot red;  // scratch reduction for setup
  int last() const { return (int)lv.size() - 1; }
  // fused-kernel V-cycle applies (point Jacobi, at least one pre-sweep)
  bool fused() const { return sm.kind == SM_JACOBI && n_pre > 0; }
  // buffer receiving the first Jacobi write of level k when its output is xout
  double* first_dst(int k, double* xout) const {
    const int W = n_pre + n_post;
    return ((W - 1) % 2 == 0) ? xout : lv[k]->xt.get();
  }
};

template <int DIM, class F>
void with_op(const Level& l, F&& f) {
  if (l.fine) {
    f(l.op->template fine<DIM>());
  } else {
    StencilOp<DIM> o;
    o.L = l.L;
    o.A = l.A.get();
    f(o);
  }
}

// launch configuration of a node kernel on level l with operator `o` in scope
#define TMG_NODE_LAUNCH(l) node_grid<DIM>((l).L), node_block<DIM>(), decltype(o)::SMEM_BYTES

template <int DIM>
void level_apply(const Level& l, const double* x, double* y, cudaStream_t s) {
  with_op<DIM>(l, [&](auto o) {
    k_apply<DIM, decltype(o)><<<TMG_NODE_LAUNCH(l), s>>>(o, x, y);
    note_launch();
  });
}

// Lanczos bound + Chebyshev coefficients (or the safeguarded Jacobi weight) for
// a level, device only.
template <int DIM>
void lanczos_setup(Hierarchy& H, Level& l, cudaStream_t s) {
  const int m = H.sm.lanczos_steps;
  DevBuf<double> v, vp, w, alpha, beta2, nrm;
  v.alloc(l.ndof, s); vp.alloc(l.ndof, s); w.alloc(l.ndof, s);
  alpha.alloc(std::max(m, 1), s); beta2.alloc(std::max(m, 1), s); nrm.alloc(1, s);
  alpha.zero(s); beta2.zero(s);
  const bool cheb = H.sm.kind == SM_CHEBYSHEV;
  if (cheb) l.coef.alloc(2 * std::max(H.sm.degree, 1), s);
  l.lmax.alloc(1, s);
  const unsigned g = grid_for(l.ndof);
  const unsigned gr = red_grid(l.ndof);
  k_splitmix<<<g, TPB, 0, s>>>(v.get(), l.ndof, (unsigned long long)H.sm.seed);
  Red rn = H.red.red();
  rn.result = nrm.get();
  k_dot<<<gr, TPB, 0, s>>>(v.get(), v.get(), l.ndof, rn);
  k_div_sqrt<<<g, TPB, 0, s>>>(v.get(), nrm.get(), l.ndof);
  note_launch(3);
  for (int j = 0; j < m; ++j) {
    with_op<DIM>(l, [&](auto o) {
      k_apply_sym<DIM, decltype(o)><<<TMG_NODE_LAUNCH(l), s>>>(o, v.get(), l.dsq.get(), w.get());
    });
    Red ra = H.red.red();
    ra.result = alpha.get() + j;
    k_dot<<<gr, TPB, 0, s>>>(w.get(), v.get(), l.ndof, ra);
    k_lz_orth<<<g, TPB, 0, s>>>(w.get(), v.get(), vp.get(), alpha.get() + j, j > 0 ? beta2.get() + j - 1 : nullptr,
                                l.ndof);
    Red rb = H.red.red();
    rb.result = beta2.get() + j;
    k_dot<<<gr, TPB, 0, s>>>(w.get(), w.get(), l.ndof, rb);
    note_launch(4);
    if (j + 1 < m) {
      k_lz_next<<<g, TPB, 0, s>>>(v.get(), vp.get(), w.get(), beta2.get() + j, l.ndof);
      note_launch();
    }
  }
  k_lz_finish<<<1, 1, 0, s>>>(alpha.get(), beta2.get(), m, H.sm.degree, cheb ? l.coef.get() : nullptr, l.lmax.get(),
                              H.sm.weight, H.sm.safeguard, cheb ? nullptr : l.wdev.get());
  note_launch();
  TMG_CUDA(cudaGetLastError());
}

template <int DIM>
void level_setup(Hierarchy& H, Level& l, bool smoother_needed, cudaStream_t s, DevBuf<unsigned>& bad) {
  const long long nd = l.ndof;
  l.diag.alloc(nd, s);
  l.dinv.alloc(nd, s);
  const bool cheb = H.sm.kind == SM_CHEBYSHEV;
  const bool guard = H.sm.kind == SM_JACOBI && H.sm.safeguard > 0.0;
  if (cheb || guard) l.dsq.alloc(nd, s);
  if (H.sm.kind == SM_BLOCK_JACOBI) l.binv.alloc(nd * DIM, s);
  with_op<DIM>(l, [&](auto o) {
    k_diag<DIM, decltype(o)><<<TMG_NODE_LAUNCH(l), s>>>(o, l.diag.get(), l.binv.get(), bad.get());
  });
  k_recip<<<grid_for(nd), TPB, 0, s>>>(l.diag.get(), l.dinv.get(), (cheb || guard) ? l.dsq.get() : nullptr, nd);
  note_launch(2);
  l.wdev.alloc(1, s);
  TMG_CUDA(cudaMemcpyAsync(l.wdev.get(), &H.sm.weight, sizeof(double), cudaMemcpyHostToDevice, s));
  l.b.alloc(nd, s); l.x.alloc(nd, s); l.xt.alloc(nd, s); l.r.alloc(nd, s);
  if (cheb) { l.rt.alloc(nd, s); l.p.alloc(nd, s); l.pt.alloc(nd, s); }
  if ((cheb || guard) && smoother_needed) lanczos_setup<DIM>(H, l, s);
}

inline int coarsen1(int d) { return std::max(1, (d + 1) / 2); }

// multigrid.py:276 gmg_level_dims (+ optional level cap)
inline std::vector<std::array<int, 3>> gmg_plan(int dim, const int* ne, long long coarse_max_dofs, int max_levels) {
  std::vector<std::array<int, 3>> plan;
  plan.push_back({ne[0], ne[1], dim == 3 ? ne[2] : 0});
  while (true) {
    auto cur = plan.back();
    long long nodes = 1;
    bool all1 = true;
    for (int d = 0; d < dim; ++d) { nodes *= (cur[d] + 1); all1 = all1 && cur[d] <= 1; }
    if (dim * nodes <= coarse_max_dofs || all1) break;
    if (max_levels > 0 && (int)plan.size() >= max_levels) break;
    std::array<int, 3> nx = cur;
    for (int d = 0; d < dim; ++d) nx[d] = coarsen1(cur[d]);
    plan.push_back(nx);
  }
  return plan;
}

template <int DIM>
std::unique_ptr<Hierarchy> build_gmg(const Operator& K, long long coarse_max_dofs, int max_levels,
                                     const SmootherCfg& sm, int n_pre, int n_post, cudaStream_t s) {
  auto H = std::make_unique<Hierarchy>();
  H->dim = DIM;
  H->n_pre = n_pre;
  H->n_post = n_post;
  H->sm = sm;
  H->red.alloc(4096, s);
  DevBuf<unsigned> bad;
  bad.alloc(1, s);
  bad.zero(s);
  auto plan = gmg_plan(DIM, K.ne, coarse_max_dofs, max_levels);
  const int nl = (int)plan.size();
  for (int k = 0; k < nl; ++k) {
    auto l = std::make_unique<Level>();
    const auto& ed = plan[k];
    for (int d = 0; d < 3; ++d) l->L.nn[d] = d < DIM ? ed[d] + 1 : 1;
    l->L.n = (long long)l->L.nn[0] * l->L.nn[1] * l->L.nn[2];
    l->ndof = l->L.n * DIM;
    if (k == 0) {
      l->fine = true;
      l->op = &K;
    } else {
      Level& f = *H->lv[k - 1];
      Coarsening T;
      T.F = f.L;
      T.C = l->L;
      for (int d = 0; d < 3; ++d) T.co[d] = (d < DIM && plan[k - 1][d] > 1) ? 1 : 0;
      f.T = T;
      l->A.alloc((size_t)Slots<DIM>::NS * DIM * DIM * l->L.n, s);
      with_op<DIM>(f, [&](auto o) {
        const long long nt = l->L.n * Slots<DIM>::NS;
        k_rap<DIM, decltype(o)><<<grid_for(nt), TPB, 0, s>>>(o, T, l->A.get());
        note_launch();
      });
      TMG_CUDA(cudaGetLastError());
    }
    H->provenance.push_back(0);
    H->lv.push_back(std::move(l));
  }
  for (int k = 0; k < nl; ++k) level_setup<DIM>(*H, *H->lv[k], k < nl - 1, s, bad);
  // coarsest: dense inverse
  Level& c = *H->lv[nl - 1];
  H->coarse.n = c.ndof;
  H->coarse.A.alloc((size_t)c.ndof * c.ndof, s);
  H->coarse.A.zero(s);
  with_op<DIM>(c, [&](auto o) {
    k_to_dense<DIM, decltype(o)><<<TMG_NODE_LAUNCH(c), s>>>(o, H->coarse.A.get());
    note_launch();
  });
  H->coarse.build(s);
  unsigned hbad = 0, cbad = 0;
  TMG_CUDA(cudaMemcpyAsync(&hbad, bad.get(), sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  TMG_CUDA(cudaMemcpyAsync(&cbad, H->coarse.bad.get(), sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  TMG_CUDA(cudaStreamSynchronize(s));
  if (hbad & 1u) throw Error(-1, "zero diagonal entry; operator not smoothable");
  if ((hbad & 2u) && sm.kind == SM_BLOCK_JACOBI) throw Error(-1, "singular nodal block in block Jacobi smoother");
  if (cbad) throw Error(-5, "coarsest operator is not positive definite");
  return H;
}

// ----------------------------------------------------------------------------
// V-cycle (multigrid.py:231), enqueue only
// ----------------------------------------------------------------------------

// Chebyshev passes on x (in place); x_zero: x holds garbage and means 0.
template <int DIM>
void smooth_cheb(Hierarchy& H, Level& l, const double* b, double* x, bool x_zero, int passes, cudaStream_t s) {
  for (int p = 0; p < passes; ++p) {
    const double* rin;
    if (x_zero) {
      rin = b;
    } else {
      with_op<DIM>(l, [&](auto o) { k_residual<DIM, decltype(o)><<<TMG_NODE_LAUNCH(l), s>>>(o, x, b, l.r.get()); });
      note_launch();
      rin = l.r.get();
    }
    const double* pin = l.p.get();
    double* rbuf[2] = {l.rt.get(), l.r.get()};
    double* pbuf[2] = {l.pt.get(), l.p.get()};
    for (int i = 0; i < H.sm.degree; ++i) {
      double* ro = rbuf[i % 2];
      double* po = pbuf[i % 2];
      if (ro == rin) ro = rbuf[(i + 1) % 2];
      if (po == pin) po = pbuf[(i + 1) % 2];
      with_op<DIM>(l, [&](auto o) {
        k_cheb<DIM, decltype(o)><<<TMG_NODE_LAUNCH(l), s>>>(o, rin, pin, l.dinv.get(), l.coef.get(), i,
                                                             (x_zero && i == 0) ? 1 : 0, x, po, ro);
      });
      note_launch();
      rin = ro;
      pin = po;
    }
    x_zero = false;
  }
}

// One Jacobi (point or block) sweep cur -> dst; cur == nullptr means x = 0.
template <int DIM, bool DOT>
void jacobi_sweep(Hierarchy& H, Level& l, const double* b, const double* cur, double* dst, const Red& red,
                  cudaStream_t s) {
  if (cur == nullptr) {
    if (H.sm.kind == SM_BLOCK_JACOBI)
      k_bscale_vec<DIM><<<grid_for(l.L.n), TPB, 0, s>>>(b, l.binv.get(), l.wdev.get(), dst, l.L.n);
    else
      k_scale_vec<<<grid_for(l.ndof), TPB, 0, s>>>(b, l.dinv.get(), l.wdev.get(), dst, l.ndof);
  } else {
    with_op<DIM>(l, [&](auto o) {
      if (H.sm.kind == SM_BLOCK_JACOBI)
        k_bjacobi<DIM, decltype(o)><<<TMG_NODE_LAUNCH(l), s>>>(o, cur, b, l.binv.get(), l.wdev.get(), dst);
      else
        k_jacobi<DIM, decltype(o), DOT><<<TMG_NODE_LAUNCH(l), s>>>(o, cur, b, l.dinv.get(), l.wdev.get(), dst, red);
    });
  }
  note_launch();
}

// V-cycle on level k: xout = MG(b).  first_done: the first pre-sweep result
// w D^-1 b already sits in H.first_dst(k, xout).  dot (level 0 only): reduce
// xout . b in the last post-sweep.  Returns true if dot was produced.
template <int DIM>
bool vcycle(Hierarchy& H, int k, const double* b, double* xout, cudaStream_t s, bool first_done = false,
            const Red* dot = nullptr) {
  Level& l = *H.lv[k];
  if (k == H.last()) {
    H.coarse.apply(b, xout, s);
    return false;
  }
  Level& c = *H.lv[k + 1];
  const bool cheb = H.sm.kind == SM_CHEBYSHEV;
  const int W = H.n_pre + H.n_post;
  auto buf = [&](int w) { return ((W - w) % 2 == 0) ? xout : l.xt.get(); };
  const Red nored{nullptr, nullptr, nullptr};
  double* xcur = nullptr;
  int widx = 0;
  if (cheb) {
    if (H.n_pre > 0) {
      smooth_cheb<DIM>(H, l, b, xout, true, H.n_pre, s);
      xcur = xout;
    }
  } else {
    for (int p = 0; p < H.n_pre; ++p) {
      double* dst = buf(++widx);
      if (!(p == 0 && first_done)) jacobi_sweep<DIM, false>(H, l, b, xcur, dst, nored, s);
      xcur = dst;
    }
  }
  const double* r = b;
  if (xcur) {
    with_op<DIM>(l, [&](auto o) { k_residual<DIM, decltype(o)><<<TMG_NODE_LAUNCH(l), s>>>(o, xcur, b, l.r.get()); });
    note_launch();
    r = l.r.get();
  }
  const bool cfirst = H.fused() && k + 1 < H.last();
  double* cx_first = cfirst ? H.first_dst(k + 1, c.x.get()) : nullptr;
  k_restrict<DIM><<<node_grid<DIM>(c.L), node_block<DIM>(), 0, s>>>(l.T, r, c.b.get(), c.dinv.get(), c.wdev.get(),
                                                                     cx_first);
  note_launch();
  vcycle<DIM>(H, k + 1, c.b.get(), c.x.get(), s, cfirst, nullptr);
  bool dot_done = false;
  if (!cheb && H.sm.kind == SM_JACOBI && H.n_post > 0) {
    if (!xcur) {  // no pre-smoothing: x = 0 before the correction
      xcur = (buf(1) == xout) ? l.xt.get() : xout;
      TMG_CUDA(cudaMemsetAsync(xcur, 0, l.ndof * sizeof(double), s));
    }
    for (int p = 0; p < H.n_post; ++p) {
      double* dst = buf(++widx);
      const bool last = p == H.n_post - 1 && dot != nullptr;
      with_op<DIM>(l, [&](auto o) {
        if (p == 0) {
          if (last)
            k_prolong_jacobi<DIM, decltype(o), true><<<TMG_NODE_LAUNCH(l), s>>>(
                o, xcur, c.x.get(), l.T, b, l.dinv.get(), l.wdev.get(), dst, *dot);
          else
            k_prolong_jacobi<DIM, decltype(o), false><<<TMG_NODE_LAUNCH(l), s>>>(
                o, xcur, c.x.get(), l.T, b, l.dinv.get(), l.wdev.get(), dst, nored);
        } else {
          if (last)
            k_jacobi<DIM, decltype(o), true><<<TMG_NODE_LAUNCH(l), s>>>(o, xcur, b, l.dinv.get(), l.wdev.get(), dst,
                                                                        *dot);
          else
            k_jacobi<DIM, decltype(o), false><<<TMG_NODE_LAUNCH(l), s>>>(o, xcur, b, l.dinv.get(), l.wdev.get(), dst,
                                                                         nored);
        }
      });
      note_launch();
      xcur = dst;
    }
    dot_done = dot != nullptr;
  } else {
    if (!xcur) {
      xcur = (cheb || H.n_post % 2 == 0) ? xout : l.xt.get();
      TMG_CUDA(cudaMemsetAsync(xcur, 0, l.ndof * sizeof(double), s));
    }
    k_prolong_add<DIM><<<node_grid<DIM>(l.L), node_block<DIM>(), 0, s>>>(l.T, c.x.get(), xcur);
    note_launch();
    if (cheb) {
      smooth_cheb<DIM>(H, l, b, xcur, false, H.n_post, s);
    } else {
      for (int p = 0; p < H.n_post; ++p) {
        double* dst = buf(++widx);
        jacobi_sweep<DIM, false>(H, l, b, xcur, dst, nored, s);
        xcur = dst;
      }
    }
  }
  if (xcur != xout) TMG_CUDA(cudaMemcpyAsync(xout, xcur, l.ndof * sizeof(double), cudaMemcpyDeviceToDevice, s));
  return dot_done;
}

}  // namespace tmg
