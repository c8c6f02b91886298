// Multigrid hierarchies on the device (reference multigrid.py:200-606):
//   build_gmg     -- level 0 is the matrix-free FineOp, coarser levels are
//                    Galerkin 3^d-point stencils (k_rap), geometric transfers;
//   build_sa_amg  -- smoothed aggregation: sparse P/P^T in BSR, BSR coarse ops;
//   build_hybrid  -- n_geo geometric levels, then SA on the last stencil level.
// The coarsest operator is inverted densely.  The V-cycle (multigrid.py:231) is
// an enqueue-only host routine so it can be captured into a CUDA graph.
//
// Kernel fusion in the weighted-Jacobi V-cycle (same arithmetic as Alg. 1):
//   * the zero-start first pre-sweep x = w D^-1 b of a coarse level is written by
//     the restriction kernel that produces b, and for level 0 by the PCG update
//     kernel that produces r;
//   * on geometric transfers the coarse-grid correction x += P e is evaluated on
//     the fly inside the first post-smoothing sweep (k_prolong_jacobi);
//   * the last level-0 sweep also reduces r.z for PCG.
#pragma once
#include <string>
#include <type_traits>

#include "tmg_amg.cuh"
#include "tmg_kern.cuh"
#include "tmg_sor.cuh"

namespace tmg {

enum OpKind { OP_FINE = 0, OP_STENCIL = 1, OP_BSR = 2 };
enum XferKind { XF_NONE = 0, XF_GEO = 1, XF_SPARSE = 2 };

struct Level {
  int opkind = OP_FINE;
  Lat L{};        // lattice levels
  int bs = 2;     // dofs per node (lattice) / block size (BSR)
  long long ndof = 0;
  const Operator* op = nullptr;  // OP_FINE
  DevBuf<double> A;              // OP_STENCIL storage
  Bsr Ab;                        // OP_BSR operator
  DevBuf<double> diag, dinv, dsq, binv;
  DevBuf<double> b, x, xt, r, rt, p, pt, tmp;
  int xfer = XF_NONE;  // transfer to the next level
  Coarsening T{};
  Bsr P, Pt;
  DevBuf<double> coef, lmax, wdev;
  // smoothed-aggregation provenance (exported for parity tests)
  DevBuf<int> agg, sptr, scol;
  int n_agg = 0, n_dropped = 0;  // n_dropped: unaggregated (-1) nodes
  Bsr Tm;                        // tentative prolongation (BSR)
  DevBuf<double> Tnode;          // its blocks indexed by node (zero when unaggregated)
  DevBuf<double> rho;
  // SOR smoothers (tmg_sor.cuh): BSR form of a lattice level, diagonal-block
  // positions, topological ticket order, ready flags + epoch/ticket counters, and
  // work vectors (z: SOR solve; gm*: SOR-GMRES basis V, Z, w and scalars)
  Bsr Asor;
  DevBuf<int> sor_diag, sor_order, sor_flag, sor_ctl;
  DevBuf<double> z, gmV, gmZ, gmw, gmg;
  bool lattice() const { return opkind != OP_BSR; }
};

struct Hierarchy {
  int dim = 2;
  int n_pre = 1, n_post = 1;
  SmootherCfg sm;
  std::vector<std::unique_ptr<Level>> lv;
  DenseInverse coarse;
  std::vector<int> provenance;  // 0 geometric, 1 algebraic (per level)
  std::vector<std::string> flags;
  bool drop_isolated = false;  // SA: leave strength-isolated nodes unaggregated (extension)
  bool smoother_only = false;  // build_smoother: level 0 and its smoother, nothing else
  RedSlot red;                 // scratch reduction for setup
  int last() const { return (int)lv.size() - 1; }
  // fused-kernel V-cycle applies (point Jacobi, at least one pre-sweep)
  bool fused() const { return sm.kind == SM_JACOBI && n_pre > 0; }
  // buffer receiving the first Jacobi write of level k when its output is xout
  double* first_dst(int k, double* xout) const {
    const int W = n_pre + n_post;
    return ((W - 1) % 2 == 0) ? xout : lv[k]->xt.get();
  }
};

// ----------------------------------------------------------------------------
// operator dispatch
// ----------------------------------------------------------------------------
template <int DIM, class F>
void with_lattice(const Level& l, F&& f) {
  if (l.opkind == OP_FINE) {
    f(l.op->template fine<DIM>());
  } else {
    StencilOp<DIM> o;
    o.L = l.L;
    o.A = l.A.get();
    f(o);
  }
}
template <class F>
void with_bsr(const Level& l, F&& f) {
  TMG_BSR_SQUARE_DISPATCH(l.bs, f(view<RR, RR>(l.Ab), std::integral_constant<int, RR>{}))
}
// lattice level operator -> BSR (its 3^d neighbour blocks)
template <int DIM>
void lattice_to_bsr(const Level& l, Bsr& out, cudaStream_t s) {
  const int n = (int)l.L.n;
  out.nrows = out.ncols = n;
  out.R = out.C = DIM;
  DevBuf<int> cnt;
  cnt.alloc(n + 1, s);
  cnt.zero(s);
  with_lattice<DIM>(l, [&](auto o) {
    k_lattice_bsr_count<DIM, decltype(o)><<<node_grid<DIM>(l.L), node_block<DIM>(), 0, s>>>(o, cnt.get());
  });
  rowptr_from_counts(cnt, out.rowptr, n, s);
  out.nnzb = read_int(out.rowptr.get() + n, s);
  out.col.alloc(out.nnzb, s);
  out.val.alloc(out.nnzb * DIM * DIM, s);
  with_lattice<DIM>(l, [&](auto o) {
    k_lattice_bsr_fill<DIM, decltype(o)><<<node_grid<DIM>(l.L), node_block<DIM>(), 0, s>>>(
        o, out.rowptr.get(), out.col.get(), out.val.get());
  });
  note_launch(2);
  TMG_CUDA(cudaGetLastError());
}

// launch configuration of a node kernel on level l with operator `o` in scope
#define TMG_NODE_LAUNCH(l) node_grid<DIM>((l).L), node_block<DIM>(), decltype(o)::SMEM_BYTES
// row kernels (k_apply, k_residual, k_jacobi, k_bjacobi, k_cheb, k_apply_sym, k_cg_pq):
// geometry of the operator's row path (row_grid / row_block / row_smem)
#define TMG_ROW_OP_LAUNCH(l) TMG_ROW_OP_LAUNCH_L((l).L, o)
#define TMG_ROW_LAUNCH(l) bsr_grid((l).Ab), TPB, 0

template <int DIM>
void lvl_apply(const Level& l, const double* x, double* y, cudaStream_t s) {
  if (l.lattice())
    with_lattice<DIM>(l, [&](auto o) { launch(k_apply<DIM, decltype(o)>, TMG_ROW_OP_LAUNCH(l), s, o, x, y); });
  else
    with_bsr(l, [&](auto A, auto rr) { launch(k_bsr_apply<decltype(rr)::value, decltype(rr)::value>, TMG_ROW_LAUNCH(l), s, A, x, y, 0); });
  note_launch();
}
template <int DIM>
void lvl_residual(const Level& l, const double* x, const double* b, double* r, cudaStream_t s) {
  if (l.lattice())
    with_lattice<DIM>(l, [&](auto o) { launch(k_residual<DIM, decltype(o)>, TMG_ROW_OP_LAUNCH(l), s, o, x, b, r); });
  else
    with_bsr(l, [&](auto A, auto rr) { launch(k_bsr_residual<decltype(rr)::value>, TMG_ROW_LAUNCH(l), s, A, x, b, r); });
  note_launch();
}
// one Jacobi sweep cur -> dst (cur == nullptr: zero start, x = w D^-1 b)
template <int DIM, bool DOT>
void lvl_sweep(const Hierarchy& H, const Level& l, const double* b, const double* cur, double* dst, const Red& red,
               cudaStream_t s) {
  const bool block = H.sm.kind == SM_BLOCK_JACOBI;
  if (block && !l.lattice()) {  // nodal blocks of the SA level (multigrid.py:64 with block_size = nvec)
    with_bsr(l, [&](auto A, auto rr) {
      launch(k_bsr_bjacobi<decltype(rr)::value>, TMG_ROW_LAUNCH(l), s, A, cur, b, l.binv.get(), l.wdev.get(), dst);
    });
    note_launch();
    return;
  }
  if (cur == nullptr && !DOT) {
    if (block)
      launch(k_bscale_vec<DIM>, grid_for(l.L.n), TPB, 0, s, b, l.binv.get(), l.wdev.get(), dst, l.L.n);
    else
      launch(k_scale_vec, grid_for(l.ndof), TPB, 0, s, b, l.dinv.get(), l.wdev.get(), dst, l.ndof);
  } else if (l.lattice()) {
    with_lattice<DIM>(l, [&](auto o) {
      if (block)
        launch(k_bjacobi<DIM, decltype(o)>, TMG_ROW_OP_LAUNCH(l), s, o, cur, b, l.binv.get(), l.wdev.get(), dst);
      else
        launch(k_jacobi<DIM, decltype(o), DOT>, TMG_ROW_OP_LAUNCH(l), s, o, cur, b, l.dinv.get(), l.wdev.get(), dst, red);
    });
  } else {
    with_bsr(l, [&](auto A, auto rr) {
      launch(k_bsr_jacobi<decltype(rr)::value, DOT>, TMG_ROW_LAUNCH(l), s, A, cur, b, l.dinv.get(), l.wdev.get(), dst, red);
    });
  }
  note_launch();
}
template <int DIM>
void lvl_cheb_step(const Level& l, const double* rin, const double* zs, const double* dv, const double* pin, int i,
                   bool x_zero, double* x, double* po, double* ro, cudaStream_t s, bool store_p = true) {
  if (l.lattice()) {
    // !store_p / ro == nullptr: p' / r' not stored (the last step of a pass;
    // r' is kept when the V-cycle reads it as its pre-smoothing residual).
    // Lattice rows form p' of their neighbours on the fly; the BSR path below
    // materialises p' (po) first.
    with_lattice<DIM>(l, [&](auto o) {
      launch(k_cheb<DIM, decltype(o)>, TMG_ROW_OP_LAUNCH(l), s, o, rin, zs, pin, dv, l.coef.get(), i, x_zero ? 1 : 0, x,
             store_p ? po : nullptr, ro);
    });
    note_launch();
  } else {
    launch(k_bsr_cheb_p, grid_for(l.ndof), TPB, 0, s, zs, pin, dv, l.coef.get(), i, po, l.ndof);
    with_bsr(l, [&](auto A, auto rr) {
      launch(k_bsr_cheb<decltype(rr)::value>, TMG_ROW_LAUNCH(l), s, A, rin, po, l.coef.get(), i, x_zero ? 1 : 0, x, ro);
    });
    note_launch(2);
  }
}
template <int DIM>
void lvl_apply_sym(Level& l, const double* v, double* y, cudaStream_t s) {
  if (l.lattice()) {
    with_lattice<DIM>(l, [&](auto o) { launch(k_apply_sym<DIM, decltype(o)>, TMG_ROW_OP_LAUNCH(l), s, o, v, l.dsq.get(), y); });
    note_launch();
  } else {
    launch(k_vmul, grid_for(l.ndof), TPB, 0, s, v, l.dsq.get(), l.tmp.get(), l.ndof);
    with_bsr(l, [&](auto A, auto rr) {
      launch(k_bsr_apply_sym<decltype(rr)::value>, TMG_ROW_LAUNCH(l), s, A, v, l.dsq.get(), l.tmp.get(), y);
    });
    note_launch(2);
  }
}

// ----------------------------------------------------------------------------
// SOR smoothers (multigrid.py:97-176): setup and the enqueue-only solve
// ----------------------------------------------------------------------------
inline const Bsr& sor_matrix(const Level& l) { return l.lattice() ? l.Asor : l.Ab; }

inline void dot_to(const Hierarchy& H, const double* a, const double* b, long long n, double* out, cudaStream_t s) {
  Red r = H.red.red();
  r.result = out;
  launch(k_dot, red_grid(n), TPB, 0, s, a, b, n, r);
  note_launch();
}

// Ticket order of the sync-free solve: block rows sorted by level set (length of
// the longest chain of strictly-lower blocks ending at the row), row order inside
// a set.  Computed on the host from the block pattern, once per level.
inline void sor_order(const Bsr& A, DevBuf<int>& order, cudaStream_t s) {
  const int n = A.nrows;
  std::vector<int> rp(n + 1), col(std::max<long long>(A.nnzb, 1));
  TMG_CUDA(cudaMemcpyAsync(rp.data(), A.rowptr.get(), (n + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
  TMG_CUDA(cudaMemcpyAsync(col.data(), A.col.get(), A.nnzb * sizeof(int), cudaMemcpyDeviceToHost, s));
  TMG_CUDA(cudaStreamSynchronize(s));
  std::vector<int> depth(n);
  int maxd = 0;
  for (int i = 0; i < n; ++i) {
    int d = 0;
    for (int p = rp[i]; p < rp[i + 1]; ++p)
      if (col[p] < i) d = std::max(d, depth[col[p]] + 1);
    depth[i] = d;
    maxd = std::max(maxd, d);
  }
  std::vector<int> start(maxd + 2, 0), ord(n);
  for (int i = 0; i < n; ++i) ++start[depth[i] + 1];
  for (int d = 0; d <= maxd; ++d) start[d + 1] += start[d];
  for (int i = 0; i < n; ++i) ord[start[depth[i]]++] = i;
  order.alloc(n, s);
  TMG_CUDA(cudaMemcpyAsync(order.get(), ord.data(), n * sizeof(int), cudaMemcpyHostToDevice, s));
  TMG_CUDA(cudaStreamSynchronize(s));
}

template <int DIM>
void sor_setup(Level& l, cudaStream_t s, DevBuf<unsigned>& bad) {
  if (l.lattice()) lattice_to_bsr<DIM>(l, l.Asor, s);
  const Bsr& A = sor_matrix(l);
  l.sor_diag.alloc(A.nrows, s);
  TMG_BSR_SQUARE_DISPATCH(A.R, launch(k_sor_diagpos<RR>, grid_for(A.nrows), TPB, 0, s, view<RR, RR>(A),
                                      l.sor_diag.get(), bad.get()))
  note_launch();
  sor_order(A, l.sor_order, s);
  l.sor_flag.alloc(A.nrows, s);
  l.sor_flag.zero(s);
  l.sor_ctl.alloc(2, s);
  l.sor_ctl.zero(s);
  l.z.alloc(l.ndof, s);
}

// z = tril(A)^-1 v  (multigrid.py:105 spsolve_triangular), two launches
inline void sor_solve(const Level& l, const double* v, double* z, cudaStream_t s) {
  const Bsr& A = sor_matrix(l);
  launch(k_sor_prep, 1, 1, 0, s, l.sor_ctl.get());
  static const int sleep_ns = [] {
    const char* e = std::getenv("TMG_SOR_SLEEP");
    return e ? std::max(0, std::atoi(e)) : 64;
  }();
  static const int acquire = [] {
    const char* e = std::getenv("TMG_SOR_ACQUIRE");
    return e ? std::atoi(e) : 1;
  }();
  const SorView S{A.rowptr.get(), A.col.get(), A.val.get(), l.sor_diag.get(), l.sor_order.get(), A.nrows,
                  l.sor_flag.get(), l.sor_ctl.get(), sleep_ns, acquire};
  // Only a few level sets' worth of rows can be ready at a time; more resident
  // warps only add flag polls to the L2 (TMG_SOR_CTAS overrides, A/B)
  static const int ctas = [] {
    const char* e = std::getenv("TMG_SOR_CTAS");
    return e ? std::max(1, std::atoi(e)) : 148 * 2;
  }();
  const unsigned grid = (unsigned)std::min<long long>(((long long)A.nrows * 32 + SOR_TPB - 1) / SOR_TPB, ctas);
  TMG_BSR_SQUARE_DISPATCH(A.R, launch(k_sor_solve<RR>, grid, SOR_TPB, 0, s, S, v, z))
  note_launch(2);
}

// lambda of tril(A)^-1 A by 10 power steps (multigrid.py:116-128) and the
// Chebyshev coefficients on [0.1, 1.1] * lambda
template <int DIM>
void sor_cheb_setup(Hierarchy& H, Level& l, cudaStream_t s) {
  TMG_REQUIRE(H.sm.power_start != nullptr, "sor_chebyshev needs the power-method start vector");
  const long long nd = l.ndof;
  DevBuf<double> v, t, nrm;
  v.alloc(nd, s); t.alloc(nd, s); nrm.alloc(1, s);
  TMG_CUDA(cudaMemcpyAsync(v.get(), H.sm.power_start, nd * sizeof(double), cudaMemcpyDeviceToDevice, s));
  l.coef.alloc(2 * std::max(H.sm.degree, 1), s);
  l.lmax.alloc(1, s);
  for (int it = 0; it < 10; ++it) {
    dot_to(H, v.get(), v.get(), nd, nrm.get(), s);
    launch(k_div_sqrt, grid_for(nd), TPB, 0, s, v.get(), nrm.get(), nd);
    note_launch();
    lvl_apply<DIM>(l, v.get(), t.get(), s);
    sor_solve(l, t.get(), v.get(), s);
  }
  dot_to(H, v.get(), v.get(), nd, nrm.get(), s);
  launch(k_sor_cheb_coef, 1, 1, 0, s, nrm.get(), H.sm.degree, l.coef.get(), l.lmax.get());
  note_launch();
  TMG_CUDA(cudaGetLastError());
}

template <int DIM>
void sor_gmres_setup(Hierarchy& H, Level& l, cudaStream_t s) {
  const GmLayout G{H.sm.degree};
  l.gmV.alloc((size_t)G.M * l.ndof, s);
  l.gmZ.alloc((size_t)G.M * l.ndof, s);
  l.gmw.alloc(l.ndof, s);
  l.gmg.alloc(G.size(), s);
  l.gmg.zero(s);
}

// `passes` SOR-GMRES passes on x (in place; x_zero: x holds garbage and means 0)
template <int DIM>
void smooth_sor_gmres(Hierarchy& H, Level& l, const double* b, double* x, bool x_zero, int passes, cudaStream_t s) {
  const GmLayout G{H.sm.degree};
  const long long n = l.ndof;
  double* g = l.gmg.get();
  double* V = l.gmV.get();
  double* Z = l.gmZ.get();
  double* w = l.gmw.get();
  const unsigned gv = grid_for(n);
  for (int pass = 0; pass < passes; ++pass) {
    const double* r = b;
    if (!x_zero) {
      lvl_residual<DIM>(l, x, b, l.r.get(), s);
      r = l.r.get();
    }
    dot_to(H, b, b, n, g + G.bb(), s);
    dot_to(H, r, r, n, g + G.rr(), s);
    launch(k_gm_init, 1, 1, 0, s, g, G);
    launch(k_gm_start, gv, TPB, 0, s, r, V, g, G, n);
    note_launch(2);
    for (int j = 0; j < G.M; ++j) {
      double* vj = V + (size_t)j * n;
      double* zj = Z + (size_t)j * n;
      sor_solve(l, vj, zj, s);
      lvl_apply<DIM>(l, zj, w, s);
      for (int i = 0; i <= j; ++i) {  // modified Gram-Schmidt (krylov.py:98-100)
        dot_to(H, V + (size_t)i * n, w, n, g + G.H(i, j), s);
        launch(k_gm_axpy, gv, TPB, 0, s, w, V + (size_t)i * n, g, G.H(i, j), n);
        note_launch();
      }
      dot_to(H, w, w, n, g + G.hn2(), s);
      launch(k_gm_rot, 1, 1, 0, s, g, G, j);
      note_launch();
      if (j + 1 < G.M) {
        launch(k_gm_next, gv, TPB, 0, s, w, V + (size_t)(j + 1) * n, g, G, n);
        note_launch();
      }
    }
    launch(k_gm_solve, 1, 1, 0, s, g, G);
    launch(k_gm_update, gv, TPB, 0, s, x, x_zero ? 1 : 0, Z, n, g, G, n);
    note_launch(2);
    x_zero = false;
  }
}

// ----------------------------------------------------------------------------
// smoother setup
// ----------------------------------------------------------------------------
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
  launch(k_splitmix, g, TPB, 0, s, v.get(), l.ndof, (unsigned long long)H.sm.seed);
  Red rn = H.red.red();
  rn.result = nrm.get();
  launch(k_dot, gr, TPB, 0, s, v.get(), v.get(), l.ndof, rn);
  launch(k_div_sqrt, g, TPB, 0, s, v.get(), nrm.get(), l.ndof);
  note_launch(3);
  for (int j = 0; j < m; ++j) {
    lvl_apply_sym<DIM>(l, v.get(), w.get(), s);
    Red ra = H.red.red();
    ra.result = alpha.get() + j;
    launch(k_dot, gr, TPB, 0, s, w.get(), v.get(), l.ndof, ra);
    launch(k_lz_orth, g, TPB, 0, s, w.get(), v.get(), vp.get(), alpha.get() + j, j > 0 ? beta2.get() + j - 1 : nullptr,
                                l.ndof);
    Red rb = H.red.red();
    rb.result = beta2.get() + j;
    launch(k_dot, gr, TPB, 0, s, w.get(), w.get(), l.ndof, rb);
    note_launch(3);
    if (j + 1 < m) {
      launch(k_lz_next, g, TPB, 0, s, v.get(), vp.get(), w.get(), beta2.get() + j, l.ndof);
      note_launch();
    }
  }
  launch(k_lz_finish, 1, 1, 0, s, alpha.get(), beta2.get(), m, H.sm.degree, cheb ? l.coef.get() : nullptr, l.lmax.get(),
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
  if (H.sm.kind == SM_BLOCK_JACOBI) {
    if (l.lattice()) {
      l.binv.alloc(nd * DIM, s);
    } else if (smoother_needed) {  // nvec x nvec nodal blocks of an SA level
      l.binv.alloc(nd * l.Ab.R, s);
      with_bsr(l, [&](auto A, auto rr) {
        launch(k_bsr_block_inv<decltype(rr)::value>, grid_for(l.Ab.nrows), TPB, 0, s, A, l.binv.get(), bad.get());
      });
      note_launch();
    }
  }
  if (l.lattice())
    with_lattice<DIM>(l, [&](auto o) {
      launch(k_diag<DIM, decltype(o)>, TMG_NODE_LAUNCH(l), s, o, l.diag.get(), l.binv.get(), bad.get());
    });
  else
    with_bsr(l, [&](auto A, auto rr) {
      launch(k_bsr_diag<decltype(rr)::value>, TMG_ROW_LAUNCH(l), s, A, l.diag.get(), bad.get());
    });
  launch(k_recip, grid_for(nd), TPB, 0, s, l.diag.get(), l.dinv.get(), (cheb || guard) ? l.dsq.get() : nullptr, nd);
  note_launch(2);
  l.wdev.alloc(1, s);
  TMG_CUDA(cudaMemcpyAsync(l.wdev.get(), &H.sm.weight, sizeof(double), cudaMemcpyHostToDevice, s));
  l.b.alloc(nd, s); l.x.alloc(nd, s); l.xt.alloc(nd, s); l.r.alloc(nd, s);
  if (cheb_kind(H.sm.kind)) { l.rt.alloc(nd, s); l.p.alloc(nd, s); l.pt.alloc(nd, s); }
  if (!l.lattice()) l.tmp.alloc(nd, s);
  if ((cheb || guard) && smoother_needed) lanczos_setup<DIM>(H, l, s);
  if (sor_kind(H.sm.kind) && smoother_needed) {
    sor_setup<DIM>(l, s, bad);
    if (H.sm.kind == SM_SOR_CHEBYSHEV) sor_cheb_setup<DIM>(H, l, s);
    else sor_gmres_setup<DIM>(H, l, s);
  }
}

template <int DIM>
void coarse_setup(Hierarchy& H, cudaStream_t s) {
  Level& c = *H.lv.back();
  H.coarse.n = c.ndof;
  H.coarse.A.alloc((size_t)c.ndof * c.ndof, s);
  H.coarse.A.zero(s);
  if (c.lattice())
    with_lattice<DIM>(c, [&](auto o) { launch(k_to_dense<DIM, decltype(o)>, TMG_NODE_LAUNCH(c), s, o, H.coarse.A.get()); });
  else
    with_bsr(c, [&](auto A, auto rr) {
      launch(k_bsr_to_dense<decltype(rr)::value>, TMG_ROW_LAUNCH(c), s, A, H.coarse.A.get(), c.ndof);
    });
  note_launch();
  H.coarse.build(s);
}

// padded copies of the odd-block algebraic operators for the V-cycle row kernels
// (after every setup kernel that indexes the unpadded values); TMG_BSR_PAD=0: off
inline void pad_cycle_operators(Hierarchy& H, cudaStream_t s) {
  const char* e = std::getenv("TMG_BSR_PAD");
  if (e && e[0] == '0') return;
  for (auto& lp : H.lv) {
    if (!lp->lattice()) bsr_pad_blocks(lp->Ab, s);
    if (lp->xfer == XF_SPARSE) {  // 3x3 transfers between algebraic levels
      bsr_pad_blocks(lp->P, s);
      bsr_pad_blocks(lp->Pt, s);
    }
  }
}

inline void finalize_checks(Hierarchy& H, DevBuf<unsigned>& bad, cudaStream_t s) {
  pad_cycle_operators(H, s);
  unsigned hbad = 0, cbad = 0;
  TMG_CUDA(cudaMemcpyAsync(&hbad, bad.get(), sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  TMG_CUDA(cudaMemcpyAsync(&cbad, H.coarse.bad.get(), sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  TMG_CUDA(cudaStreamSynchronize(s));
  if ((hbad & 5u) && sor_kind(H.sm.kind)) throw Error(-1, "zero diagonal; SOR sweep undefined");
  if (hbad & 1u) throw Error(-1, "zero diagonal entry; operator not smoothable");
  if ((hbad & 2u) && H.sm.kind == SM_BLOCK_JACOBI) throw Error(-1, "singular nodal block in block Jacobi smoother");
  if (cbad) throw Error(-5, "coarsest operator is not positive definite");
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
std::unique_ptr<Hierarchy> new_hierarchy(const SmootherCfg& sm, int n_pre, int n_post, cudaStream_t s) {
  auto H = std::make_unique<Hierarchy>();
  H->dim = DIM;
  H->n_pre = n_pre;
  H->n_post = n_post;
  H->sm = sm;
  H->red.alloc(4096, s);
  return H;
}

template <int DIM>
std::unique_ptr<Level> fine_level(const Operator& K) {
  auto l = std::make_unique<Level>();
  l->opkind = OP_FINE;
  l->op = &K;
  l->L = K.L;
  l->bs = DIM;
  l->ndof = K.ndof;
  return l;
}

// append geometric coarse levels for the element dims plan[1..] (multigrid.py:326-332)
template <int DIM>
void add_geometric_levels(Hierarchy& H, const std::vector<std::array<int, 3>>& plan, cudaStream_t s) {
  for (size_t k = 1; k < plan.size(); ++k) {
    auto l = std::make_unique<Level>();
    const auto& ed = plan[k];
    for (int d = 0; d < 3; ++d) l->L.nn[d] = d < DIM ? ed[d] + 1 : 1;
    l->L.n = (long long)l->L.nn[0] * l->L.nn[1] * l->L.nn[2];
    l->ndof = l->L.n * DIM;
    l->bs = DIM;
    l->opkind = OP_STENCIL;
    Level& f = *H.lv.back();
    Coarsening T;
    T.F = f.L;
    T.C = l->L;
    for (int d = 0; d < 3; ++d) T.co[d] = (d < DIM && plan[k - 1][d] > 1) ? 1 : 0;
    f.T = T;
    f.xfer = XF_GEO;
    H.provenance.back() = 0;
    l->A.alloc((size_t)StencilOp<DIM>::NH * DIM * DIM * l->L.n, s);
    with_lattice<DIM>(f, [&](auto o) {
      const long long nt = l->L.n * StencilOp<DIM>::NH;
      launch(k_rap<DIM, decltype(o)>, grid_for(nt), TPB, 0, s, o, T, l->A.get());
      note_launch();
    });
    TMG_CUDA(cudaGetLastError());
    H.lv.push_back(std::move(l));
    H.provenance.push_back(0);
  }
}

template <int DIM>
std::unique_ptr<Hierarchy> build_gmg(const Operator& K, long long coarse_max_dofs, int max_levels,
                                     const SmootherCfg& sm, int n_pre, int n_post, cudaStream_t s) {
  auto H = new_hierarchy<DIM>(sm, n_pre, n_post, s);
  DevBuf<unsigned> bad;
  bad.alloc(1, s);
  bad.zero(s);
  PhaseLog log(s);
  auto plan = gmg_plan(DIM, K.ne, coarse_max_dofs, max_levels);
  H->lv.push_back(fine_level<DIM>(K));
  H->provenance.push_back(0);
  add_geometric_levels<DIM>(*H, plan, s);
  log.mark("gmg: Galerkin stencils");
  const int nl = (int)H->lv.size();
  for (int k = 0; k < nl; ++k) level_setup<DIM>(*H, *H->lv[k], k < nl - 1, s, bad);
  log.mark("gmg: smoother setup");
  coarse_setup<DIM>(*H, s);
  log.mark("gmg: coarse inverse (n)", H->coarse.n);
  finalize_checks(*H, bad, s);
  return H;
}

// make_smoother(config, K) (multigrid.py:179): a one-level "hierarchy" that
// only carries the finest level's smoother (no coarse operator, no V-cycle)
template <int DIM>
std::unique_ptr<Hierarchy> build_smoother(const Operator& K, const SmootherCfg& sm, cudaStream_t s) {
  auto H = new_hierarchy<DIM>(sm, 0, 0, s);
  DevBuf<unsigned> bad;
  bad.alloc(1, s);
  bad.zero(s);
  H->lv.push_back(fine_level<DIM>(K));
  H->provenance.push_back(0);
  level_setup<DIM>(*H, *H->lv[0], true, s, bad);
  unsigned hbad = 0;
  TMG_CUDA(cudaMemcpyAsync(&hbad, bad.get(), sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  TMG_CUDA(cudaStreamSynchronize(s));
  if ((hbad & 5u) && sor_kind(sm.kind)) throw Error(-1, "zero diagonal; SOR sweep undefined");
  if (hbad & 1u) throw Error(-1, "zero diagonal entry; operator not smoothable");
  if ((hbad & 2u) && sm.kind == SM_BLOCK_JACOBI) throw Error(-1, "singular nodal block in block Jacobi smoother");
  H->smoother_only = true;
  return H;
}

// ----------------------------------------------------------------------------
// V-cycle (multigrid.py:231), enqueue only
// ----------------------------------------------------------------------------

// Chebyshev passes on x (in place); x_zero: x holds garbage and means 0.
// `passes` Chebyshev passes on level l, x in/out.  want_r: the last step also
// stores its maintained residual r' = r - alpha A p' (= b - A x in exact
// arithmetic) and the buffer holding it is returned, so the V-cycle's residual
// after pre-smoothing costs no operator application (the reference recomputes
// b - A x, multigrid.py:238-239; the two differ by fp64 rounding only).
template <int DIM>
const double* smooth_cheb(Hierarchy& H, Level& l, const double* b, double* x, bool x_zero, int passes,
                          cudaStream_t s, bool want_r = false, const Red* dot = nullptr, bool* dot_done = nullptr) {
  const double* rlast = nullptr;
  for (int p = 0; p < passes; ++p) {
    const double* rin;
    if (x_zero) {
      rin = b;
    } else {
      lvl_residual<DIM>(l, x, b, l.r.get(), s);
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
      const double* zs = rin;
      const double* dv = l.dinv.get();
      if (H.sm.kind == SM_SOR_CHEBYSHEV) {  // z = SOR solve of r (multigrid.py:138)
        sor_solve(l, rin, l.z.get(), s);
        zs = l.z.get();
        dv = nullptr;
      }
      // the last step's r' is read only by the V-cycle (want_r, last pass); p'
      // of the last step is never read
      const bool last = i + 1 == H.sm.degree;
      const bool keep_r = !last || (want_r && p + 1 == passes);
      static const bool x_only = [] {
        const char* e = std::getenv("TMG_CHEB_XONLY");
        return !(e && e[0] == '0');  // 0: the full step (operator applied, result dropped) -- A/B
      }();
      if (last && !keep_r && x_only) {
        // neither p' nor r' of this step is read: x += alpha p' needs no operator application
        // (the very last kernel of a level-0 V-cycle inside PCG also reduces r.z = x'.b)
        const bool with_dot = dot != nullptr && p + 1 == passes;
        const Red nored{nullptr, nullptr, nullptr};
        launch(k_cheb_x_only, with_dot ? std::min<unsigned>(grid_for(l.ndof), RED_BLOCKS * 4u) : grid_for(l.ndof), TPB, 0,
               s, zs, pin, dv, (const double*)l.coef.get(), i, (x_zero && i == 0) ? 1 : 0, x, l.ndof,
               with_dot ? b : (const double*)nullptr, with_dot ? *dot : nored);
        note_launch();
        if (with_dot && dot_done) *dot_done = true;
      } else {
        lvl_cheb_step<DIM>(l, rin, zs, dv, pin, i, x_zero && i == 0, x, po, keep_r ? ro : nullptr, s, !last);
      }
      if (last && keep_r) rlast = ro;
      rin = ro;
      pin = po;
    }
    x_zero = false;
  }
  return rlast;
}

template <int DIM>
void xfer_restrict(Hierarchy& H, int k, const double* r, double* xc_first, cudaStream_t s) {
  Level& l = *H.lv[k];
  Level& c = *H.lv[k + 1];
  if (l.xfer == XF_GEO) {
    launch(k_restrict<DIM>, node_grid<DIM>(c.L), node_block<DIM>(), 0, s, l.T, r, c.b.get(), c.dinv.get(), c.wdev.get(),
                                                                       xc_first);
  } else {
    TMG_BSR_RECT_DISPATCH(l.Pt.R, l.Pt.C,
                          launch(k_bsr_restrict<RR, CC>, bsr_grid(l.Pt), TPB, 0, s, 
                              view<RR, CC>(l.Pt), r, c.b.get(), c.dinv.get(), c.wdev.get(), xc_first))
  }
  note_launch();
}
template <int DIM>
void xfer_prolong_add(Hierarchy& H, int k, double* x, cudaStream_t s) {
  Level& l = *H.lv[k];
  Level& c = *H.lv[k + 1];
  if (l.xfer == XF_GEO) {
    launch(k_prolong_add<DIM>, node_grid<DIM>(l.L), node_block<DIM>(), 0, s, l.T, c.x.get(), x);
  } else {
    TMG_BSR_RECT_DISPATCH(l.P.R, l.P.C,
                          launch(k_bsr_apply<RR, CC>, bsr_grid(l.P), TPB, 0, s, view<RR, CC>(l.P), c.x.get(), x, 1))
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
  const bool cheb = cheb_kind(H.sm.kind) || H.sm.kind == SM_SOR_GMRES;  // in-place polynomial / Krylov smoothers
  static const bool reuse_r = [] {
    const char* e = std::getenv("TMG_CHEB_RESIDUAL");
    return !(e && e[0] == '0');  // 0: recompute b - A x after pre-smoothing (the reference's order of work)
  }();
  const double* r_pre = nullptr;
  bool cheb_dot = false;
  auto smooth_poly = [&](double* x, bool x_zero, int passes, bool want_r, const Red* d = nullptr) {
    if (H.sm.kind == SM_SOR_GMRES) smooth_sor_gmres<DIM>(H, l, b, x, x_zero, passes, s);
    else r_pre = smooth_cheb<DIM>(H, l, b, x, x_zero, passes, s, want_r && reuse_r, d, &cheb_dot);
  };
  const int W = H.n_pre + H.n_post;
  auto buf = [&](int w) { return ((W - w) % 2 == 0) ? xout : l.xt.get(); };
  const Red nored{nullptr, nullptr, nullptr};
  double* xcur = nullptr;
  int widx = 0;
  if (cheb) {
    if (H.n_pre > 0) {
      smooth_poly(xout, true, H.n_pre, true);
      xcur = xout;
    }
  } else {
    for (int p = 0; p < H.n_pre; ++p) {
      double* dst = buf(++widx);
      if (!(p == 0 && first_done)) lvl_sweep<DIM, false>(H, l, b, xcur, dst, nored, s);
      xcur = dst;
    }
  }
  const double* r = b;
  if (r_pre) {
    r = r_pre;  // maintained by the last Chebyshev step
  } else if (xcur) {
    lvl_residual<DIM>(l, xcur, b, l.r.get(), s);
    r = l.r.get();
  }
  const bool cfirst = H.fused() && k + 1 < H.last();
  xfer_restrict<DIM>(H, k, r, cfirst ? H.first_dst(k + 1, c.x.get()) : nullptr, s);
  vcycle<DIM>(H, k + 1, c.b.get(), c.x.get(), s, cfirst, nullptr);
  bool dot_done = false;
  if (!xcur) {  // no pre-smoothing: x = 0 before the correction
    xcur = cheb ? xout : ((buf(widx + 1) == xout) ? l.xt.get() : xout);
    if (H.n_post == 0) xcur = xout;
    TMG_CUDA(cudaMemsetAsync(xcur, 0, l.ndof * sizeof(double), s));
  }
  static const int fuse_mode = [] {
    const char* e = std::getenv("TMG_FUSE_PROLONG");
    return e ? std::atoi(e) : 0;  // measured: unfused is faster on every level
  }();
  // (not on a streamed 3D level 0: its row kernels have their own launch shape)
  const bool fuse_prolong = !cheb && H.sm.kind == SM_JACOBI && H.n_post > 0 && l.xfer == XF_GEO && l.lattice() &&
                            !(DIM == 3 && l.opkind == OP_FINE) &&
                            (fuse_mode == 2 || (fuse_mode == 1 && l.opkind == OP_FINE));
  if (!fuse_prolong) xfer_prolong_add<DIM>(H, k, xcur, s);
  if (cheb) {
    // (the dot is valid only if the smoothed vector IS the V-cycle's output buffer)
    smooth_poly(xcur, false, H.n_post, false, (dot && xcur == xout && H.n_post > 0) ? dot : nullptr);
    dot_done |= cheb_dot;
  } else {
    for (int p = 0; p < H.n_post; ++p) {
      double* dst = buf(++widx);
      const bool last = p == H.n_post - 1 && dot != nullptr && H.sm.kind == SM_JACOBI;
      if (p == 0 && fuse_prolong) {
        with_lattice<DIM>(l, [&](auto o) {
          if (last)
            launch(k_prolong_jacobi<DIM, decltype(o), true>, TMG_ROW_OP_LAUNCH(l), s, 
                o, xcur, c.x.get(), l.T, b, l.dinv.get(), l.wdev.get(), dst, *dot);
          else
            launch(k_prolong_jacobi<DIM, decltype(o), false>, TMG_ROW_OP_LAUNCH(l), s, 
                o, xcur, c.x.get(), l.T, b, l.dinv.get(), l.wdev.get(), dst, nored);
        });
        note_launch();
      } else if (last) {
        lvl_sweep<DIM, true>(H, l, b, xcur, dst, *dot, s);
      } else {
        lvl_sweep<DIM, false>(H, l, b, xcur, dst, nored, s);
      }
      dot_done |= last;
      xcur = dst;
    }
  }
  if (xcur != xout) TMG_CUDA(cudaMemcpyAsync(xout, xcur, l.ndof * sizeof(double), cudaMemcpyDeviceToDevice, s));
  return dot_done;
}

// `passes` passes of the configured smoother on level l, x in/out (the
// smoother classes' apply(x, b, passes), multigrid.py:57/90/131/161)
template <int DIM>
void level_smooth(Hierarchy& H, Level& l, const double* b, double* x, int passes, cudaStream_t s) {
  if (passes <= 0) return;
  const int kind = H.sm.kind;
  if (cheb_kind(kind)) {
    smooth_cheb<DIM>(H, l, b, x, false, passes, s);
  } else if (kind == SM_SOR_GMRES) {
    smooth_sor_gmres<DIM>(H, l, b, x, false, passes, s);
  } else {
    const Red nored{nullptr, nullptr, nullptr};
    double* cur = x;
    double* other = l.xt.get();
    for (int p = 0; p < passes; ++p) {
      lvl_sweep<DIM, false>(H, l, b, cur, other, nored, s);
      std::swap(cur, other);
    }
    if (cur != x) TMG_CUDA(cudaMemcpyAsync(x, cur, l.ndof * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
}

}  // namespace tmg
