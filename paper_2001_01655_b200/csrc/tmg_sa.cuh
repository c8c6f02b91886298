// Host orchestration of the smoothed-aggregation levels (multigrid.py:528-606):
// strength graph -> exact greedy aggregation -> tentative QR prolongation ->
// power-method omega -> smoothed P -> P^T -> Galerkin P^T A P, per level, all on
// the device.  The host only reads back a handful of integers per level
// (aggregate counts, overflow/error flags) to size the next allocations.
#pragma once
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "tmg_gmg.cuh"

namespace tmg {

// TMG_VERBOSE=1: per-phase setup timings on stderr (synchronises the stream).

__global__ void k_sqrt_to(const double* __restrict__ v2, double* __restrict__ out) {
  TMG_PDL_ENTRY; *out = sqrt(*v2); }
__global__ void k_clamp_agg(int* __restrict__ agg, int n, int n_reg) {
  TMG_PDL_ENTRY;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && agg[i] >= n_reg) agg[i] = n_reg - 1;
}

inline void bsr_transpose(const Bsr& P, Bsr& Pt, cudaStream_t s) {
  const long long nnz = P.nnzb;
  Pt.nrows = P.ncols;
  Pt.ncols = P.nrows;
  Pt.R = P.C;
  Pt.C = P.R;
  Pt.nnzb = nnz;
  DevBuf<int> rowof, iota, keys_out, perm, cnt;
  rowof.alloc(nnz, s); iota.alloc(nnz, s); keys_out.alloc(nnz, s); perm.alloc(nnz, s);
  k_row_of<<<grid_for(P.nrows), TPB, 0, s>>>(P.rowptr.get(), P.nrows, rowof.get());
  k_iota<<<grid_for(nnz), TPB, 0, s>>>(iota.get(), nnz);
  size_t tb = 0;
  TMG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, P.col.get(), keys_out.get(), iota.get(), perm.get(), (int)nnz,
                                           0, 32, s));
  DevBuf<char> tmp;
  tmp.alloc(tb, s);
  TMG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, P.col.get(), keys_out.get(), iota.get(), perm.get(),
                                           (int)nnz, 0, 32, s));
  cnt.alloc(Pt.nrows + 1, s);
  cnt.zero(s);
  k_count_cols<<<grid_for(nnz), TPB, 0, s>>>(P.col.get(), nnz, cnt.get());
  rowptr_from_counts(cnt, Pt.rowptr, Pt.nrows, s);
  Pt.col.alloc(nnz, s);
  Pt.val.alloc(nnz * P.R * P.C, s);
  k_transpose_fill<<<grid_for(nnz), TPB, 0, s>>>(perm.get(), rowof.get(), P.val.get(), P.R, P.C, nnz, Pt.col.get(),
                                                 Pt.val.get());
  note_launch(4);
  TMG_CUDA(cudaGetLastError());
}

// C = X * Y (block shapes X: R1 x K1, Y: K1 x C2)
inline void bsr_spgemm(const Bsr& X, const Bsr& Y, Bsr& Cm, cudaStream_t s) {
  TMG_REQUIRE(X.C == Y.R && X.ncols == Y.nrows, "spgemm shape mismatch");
  const int n = X.nrows;
  Cm.nrows = n;
  Cm.ncols = Y.ncols;
  Cm.R = X.R;
  Cm.C = Y.C;
  DevBuf<int> cnt, heavy;
  cnt.alloc(n + 1, s);
  cnt.zero(s);
  heavy.alloc(n, s);
  heavy.zero(s);
  const unsigned g = (unsigned)((n + SG_WARPS - 1) / SG_WARPS);
  k_spgemm_count<<<g, SG_WARPS * 32, 0, s>>>(X.rowptr.get(), X.col.get(), Y.rowptr.get(), Y.col.get(), n, cnt.get(),
                                             heavy.get());
  note_launch();
  // rows whose column set overflows the shared-memory hash: sort+unique in global memory
  std::vector<int> hheavy(n);
  TMG_CUDA(cudaMemcpyAsync(hheavy.data(), heavy.get(), n * sizeof(int), cudaMemcpyDeviceToHost, s));
  TMG_CUDA(cudaStreamSynchronize(s));
  std::vector<int> heavy_rows;
  for (int r = 0; r < n; ++r)
    if (hheavy[r]) heavy_rows.push_back(r);
  std::vector<DevBuf<int>> heavy_cols(heavy_rows.size());
  std::vector<int> heavy_n(heavy_rows.size());
  for (size_t t = 0; t < heavy_rows.size(); ++t) {
    const int r = heavy_rows[t];
    DevBuf<unsigned long long> bnd, pos;
    bnd.alloc(1, s); bnd.zero(s); pos.alloc(1, s); pos.zero(s);
    k_heavy_bound<<<1, 256, 0, s>>>(X.rowptr.get(), X.col.get(), Y.rowptr.get(), r, bnd.get());
    unsigned long long hb = 0;
    TMG_CUDA(cudaMemcpyAsync(&hb, bnd.get(), sizeof(hb), cudaMemcpyDeviceToHost, s));
    TMG_CUDA(cudaStreamSynchronize(s));
    DevBuf<int> cand, sorted, nsel;
    cand.alloc(hb, s); sorted.alloc(hb, s); nsel.alloc(1, s);
    heavy_cols[t].alloc(hb, s);
    k_heavy_gather<<<1024, 256, 0, s>>>(X.rowptr.get(), X.col.get(), Y.rowptr.get(), Y.col.get(), r, cand.get(),
                                        pos.get());
    size_t tb = 0;
    TMG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, cand.get(), sorted.get(), (int)hb, 0, 32, s));
    size_t tb2 = 0;
    TMG_CUDA(cub::DeviceSelect::Unique(nullptr, tb2, sorted.get(), heavy_cols[t].get(), nsel.get(), (int)hb, s));
    DevBuf<char> tmp;
    tmp.alloc(std::max(tb, tb2), s);
    TMG_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(), tb, cand.get(), sorted.get(), (int)hb, 0, 32, s));
    TMG_CUDA(cub::DeviceSelect::Unique(tmp.get(), tb2, sorted.get(), heavy_cols[t].get(), nsel.get(), (int)hb, s));
    TMG_CUDA(cudaMemcpyAsync(cnt.get() + r, nsel.get(), sizeof(int), cudaMemcpyDeviceToDevice, s));
    heavy_n[t] = read_int(nsel.get(), s);
    note_launch(2);
  }
  rowptr_from_counts(cnt, Cm.rowptr, n, s);
  Cm.nnzb = read_int(Cm.rowptr.get() + n, s);
  Cm.col.alloc(std::max<long long>(Cm.nnzb, 1), s);
  Cm.val.alloc(std::max<long long>(Cm.nnzb, 1) * Cm.R * Cm.C, s);
  for (size_t t = 0; t < heavy_rows.size(); ++t) {
    const int off = read_int(Cm.rowptr.get() + heavy_rows[t], s);
    TMG_CUDA(cudaMemcpyAsync(Cm.col.get() + off, heavy_cols[t].get(), heavy_n[t] * sizeof(int),
                             cudaMemcpyDeviceToDevice, s));
  }
#define TMG_SPGEMM_CASE(a, b, c)                                                                               \
  if (X.R == a && X.C == b && Y.C == c) {                                                                       \
    k_spgemm_fill<a, b, c><<<g, SG_WARPS * 32, 0, s>>>(X.rowptr.get(), X.col.get(), X.val.get(), Y.rowptr.get(), \
                                                       Y.col.get(), Y.val.get(), n, Cm.rowptr.get(), Cm.col.get(), \
                                                       Cm.val.get(), heavy.get());                             \
    for (size_t t = 0; t < heavy_rows.size(); ++t)                                                              \
      k_heavy_fill<a, b, c><<<grid_for(heavy_n[t]), TPB, 0, s>>>(X.rowptr.get(), X.col.get(), X.val.get(),      \
                                                                 Y.rowptr.get(), Y.col.get(), Y.val.get(),      \
                                                                 heavy_rows[t], Cm.rowptr.get(), Cm.col.get(),  \
                                                                 Cm.val.get());                                 \
  } else
  TMG_SPGEMM_CASE(2, 2, 3)
  TMG_SPGEMM_CASE(3, 2, 3)
  TMG_SPGEMM_CASE(3, 3, 6)
  TMG_SPGEMM_CASE(6, 3, 6)
  TMG_SPGEMM_CASE(3, 3, 3)
  TMG_SPGEMM_CASE(6, 6, 6)
  TMG_SPGEMM_CASE(1, 1, 1)
  TMG_SPGEMM_CASE(1, 1, 3)
  TMG_SPGEMM_CASE(3, 1, 3)
  TMG_SPGEMM_CASE(1, 1, 6)
  TMG_SPGEMM_CASE(6, 1, 6)
  throw Error(-1, "unsupported SpGEMM block shape");
#undef TMG_SPGEMM_CASE
  note_launch(2);
  TMG_CUDA(cudaGetLastError());
}

// aggregate_nodes + _merge_small_aggregates on the strength graph of A
inline void aggregate_level(const Bsr& A, double beta, int bs, int nvec, bool drop_isolated, Level& l,
                            std::vector<std::string>& flags, cudaStream_t s) {
  const int n = A.nrows;
  DevBuf<double> md;
  md.alloc(n, s);
  DevBuf<unsigned> bad;
  bad.alloc(1, s);
  bad.zero(s);
  TMG_BSR_SQUARE_DISPATCH(bs, k_strength_diag<RR><<<grid_for(n), TPB, 0, s>>>(view<RR, RR>(A), md.get(), bad.get()))
  unsigned hb = 0;
  TMG_CUDA(cudaMemcpyAsync(&hb, bad.get(), sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  TMG_CUDA(cudaStreamSynchronize(s));
  if (hb) throw Error(-1, "zero diagonal block; input looks unassembled or singular");
  DevBuf<int> cnt;
  cnt.alloc(n + 1, s);
  cnt.zero(s);
  TMG_BSR_SQUARE_DISPATCH(bs, k_strength<RR, false><<<grid_for(n), TPB, 0, s>>>(view<RR, RR>(A), md.get(), beta,
                                                                                  cnt.get(), nullptr, nullptr))
  rowptr_from_counts(cnt, l.sptr, n, s);
  const int snnz = read_int(l.sptr.get() + n, s);
  l.scol.alloc(std::max(snnz, 1), s);
  TMG_BSR_SQUARE_DISPATCH(bs, k_strength<RR, true><<<grid_for(n), TPB, 0, s>>>(view<RR, RR>(A), md.get(), beta,
                                                                                 nullptr, l.sptr.get(), l.scol.get()))
  note_launch(3);
  // pass 1: distance-2 LFMIS (cooperative rounds)
  DevBuf<int> st, flag, rounds;
  st.alloc(n, s); flag.alloc(1, s); flag.zero(s); rounds.alloc(1, s); rounds.zero(s);
  k_agg_init<<<grid_for(n), TPB, 0, s>>>(l.sptr.get(), n, st.get());
  {
    // flat lower-numbered distance-2 lists (count, scan, fill)
    DevBuf<int> n2cnt, n2ptr, n2col;
    n2cnt.alloc(n + 1, s);
    n2cnt.zero(s);
    k_n2<false><<<grid_for(n), TPB, 0, s>>>(l.sptr.get(), l.scol.get(), n, n2cnt.get(), nullptr, nullptr);
    rowptr_from_counts(n2cnt, n2ptr, n, s);
    const int n2nnz = read_int(n2ptr.get() + n, s);
    n2col.alloc(std::max(n2nnz, 1), s);
    k_n2<true><<<grid_for(n), TPB, 0, s>>>(l.sptr.get(), l.scol.get(), n, nullptr, n2ptr.get(), n2col.get());
    note_launch(2);
    int dev = 0, nsm = 0, per = 0;
    TMG_CUDA(cudaGetDevice(&dev));
    TMG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    // Barrier-free sweeps win while a thread owns ~1 node (config 1 level 0:
    // 3.4 vs 6.4 ms); with several nodes per thread every re-sweep gets longer
    // and grid-synchronised rounds win (config 2 level 0: 13.2 vs 20.1 ms).
    // TMG_LFMIS_ASYNC=0/1 forces one of them.
    static const int force = [] {
      const char* e = std::getenv("TMG_LFMIS_ASYNC");
      return e ? std::atoi(e) : -1;
    }();
    int per_a = 0, per_r = 0;
    TMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_a, k_lfmis2, TPB, 0));
    TMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_r, k_lfmis2_rounds, TPB, 0));
    const bool async = force >= 0 ? force == 1 : (long long)n <= 2LL * nsm * per_a * TPB;
    void* kfun = async ? (void*)k_lfmis2 : (void*)k_lfmis2_rounds;
    per = async ? per_a : per_r;
    const int blocks = std::max(1, std::min(nsm * per, (int)grid_for(n)));
    const int* a0 = n2ptr.get();
    const int* a1 = n2col.get();
    int* a3 = st.get();
    int* a4 = flag.get();
    int* a5 = rounds.get();
    void* args[] = {(void*)&a0, (void*)&a1, (void*)&n, (void*)&a3, (void*)&a4, (void*)&a5};
    PhaseLog lg(s);
    lg.mark("  strength graph (nnz)", snnz);
    TMG_CUDA(cudaLaunchCooperativeKernel(kfun, blocks, TPB, args, 0, s));
    note_launch();
    if (lg.on) lg.mark("  LFMIS (max sweeps)", read_int(rounds.get(), s));
  }
  DevBuf<int> isroot, rank, agg1, ptr, isoflag, isorank;
  isroot.alloc(n + 1, s); rank.alloc(n + 1, s); agg1.alloc(n, s); ptr.alloc(n, s);
  isroot.zero(s);
  k_flag_eq<<<grid_for(n), TPB, 0, s>>>(st.get(), n, ST_ROOT, isroot.get());
  exclusive_scan(isroot.get(), rank.get(), n + 1, s);
  k_agg_pass1<<<grid_for(n), TPB, 0, s>>>(l.sptr.get(), l.scol.get(), n, st.get(), rank.get(), agg1.get());
  k_agg_pass2_ptr<<<grid_for(n), TPB, 0, s>>>(l.sptr.get(), l.scol.get(), n, agg1.get(), ptr.get());
  l.agg.alloc(n, s);
  k_agg_pass2_resolve<<<grid_for(n), TPB, 0, s>>>(n, agg1.get(), ptr.get(), l.agg.get());
  isoflag.alloc(n + 1, s); isorank.alloc(n + 1, s);
  isoflag.zero(s);
  k_flag_eq<<<grid_for(n), TPB, 0, s>>>(l.agg.get(), n, -1, isoflag.get());
  exclusive_scan(isoflag.get(), isorank.get(), n + 1, s);
  note_launch(7);
  const int n_root = read_int(rank.get() + n, s);
  const int U = read_int(isorank.get() + n, s);
  int n_agg = n_root;
  bool forced = false;
  if (n_agg == 0 || (long long)n_agg + U >= n) {
    k_pairwise<<<grid_for(n), TPB, 0, s>>>(l.agg.get(), n);
    note_launch();
    n_agg = (n + 1) / 2;
    forced = true;
    flags.push_back("forced_pairwise_aggregation");
  } else if (U > 0) {
    if (!drop_isolated) {
      k_assign_isolated<<<grid_for(n), TPB, 0, s>>>(n, isorank.get(), n_agg, l.agg.get());
      note_launch();
      n_agg += U;
    }
    flags.push_back("isolated_nodes");
  }
  l.n_dropped = (forced || !drop_isolated) ? 0 : U;
  // _merge_small_aggregates
  const int min_size = std::max(2, (nvec + bs - 1) / bs);
  DevBuf<int> size;
  size.alloc(n_agg, s);
  size.zero(s);
  k_histogram<<<grid_for(n), TPB, 0, s>>>(l.agg.get(), n, size.get());
  note_launch();
  std::vector<int> hsize(n_agg);
  TMG_CUDA(cudaMemcpyAsync(hsize.data(), size.get(), n_agg * sizeof(int), cudaMemcpyDeviceToHost, s));
  TMG_CUDA(cudaStreamSynchronize(s));
  int n_small = 0;
  for (int a = 0; a < n_agg; ++a) n_small += hsize[a] < min_size ? 1 : 0;
  if (n_small > 0) {
    if (!forced && !drop_isolated && min_size == 2 && n_small == U) {
      // the small aggregates are exactly the isolated singletons: they have no
      // strong neighbour, so the index-neighbour fallback folds each into the
      // last regular aggregate (multigrid.py:457-467)
      k_clamp_agg<<<grid_for(n), TPB, 0, s>>>(l.agg.get(), n, n_root);
      note_launch();
      n_agg = n_root;
    } else {
      DevBuf<int> remap, nout;
      remap.alloc(n_agg, s);
      nout.alloc(1, s);
      k_merge_small_seq<<<1, 1, 0, s>>>(l.sptr.get(), l.scol.get(), n, l.agg.get(), size.get(), n_agg, min_size,
                                         remap.get(), nout.get());
      note_launch();
      n_agg = read_int(nout.get(), s);
    }
  }
  l.n_agg = n_agg;
  TMG_CUDA(cudaGetLastError());
}

// tentative prolongation T (BSR, one bs x nv block per node) and coarse candidates Bc
inline void tentative_level(Level& l, const double* B, int n, int bs, int nv, DevBuf<double>& Bc, cudaStream_t s) {
  const int na = l.n_agg;
  DevBuf<int> iota, keys, members, size, offs;
  iota.alloc(n, s); keys.alloc(n, s); members.alloc(n, s);
  k_iota<<<grid_for(n), TPB, 0, s>>>(iota.get(), n);
  size_t tb = 0;
  TMG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, l.agg.get(), keys.get(), iota.get(), members.get(), n, 0, 32, s));
  DevBuf<char> tmp;
  tmp.alloc(tb, s);
  TMG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, l.agg.get(), keys.get(), iota.get(), members.get(), n, 0, 32,
                                           s));
  size.alloc(na + 1, s);
  size.zero(s);
  k_histogram<<<grid_for(n), TPB, 0, s>>>(l.agg.get(), n, size.get());
  offs.alloc(na + 1, s);
  exclusive_scan(size.get(), offs.get(), na + 1, s);
  // per-aggregate scratch offsets (m * nv doubles each)
  std::vector<int> hsize(na);
  TMG_CUDA(cudaMemcpyAsync(hsize.data(), size.get(), na * sizeof(int), cudaMemcpyDeviceToHost, s));
  TMG_CUDA(cudaStreamSynchronize(s));
  std::vector<long long> hoff(na + 1, 0);
  for (int a = 0; a < na; ++a) hoff[a + 1] = hoff[a] + (long long)hsize[a] * bs * nv;
  DevBuf<long long> woff;
  woff.alloc(na + 1, s);
  TMG_CUDA(cudaMemcpyAsync(woff.get(), hoff.data(), (na + 1) * sizeof(long long), cudaMemcpyHostToDevice, s));
  DevBuf<double> work;
  work.alloc(std::max<long long>(hoff[na], 1), s);
  // node-indexed blocks (zero for unaggregated nodes), then the BSR view
  l.Tnode.alloc((long long)n * bs * nv, s);
  l.Tnode.zero(s);
  Bc.alloc((long long)na * nv * nv, s);
  DevBuf<int> bad;
  bad.alloc(1, s);
  bad.zero(s);
  // radix sort puts the unaggregated (-1) nodes first: skip them
  k_tentative_qr<<<na, 128, 0, s>>>(offs.get(), members.get() + l.n_dropped, bs, nv, B, work.get(), woff.get(),
                                    l.Tnode.get(), Bc.get(), bad.get());
  note_launch(4);
  const int hbad = read_int(bad.get(), s);
  if (hbad)
    throw Error(-1, "aggregate with " + std::to_string(hbad) + " dofs cannot carry " + std::to_string(nv) +
                        " candidates");
  Bsr& T = l.Tm;
  T.nrows = n;
  T.ncols = na;
  T.R = bs;
  T.C = nv;
  DevBuf<int> cnt;
  cnt.alloc(n + 1, s);
  cnt.zero(s);
  k_flag_nonneg<<<grid_for(n), TPB, 0, s>>>(l.agg.get(), n, cnt.get());
  rowptr_from_counts(cnt, T.rowptr, n, s);
  T.nnzb = n - l.n_dropped;
  T.col.alloc(std::max<long long>(T.nnzb, 1), s);
  T.val.alloc(std::max<long long>(T.nnzb, 1) * bs * nv, s);
  k_compact_T<<<grid_for(n), TPB, 0, s>>>(n, l.agg.get(), T.rowptr.get(), l.Tnode.get(), bs * nv, T.col.get(),
                                          T.val.get());
  note_launch(2);
  TMG_CUDA(cudaGetLastError());
}

// omega = 4 / (3 rho(D^-1 A)), rho from 10 power steps from v0 (multigrid.py:504)
inline void spectral_radius(Hierarchy& H, const Bsr& A, int bs, const double* dinv, const double* v0, long long nd,
                            DevBuf<double>& rho, cudaStream_t s) {
  DevBuf<double> v, t, nrm;
  v.alloc(nd, s); t.alloc(nd, s); nrm.alloc(1, s);
  rho.alloc(1, s);
  TMG_CUDA(cudaMemcpyAsync(v.get(), v0, nd * sizeof(double), cudaMemcpyDeviceToDevice, s));
  const unsigned g = grid_for(nd), gr = red_grid(nd);
  for (int it = 0; it < 10; ++it) {
    Red rn = H.red.red();
    rn.result = nrm.get();
    k_dot<<<gr, TPB, 0, s>>>(v.get(), v.get(), nd, rn);
    k_div_sqrt<<<g, TPB, 0, s>>>(v.get(), nrm.get(), nd);
    TMG_BSR_SQUARE_DISPATCH(bs, k_bsr_apply<RR, RR><<<bsr_grid(A), TPB, 0, s>>>(view<RR, RR>(A), v.get(),
                                                                                       t.get(), 0))
    k_vmul<<<g, TPB, 0, s>>>(dinv, t.get(), v.get(), nd);
    note_launch(4);
  }
  Red rn = H.red.red();
  rn.result = nrm.get();
  k_dot<<<gr, TPB, 0, s>>>(v.get(), v.get(), nd, rn);
  k_sqrt_to<<<1, 1, 0, s>>>(nrm.get(), rho.get());
  note_launch(2);
}

// P = T - omega D^-1 (A T): AT by the BSR SpGEMM (heavy rows included), then the
// scaling/own-block update in place (multigrid.py:518-525).
template <int BS, int NV>
void smooth_p_typed(const Bsr& A, const Level& l, const double* dinv, Bsr& P, cudaStream_t s) {
  bsr_spgemm(A, l.Tm, P, s);
  k_p_from_at<BS, NV><<<grid_for(P.nrows), TPB, 0, s>>>(P.nrows, P.rowptr.get(), P.col.get(), P.val.get(),
                                                        l.agg.get(), l.Tnode.get(), dinv, l.rho.get());
  note_launch();
  TMG_CUDA(cudaGetLastError());
}
inline void smooth_p(const Bsr& A, const Level& l, const double* dinv, int bs, int nv, Bsr& P, cudaStream_t s) {
  if (bs == 2 && nv == 3) smooth_p_typed<2, 3>(A, l, dinv, P, s);
  else if (bs == 3 && nv == 6) smooth_p_typed<3, 6>(A, l, dinv, P, s);
  else if (bs == 3 && nv == 3) smooth_p_typed<3, 3>(A, l, dinv, P, s);
  else if (bs == 6 && nv == 6) smooth_p_typed<6, 6>(A, l, dinv, P, s);
  else if (bs == 1 && nv == 3) smooth_p_typed<1, 3>(A, l, dinv, P, s);
  else if (bs == 1 && nv == 6) smooth_p_typed<1, 6>(A, l, dinv, P, s);
  else if (bs == 1 && nv == 1) smooth_p_typed<1, 1>(A, l, dinv, P, s);
  else throw Error(-1, "unsupported (block size, candidates) combination");
}

// _sa_levels (multigrid.py:528): append SA levels below H.lv.back()
template <int DIM>
void sa_levels(Hierarchy& H, const double* B_dev, int nvec, int bs, long long coarse_max_dofs, double beta,
               const double* v0, cudaStream_t s, int max_levels = 30) {
  DevBuf<double> Bcur;  // candidates of the current level (device)
  const double* B = B_dev;
  int added = 0;
  PhaseLog log(s);
  while (H.lv.back()->ndof > coarse_max_dofs && added < max_levels) {
    Level& l = *H.lv.back();
    log.mark("sa level start (ndof)", l.ndof);
    Bsr Atmp;
    const Bsr* A = &l.Ab;
    if (l.lattice()) {
      lattice_to_bsr<DIM>(l, Atmp, s);
      A = &Atmp;
      log.mark("lattice->bsr (nnzb)", Atmp.nnzb);
    }
    const int n = A->nrows;
    std::vector<std::string> f;
    aggregate_level(*A, beta, bs, nvec, H.drop_isolated, l, f, s);
    log.mark("strength+aggregation (n_agg)", l.n_agg);
    H.flags.insert(H.flags.end(), f.begin(), f.end());
    if ((long long)l.n_agg * nvec >= l.ndof) {
      H.flags.push_back("aggregation_stalled");
      break;
    }
    DevBuf<double> Bc;
    tentative_level(l, B, n, bs, nvec, Bc, s);
    log.mark("tentative QR");
    // D^-1 of this level and omega
    DevBuf<double> d, dinv;
    DevBuf<unsigned> bad;
    d.alloc(l.ndof, s); dinv.alloc(l.ndof, s); bad.alloc(1, s); bad.zero(s);
    TMG_BSR_SQUARE_DISPATCH(bs, k_bsr_diag<RR><<<grid_for(n), TPB, 0, s>>>(view<RR, RR>(*A), d.get(), bad.get()))
    k_recip<<<grid_for(l.ndof), TPB, 0, s>>>(d.get(), dinv.get(), nullptr, l.ndof);
    note_launch(2);
    spectral_radius(H, *A, bs, dinv.get(), v0, l.ndof, l.rho, s);
    log.mark("spectral radius");
    smooth_p(*A, l, dinv.get(), bs, nvec, l.P, s);
    log.mark("smoothed P (nnzb)", l.P.nnzb);
    bsr_transpose(l.P, l.Pt, s);
    Bsr AP;
    bsr_spgemm(*A, l.P, AP, s);
    log.mark("P^T, A*P (nnzb)", AP.nnzb);
    auto c = std::make_unique<Level>();
    c->opkind = OP_BSR;
    c->bs = nvec;
    bsr_spgemm(l.Pt, AP, c->Ab, s);
    log.mark("P^T*(A*P) (nnzb)", c->Ab.nnzb);
    c->ndof = (long long)l.n_agg * nvec;
    l.xfer = XF_SPARSE;
    H.provenance.back() = 1;
    H.lv.push_back(std::move(c));
    H.provenance.push_back(1);
    Bcur = std::move(Bc);
    B = Bcur.get();
    bs = nvec;
    ++added;
  }
}

template <int DIM>
std::unique_ptr<Hierarchy> build_sa_amg(const Operator& K, const double* B_dev, int nvec, long long coarse_max_dofs,
                                        double beta, const double* v0, const SmootherCfg& sm, int n_pre, int n_post,
                                        bool drop_isolated, cudaStream_t s) {
  auto H = new_hierarchy<DIM>(sm, n_pre, n_post, s);
  H->drop_isolated = drop_isolated;
  const int bs = nvec == 3 ? 2 : nvec == 6 ? 3 : 1;
  TMG_REQUIRE(bs == DIM, "near-nullspace columns do not match the mesh dimension (3 in 2D, 6 in 3D)");
  H->lv.push_back(fine_level<DIM>(K));
  H->provenance.push_back(1);
  sa_levels<DIM>(*H, B_dev, nvec, bs, coarse_max_dofs, beta, v0, s);
  PhaseLog log(s);
  DevBuf<unsigned> bad;
  bad.alloc(1, s);
  bad.zero(s);
  const int nl = (int)H->lv.size();
  for (int k = 0; k < nl; ++k) level_setup<DIM>(*H, *H->lv[k], k < nl - 1, s, bad);
  log.mark("sa: smoother setup");
  coarse_setup<DIM>(*H, s);
  log.mark("sa: coarse inverse (n)", H->coarse.n);
  finalize_checks(*H, bad, s);
  return H;
}

// multigrid.py:573: n_geo geometric levels, then SA on the last geometric operator
// with the (un-zeroed) rigid-body modes of the coarse mesh (B_coarse, host-built).
template <int DIM>
std::unique_ptr<Hierarchy> build_hybrid(const Operator& K, int n_geo, const double* B_coarse, int nvec,
                                        long long coarse_max_dofs, double beta, const double* v0,
                                        const SmootherCfg& sm, int n_pre, int n_post, long long expect_sa_ndof,
                                        bool drop_isolated, cudaStream_t s) {
  auto H = new_hierarchy<DIM>(sm, n_pre, n_post, s);
  H->drop_isolated = drop_isolated;
  H->lv.push_back(fine_level<DIM>(K));
  H->provenance.push_back(0);
  std::vector<std::array<int, 3>> plan;
  plan.push_back({K.ne[0], K.ne[1], DIM == 3 ? K.ne[2] : 0});
  long long nd = K.ndof;
  for (int g = 0; g < n_geo; ++g) {
    auto cur = plan.back();
    bool all1 = true;
    for (int d = 0; d < DIM; ++d) all1 = all1 && cur[d] <= 1;
    if (all1) {
      H->flags.push_back("geometric_coarsening_exhausted");
      break;
    }
    if (nd <= coarse_max_dofs) break;
    std::array<int, 3> nx = cur;
    for (int d = 0; d < DIM; ++d) nx[d] = coarsen1(cur[d]);
    plan.push_back(nx);
    nd = DIM;
    for (int d = 0; d < DIM; ++d) nd *= nx[d] + 1;
  }
  add_geometric_levels<DIM>(*H, plan, s);
  TMG_REQUIRE(H->lv.back()->ndof == expect_sa_ndof, "hybrid: coarse candidate size does not match the plan");
  sa_levels<DIM>(*H, B_coarse, nvec, DIM, coarse_max_dofs, beta, v0, s);
  H->provenance.back() = 1;  // the coarsest level comes from _sa_levels: "algebraic"
  DevBuf<unsigned> bad;
  bad.alloc(1, s);
  bad.zero(s);
  const int nl = (int)H->lv.size();
  for (int k = 0; k < nl; ++k) level_setup<DIM>(*H, *H->lv[k], k < nl - 1, s, bad);
  coarse_setup<DIM>(*H, s);
  finalize_checks(*H, bad, s);
  return H;
}

}  // namespace tmg
