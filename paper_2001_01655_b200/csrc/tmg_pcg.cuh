// Preconditioned CG (extension of the reference's krylov module, krylov.py:134
// documents CG as the natural extension for SPD K and M) executed as ONE CUDA
// graph: a prologue (initial residual, tolerance) followed by a device-side WHILE
// conditional node whose body is [V-cycle z=M r] [r.z] [p=z+beta p, q=A p, p.q]
// [x+=alpha p, r-=alpha q, r.r] [convergence check -> cudaGraphSetConditional].
// No host round trip per iteration; dot products use deterministic two-level
// reductions so the iterate sequence is bitwise reproducible.
#pragma once
#include "tmg_gmg.cuh"

namespace tmg {

struct CgCfg {
  double rtol;
  int maxit;
};
struct CgState {
  double rz, tol;
  int it, converged;
};

__global__ void k_cg_init(const CgCfg* __restrict__ cfg, CgState* __restrict__ st, const double* __restrict__ bb,
                          const double* __restrict__ rr, double* __restrict__ hist, cudaGraphConditionalHandle h) {
  const double tol = cfg->rtol * sqrt(*bb);
  const double r0 = sqrt(*rr);
  st->tol = tol;
  st->it = 0;
  st->rz = 0.0;
  hist[0] = r0;
  st->converged = r0 <= tol;
  cudaGraphSetConditional(h, (!(r0 <= tol) && cfg->maxit > 0) ? 1u : 0u);
}

template <int DIM, class Op>
__global__ void __launch_bounds__(TPB) k_cg_pq(Op op, const double* __restrict__ z, const double* __restrict__ p,
                                               double* __restrict__ pn, double* __restrict__ q,
                                               const CgState* __restrict__ st, const double* __restrict__ rz_new,
                                               Red red) {
  TMG_NODE_PROLOGUE
  const double beta = st->it == 0 ? 0.0 : (*rz_new / st->rz);
  double v = 0.0;
  if (active) {
    AxpySrc<DIM> src{z, p, beta};
    double out[DIM];
    op.row(node, ci, cj, ck, src, out);
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
      const double pv = src(node, c);
      pn[node * DIM + c] = pv;
      q[node * DIM + c] = out[c];
      v += pv * out[c];
    }
  }
  grid_reduce(v, red);
}

__global__ void __launch_bounds__(TPB) k_cg_update(double* __restrict__ x, double* __restrict__ r, double* __restrict__ p,
                                                   const double* __restrict__ pn, const double* __restrict__ q,
                                                   long long n, const double* __restrict__ rz_new,
                                                   const double* __restrict__ pq, Red red) {
  const double alpha = *rz_new / *pq;
  double v = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double pv = pn[i];
    x[i] += alpha * pv;
    const double ri = r[i] - alpha * q[i];
    r[i] = ri;
    p[i] = pv;
    v += ri * ri;
  }
  grid_reduce(v, red);
}

__global__ void k_cg_check(const CgCfg* __restrict__ cfg, CgState* __restrict__ st, const double* __restrict__ rz_new,
                           const double* __restrict__ rr, double* __restrict__ hist, cudaGraphConditionalHandle h) {
  st->rz = *rz_new;
  const int it = st->it + 1;
  st->it = it;
  const double rn = sqrt(*rr);
  hist[it] = rn;
  const bool conv = rn <= st->tol;
  st->converged = conv;
  cudaGraphSetConditional(h, (!conv && it < cfg->maxit) ? 1u : 0u);
}

struct PcgCtx {
  long long ndof = 0;
  int hist_cap = 0;
  DevBuf<double> b, x, r, z, p, pn, q, hist;
  DevBuf<CgCfg> cfg;
  DevBuf<CgState> st;
  RedSlot bb, rr, rz, pq;
  cudaStream_t cs = nullptr, cs2 = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  bool use_x0_graph = false;
  long long prologue_launches = 0, body_launches = 0;
  ~PcgCtx() {
    if (exec) cudaGraphExecDestroy(exec);
    if (cs) cudaStreamDestroy(cs);
    if (cs2) cudaStreamDestroy(cs2);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
  }
};

template <int DIM>
void pcg_build_graph(PcgCtx& C, const Operator& K, Hierarchy* H, bool use_x0) {
  const long long n = C.ndof;
  const unsigned gn = grid_for(K.L.n);
  const unsigned gv = std::min<unsigned>(grid_for(n), 1184);
  if (C.exec) { cudaGraphExecDestroy(C.exec); C.exec = nullptr; }
  cudaStream_t s = C.cs;
  TMG_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  cudaStreamCaptureStatus cst;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  TMG_CUDA(cudaStreamGetCaptureInfo(s, &cst, nullptr, &g, &deps, &ndeps));
  cudaGraphConditionalHandle handle;
  TMG_CUDA(cudaGraphConditionalHandleCreate(&handle, g, 0, 0));
  auto op0 = K.template fine<DIM>();
  const long long c0 = launch_counter().load();
  // prologue
  if (use_x0) {
    k_residual<DIM, decltype(op0)><<<gn, TPB, smem_of(op0), s>>>(op0, C.x.get(), C.b.get(), C.r.get()); ::tmg::note_launch();
  } else {
    TMG_CUDA(cudaMemsetAsync(C.x.get(), 0, n * sizeof(double), s));
    TMG_CUDA(cudaMemcpyAsync(C.r.get(), C.b.get(), n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  k_dot<<<gv, TPB, 0, s>>>(C.b.get(), C.b.get(), n, C.bb.red()); ::tmg::note_launch();
  k_dot<<<gv, TPB, 0, s>>>(C.r.get(), C.r.get(), n, C.rr.red()); ::tmg::note_launch();
  k_cg_init<<<1, 1, 0, s>>>(C.cfg.get(), C.st.get(), C.bb.res.get(), C.rr.res.get(), C.hist.get(), handle); ::tmg::note_launch();
  TMG_CUDA(cudaGetLastError());
  const long long c1 = launch_counter().load();
  // while node
  TMG_CUDA(cudaStreamGetCaptureInfo(s, &cst, nullptr, &g, &deps, &ndeps));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = handle;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cnode;
  TMG_CUDA(cudaGraphAddNode(&cnode, g, deps, ndeps, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  TMG_CUDA(cudaStreamUpdateCaptureDependencies(s, &cnode, 1, cudaStreamSetCaptureDependencies));
  cudaStream_t b2 = C.cs2;
  TMG_CUDA(cudaStreamBeginCaptureToGraph(b2, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  const double* z = C.r.get();
  if (H) {
    vcycle<DIM>(*H, 0, C.r.get(), C.z.get(), b2);
    z = C.z.get();
  }
  k_dot<<<gv, TPB, 0, b2>>>(C.r.get(), z, n, C.rz.red()); ::tmg::note_launch();
  k_cg_pq<DIM, decltype(op0)><<<gn, TPB, smem_of(op0), b2>>>(op0, z, C.p.get(), C.pn.get(), C.q.get(), C.st.get(),
                                                             C.rz.res.get(), C.pq.red()); ::tmg::note_launch();
  k_cg_update<<<gv, TPB, 0, b2>>>(C.x.get(), C.r.get(), C.p.get(), C.pn.get(), C.q.get(), n, C.rz.res.get(),
                                  C.pq.res.get(), C.rr.red()); ::tmg::note_launch();
  k_cg_check<<<1, 1, 0, b2>>>(C.cfg.get(), C.st.get(), C.rz.res.get(), C.rr.res.get(), C.hist.get(), handle); ::tmg::note_launch();
  TMG_CUDA(cudaGetLastError());
  const long long c2 = launch_counter().load();
  C.prologue_launches = c1 - c0;
  C.body_launches = c2 - c1;
  note_launch(-(c2 - c0));  // captured, not executed
  cudaGraph_t body_out = nullptr;
  TMG_CUDA(cudaStreamEndCapture(b2, &body_out));
  cudaGraph_t gout = nullptr;
  TMG_CUDA(cudaStreamEndCapture(s, &gout));
  TMG_CUDA(cudaGraphInstantiate(&C.exec, gout, 0));
  cudaGraphDestroy(gout);
  C.use_x0_graph = use_x0;
}

struct PcgResult {
  int iterations = 0, converged = 0;
  double r0 = 0, rfinal = 0, ms = 0;
  std::vector<double> hist;
};

template <int DIM>
PcgResult pcg_solve(std::unique_ptr<PcgCtx>& slot, const Operator& K, Hierarchy* H, const double* b, double* x,
                    bool use_x0, double rtol, int maxit, cudaStream_t user) {
  TMG_REQUIRE(rtol > 0.0 && rtol < 1.0, "rtol must be in (0, 1)");
  TMG_REQUIRE(maxit >= 0, "max_iterations must be >= 0");
  if (!slot) slot = std::make_unique<PcgCtx>();
  PcgCtx& C = *slot;
  const long long n = K.ndof;
  bool rebuild = C.exec == nullptr || C.use_x0_graph != use_x0;
  if (C.ndof != n) {
    C.ndof = n;
    const unsigned gmax = std::max(grid_for(K.L.n), 1184u);
    cudaStream_t s = user;
    C.b.alloc(n, s); C.x.alloc(n, s); C.r.alloc(n, s); C.z.alloc(n, s);
    C.p.alloc(n, s); C.pn.alloc(n, s); C.q.alloc(n, s);
    C.cfg.alloc(1, s); C.st.alloc(1, s);
    C.bb.alloc(gmax, s); C.rr.alloc(gmax, s); C.rz.alloc(gmax, s); C.pq.alloc(gmax, s);
    TMG_CUDA(cudaStreamCreateWithFlags(&C.cs, cudaStreamNonBlocking));
    TMG_CUDA(cudaStreamCreateWithFlags(&C.cs2, cudaStreamNonBlocking));
    TMG_CUDA(cudaEventCreate(&C.e0));
    TMG_CUDA(cudaEventCreate(&C.e1));
    rebuild = true;
  }
  if (maxit + 1 > C.hist_cap) {
    C.hist_cap = std::max(maxit + 1, 1024);
    C.hist.alloc(C.hist_cap, user);
    rebuild = true;
  }
  if (rebuild) {
    TMG_CUDA(cudaStreamSynchronize(user));  // buffers allocated on `user` must exist before capture
    pcg_build_graph<DIM>(C, K, H, use_x0);
  }
  CgCfg hc{rtol, maxit};
  TMG_CUDA(cudaEventRecord(C.e0, user));
  TMG_CUDA(cudaMemcpyAsync(C.cfg.get(), &hc, sizeof(hc), cudaMemcpyHostToDevice, user));
  TMG_CUDA(cudaMemcpyAsync(C.b.get(), b, n * sizeof(double), cudaMemcpyDeviceToDevice, user));
  if (use_x0) TMG_CUDA(cudaMemcpyAsync(C.x.get(), x, n * sizeof(double), cudaMemcpyDeviceToDevice, user));
  TMG_CUDA(cudaGraphLaunch(C.exec, user));
  TMG_CUDA(cudaMemcpyAsync(x, C.x.get(), n * sizeof(double), cudaMemcpyDeviceToDevice, user));
  TMG_CUDA(cudaEventRecord(C.e1, user));
  CgState hs;
  TMG_CUDA(cudaMemcpyAsync(&hs, C.st.get(), sizeof(hs), cudaMemcpyDeviceToHost, user));
  TMG_CUDA(cudaStreamSynchronize(user));
  note_launch(C.prologue_launches + (long long)hs.it * C.body_launches);
  PcgResult res;
  res.iterations = hs.it;
  res.converged = hs.converged;
  res.hist.resize(hs.it + 1);
  TMG_CUDA(cudaMemcpy(res.hist.data(), C.hist.get(), (hs.it + 1) * sizeof(double), cudaMemcpyDeviceToHost));
  res.r0 = res.hist.front();
  res.rfinal = res.hist.back();
  float ms = 0.f;
  TMG_CUDA(cudaEventElapsedTime(&ms, C.e0, C.e1));
  res.ms = ms;
  return res;
}

}  // namespace tmg
