// Hex8 matrix-free operator rows, two x-adjacent nodes per thread (A/B build
// option -DTMG_FINE3_PAIR; the default 3D path is tmg_fine3h.cuh).
//
// The 3D level-0 product K u (mesh.py:327, Z K Z + I_fixed) costs 576 FMA per
// node (24 x 24 KE per element) against ~104 B of HBM traffic: on B200 it is
// bound by the FP64 pipe and the instruction issue around it, not by HBM.  In
// the node-per-thread tile (FineOp::row) every KE coefficient fetched from the
// constant bank (LDCU + UMOV into uniform registers) feeds ONE DFMA, and every
// neighbour value is re-masked per use.  Here a thread owns nodes (x, x+1):
// element e(-1)/e(0) of node x and e(0)/e(+1) of node x+1 sit at the same local
// corner, so each coefficient feeds two DFMAs; the staged tile holds masked
// values, so the inner loop is loads + DFMAs only.  Per node the arithmetic and
// its order are those of FineOp::row (same results bit for bit).
//
// Measured alternative (kept out): element products on the FP64 tensor pipe
// (DMMA m8n8k4, KE in A-fragments, slab-streamed 16x16 node columns) was slower
// (316 vs 194 us per config-4 sweep): each CTA walks its planes with exposed
// load / barrier latency at 2 CTAs per SM, and the B200 FP64 tensor peak is no
// higher than the DFMA peak.
#pragma once

namespace tmg {
namespace f3 {
constexpr int PX = 64, PY = 4, PZ = 2, NT = 256;   // nodes per CTA (x pairs per thread)
constexpr int HX = PX + 2, HY = PY + 2, HZ = PZ + 2, NH = HX * HY * HZ;  // staged nodes
constexpr int EX = PX + 1, EY = PY + 1, EZ = PZ + 1, NEL = EX * EY * EZ;  // staged elements
constexpr int SPN = (NH + NT - 1) / NT, SPE = (NEL + NT - 1) / NT;
constexpr size_t SMEM_BYTES = sizeof(double) * (NH * 3 + NEL);

inline dim3 grid(const Lat& L) {
  return dim3((L.nn[0] + PX - 1) / PX, (L.nn[1] + PY - 1) / PY, (L.nn[2] + PZ - 1) / PZ);
}
}  // namespace f3

// epi(node, i, j, k, out, self) for every node of the CTA inside the lattice:
// out = row of Z K Z + I_fixed applied to the source, self = source at the node.
// Called by all threads of the block.
template <class Src, class Epi>
__device__ __forceinline__ void fine3_pair_rows(const FineOp<3>& op, const Src& src, Epi&& epi) {
  using namespace f3;
  extern __shared__ __align__(16) double f3_sm[];
  double* xs = f3_sm;          // masked source, [node][3]
  double* es = xs + NH * 3;    // moduli
  const int t = threadIdx.x;
  const int i0 = blockIdx.x * PX - 1, j0 = blockIdx.y * PY - 1, k0 = blockIdx.z * PZ - 1;
  {  // stage: all loads in flight before the first shared store
    double v[SPN][3];
    double ev[SPE];
#pragma unroll
    for (int u = 0; u < SPN; ++u) {
      const int h = t + u * NT;
      const int hx = h % HX, hy = (h / HX) % HY, hz = h / (HX * HY);
      const int gi = i0 + hx, gj = j0 + hy, gk = k0 + hz;
#pragma unroll
      for (int c = 0; c < 3; ++c) v[u][c] = 0.0;
      if (h < NH && op.L.inside(gi, gj, gk)) {
        const int m = op.L.id(gi, gj, gk);
        src.load(m, gi, gj, gk, v[u]);
        const unsigned mk = __ldg(op.mask + m);
#pragma unroll
        for (int c = 0; c < 3; ++c)
          if (!((mk >> c) & 1u)) v[u][c] = 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < SPE; ++u) {
      const int e = t + u * NT;
      const int ex = i0 + e % EX, ey = j0 + (e / EX) % EY, ez = k0 + e / (EX * EY);
      const bool ok = e < NEL && ex >= 0 && ex < op.ne[0] && ey >= 0 && ey < op.ne[1] && ez >= 0 && ez < op.ne[2];
      ev[u] = ok ? __ldg(op.E + op.elem_id(ex, ey, ez)) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < SPN; ++u) {
      const int h = t + u * NT;
      if (h < NH)
#pragma unroll
        for (int c = 0; c < 3; ++c) xs[h * 3 + c] = v[u][c];
    }
#pragma unroll
    for (int u = 0; u < SPE; ++u) {
      const int e = t + u * NT;
      if (e < NEL) es[e] = ev[u];
    }
  }
  __syncthreads();
  const int tx = t & 31, ty = (t >> 5) & 3, tz = t >> 7;
  const int ax = 2 * tx;  // halo x of the element column left of node A (= node A's x - 1)
  double accA[3] = {0.0, 0.0, 0.0}, accB[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int ez = 0; ez < 2; ++ez)
#pragma unroll
    for (int ey = 0; ey < 2; ++ey)
#pragma unroll
      for (int ex = 0; ex < 2; ++ex) {
        // node A: element (ax+ex, ty+ey, tz+ez) of the staged element grid; node B: one to the right
        const double EA = es[(ax + ex) + EX * ((ty + ey) + EY * (tz + ez))];
        const double EB = es[(ax + ex + 1) + EX * ((ty + ey) + EY * (tz + ez))];
        const int ln = corner_of(1 - ex, 1 - ey, 1 - ez);
        double tA[3] = {0.0, 0.0, 0.0}, tB[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const int hx = ax + ex + corner_x(m), hy = ty + ey + corner_y(m), hz = tz + ez + corner_z(m);
          const double* pa = xs + 3 * (hx + HX * (hy + HY * hz));
          double ua[3], ub[3];
#pragma unroll
          for (int d = 0; d < 3; ++d) { ua[d] = pa[d]; ub[d] = pa[3 + d]; }
#pragma unroll
          for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              const double k = op.ke[(ln * 3 + c) * 24 + m * 3 + d];
              tA[c] += k * ua[d];
              tB[c] += k * ub[d];
            }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          accA[c] += EA * tA[c];
          accB[c] += EB * tB[c];
        }
      }
  const int gj = j0 + 1 + ty, gk = k0 + 1 + tz;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int gi = i0 + 1 + ax + h;
    if (gi < op.L.nn[0] && gj < op.L.nn[1] && gk < op.L.nn[2]) {
      const int node = op.L.id(gi, gj, gk);
      double self[3], out[3];
      src.load(node, gi, gj, gk, self);
      const unsigned mk = __ldg(op.mask + node);
      const double* acc = h ? accB : accA;
#pragma unroll
      for (int c = 0; c < 3; ++c) out[c] = ((mk >> c) & 1u) ? acc[c] : self[c];
      epi(node, gi, gj, gk, out, self);
    }
  }
}

}  // namespace tmg
