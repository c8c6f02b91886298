// C ABI (include/topomg_b200.h) over the B200 MG-PCG kernels.
#include <cstring>
#include <string>

#include "../../include/topomg_b200.h"
#include "tmg_pcg.cuh"
#include "tmg_gmres.cuh"
#include "tmg_sa.cuh"

using namespace tmg;

struct tmg_operator {
  Operator op;
  std::unique_ptr<PcgCtx> pcg;  // unpreconditioned CG workspace
  RedSlot sens;                 // compliance reduction of the sensitivity kernel (allocated once)
  double* comp_host = nullptr;  // pinned landing slot of the compliance scalar
  ~tmg_operator() {
    if (comp_host) cudaFreeHost(comp_host);
  }
};
struct tmg_hierarchy {
  std::unique_ptr<Hierarchy> h;
  const tmg_operator* K = nullptr;
  std::unique_ptr<PcgCtx> pcg;
};

static thread_local std::string g_err;

#define ABI_BEGIN try {
#define ABI_END                                   \
  }                                               \
  catch (const tmg::Error& e) {                   \
    g_err = e.what();                             \
    return e.code;                                \
  }                                               \
  catch (const std::exception& e) {               \
    g_err = e.what();                             \
    return TMG_ECUDA;                             \
  }                                               \
  return TMG_OK;

static cudaStream_t S(void* s) { return (cudaStream_t)s; }

static void require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw Error(TMG_ENODEV, "no CUDA device: the B200 path has no CPU fallback");
  }
  // Keep freed stream-ordered memory in the pool: a hierarchy is rebuilt every
  // optimisation step, and with the default release threshold (0) every
  // synchronisation hands the pool back to the driver, so the next build pays
  // for fresh page mappings (observed: AMG setup 48 ms vs 270 ms run to run).
  static const bool pool_ready = [] {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
    return true;
  }();
  (void)pool_ready;
}

static void check_mesh(const tmg_mesh_desc* m) {
  TMG_REQUIRE(m != nullptr, "mesh descriptor is NULL");
  TMG_REQUIRE(m->ndim == 2 || m->ndim == 3, "mesh must be 2D or 3D");
  for (int d = 0; d < m->ndim; ++d) {
    TMG_REQUIRE(m->dims[d] >= 1, "all dims must be >= 1");
    TMG_REQUIRE(m->h[d] > 0.0, "all element sizes must be > 0");
  }
}

// ----------------------------------------------------------------------------
// element kernels
// ----------------------------------------------------------------------------
__global__ void k_simp(const double* __restrict__ rho, long long n, double p, double e0, double emin,
                       double* __restrict__ E, unsigned* __restrict__ bad) {
  TMG_PDL_ENTRY;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double r = rho[i];
  if (!(r >= 0.0 && r <= 1.0)) atomicOr(bad, 1u);
  E[i] = emin + (e0 - emin) * pow(r, p);
}

__global__ void k_check_pos(const double* __restrict__ v, long long n, unsigned* __restrict__ bad) {
  TMG_PDL_ENTRY;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n && !(v[i] > 0.0)) atomicOr(bad, 1u);
}

// rho^(p-1) of the SIMP derivative: small integer exponents (p = 1, 2, 3, 4 --
// the reference's penal = 3) as exact-rounded products instead of the ~300
// instruction generic pow (a third of the sensitivity kernel's time).
__device__ __forceinline__ double simp_pow_m1(double r, double p) {
  if (p == 3.0) return r * r;
  if (p == 2.0) return r;
  if (p == 1.0) return 1.0;
  if (p == 4.0) return r * r * r;
  return pow(r, p - 1.0);
}

// Per-element strain energy ce_e = u_e^T KE u_e, the sensitivity
// dc_e = -dE/drho(rho_e) ce_e, and (f != nullptr) the compliance f.u in the
// same launch (optimization.py:106-111, 124-129).  Grid-stride over elements
// (x fastest: a warp's corner gathers are contiguous node runs) and over dofs
// (the compliance dot, reduced deterministically).  3D: the quadratic form in
// the reflection-character basis of tmg_fine3h.cuh -- u^ = T u_e (a 2x2x2
// Walsh-Hadamard transform per component) and u_e^T KE u_e = u^T KE^ u^ with
// the 45-term KE^ (~140 FP64 operations instead of 600).
template <int DIM>
__global__ void __launch_bounds__(TPB) k_sens(const __grid_constant__ FineOp<DIM> op, const double* __restrict__ u,
                                              const double* __restrict__ f, long long nelem, long long ndof,
                                              double* __restrict__ ce, const double* __restrict__ rho, double p,
                                              double e0, double emin, double* __restrict__ dc, Red red) {
  TMG_PDL_ENTRY;
  constexpr int NN = 1 << DIM, NE = DIM * NN;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nelem; e += stride) {
    const int ex = (int)(e % op.ne[0]);
    const long long t = e / op.ne[0];
    const int ey = (int)(t % op.ne[1]);
    const int ez = DIM == 3 ? (int)(t / op.ne[1]) : 0;
    double s = 0.0;
    if constexpr (DIM == 3) {
      double v[8][3];  // corner a = x + 2y + 4z
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const long long node = op.L.id(ex + (a & 1), ey + ((a >> 1) & 1), ez + (a >> 2));
#pragma unroll
        for (int c = 0; c < 3; ++c) v[a][c] = __ldg(u + node * 3 + c);
      }
#pragma unroll
      for (int b = 1; b < 8; b <<= 1)  // in-place Walsh-Hadamard: v[s] = sum_a (-1)^{popcount(s & a)} v[a]
#pragma unroll
        for (int a = 0; a < 8; ++a)
          if (!(a & b))
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              const double x0 = v[a][c], x1 = v[a | b][c];
              v[a][c] = x0 + x1;
              v[a | b][c] = x0 - x1;
            }
#pragma unroll
      for (int chi = 0; chi < 8; ++chi)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const int mi = f3h::blk_member(chi, i);
          if (mi < 3) continue;  // the mean character: zero row
          double y = 0.0;
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const int mj = f3h::blk_member(chi, j);
            if (f3h::blk_coef(chi, i, j) >= 0) y = fma(op.keh[f3h::blk_coef(chi, i, j)], v[mj / 3][mj % 3], y);
          }
          s = fma(v[mi / 3][mi % 3], y, s);
        }
    } else {
      double ue[NE];
#pragma unroll
      for (int m = 0; m < NN; ++m) {
        const long long node = op.L.id(ex + corner_x(m), ey + corner_y(m), 0);
#pragma unroll
        for (int c = 0; c < DIM; ++c) ue[m * DIM + c] = __ldg(u + node * DIM + c);
      }
#pragma unroll
      for (int i = 0; i < NE; ++i) {
        double ki = 0.0;
#pragma unroll
        for (int j = 0; j < NE; ++j) ki += op.ke[i * NE + j] * ue[j];
        s += ue[i] * ki;
      }
    }
    if (ce) ce[e] = s;
    if (dc) {
      const double r = rho[e];
      const double dE = p * (e0 - emin) * simp_pow_m1(r, p);
      dc[e] = -dE * s;
    }
  }
  if (f) {
    double a = 0.0, b = 0.0;
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    for (; i + stride < ndof; i += 2 * stride) {
      a += __ldg(f + i) * __ldg(u + i);
      b += __ldg(f + i + stride) * __ldg(u + i + stride);
    }
    if (i < ndof) a += __ldg(f + i) * __ldg(u + i);
    grid_reduce(a + b, red);
  }
}

// The 3D form of k_sens, streamed: a CTA owns a 32 x 8 tile of element columns
// and walks a z chunk one element layer per step.  Each node plane of the tile
// (33 x 9 nodes) is read ONCE, by coalesced row loads (register-staged one step
// ahead, then a double-buffered shared plane); a thread keeps the x-y character
// transform of its element's bottom face in registers, so an element costs 12
// shared loads instead of 24 strided global ones.  The compliance f.u is reduced
// from the same staged values (every node is owned by exactly one tile), so u is
// not read a second time.
namespace sens3 {
constexpr int TX = 32, TY = 8, NT = TX * TY;
constexpr int NRX = 3 * (TX + 1), NRY = TY + 1;   // doubles per staged row, rows per plane
constexpr int PITCH = NRX + 1;                    // (100 doubles: rows 8 banks apart)
constexpr int NLD = (NRX * NRY + NT - 1) / NT;    // staged doubles per thread and plane
}  // namespace sens3
__global__ void __launch_bounds__(sens3::NT, 2) k_sens3(const __grid_constant__ FineOp<3> op,
                                                        const double* __restrict__ u, const double* __restrict__ f,
                                                        double* __restrict__ ce, const double* __restrict__ rho,
                                                        double p, double e0, double emin, double* __restrict__ dc,
                                                        Red red) {
  TMG_PDL_ENTRY;
  using namespace sens3;
  __shared__ double sm[2][NRY * PITCH];
  const int t = threadIdx.x, tx = t % TX, ty = t / TX;
  const int nn0 = op.L.nn[0], nn1 = op.L.nn[1], nn2 = op.L.nn[2];
  const int ne0 = op.ne[0], ne1 = op.ne[1], ne2 = op.ne[2];
  const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
  const int zc = (ne2 + gridDim.z - 1) / gridDim.z;
  const int z0 = blockIdx.z * zc, z1 = min(ne2, z0 + zc);  // element layers [z0, z1), node planes [z0, z1]
  double dot = 0.0;
  if (z0 < z1) {
    // the staged doubles of this thread: row r, offset q in the row, global
    // offset inside a plane, and whether this tile owns the node (f.u)
    int soff[NLD];
    long long goff[NLD];
    bool ld_ok[NLD], own[NLD];
#pragma unroll
    for (int l = 0; l < NLD; ++l) {
      const int idx = t + l * NT, r = idx / NRX, q = idx % NRX;
      const int gi = i0 + q / 3, gj = j0 + r;
      ld_ok[l] = idx < NRX * NRY && gi < nn0 && gj < nn1;
      soff[l] = r * PITCH + q;
      goff[l] = 3 * ((long long)gj * nn0 + i0) + q;
      own[l] = ld_ok[l] && (q < 3 * TX || gi == nn0 - 1) && (r < TY || gj == nn1 - 1);
    }
    const long long plane3 = 3 * (long long)nn0 * nn1;
    double stage[NLD];
    auto load_plane = [&](int pz) {
      const bool own_z = f != nullptr && (pz < z1 || pz == nn2 - 1);
#pragma unroll
      for (int l = 0; l < NLD; ++l) {
        stage[l] = ld_ok[l] ? __ldg(u + plane3 * pz + goff[l]) : 0.0;
        if (own_z && own[l]) dot = fma(__ldg(f + plane3 * pz + goff[l]), stage[l], dot);
      }
    };
    auto store_plane = [&](int b) {
#pragma unroll
      for (int l = 0; l < NLD; ++l)
        if (t + l * NT < NRX * NRY) sm[b][soff[l]] = stage[l];
    };
    auto face = [&](int b, double (*F)[3]) {
      const double* S = sm[b] + ty * PITCH + 3 * tx;
      double v[4][3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        v[0][c] = S[c];
        v[1][c] = S[3 + c];
        v[2][c] = S[PITCH + c];
        v[3][c] = S[PITCH + 3 + c];
      }
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
    const int ex = i0 + tx, ey = j0 + ty;
    const bool el_ok = ex < ne0 && ey < ne1;
    const double de = e0 - emin;
    double Fb[4][3], Ft[4][3];
    load_plane(z0);
    store_plane(z0 & 1);
    load_plane(z0 + 1);
    __syncthreads();
    face(z0 & 1, Fb);
    for (int k = z0; k < z1; ++k) {
      store_plane((k + 1) & 1);            // plane k+1 (loaded one step ago)
      if (k + 2 <= z1) load_plane(k + 2);  // in flight during this layer
      __syncthreads();
      face((k + 1) & 1, Ft);
      double v[8][3];  // character s = q + 4 qz
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          v[q][c] = Fb[q][c] + Ft[q][c];
          v[q + 4][c] = Fb[q][c] - Ft[q][c];
          Fb[q][c] = Ft[q][c];
        }
      double s = 0.0;
#pragma unroll
      for (int chi = 0; chi < 8; ++chi)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const int mi = f3h::blk_member(chi, i);
          if (mi < 3) continue;  // the mean character: zero row
          double y = 0.0;
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const int mj = f3h::blk_member(chi, j);
            if (f3h::blk_coef(chi, i, j) >= 0) y = fma(op.keh[f3h::blk_coef(chi, i, j)], v[mj / 3][mj % 3], y);
          }
          s = fma(v[mi / 3][mi % 3], y, s);
        }
      if (el_ok) {
        const long long e = ((long long)k * ne1 + ey) * ne0 + ex;
        if (ce) ce[e] = s;
        if (dc) {
          const double r = __ldg(rho + e);
          const double dE = p * de * simp_pow_m1(r, p);
          dc[e] = -dE * s;
        }
      }
      // (no second barrier: the next step stores into the OTHER buffer, whose
      // last readers finished before this step's barrier)
    }
  }
  if (f) grid_reduce(dot, red);
}

// The 3D form of k_sens on bricks: a CTA owns 32 x 4 x 2 elements, one per
// thread.  The brick's 33 x 5 x 3 nodes are staged ONCE in shared memory by
// coalesced row loads (15 rows of 99 contiguous doubles), so an element costs
// 24 conflict-free shared loads instead of 24 strided global ones and every load
// of the CTA is in flight at once (no dependent steps: latency is hidden by the
// ~7000 independent CTAs).  The compliance f.u is reduced from the staged values
// (every node is owned by exactly one brick), so u is read from HBM once.
namespace sensb {
constexpr int BX = 32, BY = 4, BZ = 2, NT = BX * BY * BZ;
constexpr int NRX = 3 * (BX + 1), NROW = (BY + 1) * (BZ + 1);  // doubles per staged row, rows per brick
constexpr int PITCH = NRX + 1;                                 // (100 doubles: rows 8 banks apart)
constexpr int NLD = (NRX * NROW + NT - 1) / NT;                // staged doubles per thread
}  // namespace sensb
__global__ void __launch_bounds__(sensb::NT, 3) k_sensb(const __grid_constant__ FineOp<3> op,
                                                        const double* __restrict__ u, const double* __restrict__ f,
                                                        double* __restrict__ ce, const double* __restrict__ rho,
                                                        double p, double e0, double emin, double* __restrict__ dc,
                                                        Red red) {
  TMG_PDL_ENTRY;
  using namespace sensb;
  __shared__ double sm[NROW * PITCH];
  const int t = threadIdx.x;
  const int nn0 = op.L.nn[0], nn1 = op.L.nn[1], nn2 = op.L.nn[2];
  const int ne0 = op.ne[0], ne1 = op.ne[1], ne2 = op.ne[2];
  const int i0 = blockIdx.x * BX, j0 = blockIdx.y * BY, k0 = blockIdx.z * BZ;
  double dot = 0.0;
#pragma unroll
  for (int l = 0; l < NLD; ++l) {
    const int idx = t + l * NT;
    if (idx >= NRX * NROW) break;
    const int row = idx / NRX, q = idx - row * NRX;
    const int ry = row % (BY + 1), rz = row / (BY + 1);
    const int gi = i0 + q / 3, gj = j0 + ry, gk = k0 + rz;
    double v = 0.0;
    if (gi < nn0 && gj < nn1 && gk < nn2) {
      const long long g = 3 * (((long long)gk * nn1 + gj) * nn0 + i0) + q;
      v = __ldg(u + g);
      const bool own = (q < 3 * BX || gi == nn0 - 1) && (ry < BY || gj == nn1 - 1) && (rz < BZ || gk == nn2 - 1);
      if (f != nullptr && own) dot = fma(__ldg(f + g), v, dot);
    }
    sm[row * PITCH + q] = v;
  }
  __syncthreads();
  const int tx = t % BX, ty = (t / BX) % BY, tz = t / (BX * BY);
  const int ex = i0 + tx, ey = j0 + ty, ez = k0 + tz;
  if (ex < ne0 && ey < ne1 && ez < ne2) {
    double v[8][3];  // corner a = x + 2y + 4z
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const double* S = sm + ((tz + (a >> 2)) * (BY + 1) + ty + ((a >> 1) & 1)) * PITCH + 3 * (tx + (a & 1));
#pragma unroll
      for (int c = 0; c < 3; ++c) v[a][c] = S[c];
    }
#pragma unroll
    for (int b = 1; b < 8; b <<= 1)  // in-place Walsh-Hadamard: v[s] = sum_a (-1)^{popcount(s & a)} v[a]
#pragma unroll
      for (int a = 0; a < 8; ++a)
        if (!(a & b))
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const double x0 = v[a][c], x1 = v[a | b][c];
            v[a][c] = x0 + x1;
            v[a | b][c] = x0 - x1;
          }
    double s = 0.0;
#pragma unroll
    for (int chi = 0; chi < 8; ++chi)
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int mi = f3h::blk_member(chi, i);
        if (mi < 3) continue;  // the mean character: zero row
        double y = 0.0;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const int mj = f3h::blk_member(chi, j);
          if (f3h::blk_coef(chi, i, j) >= 0) y = fma(op.keh[f3h::blk_coef(chi, i, j)], v[mj / 3][mj % 3], y);
        }
        s = fma(v[mi / 3][mi % 3], y, s);
      }
    const long long e = ((long long)ez * ne1 + ey) * ne0 + ex;
    if (ce) ce[e] = s;
    if (dc) {
      const double r = __ldg(rho + e);
      dc[e] = -(p * (e0 - emin) * simp_pow_m1(r, p)) * s;
    }
  }
  if (f) grid_reduce(dot, red);
}

// ----------------------------------------------------------------------------
// ABI
// ----------------------------------------------------------------------------
extern "C" {

const char* tmg_last_error(void) { return g_err.c_str(); }
int tmg_version(void) { return 100; }
int64_t tmg_launch_count(void) { return launch_counter().load(); }
int tmg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int tmg_element_stiffness(const tmg_mesh_desc* mesh, double E, double nu, double* ke_host) {
  ABI_BEGIN
  check_mesh(mesh);
  TMG_REQUIRE(nu >= 0.0 && nu < 0.5, "nu must be in [0, 0.5)");
  TMG_REQUIRE(E > 0.0, "E must be positive");
  auto ke = element_stiffness(mesh->ndim, mesh->h, E, nu);
  std::memcpy(ke_host, ke.data(), ke.size() * sizeof(double));
  ABI_END
}

int tmg_simp_modulus(const double* rho_dev, int64_t n, double penalty, double e0, double emin, double* E_dev,
                     void* stream) {
  ABI_BEGIN
  require_device();
  DevBuf<unsigned> bad;
  bad.alloc(1, S(stream));
  bad.zero(S(stream));
  if (n > 0) { k_simp<<<grid_for(n), TPB, 0, S(stream)>>>(rho_dev, n, penalty, e0, emin, E_dev, bad.get()); ::tmg::note_launch(); }
  unsigned hb = 0;
  TMG_CUDA(cudaMemcpyAsync(&hb, bad.get(), sizeof(unsigned), cudaMemcpyDeviceToHost, S(stream)));
  TMG_CUDA(cudaStreamSynchronize(S(stream)));
  TMG_REQUIRE(hb == 0, "rho must lie in [0, 1]");
  ABI_END
}

int tmg_operator_create(const tmg_mesh_desc* mesh, const double* element_moduli_dev, const int64_t* fixed_dofs_host,
                        int64_t n_fixed, double nu, void* stream, tmg_operator** out) {
  ABI_BEGIN
  check_mesh(mesh);
  TMG_REQUIRE(nu >= 0.0 && nu < 0.5, "nu must be in [0, 0.5)");
  require_device();
  cudaStream_t s = S(stream);
  auto K = std::make_unique<tmg_operator>();
  Operator& o = K->op;
  o.dim = mesh->ndim;
  for (int d = 0; d < 3; ++d) {
    o.ne[d] = d < o.dim ? mesh->dims[d] : 1;
    o.h[d] = d < o.dim ? mesh->h[d] : 1.0;
    o.L.nn[d] = d < o.dim ? mesh->dims[d] + 1 : 1;
  }
  o.L.n = (long long)o.L.nn[0] * o.L.nn[1] * o.L.nn[2];
  o.nelem = (long long)o.ne[0] * o.ne[1] * (o.dim == 3 ? o.ne[2] : 1);
  o.ndof = o.L.n * o.dim;
  o.nu = nu;
  o.ke_host = element_stiffness(o.dim, o.h, 1.0, nu);
  if (o.dim == 3) {
    o.keh_host.assign(f3h::NZ, 0.0);
    // the box element's mirror symmetry puts KE in 8 character blocks (45 terms)
    TMG_REQUIRE(f3h::hat_coefficients(o.ke_host.data(), o.keh_host.data()) <= 1e-12,
                "element matrix lacks the mirror symmetry of a box element");
  }
  std::vector<uint8_t> mask(o.L.n, (uint8_t)((1u << o.dim) - 1u));
  for (int64_t t = 0; t < n_fixed; ++t) {
    const int64_t d = fixed_dofs_host[t];
    TMG_REQUIRE(d >= 0 && d < o.ndof, "fixed dof index out of range");
    mask[d / o.dim] &= (uint8_t)~(1u << (d % o.dim));
  }
  o.E.alloc(o.nelem, s);
  o.ke.alloc(o.ke_host.size(), s);
  o.mask.alloc(o.L.n, s);
  TMG_CUDA(cudaMemcpyAsync(o.E.get(), element_moduli_dev, o.nelem * sizeof(double), cudaMemcpyDeviceToDevice, s));
  TMG_CUDA(cudaMemcpyAsync(o.ke.get(), o.ke_host.data(), o.ke_host.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  TMG_CUDA(cudaMemcpyAsync(o.mask.get(), mask.data(), mask.size(), cudaMemcpyHostToDevice, s));
  DevBuf<unsigned> bad;
  bad.alloc(1, s);
  bad.zero(s);
  k_check_pos<<<grid_for(o.nelem), TPB, 0, s>>>(o.E.get(), o.nelem, bad.get()); ::tmg::note_launch();
  unsigned hb = 0;
  TMG_CUDA(cudaMemcpyAsync(&hb, bad.get(), sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  TMG_CUDA(cudaStreamSynchronize(s));  // also makes the pageable H2D sources safe to release
  TMG_REQUIRE(hb == 0, "element moduli must be positive");
  *out = K.release();
  ABI_END
}

int tmg_operator_destroy(tmg_operator* op) {
  ABI_BEGIN
  delete op;
  ABI_END
}

int64_t tmg_operator_size(const tmg_operator* op) { return op ? op->op.ndof : -1; }

int tmg_operator_apply(tmg_operator* K, const double* x, double* y, void* stream) {
  ABI_BEGIN
  TMG_REQUIRE(K, "operator is NULL");
  const Operator& o = K->op;
  if (o.dim == 2) {
    auto f = o.fine<2>();
    launch(k_apply<2, FineOp<2>>, row_grid<2, FineOp<2>>(o.L), row_block<2, FineOp<2>>(), row_smem<FineOp<2>>(), S(stream), f, x, y);
    ::tmg::note_launch();
  } else {
    auto f = o.fine<3>();
    launch(k_apply<3, FineOp<3>>, row_grid<3, FineOp<3>>(o.L), row_block<3, FineOp<3>>(), row_smem<FineOp<3>>(), S(stream), f, x, y);
    ::tmg::note_launch();
  }
  TMG_CUDA(cudaGetLastError());
  ABI_END
}

int tmg_operator_diagonal(tmg_operator* K, double* d, void* stream) {
  ABI_BEGIN
  TMG_REQUIRE(K, "operator is NULL");
  const Operator& o = K->op;
  DevBuf<unsigned> bad;
  bad.alloc(1, S(stream));
  bad.zero(S(stream));
  if (o.dim == 2) {
    auto f = o.fine<2>();
    k_diag<2, FineOp<2>><<<node_grid<2>(o.L), node_block<2>(), 0, S(stream)>>>(f, d, nullptr, bad.get()); ::tmg::note_launch();
  } else {
    auto f = o.fine<3>();
    k_diag<3, FineOp<3>><<<node_grid<3>(o.L), node_block<3>(), 0, S(stream)>>>(f, d, nullptr, bad.get()); ::tmg::note_launch();
  }
  TMG_CUDA(cudaGetLastError());
  ABI_END
}

// ndof0: rows of the finest level; keep: device copy of the sor_chebyshev power
// start vector (host or device input), alive for the build
static SmootherCfg to_cfg(const tmg_smoother_desc* d, long long ndof0, DevBuf<double>& keep, cudaStream_t s) {
  SmootherCfg c;
  if (d) {
    c.kind = d->kind;
    c.weight = d->weight;
    c.degree = d->inner_iterations;
    c.lanczos_steps = d->lanczos_steps > 0 ? d->lanczos_steps : 10;
    c.seed = d->seed;
    c.safeguard = d->safeguard;
  }
  TMG_REQUIRE(c.safeguard == 0.0 || (c.kind == SM_JACOBI && c.safeguard > 0.0 && c.safeguard < 2.0),
              "safeguard applies to weighted_jacobi only and must be in (0, 2)");
  TMG_REQUIRE(c.kind >= 0 && c.kind <= SM_SOR_GMRES, "unknown smoother kind");
  if (c.kind == SM_SOR_CHEBYSHEV) {
    TMG_REQUIRE(d->power_start != nullptr, "sor_chebyshev needs power_start (default_rng(0).standard_normal(ndofs))");
    keep.alloc(ndof0, s);
    TMG_CUDA(cudaMemcpyAsync(keep.get(), d->power_start, ndof0 * sizeof(double), cudaMemcpyDefault, s));
    c.power_start = keep.get();
  }
  TMG_REQUIRE(c.weight > 0.0 && c.weight <= 1.0, "smoother weight must be in (0, 1]");
  TMG_REQUIRE(c.degree >= 1, "inner_iterations must be >= 1");
  return c;
}

int tmg_gmg_build(tmg_operator* K, int64_t coarse_max_dofs, int32_t max_levels, const tmg_smoother_desc* smoother,
                  int32_t n_pre, int32_t n_post, void* stream, tmg_hierarchy** out) {
  ABI_BEGIN
  TMG_REQUIRE(K, "operator is NULL");
  TMG_REQUIRE(n_pre >= 0 && n_post >= 0, "n_pre/n_post must be >= 0");
  DevBuf<double> ps;
  const SmootherCfg c = to_cfg(smoother, K->op.ndof, ps, S(stream));
  auto H = std::make_unique<tmg_hierarchy>();
  H->K = K;
  if (K->op.dim == 2)
    H->h = build_gmg<2>(K->op, coarse_max_dofs, max_levels, c, n_pre, n_post, S(stream));
  else
    H->h = build_gmg<3>(K->op, coarse_max_dofs, max_levels, c, n_pre, n_post, S(stream));
  *out = H.release();
  ABI_END
}

int tmg_sa_amg_build(tmg_operator* K, const double* B_host, int32_t nvec, int64_t coarse_max_dofs, double beta,
                     const double* v0_host, const tmg_smoother_desc* smoother, int32_t n_pre, int32_t n_post,
                     int32_t isolated_mode, void* stream, tmg_hierarchy** out) {
  ABI_BEGIN
  TMG_REQUIRE(K && B_host && v0_host, "operator/near_nullspace/start vector is NULL");
  TMG_REQUIRE(isolated_mode == 0 || isolated_mode == 1, "isolated_mode must be 0 (merge) or 1 (drop)");
  TMG_REQUIRE(n_pre >= 0 && n_post >= 0, "n_pre/n_post must be >= 0");
  TMG_REQUIRE(nvec == 3 || nvec == 6, "near_nullspace must be (ndofs, 3) in 2D or (ndofs, 6) in 3D");
  cudaStream_t s = S(stream);
  DevBuf<double> ps;
  const SmootherCfg c = to_cfg(smoother, K->op.ndof, ps, s);
  const long long nd = K->op.ndof;
  DevBuf<double> B, v0;
  B.alloc(nd * nvec, s);
  v0.alloc(nd, s);
  // host or device pointers (unified addressing picks the direction)
  TMG_CUDA(cudaMemcpyAsync(B.get(), B_host, nd * nvec * sizeof(double), cudaMemcpyDefault, s));
  TMG_CUDA(cudaMemcpyAsync(v0.get(), v0_host, nd * sizeof(double), cudaMemcpyDefault, s));
  auto H = std::make_unique<tmg_hierarchy>();
  H->K = K;
  if (K->op.dim == 2)
    H->h = build_sa_amg<2>(K->op, B.get(), nvec, coarse_max_dofs, beta, v0.get(), c, n_pre, n_post,
                           isolated_mode == 1, s);
  else
    H->h = build_sa_amg<3>(K->op, B.get(), nvec, coarse_max_dofs, beta, v0.get(), c, n_pre, n_post,
                           isolated_mode == 1, s);
  TMG_CUDA(cudaStreamSynchronize(s));
  *out = H.release();
  ABI_END
}

int tmg_hybrid_build(tmg_operator* K, int32_t n_geo, const double* Bc_host, int64_t coarse_ndof, int32_t nvec,
                     int64_t coarse_max_dofs, double beta, const double* v0_host, const tmg_smoother_desc* smoother,
                     int32_t n_pre, int32_t n_post, int32_t isolated_mode, void* stream, tmg_hierarchy** out) {
  ABI_BEGIN
  TMG_REQUIRE(K && Bc_host && v0_host, "operator/near_nullspace/start vector is NULL");
  TMG_REQUIRE(isolated_mode == 0 || isolated_mode == 1, "isolated_mode must be 0 (merge) or 1 (drop)");
  TMG_REQUIRE(n_geo >= 1, "n_geo must be >= 1 (n_geo = 0 is build_sa_amg)");
  TMG_REQUIRE(n_pre >= 0 && n_post >= 0, "n_pre/n_post must be >= 0");
  TMG_REQUIRE(nvec == 3 || nvec == 6, "near_nullspace must be (ndofs, 3) in 2D or (ndofs, 6) in 3D");
  cudaStream_t s = S(stream);
  DevBuf<double> ps;
  const SmootherCfg c = to_cfg(smoother, K->op.ndof, ps, s);
  DevBuf<double> B, v0;
  B.alloc(coarse_ndof * nvec, s);
  v0.alloc(coarse_ndof, s);
  TMG_CUDA(cudaMemcpyAsync(B.get(), Bc_host, coarse_ndof * nvec * sizeof(double), cudaMemcpyDefault, s));
  TMG_CUDA(cudaMemcpyAsync(v0.get(), v0_host, coarse_ndof * sizeof(double), cudaMemcpyDefault, s));
  auto H = std::make_unique<tmg_hierarchy>();
  H->K = K;
  if (K->op.dim == 2)
    H->h = build_hybrid<2>(K->op, n_geo, B.get(), nvec, coarse_max_dofs, beta, v0.get(), c, n_pre, n_post,
                           coarse_ndof, isolated_mode == 1, s);
  else
    H->h = build_hybrid<3>(K->op, n_geo, B.get(), nvec, coarse_max_dofs, beta, v0.get(), c, n_pre, n_post,
                           coarse_ndof, isolated_mode == 1, s);
  TMG_CUDA(cudaStreamSynchronize(s));
  *out = H.release();
  ABI_END
}

int tmg_hierarchy_destroy(tmg_hierarchy* h) {
  ABI_BEGIN
  delete h;
  ABI_END
}

int tmg_hierarchy_num_levels(const tmg_hierarchy* h) { return h ? (int)h->h->lv.size() : -1; }

int tmg_hierarchy_level_info(const tmg_hierarchy* h, int32_t level, tmg_level_info* info) {
  ABI_BEGIN
  TMG_REQUIRE(h, "hierarchy is NULL");
  if (level < 0 || level >= (int)h->h->lv.size()) throw Error(TMG_ERANGE, "level index out of range");
  const Level& l = *h->h->lv[level];
  const int D = h->h->dim;
  info->size = l.ndof;
  info->provenance = h->h->provenance[level];
  if (level == h->h->last() && level > 0) {
    info->storage = 3;
    info->nonzeros = l.ndof * l.ndof;
  } else if (l.opkind == OP_FINE) {
    info->storage = 0;
    info->nonzeros = l.op->nelem;
  } else if (l.opkind == OP_STENCIL) {
    info->storage = 1;
    info->nonzeros = (D == 2 ? StencilOp<2>::NH : StencilOp<3>::NH) * (long long)D * D * l.L.n;  // symmetric: upper slots
  } else {
    info->storage = 2;
    info->nonzeros = l.Ab.scalar_nnz();
  }
  ABI_END
}

int tmg_hierarchy_flags(const tmg_hierarchy* h, char* buf, int32_t cap) {
  ABI_BEGIN
  TMG_REQUIRE(h && buf && cap > 0, "bad arguments");
  std::string s;
  for (const auto& f : h->h->flags) s += (s.empty() ? "" : ",") + f;
  std::strncpy(buf, s.c_str(), cap - 1);
  buf[cap - 1] = '\0';
  ABI_END
}

static void copy_bsr(const Bsr& m, int64_t* dims, int32_t* rowptr, int32_t* col, double* val, cudaStream_t s) {
  dims[0] = m.nrows;
  dims[1] = m.ncols;
  dims[2] = m.nnzb;
  dims[3] = (int64_t)m.R * 1000 + m.C;
  if (rowptr) TMG_CUDA(cudaMemcpyAsync(rowptr, m.rowptr.get(), (m.nrows + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
  if (col) TMG_CUDA(cudaMemcpyAsync(col, m.col.get(), m.nnzb * sizeof(int), cudaMemcpyDeviceToHost, s));
  if (val)
    TMG_CUDA(cudaMemcpyAsync(val, m.val.get(), m.nnzb * m.R * m.C * sizeof(double), cudaMemcpyDeviceToHost, s));
  TMG_CUDA(cudaStreamSynchronize(s));
}

int tmg_hierarchy_export(tmg_hierarchy* h, int32_t level, int32_t what, int64_t* dims, int32_t* rowptr, int32_t* col,
                         double* val, void* stream) {
  ABI_BEGIN
  TMG_REQUIRE(h && dims, "hierarchy/dims is NULL");
  if (level < 0 || level >= (int)h->h->lv.size()) throw Error(TMG_ERANGE, "level index out of range");
  Level& l = *h->h->lv[level];
  cudaStream_t s = S(stream);
  switch (what) {
    case 0: {  // level operator as BSR
      if (l.lattice()) {
        Bsr tmp;
        if (h->h->dim == 2) lattice_to_bsr<2>(l, tmp, s);
        else lattice_to_bsr<3>(l, tmp, s);
        copy_bsr(tmp, dims, rowptr, col, val, s);
      } else {
        copy_bsr(l.Ab, dims, rowptr, col, val, s);
      }
      break;
    }
    case 1:
      TMG_REQUIRE(l.xfer == XF_SPARSE, "level has no algebraic prolongation");
      copy_bsr(l.P, dims, rowptr, col, val, s);
      break;
    case 4:
      TMG_REQUIRE(l.xfer == XF_SPARSE, "level has no tentative prolongation");
      copy_bsr(l.Tm, dims, rowptr, col, val, s);
      break;
    case 2: {  // strength graph
      TMG_REQUIRE(l.xfer == XF_SPARSE, "level has no strength graph");
      const int n = (int)(l.ndof / l.bs);
      int nnz = 0;
      TMG_CUDA(cudaMemcpyAsync(&nnz, l.sptr.get() + n, sizeof(int), cudaMemcpyDeviceToHost, s));
      TMG_CUDA(cudaStreamSynchronize(s));
      dims[0] = n; dims[1] = n; dims[2] = nnz; dims[3] = 0;
      if (rowptr) TMG_CUDA(cudaMemcpyAsync(rowptr, l.sptr.get(), (n + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
      if (col && nnz) TMG_CUDA(cudaMemcpyAsync(col, l.scol.get(), nnz * sizeof(int), cudaMemcpyDeviceToHost, s));
      TMG_CUDA(cudaStreamSynchronize(s));
      break;
    }
    case 3: {  // aggregates
      TMG_REQUIRE(l.xfer == XF_SPARSE, "level has no aggregates");
      const int n = (int)(l.ndof / l.bs);
      dims[0] = n; dims[1] = l.n_agg; dims[2] = n; dims[3] = 0;
      if (col) TMG_CUDA(cudaMemcpyAsync(col, l.agg.get(), n * sizeof(int), cudaMemcpyDeviceToHost, s));
      if (val) TMG_CUDA(cudaMemcpyAsync(val, l.rho.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
      TMG_CUDA(cudaStreamSynchronize(s));
      break;
    }
    default:
      throw Error(TMG_EINVAL, "unknown export kind");
  }
  ABI_END
}

int tmg_hierarchy_vcycle(tmg_hierarchy* h, int32_t level, const double* b, double* x, void* stream) {
  ABI_BEGIN
  TMG_REQUIRE(h, "hierarchy is NULL");
  TMG_REQUIRE(!h->h->smoother_only, "a smoother-only hierarchy has no V-cycle");
  if (level < 0 || level >= (int)h->h->lv.size()) throw Error(TMG_ERANGE, "level index out of range");
  if (h->h->dim == 2) vcycle<2>(*h->h, level, b, x, S(stream));
  else vcycle<3>(*h->h, level, b, x, S(stream));
  TMG_CUDA(cudaGetLastError());
  ABI_END
}

int tmg_smoother_create(tmg_operator* K, const tmg_smoother_desc* smoother, void* stream, tmg_hierarchy** out) {
  ABI_BEGIN
  TMG_REQUIRE(K && out, "operator/out is NULL");
  cudaStream_t s = S(stream);
  DevBuf<double> ps;
  const SmootherCfg c = to_cfg(smoother, K->op.ndof, ps, s);
  auto H = std::make_unique<tmg_hierarchy>();
  H->K = K;
  if (K->op.dim == 2) H->h = build_smoother<2>(K->op, c, s);
  else H->h = build_smoother<3>(K->op, c, s);
  *out = H.release();
  ABI_END
}

int tmg_hierarchy_smooth(tmg_hierarchy* h, int32_t level, const double* b, double* x, int32_t passes,
                         void* stream) {
  ABI_BEGIN
  TMG_REQUIRE(h, "hierarchy is NULL");
  TMG_REQUIRE(passes >= 0, "passes must be >= 0");
  if (level < 0 || level >= (int)h->h->lv.size()) throw Error(TMG_ERANGE, "level index out of range");
  if (level == h->h->last() && !h->h->smoother_only) throw Error(TMG_ERANGE, "the coarsest level has no smoother");
  if (h->h->dim == 2) level_smooth<2>(*h->h, *h->h->lv[level], b, x, passes, S(stream));
  else level_smooth<3>(*h->h, *h->h->lv[level], b, x, passes, S(stream));
  TMG_CUDA(cudaGetLastError());
  ABI_END
}

int tmg_hierarchy_level_apply(tmg_hierarchy* h, int32_t level, const double* x, double* y, void* stream) {
  ABI_BEGIN
  TMG_REQUIRE(h, "hierarchy is NULL");
  if (level < 0 || level >= (int)h->h->lv.size()) throw Error(TMG_ERANGE, "level index out of range");
  if (h->h->dim == 2) lvl_apply<2>(*h->h->lv[level], x, y, S(stream));
  else lvl_apply<3>(*h->h->lv[level], x, y, S(stream));
  TMG_CUDA(cudaGetLastError());
  ABI_END
}

int tmg_hierarchy_level_lmax(tmg_hierarchy* h, int32_t level, double* lmax, void* stream) {
  ABI_BEGIN
  TMG_REQUIRE(h, "hierarchy is NULL");
  if (level < 0 || level >= (int)h->h->lv.size()) throw Error(TMG_ERANGE, "level index out of range");
  const Level& l = *h->h->lv[level];
  *lmax = std::nan("");
  if (l.lmax.get()) {
    TMG_CUDA(cudaMemcpyAsync(lmax, l.lmax.get(), sizeof(double), cudaMemcpyDeviceToHost, S(stream)));
    TMG_CUDA(cudaStreamSynchronize(S(stream)));
  }
  ABI_END
}

// reps enqueues of `body` captured into one CUDA graph on a private stream and
// timed as one replay (after a warm-up replay): the kernels run back to back as
// they do inside the PCG graph, without host launch overhead in the number.
extern "C++" {
template <class F>
static double time_graph(int reps, cudaStream_t user, F&& body) {
  cudaStream_t cs;
  TMG_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  TMG_CUDA(cudaStreamSynchronize(user));
  TMG_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  const long long c0 = launch_counter().load();
  for (int r = 0; r < reps; ++r) body(cs);
  note_launch(-(launch_counter().load() - c0));  // captured, counted when replayed
  cudaGraph_t g = nullptr;
  TMG_CUDA(cudaStreamEndCapture(cs, &g));
  cudaGraphExec_t ge = nullptr;
  TMG_CUDA(cudaGraphInstantiate(&ge, g, 0));
  cudaEvent_t a, b;
  TMG_CUDA(cudaEventCreate(&a));
  TMG_CUDA(cudaEventCreate(&b));
  TMG_CUDA(cudaGraphLaunch(ge, cs));
  TMG_CUDA(cudaEventRecord(a, cs));
  TMG_CUDA(cudaGraphLaunch(ge, cs));
  TMG_CUDA(cudaEventRecord(b, cs));
  TMG_CUDA(cudaEventSynchronize(b));
  float t = 0.f;
  TMG_CUDA(cudaEventElapsedTime(&t, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(cs);
  return (double)t / reps;
}
}  // extern "C++"

int tmg_hierarchy_time_smoother(tmg_hierarchy* h, int32_t level, int32_t reps, double* ms, void* stream) {
  ABI_BEGIN
  TMG_REQUIRE(h && reps > 0, "hierarchy is NULL or reps <= 0");
  if (level < 0 || level >= h->h->last()) throw Error(TMG_ERANGE, "level has no smoother");
  auto run = [&](auto dimtag) {
    constexpr int DIM = decltype(dimtag)::value;
    Hierarchy& H = *h->h;
    Level& l = *H.lv[level];
    const Red nored{nullptr, nullptr, nullptr};
    *ms = time_graph(reps, S(stream), [&](cudaStream_t cs) {
      if (sor_kind(H.sm.kind))  // the SOR triangular solve
        sor_solve(l, l.b.get(), l.xt.get(), cs);
      else if (H.sm.kind == SM_CHEBYSHEV)
        lvl_cheb_step<DIM>(l, l.r.get(), l.r.get(), l.dinv.get(), l.p.get(), 1, false, l.x.get(), l.pt.get(),
                           l.rt.get(), cs);
      else
        lvl_sweep<DIM, false>(H, l, l.b.get(), l.x.get(), l.xt.get(), nored, cs);
    });
  };
  if (h->h->dim == 2) run(std::integral_constant<int, 2>());
  else run(std::integral_constant<int, 3>());
  ABI_END
}

int tmg_hierarchy_time_vcycle(tmg_hierarchy* h, int32_t level, int32_t reps, double* ms, void* stream) {
  ABI_BEGIN
  TMG_REQUIRE(h && reps > 0, "hierarchy is NULL or reps <= 0");
  if (level < 0 || level > h->h->last()) throw Error(TMG_ERANGE, "level out of range");
  auto run = [&](auto dimtag) {
    constexpr int DIM = decltype(dimtag)::value;
    Hierarchy& H = *h->h;
    Level& l = *H.lv[level];
    *ms = time_graph(reps, S(stream), [&](cudaStream_t cs) { vcycle<DIM>(H, level, l.b.get(), l.x.get(), cs); });
  };
  if (h->h->dim == 2) run(std::integral_constant<int, 2>());
  else run(std::integral_constant<int, 3>());
  ABI_END
}

int tmg_hierarchy_time_phase(tmg_hierarchy* h, int32_t level, int32_t phase, int32_t reps, double* ms,
                             void* stream) {
  ABI_BEGIN
  TMG_REQUIRE(h && reps > 0, "hierarchy is NULL or reps <= 0");
  if (level < 0 || level > h->h->last()) throw Error(TMG_ERANGE, "level out of range");
  const bool coarse = level == h->h->last();
  if (coarse != (phase == TMG_PHASE_COARSE) || phase < 0 || phase > TMG_PHASE_COARSE)
    throw Error(TMG_ERANGE, "phase not defined on this level");
  auto run = [&](auto dimtag) {
    constexpr int DIM = decltype(dimtag)::value;
    Hierarchy& H = *h->h;
    Level& l = *H.lv[level];
    *ms = time_graph(reps, S(stream), [&](cudaStream_t cs) {
      switch (phase) {
        case TMG_PHASE_RESIDUAL: lvl_residual<DIM>(l, l.x.get(), l.b.get(), l.r.get(), cs); break;
        case TMG_PHASE_RESTRICT: xfer_restrict<DIM>(H, level, l.r.get(), nullptr, cs); break;
        case TMG_PHASE_PROLONG: xfer_prolong_add<DIM>(H, level, l.x.get(), cs); break;
        default: H.coarse.apply(l.b.get(), l.x.get(), cs); break;
      }
    });
  };
  if (h->h->dim == 2) run(std::integral_constant<int, 2>());
  else run(std::integral_constant<int, 3>());
  ABI_END
}

int tmg_gmres_solve(tmg_operator* K, tmg_hierarchy* h, const double* b, double* x, int32_t use_x0,
                    const tmg_gmres_desc* cfg, double* hist, tmg_solve_record* rec, void* stream) {
  ABI_BEGIN
  TMG_REQUIRE(K && cfg, "operator/config is NULL");
  TMG_REQUIRE(!h || !h->h->smoother_only, "a smoother-only hierarchy cannot precondition (no V-cycle)");
  Hierarchy* H = h ? h->h.get() : nullptr;
  if (h) TMG_REQUIRE(h->h->lv[0]->op == &K->op, "hierarchy was built for a different operator");
  GmresResult r = K->op.dim == 2
                      ? gmres_solve<2>(K->op, H, b, x, use_x0 != 0, cfg->rtol, cfg->max_iterations, cfg->restart,
                                       cfg->flexible != 0, S(stream))
                      : gmres_solve<3>(K->op, H, b, x, use_x0 != 0, cfg->rtol, cfg->max_iterations, cfg->restart,
                                       cfg->flexible != 0, S(stream));
  if (hist) std::copy(r.hist.begin(), r.hist.end(), hist);
  if (rec) {
    rec->iterations = r.iterations;
    rec->converged = r.converged;
    rec->initial_residual = r.hist.front();
    rec->final_residual = r.hist.back();
    rec->solve_ms = r.ms;
    rec->recursive_residual = r.hist.back();
    rec->restarts = 0;
    rec->reserved = 0;
  }
  ABI_END
}

int tmg_pcg_solve(tmg_operator* K, tmg_hierarchy* h, const double* b, double* x, int32_t use_x0,
                  const tmg_solve_desc* cfg, double* hist, tmg_solve_record* rec, void* stream) {
  ABI_BEGIN
  TMG_REQUIRE(K && cfg, "operator/config is NULL");
  TMG_REQUIRE(!h || !h->h->smoother_only, "a smoother-only hierarchy cannot precondition (no V-cycle)");
  Hierarchy* H = h ? h->h.get() : nullptr;
  if (h) TMG_REQUIRE(h->h->lv[0]->op == &K->op, "hierarchy was built for a different operator");
  std::unique_ptr<PcgCtx>& slot = h ? h->pcg : K->pcg;
  PcgResult r = K->op.dim == 2
                    ? pcg_solve<2>(slot, K->op, H, b, x, use_x0 != 0, cfg->rtol, cfg->max_iterations, S(stream))
                    : pcg_solve<3>(slot, K->op, H, b, x, use_x0 != 0, cfg->rtol, cfg->max_iterations, S(stream));
  if (rec) {
    rec->iterations = r.iterations;
    rec->converged = r.converged;
    rec->initial_residual = r.r0;
    rec->final_residual = r.rfinal;
    rec->solve_ms = r.ms;
    rec->recursive_residual = r.rrecursive;
    rec->restarts = r.restarts;
    rec->reserved = 0;
  }
  if (hist) std::memcpy(hist, r.hist.data(), r.hist.size() * sizeof(double));
  ABI_END
}

static unsigned sens_grid(long long nelem) { return std::min<unsigned>(grid_for(nelem), RED_BLOCKS * 4u); }
// 3D: 32 x 8 element-column tiles, z chunked so the grid is about four CTAs per SM
static dim3 sens3_grid(const Operator& o) {
  const unsigned gx = (o.ne[0] + sens3::TX - 1) / sens3::TX, gy = (o.ne[1] + sens3::TY - 1) / sens3::TY;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const unsigned want = std::max(1u, (4u * (unsigned)sms + gx * gy - 1) / (gx * gy));
  return dim3(gx, gy, std::min<unsigned>(want, (unsigned)std::max(1, o.ne[2])));
}
// 3D sensitivity kernel (TMG_SENS=gather|stream|brick): 0 per-element gather (k_sens<3>, default: 65 us on
// config 4), 1 z-streamed tiles (k_sens3: 87 us), 2 bricks staged in shared memory (k_sensb: 108 us) -- the two
// staged forms read u once and coalesced but run at 2-3 CTAs per SM; the gather at full occupancy hides its
// L1-served 8-fold node reuse better (profiles/r02_sens_ab.txt)
static int sens_mode(const Operator& o) {
  static const int mode = [] {
    const char* e = std::getenv("TMG_SENS");
    if (!e) return 0;
    return e[0] == 'b' ? 2 : (e[0] == 's' ? 1 : 0);
  }();
  return o.dim == 3 ? mode : 0;
}
static bool sens_streamed(const Operator& o) { return sens_mode(o) == 1; }
static dim3 sensb_grid(const Operator& o) {
  return dim3((o.ne[0] + sensb::BX - 1) / sensb::BX, (o.ne[1] + sensb::BY - 1) / sensb::BY,
              (o.ne[2] + sensb::BZ - 1) / sensb::BZ);
}

static void launch_sens(tmg_operator& K, const double* u, const double* f, double* ce, const double* rho, double p,
                        double e0, double emin, double* dc, cudaStream_t s) {
  const Operator& o = K.op;
  const int mode = sens_mode(o);
  const dim3 g3 = mode == 1 ? sens3_grid(o) : (mode == 2 ? sensb_grid(o) : dim3(1, 1, 1));
  const unsigned g = mode ? g3.x * g3.y * g3.z : sens_grid(o.nelem);
  if (f && K.sens.part.n < g) K.sens.alloc(g, s);
  const Red red = f ? K.sens.red() : Red{nullptr, nullptr, nullptr};
  if (mode == 1)
    launch(k_sens3, g3, sens3::NT, 0, s, o.fine<3>(), u, f, ce, rho, p, e0, emin, dc, red);
  else if (mode == 2)
    launch(k_sensb, g3, sensb::NT, 0, s, o.fine<3>(), u, f, ce, rho, p, e0, emin, dc, red);
  else if (o.dim == 2)
    launch(k_sens<2>, g, TPB, 0, s, o.fine<2>(), u, f, o.nelem, o.ndof, ce, rho, p, e0, emin, dc, red);
  else
    launch(k_sens<3>, g, TPB, 0, s, o.fine<3>(), u, f, o.nelem, o.ndof, ce, rho, p, e0, emin, dc, red);
  note_launch();
  TMG_CUDA(cudaGetLastError());
}

int tmg_strain_energy(tmg_operator* K, const double* u, double* ce, void* stream) {
  ABI_BEGIN
  TMG_REQUIRE(K, "operator is NULL");
  launch_sens(*K, u, nullptr, ce, nullptr, 1.0, 1.0, 0.0, nullptr, S(stream));
  ABI_END
}

// one launch: dc, and the compliance f.u (landed in pinned memory; the call
// returns it, so it waits for that one scalar -- no allocation per call)
int tmg_compliance_sensitivity(tmg_operator* K, const double* rho, const double* f, const double* u, double penalty,
                               double e0, double emin, double* dc, double* compliance, void* stream) {
  ABI_BEGIN
  TMG_REQUIRE(K, "operator is NULL");
  cudaStream_t s = S(stream);
  launch_sens(*K, u, compliance ? f : nullptr, nullptr, rho, penalty, e0, emin, dc, s);
  if (compliance) {
    if (!K->comp_host) TMG_CUDA(cudaMallocHost((void**)&K->comp_host, sizeof(double)));
    TMG_CUDA(cudaMemcpyAsync(K->comp_host, K->sens.res.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
    TMG_CUDA(cudaStreamSynchronize(s));
    *compliance = *K->comp_host;
  }
  ABI_END
}

// Average device time of the fused compliance + sensitivity kernel (bench.py's
// `sensitivity` roofline entry): `reps` launches in one CUDA graph, rotating over
// three copies of u and f so that consecutive launches stream them from HBM
// instead of finding them in the 126 MB L2.
int tmg_operator_time_sensitivity(tmg_operator* K, const double* rho, const double* f, const double* u,
                                  double penalty, double e0, double emin, double* dc, int32_t reps, double* ms,
                                  void* stream) {
  ABI_BEGIN
  TMG_REQUIRE(K && reps > 0, "operator is NULL or reps <= 0");
  cudaStream_t s = S(stream);
  const long long n = K->op.ndof;
  DevBuf<double> uc[2], fc[2];
  const double* us[3] = {u, nullptr, nullptr};
  const double* fs[3] = {f, nullptr, nullptr};
  for (int i = 0; i < 2; ++i) {
    uc[i].alloc(n, s);
    fc[i].alloc(n, s);
    TMG_CUDA(cudaMemcpyAsync(uc[i].get(), u, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    TMG_CUDA(cudaMemcpyAsync(fc[i].get(), f, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    us[i + 1] = uc[i].get();
    fs[i + 1] = fc[i].get();
  }
  int turn = 0;
  *ms = time_graph(reps, s, [&](cudaStream_t cs) {
    launch_sens(*K, us[turn % 3], fs[turn % 3], nullptr, rho, penalty, e0, emin, dc, cs);
    ++turn;
  });
  TMG_CUDA(cudaStreamSynchronize(s));
  ABI_END
}

int tmg_solve_compliance_host(const tmg_mesh_desc* mesh, const double* rho_host, const int64_t* fixed_host,
                              int64_t n_fixed, const double* f_host, double penalty, double e0, double emin,
                              double nu, const tmg_mg_desc* mg, const tmg_solve_desc* cfg, double* u_host,
                              double* dc_host, double* compliance_host, tmg_solve_record* rec) {
  ABI_BEGIN
  check_mesh(mesh);
  TMG_REQUIRE(mg && cfg, "mg/solve descriptor is NULL");
  TMG_REQUIRE(mg->strategy >= 0 && mg->strategy <= 2, "unknown preconditioner strategy");
  require_device();
  cudaStream_t s;
  TMG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamSynchronize(s); cudaStreamDestroy(s); }
  } guard{s};
  long long nel = 1, nnode = 1;
  for (int d = 0; d < mesh->ndim; ++d) { nel *= mesh->dims[d]; nnode *= mesh->dims[d] + 1; }
  const long long ndof = nnode * mesh->ndim;
  DevBuf<double> rho, E, f, u, dc;
  rho.alloc(nel, s); E.alloc(nel, s); f.alloc(ndof, s); u.alloc(ndof, s); dc.alloc(nel, s);
  TMG_CUDA(cudaMemcpyAsync(rho.get(), rho_host, nel * sizeof(double), cudaMemcpyHostToDevice, s));
  TMG_CUDA(cudaMemcpyAsync(f.get(), f_host, ndof * sizeof(double), cudaMemcpyHostToDevice, s));
  int rc = tmg_simp_modulus(rho.get(), nel, penalty, e0, emin, E.get(), s);
  if (rc) return rc;
  tmg_operator* K = nullptr;
  rc = tmg_operator_create(mesh, E.get(), fixed_host, n_fixed, nu, s, &K);
  if (rc) return rc;
  std::unique_ptr<tmg_operator> Kg(K);
  tmg_hierarchy* H = nullptr;
  if (mg->strategy == 0)
    rc = tmg_gmg_build(K, mg->coarse_max_dofs, mg->max_levels, &mg->smoother, mg->n_pre, mg->n_post, s, &H);
  else if (mg->strategy == 1)
    rc = tmg_sa_amg_build(K, mg->near_nullspace_host, mg->nvec, mg->coarse_max_dofs, mg->beta, mg->v0_host,
                          &mg->smoother, mg->n_pre, mg->n_post, mg->isolated_mode, s, &H);
  else
    rc = tmg_hybrid_build(K, mg->n_geo, mg->near_nullspace_host, mg->coarse_ndof, mg->nvec, mg->coarse_max_dofs,
                          mg->beta, mg->v0_host, &mg->smoother, mg->n_pre, mg->n_post, mg->isolated_mode, s, &H);
  if (rc) return rc;
  std::unique_ptr<tmg_hierarchy> Hg(H);
  TMG_REQUIRE(cfg->method >= 0 && cfg->method <= 2, "unknown Krylov method");
  // optimization.py:90-95: a non-stationary V-cycle (the SOR smoothers) is always
  // run under FGMRES; the PCG extension needs a stationary symmetric one
  const bool stationary = mg->smoother.kind <= 2;
  TMG_REQUIRE(stationary || cfg->method != 0, "PCG needs a stationary smoother (sor_* kinds need FGMRES)");
  if (cfg->method == 0) {
    rc = tmg_pcg_solve(K, H, f.get(), u.get(), 0, cfg, nullptr, rec, s);
  } else {
    const tmg_gmres_desc g{cfg->rtol, cfg->max_iterations, cfg->restart > 0 ? cfg->restart : 200,
                           (cfg->method == 2 || !stationary) ? 1 : 0};
    rc = tmg_gmres_solve(K, H, f.get(), u.get(), 0, &g, nullptr, rec, s);
  }
  if (rc) return rc;
  rc = tmg_compliance_sensitivity(K, rho.get(), f.get(), u.get(), penalty, e0, emin, dc.get(), compliance_host, s);
  if (rc) return rc;
  TMG_CUDA(cudaMemcpyAsync(u_host, u.get(), ndof * sizeof(double), cudaMemcpyDeviceToHost, s));
  TMG_CUDA(cudaMemcpyAsync(dc_host, dc.get(), nel * sizeof(double), cudaMemcpyDeviceToHost, s));
  TMG_CUDA(cudaStreamSynchronize(s));
  ABI_END
}

}  // extern "C"
