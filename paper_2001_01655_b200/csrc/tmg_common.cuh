// Common device/host plumbing for the B200 MG-PCG library.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace tmg {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define TMG_CUDA(x)                                                                    \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess)                                                             \
      throw ::tmg::Error(-3, std::string(#x) + " -> " + cudaGetErrorString(e_) + " @" + \
                                 __FILE__ + ":" + std::to_string(__LINE__));           \
  } while (0)

#define TMG_REQUIRE(cond, msg) \
  do {                         \
    if (!(cond)) throw ::tmg::Error(-1, msg); \
  } while (0)

constexpr int TPB = 256;  // threads per block for node-parallel kernels

// Count of this library's kernel launches (graph replays included), for the
// bench's gpu_launches claim.
inline std::atomic<long long>& launch_counter() {
  static std::atomic<long long> c{0};
  return c;
}
inline void note_launch(long long n = 1) { launch_counter().fetch_add(n, std::memory_order_relaxed); }

inline unsigned grid_for(long long n, int tpb = TPB) {
  long long g = (n + tpb - 1) / tpb;
  return (unsigned)(g < 1 ? 1 : g);
}

// Programmatic dependent launch.  Every kernel of the library starts with
// TMG_PDL_ENTRY: wait until the preceding grid in the stream has completed and
// its writes are visible (a no-op when launched without the PDL attribute), then
// allow the next grid to be scheduled.  launch() adds the attribute, so the
// next kernel's launch and block rasterisation overlap this kernel's tail -- the
// V-cycle is ~40 dependent kernels per PCG iteration, most of them short.
// TMG_PDL=0 disables the attribute (A/B switch).
#define TMG_PDL_ENTRY                                                  \
  do {                                                                 \
    asm volatile("griddepcontrol.wait;" ::: "memory");                 \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");    \
  } while (0)

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TMG_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
template <typename... KArgs, typename... Args>
inline void launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  if (smem > 48 * 1024)  // opt in to large dynamic shared memory (host-side attribute, capture-safe)
    TMG_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  TMG_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// Stream-ordered device buffer (cudaMallocAsync) -- setup never forces a device sync.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept { *this = std::move(o); }
  DevBuf& operator=(DevBuf&& o) noexcept {
    release();
    p = o.p; n = o.n; s = o.s;
    o.p = nullptr; o.n = 0;
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    if (count) TMG_CUDA(cudaMallocAsync((void**)&p, count * sizeof(T), st));
  }
  void zero(cudaStream_t st) {
    if (n) TMG_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), st));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  T* get() const { return p; }
};

// Node lattice of a structured level: nodes lexicographic with x fastest
// (reference mesh.py:65 node_index).  In 2D nn[2] == 1.
// Node ids are 32-bit (checked on the host: n * dofs_per_node < 2^31).
struct Lat {
  int nn[3];
  long long n;
  __host__ __device__ int id(int i, int j, int k) const { return i + nn[0] * (j + nn[1] * k); }
  __device__ void ijk(long long node, int& i, int& j, int& k) const {
    i = (int)(node % nn[0]);
    long long t = node / nn[0];
    j = (int)(t % nn[1]);
    k = (int)(t / nn[1]);
  }
  __host__ __device__ bool inside(int i, int j, int k) const {
    return i >= 0 && i < nn[0] && j >= 0 && j < nn[1] && k >= 0 && k < nn[2];
  }
};

// 2D/3D launch geometry: one thread per lattice node, no index division.
template <int DIM>
inline dim3 node_block() { return DIM == 2 ? dim3(32, 8, 1) : dim3(32, 4, 2); }
template <int DIM>
inline dim3 node_grid(const Lat& L) {
  const dim3 b = node_block<DIM>();
  return dim3((L.nn[0] + b.x - 1) / b.x, (L.nn[1] + b.y - 1) / b.y, (L.nn[2] + b.z - 1) / b.z);
}
inline unsigned node_blocks(const dim3& g) { return g.x * g.y * g.z; }

// Deterministic grid-wide reduction: per-block partials, the last block to
// finish sums them in a fixed order and publishes one scalar (no atomics on the
// value itself, so results are bitwise reproducible run to run).
struct Red {
  double* partials;   // >= gridDim.x entries
  unsigned* counter;  // zero-initialised, reset by the last block
  double* result;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// linear thread / block ids for 1D, 2D and 3D launches
__device__ __forceinline__ int lin_tid() { return threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z); }
__device__ __forceinline__ int lin_nthreads() { return blockDim.x * blockDim.y * blockDim.z; }
__device__ __forceinline__ unsigned lin_bid() { return blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z); }
__device__ __forceinline__ unsigned lin_nblocks() { return gridDim.x * gridDim.y * gridDim.z; }

// Block-level sum (thread count multiple of 32, <= 1024). Valid in linear thread 0.
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double ws[32];
  const int t = lin_tid();
  const int lane = t & 31, w = t >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) ws[w] = v;
  __syncthreads();
  const int nw = lin_nthreads() >> 5;
  v = (t < nw) ? ws[t] : 0.0;
  if (w == 0) v = warp_sum(v);
  return v;
}

// Every thread of every block must call this (uniform control flow).  fin(s)
// runs once, in thread 0 of the last block, after the result is published.
struct NoFinish {
  __device__ void operator()(double) const {}
};
template <class Fin = NoFinish>
__device__ __forceinline__ void grid_reduce(double v, const Red& r, Fin fin = Fin{}) {
  __shared__ bool last;
  const int t = lin_tid();
  const unsigned nb = lin_nblocks();
  double b = block_sum(v);
  if (t == 0) {
    r.partials[lin_bid()] = b;
    __threadfence();
    unsigned done = atomicAdd(r.counter, 1u);
    last = (done == nb - 1);
  }
  __syncthreads();
  if (last) {
    __threadfence();
    double s = 0.0;
    for (unsigned i = t; i < nb; i += lin_nthreads()) s += ((volatile double*)r.partials)[i];
    s = block_sum(s);
    if (t == 0) {
      *r.result = s;
      *r.counter = 0u;
      fin(s);
    }
  }
}

// Setup phase timer (TMG_VERBOSE=1: synchronises and prints per phase).
struct PhaseLog {
  bool on = false;
  cudaStream_t s;
  std::chrono::steady_clock::time_point t0;
  explicit PhaseLog(cudaStream_t st) : s(st) {
    const char* e = std::getenv("TMG_VERBOSE");
    on = e && e[0] == '1';
    t0 = std::chrono::steady_clock::now();
  }
  void mark(const char* what, long long a = -1) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[tmg] %-28s %9.3f ms  %lld\n", what,
                 std::chrono::duration<double, std::milli>(t - t0).count(), a);
    t0 = t;
  }
};

// A reduction slot with its own storage.
struct RedSlot {
  DevBuf<double> part;
  DevBuf<unsigned> cnt;
  DevBuf<double> res;
  void alloc(unsigned max_blocks, cudaStream_t s) {
    part.alloc(max_blocks, s);
    cnt.alloc(1, s);
    cnt.zero(s);
    res.alloc(1, s);
    res.zero(s);
  }
  Red red() const { return Red{part.get(), cnt.get(), res.get()}; }
};

}  // namespace tmg
