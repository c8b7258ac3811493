// common.cuh -- shared plumbing for the densegraph B200 library:
// status/exception mapping, the library stream, stream-ordered device
// buffers, splitmix64, exact 128-bit density compare, block scans and the
// grid barrier used by the persistent kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <new>
#include <stdexcept>
#include <string>
#include <utility>

#include "dg_b200.h"

namespace dgb {

constexpr uint32_t kNoVertex = 0xffffffffu;  // graph.hpp:12

struct DgError : std::runtime_error {
  dg_status code;
  DgError(dg_status c, const std::string& w) : std::runtime_error(w), code(c) {}
};

[[noreturn]] inline void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  char buf[512];
  snprintf(buf, sizeof buf, "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
           cudaGetErrorString(e), what, file, line);
  if (e == cudaErrorMemoryAllocation) throw DgError(DG_E_NOMEM, buf);
  throw DgError(DG_E_CUDA, buf);
}

#define DG_CUDA(call)                                                  \
  do {                                                                 \
    cudaError_t e_ = (call);                                           \
    if (e_ != cudaSuccess) ::dgb::throw_cuda(e_, #call, __FILE__, __LINE__); \
  } while (0)

void count_launch();
void set_last_error(const char* what);  // the thread's dg_last_error() text

// Every extern "C" entry point: exceptions never cross the ABI; the status
// code maps onto the reference's exception type and dg_last_error() holds
// the message.
#define DG_API_BEGIN try {
#define DG_API_END                                  \
  return DG_OK;                                     \
  }                                                 \
  catch (const ::dgb::DgError& e) {                 \
    ::dgb::set_last_error(e.what());                \
    return e.code;                                  \
  }                                                 \
  catch (const std::bad_alloc&) {                   \
    ::dgb::set_last_error("host allocation failed"); \
    return DG_E_NOMEM;                              \
  }                                                 \
  catch (const std::exception& e) {                 \
    ::dgb::set_last_error(e.what());                \
    return DG_E_INVARIANT;                          \
  }
#define DG_CHECK_LAUNCH()            \
  do {                               \
    DG_CUDA(cudaGetLastError());     \
    ::dgb::count_launch();           \
  } while (0)

// The library's stream on the current device (one per device, created
// lazily).  Every entry point enqueues on it and synchronises before
// returning, so calls are externally synchronous like the reference's.
cudaStream_t stream();
cudaMemPool_t mem_pool();  // the library's private stream-ordered pool
void trim_memory();        // release every cached block of mem_pool()
int num_sms();
void stream_sync();

// Stream-ordered device buffer (the library's private pool, library stream).
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr, o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p, n = o.n;
      o.p = nullptr, o.n = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    // +16 bytes of slack: kernels may read a whole 16-byte vector that
    // straddles the end of an array (e.g. the last adjacency quad)
    if (count)
      DG_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p), count * sizeof(T) + 16,
                                      mem_pool(), stream()));
  }
  void release() {
    if (p) cudaFreeAsync(p, stream());
    p = nullptr, n = 0;
  }
  void zero() {
    if (n) DG_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), stream()));
  }
  void fill_ff() {
    if (n) DG_CUDA(cudaMemsetAsync(p, 0xff, n * sizeof(T), stream()));
  }
  T* get() const { return p; }
};

template <class T>
inline void h2d(T* dst, const T* src, size_t count) {
  if (count) DG_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyHostToDevice, stream()));
}
template <class T>
inline void d2h(T* dst, const T* src, size_t count) {
  if (count) DG_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToHost, stream()));
}
template <class T>
inline void d2d(T* dst, const T* src, size_t count) {
  if (count)
    DG_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToDevice, stream()));
}
template <class T>
inline T read_scalar(const T* dptr) {
  T v;
  DG_CUDA(cudaMemcpyAsync(&v, dptr, sizeof(T), cudaMemcpyDeviceToHost, stream()));
  stream_sync();
  return v;
}

inline unsigned grid_for(uint64_t work, unsigned block, unsigned cap_per_sm = 8) {
  uint64_t g = (work + block - 1) / block;
  uint64_t cap = uint64_t(num_sms()) * cap_per_sm;
  if (g > cap) g = cap;
  return g ? unsigned(g) : 1u;
}

// ------------------------------------------------------------------ device helpers

// splitmix64 (reference parallel.hpp:92-97)
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// Exact Density compare a_e/a_v > b_e/b_v by 128-bit cross products
// (reference density.hpp:32-36).
__device__ __forceinline__ bool dens_gt(uint64_t ae, uint64_t av, uint64_t be, uint64_t bv) {
  uint64_t lhs_hi = __umul64hi(ae, bv), lhs_lo = ae * bv;
  uint64_t rhs_hi = __umul64hi(be, av), rhs_lo = be * av;
  return lhs_hi > rhs_hi || (lhs_hi == rhs_hi && lhs_lo > rhs_lo);
}
__device__ __forceinline__ bool dens_ge(uint64_t ae, uint64_t av, uint64_t be, uint64_t bv) {
  return !dens_gt(be, bv, ae, av);
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

template <class T>
__device__ __forceinline__ T warp_incl_scan(T x) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane_id() >= (unsigned)o) x += y;
  }
  return x;
}

template <class T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

template <class T>
__device__ __forceinline__ T warp_min(T x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    T y = __shfl_xor_sync(0xffffffffu, x, o);
    x = y < x ? y : x;
  }
  return x;
}

template <class T>
__device__ __forceinline__ T warp_max(T x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    T y = __shfl_xor_sync(0xffffffffu, x, o);
    x = y > x ? y : x;
  }
  return x;
}

// Block-wide exclusive scan of one value per thread; every thread calls it.
// `ws` is __shared__ scratch of >= 33 elements.  Returns the exclusive
// prefix; *total receives the block total.  Two __syncthreads.
template <class T>
__device__ __forceinline__ T block_excl_scan(T x, T* ws, T* total) {
  const unsigned w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  T inc = warp_incl_scan(x);
  if (lane_id() == 31) ws[w] = inc;
  __syncthreads();
  if (w == 0) {
    T v = lane_id() < nw ? ws[lane_id()] : T(0);
    T vi = warp_incl_scan(v);
    ws[lane_id()] = vi - v;
    if (lane_id() == 31) ws[32] = vi;
  }
  __syncthreads();
  T r = ws[w] + inc - x;
  *total = ws[32];
  return r;
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Sense-free generation barrier for a co-resident (cooperatively launched)
// grid.  Thread 0 of each CTA arrives with a release-ordered atomic and
// spins on the generation word with acquire loads.  A spin that exceeds
// `timeout_cycles` raises *abort (the kernel then unwinds instead of
// hanging the device).
struct GridBarrier {
  uint32_t count;
  uint32_t gen;
  uint32_t abort;
  uint32_t timeout_s;  // give up after ~timeout_s seconds of spinning (0: 60)
};

// Host side: the spin limit of grid barriers, DG_BARRIER_TIMEOUT_S (default
// 60 s; a debugger or compute-sanitizer may need more).
inline uint32_t barrier_timeout_s() {
  const char* e = getenv("DG_BARRIER_TIMEOUT_S");
  const long v = e ? atol(e) : 0;
  return v > 0 ? uint32_t(v) : 60u;
}

__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Only thread 0 of each CTA touches the barrier words; after the barrier it
// runs `fetch()` (e.g. loads the phase's global scalars into shared memory)
// so the rest of the CTA never hammers one L2 line.  *s_abort is a shared
// word the CTA reads after the closing __syncthreads.
template <class Fetch>
__device__ __forceinline__ bool grid_sync(GridBarrier* b, uint32_t nblocks, uint32_t* s_abort,
                                          Fetch fetch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    // One arrival word whose top bit flips when the last CTA arrives: CTA 0
    // adds 2^31 - (nblocks - 1), every other CTA adds 1, so the sum of one
    // barrier episode is exactly 2^31.  Waiters poll the same word; no reset
    // store, one atomic round trip on the critical path.
    const uint32_t add = blockIdx.x == 0 ? 0x80000000u - (nblocks - 1) : 1u;
    uint32_t old;  // release-ordered arrival, acquire-ordered polling: no full fences
    asm volatile("atom.add.release.gpu.u32 %0, [%1], %2;"
                 : "=r"(old)
                 : "l"(&b->count), "r"(add)
                 : "memory");
    const long long t0 = clock64();
    uint32_t spins = 0;
    while (((old ^ ld_acquire_u32(&b->count)) & 0x80000000u) == 0) {
      if ((++spins & 1023u) == 0) {
        if (ld_relaxed_u32(&b->abort)) break;
        const long long lim = (long long)(b->timeout_s ? b->timeout_s : 60u) << 31;
        if (clock64() - t0 > lim) {  // ~timeout_s seconds at 2 GHz: give up, do not hang
          atomicExch(&b->abort, 1u);
          break;
        }
      }
    }
    *s_abort = ld_relaxed_u32(&b->abort);
    fetch();
  }
  __syncthreads();
  return *s_abort == 0;
}

__device__ __forceinline__ bool grid_sync(GridBarrier* b, uint32_t nblocks, uint32_t* s_abort) {
  return grid_sync(b, nblocks, s_abort, [] {});
}

}  // namespace dgb
