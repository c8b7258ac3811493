#include <vector>
// microbench.cu -- latency floors that bound the per-round (k-core) and
// per-batch (Greedy++) costs on this B200: grid barrier, cooperative-groups
// grid.sync, cluster barrier, CTA barrier, dependent L2 load chain, shared
// atomics (spread / plain RMW).  Diagnostic only (dg_microbench).
#include <cooperative_groups.h>

#include "internal.cuh"
#include "dg_b200_diag.h"

namespace cg = cooperative_groups;

namespace dgb {
namespace {

__global__ void k_mb_grid(GridBarrier* b, uint64_t iters) {
  __shared__ uint32_t ab;
  for (uint64_t i = 0; i < iters; ++i)
    if (!grid_sync(b, gridDim.x, &ab)) break;
}

__global__ void k_mb_cg(uint64_t iters) {
  cg::grid_group g = cg::this_grid();
  for (uint64_t i = 0; i < iters; ++i) g.sync();
}

__global__ void __cluster_dims__(8, 1, 1) k_mb_cluster(uint64_t iters) {
  cg::cluster_group c = cg::this_cluster();
  for (uint64_t i = 0; i < iters; ++i) c.sync();
}

__global__ void k_mb_cluster_dyn(uint64_t iters) {  // cluster size from the launch
  cg::cluster_group c = cg::this_cluster();
  for (uint64_t i = 0; i < iters; ++i) c.sync();
}

__global__ void k_mb_bar(uint64_t iters, uint32_t* sink) {
  uint32_t x = threadIdx.x;
  for (uint64_t i = 0; i < iters; ++i) {
    __syncthreads();
    x = x * 1664525u + 1013904223u;
  }
  if (x == 7) *sink = x;
}

__global__ void k_mb_chase(const uint32_t* next, uint64_t iters, uint32_t* sink) {
  uint32_t p = 0;
  for (uint64_t i = 0; i < iters; ++i) p = next[p];
  *sink = p;
}

__global__ void k_mb_atoms(uint64_t iters, uint32_t* sink, int plain) {
  __shared__ uint32_t a[8192];
  for (uint32_t i = threadIdx.x; i < 8192; i += blockDim.x) a[i] = 0;
  __syncthreads();
  uint32_t idx = (threadIdx.x * 2654435761u) & 8191u;
  for (uint64_t i = 0; i < iters; ++i) {
    if (plain)
      a[idx] = a[idx] + 1;
    else
      atomicAdd(&a[idx], 1u);
    idx = (idx + 1031u) & 8191u;
  }
  __syncthreads();
  if (a[threadIdx.x] == 0xdeadbeef) *sink = 1;
}

// shared-memory primitives on one SM: 11 ATOMS with the result used (spread
// addresses, throughput per warp instruction, 32 warps), 12 LDS at spread
// addresses (throughput, 32 warps), 13 dependent LDS chain (latency, one
// warp), 14 dependent redux.sync chain (latency, one warp), 15 dependent
// ATOMS chain (latency, one warp)
__global__ void k_mb_smem(int mode, uint64_t iters, uint32_t* sink) {
  __shared__ uint32_t a[8192];
  for (uint32_t i = threadIdx.x; i < 8192; i += blockDim.x) a[i] = (i * 40503u + 7919u) & 8191u;
  __syncthreads();
  uint32_t idx = (threadIdx.x * 2654435761u) & 8191u, acc = 0;
  const uint32_t lane = threadIdx.x & 31;
  const long long t0 = clock64();
  for (uint64_t i = 0; i < iters; ++i) {
    if (mode == 11) {
      acc += atomicAdd(&a[idx], 1u);
      idx = (idx + 1031u) & 8191u;
    } else if (mode == 12) {
      acc += a[idx];
      idx = (idx + 1031u) & 8191u;
    } else if (mode == 13) {
      idx = a[(idx + lane) & 8191u];
    } else if (mode == 14) {
      idx = __reduce_min_sync(~0u, idx + lane) + 1u;
    } else {
      idx = (atomicAdd(&a[(idx + lane * 33u) & 8191u], 0u) + 1u) & 8191u;
    }
  }
  const long long t1 = clock64();
  if ((acc ^ idx) == 0xdeadbeefu) *sink = acc;
  if (threadIdx.x == 0) reinterpret_cast<unsigned long long*>(sink)[1] = (unsigned long long)(t1 - t0);
}

// throughput with 8 independent ops in flight per thread (32 warps, random
// bank-spread addresses): 16 LDS, 17 RED (no return), 18 ATOMS (return used
// after all 8 are issued)
__global__ void k_mb_smem_tp(int mode, uint64_t iters, uint32_t* sink) {
  __shared__ uint32_t a[8192];
  for (uint32_t i = threadIdx.x; i < 8192; i += blockDim.x) a[i] = i;
  __syncthreads();
  uint32_t x = threadIdx.x * 2654435761u + 12345u, acc = 0;
  const long long t0 = clock64();
  for (uint64_t i = 0; i < iters; ++i) {
    uint32_t idx[8], r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x = x * 1664525u + 1013904223u;
      idx[k] = x >> 19;  // random over 8192 words
    }
    if (mode == 16) {
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] = a[idx[k]];
    } else if (mode == 17) {
#pragma unroll
      for (int k = 0; k < 8; ++k) atomicAdd(&a[idx[k]], 1u);
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] = 0;
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] = atomicAdd(&a[idx[k]], 1u);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += r[k];
  }
  __syncthreads();
  const long long t1 = clock64();
  if (acc == 0xdeadbeefu) *sink = acc;
  if (threadIdx.x == 0) reinterpret_cast<unsigned long long*>(sink)[1] = (unsigned long long)(t1 - t0);
}

__global__ void k_mb_init_chase(uint32_t* next, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    next[i] = uint32_t((uint64_t(i) * 40503u + 7919u) % n);  // full-cycle-ish stride walk
}

}  // namespace
}  // namespace dgb

using namespace dgb;

extern "C" dg_status dg_microbench(int which, uint64_t iters, double* ns_per_op) {
  try {
    const bool g_mb_cycles = which >= 111 && which <= 118;  // 100 + mode: SM cycles per op
    if (g_mb_cycles) which -= 100;
    DevBuf<uint32_t> sink(4);  // [0] sink, [2..3] SM cycles of the timed loop (smem modes)
    cudaEvent_t e0, e1;
    DG_CUDA(cudaEventCreate(&e0));
    DG_CUDA(cudaEventCreate(&e1));
    const int sms = num_sms();
    DG_CUDA(cudaEventRecord(e0, stream()));
    if (which == 0) {
      DevBuf<GridBarrier> b(1);
      b.zero();
      void* p[] = {&b.p, &iters};
      DG_CUDA(cudaLaunchCooperativeKernel((void*)k_mb_grid, dim3(sms), dim3(1024), p, 0,
                                          stream()));
    } else if (which == 1) {
      void* p[] = {&iters};
      DG_CUDA(cudaLaunchCooperativeKernel((void*)k_mb_cg, dim3(sms), dim3(1024), p, 0, stream()));
    } else if (which == 2) {
      k_mb_cluster<<<8, 1024, 0, stream()>>>(iters);
    } else if (which == 3) {
      k_mb_bar<<<1, 1024, 0, stream()>>>(iters, sink.get());
    } else if (which == 4 || which == 7 || which == 8) {
      // 4 MiB (L2-resident), 64 MiB (half the L2), 1 GiB (HBM)
      const uint32_t n = which == 4 ? (1u << 20) : which == 7 ? (1u << 24) : (1u << 28);
      DevBuf<uint32_t> next(n);
      k_mb_init_chase<<<256, 256, 0, stream()>>>(next.get(), n);
      k_mb_chase<<<1, 1, 0, stream()>>>(next.get(), which == 4 ? 1000 : n / 4, sink.get());
      DG_CUDA(cudaEventRecord(e0, stream()));
      k_mb_chase<<<1, 1, 0, stream()>>>(next.get(), iters, sink.get());
    } else if (which == 9 || which == 10) {  // 16- / 4-CTA cluster barrier, 1024 threads
      const int cs = which == 9 ? 16 : 4;
      if (cs > 8)
        DG_CUDA(cudaFuncSetAttribute(k_mb_cluster_dyn,
                                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(1024);
      cfg.stream = stream();
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      DG_CUDA(cudaLaunchKernelEx(&cfg, k_mb_cluster_dyn, iters));
    } else if (which == 5 || which == 6) {
      k_mb_atoms<<<1, 1024, 0, stream()>>>(iters, sink.get(), which == 6);
    } else if (which >= 16 && which <= 18) {
      k_mb_smem_tp<<<1, 1024, 0, stream()>>>(which, iters, sink.get());
    } else if (which >= 11 && which <= 15) {
      k_mb_smem<<<1, which <= 12 ? 1024 : 32, 0, stream()>>>(which, iters, sink.get());
    } else {
      throw DgError(DG_E_PARAM, "unknown microbenchmark");
    }
    DG_CUDA(cudaGetLastError());
    DG_CUDA(cudaEventRecord(e1, stream()));
    stream_sync();
    float ms = 0;
    DG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    // per op: barriers per iteration; atomics per warp-instruction (32 lanes x 32 warps)
    double ops = double(iters);
    if (which == 5 || which == 6 || which == 11 || which == 12)
      ops = double(iters) * 32;  // warp instructions per SM
    if (which >= 16 && which <= 18) ops = double(iters) * 32 * 8;
    *ns_per_op = ms * 1e6 / ops;
    if (g_mb_cycles && which >= 11 && which <= 18) {
      unsigned long long cyc = 0;
      d2h(&cyc, reinterpret_cast<unsigned long long*>(sink.get()) + 1, 1);
      stream_sync();
      *ns_per_op = double(cyc) / ops;  // SM cycles per op instead of ns
    }
    return DG_OK;
  } catch (const DgError& e) {
    return e.code;
  }
}

extern "C" dg_status dg_peel_profile(uint64_t out[16]) {
  try {
    unsigned long long o[16];
    peel_profile(o);
    for (int i = 0; i < 16; ++i) out[i] = o[i];
    return DG_OK;
  } catch (const DgError& e) {
    return e.code;
  }
}

extern "C" dg_status dg_peel_trace_arm(uint32_t first_batch) {
  try {
    peel_trace_arm(first_batch);
    return DG_OK;
  } catch (const DgError& e) {
    return e.code;
  }
}

extern "C" dg_status dg_peel_trace_read(uint64_t* out) {
  try {
    std::vector<unsigned long long> o(kPeelTraceWords);
    peel_trace_read(o.data());
    for (size_t i = 0; i < kPeelTraceWords; ++i) out[i] = o[i];
    return DG_OK;
  } catch (const DgError& e) {
    return e.code;
  }
}

extern "C" dg_status dg_kcore_profile(uint64_t out[DG_KCORE_PROFILE_WORDS]) {
  try {
    static unsigned long long o[DG_KCORE_PROFILE_WORDS];
    kcore_profile(o);
    for (int i = 0; i < DG_KCORE_PROFILE_WORDS; ++i) out[i] = o[i];
    return DG_OK;
  } catch (const DgError& e) {
    return e.code;
  }
}

