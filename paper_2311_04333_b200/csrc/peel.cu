// peel.cu -- Greedy++ ordering and Algorithm 3 (reference refine.cpp).
//
// k_peel: the whole min-key batch chain of one iteration in ONE CTA
// (refine.cpp:20-156 semantics).  Keys (load - base + residual degree) live
// in shared memory when they fit (u32 keys when the key range allows, u64
// otherwise), so every batch is: CTA-wide min + ordered batch extraction
// (one barrier: warp min/count -> warp table -> every warp re-reduces the 32
// entries), then a load-balanced pass over the batch's adjacency lists that
// decrements alive neighbours' keys with shared-memory atomics and, fused,
// counts Algorithm 3's charge A[pos(v)] (= alive neighbours after v's batch
// + same-batch neighbours with a larger id, refine.cpp:195-199).  No host
// round trip and no global barrier per batch.
//
// k_alg3: suffix sums of A, first strict argmax of B[i]/(n-i) with exact
// 128-bit compares, width = max A, loads += A, the sampled slack audit on the
// pre-update loads, and the next iteration's key range -- one CTA.
#include <cub/cub.cuh>

#include <atomic>

#include "internal.cuh"
#include "peel_kernel.cuh"
#include "peel_cluster.cuh"
#include "peel_queue.cuh"

namespace dgb {

namespace {

constexpr int PT = 1024;  // peel CTA size
constexpr size_t kSmemCap = 227 * 1024;

}  // namespace

constexpr uint64_t kQueueMinN = 16384;
// batch mode: the cluster kernel from here up.  Measured us/batch, single CTA
// vs cluster: 9.1K vertices (RMAT-22) 1.62 / 1.66, 10.9K (RMAT-23) 2.28 / 1.71,
// 12.9K (RMAT-24) 2.31 / 1.77, 15.3K (RMAT-25) 2.63 / 1.79
constexpr uint64_t kClusterMinN = 9600;
// ... and smaller cores with long rows, whose removal one SM streams alone:
// Chung-Lu 50M's 6.6K core (average degree 2,301) 1.85 / 1.74, while RMAT-22's
// 9.1K core (1,373) stays on the single CTA
constexpr uint64_t kClusterDenseMinN = 4096, kClusterDenseDeg = 2000;
std::atomic<int> g_peel_mode{0};  // dg_set_peel_mode: 0 auto, 1 scanning single-CTA kernel, 2 cluster, 3 candidate list

namespace {

// ---- key range: min load, max (load - min + deg)
__global__ void k_key_range(const uint64_t* offs, const uint64_t* loads, uint64_t n,
                            unsigned long long* mn, unsigned long long* mx) {
  uint64_t lmin = ~0ULL;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    lmin = min(lmin, loads[i]);
  lmin = warp_min(lmin);
  if (lane_id() == 0) atomicMin(mn, (unsigned long long)lmin);
}
__global__ void k_key_max(const uint64_t* offs, const uint64_t* loads, uint64_t n,
                          const unsigned long long* mn, unsigned long long* mx) {
  const uint64_t base = *mn;
  uint64_t lmax = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    lmax = max(lmax, loads[i] - base + (offs[i + 1] - offs[i]));
  lmax = warp_max(lmax);
  if (lane_id() == 0) atomicMax(mx, (unsigned long long)lmax);
}

// ---- Algorithm 3 ----
struct A3Args {
  const uint64_t* offs;
  uint32_t n;
  const uint32_t* perm;
  const uint32_t* A;    // final charges, or
  const uint64_t* raw;  // raw fused-peel charges: A[i] = raw[i] - (loads[perm[i]] - base)
  uint64_t base;
  uint64_t* loads;
  uint64_t slack_samples, slack_allowed, slack_seed;
  uint64_t* suffix;
  Alg3Out* out;
  uint64_t* cs;  // scratch: the charges A[i], n entries
};

__device__ __forceinline__ bool better(uint64_t e1, uint64_t v1, uint64_t i1, uint64_t e2,
                                       uint64_t v2, uint64_t i2) {
  // strictly denser, or equally dense at a smaller position
  if (dens_gt(e1, v1, e2, v2)) return true;
  if (dens_gt(e2, v2, e1, v1)) return false;
  return i1 < i2;
}

__device__ __forceinline__ uint64_t charge(const A3Args& a, uint32_t i) {
  return a.A ? uint64_t(a.A[i]) : a.raw[i] - (a.loads[a.perm[i]] - a.base);
}

__global__ void __launch_bounds__(PT, 1) k_alg3(A3Args a) {
  __shared__ uint64_t ws[33];
  __shared__ uint64_t r_e[32], r_v[32], r_i[32], r_w[32], r_x[32], r_y[32];
  const uint32_t tid = threadIdx.x, lane = lane_id(), w = tid >> 5, nw = blockDim.x >> 5;
  const uint32_t n = a.n;
  // slack audit on the pre-update loads (refine.cpp:229-242)
  uint64_t bad = 0;
  if (n >= 2)
    for (uint64_t t = tid; t < a.slack_samples; t += blockDim.x) {
      uint64_t i = mix64(a.slack_seed ^ (2 * t + 1)) % n;
      uint64_t j = mix64(a.slack_seed ^ (2 * t + 2)) % n;
      if (i == j) continue;
      if (i > j) {
        uint64_t s = i;
        i = j;
        j = s;
      }
      if (a.loads[a.perm[i]] > a.loads[a.perm[j]] + a.slack_allowed) ++bad;
    }
  uint64_t badsum;
  block_excl_scan(bad, ws, &badsum);

  // the charges, once, position-strided (coalesced perm / raw reads, four
  // independent perm -> loads gathers in flight per thread) into scratch
  uint64_t wmax = 0;
  {
    uint32_t i = tid;
    for (; i + 3 * blockDim.x < n; i += 4 * blockDim.x) {
      uint64_t x[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) x[k] = charge(a, i + k * blockDim.x);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        a.cs[i + k * blockDim.x] = x[k];
        wmax = max(wmax, x[k]);
      }
    }
    for (; i < n; i += blockDim.x) {
      const uint64_t x = charge(a, i);
      a.cs[i] = x;
      wmax = max(wmax, x);
    }
  }
  __syncthreads();  // scratch written by the whole block

  // chunked suffix sums over the scratch copy
  const uint32_t c = (n + blockDim.x - 1) / blockDim.x;
  const uint32_t lo = min(n, tid * c), hi = min(n, lo + c);
  uint64_t local = 0;
  for (uint32_t i = lo; i < hi; ++i) local += a.cs[i];
  uint64_t total;
  const uint64_t ex = block_excl_scan(local, ws, &total);
  uint64_t run = total - ex - local;  // sum of A beyond my chunk
  uint64_t be = 0, bv = 1, bi = ~0ULL;
  for (uint32_t i = hi; i-- > lo;) {
    run += a.cs[i];
    if (a.suffix) a.suffix[i] = run;
    const uint64_t d = n - i;
    if (!dens_gt(be, bv, run, d)) {  // >= : walking down, smaller i wins ties
      be = run;
      bv = d;
      bi = i;
    }
  }
  // block argmax (tie -> smaller position), width
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    uint64_t e2 = __shfl_xor_sync(0xffffffffu, be, o);
    uint64_t v2 = __shfl_xor_sync(0xffffffffu, bv, o);
    uint64_t i2 = __shfl_xor_sync(0xffffffffu, bi, o);
    if (better(e2, v2, i2, be, bv, bi)) be = e2, bv = v2, bi = i2;
  }
  wmax = warp_max(wmax);
  if (lane == 0) r_e[w] = be, r_v[w] = bv, r_i[w] = bi, r_w[w] = wmax;
  __syncthreads();
  if (w == 0) {
    be = lane < nw ? r_e[lane] : 0;
    bv = lane < nw ? r_v[lane] : 1;
    bi = lane < nw ? r_i[lane] : ~0ULL;
    uint64_t wm = lane < nw ? r_w[lane] : 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      uint64_t e2 = __shfl_xor_sync(0xffffffffu, be, o);
      uint64_t v2 = __shfl_xor_sync(0xffffffffu, bv, o);
      uint64_t i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      if (better(e2, v2, i2, be, bv, bi)) be = e2, bv = v2, bi = i2;
    }
    wm = warp_max(wm);
    if (lane == 0) {
      if (be == 0) {  // every suffix has density 0: rho stays {0,1} at prefix 0
        a.out->rho_edges = 0;
        a.out->rho_verts = 1;
        a.out->best_prefix = 0;
      } else {
        a.out->rho_edges = be;
        a.out->rho_verts = bv;
        a.out->best_prefix = bi;
      }
      a.out->width = wm;
      a.out->total = total;
      a.out->slack_bad = badsum;
    }
  }
  // loads += A (refine.cpp:213); every position's vertex is distinct, and
  // every charge was read before this point (the barrier above the scan)
  for (uint32_t i = tid; i < n; i += blockDim.x) a.loads[a.perm[i]] += a.cs[i];
  __syncthreads();
  // next key range over vertices
  uint64_t mn = ~0ULL;
  for (uint32_t v = tid; v < n; v += blockDim.x) mn = min(mn, a.loads[v]);
  mn = warp_min(mn);
  if (lane == 0) r_x[w] = mn;
  __syncthreads();
  if (w == 0) {
    uint64_t x = lane < nw ? r_x[lane] : ~0ULL;
    x = warp_min(x);
    if (lane == 0) r_x[0] = x;
  }
  __syncthreads();
  const uint64_t base = r_x[0];
  uint64_t mk = 0;
  for (uint32_t v = tid; v < n; v += blockDim.x)
    mk = max(mk, a.loads[v] - base + (a.offs[v + 1] - a.offs[v]));
  mk = warp_max(mk);
  if (lane == 0) r_y[w] = mk;
  __syncthreads();
  if (w == 0) {
    uint64_t x = lane < nw ? r_y[lane] : 0;
    x = warp_max(x);
    if (lane == 0) {
      a.out->min_load = n ? base : 0;
      a.out->max_key = x;
    }
  }
}

// ---- charges from an arbitrary permutation (refine.cpp:186-199)
__global__ void k_pos_from_perm(const uint32_t* perm, uint64_t n, uint64_t* pos, uint32_t* err) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t v = perm[i];
    if (v >= n) {
      *err = 1;
      continue;
    }
    unsigned long long old =
        atomicCAS(reinterpret_cast<unsigned long long*>(&pos[v]), ~0ULL, (unsigned long long)i);
    if (old != ~0ULL) *err = 1;
  }
}

// A[pos(v)] = #neighbours positioned after v (refine.cpp:195-199: every edge
// charged to its earlier endpoint): a warp per row counts them and writes its
// own position -- no atomics, no zero fill
template <class P>
__global__ void k_charges_rows(const uint64_t* offs, const uint32_t* adj, uint64_t n,
                               const P* pos, uint32_t* A) {
  const uint64_t warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t v = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; v < n; v += warps) {
    const P pv = pos[v];
    uint32_t c = 0;
    for (uint64_t p = offs[v] + lane_id(); p < offs[v + 1]; p += 32) c += pos[adj[p]] > pv;
    c = __reduce_add_sync(~0u, c);
    if (lane_id() == 0) A[pv] = c;
  }
}

__global__ void k_pos32(const uint32_t* perm, uint64_t n, uint32_t* pos) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    pos[perm[i]] = uint32_t(i);
}

__global__ void k_sort_keys32(const uint64_t* loads, uint64_t n, uint64_t base, uint32_t* keys) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    keys[i] = uint32_t(loads[i] - base);
}

__global__ void k_iota(uint32_t* p, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    p[i] = uint32_t(i);
}

unsigned long long* peel_prof_buffer() {
  static unsigned long long* buf[64] = {};
  int d = 0;
  DG_CUDA(cudaGetDevice(&d));
  if (!buf[d]) {
    constexpr size_t N = 16 + kPeelTraceWords;  // counters, then the armed timeline
    DG_CUDA(cudaMalloc(&buf[d], N * sizeof(unsigned long long)));
    DG_CUDA(cudaMemset(buf[d], 0, N * sizeof(unsigned long long)));
  }
  return buf[d];
}

bool g_peel_trace_armed[64] = {};  // dg_peel_trace_arm: launch the timeline variant

bool peel_trace_armed() {
  int d = 0;
  DG_CUDA(cudaGetDevice(&d));
  return g_peel_trace_armed[d];
}

template <class K, bool SMEM, bool OFFS, int VQ, bool TR = false, bool SMALL = false>
void launch_peel(const dg_graph& g, const uint64_t* d_loads, uint64_t base, bool one,
                 uint32_t chunk, uint32_t* d_perm, uint64_t* d_raw,
                 unsigned long long* d_batches) {
  // just enough warps to hold the keys: idle warps still issue the
  // per-warp table reduction of every batch (RMAT-22's 9.1K core: 24 warps
  // instead of 32, 1.95 -> 1.85 us per batch)
  const uint64_t wkeys = uint64_t(chunk) * 32;
  const uint32_t nt = uint32_t(
      std::min<uint64_t>(peelk::PT, std::max<uint64_t>(1, (g.n + wkeys - 1) / wkeys) * 32));
  DevBuf<K> gk;
  if (!SMEM) gk.alloc(size_t(chunk) * nt);
  const size_t smem = peelk::smem_bytes<K, OFFS>(chunk, SMEM, nt);
  auto kern = peelk::k_peel<K, SMEM, OFFS, VQ, TR, SMALL ? 768 : peelk::PT>;
  if (TR)  // timeline of this launch only
    DG_CUDA(cudaMemsetAsync(peel_prof_buffer() + 16, 0, kPeelTraceWords * 8, stream()));
  DG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  peelk::Args<K> a{g.offs.get(), g.adj.get(), uint32_t(g.n), d_loads, base, one ? 1 : 0,
                   gk.get(), chunk, d_perm, d_raw, d_batches, peel_prof_buffer()};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream();
  DG_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  DG_CHECK_LAUNCH();
}

// u32 keys in shared memory: compile-time chunk of 4*VQ keys (VQ odd)
template <bool OFFS>
bool launch_vec(const dg_graph& g, const uint64_t* d_loads, uint64_t base, bool one, uint32_t vq,
                uint32_t* d_perm, uint64_t* d_raw, unsigned long long* d_batches) {
  switch (vq) {
#define DG_VQ(V)                                                                         \
  case V:                                                                                \
    if (OFFS && peel_trace_armed())                                                      \
      launch_peel<uint32_t, true, OFFS, V, OFFS>(g, d_loads, base, one, 4 * V, d_perm,   \
                                                 d_raw, d_batches);                      \
    else if (g.n <= 768ULL * V * 4)                                                      \
      launch_peel<uint32_t, true, OFFS, V, false, true>(g, d_loads, base, one, 4 * V,    \
                                                        d_perm, d_raw, d_batches);       \
    else                                                                                 \
      launch_peel<uint32_t, true, OFFS, V>(g, d_loads, base, one, 4 * V, d_perm, d_raw,  \
                                           d_batches);                                   \
    return true;
    DG_VQ(1) DG_VQ(3) DG_VQ(5) DG_VQ(7) DG_VQ(9) DG_VQ(11) DG_VQ(13)
#undef DG_VQ
    default:
      return false;
  }
}

// Candidate-list kernel (batch mode, u32 keys): smallest odd VQ covering n
template <bool OFFS, int VQ, bool TR = false>
bool launch_queue1(const dg_graph& g, const uint64_t* d_loads, uint64_t base, uint32_t* d_perm,
                   uint64_t* d_raw, unsigned long long* d_batches) {
  constexpr size_t smem = peelq::smem_bytes<VQ, OFFS>();
  if (smem > kSmemCap) return false;
  auto kern = peelq::k_peel_queue<OFFS, VQ, TR>;
  if (TR)  // timeline of this launch only
    DG_CUDA(cudaMemsetAsync(peel_prof_buffer() + 16, 0, kPeelTraceWords * 8, stream()));
  DG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  peelq::Args a{g.offs.get(), g.adj.get(), uint32_t(g.n), d_loads, base,
                d_perm,       d_raw,       d_batches,     peel_prof_buffer()};
  kern<<<1, peelq::PT, smem, stream()>>>(a);
  DG_CHECK_LAUNCH();
  return true;
}

template <bool OFFS>
bool launch_queue(const dg_graph& g, const uint64_t* d_loads, uint64_t base, uint32_t vq,
                  uint32_t* d_perm, uint64_t* d_raw, unsigned long long* d_batches) {
  switch (vq) {
#define DG_VQ(V)                                                                        \
  case V:                                                                               \
    return peel_trace_armed()                                                           \
               ? launch_queue1<OFFS, V, true>(g, d_loads, base, d_perm, d_raw, d_batches) \
               : launch_queue1<OFFS, V>(g, d_loads, base, d_perm, d_raw, d_batches);
    DG_VQ(1) DG_VQ(3) DG_VQ(5) DG_VQ(7) DG_VQ(9)
#undef DG_VQ
    default:
      return false;
  }
}

}  // namespace

KeyRange key_range(const dg_graph& g, const uint64_t* d_loads) {
  KeyRange kr;
  if (!g.n) return kr;
  DevBuf<unsigned long long> mm(2);
  unsigned long long init[2] = {~0ULL, 0ULL};
  h2d(mm.get(), init, 2);
  k_key_range<<<grid_for(g.n, 256), 256, 0, stream()>>>(g.offs.get(), d_loads, g.n, mm.get(),
                                                        mm.get() + 1);
  DG_CHECK_LAUNCH();
  k_key_max<<<grid_for(g.n, 256), 256, 0, stream()>>>(g.offs.get(), d_loads, g.n, mm.get(),
                                                      mm.get() + 1);
  DG_CHECK_LAUNCH();
  unsigned long long h[2];
  d2h(h, mm.get(), 2);
  stream_sync();
  kr.min_load = h[0];
  kr.max_key = h[1];
  return kr;
}

// Per-row CTA slices for the cluster kernel: seg[v*(CS+1) + r] = index
// inside row v of its first neighbour >= r * no (rows ascend; CTA r owns ids
// [r*no, (r+1)*no)), one thread per (row, r) by binary search.
template <int CS>
__global__ void k_seg_table(const uint64_t* offs, const uint32_t* adj, uint64_t n, uint32_t no,
                            uint32_t* seg) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n * (CS + 1);
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t v = i / (CS + 1);
    const uint32_t r = uint32_t(i % (CS + 1));
    const uint64_t o0 = offs[v];
    uint32_t lo = 0, hi = uint32_t(offs[v + 1] - o0);
    if (r == 0) {
      hi = 0;
    } else if (r < CS) {
      const uint32_t x = r * no;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (adj[o0 + mid] < x) lo = mid + 1; else hi = mid;
      }
    }
    seg[i] = hi;
  }
}

// Cluster variant: returns false when no cluster configuration fits.
template <int CS, int PT>
bool launch_cluster_pt(const dg_graph& g, const uint64_t* d_loads, uint64_t base, bool one,
                       uint32_t nc, uint32_t no, uint32_t* d_perm, uint64_t* d_raw,
                       unsigned long long* d_batches) {
  const uint64_t n = g.n;
  const bool offs32 = 2 * g.m < 0xffffffffULL;
  // 64-bit row offsets in the kernel (DG_CLUSTER_O64=1 forces them: tests)
  const bool o64 = 2 * g.m + 64 >= 0xffffffffULL || getenv("DG_CLUSTER_O64");
  bool offs_smem = offs32 && peelc::smem_bytes(nc, true) <= kSmemCap;
  if (!offs_smem && peelc::smem_bytes(nc, false) > kSmemCap) return false;
  // every row's slice bounds in shared memory when they fit (rows < 2^16 arcs)
  const bool slice_smem = PT == 512 && g.maxdeg < 65536 &&
                          peelc::smem_bytes(nc, offs_smem, n) <= kSmemCap &&
                          !getenv("DG_NO_SLICE_SMEM");
  // slice cache: 16 slots of up to 256 quads (4 KB) in what shared memory is left
  uint32_t slotq = 0;
  if (slice_smem && !getenv("DG_NO_SLICE_CACHE"))
    for (uint32_t q = getenv("DG_SLICE_SLOTQ") ? atoi(getenv("DG_SLICE_SLOTQ")) : 256;
         q >= 32 && !slotq; q >>= 1)
      if (peelc::smem_bytes(nc, offs_smem, n, q) <= kSmemCap) slotq = q;
  const size_t smem = peelc::smem_bytes(nc, offs_smem, slice_smem ? n : 0, slotq);
  auto kern = o64 ? peelc::k_peel_cluster<CS, PT, true> : peelc::k_peel_cluster<CS, PT, false>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) !=
      cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (CS > 8 &&
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
          cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS);
  cfg.blockDim = dim3(PT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream();
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) != cudaSuccess || nclusters < 1) {
    cudaGetLastError();
    return false;
  }
  // raw charges are accumulated with atomics (see peel_cluster.cuh)
  DG_CUDA(cudaMemsetAsync(d_raw, 0, n * sizeof(uint64_t), stream()));
  DevBuf<uint32_t> seg(n * (CS + 1));
  k_seg_table<CS><<<grid_for(n * (CS + 1), 256), 256, 0, stream()>>>(g.offs.get(), g.adj.get(), n,
                                                                      no, seg.get());
  DG_CHECK_LAUNCH();
  peelc::Args a{g.offs.get(), g.adj.get(), uint32_t(n), d_loads, base, one ? 1 : 0,
                nc, nc / PT, no, offs_smem ? 1 : 0, d_perm, d_raw, seg.get(),
                slice_smem ? 1 : 0, slotq, d_batches, peel_prof_buffer()};
  DG_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  count_launch();
  return true;
}

// CTA size by block size (see below); DG_CLUSTER_PT=512|1024 overrides (tuning).
template <int CS>
bool launch_cluster(const dg_graph& g, const uint64_t* d_loads, uint64_t base, bool one,
                    uint32_t* d_perm, uint64_t* d_raw, unsigned long long* d_batches) {
  // NO = ceil(n / CS) ids owned per CTA, in NC key slots (the smallest
  // multiple of the CTA size covering NO), so every CTA of the cluster holds
  // the same share of the vertices (NO rounded up to a multiple of the CTA
  // size left 4 of 16 CTAs empty on RMAT-26's 17.9K core, and power-of-two
  // blocks 7); DG_CLUSTER_POW2=1 restores power-of-two blocks.
  uint64_t per_cta = (g.n + CS - 1) / CS;
  // 512-thread CTAs while their keys fit S1's 8-key register tier, 1024
  // beyond (RMAT-26's 84K core, 5.2K ids per CTA: 3.50 us/batch at 1024 with
  // 6 keys per thread in registers vs 3.55 at 512 with 11 keys reloaded)
  int pt = per_cta <= 4096 ? 512 : 1024;
  if (const char* e = getenv("DG_CLUSTER_PT")) pt = atoi(e) == 512 ? 512 : 1024;
  uint64_t c = (per_cta + pt - 1) / pt;  // keys per thread
  // an odd number of keys per thread: S1's scalar shared loads at an even
  // word stride hit each bank from 2 (4 at stride 4) lanes of the warp
  // (ncu on the 84K core at 6 keys: 52 % of its shared wavefronts were
  // excess); 8 stays (the two-vector tier)
  if (c < 8 && (c & 1) == 0 && !getenv("DG_CLUSTER_EVEN")) ++c;
  if (getenv("DG_CLUSTER_POW2") && getenv("DG_CLUSTER_POW2")[0] == '1') {
    uint64_t nc = 512;
    while (nc * CS < g.n) nc *= 2;
    if (nc < uint64_t(pt)) nc = pt;
    c = nc / pt;
    per_cta = nc;
  }
  if (c > 32) return false;  // <= 32 keys per thread (the S1 match mask)
  const uint32_t nc = uint32_t(c * pt);
  if (getenv("DG_CLUSTER_NCOWN") && getenv("DG_CLUSTER_NCOWN")[0] == '1') per_cta = nc;
  const uint32_t no = uint32_t(per_cta);
  if (pt == 512)
    return launch_cluster_pt<CS, 512>(g, d_loads, base, one, nc, no, d_perm, d_raw, d_batches);
  return launch_cluster_pt<CS, 1024>(g, d_loads, base, one, nc, no, d_perm, d_raw, d_batches);
}

void peel_order(const dg_graph& g, const uint64_t* d_loads, const KeyRange& kr,
                bool one_at_a_time, uint32_t* d_perm, uint64_t* d_raw,
                unsigned long long* d_batches) {
  if (g.n == 0) return;
  const uint32_t n = uint32_t(g.n);
  const uint32_t per = (n + peelk::PT - 1) / peelk::PT;
  // alive keys must stay below 2^(bits-1) and degrees below 2^28 (see the
  // key ranges in peel_kernel.cuh)
  if (g.maxdeg >= (1ULL << 28)) throw DgError(DG_E_PARAM, "degree too large for the peel kernel");
  if (kr.max_key >= (1ULL << 62)) throw DgError(DG_E_PARAM, "load range exceeds 2^62");
  const bool k32 = kr.max_key < 0x80000000ULL;
  // u32 keys in shared memory are scanned with 128-bit loads: chunk = 4q with
  // q odd keeps a warp's vector loads bank-conflict free; otherwise an odd
  // chunk keeps scalar scans conflict free.
  const uint32_t vq = ((per + 3) / 4) | 1u;
  const uint32_t chunk_odd = per | 1u;
  const bool offs32 = 2 * g.m < 0xffffffffULL;
  const uint64_t base = kr.min_load;
  // Cores whose u32 keys + offsets do not fit one SM: a 16- (or 8-) CTA cluster
  // with the keys spread over distributed shared memory.
  // Preference: one CTA with u32 keys in shared memory (fastest per batch);
  // when the core's keys do not fit one SM, a 16- (or 8-) CTA cluster with the
  // keys spread over distributed shared memory; then the u64 / global-key
  // single-CTA fallbacks.  dg_set_peel_mode can force either kernel.
  // batch mode beyond kQueueMinN: the cluster kernel (RMAT-22's 35K core
  // 3.52 vs 4.22 us per batch for the candidate-list kernel, RMAT-26's 17.9K
  // core 2.98 vs 3.20), the candidate-list kernel when no cluster fits
  const int mode = g_peel_mode.load(std::memory_order_relaxed);
  const bool dense_mid = g.n > kClusterDenseMinN && 2 * g.m >= kClusterDenseDeg * g.n;
  if (k32 && !one_at_a_time && mode == 0 && (g.n > kClusterMinN || dense_mid)) {
    // DG_CLUSTER_CS=8 prefers the 8-CTA cluster (tuning)
    static const bool pref8 = getenv("DG_CLUSTER_CS") && atoi(getenv("DG_CLUSTER_CS")) == 8;
    if (pref8 && launch_cluster<8>(g, d_loads, base, false, d_perm, d_raw, d_batches)) return;
    if (launch_cluster<16>(g, d_loads, base, false, d_perm, d_raw, d_batches)) return;
    if (launch_cluster<8>(g, d_loads, base, false, d_perm, d_raw, d_batches)) return;
  }
  if (k32 && !one_at_a_time &&
      ((mode == 0 && g.n > kQueueMinN) || mode == 3)) {
    if (offs32 && launch_queue<true>(g, d_loads, base, vq, d_perm, d_raw, d_batches)) return;
    if (launch_queue<false>(g, d_loads, base, vq, d_perm, d_raw, d_batches)) return;
  }
  if (k32 && mode == 2) {
    if (launch_cluster<16>(g, d_loads, base, one_at_a_time, d_perm, d_raw, d_batches)) return;
    if (launch_cluster<8>(g, d_loads, base, one_at_a_time, d_perm, d_raw, d_batches)) return;
  }
  if (k32) {
    if (offs32 && peelk::smem_bytes<uint32_t, true>(4 * vq, true) <= kSmemCap &&
        launch_vec<true>(g, d_loads, base, one_at_a_time, vq, d_perm, d_raw, d_batches))
      return;
    if (peelk::smem_bytes<uint32_t, false>(4 * vq, true) <= kSmemCap &&
        launch_vec<false>(g, d_loads, base, one_at_a_time, vq, d_perm, d_raw, d_batches))
      return;
    if (mode != 1) {
      if (launch_cluster<16>(g, d_loads, base, one_at_a_time, d_perm, d_raw, d_batches)) return;
      if (launch_cluster<8>(g, d_loads, base, one_at_a_time, d_perm, d_raw, d_batches)) return;
    }
  }
#define DG_PEEL_TRY(K, SM, OF)                                                               \
  if ((sizeof(K) == 4) == k32 && (!OF || offs32) &&                                          \
      peelk::smem_bytes<K, OF>(chunk_odd, SM) <= kSmemCap) {                                 \
    launch_peel<K, SM, OF, 0>(g, d_loads, base, one_at_a_time, chunk_odd, d_perm, d_raw,     \
                              d_batches);                                                    \
    return;                                                                                  \
  }
  DG_PEEL_TRY(uint32_t, true, true)
  DG_PEEL_TRY(uint32_t, true, false)
  DG_PEEL_TRY(uint64_t, true, true)
  DG_PEEL_TRY(uint64_t, true, false)
  DG_PEEL_TRY(uint32_t, false, false)
  DG_PEEL_TRY(uint64_t, false, false)
#undef DG_PEEL_TRY
  throw DgError(DG_E_INVARIANT, "no peel kernel variant fits");
}

void peel_profile(unsigned long long out[16]) {
  d2h(out, peel_prof_buffer(), 16);
  stream_sync();
}

void peel_trace_arm(uint32_t first_batch) {
  int d = 0;
  DG_CUDA(cudaGetDevice(&d));
  g_peel_trace_armed[d] = first_batch != 0xffffffffu;
  const unsigned long long w = g_peel_trace_armed[d] ? first_batch + 1ULL : 0ULL;  // 0 = disarmed
  h2d(peel_prof_buffer() + 15, &w, 1);
  stream_sync();
}

void peel_trace_read(unsigned long long* out) {
  d2h(out, peel_prof_buffer() + 16, kPeelTraceWords);
  stream_sync();
}

void sort_order(uint64_t n, const uint64_t* d_loads, uint32_t* d_perm) {
  if (!n) return;
  DevBuf<uint32_t> ids(n);
  DevBuf<uint64_t> ksorted(n);
  k_iota<<<grid_for(n, 256), 256, 0, stream()>>>(ids.get(), n);
  DG_CHECK_LAUNCH();
  size_t tmp = 0;
  DG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, d_loads, ksorted.get(), ids.get(), d_perm,
                                          n, 0, 64, stream()));
  DevBuf<char> t(tmp);
  DG_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, d_loads, ksorted.get(), ids.get(),
                                          d_perm, n, 0, 64, stream()));
}

void charges_from_perm(const dg_graph& g, const uint32_t* d_perm, uint32_t* d_charges) {
  const uint64_t n = g.n;
  if (!n) return;
  DevBuf<uint64_t> pos(n);
  pos.fill_ff();
  DevBuf<uint32_t> err(1);
  err.zero();
  k_pos_from_perm<<<grid_for(n, 256), 256, 0, stream()>>>(d_perm, n, pos.get(), err.get());
  DG_CHECK_LAUNCH();
  if (read_scalar(err.get())) throw DgError(DG_E_INVARIANT, "ordering is not a permutation");
  k_charges_rows<uint64_t><<<grid_for(n * 32, 256), 256, 0, stream()>>>(g.offs.get(), g.adj.get(),
                                                                         n, pos.get(), d_charges);
  DG_CHECK_LAUNCH();
}

void charges_trusted(const dg_graph& g, const uint32_t* d_perm, uint32_t* d_charges) {
  const uint64_t n = g.n;
  if (!n) return;
  DevBuf<uint32_t> pos(n);
  k_pos32<<<grid_for(n, 256), 256, 0, stream()>>>(d_perm, n, pos.get());
  DG_CHECK_LAUNCH();
  k_charges_rows<uint32_t><<<grid_for(n * 32, 256), 256, 0, stream()>>>(g.offs.get(), g.adj.get(),
                                                                         n, pos.get(), d_charges);
  DG_CHECK_LAUNCH();
}

void sort_order_range(uint64_t n, const uint64_t* d_loads, const KeyRange& kr, uint32_t* d_perm) {
  if (!n) return;
  uint32_t bits = 0;
  while (bits < 64 && (kr.max_key >> bits)) ++bits;  // loads - base <= max_key
  if (bits > 32) {
    sort_order(n, d_loads, d_perm);
    return;
  }
  if (bits == 0) {
    k_iota<<<grid_for(n, 256), 256, 0, stream()>>>(d_perm, n);
    DG_CHECK_LAUNCH();
    return;
  }
  DevBuf<uint32_t> ids(n), k32(n), ks(n);
  k_iota<<<grid_for(n, 256), 256, 0, stream()>>>(ids.get(), n);
  DG_CHECK_LAUNCH();
  k_sort_keys32<<<grid_for(n, 256), 256, 0, stream()>>>(d_loads, n, kr.min_load, k32.get());
  DG_CHECK_LAUNCH();
  size_t tmp = 0;
  DG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k32.get(), ks.get(), ids.get(), d_perm, n,
                                          0, int(bits), stream()));
  DevBuf<char> t(tmp);
  DG_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, k32.get(), ks.get(), ids.get(), d_perm, n,
                                          0, int(bits), stream()));
}

void alg3(const dg_graph& g, const uint32_t* d_perm, const uint32_t* d_charges,
          const uint64_t* d_raw, uint64_t raw_base, uint64_t* d_loads,
          uint64_t slack_samples, uint64_t slack_allowed, uint64_t slack_seed, uint64_t* d_suffix,
          Alg3Out* d_out) {
  DevBuf<uint64_t> cs(g.n ? g.n : 1);
  A3Args a{g.offs.get(), uint32_t(g.n), d_perm, d_charges, d_raw, raw_base, d_loads,
           slack_samples, slack_allowed,
           slack_seed, d_suffix, d_out, cs.get()};
  k_alg3<<<1, PT, 0, stream()>>>(a);
  DG_CHECK_LAUNCH();
}

}  // namespace dgb

extern "C" dg_status dg_set_peel_mode(int mode) {
  if (mode < 0 || mode > 3) return DG_E_PARAM;
  dgb::g_peel_mode.store(mode, std::memory_order_relaxed);
  return DG_OK;
}
