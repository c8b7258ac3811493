// oracle_search.cu -- the reference's exhaustive densest-subgraph search
// (proj/include/densegraph/oracle.hpp:16-19, proj/src/oracle.cpp:70-108) on
// the device: every nonempty vertex subset of a graph with <= 32 vertices.
//
// Contract (oracle.hpp:16-19): rho* reduced; ties prefer fewer vertices,
// then the lexicographically smallest sorted id set; the witness is the
// ORIGINAL ids, ascending.  These three keys order distinct subsets totally,
// so the maximum is unique and any reduction order finds it.
//
// Mapping: 2^n - 1 Gray-code states are cut into contiguous ranges, one per
// thread; a state differs from its predecessor in one vertex, so the edge
// count of the subset updates with one popcount of that vertex's adjacency
// mask (masks in shared memory).  Each thread keeps its best candidate,
// warps and CTAs reduce with the same order, and a one-CTA pass reduces the
// CTA winners.  2^22 subsets take a few microseconds of a B200.
#include <string>

#include "internal.cuh"

namespace dgb {
namespace {

struct Cand {
  uint32_t edges, verts, mask;
};

// lexicographic order of sorted id lists for equal-size sets: the smaller
// set owns the lowest bit of the symmetric difference
__device__ __forceinline__ bool lex_smaller(uint32_t a, uint32_t b) {
  const uint32_t d = a ^ b;
  return (a & (d & (0u - d))) != 0;
}

__device__ __forceinline__ bool better(const Cand& a, const Cand& b) {
  if (a.verts == 0) return false;
  if (b.verts == 0) return true;
  const uint64_t l = uint64_t(a.edges) * b.verts, r = uint64_t(b.edges) * a.verts;
  if (l != r) return l > r;
  if (a.verts != b.verts) return a.verts < b.verts;
  return lex_smaller(a.mask, b.mask);
}

__device__ __forceinline__ Cand warp_best(Cand c) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    Cand x{__shfl_xor_sync(~0u, c.edges, o), __shfl_xor_sync(~0u, c.verts, o),
           __shfl_xor_sync(~0u, c.mask, o)};
    if (better(x, c)) c = x;
  }
  return c;
}

__device__ __forceinline__ Cand block_best(Cand c, Cand* sm) {
  c = warp_best(c);
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) sm[w] = c;
  __syncthreads();
  if (w == 0) {
    c = (threadIdx.x < nw) ? sm[threadIdx.x] : Cand{0, 0, 0};
    c = warp_best(c);
  }
  return c;
}

__device__ __forceinline__ uint32_t subset_edges(const uint32_t* adjm, uint32_t members) {
  uint32_t e = 0;
  for (uint32_t rest = members; rest; rest &= rest - 1)
    e += __popc(adjm[__ffs(rest) - 1] & members);
  return e / 2;
}

__global__ void k_oracle_scan(const uint32_t* g_adjm, uint32_t n, uint64_t total, Cand* out) {
  __shared__ uint32_t adjm[32];
  __shared__ Cand sm[32];
  if (threadIdx.x < 32) adjm[threadIdx.x] = threadIdx.x < n ? g_adjm[threadIdx.x] : 0u;
  __syncthreads();
  const uint64_t T = uint64_t(gridDim.x) * blockDim.x;
  const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  // states 1..total, thread t takes [lo, hi)
  const uint64_t lo = 1 + total * t / T, hi = 1 + total * (t + 1) / T;
  Cand best{0, 0, 0};
  if (lo < hi) {
    uint32_t members = uint32_t(lo ^ (lo >> 1));
    uint32_t edges = subset_edges(adjm, members);
    for (uint64_t s = lo;;) {
      const Cand cur{edges, uint32_t(__popc(members)), members};
      if (better(cur, best)) best = cur;
      if (++s >= hi) break;
      const uint32_t v = __ffsll((long long)s) - 1;  // the bit Gray state s flips
      const uint32_t bit = 1u << v;
      if (members & bit) {
        members ^= bit;
        edges -= __popc(adjm[v] & members);
      } else {
        edges += __popc(adjm[v] & members);
        members ^= bit;
      }
    }
  }
  best = block_best(best, sm);
  if (threadIdx.x == 0) out[blockIdx.x] = best;
}

__global__ void k_oracle_reduce(const Cand* in, uint32_t k, Cand* out) {
  __shared__ Cand sm[32];
  Cand best{0, 0, 0};
  for (uint32_t i = threadIdx.x; i < k; i += blockDim.x)
    if (better(in[i], best)) best = in[i];
  best = block_best(best, sm);
  if (threadIdx.x == 0) *out = best;
}

// adjacency masks of a <= 32-vertex graph, one warp per row
__global__ void k_oracle_masks(const uint64_t* offs, const uint32_t* adj, uint32_t n,
                               uint32_t* adjm) {
  const uint32_t v = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (v >= n) return;
  uint32_t m = 0;
  for (uint64_t i = offs[v] + lane; i < offs[v + 1]; i += 32) m |= 1u << adj[i];
  m = __reduce_or_sync(~0u, m);
  if (lane == 0) adjm[v] = m;
}

uint64_t gcd64(uint64_t a, uint64_t b) {
  while (b) {
    const uint64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

}  // namespace
}  // namespace dgb

using namespace dgb;

extern "C" dg_status dg_brute_force_densest(const dg_graph* g, uint32_t limit, uint64_t* edges,
                                            uint64_t* verts, uint64_t* witness,
                                            uint64_t* witness_n) {
  DG_API_BEGIN
  if (!g || !edges || !verts || !witness_n) throw DgError(DG_E_PARAM, "null argument");
  if (g->n == 0) throw DgError(DG_E_EMPTY, "oracle on empty graph");
  if (g->n > limit || g->n > 32)
    throw DgError(DG_E_ORACLE_SIZE, "graph has " + std::to_string(g->n) +
                                        " vertices, oracle limit is " + std::to_string(limit));
  const uint32_t n = uint32_t(g->n);
  DevBuf<uint32_t> adjm(32);
  k_oracle_masks<<<1, 32 * n, 0, stream()>>>(g->offs.get(), g->adj.get(), n, adjm.get());
  DG_CHECK_LAUNCH();
  const uint64_t total = (n == 32) ? 0xffffffffULL : (1ULL << n) - 1;
  // ~64 states per thread at least; up to 8 CTAs of 256 per SM
  uint64_t want = (total + 63) / 64;
  unsigned threads = 256;
  unsigned blocks = unsigned(std::min<uint64_t>((want + threads - 1) / threads,
                                                uint64_t(num_sms()) * 8));
  if (blocks == 0) blocks = 1;
  DevBuf<Cand> part(blocks), best(1);
  k_oracle_scan<<<blocks, threads, 0, stream()>>>(adjm.get(), n, total, part.get());
  DG_CHECK_LAUNCH();
  k_oracle_reduce<<<1, 1024, 0, stream()>>>(part.get(), blocks, best.get());
  DG_CHECK_LAUNCH();
  Cand c;
  d2h(&c, best.get(), 1);
  uint64_t orig[32];
  d2h(orig, g->orig.get(), n);
  stream_sync();
  if (c.verts == 0) throw DgError(DG_E_INVARIANT, "oracle search found no subset");
  const uint64_t gg = gcd64(c.edges, c.verts);  // Density::reduced (density.hpp:23-26)
  *edges = c.edges / gg;
  *verts = c.verts / gg;
  uint64_t k = 0;
  for (uint32_t v = 0; v < n; ++v)
    if ((c.mask >> v) & 1u) {
      if (witness) witness[k] = orig[v];
      ++k;
    }
  *witness_n = k;
  DG_API_END
}
