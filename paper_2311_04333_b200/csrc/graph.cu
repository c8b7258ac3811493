// graph.cu -- device CSR build and induced-subgraph compaction.
//
// CSR build (reference io.cpp:51-92 semantics):
//   1. dense ids: presence flags over the original-id range + exclusive scan
//      (rank = dense id), or for huge/sparse id spaces a sort + unique of the
//      endpoints with binary-search ranks;
//   2. canonical pair keys (min<<B | max) over dense ids, CUB onesweep radix
//      sort on the 2B significant bits, unique;
//   3. both arc directions, radix sort on (src, dst) -> rows ascending; adj =
//      low bits, offs from the row boundaries (every dense id has an edge).
// Induced subgraph (graph.hpp:50-80): keep scan -> map; rows cut into
// segments of <= kSeg arcs so hub rows are spread over many warps; per-
// segment kept-neighbour counts, one exclusive scan gives both the new
// offsets and every segment's output position; an order-preserving
// ballot-compaction pass fills the new rows.
#include <cub/cub.cuh>

#include "internal.cuh"

namespace dgb {

namespace {

constexpr uint32_t kSeg = 2048;

__global__ void k_max_id(const uint64_t* u, const uint64_t* v, uint64_t k,
                         unsigned long long* out) {
  uint64_t mx = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < k;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t a = u[i], b = v[i];
    if (a != b) mx = max(mx, max(a, b));
  }
  mx = warp_max(mx);
  if (lane_id() == 0 && mx) atomicMax(out, (unsigned long long)mx);
}

__global__ void k_mark_present(const uint64_t* u, const uint64_t* v, uint64_t k,
                               uint32_t* flags) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < k;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t a = u[i], b = v[i];
    if (a != b) {
      flags[a] = 1;
      flags[b] = 1;
    }
  }
}

__global__ void k_scatter_orig(const uint32_t* flags, const uint32_t* rank, uint64_t count,
                               uint64_t* orig) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
       i += uint64_t(gridDim.x) * blockDim.x)
    if (flags[i]) orig[rank[i]] = i;
}

__global__ void k_endpoints(const uint64_t* u, const uint64_t* v, uint64_t k, uint64_t* ep,
                            uint8_t* keep) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < k;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t a = u[i], b = v[i];
    ep[2 * i] = a;
    ep[2 * i + 1] = b;
    keep[2 * i] = keep[2 * i + 1] = a != b;
  }
}

__device__ __forceinline__ uint64_t lower_bound_dev(const uint64_t* a, uint64_t n, uint64_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    uint64_t mid = (lo + hi) >> 1;
    if (a[mid] < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// mode 0: rank table lookup (ids < table size); mode 1: binary search in orig.
__global__ void k_pair_keys(const uint64_t* u, const uint64_t* v, uint64_t k, int mode,
                            const uint32_t* rank, const uint64_t* orig, uint64_t n, uint32_t B,
                            uint64_t* keys) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < k;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t a = u[i], b = v[i];
    if (a == b) {
      keys[i] = ~0ULL;
      continue;
    }
    uint64_t lo = min(a, b), hi = max(a, b);
    uint64_t x = mode == 0 ? rank[lo] : lower_bound_dev(orig, n, lo);
    uint64_t y = mode == 0 ? rank[hi] : lower_bound_dev(orig, n, hi);
    keys[i] = (x << B) | y;
  }
}

__global__ void k_arcs(const uint64_t* pkeys, uint64_t m, uint32_t B, uint64_t* arcs) {
  const uint64_t mask = (1ULL << B) - 1;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < m;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t key = pkeys[i];
    arcs[2 * i] = key;
    arcs[2 * i + 1] = ((key & mask) << B) | (key >> B);
  }
}

__global__ void k_csr_from_arcs(const uint64_t* arcs, uint64_t arcs_n, uint32_t B, uint64_t n,
                                uint32_t* adj, uint64_t* offs) {
  const uint64_t mask = (1ULL << B) - 1;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < arcs_n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t key = arcs[i];
    adj[i] = uint32_t(key & mask);
    uint64_t s = key >> B;
    if (i == 0 || (arcs[i - 1] >> B) != s) offs[s] = i;
    if (i == 0) offs[n] = arcs_n;
  }
}

__global__ void k_max_degree(const uint64_t* offs, uint64_t n, unsigned long long* out) {
  uint64_t mx = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    mx = max(mx, offs[i + 1] - offs[i]);
  mx = warp_max(mx);
  if (lane_id() == 0 && mx) atomicMax(out, (unsigned long long)mx);
}

// ---- induced subgraph ----
// keep flags (scanned into the old -> new map) and the same as a bitmap: the
// per-arc membership tests of the count and fill passes read n / 8 bytes that
// stay in L2 (RMAT-26: 4 MB) instead of gathering from a 4n-byte array
__global__ void k_keep_flags(const uint8_t* keep8, const uint32_t* labels, uint32_t k, uint64_t n,
                             uint32_t* keep, uint32_t* bits) {
  const uint64_t step = uint64_t(gridDim.x) * blockDim.x;  // a multiple of 32
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < ((n + 31) & ~uint64_t(31));
       i += step) {
    const bool f = i < n && (keep8 ? (keep8[i] != 0) : (labels[i] >= k));
    if (i < n) keep[i] = f;
    const uint32_t b = __ballot_sync(0xffffffffu, f);
    if (lane_id() == 0) bits[i >> 5] = b;
  }
}

// wrank[w] = new id of the first kept vertex at or after id 32w, so that
// map[u] = wrank[u >> 5] + popc(bits[u >> 5] below bit u & 31)
__global__ void k_word_ranks(const uint32_t* map, uint64_t n, uint32_t* wrank) {
  const uint64_t W = (n + 31) >> 5;
  for (uint64_t w = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; w < W;
       w += uint64_t(gridDim.x) * blockDim.x)
    wrank[w] = map[w << 5];
}

__device__ __forceinline__ bool bit_of(const uint32_t* bits, uint32_t u) {
  return (__ldg(bits + (u >> 5)) >> (u & 31)) & 1u;
}

__global__ void k_nseg(const uint32_t* keep, const uint64_t* offs, uint64_t n, uint64_t* nseg) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t d = offs[i + 1] - offs[i];
    nseg[i] = keep[i] ? max(uint64_t(1), (d + kSeg - 1) / kSeg) : uint64_t(0);
  }
}

__global__ void k_seg_rows(const uint32_t* keep, const uint64_t* nseg, const uint64_t* segoff,
                           uint64_t n, uint32_t* seg_row) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    if (!keep[i]) continue;
    for (uint64_t j = 0; j < nseg[i]; ++j) seg_row[segoff[i] + j] = uint32_t(i);
  }
}

// warp per segment: count kept neighbours
__global__ void k_seg_count(const uint32_t* seg_row, const uint64_t* segoff, uint64_t S,
                            const uint64_t* offs, const uint32_t* adj, const uint32_t* bits,
                            uint64_t* segcnt) {
  const uint64_t warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t s = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; s < S; s += warps) {
    uint32_t v = seg_row[s];
    uint64_t j = s - segoff[v];
    uint64_t b = offs[v] + j * kSeg, e = min(offs[v + 1], b + kSeg);
    uint32_t c = 0;
    constexpr int U = 8;  // arcs in flight per lane
    for (uint64_t p0 = b + lane_id(); p0 < e; p0 += 32 * U) {
      uint32_t u[U];
#pragma unroll
      for (int q = 0; q < U; ++q) u[q] = p0 + 32 * q < e ? __ldg(adj + p0 + 32 * q) : kNoVertex;
#pragma unroll
      for (int q = 0; q < U; ++q)
        if (u[q] != kNoVertex) c += bit_of(bits, u[q]);
    }
    c = warp_sum(c);
    if (lane_id() == 0) segcnt[s] = c;
  }
}

__global__ void k_seg_fill(const uint32_t* seg_row, const uint64_t* segoff, uint64_t S,
                           const uint64_t* offs, const uint32_t* adj, const uint32_t* bits,
                           const uint32_t* wrank, const uint64_t* segpos, uint32_t* nadj) {
  const uint64_t warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t s = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; s < S; s += warps) {
    uint32_t v = seg_row[s];
    uint64_t j = s - segoff[v];
    uint64_t b = offs[v] + j * kSeg, e = min(offs[v + 1], b + kSeg);
    uint64_t w = segpos[s];
    constexpr int U = 4;  // 32-arc steps in flight
    for (uint64_t p0 = b; p0 < e; p0 += 32 * U) {
      uint32_t u[U], wd[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const uint64_t p = p0 + 32 * q + lane_id();
        u[q] = p < e ? __ldg(adj + p) : kNoVertex;
      }
#pragma unroll
      for (int q = 0; q < U; ++q) wd[q] = u[q] != kNoVertex ? __ldg(bits + (u[q] >> 5)) : 0u;
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const bool k = (wd[q] >> (u[q] & 31)) & 1u;
        const uint32_t bal = __ballot_sync(0xffffffffu, k);
        if (k)
          nadj[w + __popc(bal & ((1u << lane_id()) - 1))] =
              __ldg(wrank + (u[q] >> 5)) + __popc(wd[q] & ((1u << (u[q] & 31)) - 1));
        w += __popc(bal);
      }
    }
  }
}

__global__ void k_new_rows(const uint32_t* keep, const uint32_t* map, const uint64_t* segoff,
                           const uint64_t* segpos, const uint64_t* orig, uint64_t n,
                           uint64_t new_n, uint64_t total, uint64_t* noffs, uint64_t* norig,
                           uint32_t* old_to_new) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    if (keep[i]) {
      noffs[map[i]] = segpos[segoff[i]];
      norig[map[i]] = orig[i];
    }
    if (old_to_new) old_to_new[i] = keep[i] ? map[i] : kNoVertex;
    if (i == 0) noffs[new_n] = total;
  }
}

__global__ void k_gather_map_u32(const uint32_t* in, const uint32_t* map, uint64_t n,
                                 uint32_t* out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    if (map[i] != kNoVertex) out[map[i]] = in[i];
}
__global__ void k_gather_map_u64(const uint64_t* in, const uint32_t* map, uint64_t n,
                                 uint64_t* out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    if (map[i] != kNoVertex) out[map[i]] = in[i];
}

template <class T>
T excl_scan(const T* d_in, T* d_out, uint64_t count) {
  if (count == 0) return T(0);
  size_t tmp = 0;
  DG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, d_in, d_out, count, stream()));
  DevBuf<char> t(tmp);
  DG_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, d_in, d_out, count, stream()));
  T a, b;
  d2h(&a, d_in + count - 1, 1);
  d2h(&b, d_out + count - 1, 1);
  stream_sync();
  return a + b;
}

uint32_t bits_for(uint64_t n) {  // bits to hold ids 0..n-1 (>= 1)
  uint32_t b = 1;
  while ((1ULL << b) < n) ++b;
  return b;
}

void radix_sort_u64(DevBuf<uint64_t>& keys, uint64_t count, uint32_t end_bit) {
  if (count < 2) return;
  DevBuf<uint64_t> alt(count);
  cub::DoubleBuffer<uint64_t> db(keys.get(), alt.get());
  size_t tmp = 0;
  DG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, db, count, 0, int(end_bit), stream()));
  DevBuf<char> t(tmp);
  DG_CUDA(cub::DeviceRadixSort::SortKeys(t.get(), tmp, db, count, 0, int(end_bit), stream()));
  if (db.Current() != keys.get()) std::swap(keys, alt);
}

}  // namespace

uint64_t device_max_degree(const uint64_t* d_offs, uint64_t n) {
  DevBuf<unsigned long long> mx(1);
  mx.zero();
  k_max_degree<<<grid_for(n, 256), 256, 0, stream()>>>(d_offs, n, mx.get());
  DG_CHECK_LAUNCH();
  return read_scalar(mx.get());
}

GraphPtr build_from_pairs(const uint64_t* d_u, const uint64_t* d_v, uint64_t k) {
  const unsigned T = 256;
  DevBuf<unsigned long long> mx(1);
  mx.zero();
  if (k) k_max_id<<<grid_for(k, T), T, 0, stream()>>>(d_u, d_v, k, mx.get());
  DG_CHECK_LAUNCH();
  const uint64_t maxid = read_scalar(mx.get());

  auto g = std::make_unique<dg_graph>();
  DevBuf<uint32_t> rank;
  int mode;
  // Any non-loop pair has max(u,v) >= 1, so maxid == 0 <=> no edge.
  if (maxid == 0) throw DgError(DG_E_EMPTY, "no edges after removing self-loops and duplicates");

  size_t free_b = 0, total_b = 0;
  DG_CUDA(cudaMemGetInfo(&free_b, &total_b));
  if (maxid < 0xffffffffULL && (maxid + 1) * 8 <= free_b / 4) {
    // presence flags -> rank table (dense id = rank among present ids)
    mode = 0;
    const uint64_t R = maxid + 1;
    DevBuf<uint32_t> flags(R);
    flags.zero();
    k_mark_present<<<grid_for(k, T), T, 0, stream()>>>(d_u, d_v, k, flags.get());
    DG_CHECK_LAUNCH();
    rank.alloc(R);
    g->n = excl_scan(flags.get(), rank.get(), R);
    g->orig.alloc(g->n);
    k_scatter_orig<<<grid_for(R, T), T, 0, stream()>>>(flags.get(), rank.get(), R, g->orig.get());
    DG_CHECK_LAUNCH();
  } else {
    // sparse / 64-bit ids: sort + unique endpoints, binary-search ranks
    mode = 1;
    DevBuf<uint64_t> ep(2 * k), sel(2 * k);
    DevBuf<uint8_t> keep(2 * k);
    k_endpoints<<<grid_for(k, T), T, 0, stream()>>>(d_u, d_v, k, ep.get(), keep.get());
    DG_CHECK_LAUNCH();
    DevBuf<uint64_t> cnt(1);
    size_t tmp = 0;
    DG_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, ep.get(), keep.get(), sel.get(), cnt.get(),
                                       2 * k, stream()));
    {
      DevBuf<char> t(tmp);
      DG_CUDA(cub::DeviceSelect::Flagged(t.get(), tmp, ep.get(), keep.get(), sel.get(), cnt.get(),
                                         2 * k, stream()));
    }
    uint64_t c = read_scalar(cnt.get());
    radix_sort_u64(sel, c, 64);
    g->orig.alloc(c);
    tmp = 0;
    DG_CUDA(cub::DeviceSelect::Unique(nullptr, tmp, sel.get(), g->orig.get(), cnt.get(), c,
                                      stream()));
    {
      DevBuf<char> t(tmp);
      DG_CUDA(cub::DeviceSelect::Unique(t.get(), tmp, sel.get(), g->orig.get(), cnt.get(), c,
                                        stream()));
    }
    g->n = read_scalar(cnt.get());
  }
  if (g->n > 0xfffffffeULL) throw DgError(DG_E_PARAM, "more than 2^32-2 vertices");
  const uint32_t B = bits_for(g->n);

  // canonical pair keys, sort on 2B bits, unique
  DevBuf<uint64_t> keys(k);
  k_pair_keys<<<grid_for(k, T), T, 0, stream()>>>(d_u, d_v, k, mode, rank.get(), g->orig.get(),
                                                  g->n, B, keys.get());
  DG_CHECK_LAUNCH();
  rank.release();
  radix_sort_u64(keys, k, 2 * B);
  DevBuf<uint64_t> ukeys(k), cnt(1);
  {
    size_t tmp = 0;
    DG_CUDA(cub::DeviceSelect::Unique(nullptr, tmp, keys.get(), ukeys.get(), cnt.get(), k,
                                      stream()));
    DevBuf<char> t(tmp);
    DG_CUDA(cub::DeviceSelect::Unique(t.get(), tmp, keys.get(), ukeys.get(), cnt.get(), k,
                                      stream()));
  }
  keys.release();
  uint64_t m = read_scalar(cnt.get());
  if (m) {
    uint64_t last = read_scalar(ukeys.get() + m - 1);
    const uint64_t sentinel_lo = (2 * B == 64) ? ~0ULL : ((1ULL << (2 * B)) - 1);
    if ((last & sentinel_lo) == sentinel_lo) --m;  // the self-loop sentinel group
  }
  if (m == 0) throw DgError(DG_E_EMPTY, "no edges after removing self-loops and duplicates");
  g->m = m;

  // both arc directions -> sorted rows
  DevBuf<uint64_t> arcs(2 * m);
  k_arcs<<<grid_for(m, T), T, 0, stream()>>>(ukeys.get(), m, B, arcs.get());
  DG_CHECK_LAUNCH();
  ukeys.release();
  radix_sort_u64(arcs, 2 * m, 2 * B);
  g->adj.alloc(2 * m);
  g->offs.alloc(g->n + 1);
  k_csr_from_arcs<<<grid_for(2 * m, T), T, 0, stream()>>>(arcs.get(), 2 * m, B, g->n,
                                                          g->adj.get(), g->offs.get());
  DG_CHECK_LAUNCH();
  arcs.release();
  g->maxdeg = device_max_degree(g->offs.get(), g->n);
  return g;
}

GraphPtr graph_from_device_csr(uint64_t n, const uint64_t* d_offs, const uint32_t* d_adj,
                               const uint64_t* d_orig) {
  auto g = std::make_unique<dg_graph>();
  g->n = n;
  g->offs.alloc(n + 1);
  d2d(g->offs.get(), d_offs, n + 1);
  uint64_t arcs = read_scalar(g->offs.get() + n);
  if (arcs & 1) throw DgError(DG_E_INVARIANT, "CSR arc count is odd");
  g->m = arcs / 2;
  g->adj.alloc(arcs);
  d2d(g->adj.get(), d_adj, arcs);
  g->orig.alloc(n);
  d2d(g->orig.get(), d_orig, n);
  g->maxdeg = n ? device_max_degree(g->offs.get(), n) : 0;
  return g;
}

GraphPtr induced(const dg_graph& g, const uint8_t* d_keep, const uint32_t* d_labels, uint32_t k,
                 uint32_t* d_old_to_new) {
  const unsigned T = 256;
  const uint64_t n = g.n;
  auto h = std::make_unique<dg_graph>();
  if (n == 0) {
    h->offs.alloc(1);
    h->offs.zero();
    return h;
  }
  DevBuf<uint32_t> keep(n), map(n), bits((n + 31) / 32), wrank((n + 31) / 32);
  k_keep_flags<<<grid_for(n, T), T, 0, stream()>>>(d_keep, d_labels, k, n, keep.get(), bits.get());
  DG_CHECK_LAUNCH();
  const uint64_t new_n = excl_scan(keep.get(), map.get(), n);
  k_word_ranks<<<grid_for((n + 31) / 32, T), T, 0, stream()>>>(map.get(), n, wrank.get());
  DG_CHECK_LAUNCH();
  DevBuf<uint64_t> nseg(n), segoff(n);
  k_nseg<<<grid_for(n, T), T, 0, stream()>>>(keep.get(), g.offs.get(), n, nseg.get());
  DG_CHECK_LAUNCH();
  const uint64_t S = excl_scan(nseg.get(), segoff.get(), n);
  DevBuf<uint32_t> seg_row(S);
  DevBuf<uint64_t> segcnt(S), segpos(S);
  uint64_t total = 0;
  if (S) {
    k_seg_rows<<<grid_for(n, T), T, 0, stream()>>>(keep.get(), nseg.get(), segoff.get(), n,
                                                   seg_row.get());
    DG_CHECK_LAUNCH();
  }
  nseg.release();
  h->n = new_n;
  h->offs.alloc(new_n + 1);
  h->orig.alloc(new_n);
  if (S) {
    k_seg_count<<<grid_for(S * 32, T), T, 0, stream()>>>(seg_row.get(), segoff.get(), S,
                                                         g.offs.get(), g.adj.get(), bits.get(),
                                                         segcnt.get());
    DG_CHECK_LAUNCH();
    total = excl_scan(segcnt.get(), segpos.get(), S);
  }
  k_new_rows<<<grid_for(n, T), T, 0, stream()>>>(keep.get(), map.get(), segoff.get(),
                                                 segpos.get(), g.orig.get(), n, new_n, total,
                                                 h->offs.get(), h->orig.get(), d_old_to_new);
  DG_CHECK_LAUNCH();
  h->adj.alloc(total);
  h->m = total / 2;
  if (S && total) {
    k_seg_fill<<<grid_for(S * 32, T), T, 0, stream()>>>(seg_row.get(), segoff.get(), S,
                                                        g.offs.get(), g.adj.get(), bits.get(),
                                                        wrank.get(), segpos.get(), h->adj.get());
    DG_CHECK_LAUNCH();
  }
  h->maxdeg = new_n ? device_max_degree(h->offs.get(), new_n) : 0;
  return h;
}

// ---- arcs of a vertex list into a vertex set (the witness recount) ----
namespace {
__global__ void k_list_nseg(const uint32_t* rows, uint64_t nrows, const uint64_t* offs,
                            uint32_t* nseg) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nrows;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t d = offs[rows[i] + 1] - offs[rows[i]];
    nseg[i] = uint32_t((d + kSeg - 1) / kSeg);
  }
}
// warp per segment of <= kSeg arcs: its row by binary search over the scanned
// segment counts (hub rows of the input graph spread over many warps)
__global__ void k_list_seg_count(const uint32_t* rows, uint64_t nrows, const uint32_t* segoff,
                                 uint64_t S, const uint64_t* offs, const uint32_t* adj,
                                 const uint32_t* bits, unsigned long long* total) {
  const uint64_t warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  unsigned long long c = 0;
  for (uint64_t s = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; s < S; s += warps) {
    uint64_t lo = 0, hi = nrows;  // last row with segoff <= s
    while (hi - lo > 1) {
      const uint64_t mid = (lo + hi) >> 1;
      if (segoff[mid] <= s) lo = mid; else hi = mid;
    }
    const uint32_t v = rows[lo];
    const uint64_t b = offs[v] + (s - segoff[lo]) * kSeg, e = min(offs[v + 1], b + kSeg);
    constexpr int U = 8;
    for (uint64_t p0 = b + lane_id(); p0 < e; p0 += 32 * U) {
      uint32_t u[U];
#pragma unroll
      for (int q = 0; q < U; ++q) u[q] = p0 + 32 * q < e ? __ldg(adj + p0 + 32 * q) : kNoVertex;
#pragma unroll
      for (int q = 0; q < U; ++q)
        if (u[q] != kNoVertex) c += bit_of(bits, u[q]);
    }
  }
  c = warp_sum(c);
  if (lane_id() == 0 && c) atomicAdd(total, c);
}
}  // namespace

uint64_t count_arcs_into_set(const dg_graph& g, const uint32_t* d_rows, uint64_t nrows,
                             const uint32_t* d_bits) {
  if (!nrows) return 0;
  const unsigned T = 256;
  DevBuf<uint32_t> nseg(nrows), segoff(nrows);
  k_list_nseg<<<grid_for(nrows, T), T, 0, stream()>>>(d_rows, nrows, g.offs.get(), nseg.get());
  DG_CHECK_LAUNCH();
  const uint64_t S = excl_scan(nseg.get(), segoff.get(), nrows);
  DevBuf<unsigned long long> total(1);
  total.zero();
  if (S) {
    k_list_seg_count<<<grid_for(S * 32, T), T, 0, stream()>>>(
        d_rows, nrows, segoff.get(), S, g.offs.get(), g.adj.get(), d_bits, total.get());
    DG_CHECK_LAUNCH();
  }
  return read_scalar(total.get());
}

void gather_by_map_u32(const uint32_t* in, const uint32_t* map, uint64_t n, uint32_t* out) {
  if (!n) return;
  k_gather_map_u32<<<grid_for(n, 256), 256, 0, stream()>>>(in, map, n, out);
  DG_CHECK_LAUNCH();
}
void gather_by_map_u64(const uint64_t* in, const uint32_t* map, uint64_t n, uint64_t* out) {
  if (!n) return;
  k_gather_map_u64<<<grid_for(n, 256), 256, 0, stream()>>>(in, map, n, out);
  DG_CHECK_LAUNCH();
}

}  // namespace dgb
