// dist_build.cu -- the per-rank device work of the distributed CSR build and
// of the per-shard get_core, so a multi-GPU job never holds
// the whole graph: paper_2311_04333_b200/sharded_build.py moves the buffers
// between ranks (NCCL all-to-all / all-gather) and calls these kernels on
// each rank's slice.  Semantics are the reference's CSR build (io.cpp:51-92:
// canonical pairs, loops dropped, duplicates collapsed, dense id = rank of
// the original id, rows ascending) and induced_subgraph (graph.hpp:50-80:
// kept vertices renumbered in old order, rows keep their order), cut along
// contiguous ranges of the original id space.
//
//   route   sample pairs -> both arc directions as (src << 32 | dst) keys,
//           grouped by the owner of src (original-id ranges)
//   rows    received keys -> sort, unique -> the owner's rows: distinct
//           sources, row offsets, neighbour original ids
//   unique  distinct neighbour ids + each arc's index into them (the ids
//           are then asked of their owners)
//   lookup  an owner's answers: dense id = rank base + position among its
//           sources (binary search)
//   relabel adjacency in dense ids
//   keep / core_rows   get_core on a shard: kept-vertex map, kept rows with
//           the kept neighbours renamed through the all-gathered map
#include <cub/cub.cuh>

#include <vector>

#include "internal.cuh"

namespace dgb {
namespace {

constexpr uint32_t kNone = 0xffffffffu;
constexpr uint32_t kMaxRanks = 64;

__device__ __forceinline__ uint32_t owner_of_id(const uint64_t* sb, uint32_t P, uint64_t x) {
  uint32_t lo = 0, hi = P - 1;  // largest r with sb[r] <= x
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (sb[mid] <= x) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void k_dist_max(const uint64_t* u, const uint64_t* v, uint64_t k,
                           unsigned long long* out) {
  unsigned long long m = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < k;
       i += uint64_t(gridDim.x) * blockDim.x)
    if (u[i] != v[i]) m = max(m, (unsigned long long)max(u[i], v[i]));
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(~0u, m, o));
  if (lane_id() == 0 && m) atomicMax(out, m);
}

// histogram of non-loop endpoints >> shift into nb buckets (nb <= 4096)
__global__ void k_dist_hist(const uint64_t* u, const uint64_t* v, uint64_t k, uint32_t shift,
                            uint32_t nb, unsigned long long* hist) {
  __shared__ unsigned int sh[4096];
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < k;
       i += uint64_t(gridDim.x) * blockDim.x) {
    if (u[i] == v[i]) continue;
    atomicAdd(&sh[min(u[i] >> shift, uint64_t(nb - 1))], 1u);
    atomicAdd(&sh[min(v[i] >> shift, uint64_t(nb - 1))], 1u);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], (unsigned long long)sh[i]);
}

// per-owner arc counts (both directions of every non-loop pair)
__global__ void k_dist_count(const uint64_t* u, const uint64_t* v, uint64_t k,
                             const uint64_t* bounds, uint32_t P, unsigned long long* cnt) {
  __shared__ uint64_t sb[kMaxRanks + 1];
  __shared__ unsigned long long sc[kMaxRanks];
  for (uint32_t i = threadIdx.x; i <= P; i += blockDim.x) sb[i] = bounds[i];
  for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) sc[i] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < k;
       i += uint64_t(gridDim.x) * blockDim.x) {
    if (u[i] == v[i]) continue;
    atomicAdd(&sc[owner_of_id(sb, P, u[i])], 1ULL);
    atomicAdd(&sc[owner_of_id(sb, P, v[i])], 1ULL);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < P; i += blockDim.x)
    if (sc[i]) atomicAdd(&cnt[i], sc[i]);
}

// scatter keys into owner segments (cursor[r] starts at the segment base)
__global__ void k_dist_scatter(const uint64_t* u, const uint64_t* v, uint64_t k,
                               const uint64_t* bounds, uint32_t P, unsigned long long* cursor,
                               uint64_t* keys) {
  __shared__ uint64_t sb[kMaxRanks + 1];
  for (uint32_t i = threadIdx.x; i <= P; i += blockDim.x) sb[i] = bounds[i];
  __syncthreads();
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < k;
       i += uint64_t(gridDim.x) * blockDim.x) {
    if (u[i] == v[i]) continue;
    const uint64_t a = u[i], b = v[i];
    keys[atomicAdd(&cursor[owner_of_id(sb, P, a)], 1ULL)] = (a << 32) | b;
    keys[atomicAdd(&cursor[owner_of_id(sb, P, b)], 1ULL)] = (b << 32) | a;
  }
}

// sorted unique keys -> row starts (first key of each source) as flags
__global__ void k_dist_src_flags(const uint64_t* keys, uint64_t n, uint32_t* flag,
                                 uint32_t* dst) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    flag[i] = (i == 0 || (keys[i] >> 32) != (keys[i - 1] >> 32)) ? 1u : 0u;
    dst[i] = uint32_t(keys[i]);
  }
}

// flags' exclusive scan -> row offsets and the distinct sources
__global__ void k_dist_rows(const uint64_t* keys, const uint32_t* flag, const uint32_t* pos,
                            uint64_t n, uint64_t* offs, uint64_t* verts) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    if (flag[i]) {
      offs[pos[i]] = i;
      verts[pos[i]] = keys[i] >> 32;
    }
}

__global__ void k_dist_iota(uint32_t* a, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    a[i] = uint32_t(i);
}

// sorted (value, index) pairs -> run starts; inv[index] = run id
__global__ void k_dist_run_flags(const uint32_t* sv, uint64_t n, uint32_t* flag) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    flag[i] = (i == 0 || sv[i] != sv[i - 1]) ? 1u : 0u;
}

__global__ void k_dist_inverse(const uint32_t* sv, const uint32_t* si, const uint32_t* flag,
                               const uint32_t* pos, uint64_t n, uint32_t* uniq, uint32_t* inv) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t r = pos[i] + flag[i] - 1;  // inclusive run id
    inv[si[i]] = r;
    if (flag[i]) uniq[r] = sv[i];
  }
}

__global__ void k_dist_lookup(const uint64_t* verts, uint64_t nv, const uint32_t* asked,
                              uint64_t na, uint64_t base, uint32_t* out, uint32_t* miss) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < na;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t x = asked[i];
    uint64_t lo = 0, hi = nv;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (verts[mid] < x) lo = mid + 1; else hi = mid;
    }
    if (lo >= nv || verts[lo] != x) *miss = 1;
    out[i] = uint32_t(base + lo);
  }
}

__global__ void k_dist_relabel(const uint32_t* back, const uint32_t* inv, uint64_t n,
                               uint32_t* adj) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    adj[i] = back[inv[i]];
}

__global__ void k_dist_keep(const uint32_t* labels, uint64_t nl, uint32_t k, uint32_t* flag) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nl;
       i += uint64_t(gridDim.x) * blockDim.x)
    flag[i] = labels[i] >= k ? 1u : 0u;
}

__global__ void k_dist_map(const uint32_t* flag, const uint32_t* pos, uint64_t nl, uint64_t base,
                           uint32_t* map) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nl;
       i += uint64_t(gridDim.x) * blockDim.x)
    map[i] = flag[i] ? uint32_t(base + pos[i]) : kNone;
}

// kept rows: warp per row, count of kept neighbours (full map: global old id -> new id)
__global__ void k_dist_core_count(const uint64_t* offs, const uint32_t* adj, uint64_t nl,
                                  const uint32_t* keepf, const uint32_t* full, uint64_t* deg) {
  const uint64_t warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t r = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; r < nl; r += warps) {
    uint64_t c = 0;
    if (keepf[r])
      for (uint64_t j = offs[r] + lane_id(); j < offs[r + 1]; j += 32) c += full[adj[j]] != kNone;
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(~0u, c, o);
    if (lane_id() == 0) deg[r] = c;
  }
}

// fill in row order (ballot compaction keeps the neighbours' order)
__global__ void k_dist_core_fill(const uint64_t* offs, const uint32_t* adj, uint64_t nl,
                                 const uint32_t* keepf, const uint32_t* full,
                                 const uint64_t* noffs, const uint32_t* kpos, uint32_t* nadj) {
  const uint64_t warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint32_t lane = lane_id();
  for (uint64_t r = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; r < nl; r += warps) {
    if (!keepf[r]) continue;
    uint64_t o = noffs[kpos[r]];
    for (uint64_t j0 = offs[r]; j0 < offs[r + 1]; j0 += 32) {
      const uint64_t j = j0 + lane;
      uint32_t x = kNone;
      if (j < offs[r + 1]) x = full[adj[j]];
      const uint32_t m = __ballot_sync(~0u, x != kNone);
      if (x != kNone) nadj[o + __popc(m & ((1u << lane) - 1u))] = x;
      o += __popc(m);
    }
  }
}

// counts of sorted values per owner range: binary search per bound
__global__ void k_dist_bucket(const uint32_t* vals, uint64_t n, const uint64_t* bounds, uint32_t P,
                              unsigned long long* pos) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > P) return;
  uint64_t lo = 0, hi = n;  // first index with vals >= bounds[r]
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (vals[mid] < bounds[r]) lo = mid + 1; else hi = mid;
  }
  pos[r] = lo;
}

// out[map[i] - base] = in[i] for kept i (elements of `es` bytes: 4 or 8)
__global__ void k_dist_take(const void* in, const uint32_t* map, uint64_t nl, uint64_t base,
                            uint32_t es, void* out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nl;
       i += uint64_t(gridDim.x) * blockDim.x) {
    if (map[i] == kNone) continue;
    const uint64_t o = map[i] - base;
    if (es == 8)
      static_cast<uint64_t*>(out)[o] = static_cast<const uint64_t*>(in)[i];
    else
      static_cast<uint32_t*>(out)[o] = static_cast<const uint32_t*>(in)[i];
  }
}

__global__ void k_dist_not_none(const uint32_t* map, uint64_t nl, uint32_t* flag) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nl;
       i += uint64_t(gridDim.x) * blockDim.x)
    flag[i] = map[i] != kNone ? 1u : 0u;
}

__global__ void k_dist_compact_rows(const uint64_t* deg, const uint32_t* keepf,
                                    const uint32_t* kpos, uint64_t nl, uint64_t* kdeg) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nl;
       i += uint64_t(gridDim.x) * blockDim.x)
    if (keepf[i]) kdeg[kpos[i]] = deg[i];
}

template <class T>
T scan_total(const T* in, T* out, uint64_t n) {
  if (!n) return T(0);
  size_t tmp = 0;
  DG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, stream()));
  DevBuf<char> t(tmp);
  DG_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, in, out, n, stream()));
  T a, b;
  d2h(&a, in + n - 1, 1);
  d2h(&b, out + n - 1, 1);
  stream_sync();
  return a + b;
}

}  // namespace
}  // namespace dgb

using namespace dgb;

extern "C" {

dg_status dg_dist_max_id(const uint64_t* u, const uint64_t* v, uint64_t k, uint64_t* out) {
  DG_API_BEGIN
  if (!out) throw DgError(DG_E_PARAM, "null argument");
  DevBuf<unsigned long long> m(1);
  m.zero();
  if (k) {
    k_dist_max<<<grid_for(k, 256), 256, 0, stream()>>>(u, v, k, m.get());
    DG_CHECK_LAUNCH();
  }
  *out = read_scalar(m.get());
  DG_API_END
}

dg_status dg_dist_endpoint_hist(const uint64_t* u, const uint64_t* v, uint64_t k, uint32_t shift,
                                uint32_t nb, uint64_t* hist) {
  DG_API_BEGIN
  if (!hist || nb == 0 || nb > 4096) throw DgError(DG_E_PARAM, "bad arguments");
  DevBuf<unsigned long long> h(nb);
  h.zero();
  if (k) {
    k_dist_hist<<<grid_for(k, 256), 256, 0, stream()>>>(u, v, k, shift, nb, h.get());
    DG_CHECK_LAUNCH();
  }
  d2h(reinterpret_cast<unsigned long long*>(hist), h.get(), nb);
  stream_sync();
  DG_API_END
}

dg_status dg_dist_route(const uint64_t* u, const uint64_t* v, uint64_t k,
                        const uint64_t* id_bounds, uint32_t P, uint64_t* keys, uint64_t* counts) {
  DG_API_BEGIN
  if (!id_bounds || !counts || P == 0 || P > kMaxRanks) throw DgError(DG_E_PARAM, "bad arguments");
  DevBuf<uint64_t> b(P + 1);
  h2d(b.get(), id_bounds, P + 1);
  DevBuf<unsigned long long> cnt(P);
  cnt.zero();
  if (k) {
    k_dist_count<<<grid_for(k, 256), 256, 0, stream()>>>(u, v, k, b.get(), P, cnt.get());
    DG_CHECK_LAUNCH();
  }
  std::vector<unsigned long long> h(P), cur(P);
  d2h(h.data(), cnt.get(), P);
  stream_sync();
  unsigned long long s = 0;
  for (uint32_t r = 0; r < P; ++r) {
    cur[r] = s;
    s += h[r];
    counts[r] = h[r];
  }
  if (k && s) {
    h2d(cnt.get(), cur.data(), P);
    k_dist_scatter<<<grid_for(k, 256), 256, 0, stream()>>>(u, v, k, b.get(), P, cnt.get(), keys);
    DG_CHECK_LAUNCH();
  }
  stream_sync();
  DG_API_END
}

dg_status dg_dist_rows(uint64_t* keys, uint64_t n, uint64_t* offs, uint64_t* verts,
                       uint32_t* dst, uint64_t* nverts, uint64_t* narcs) {
  DG_API_BEGIN
  if (!nverts || !narcs) throw DgError(DG_E_PARAM, "null argument");
  uint64_t m = 0, nv = 0;
  if (n) {
    // sort + unique (sorted keys = rows in source order, neighbours ascending)
    DevBuf<uint64_t> alt(n), uk(n);
    cub::DoubleBuffer<uint64_t> db(keys, alt.get());
    size_t tmp = 0;
    DG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, db, n, 0, 64, stream()));
    {
      DevBuf<char> t(tmp);
      DG_CUDA(cub::DeviceRadixSort::SortKeys(t.get(), tmp, db, n, 0, 64, stream()));
    }
    DevBuf<unsigned long long> cnt(1);
    tmp = 0;
    DG_CUDA(cub::DeviceSelect::Unique(nullptr, tmp, db.Current(), uk.get(), cnt.get(), n, stream()));
    {
      DevBuf<char> t(tmp);
      DG_CUDA(cub::DeviceSelect::Unique(t.get(), tmp, db.Current(), uk.get(), cnt.get(), n,
                                        stream()));
    }
    m = read_scalar(cnt.get());
    DevBuf<uint32_t> flag(m), pos(m);
    k_dist_src_flags<<<grid_for(m, 256), 256, 0, stream()>>>(uk.get(), m, flag.get(), dst);
    DG_CHECK_LAUNCH();
    nv = scan_total(flag.get(), pos.get(), m);
    k_dist_rows<<<grid_for(m, 256), 256, 0, stream()>>>(uk.get(), flag.get(), pos.get(), m, offs,
                                                        verts);
    DG_CHECK_LAUNCH();
  }
  h2d(offs + nv, &m, 1);
  stream_sync();
  *nverts = nv;
  *narcs = m;
  DG_API_END
}

dg_status dg_dist_unique(const uint32_t* vals, uint64_t n, uint32_t* uniq, uint32_t* inv,
                         uint64_t* nuniq) {
  DG_API_BEGIN
  if (!nuniq) throw DgError(DG_E_PARAM, "null argument");
  uint64_t nu = 0;
  if (n) {
    DevBuf<uint32_t> idx(n), sv(n), si(n), flag(n), pos(n);
    k_dist_iota<<<grid_for(n, 256), 256, 0, stream()>>>(idx.get(), n);
    DG_CHECK_LAUNCH();
    size_t tmp = 0;
    DG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, vals, sv.get(), idx.get(), si.get(), n,
                                            0, 32, stream()));
    {
      DevBuf<char> t(tmp);
      DG_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, vals, sv.get(), idx.get(), si.get(), n,
                                              0, 32, stream()));
    }
    k_dist_run_flags<<<grid_for(n, 256), 256, 0, stream()>>>(sv.get(), n, flag.get());
    DG_CHECK_LAUNCH();
    nu = scan_total(flag.get(), pos.get(), n);
    k_dist_inverse<<<grid_for(n, 256), 256, 0, stream()>>>(sv.get(), si.get(), flag.get(),
                                                           pos.get(), n, uniq, inv);
    DG_CHECK_LAUNCH();
    stream_sync();
  }
  *nuniq = nu;
  DG_API_END
}

dg_status dg_dist_lookup(const uint64_t* verts, uint64_t nv, const uint32_t* asked, uint64_t na,
                         uint64_t base, uint32_t* out) {
  DG_API_BEGIN
  if (na) {
    DevBuf<uint32_t> miss(1);
    miss.zero();
    k_dist_lookup<<<grid_for(na, 256), 256, 0, stream()>>>(verts, nv, asked, na, base, out,
                                                           miss.get());
    DG_CHECK_LAUNCH();
    if (read_scalar(miss.get())) throw DgError(DG_E_INVARIANT, "asked for a vertex its owner lacks");
  }
  DG_API_END
}

dg_status dg_dist_bucket_counts(const uint32_t* vals, uint64_t n, const uint64_t* id_bounds,
                                uint32_t P, uint64_t* counts) {
  DG_API_BEGIN
  if (!id_bounds || !counts || P == 0 || P > kMaxRanks) throw DgError(DG_E_PARAM, "bad arguments");
  DevBuf<uint64_t> b(P + 1);
  h2d(b.get(), id_bounds, P + 1);
  DevBuf<unsigned long long> pos(P + 1);
  k_dist_bucket<<<1, 128, 0, stream()>>>(vals, n, b.get(), P, pos.get());
  DG_CHECK_LAUNCH();
  std::vector<unsigned long long> h(P + 1);
  d2h(h.data(), pos.get(), P + 1);
  stream_sync();
  for (uint32_t r = 0; r < P; ++r) counts[r] = r + 1 < P ? h[r + 1] - h[r] : n - h[r];
  DG_API_END
}

dg_status dg_dist_take(const void* in, const uint32_t* map, uint64_t nl, uint64_t base,
                       uint32_t elem_bytes, void* out) {
  DG_API_BEGIN
  if (elem_bytes != 4 && elem_bytes != 8) throw DgError(DG_E_PARAM, "elements are 4 or 8 bytes");
  if (nl) {
    k_dist_take<<<grid_for(nl, 256), 256, 0, stream()>>>(in, map, nl, base, elem_bytes, out);
    DG_CHECK_LAUNCH();
    stream_sync();
  }
  DG_API_END
}

dg_status dg_dist_relabel(const uint32_t* back, const uint32_t* inv, uint64_t n, uint32_t* adj) {
  DG_API_BEGIN
  if (n) {
    k_dist_relabel<<<grid_for(n, 256), 256, 0, stream()>>>(back, inv, n, adj);
    DG_CHECK_LAUNCH();
    stream_sync();
  }
  DG_API_END
}

dg_status dg_dist_keep_map(const uint32_t* labels, uint64_t nl, uint32_t k, uint64_t base,
                           uint32_t* map, uint64_t* kept) {
  DG_API_BEGIN
  if (!kept) throw DgError(DG_E_PARAM, "null argument");
  uint64_t c = 0;
  if (nl) {
    DevBuf<uint32_t> flag(nl), pos(nl);
    k_dist_keep<<<grid_for(nl, 256), 256, 0, stream()>>>(labels, nl, k, flag.get());
    DG_CHECK_LAUNCH();
    c = scan_total(flag.get(), pos.get(), nl);
    k_dist_map<<<grid_for(nl, 256), 256, 0, stream()>>>(flag.get(), pos.get(), nl, base, map);
    DG_CHECK_LAUNCH();
    stream_sync();
  }
  *kept = c;
  DG_API_END
}

dg_status dg_dist_core_rows(const uint64_t* offs, const uint32_t* adj, uint64_t nl,
                            const uint32_t* local_map, const uint32_t* full_map,
                            uint64_t* noffs, uint32_t* nadj, uint64_t* nkept, uint64_t* narcs) {
  DG_API_BEGIN
  if (!narcs || !nkept) throw DgError(DG_E_PARAM, "null argument");
  uint64_t m = 0, kn = 0;
  if (nl) {
    DevBuf<uint32_t> keepf(nl), kpos(nl);
    DevBuf<uint64_t> deg(nl), kdeg(nl);
    k_dist_not_none<<<grid_for(nl, 256), 256, 0, stream()>>>(local_map, nl, keepf.get());
    DG_CHECK_LAUNCH();
    kn = scan_total(keepf.get(), kpos.get(), nl);
    k_dist_core_count<<<grid_for(nl * 32, 256), 256, 0, stream()>>>(offs, adj, nl, keepf.get(),
                                                                   full_map, deg.get());
    DG_CHECK_LAUNCH();
    if (kn) {
      k_dist_compact_rows<<<grid_for(nl, 256), 256, 0, stream()>>>(deg.get(), keepf.get(),
                                                                   kpos.get(), nl, kdeg.get());
      DG_CHECK_LAUNCH();
      m = scan_total(kdeg.get(), noffs, kn);
      k_dist_core_fill<<<grid_for(nl * 32, 256), 256, 0, stream()>>>(
          offs, adj, nl, keepf.get(), full_map, noffs, kpos.get(), nadj);
      DG_CHECK_LAUNCH();
    }
  }
  h2d(noffs + kn, &m, 1);
  stream_sync();
  *nkept = kn;
  *narcs = m;
  DG_API_END
}

}  // extern "C"
