// graph_stream.cu -- CSR build straight from a device generator (gen.cuh), in
// source-range parts, without materialising the sample pairs.
//
// Same result as build_from_pairs on the generated pairs (io.cpp:51-92
// semantics: loops dropped, duplicates merged, dense id = rank of the original
// id among present ones, rows ascending) -- pinned by tests.  Memory is what
// lets BASELINE's largest configuration (RMAT-28, 4.3e9 samples, ~8.5e9 arcs)
// build on ONE B200: the pair arrays alone would be 69 GB and the global sorts
// of build_from_pairs need ~3x that.  Here:
//   pass 0   regenerate the samples: presence flags of the original ids and
//            per-bucket counts of arc emissions (both directions, loops out)
//   scan     dense ids = exclusive scan of the flags (rank table), orig ids
//   parts    bucket ranges cut so one part's emissions fit a budget; for each
//            part regenerate the samples and emit the arcs whose SOURCE lies in
//            the part as keys (src << B | dst), radix sort, unique: the part's
//            rows in order, neighbours ascending; offsets from the run starts,
//            adjacency appended.
// Peak memory ~ rank table + final adjacency + one part (3 x 8 B per emission).
#include <algorithm>
#include <vector>

#include <cub/cub.cuh>

#include "gen.cuh"

namespace dgb {

namespace {

constexpr uint32_t kNB = 8192;  // emission-count buckets over the original id range (32 KB of shared)

template <class Gen>
__global__ void k_presence(Gen gen, uint64_t k, uint32_t shift, uint32_t* flags,
                           unsigned long long* bcnt) {
  __shared__ uint32_t hist[kNB];
  for (uint32_t i = threadIdx.x; i < kNB; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  for (uint64_t s = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; s < k;
       s += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t a, b;
    gen(s, a, b);
    if (a == b) continue;  // self-loop: dropped (io.cpp:59)
    flags[a] = 1;
    flags[b] = 1;
    atomicAdd(&hist[a >> shift], 1u);
    atomicAdd(&hist[b >> shift], 1u);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < kNB; i += blockDim.x)
    if (hist[i]) atomicAdd(&bcnt[i], (unsigned long long)hist[i]);
}

__global__ void k_orig_from_flags(const uint32_t* flags, const uint32_t* rank, uint64_t R,
                                  uint64_t* orig) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < R;
       i += uint64_t(gridDim.x) * blockDim.x)
    if (flags[i]) orig[rank[i]] = i;
}

// arcs with source in [lo, hi) (original ids) as keys src << B | dst (dense)
template <class Gen>
__global__ void k_part_arcs(Gen gen, uint64_t k, const uint32_t* rank, uint64_t lo, uint64_t hi,
                            uint32_t B, uint64_t* out, unsigned long long* cnt) {
  for (uint64_t s0 = blockIdx.x * uint64_t(blockDim.x); s0 < k;
       s0 += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t s = s0 + threadIdx.x;
    uint64_t key[2];
    uint32_t nk = 0;
    if (s < k) {
      uint64_t a, b;
      gen(s, a, b);
      if (a != b) {
        if (a >= lo && a < hi) key[nk++] = (uint64_t(rank[a]) << B) | rank[b];
        if (b >= lo && b < hi) key[nk++] = (uint64_t(rank[b]) << B) | rank[a];
      }
    }
    // warp-aggregated append
    const uint32_t lane = lane_id();
    uint32_t incl = nk;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(~0u, incl, o);
      if (lane >= uint32_t(o)) incl += y;
    }
    const uint32_t tot = __shfl_sync(~0u, incl, 31);
    unsigned long long base = 0;
    if (lane == 31 && tot) base = atomicAdd(cnt, (unsigned long long)tot);
    base = __shfl_sync(~0u, base, 31);
    for (uint32_t j = 0; j < nk; ++j) out[base + incl - nk + j] = key[j];
  }
}

// sorted unique keys of one part -> row starts (offsets) and adjacency
__global__ void k_part_rows(const uint64_t* keys, uint64_t c, uint32_t B, uint64_t base,
                            uint64_t* offs, uint32_t* adj) {
  const uint64_t mask = (B == 64) ? ~0ULL : ((1ULL << B) - 1);
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < c;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t x = keys[i], row = x >> B;
    if (i == 0 || (keys[i - 1] >> B) != row) offs[row] = base + i;
    adj[base + i] = uint32_t(x & mask);
  }
}

uint32_t bits_for(uint64_t n) {
  uint32_t b = 1;
  while ((1ULL << b) < n) ++b;
  return b;
}

template <class Gen>
GraphPtr build_streamed(const Gen& gen, uint64_t k, uint64_t part_cap) {
  const unsigned T = 256;
  const uint64_t R = gen.id_bound();
  if (R == 0 || R > 0xffffffffULL)
    throw DgError(DG_E_PARAM, "generator ids must be below 2^32 for the streamed build");
  uint32_t shift = 0;
  while ((R - 1) >> shift >= kNB) ++shift;

  // pass 0: presence flags + emission counts per bucket
  DevBuf<uint32_t> flags(R), rank(R);
  flags.zero();
  DevBuf<unsigned long long> bcnt(kNB);
  bcnt.zero();
  if (k) {
    k_presence<<<num_sms() * 4, 512, 0, stream()>>>(gen, k, shift, flags.get(), bcnt.get());
    DG_CHECK_LAUNCH();
  }
  std::vector<unsigned long long> hb(kNB);
  d2h(hb.data(), bcnt.get(), kNB);
  size_t tmp = 0;
  DG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, flags.get(), rank.get(), R, stream()));
  {
    DevBuf<char> t(tmp);
    DG_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, flags.get(), rank.get(), R, stream()));
  }
  uint32_t lastf = 0, lastr = 0;
  d2h(&lastf, flags.get() + R - 1, 1);
  d2h(&lastr, rank.get() + R - 1, 1);
  stream_sync();
  const uint64_t n = uint64_t(lastf) + lastr;
  if (n == 0) throw DgError(DG_E_EMPTY, "no edges after removing self-loops and duplicates");
  if (n > 0xfffffffeULL) throw DgError(DG_E_PARAM, "more than 2^32-2 vertices");
  const uint32_t B = bits_for(n);
  uint64_t emissions = 0;
  for (auto c : hb) emissions += c;

  auto g = std::make_unique<dg_graph>();
  g->n = n;
  g->orig.alloc(n);
  k_orig_from_flags<<<grid_for(R, T), T, 0, stream()>>>(flags.get(), rank.get(), R,
                                                         g->orig.get());
  DG_CHECK_LAUNCH();
  flags.release();
  g->offs.alloc(n + 1);
  g->adj.alloc(emissions);  // upper bound of 2m (duplicates merge)

  // part budget (emissions): a third of the free memory over key + sort buffer + unique out
  size_t free_b = 0, total_b = 0;
  DG_CUDA(cudaMemGetInfo(&free_b, &total_b));
  uint64_t cap = part_cap ? part_cap : uint64_t(free_b / 3) / 24;
  cap = std::min<uint64_t>(cap, 1ULL << 31);
  DevBuf<unsigned long long> cnt(2);
  uint64_t base = 0;
  for (uint32_t b0 = 0; b0 < kNB;) {
    // widest bucket range within the budget (at least one bucket)
    uint64_t sz = hb[b0];
    uint32_t b1 = b0 + 1;
    while (b1 < kNB && sz + hb[b1] <= cap) sz += hb[b1++];
    if (sz > (1ULL << 31)) throw DgError(DG_E_NOMEM, "one id bucket exceeds the sort limit");
    if (sz) {
      const uint64_t lo = uint64_t(b0) << shift, hi = std::min<uint64_t>(uint64_t(b1) << shift, R);
      DevBuf<uint64_t> keys(sz), alt(sz), uniq(sz);
      cnt.zero();
      k_part_arcs<<<num_sms() * 8, T, 0, stream()>>>(gen, k, rank.get(), lo, hi, B, keys.get(),
                                                     cnt.get());
      DG_CHECK_LAUNCH();
      cub::DoubleBuffer<uint64_t> db(keys.get(), alt.get());
      tmp = 0;
      DG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, db, int64_t(sz), 0, int(2 * B),
                                             stream()));
      {
        DevBuf<char> t(tmp);
        DG_CUDA(cub::DeviceRadixSort::SortKeys(t.get(), tmp, db, int64_t(sz), 0, int(2 * B),
                                               stream()));
      }
      tmp = 0;
      DG_CUDA(cub::DeviceSelect::Unique(nullptr, tmp, db.Current(), uniq.get(), cnt.get() + 1,
                                        int64_t(sz), stream()));
      {
        DevBuf<char> t(tmp);
        DG_CUDA(cub::DeviceSelect::Unique(t.get(), tmp, db.Current(), uniq.get(), cnt.get() + 1,
                                          int64_t(sz), stream()));
      }
      const uint64_t c = read_scalar(cnt.get() + 1);
      k_part_rows<<<grid_for(c, T), T, 0, stream()>>>(uniq.get(), c, B, base, g->offs.get(),
                                                      g->adj.get());
      DG_CHECK_LAUNCH();
      base += c;
    }
    b0 = b1;
  }
  rank.release();
  h2d(g->offs.get() + n, &base, 1);
  stream_sync();
  if (base & 1) throw DgError(DG_E_INVARIANT, "streamed build: odd arc count");
  g->m = base / 2;
  g->maxdeg = device_max_degree(g->offs.get(), n);
  return g;
}

}  // namespace

GraphPtr build_rmat_streamed(uint32_t scale, uint64_t samples, uint64_t seed, uint64_t part_cap) {
  if (scale == 0 || scale > 32) throw DgError(DG_E_PARAM, "rmat scale must be in [1, 32]");
  return build_streamed(RmatGen{scale, mix64(seed ^ 0x524d4154ULL)}, samples, part_cap);
}

GraphPtr build_chung_lu_streamed(uint64_t n, uint64_t pairs, double R, uint64_t seed,
                                 uint64_t part_cap) {
  if (n == 0) throw DgError(DG_E_PARAM, "chung-lu needs n > 0");
  return build_streamed(ChungLuGen{n, R, mix64(seed ^ 0x434cULL)}, pairs, part_cap);
}

}  // namespace dgb
