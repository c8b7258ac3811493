// shard.cu -- one GPU's shard of a 1D vertex-range-partitioned coreness
// (SURVEY.md §8e).  Rank r owns the contiguous dense-id range [lo, hi): its
// residual degrees and labels; frontier expansion decrements owned
// neighbours in place (atomicSub crossing detection, as in kcore.cu) and
// buckets every remote neighbour id by its owner rank for the per-round
// exchange; received decrements are applied with the same crossing rule.
// The round / level protocol (frontier-size sum, min-degree agreement,
// decrement all-to-all) lives in paper_2311_04333_b200/sharded.py over NCCL.
//
// Peer mode (fused compute + exchange): the state the owners' decrements
// touch -- degrees, labels, the two frontier queues and their counters -- is
// ONE cudaMalloc'd block per shard, exported by CUDA IPC (or shared directly
// between shards of one process).  dg_shard_expand_peer decrements every
// neighbour at its owner with system-scope atomics over NVLink peer memory,
// and the decrement that crosses the bound labels the vertex and appends it
// to the owner's next-frontier queue: no send buffers, no all-to-all, one
// all-reduce (the produced crossings) per round.
#include <cstring>
#include <vector>

#include "shard.cuh"

namespace dgb {
namespace {

constexpr uint32_t kUnset = 0xffffffffu;

__global__ void k_sh_init(const uint64_t* offs, uint64_t nl, uint32_t* deg, uint32_t* labels) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nl;
       i += uint64_t(gridDim.x) * blockDim.x) {
    deg[i] = uint32_t(offs[i + 1] - offs[i]);
    labels[i] = kUnset;
  }
}

// local offsets of rows [lo, hi) of a global CSR (rebased to 0)
__global__ void k_sh_rebase(const uint64_t* goffs, uint64_t lo, uint64_t nl, uint64_t* loffs) {
  const uint64_t b = goffs[lo];
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i <= nl;
       i += uint64_t(gridDim.x) * blockDim.x)
    loffs[i] = goffs[lo + i] - b;
}

__global__ void k_sh_min(const uint32_t* deg, const uint32_t* labels, uint64_t nl,
                         unsigned long long* out) {
  uint32_t m = kUnset;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nl;
       i += uint64_t(gridDim.x) * blockDim.x)
    if (labels[i] == kUnset) m = min(m, deg[i]);
  m = __reduce_min_sync(~0u, m);
  if (lane_id() == 0 && m != kUnset) atomicMin(out, (unsigned long long)m);
}

__global__ void k_sh_collect(uint32_t* deg, uint32_t* labels, uint64_t nl, uint32_t bound,
                             uint32_t label, uint32_t* front, unsigned long long* cnt) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nl;
       i += uint64_t(gridDim.x) * blockDim.x)
    if (labels[i] == kUnset && deg[i] <= bound) {
      labels[i] = label;
      front[atomicAdd(cnt, 1ULL)] = uint32_t(i);
    }
}

__device__ __forceinline__ uint32_t owner_of(const uint64_t* bounds, uint32_t P, uint64_t u) {
  uint32_t r = 0;
  while (r + 1 < P && u >= bounds[r + 1]) ++r;
  return r;
}

// crossing rule of kcore.cu: the decrement that takes deg from bound+1 to
// bound enrols the vertex in the next round's frontier
__device__ __forceinline__ void dec_local(uint32_t* deg, uint32_t* labels, uint32_t i,
                                          uint32_t bound, uint32_t label, uint32_t* next,
                                          unsigned long long* cnt) {
  if (deg[i] <= bound) return;
  if (atomicSub(&deg[i], 1u) == bound + 1) {
    labels[i] = label;
    next[atomicAdd(cnt, 1ULL)] = i;
  }
}

// pass 1 (count) / pass 2 (fill + local decrements): warp per frontier vertex
template <bool FILL>
__global__ void k_sh_expand(const uint64_t* offs, const uint32_t* adj, uint64_t lo, uint64_t hi,
                            const uint32_t* front, uint64_t nfront, const uint64_t* bounds,
                            uint32_t P, uint32_t* deg, uint32_t* labels, uint32_t bound,
                            uint32_t label, uint32_t* next, unsigned long long* cnt,
                            unsigned long long* cursor, uint32_t* send) {
  const uint64_t warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t f = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; f < nfront;
       f += warps) {
    const uint64_t v = front[f];  // local row
    for (uint64_t p = offs[v] + lane_id(); p < offs[v + 1]; p += 32) {
      const uint64_t u = adj[p];
      if (u >= lo && u < hi) {
        if (FILL) dec_local(deg, labels, uint32_t(u - lo), bound, label, next, cnt);
      } else {
        const uint32_t r = owner_of(bounds, P, u);
        if (FILL)
          send[atomicAdd(&cursor[r], 1ULL)] = uint32_t(u);
        else
          atomicAdd(&cnt[2 + r], 1ULL);
      }
    }
  }
}

__global__ void k_sh_apply(const uint32_t* recv, uint64_t nrecv, uint64_t lo, uint32_t* deg,
                           uint32_t* labels, uint32_t bound, uint32_t label, uint32_t* next,
                           unsigned long long* cnt) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nrecv;
       i += uint64_t(gridDim.x) * blockDim.x)
    dec_local(deg, labels, uint32_t(recv[i] - lo), bound, label, next, cnt);
}

// Peer mode: warp per frontier vertex; every neighbour is decremented at its
// owner (peers[r] maps rank r's block: NVLink peer memory, or this GPU) with
// system-scope atomics; the crossing decrement labels the vertex and appends
// it to the owner's queue qn.  `produced` counts this shard's crossings (the
// per-round all-reduce sums them).
constexpr uint32_t kMaxPeers = 64;

__global__ void k_sh_expand_peer(const uint64_t* offs, const uint32_t* adj, const uint32_t* front,
                                 uint64_t nfront, const uint64_t* bounds, uint32_t P,
                                 const PeerView* peers, uint32_t bound, uint32_t label,
                                 uint32_t qn, unsigned long long* produced) {
  __shared__ uint64_t sb[kMaxPeers + 1];
  __shared__ PeerView sp[kMaxPeers];
  for (uint32_t i = threadIdx.x; i <= P; i += blockDim.x) sb[i] = bounds[i];
  for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) sp[i] = peers[i];
  __syncthreads();
  uint32_t made = 0;
  const uint64_t warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t f = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; f < nfront;
       f += warps) {
    const uint64_t v = front[f];  // local row
    for (uint64_t p = offs[v] + lane_id(); p < offs[v + 1]; p += 32) {
      const uint64_t u = adj[p];
      uint32_t r = 0;
      while (r + 1 < P && u >= sb[r + 1]) ++r;
      const PeerView& pv = sp[r];
      const uint32_t i = uint32_t(u - sb[r]);
      // a stale (higher) degree only costs an extra atomic: degrees only fall
      if (pv.deg[i] <= bound) continue;
      if (atomicSub_system(&pv.deg[i], 1u) == bound + 1) {
        pv.labels[i] = label;
        const unsigned long long slot = atomicAdd_system(&pv.ctr[qn], 1ULL);
        pv.q[qn][slot] = i;
        ++made;
      }
    }
  }
  __threadfence_system();  // peer stores visible before the round's barrier
  made = __reduce_add_sync(~0u, made);
  if (lane_id() == 0 && made) atomicAdd(produced, (unsigned long long)made);
}

}  // namespace
}  // namespace dgb

using namespace dgb;

extern "C" {

static void shard_init_state(dg_shard* s, const uint64_t* bounds, uint32_t P) {
  const uint64_t nl = s->hi - s->lo;
  DG_CUDA(cudaMalloc(&s->block, shard_block_bytes(nl)));
  s->own = shard_block_view(s->block, nl);
  DG_CUDA(cudaMemsetAsync(s->block, 0, 128 + sizeof(XCtrl), stream()));
  s->peers.assign(P, PeerView{});
  s->cnt.alloc(2 + P);
  s->bounds.alloc(P + 1);
  h2d(s->bounds.get(), bounds, P + 1);
  s->hbounds.assign(bounds, bounds + P + 1);
  if (nl) {
    k_sh_init<<<grid_for(nl, 256), 256, 0, stream()>>>(s->offs.get(), nl, s->own.deg,
                                                        s->own.labels);
    DG_CHECK_LAUNCH();
  }
  stream_sync();
}

static void shard_check(uint64_t n, const uint64_t* bounds, uint32_t P, uint32_t rank) {
  if (!bounds || rank >= P) throw DgError(DG_E_PARAM, "bad shard arguments");
  if (bounds[0] != 0 || bounds[P] != n) throw DgError(DG_E_PARAM, "bounds must cover [0, n)");
  for (uint32_t r = 0; r < P; ++r)
    if (bounds[r] > bounds[r + 1]) throw DgError(DG_E_PARAM, "bounds must ascend");
}

dg_status dg_shard_create(const dg_graph* g, const uint64_t* bounds, uint32_t P, uint32_t rank,
                          dg_shard** out) {
  DG_API_BEGIN
  if (!g || !out) throw DgError(DG_E_PARAM, "bad shard arguments");
  shard_check(g->n, bounds, P, rank);
  auto s = std::make_unique<dg_shard>();
  s->n = g->n;
  s->P = P;
  s->lo = bounds[rank];
  s->hi = bounds[rank + 1];
  s->rank = rank;
  const uint64_t nl = s->hi - s->lo;
  // the rank's own rows (the source graph may be freed afterwards)
  s->offs.alloc(nl + 1);
  k_sh_rebase<<<grid_for(nl + 1, 256), 256, 0, stream()>>>(g->offs.get(), s->lo, nl,
                                                            s->offs.get());
  DG_CHECK_LAUNCH();
  uint64_t a0 = 0, a1 = 0;
  d2h(&a0, g->offs.get() + s->lo, 1);
  d2h(&a1, g->offs.get() + s->hi, 1);
  stream_sync();
  s->adj.alloc(a1 - a0);
  if (a1 > a0)
    DG_CUDA(cudaMemcpyAsync(s->adj.get(), g->adj.get() + a0, (a1 - a0) * 4,
                            cudaMemcpyDeviceToDevice, stream()));
  shard_init_state(s.get(), bounds, P);
  s->peers[rank] = s->own;
  *out = s.release();
  DG_API_END
}

dg_status dg_shard_create_rows(uint64_t n, const uint64_t* bounds, uint32_t P, uint32_t rank,
                               const uint64_t* offs, const uint32_t* adj, int on_device,
                               dg_shard** out) {
  DG_API_BEGIN
  if (!out || !offs) throw DgError(DG_E_PARAM, "bad shard arguments");
  shard_check(n, bounds, P, rank);
  auto s = std::make_unique<dg_shard>();
  s->n = n;
  s->P = P;
  s->lo = bounds[rank];
  s->hi = bounds[rank + 1];
  s->rank = rank;
  const uint64_t nl = s->hi - s->lo;
  uint64_t o[2] = {0, 0};
  if (on_device) {
    d2h(&o[0], offs, 1);
    d2h(&o[1], offs + nl, 1);
    stream_sync();
  } else {
    o[0] = offs[0];
    o[1] = offs[nl];
  }
  if (o[1] < o[0]) throw DgError(DG_E_PARAM, "row offsets must ascend");
  s->offs.alloc(nl + 1);
  DevBuf<uint64_t> tmp(nl + 1);
  DG_CUDA(cudaMemcpyAsync(tmp.get(), offs, (nl + 1) * 8,
                          on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, stream()));
  k_sh_rebase<<<grid_for(nl + 1, 256), 256, 0, stream()>>>(tmp.get(), 0, nl, s->offs.get());
  DG_CHECK_LAUNCH();
  s->adj.alloc(o[1] - o[0]);
  if (o[1] > o[0]) {
    if (!adj) throw DgError(DG_E_PARAM, "null adjacency");
    DG_CUDA(cudaMemcpyAsync(s->adj.get(), adj, (o[1] - o[0]) * 4,
                            on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                            stream()));
  }
  shard_init_state(s.get(), bounds, P);
  s->peers[rank] = s->own;
  *out = s.release();
  DG_API_END
}

void dg_shard_free(dg_shard* s) {
  try {
    delete s;
  } catch (...) {
  }
}

dg_status dg_shard_min_alive(dg_shard* s, uint32_t* out) {
  DG_API_BEGIN
  const uint64_t nl = s->hi - s->lo;
  unsigned long long init = kUnset;
  h2d(s->cnt.get() + 1, &init, 1);
  if (nl) {
    k_sh_min<<<grid_for(nl, 256), 256, 0, stream()>>>(s->own.deg, s->own.labels, nl,
                                                       s->cnt.get() + 1);
    DG_CHECK_LAUNCH();
  }
  *out = uint32_t(read_scalar(s->cnt.get() + 1));
  DG_API_END
}

dg_status dg_shard_collect(dg_shard* s, uint32_t bound, uint32_t label, uint64_t* nfront) {
  DG_API_BEGIN
  const uint64_t nl = s->hi - s->lo;
  s->cnt.zero();
  if (nl) {
    k_sh_collect<<<grid_for(nl, 256), 256, 0, stream()>>>(s->own.deg, s->own.labels, nl,
                                                           bound, label, s->own.q[s->cur],
                                                           s->cnt.get());
    DG_CHECK_LAUNCH();
  }
  s->nfront = read_scalar(s->cnt.get());
  *nfront = s->nfront;
  DG_API_END
}

dg_status dg_shard_count_remote(dg_shard* s, uint64_t* counts) {
  DG_API_BEGIN
  s->cnt.zero();
  if (s->nfront) {
    k_sh_expand<false><<<grid_for(s->nfront * 32, 256), 256, 0, stream()>>>(
        s->offs.get(), s->adj.get(), s->lo, s->hi, s->own.q[s->cur], s->nfront,
        s->bounds.get(), s->P, s->own.deg, s->own.labels, 0, 0, nullptr, s->cnt.get(),
        nullptr, nullptr);
    DG_CHECK_LAUNCH();
  }
  std::vector<unsigned long long> h(s->P);
  d2h(h.data(), s->cnt.get() + 2, s->P);
  stream_sync();
  for (uint32_t r = 0; r < s->P; ++r) counts[r] = h[r];
  DG_API_END
}

dg_status dg_shard_expand(dg_shard* s, uint32_t bound, uint32_t label, const uint64_t* displs,
                          uint32_t* d_send) {
  DG_API_BEGIN
  DevBuf<unsigned long long> cur(s->P);
  std::vector<unsigned long long> h(displs, displs + s->P);
  h2d(cur.get(), h.data(), s->P);
  s->cnt.zero();
  if (s->nfront) {
    k_sh_expand<true><<<grid_for(s->nfront * 32, 256), 256, 0, stream()>>>(
        s->offs.get(), s->adj.get(), s->lo, s->hi, s->own.q[s->cur], s->nfront,
        s->bounds.get(), s->P, s->own.deg, s->own.labels, bound, label, s->own.q[s->cur ^ 1],
        s->cnt.get(), cur.get(), d_send);
    DG_CHECK_LAUNCH();
  }
  stream_sync();
  DG_API_END
}

dg_status dg_shard_apply(dg_shard* s, const uint32_t* d_recv, uint64_t nrecv, uint32_t bound,
                         uint32_t label, uint64_t* nnext) {
  DG_API_BEGIN
  if (nrecv) {
    k_sh_apply<<<grid_for(nrecv, 256), 256, 0, stream()>>>(d_recv, nrecv, s->lo, s->own.deg,
                                                           s->own.labels, bound, label,
                                                           s->own.q[s->cur ^ 1], s->cnt.get());
    DG_CHECK_LAUNCH();
  }
  s->nfront = read_scalar(s->cnt.get());
  s->cur ^= 1;
  *nnext = s->nfront;
  DG_API_END
}

// ---- peer mode
static void peer_set(dg_shard* s, uint32_t rank, void* block) {
  if (rank >= s->P) throw DgError(DG_E_PARAM, "peer rank out of range");
  s->peers[rank] = shard_block_view(block, s->hbounds[rank + 1] - s->hbounds[rank]);
  s->peers_ready = false;
}



dg_status dg_shard_ipc_handle(const dg_shard* s, void* handle) {
  DG_API_BEGIN
  if (!s || !handle) throw DgError(DG_E_PARAM, "null argument");
  cudaIpcMemHandle_t h;
  DG_CUDA(cudaIpcGetMemHandle(&h, s->block));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle, &h, sizeof h);
  DG_API_END
}

dg_status dg_shard_peer_open(dg_shard* s, uint32_t rank, const void* handle) {
  DG_API_BEGIN
  if (!s || !handle) throw DgError(DG_E_PARAM, "null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  void* p = nullptr;
  DG_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  s->opened.push_back(p);
  peer_set(s, rank, p);
  DG_API_END
}

dg_status dg_shard_peer_link(dg_shard* s, uint32_t rank, const dg_shard* other) {
  DG_API_BEGIN
  if (!s || !other) throw DgError(DG_E_PARAM, "null argument");
  if (other->P != s->P || other->n != s->n) throw DgError(DG_E_PARAM, "shards of different graphs");
  peer_set(s, rank, other->block);
  DG_API_END
}

dg_status dg_shard_expand_peer(dg_shard* s, uint32_t bound, uint32_t label, uint64_t* produced) {
  DG_API_BEGIN
  if (!s || !produced) throw DgError(DG_E_PARAM, "null argument");
  shard_device_peers(s);
  // the current queue's counter restarts: remote ranks append into this
  // queue only in the next round, after the round barrier
  DG_CUDA(cudaMemsetAsync(s->own.ctr + s->cur, 0, 8, stream()));
  s->cnt.zero();
  if (s->nfront) {
    k_sh_expand_peer<<<grid_for(s->nfront * 32, 256), 256, 0, stream()>>>(
        s->offs.get(), s->adj.get(), s->own.q[s->cur], s->nfront, s->bounds.get(), s->P,
        s->d_peers.get(), bound, label, s->cur ^ 1, s->cnt.get());
    DG_CHECK_LAUNCH();
  }
  *produced = read_scalar(s->cnt.get());
  DG_API_END
}

dg_status dg_shard_finish_round(dg_shard* s, uint64_t* nnext) {
  DG_API_BEGIN
  if (!s || !nnext) throw DgError(DG_E_PARAM, "null argument");
  s->nfront = read_scalar(s->own.ctr + (s->cur ^ 1));
  s->cur ^= 1;
  *nnext = s->nfront;
  DG_API_END
}

dg_status dg_shard_labels(const dg_shard* s, uint32_t* labels) {
  DG_API_BEGIN
  d2h(labels, s->own.labels, s->hi - s->lo);
  stream_sync();
  DG_API_END
}

}  // extern "C"

namespace dgb {
const PeerView* shard_device_peers(dg_shard* s) {
  if (s->P > 64) throw DgError(DG_E_PARAM, "peer mode supports at most 64 shards");
  if (!s->peers_ready) {
    for (const PeerView& v : s->peers)
      if (!v.deg) throw DgError(DG_E_PARAM, "peer mode needs every rank linked or opened");
    s->d_peers.alloc(s->P);
    h2d(s->d_peers.get(), s->peers.data(), s->P);
    s->peers_ready = true;
  }
  return s->d_peers.get();
}
}  // namespace dgb
