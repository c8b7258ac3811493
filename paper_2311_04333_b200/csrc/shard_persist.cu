// shard_persist.cu -- the sharded coreness as ONE persistent kernel per GPU
// (SURVEY.md §8e): the round loop of core.cpp:89-119 runs on the device, the
// decrement exchange is fused into the expansion (system-scope atomics on the
// owners' degrees through peer memory -- NVLink peer mappings across GPUs),
// and rounds are separated by a device-side barrier across shards instead of
// host round trips and collectives.
//
// Each shard is served by a GROUP of CTAs: on a multi-GPU job one group per
// GPU (the whole GPU), on one GPU any number of groups in one cooperative
// launch (every CTA co-resident, so the cross-group barrier cannot deadlock;
// tests run P shards this way).  Per round, with b the bound:
//
//   expand   warps take the group's frontier entries (its queue) dynamically;
//            rows longer than kPiece arcs are cut into pieces taken after a
//            group barrier; every arc decrements its target at the owner
//            (atomicSub / atomicSub_system); the decrement that lands the
//            degree on b labels the vertex and appends it to the OWNER's next
//            queue (atomicAdd_system on its counter).
//   barrier  group barrier, then the group leader arrives at the cross-shard
//            flip barrier in shard 0's control block (XCtrl) adding its
//            crossings, spins, reads the global sum; group barrier.
//   level    when the global frontier is empty: each group scans its live
//            list (min alive degree, compaction), cross-shard min, the new
//            bound (exact: the min; approximate: the geometric phases of
//            core.cpp:105-110), each group collects its vertices at the bound
//            into its queue, cross-shard sum.
//
// peel_rounds counts non-empty global rounds, kmax the last label: the same
// values as the single-GPU kernel and the reference.
#include <cstring>
#include <vector>

#include "shard.cuh"

namespace dgb {
namespace {

constexpr uint32_t kUnset = 0xffffffffu;
constexpr uint32_t kThreads = 512;
constexpr uint64_t kPiece = 128;   // arcs per piece (one warp step of 4 arcs per lane)
constexpr int kTiny = 4;           // rows of at most kTiny arcs: one thread each
constexpr uint64_t kHub = 512 * kPiece;  // longer rows: shared by every warp of the group
constexpr uint32_t kMaxP = 64;
#ifndef DG_SP_PROF
#define DG_SP_PROF 0  // tuning build: group-0 phase cycles into out[3..9]
#endif

struct GroupShard {  // one per group of this launch
  const uint64_t* offs;  // local rows (local offsets), nl + 1
  const uint32_t* adj;   // global neighbour ids
  uint64_t lo, nl;
  uint32_t rank;         // global shard index
  PeerView own;
  uint32_t* live[2];     // live lists (local ids), nl each
  uint64_t* piece;       // pieces of medium rows: (start, end) arc pairs
  uint64_t piece_cap;
  uint64_t* hub;         // rows longer than kHub: (start, end) pairs
  GridBarrier* bar;      // group barrier
  unsigned long long* wk;  // [16] group scratch (work counters, group reductions)
};

struct PArgs {
  GroupShard* gs;  // [G]
  uint32_t G, P, per;  // groups here, shards in all, CTAs per group
  const PeerView* peers;
  const uint64_t* bounds;  // P + 1
  XCtrl* x;                // shard 0's control block (mapped here)
  uint64_t n;
  int approx;
  uint64_t c_num, c_den;
  uint32_t* out;  // kmax, rounds, err (written by group 0)
  int sys;        // some shard lives in another process / GPU: system-scope sync
};

// work-counter slots in GroupShard::wk, rotated by round parity where a slot
// is reset one phase before its next use
enum : int { W_HUB = 0, W_PCN = 4, W_LIVE = 6, W_GMIN = 8, W_GSUM = 10 };
// W_GMIN / W_GSUM are used by the phase ending in cross-shard episode e at
// slot (e & 1) and reset by the leader right after that episode, W_LIVE is
// reset once every CTA read it (after the collect's group barrier)

__device__ __forceinline__ uint32_t gsync(GroupShard& g, uint32_t per, uint32_t rel,
                                          uint32_t* s_abort, bool sysfence = false) {
  // group barrier: grid_sync over the group's CTAs (group-relative CTA 0 leads)
  __syncthreads();
  if (threadIdx.x == 0) {
    // after the CTA barrier, one system-scope fence per CTA covers every
    // thread's peer-memory writes of the phase (cumulativity)
    if (sysfence) __threadfence_system();
    const uint32_t add = rel == 0 ? 0x80000000u - (per - 1) : 1u;
    uint32_t old;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], %2;"
                 : "=r"(old)
                 : "l"(&g.bar->count), "r"(add)
                 : "memory");
    const long long t0 = clock64();
    uint32_t spins = 0;
    while (((old ^ ld_acquire_u32(&g.bar->count)) & 0x80000000u) == 0) {
      if ((++spins & 1023u) == 0) {
        if (ld_relaxed_u32(&g.bar->abort)) break;
        if (clock64() - t0 > ((long long)(g.bar->timeout_s ? g.bar->timeout_s : 60u) << 31)) {
          atomicExch(&g.bar->abort, 1u);
          break;
        }
      }
    }
    *s_abort = ld_relaxed_u32(&g.bar->abort);
  }
  __syncthreads();
  return *s_abort;
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct Shared {
  GroupShard g;  // this group's shard (copied: asm memory clobbers would
                 // otherwise re-read every field from global memory)
  uint64_t bounds[kMaxP + 1];
  PeerView peers[kMaxP];
  uint32_t abort;
  unsigned long long xsum;  // results of the last cross-shard episode
  uint32_t xmin;
  unsigned long long csum;  // this CTA's contribution to the next episode
  uint32_t cmin;
  unsigned long long ws[33];
  unsigned long long base;
};

// Flat barrier over every CTA of the launch on a flip word (the launch holds
// every shard: one GPU).  Thread 0 only; returns false on abort.
__device__ __forceinline__ bool flat_arrive(uint32_t* word, uint32_t* abort_w, uint32_t timeout_s) {
  const uint32_t add = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
  uint32_t old;
  asm volatile("atom.add.release.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(word), "r"(add) : "memory");
  const long long t0 = clock64();
  uint32_t spins = 0;
  while (((old ^ ld_acquire_u32(word)) & 0x80000000u) == 0) {
    if ((++spins & 1023u) == 0) {
      if (ld_relaxed_u32(abort_w)) return false;
      if (clock64() - t0 > ((long long)(timeout_s ? timeout_s : 60u) << 31)) {
        atomicExch(abort_w, 1u);
        return false;
      }
    }
  }
  return true;
}

// Cross-shard episode: every CTA of every group calls it after adding its
// share to s.csum / s.cmin; afterwards s.xsum / s.xmin hold the global sum /
// min over all shards.  One launch holding every shard: one flat barrier of
// all CTAs.  Shards in other processes (multi-GPU): group barrier, the group
// leader meets the other leaders in shard 0's control block with
// system-scope atomics, group barrier.
__device__ bool xsync(const PArgs& a, GroupShard& g, uint32_t rel, uint32_t& episode, Shared& s) {
  XCtrl* x = a.x;
  const uint32_t e = episode & 3u;
  ++episode;
  if (!a.sys) {
    __syncthreads();
    if (threadIdx.x == 0) {
      if (s.csum) atomicAdd(&x->sum[e], s.csum);
      if (s.cmin != kUnset) atomicMin(&x->minv[e], s.cmin);
      s.abort = !flat_arrive(&x->arrive, &x->abort, g.bar->timeout_s);
      s.xsum = *reinterpret_cast<volatile unsigned long long*>(&x->sum[e]);
      s.xmin = *reinterpret_cast<volatile unsigned int*>(&x->minv[e]);
      // slot e + 2 is written again only after every CTA passed episode e + 1
      if (blockIdx.x == 0) {
        x->sum[(e + 2) & 3u] = 0;
        x->minv[(e + 2) & 3u] = kUnset;
      }
      s.csum = 0;
      s.cmin = kUnset;
    }
    __syncthreads();
    return !s.abort;
  }
  unsigned long long* gs = &g.wk[W_GSUM + (e & 1u)];
  unsigned long long* gm = &g.wk[W_GMIN + (e & 1u)];
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s.csum) atomicAdd(gs, s.csum);
    if (s.cmin != kUnset) atomicMin(gm, (unsigned long long)s.cmin);
    s.csum = 0;
    s.cmin = kUnset;
  }
  if (gsync(g, a.per, rel, &s.abort, true)) return false;
  if (rel == 0 && threadIdx.x == 0) {
    const unsigned long long gsum = *reinterpret_cast<volatile unsigned long long*>(gs);
    const uint32_t gmin = uint32_t(*reinterpret_cast<volatile unsigned long long*>(gm));
    *gs = 0;  // only the leader reads the group slots
    *gm = kUnset;
    if (gsum) atomicAdd_system(&x->sum[e], gsum);
    if (gmin != kUnset) atomicMin_system(&x->minv[e], gmin);
    const uint32_t add = g.rank == 0 ? 0x80000000u - (a.P - 1) : 1u;
    uint32_t old;
    asm volatile("atom.add.release.sys.u32 %0, [%1], %2;"
                 : "=r"(old)
                 : "l"(&x->arrive), "r"(add)
                 : "memory");
    const long long t0 = clock64();
    uint32_t spins = 0;
    while (((old ^ ld_acquire_sys(&x->arrive)) & 0x80000000u) == 0) {
      if ((++spins & 1023u) == 0) {
        if (ld_acquire_sys(&x->abort)) break;
        if (clock64() - t0 > ((long long)(g.bar->timeout_s ? g.bar->timeout_s : 60u) << 31)) {
          atomicExch_system(&x->abort, 1u);
          break;
        }
      }
    }
    if (ld_relaxed_u32(&x->abort)) atomicExch(&g.bar->abort, 1u);
    g.wk[14] = *reinterpret_cast<volatile unsigned long long*>(&x->sum[e]);
    g.wk[15] = *reinterpret_cast<volatile unsigned int*>(&x->minv[e]);
    if (g.rank == 0) {
      x->sum[(e + 2) & 3u] = 0;
      x->minv[(e + 2) & 3u] = kUnset;
    }
  }
  if (gsync(g, a.per, rel, &s.abort)) return false;
  if (threadIdx.x == 0) {
    s.xsum = *reinterpret_cast<volatile unsigned long long*>(&g.wk[14]);
    s.xmin = uint32_t(*reinterpret_cast<volatile unsigned long long*>(&g.wk[15]));
  }
  __syncthreads();
  return true;
}

// barrier over the group's CTAs (one launch holding every shard: all CTAs)
__device__ __forceinline__ bool bsync(const PArgs& a, GroupShard& g, uint32_t rel, Shared& s) {
  if (!a.sys) {
    __syncthreads();
    if (threadIdx.x == 0) s.abort = !flat_arrive(&a.x->arrive2, &a.x->abort, g.bar->timeout_s);
    __syncthreads();
    return !s.abort;
  }
  return gsync(g, a.per, rel, &s.abort) == 0;
}

// Decrement K targets per lane (global ids; act = present) at their owners:
// device-scope atomics for this shard's own vertices after a cached degree
// test, system-scope atomics -- NVLink for another GPU -- for the others.
// The decrement that lands a degree on the bound labels the vertex and
// appends it to the owner's (append-only) queue, warp-aggregated per owner.  All K loads
// and atomics of a lane are in flight together.  Returns this lane's
// crossings.  Every lane of the warp must call it (warp-collective).
template <int K>
__device__ __forceinline__ uint32_t process_targets(const Shared& s, uint32_t P, uint32_t me,
                                                   bool (&act)[K], const uint32_t (&u)[K],
                                                   uint32_t bound, uint32_t label) {
  const uint32_t lane = lane_id();
  uint32_t own[K], idx[K], old[K], made = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    own[k] = 0;
    idx[k] = 0;
    if (act[k]) {
      uint32_t lo = 0, hi = P - 1;  // owner: largest r with bounds[r] <= u
      while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (s.bounds[mid] <= u[k]) lo = mid; else hi = mid - 1;
      }
      own[k] = lo;
      idx[k] = uint32_t(u[k] - s.bounds[lo]);
    }
  }
#pragma unroll
  for (int k = 0; k < K; ++k)  // own targets: skip the dead (degree at/below the bound)
    if (act[k] && own[k] == me) act[k] = __ldcg(&s.peers[me].deg[idx[k]]) > bound;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    old[k] = 0;
    if (!act[k]) continue;
    // a remote dead target's degree is already <= bound and only falls, so
    // the crossing test never fires for it: no remote liveness load
    old[k] = own[k] == me ? atomicSub(&s.peers[me].deg[idx[k]], 1u)
                          : atomicSub_system(&s.peers[own[k]].deg[idx[k]], 1u);
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const bool cross = act[k] && old[k] == bound + 1;
    if (!__any_sync(~0u, cross)) continue;
    const uint32_t grp = __match_any_sync(~0u, cross ? own[k] : 0xffffffffu);
    const uint32_t leader = __ffs(grp) - 1;
    const PeerView& pv = s.peers[own[k]];
    unsigned long long base = 0;
    if (cross && lane == leader)
      base = atomicAdd_system(&pv.ctr[0], (unsigned long long)__popc(grp));
    base = __shfl_sync(~0u, base, leader);
    if (cross) {
      pv.labels[idx[k]] = label;
      pv.q[0][base + __popc(grp & ((1u << lane) - 1u))] = idx[k];
      ++made;
    }
  }
  return made;
}

// arcs [st, en) of a row, 4 per lane per step (warp-collective)
__device__ __forceinline__ uint32_t expand_arcs(const Shared& s, const uint32_t* adj, uint32_t P,
                                                uint32_t me, uint64_t st, uint64_t en,
                                                uint32_t bound, uint32_t label) {
  constexpr int K = 4;
  uint32_t made = 0;
  for (uint64_t j0 = st; j0 < en; j0 += 32 * K) {
    bool act[K];
    uint32_t u[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t j = j0 + k * 32 + lane_id();
      act[k] = j < en;
      u[k] = act[k] ? adj[j] : 0u;
    }
    made += process_targets<K>(s, P, me, act, u, bound, label);
  }
  return made;
}

// Block-aggregated append: threads with `flag` write `val` to dst[base + i]
// where base comes from one atomicAdd on *ctr per call (all threads call).
__device__ __forceinline__ void block_append(bool flag, uint32_t val, unsigned long long* ctr,
                                             uint32_t* dst, Shared& s) {
  unsigned long long tot;
  const unsigned long long ex = block_excl_scan<unsigned long long>(flag ? 1ULL : 0ULL, s.ws, &tot);
  if (threadIdx.x == 0 && tot) s.base = atomicAdd(ctr, tot);
  __syncthreads();
  if (flag) dst[s.base + ex] = val;
  __syncthreads();  // ws / base reuse
}

__global__ void __launch_bounds__(kThreads, 1) k_shard_coreness(PArgs a) {
  __shared__ Shared s;
  const uint32_t grp = blockIdx.x / a.per, rel = blockIdx.x % a.per;
  if (threadIdx.x == 0) {
    s.g = a.gs[grp];
    s.csum = 0;
    s.cmin = kUnset;
  }
  GroupShard& g = s.g;
  for (uint32_t i = threadIdx.x; i <= a.P; i += blockDim.x) s.bounds[i] = a.bounds[i];
  for (uint32_t i = threadIdx.x; i < a.P; i += blockDim.x) s.peers[i] = a.peers[i];
  __syncthreads();
  const uint32_t me = g.rank, lane = lane_id();
  const uint64_t gthreads = uint64_t(a.per) * blockDim.x;
  const uint64_t gtid = uint64_t(rel) * blockDim.x + threadIdx.x;
  const uint64_t gwarps = gthreads >> 5, gwarp = gtid >> 5;
  uint32_t episode = 0, lv = 0;
  uint64_t livec = g.nl;
  bool implicit = true;
  // the queue is append-only for the whole run (a vertex enters a frontier
  // once in its life): the current frontier is q[head, tail)
  uint64_t head = 0, tail = 0;
  uint64_t bound = 0, label = 0, t = 1, remaining = a.n, total = 0;
  uint32_t kmax = 0, rounds = 0, err = 0;
  const bool L = rel == 0 && threadIdx.x == 0;  // group leader
  long long pc[7] = {}, tp = clock64();
  auto mark = [&](int k) {
    if (DG_SP_PROF && L && grp == 0) {
      const long long tt = clock64();
      pc[k] += tt - tp;
      tp = tt;
    }
  };
  uint32_t* q = g.own.q[0];
  unsigned long long* qctr = &g.own.ctr[0];

  for (uint64_t guard = 0;; ++guard) {
    if (guard > 4 * a.n + 64) { err = 1; break; }
    if (total == 0) {
      if (remaining == 0) break;
      // ---- level advance: min alive degree + compaction of the live list
      uint32_t lmin = kUnset;
      const uint32_t* lin = g.live[lv];
      uint32_t* lout = g.live[lv ^ 1];
      unsigned long long* lc = &g.wk[W_LIVE];
      // labels / degrees are written by other shards (peer memory): L2 loads
      for (uint64_t b0 = uint64_t(rel) * blockDim.x; b0 < livec;
           b0 += uint64_t(a.per) * blockDim.x) {  // CTA-uniform bound
        const uint64_t i = b0 + threadIdx.x;
        uint32_t v = 0;
        bool alive = false;
        if (i < livec) {
          v = implicit ? uint32_t(i) : lin[i];
          const uint32_t d = __ldcg(&g.own.deg[v]);
          alive = __ldcg(&g.own.labels[v]) == kUnset;
          if (alive) lmin = min(lmin, d);
        }
        block_append(alive, v, lc, lout, s);
      }
      mark(0);
      lmin = __reduce_min_sync(~0u, lmin);
      if (lane == 0 && lmin != kUnset) atomicMin(&s.cmin, lmin);
      if (!xsync(a, g, rel, episode, s)) { err = 4; break; }
      livec = *reinterpret_cast<volatile unsigned long long*>(lc);
      lv ^= 1;
      implicit = false;
      const uint64_t gmin = s.xmin;
      if (gmin == kUnset) { err = 2; break; }
      while (gmin > bound) {
        if (!a.approx) {
          bound = gmin;
          label = gmin;
        } else {  // core.cpp:105-110
          label = t;
          const uint64_t ct = (t * a.c_num) / a.c_den + ((t * a.c_num) % a.c_den != 0);
          const uint64_t nt = t + 1 > ct ? t + 1 : ct;
          bound = nt - 1;
          t = nt;
        }
      }
      // collect: alive vertices at or below the bound join the queue
      uint32_t made = 0;
      const uint32_t* l2 = g.live[lv];
      for (uint64_t b0 = uint64_t(rel) * blockDim.x; b0 < livec;
           b0 += uint64_t(a.per) * blockDim.x) {
        const uint64_t i = b0 + threadIdx.x;
        bool hit = false;
        uint32_t v = 0;
        if (i < livec) {
          v = l2[i];
          hit = __ldcg(&g.own.labels[v]) == kUnset && __ldcg(&g.own.deg[v]) <= bound;
          if (hit) g.own.labels[v] = uint32_t(label);
        }
        made += hit;
        block_append(hit, v, qctr, q, s);
      }
      made = __reduce_add_sync(~0u, made);
      if (lane == 0 && made) atomicAdd(&s.csum, (unsigned long long)made);
      if (!xsync(a, g, rel, episode, s)) { err = 4; break; }
      if (L) g.wk[W_LIVE] = 0;  // every CTA read livec before the collect
      total = s.xsum;
      if (total == 0) { err = 3; break; }
      tail = *reinterpret_cast<volatile unsigned long long*>(qctr);
      mark(1);
    }
    // ---- round: expand q[head, tail); crossings are appended at the owners
    ++rounds;
    if (label > kmax) kmax = uint32_t(label);
    remaining -= total;
    const uint64_t nq = tail - head;
    const uint32_t* fq = q + head;
    const uint32_t b32 = uint32_t(bound), l32 = uint32_t(label);
    unsigned long long* pcn = &g.wk[W_PCN + (rounds & 1)];
    unsigned long long* nhub = &g.wk[W_HUB + (rounds & 1)];
    uint32_t made = 0;
    // entries, one per thread: rows of <= kTiny arcs are decremented by
    // their thread; rows up to kHub arcs are cut into kPiece-arc pieces
    // (written by their thread); longer rows go to the hub list
    for (uint64_t b0 = gtid - lane; b0 < nq; b0 += gthreads) {  // warp-uniform
      const uint64_t e = b0 + lane;
      uint64_t r0 = 0, r1 = 0;
      if (e < nq) {
        const uint32_t v = __ldcg(&fq[e]);
        r0 = g.offs[v];
        r1 = g.offs[v + 1];
      }
      const uint64_t d = r1 - r0;
      bool act[kTiny];
      uint32_t u[kTiny];
#pragma unroll
      for (int k = 0; k < kTiny; ++k) {
        act[k] = d <= kTiny && k < d;
        u[k] = act[k] ? g.adj[r0 + k] : 0u;
      }
      made += process_targets<kTiny>(s, a.P, me, act, u, b32, l32);
      const uint32_t np = (d > kTiny && d <= kHub) ? uint32_t((d + kPiece - 1) / kPiece) : 0u;
      const uint32_t inc = warp_incl_scan(np), tot = __shfl_sync(~0u, inc, 31);
      unsigned long long at = 0;
      if (lane == 31 && tot) at = atomicAdd(pcn, (unsigned long long)tot);
      at = __shfl_sync(~0u, at, 31) + (inc - np);
      for (uint32_t k = 0; k < np; ++k) {
        g.piece[2 * (at + k)] = r0 + uint64_t(k) * kPiece;
        g.piece[2 * (at + k) + 1] = min(r0 + uint64_t(k + 1) * kPiece, r1);
      }
      const bool hub = d > kHub;
      const uint32_t hm = __ballot_sync(~0u, hub);
      unsigned long long hb = 0;
      if (hm && lane == __ffs(hm) - 1) hb = atomicAdd(nhub, (unsigned long long)__popc(hm));
      hb = __shfl_sync(~0u, hb, __ffs(hm ? hm : 1u) - 1);
      if (hub) {
        const uint64_t h = hb + __popc(hm & ((1u << lane) - 1u));
        g.hub[2 * h] = r0;
        g.hub[2 * h + 1] = r1;
      }
    }
    mark(2);
    if (!bsync(a, g, rel, s)) { err = 4; break; }
    mark(3);
    const unsigned long long npc = __ldcg(pcn), nh = __ldcg(nhub);
    for (uint64_t e = gwarp; e < npc; e += gwarps)
      made += expand_arcs(s, g.adj, a.P, me, g.piece[2 * e], g.piece[2 * e + 1], b32, l32);
    for (uint64_t h = 0; h < nh; ++h) {  // every warp takes a share of every hub row
      const uint64_t r0 = __ldcg(&g.hub[2 * h]), r1 = __ldcg(&g.hub[2 * h + 1]);
      for (uint64_t st = r0 + gwarp * kPiece; st < r1; st += gwarps * kPiece)
        made += expand_arcs(s, g.adj, a.P, me, st, min(st + kPiece, r1), b32, l32);
    }
    mark(4);
    made = __reduce_add_sync(~0u, made);
    if (lane == 0 && made) atomicAdd(&s.csum, (unsigned long long)made);
    if (L) {  // the next round's piece / hub counts (used two rounds ago)
      g.wk[W_PCN + ((rounds + 1) & 1)] = 0;
      g.wk[W_HUB + ((rounds + 1) & 1)] = 0;
    }
    if (!xsync(a, g, rel, episode, s)) { err = 4; break; }
    total = s.xsum;
    head = tail;
    tail = *reinterpret_cast<volatile unsigned long long*>(qctr);  // every append is done
    mark(5);
  }
  if (grp == 0 && rel == 0 && threadIdx.x == 0) {
    a.out[0] = kmax;
    a.out[1] = rounds;
    a.out[2] = err;
    if (DG_SP_PROF)
      for (int k = 0; k < 6; ++k) a.out[3 + k] = uint32_t(pc[k] >> 10);  // kilocycles
  }
}

__global__ void k_ps_init(const uint64_t* offs, uint64_t nl, uint32_t* deg, uint32_t* labels) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nl;
       i += uint64_t(gridDim.x) * blockDim.x) {
    deg[i] = uint32_t(offs[i + 1] - offs[i]);
    labels[i] = kUnset;
  }
}

__global__ void k_ps_wk_init(unsigned long long* wk, GridBarrier* bar, uint32_t timeout_s) {
  if (threadIdx.x < 16)
    wk[threadIdx.x] = (threadIdx.x == W_GMIN || threadIdx.x == W_GMIN + 1) ? kUnset : 0ULL;
  if (threadIdx.x == 0) *bar = GridBarrier{0, 0, 0, timeout_s};
}

__global__ void k_ps_x_init(XCtrl* x) {
  if (threadIdx.x == 0) {
    x->arrive = 0;
    x->arrive2 = 0;
    x->abort = 0;
    for (int e = 0; e < 4; ++e) {
      x->sum[e] = 0;
      x->minv[e] = kUnset;
    }
  }
}

}  // namespace
}  // namespace dgb

using namespace dgb;

extern "C" {

dg_status dg_shard_xctrl_reset(dg_shard* s) {
  DG_API_BEGIN
  if (!s) throw DgError(DG_E_PARAM, "null argument");
  k_ps_x_init<<<1, 32, 0, stream()>>>(s->own.x);
  DG_CHECK_LAUNCH();
  stream_sync();
  DG_API_END
}

dg_status dg_shard_coreness_persistent(dg_shard** shards, uint32_t count, int approx,
                                       uint64_t c_num, uint64_t c_den, uint32_t* kmax,
                                       uint32_t* rounds, float* kernel_ms) {
  DG_API_BEGIN
  if (!shards || count == 0 || !kmax || !rounds) throw DgError(DG_E_PARAM, "null argument");
  if (approx && (c_den == 0 || c_num <= c_den))
    throw DgError(DG_E_PARAM, "approximation factor must be > 1");
  dg_shard* s0 = shards[0];
  const uint32_t P = s0->P;
  if (P > kMaxP) throw DgError(DG_E_PARAM, "at most 64 shards");
  if (count > P) throw DgError(DG_E_PARAM, "more shards than the partition has");
  for (uint32_t k = 0; k < count; ++k)
    if (shards[k]->P != P || shards[k]->n != s0->n) throw DgError(DG_E_PARAM, "shards of different graphs");
  const PeerView* d_peers = shard_device_peers(s0);
  // every shard of this process sees the same peer views (its own block is
  // its entry); the control block is shard 0's as mapped here
  const XCtrl* x = s0->peers[0].x;
  // per-shard state: degrees, labels, queues reset; live lists, pieces
  std::vector<GroupShard> hg(count);
  std::vector<DevBuf<uint32_t>> lives;
  std::vector<DevBuf<uint64_t>> pieces;
  DevBuf<unsigned long long> wk(16 * count);
  DevBuf<GridBarrier> bars(count);
  for (uint32_t k = 0; k < count; ++k) {
    dg_shard* s = shards[k];
    const uint64_t nl = s->hi - s->lo;
    if (nl) {
      k_ps_init<<<grid_for(nl, 256), 256, 0, stream()>>>(s->offs.get(), nl, s->own.deg,
                                                          s->own.labels);
      DG_CHECK_LAUNCH();
    }
    DG_CUDA(cudaMemsetAsync(s->own.ctr, 0, 16, stream()));
    lives.emplace_back(nl ? nl : 1);
    lives.emplace_back(nl ? nl : 1);
    uint64_t arcs = 0;
    d2h(&arcs, s->offs.get() + nl, 1);
    stream_sync();
    const uint64_t cap = arcs / kPiece + nl + 1;
    pieces.emplace_back(2 * cap);
    pieces.emplace_back(2 * (nl + 1));
    k_ps_wk_init<<<1, 32, 0, stream()>>>(wk.get() + 16 * k, bars.get() + k, barrier_timeout_s());
    DG_CHECK_LAUNCH();
    GroupShard& gsh = hg[k];
    gsh.offs = s->offs.get();
    gsh.adj = s->adj.get();
    gsh.lo = s->lo;
    gsh.nl = nl;
    gsh.rank = s->rank;
    gsh.own = s->own;
    gsh.live[0] = lives[2 * k].get();
    gsh.live[1] = lives[2 * k + 1].get();
    gsh.piece = pieces[2 * k].get();
    gsh.hub = pieces[2 * k + 1].get();
    gsh.piece_cap = cap;
    gsh.bar = bars.get() + k;
    gsh.wk = wk.get() + 16 * k;
  }
  DevBuf<GroupShard> dg(count);
  h2d(dg.get(), hg.data(), count);
  DevBuf<uint32_t> out(10);
  out.zero();
  int occ = 0;
  DG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_shard_coreness, kThreads, 0));
  const uint32_t slots = uint32_t(occ) * uint32_t(num_sms());
  const uint32_t per = slots / count;
  if (per == 0) throw DgError(DG_E_PARAM, "more shards than co-resident CTAs");
  PArgs a{dg.get(), count, P, per, d_peers, s0->bounds.get(), const_cast<XCtrl*>(x), s0->n,
          approx ? 1 : 0, c_num, c_den, out.get(), count < P ? 1 : 0};
  void* params[] = {&a};
  cudaEvent_t e0, e1;
  DG_CUDA(cudaEventCreate(&e0));
  DG_CUDA(cudaEventCreate(&e1));
  DG_CUDA(cudaEventRecord(e0, stream()));
  DG_CUDA(cudaLaunchCooperativeKernel((void*)k_shard_coreness, dim3(per * count), dim3(kThreads),
                                      params, 0, stream()));
  count_launch();
  DG_CUDA(cudaEventRecord(e1, stream()));
  uint32_t h[10];
  d2h(h, out.get(), 10);
  stream_sync();
  float ms = 0;
  DG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (kernel_ms) *kernel_ms = ms;
  if (DG_SP_PROF)
    fprintf(stderr, "[shard prof] kcycles: level %u level-sync %u expand %u sync %u pieces %u xsync %u\n",
            h[3], h[4], h[5], h[6], h[7], h[8]);
  if (h[2] == 4)
    throw DgError(DG_E_INVARIANT,
                  "sharded coreness: barrier timeout (a shard did not arrive within "
                  "DG_BARRIER_TIMEOUT_S seconds)");
  if (h[2]) throw DgError(DG_E_INVARIANT, "sharded coreness kernel failed internal check");
  *kmax = h[0];
  *rounds = h[1];
  for (uint32_t k = 0; k < count; ++k) shards[k]->nfront = 0;
  DG_API_END
}

}  // extern "C"
