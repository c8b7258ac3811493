// kcore.cu -- exact / approximate coreness as ONE persistent cooperative
// kernel (reference core.cpp:18-131).
//
// Semantics reproduced exactly (labels, kmax, peel_rounds):
//   round at bound b: every alive vertex with residual degree <= b leaves
//   (label = current label), then alive neighbours lose one degree per removed
//   neighbour.  A round is "non-empty" iff it removes something; when none is
//   left at b the bound advances (exact: to the minimum alive degree, which
//   is what the reference's ++bound loop reaches; approximate: geometric
//   phases t_{i+1} = max(t_i + 1, ceil(c t_i)) until b >= min degree).
//
// B200 mapping:
//   * frontier of round r+1 = vertices whose degree crossed b+1 -> b during
//     round r, detected by the atomicSub return value (no bucket rescans);
//   * a frontier entry is (vertex, exclusive arc prefix, row offset), and a
//     chunk-start table cse[c] = entry holding arc 32c makes the expansion
//     perfectly load balanced: one warp step = 32 consecutive arcs; the step
//     loads its <= 32 entry starts coalesced and finds each lane's entry with
//     a 5-step shuffle search (no memory in the dependent chain).  Each warp
//     keeps UC steps in flight, so hub rows are spread over many warps and
//     small rows are packed 32 arcs per step;
//   * crossings are buffered in shared memory and published with ONE packed
//     64-bit atomic per CTA per tile: (count << 36) | arcs; a CTA whose buffer
//     overflows leaves the vertex unlabelled and raises a flag, and an extra
//     collect phase picks those up from the live list;
//   * the live list (alive vertices) is compacted at every level advance, so
//     min-degree scans shrink with the graph;
//   * one grid barrier per round (two per level advance); only thread 0 of a
//     CTA touches the barrier and the phase scalars (fetched into shared
//     memory), so no L2 line is hammered by the whole grid.
#include <cstdlib>

#include "internal.cuh"

namespace dgb {

namespace {

constexpr int KC_THREADS = 1024;
#ifndef DG_KC_SPEC
#define DG_KC_SPEC 1
#endif
constexpr uint32_t CH = 32;     // arcs per chunk = one warp step
#ifndef DG_UC
#define DG_UC 2
#endif
constexpr int UC = DG_UC;         // chunks in flight per warp (short-row steps)
constexpr int SC = 8;           // chunks per super-chunk (one warp step on long rows)
#ifndef DG_WIDE_Q
#define DG_WIDE_Q 2  // super-chunk rounds: at least DG_WIDE_Q / 4 super-chunks per warp
#endif
#ifndef DG_KC_HUBS
#define DG_KC_HUBS 4096         // big rounds: decrements of ids below this summed per CTA
#endif
constexpr uint32_t HUBS = DG_KC_HUBS;
#ifndef DG_KC_BUF
#define DG_KC_BUF 8192
#endif
constexpr uint32_t BUF = DG_KC_BUF;  // per-CTA crossing buffer
#ifndef DG_KC_LB
#define DG_KC_LB 4096
#endif
constexpr uint32_t LB = DG_KC_LB;  // per-CTA buffer of low-list entries (degree crossing theta)
constexpr uint32_t NB = 1024;   // degree histogram bins of a full level pass (= KC_THREADS)
constexpr uint32_t HS = 32;     // histogram sampling stride (one lane per warp step)
constexpr uint32_t kUnset = 0xffffffffu;
constexpr uint64_t M36 = (1ULL << 36) - 1;

struct alignas(128) Acc {  // one cache line each: no false sharing between phases
  unsigned long long front;  // (count << 36) | arcs of the frontier being built
  unsigned long long live;   // live-list entries written
  uint32_t minv;             // min alive degree (level advance)
  uint32_t ovf;              // some CTA buffer overflowed while building
  unsigned long long live2;  // live-list entries of a fallback collect (level advance)
  unsigned long long ccnt;   // level-advance candidates spilled to KcArgs::cand
};

struct Frontier {
  uint32_t* v;    // vertex
  uint64_t* fa;   // exclusive arc prefix
  uint64_t* fo;   // row offset offs[v]
  uint32_t* cse;  // cse[c] = entry holding arc CH*c
};

struct KcArgs {
  const uint64_t* offs;
  const uint32_t* adj;
  uint32_t n;
  uint32_t* deg;  // residual degrees
  uint32_t* labels;
  uint32_t* live0;
  uint32_t* live1;
  uint32_t* cand;  // level-advance candidates spilled by full CTA buffers (capacity n)
  uint32_t* alive;  // alive bitmap (n bits; large graphs only, see k_coreness<BM>)
  Frontier fr[2];
  Acc* acc;  // [3]
  // low list (exact mode): every alive vertex with degree < theta, so level
  // advances scan it instead of the whole live list (see k_coreness)
  uint32_t* low[2];
  unsigned long long* lt;  // [2] entries in low[0] / low[1]
  uint32_t* hist;          // [NB] sampled degree histogram of a full pass (zero between uses)
  GridBarrier* bar;
  uint32_t* out;               // kmax, rounds, err
  unsigned long long* rtrace;  // [3*4096] per-round expand cycles, Fc, Ftot, then
                               // [3*4096] per-level-pass cycles, live entries, spilled (diagnostic)
  unsigned long long* prof;    // [8] block-0 cycles (see dg_kcore_profile)
  int approx;
  int nolow;  // DG_KCORE_LOWLIST=0: no low list (every level advance a full pass)
  uint64_t lowmin;  // live-list length from which level advances use the low list
  uint64_t c_num, c_den;
};

struct Smem {
  uint32_t hub[HUBS > 0 ? HUBS : 1];  // per-CTA decrement sums of low ids (big rounds)
  uint32_t id[BUF];  // staged vertices (next frontier / level-advance candidates)
  uint32_t rd[BUF];  // residual degree of a level-advance candidate
  uint64_t tileA[KC_THREADS];
  uint64_t ws[33];
  uint32_t ws32[33];
  uint32_t hst[NB];  // sampled degree histogram of a full level pass
  uint32_t lid[LB];  // staged low-list entries (degree crossed theta this round)
  uint32_t cnt;
  uint32_t lcnt;
  uint32_t cmin;  // running CTA minimum of a level pass (exact mode)
  uint32_t tbin;  // scratch: histogram bin that sets theta
  uint32_t kth;   // theta (low-list threshold, 0 = no low list)
  uint32_t klb;   // low-list buffer being extended
  unsigned long long b_lc;
  unsigned long long baseF, baseL;
  // phase scalars fetched by thread 0 after each grid barrier
  uint32_t abort;
  unsigned long long b_front, b_live, b_live2, b_ccnt;
  uint32_t b_minv, b_ovf;
};

// Level advance candidates: alive vertices within LW of the current bound are
// staged in shared memory during the min scan (a CTA's overflow spills to a
// global list), so the usual small jump needs no second pass.
constexpr uint32_t LW = 16;
constexpr int LE = 4;  // live-list entries per thread in the level pass
constexpr uint32_t LFRAC = 8;  // low list ~ 1/LFRAC of the alive vertices at a rebuild
constexpr uint32_t LMIN = 8;   // ... and at least LMIN degree values past the bound
static_assert(NB == KC_THREADS, "one histogram bin per thread");

__device__ __forceinline__ void fetch_acc(Smem& s, Acc* acc) {
  s.b_front = ld_relaxed_u64(&acc->front);
  s.b_live = ld_relaxed_u64(&acc->live);
  s.b_minv = ld_relaxed_u32(&acc->minv);
  s.b_ovf = ld_relaxed_u32(&acc->ovf);
  s.b_live2 = ld_relaxed_u64(&acc->live2);
  s.b_ccnt = ld_relaxed_u64(&acc->ccnt);
}

// alive bit (BM mode)
__device__ __forceinline__ bool is_alive(const KcArgs& a, uint32_t v) {
  return ((ld_relaxed_u32(&a.alive[v >> 5]) >> (v & 31)) & 1u) != 0;
}
#ifndef DG_ALIVE_LD
#define DG_ALIVE_LD 1
#endif
// alive bit on the expansion path: may be stale (bits only ever clear, and a
// decrement of a removed vertex never reports a crossing: its degree is
// already at or below the bound), so it may come from L1
__device__ __forceinline__ bool is_alive_exp(const KcArgs& a, uint32_t v) {
  uint32_t w;
#if DG_ALIVE_LD == 1
  asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(w) : "l"(&a.alive[v >> 5]));
#elif DG_ALIVE_LD == 2
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(w) : "l"(&a.alive[v >> 5]));
#else
  w = ld_relaxed_u32(&a.alive[v >> 5]);
#endif
  return ((w >> (v & 31)) & 1u) != 0;
}

// All threads of the CTA call this with a per-thread candidate (isF, v, d, o).
// Publishes the tile's entries into the frontier with one atomic, labels
// them, and fills the chunk-start table for the tile's arc range.
__device__ __forceinline__ void emit_front_tile(bool isF, uint32_t v, uint32_t d, uint64_t o,
                                                uint32_t label, const KcArgs& a,
                                                const Frontier& F, Acc* acc, Smem& s) {
  const uint64_t pk = isF ? ((1ULL << 36) | d) : 0ULL;
  uint64_t tot;
  const uint64_t ex = block_excl_scan(pk, s.ws, &tot);
  if (tot == 0) return;  // uniform: nothing in this tile (block_excl_scan synced)
  if (threadIdx.x == 0) s.baseF = atomicAdd(&acc->front, (unsigned long long)tot);
  __syncthreads();
  const uint64_t base = s.baseF;
  const uint64_t e0 = base >> 36, A0 = base & M36;
  if (isF) {
    const uint64_t k = ex >> 36, A = A0 + (ex & M36);
    F.v[e0 + k] = v;
    F.fa[e0 + k] = A;
    F.fo[e0 + k] = o;
    a.labels[v] = label;
    if (a.alive) atomicAnd(&a.alive[v >> 5], ~(1u << (v & 31)));
    s.tileA[k] = A;
  }
  __syncthreads();
  const uint64_t cnt = tot >> 36, TA = tot & M36;
  if (TA) {
    const uint64_t c_lo = (A0 + CH - 1) / CH, c_hi = (A0 + TA - 1) / CH;
    for (uint64_t c = c_lo + threadIdx.x; c <= c_hi; c += blockDim.x) {
      const uint64_t x = c * CH;
      uint64_t lo = 0, hi = cnt - 1;  // largest k with tileA[k] <= x
      while (lo < hi) {
        const uint64_t mid = (lo + hi + 1) >> 1;
        if (s.tileA[mid] <= x)
          lo = mid;
        else
          hi = mid - 1;
      }
      F.cse[c] = uint32_t(e0 + lo);
    }
  }
  __syncthreads();
}

// Scan the live list: alive vertices with deg <= bound join the frontier,
// the other alive ones are compacted into live_out.
template <bool BM>
__device__ void collect(const KcArgs& a, uint32_t livec, bool implicit, const uint32_t* live_in,
                        uint32_t* live_out, uint32_t bound, uint32_t label, const Frontier& F,
                        Acc* acc, Smem& s, unsigned long long* live_ctr) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t base = uint64_t(blockIdx.x) * blockDim.x; base < livec; base += stride) {
    const uint64_t i = base + threadIdx.x;
    uint32_t v = 0, d = 0;
    uint64_t o = 0;
    bool isF = false, isL = false;
    if (i < livec) {
      v = implicit ? uint32_t(i) : live_in[i];
      if (BM ? is_alive(a, v) : a.labels[v] == kUnset) {
        if (a.deg[v] <= bound) {
          isF = true;
          o = a.offs[v];
          d = uint32_t(a.offs[v + 1] - o);
        } else {
          isL = true;
        }
      }
    }
    uint32_t totL;
    const uint32_t exL = block_excl_scan<uint32_t>(isL ? 1u : 0u, s.ws32, &totL);
    if (threadIdx.x == 0 && totL) s.baseL = atomicAdd(live_ctr, (unsigned long long)totL);
    __syncthreads();
    if (isL) live_out[s.baseL + exL] = v;
    emit_front_tile(isF, v, d, o, label, a, F, acc, s);
  }
}

// Level-advance pass over the live list (see k_coreness): min alive degree,
// compaction into live_out (list order kept), candidates within LW of the
// bound staged in shared memory (overflow spilled to a.cand).  E contiguous
// entries per thread: E independent load chains and one CTA scan per
// E * blockDim entries.
// hist: also sample the degrees of alive vertices (ids = 0 mod HS) into the
// CTA's histogram s.hst[min(d - hb, NB - 1)] (full passes of exact mode).
// LOCAL: the list is this CTA's own (shared memory), not a grid-strided share.
template <bool BM, int E, bool LOCAL = false>
__device__ __forceinline__ void level_pass(const KcArgs& a, Smem& s, const uint32_t* live_in,
                                           uint32_t* live_out, uint64_t livec, bool implicit,
                                           uint64_t win, bool track, Acc* acc,
                                           unsigned long long* out_ctr, bool hist, uint32_t hb,
                                           uint32_t& lmin, const Frontier* spec = nullptr) {
  const uint32_t lane = lane_id();
  const uint64_t tile = uint64_t(blockDim.x) * E;
  const uint64_t stride = LOCAL ? tile : uint64_t(gridDim.x) * tile;
  for (uint64_t base = LOCAL ? 0 : uint64_t(blockIdx.x) * tile; base < livec; base += stride) {
    const uint64_t i0 = base + uint64_t(threadIdx.x) * E;
    uint32_t v[E], d[E];
    bool alive[E];
    if (E == 4 && !LOCAL && !implicit && i0 + E <= livec) {
      const uint4 q = *reinterpret_cast<const uint4*>(live_in + i0);
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = w[e & 3];
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e)
        v[e] = implicit ? uint32_t(i0 + e) : (i0 + e < livec ? live_in[i0 + e] : 0u);
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      alive[e] = false;
      d[e] = kUnset;
      if (i0 + e < livec) {
        const uint32_t x = v[e];
        // the degree is read alongside the liveness word (not after it): one
        // dependent round trip per entry instead of two
        const uint32_t dx = a.deg[x];
        alive[e] = BM ? is_alive(a, x) : a.labels[x] == kUnset;
        if (alive[e]) d[e] = dx;
      }
    }
    uint32_t c = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      lmin = min(lmin, d[e]);
      c += alive[e];
      if (hist && alive[e] && (v[e] & (HS - 1)) == 0) atomicAdd(&s.hst[min(d[e] - hb, NB - 1)], 1u);
      bool spill = false;
      bool near;
      if (track) {
        // exact mode: the next bound IS the global minimum, so a CTA stages
        // only vertices at its running minimum (entries staged before the
        // minimum dropped are filtered at emission)
        const uint32_t wm = __reduce_min_sync(~0u, alive[e] ? d[e] : kUnset);
        if (lane == 0 && wm < *reinterpret_cast<volatile uint32_t*>(&s.cmin))
          atomicMin(&s.cmin, wm);
        __syncwarp();
        near = alive[e] && d[e] <= *reinterpret_cast<volatile uint32_t*>(&s.cmin);
      } else {
        near = alive[e] && d[e] <= win;
      }
      const uint32_t nm = __ballot_sync(~0u, near);  // one shared atomic per warp
      uint32_t nb = 0;
      if (nm && lane == uint32_t(__ffs(nm) - 1)) nb = atomicAdd(&s.cnt, uint32_t(__popc(nm)));
      if (nm) nb = __shfl_sync(~0u, nb, __ffs(nm) - 1);
      if (near) {
        const uint32_t slot = nb + __popc(nm & ((1u << lane) - 1u));
        if (slot < BUF) {
          s.id[slot] = v[e];
          s.rd[slot] = d[e];
        } else {
          spill = true;
        }
      }
      // overflow -> global candidate list, warp-aggregated
      const uint32_t cm = __ballot_sync(~0u, spill);
      if (cm) {
        unsigned long long cb = 0;
        if (lane == 0) cb = atomicAdd(&acc->ccnt, (unsigned long long)__popc(cm));
        cb = __shfl_sync(~0u, cb, 0);
        if (spill) a.cand[cb + __popc(cm & ((1u << lane) - 1u))] = v[e];
      }
    }
    uint32_t totL;
    const uint32_t exL = block_excl_scan<uint32_t>(c, s.ws32, &totL);
    if (threadIdx.x == 0 && totL) s.baseL = atomicAdd(out_ctr, (unsigned long long)totL);
    __syncthreads();
    uint64_t o = s.baseL + exL;
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (alive[e]) live_out[o++] = v[e];
    __syncthreads();  // s.baseL / ws32 reuse
    if (E == 1 && spec) {
      // speculative frontier (exact mode, short lists): the next bound is at
      // least hb, so if any alive vertex has degree hb the new frontier is
      // exactly the alive vertices of degree hb -- emitted here, before the
      // pass's grid barrier, so that advance needs no second barrier; with
      // none anywhere nothing is emitted and the usual emission follows
      const bool isF = alive[0] && d[0] == hb;
      uint64_t ro = 0;
      uint32_t dl = 0;
      if (isF) {
        ro = a.offs[v[0]];
        dl = uint32_t(a.offs[v[0] + 1] - ro);
      }
      emit_front_tile(isF, v[0], dl, ro, hb, a, *spec, acc, s);
    }
  }
}

// 64-bit warp shuffle
__device__ __forceinline__ uint64_t shfl64(uint64_t x, uint32_t src) {
  return __shfl_sync(~0u, x, src);
}


// Liveness tests and decrements of K targets per lane (kUnset = none), all
// K loads in flight before any atomic; a decrement that lands the degree
// on the bound enrols the vertex in the next frontier (warp-aggregated slot
// in the CTA's crossing buffer).
// A decrement that takes the degree from theta to theta - 1 enrols the vertex
// in the low list (staged in s.lid, flushed once per CTA at the end of the
// round; theta = 0 outside exact mode: no alive degree is ever 0 before a
// decrement).
__device__ __forceinline__ void stage_low(bool lx, uint32_t uv, Smem& s, const KcArgs& a,
                                          const uint32_t& lbs) {
  const uint32_t lm = __ballot_sync(~0u, lx);
  if (!lm) return;
  const uint32_t lane = lane_id();
  uint32_t base = 0;
  if (lane == __ffs(lm) - 1) base = atomicAdd(&s.lcnt, uint32_t(__popc(lm)));
  base = __shfl_sync(~0u, base, __ffs(lm) - 1);
  const uint32_t slot = base + __popc(lm & ((1u << lane) - 1u));
  const bool ovf = lx && slot >= LB;
  if (lx && !ovf) s.lid[slot] = uv;
  const uint32_t om = __ballot_sync(~0u, ovf);  // CTA buffer full: straight to the list
  if (om) {
    unsigned long long gb = 0;
    const uint32_t lb = lbs;
    if (lane == __ffs(om) - 1) gb = atomicAdd(&a.lt[lb], (unsigned long long)__popc(om));
    gb = __shfl_sync(~0u, gb, __ffs(om) - 1);
    if (ovf) a.low[lb][gb + __popc(om & ((1u << lane) - 1u))] = uv;
  }
}

template <bool BM, int K, bool HUB = false>
__device__ __forceinline__ void expand_targets(const KcArgs& a, const uint32_t (&u)[K],
                                               uint32_t b32, Smem& s, Acc* nacc) {
  const uint32_t theta = s.kth;
  bool live[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const uint32_t uv = u[k];
    live[k] = false;
    if (uv == kUnset) continue;
    if (HUB && uv < HUBS) {  // summed in shared memory, applied once per CTA (hub_flush)
      atomicAdd(&s.hub[uv], 1u);
      continue;
    }
    if (BM)
      live[k] = is_alive_exp(a, uv);  // removed?
    else
      live[k] = a.deg[uv] > b32;  // dead, or already at/below the bound
  }
  uint32_t old[K];
#pragma unroll
  for (int k = 0; k < K; ++k) old[k] = live[k] ? atomicSub(&a.deg[u[k]], 1u) : 0u;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const bool cross = live[k] && old[k] == b32 + 1;  // crossed: joins the next round
    const bool lx = live[k] && old[k] == theta;       // crossed theta: joins the low list
    if (!__any_sync(~0u, cross || lx)) continue;       // the usual case: one vote
    stage_low(lx, u[k], s, a, s.klb);
    const uint32_t cm = __ballot_sync(~0u, cross);
    if (!cm) continue;
    uint32_t base = 0;
    if (lane_id() == __ffs(cm) - 1) base = atomicAdd(&s.cnt, uint32_t(__popc(cm)));
    base = __shfl_sync(~0u, base, __ffs(cm) - 1);
    if (cross) {
      const uint32_t slot = base + __popc(cm & ((1u << lane_id()) - 1u));
      const uint32_t uv = u[k];
      if (slot < BUF) {
        s.id[slot] = uv;  // its row is looked up at emission, off this critical path
      } else {
        nacc->ovf = 1;  // left unlabelled; the overflow collect finds it
      }
    }
  }
}

// UC 32-arc chunks cb, cb + cs, ... (those below cend) of frontier F (nch
// chunks in all): each chunk's entry window is loaded coalesced and a 5-step
// shuffle search maps lanes to entries (no memory in the dependent chain).
template <int UC_>
__device__ __forceinline__ void load_chunks(const Frontier& F, const uint32_t* adj, uint64_t cb,
                                            uint64_t cs, uint64_t cend, uint32_t Fc,
                                            uint64_t Ftot, uint32_t lane, uint32_t (&u)[UC_],
                                            uint64_t nch = 0) {
  if (nch == 0) nch = cend;
  uint32_t ne[UC_];
  uint64_t e0[UC_], fa[UC_], fo[UC_];
#pragma unroll
  for (int k = 0; k < UC_; ++k) {
    const uint64_t c = cb + k * cs;
    ne[k] = 0;
    e0[k] = 0;
    fa[k] = ~0ULL;
    fo[k] = 0;
    if (c < cend) {
      e0[k] = F.cse[c];
      const uint64_t e1 = (c + 1 < nch) ? F.cse[c + 1] : uint64_t(Fc) - 1;
      ne[k] = uint32_t(e1 - e0[k] + 1);
      // rows of degree >= 1 need at most 32 entries for 32 arcs; only
      // zero-degree rows can push the window past 32 (slow path)
      if (ne[k] > 32 && F.fa[e0[k] + 32] > c * CH + CH - 1) ne[k] = 32;
      if (lane < ne[k]) {
        fa[k] = F.fa[e0[k] + lane];
        fo[k] = F.fo[e0[k] + lane];
      }
    }
  }
#pragma unroll
  for (int k = 0; k < UC_; ++k) {
    const uint64_t c = cb + k * cs;
    const uint64_t x = c * CH + lane;
    u[k] = kUnset;
    if (c >= cend) continue;  // warp-uniform
    uint64_t p;
    if (ne[k] <= 32) {
      uint32_t l = 0;  // largest l < ne with fa[l] <= x
#pragma unroll
      for (uint32_t step = 16; step; step >>= 1) {
        const uint32_t tl = l + step;
        const uint64_t fl = __shfl_sync(~0u, fa[k], tl < 32 ? tl : 31);
        if (tl < ne[k] && fl <= x) l = tl;
      }
      p = __shfl_sync(~0u, fo[k], l) + (x - __shfl_sync(~0u, fa[k], l));
    } else {  // > 32 entries touch 32 arcs (zero-degree rows): binary search
      uint64_t lo = e0[k], hi = e0[k] + ne[k] - 1;
      while (lo < hi) {
        const uint64_t mid = (lo + hi + 1) >> 1;
        if (F.fa[mid] <= x)
          lo = mid;
        else
          hi = mid - 1;
      }
      p = F.fo[lo] + (x - F.fa[lo]);
    }
    if (x < Ftot) u[k] = adj[p];
  }
}

// BM: liveness from an alive bitmap (n bits, cleared at labelling): arcs to
// removed vertices skip the random read of deg, and a warp's tests of a
// sorted neighbour list share sectors.
// PROF: the diagnostic variant (dg_kcore_profile, DG_KCORE_PROFILE=1) records
// block-0 phase cycles and a per-round trace; the production variant has none
// of that code.
template <bool BM, bool PROF>
__global__ void __launch_bounds__(KC_THREADS, 1) k_coreness(KcArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const uint32_t nb = gridDim.x;
  const uint32_t lane = lane_id();
  const uint64_t gwarp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;

  for (uint32_t h = threadIdx.x; h < HUBS; h += blockDim.x) s.hub[h] = 0;
  for (uint32_t h = threadIdx.x; h < NB; h += blockDim.x) s.hst[h] = 0;
  if (threadIdx.x == 0) {
    s.lcnt = 0;
    s.kth = 0;
    s.klb = 0;
  }
  uint32_t f = 0;       // frontier generation
  uint32_t lv = 0;      // live buffer holding the current live list
  uint32_t livec = a.n;
  bool implicit = true; // live list = 0..n-1 until the first compaction
  uint64_t bound = 0, label = 0, t = 1;
  uint64_t remaining = a.n;
  uint32_t kmax = 0, rounds = 0;
  uint32_t Fc = 0;
  uint64_t Ftot = 0;
  uint64_t guard = 0;
  uint32_t lb = 0;          // low list buffer
  bool hist_dirty = false;  // a.hist holds samples to clear
  const bool P = blockIdx.x == 0 && threadIdx.x == 0;
  long long pr[8] = {}, tp = PROF ? clock64() : 0;
  auto mark = [&](int k) {
    if (PROF && P) {
      const long long tt = clock64();
      pr[k] += tt - tp;
      tp = tt;
    }
  };

  for (;;) {
    if (++guard > 4ULL * a.n + 64) {
      if (P) a.out[2] = 1;
      break;
    }
    if (Fc == 0) {
      if (remaining == 0) break;
      // ---- level advance.  Exact mode keeps a LOW LIST: every alive vertex
      // of degree < theta (built at a full pass, extended by the decrements
      // that cross theta), so the minimum alive degree -- the next bound,
      // < theta while the list holds an alive vertex -- comes from a pass
      // over the low list only; a full pass over the live list (min,
      // compaction, a sampled degree histogram that sets the next theta,
      // then the low list rebuilt) runs only when the low list has run dry.
      // Either pass stages the alive vertices at the running minimum in
      // shared memory (a CTA's overflow spills to a.cand), so the frontier
      // usually needs no second pass.  Approximate mode: every level
      // advance is a full pass staging the vertices within LW of the bound.
      Acc* acc = a.acc + (f % 3);
      const uint64_t win = bound + LW;
      const bool track = !a.approx;
      // a low list pays while a full pass takes several tiles per CTA
      const bool lowok = track && !a.nolow && livec >= a.lowmin;
      uint64_t Lc = 0;
      if (lowok) {
        if (threadIdx.x == 0) s.b_lc = ld_relaxed_u64(&a.lt[lb]);
        __syncthreads();
        Lc = s.b_lc;
      }
      bool full = !lowok || Lc == 0;
      const uint32_t hb = uint32_t(bound) + 1;  // every alive degree is > bound here
      bool spec = false;  // the last pass emitted the frontier of bound hb speculatively
      for (;;) {
        if (threadIdx.x == 0) {
          s.cnt = 0;
          s.cmin = kUnset;
        }
        __syncthreads();
        uint32_t lmin = kUnset;
        const uint32_t* in;
        uint32_t* out;
        uint64_t cnt;
        bool imp = false;
        unsigned long long* octr;
        if (full) {
          in = lv ? a.live1 : a.live0;
          out = lv ? a.live0 : a.live1;
          cnt = livec;
          imp = implicit;
          octr = &acc->live;
        } else {
          in = a.low[lb];
          out = a.low[lb ^ 1];
          cnt = Lc;
          octr = &a.lt[lb ^ 1];
        }
        const bool hist = full && lowok;
        // short lists (one tile per CTA, exact mode): emit the frontier of
        // bound hb speculatively during the pass (see level_pass)
        spec = DG_KC_SPEC && track && !hist && cnt <= uint64_t(gridDim.x) * blockDim.x;
        const Frontier* fsp = spec ? &a.fr[f & 1] : nullptr;
        // wide tiles only while the list fills the grid LE times over
        if (cnt >= uint64_t(gridDim.x) * blockDim.x * LE)
          level_pass<BM, LE>(a, s, in, out, cnt, imp, win, track, acc, octr, hist, hb, lmin);
        else
          level_pass<BM, 1>(a, s, in, out, cnt, imp, win, track, acc, octr, hist, hb, lmin, fsp);
        // the low-list entries this CTA staged since the last level advance
        // (kept in shared memory, no per-round flush) join the pass; a full
        // pass rebuilds the list, so it drops them
        if (!full) {
          level_pass<BM, 1, true>(a, s, s.lid, out, min(s.lcnt, LB), false, win, track, acc, octr,
                                  false, hb, lmin, fsp);
          if (threadIdx.x == 0) s.lcnt = 0;  // level_pass ended with a CTA barrier
        } else if (hist && threadIdx.x == 0) {
          s.lcnt = 0;
        }
        lmin = __reduce_min_sync(~0u, lmin);
        if (lane == 0) s.ws32[threadIdx.x >> 5] = lmin;
        __syncthreads();
        if (threadIdx.x < 32) {
          uint32_t x = threadIdx.x < (blockDim.x >> 5) ? s.ws32[threadIdx.x] : kUnset;
          x = __reduce_min_sync(~0u, x);
          if (threadIdx.x == 0 && x != kUnset) atomicMin(&acc->minv, x);
        }
        if (hist)  // the CTA's samples into the grid histogram (NB == blockDim.x)
          for (uint32_t i = threadIdx.x; i < NB; i += blockDim.x) {
            const uint32_t c = s.hst[i];
            if (c) {
              s.hst[i] = 0;
              atomicAdd(&a.hist[i], c);
            }
          }
        if (PROF && P && pr[6] < 4096) {
          a.rtrace[3 * 4096 + 3 * pr[6]] = clock64() - tp;
          a.rtrace[3 * 4096 + 3 * pr[6] + 1] = cnt;
        }
        mark(0);
        if (!grid_sync(a.bar, nb, &s.abort, [&] { fetch_acc(s, acc); })) break;
        mark(1);
        if (PROF && P && pr[6] < 4096)
          a.rtrace[3 * 4096 + 3 * pr[6] + 2] = s.b_ccnt | (full ? (1ULL << 40) : 0ULL);
        if (PROF && P) ++pr[6];
        if (full) {
          livec = uint32_t(s.b_live);
          lv ^= 1;
          implicit = false;
        } else {
          // every CTA is past the pass over low[lb]: its counter restarts at
          // 0 for the next compaction into it
          if (P) a.lt[lb] = 0;
          lb ^= 1;
        }
        if (s.b_minv != kUnset || full) break;
        full = true;  // the low list held no alive vertex: full pass
      }
      if (s.abort) break;
      const uint64_t gmin = s.b_minv;
      if (gmin == kUnset) {  // remaining > 0 but nothing alive: inconsistent
        if (P) a.out[2] = 2;
        break;
      }
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
      // the speculative frontier is the frontier: no emission, no second barrier
      const bool fast = spec && gmin == hb;
      const bool rebuild = full && lowok;
      if (full && !lowok && threadIdx.x == 0) s.kth = 0;  // no low list from here on
      if (rebuild) {
        // next theta: the low list should hold about 1/LFRAC of the alive
        // vertices (sampled histogram of degree - hb), and at least LMIN
        // degree values beyond the new bound
        if (threadIdx.x == 0) s.tbin = NB - 1;
        uint32_t tot;
        const uint32_t hv = threadIdx.x < NB ? ld_relaxed_u32(&a.hist[threadIdx.x]) : 0u;
        const uint32_t ex = block_excl_scan<uint32_t>(hv, s.ws32, &tot);
        const uint32_t target = (tot + LFRAC - 1) / LFRAC;
        if (threadIdx.x < NB - 1 && hv && ex < target && ex + hv >= target)
          atomicMin(&s.tbin, threadIdx.x + 1);
        __syncthreads();
        uint64_t th = uint64_t(hb) + s.tbin;
        th = max(th, bound + LMIN);
        th = min(th, uint64_t(hb) + NB - 1);  // the last bin mixes every larger degree
        const uint32_t theta = uint32_t(max(th, bound + 1));
        __syncthreads();  // every thread has read s.tbin
        if (threadIdx.x == 0) {
          s.kth = theta;
          s.klb = lb;
        }
        __syncthreads();
        hist_dirty = true;
      }
      const Frontier& F0 = a.fr[f & 1];
      if (fast) {
        // s.b_front (fetched at the pass's barrier) holds the frontier
      } else if (track || bound <= win) {
        // the frontier = candidates with residual degree <= bound: this CTA's
        // staged ones, then a grid-strided share of the spilled ones
        const uint32_t cnt = min(s.cnt, BUF);
        for (uint32_t b0 = 0; b0 < cnt; b0 += blockDim.x) {
          const uint32_t i = b0 + threadIdx.x;
          const bool ok = i < cnt && s.rd[i] <= bound;
          const uint32_t v = ok ? s.id[i] : 0;
          const uint64_t o = ok ? a.offs[v] : 0;
          const uint32_t dl = ok ? uint32_t(a.offs[v + 1] - o) : 0;
          emit_front_tile(ok, v, dl, o, uint32_t(label), a, F0, acc, s);
        }
        const uint64_t cc = s.b_ccnt;
        for (uint64_t base = uint64_t(blockIdx.x) * blockDim.x; base < cc;
             base += uint64_t(gridDim.x) * blockDim.x) {
          const uint64_t i = base + threadIdx.x;
          bool ok = false;
          uint32_t v = 0, dl = 0;
          uint64_t o = 0;
          if (i < cc) {
            v = a.cand[i];
            if (a.deg[v] <= bound) {
              ok = true;
              o = a.offs[v];
              dl = uint32_t(a.offs[v + 1] - o);
            }
          }
          emit_front_tile(ok, v, dl, o, uint32_t(label), a, F0, acc, s);
        }
        if (rebuild) {
          // the low list of the new theta from the compacted live list (into
          // low[lb], empty here); this round's frontier vertices may enter
          // too (dead by the next pass, which drops them)
          // (LE entries per thread, one 16-byte load of the list)
          const uint32_t* lin = lv ? a.live1 : a.live0;
          const uint64_t tile = uint64_t(blockDim.x) * LE;
          for (uint64_t base = uint64_t(blockIdx.x) * tile; base < livec;
               base += uint64_t(gridDim.x) * tile) {
            const uint64_t i0 = base + uint64_t(threadIdx.x) * LE;
            uint32_t v[LE];
            bool in[LE];
            if (i0 + LE <= livec) {
              const uint4 q = *reinterpret_cast<const uint4*>(lin + i0);
              v[0] = q.x, v[1] = q.y, v[2] = q.z, v[3] = q.w;
            } else {
#pragma unroll
              for (int e = 0; e < LE; ++e) v[e] = i0 + e < livec ? lin[i0 + e] : 0u;
            }
            uint32_t c = 0;
#pragma unroll
            for (int e = 0; e < LE; ++e) {
              in[e] = i0 + e < livec && a.deg[v[e]] < s.kth;
              c += in[e];
            }
            uint32_t tl;
            const uint32_t el = block_excl_scan<uint32_t>(c, s.ws32, &tl);
            if (threadIdx.x == 0 && tl) s.baseL = atomicAdd(&a.lt[lb], (unsigned long long)tl);
            __syncthreads();
            uint64_t o = s.baseL + el;
#pragma unroll
            for (int e = 0; e < LE; ++e)
              if (in[e]) a.low[lb][o++] = v[e];
            __syncthreads();
          }
        }
        mark(2);
        if (!grid_sync(a.bar, nb, &s.abort, [&] { fetch_acc(s, acc); })) break;
        mark(1);
      } else {
        // larger jump: collect from the compacted list
        collect<BM>(a, livec, false, lv ? a.live1 : a.live0, lv ? a.live0 : a.live1,
                    uint32_t(bound), uint32_t(label), F0, acc, s, &acc->live2);
        mark(2);
        if (!grid_sync(a.bar, nb, &s.abort, [&] { fetch_acc(s, acc); })) break;
        mark(1);
        livec = uint32_t(s.b_live2);
        lv ^= 1;
      }
      if (threadIdx.x == 0) s.klb = lb;
      const unsigned long long pk = s.b_front;
      Fc = uint32_t(pk >> 36);
      Ftot = pk & M36;
      if (Fc == 0) {
        if (P) a.out[2] = 3;
        break;
      }
    }

    // ---- expand frontier f into frontier f+1
    ++rounds;
    if (label > kmax) kmax = uint32_t(label);
    remaining -= Fc;
    Acc* nacc = a.acc + ((f + 1) % 3);
    if (P) {
      Acc* r = a.acc + ((f + 2) % 3);
      r->front = 0;
      r->live = 0;
      r->minv = kUnset;
      r->ovf = 0;
      r->live2 = 0;
      r->ccnt = 0;
    }
    if (threadIdx.x == 0) s.cnt = 0;
    if (hist_dirty) {  // every CTA read the histogram before the last grid barrier
      if (blockIdx.x == 0)
        for (uint32_t i = threadIdx.x; i < NB; i += blockDim.x) a.hist[i] = 0;
      hist_dirty = false;
    }
    __syncthreads();
    const uint32_t b32r = uint32_t(bound);
    // big rounds: one super-chunk = SC consecutive 32-arc chunks of the
    // frontier's virtual arc space per warp step; rounds too small to give
    // every warp two super-chunks keep one 32-arc chunk per step (UC in
    // flight), so their work spreads over the whole grid
    const bool wide = (Ftot + CH - 1) / CH * 4 >= uint64_t(nwarps) * SC * DG_WIDE_Q;
    {
      const Frontier& F = a.fr[f & 1];
      const uint32_t b32 = uint32_t(bound);
      const uint64_t nch = (Ftot + CH - 1) / CH;
      const uint64_t nsc = wide ? (nch + SC - 1) / SC : 0;
      if (!wide)
        for (uint64_t cb = gwarp; cb < nch; cb += nwarps * UC) {
          uint32_t u[UC];
          load_chunks<UC>(F, a.adj, cb, nwarps, nch, Fc, Ftot, lane, u);
          expand_targets<BM, UC>(a, u, b32, s, nacc);
        }
      // super-chunks go warp-major across the CTAs, so a round of fewer
      // super-chunks than warps still spreads over every SM
      const uint64_t swarp = uint64_t(threadIdx.x >> 5) * gridDim.x + blockIdx.x;
      for (uint64_t sc = swarp; sc < nsc; sc += nwarps) {
        const uint64_t c0 = sc * SC;
        const uint64_t clast = min(c0 + SC, nch) - 1;
        const uint64_t e0 = F.cse[c0];
        const uint64_t e1 = (clast + 1 < nch) ? F.cse[clast + 1] : uint64_t(Fc) - 1;
        if (e1 - e0 < 32) {
          // <= 32 entries cover the super-chunk (rows average >= SC arcs):
          // lane l holds entry e0 + l; SC independent adjacency loads, then SC
          // liveness tests, then the decrements -- SC x the memory-level
          // parallelism of one step per warp
          const uint32_t ne = uint32_t(e1 - e0 + 1);
          uint64_t fa = ~0ULL, fo = 0;
          if (lane < ne) {
            fa = F.fa[e0 + lane];
            fo = F.fo[e0 + lane];
          }
          uint32_t u[SC];
#pragma unroll
          for (int k = 0; k < SC; ++k) {
            const uint64_t x = (c0 + k) * CH + lane;
            uint32_t l = 0;  // largest l < ne with fa[l] <= x (every lane searches)
            if (ne > 1) {    // warp-uniform
#pragma unroll
              for (uint32_t step = 16; step; step >>= 1) {
                const uint32_t tl = l + step;
                const uint64_t fl = shfl64(fa, tl < 32 ? tl : 31);
                if (tl < ne && fl <= x) l = tl;
              }
            }
            const uint64_t p = shfl64(fo, l) + (x - shfl64(fa, l));
            u[k] = x < Ftot ? a.adj[p] : kUnset;
          }
          expand_targets<BM, SC, (HUBS > 0)>(a, u, b32, s, nacc);
        } else {
          // many short rows: one 32-arc chunk per step, UC in flight
          for (uint64_t cb = c0; cb <= clast; cb += UC) {
            uint32_t u[UC];
            load_chunks<UC>(F, a.adj, cb, 1, clast + 1, Fc, Ftot, lane, u, nch);
            expand_targets<BM, UC, (HUBS > 0)>(a, u, b32, s, nacc);
          }
        }
      }
    }
    __syncthreads();
    if (HUBS > 0 && wide) {
      // big round: every CTA applies its summed decrements of the low ids
      // (RMAT's hubs) with one atomic each; the sum that takes the degree
      // from above the bound to at/below it enrols the vertex
      for (uint32_t h0 = 0; h0 < HUBS; h0 += blockDim.x) {
        const uint32_t h = h0 + threadIdx.x;
        const uint32_t c = h < HUBS ? s.hub[h] : 0u;
        bool cross = false, lx = false;
        if (c) {
          s.hub[h] = 0;
          const bool alive = BM ? is_alive(a, h) : a.labels[h] == kUnset;
          if (alive) {
            const uint32_t old = atomicSub(&a.deg[h], c);
            cross = old > b32r && old - c <= b32r;
            lx = old >= s.kth && old - c < s.kth;
          }
        }
        stage_low(lx, h, s, a, s.klb);
        const uint32_t cm = __ballot_sync(~0u, cross);
        if (cm) {
          uint32_t base = 0;
          if (lane == __ffs(cm) - 1) base = atomicAdd(&s.cnt, uint32_t(__popc(cm)));
          base = __shfl_sync(~0u, base, __ffs(cm) - 1);
          if (cross) {
            const uint32_t slot = base + __popc(cm & ((1u << lane) - 1u));
            if (slot < BUF) s.id[slot] = h;
            else nacc->ovf = 1;
          }
        }
      }
      __syncthreads();
    }
    if (PROF && P && rounds <= 4096) {
      a.rtrace[3 * (rounds - 1)] = clock64() - tp;
      a.rtrace[3 * (rounds - 1) + 1] = Fc | ((remaining + Fc) << 32);  // alive at round start
      a.rtrace[3 * (rounds - 1) + 2] = Ftot;
    }
    mark(3);
    {
      const uint32_t cnt = min(s.cnt, BUF);
      const Frontier& NF = a.fr[(f + 1) & 1];
      for (uint32_t b0 = 0; b0 < cnt; b0 += blockDim.x) {
        const uint32_t i = b0 + threadIdx.x;
        const bool ok = i < cnt;
        const uint32_t v = ok ? s.id[i] : 0;
        const uint64_t o = ok ? a.offs[v] : 0;
        const uint32_t dl = ok ? uint32_t(a.offs[v + 1] - o) : 0;
        emit_front_tile(ok, v, dl, o, uint32_t(label), a, NF, nacc, s);
      }
    }
    mark(4);
    if (!grid_sync(a.bar, nb, &s.abort, [&] { fetch_acc(s, nacc); })) break;
    mark(5);
    ++f;
    if (s.b_ovf) {
      if (PROF && P) ++pr[7];
      collect<BM>(a, livec, implicit, lv ? a.live1 : a.live0, lv ? a.live0 : a.live1, uint32_t(bound),
              uint32_t(label), a.fr[f & 1], nacc, s, &nacc->live);
      if (!grid_sync(a.bar, nb, &s.abort, [&] { fetch_acc(s, nacc); })) break;
      livec = uint32_t(s.b_live);
      lv ^= 1;
      implicit = false;
    }
    const unsigned long long pk = s.b_front;
    Fc = uint32_t(pk >> 36);
    Ftot = pk & M36;
  }
  if (P) {
    a.out[0] = kmax;
    a.out[1] = rounds;
    if (ld_relaxed_u32(&a.bar->abort)) a.out[2] = 4;
    if (PROF)
      for (int k = 0; k < 8; ++k) a.prof[k] = pr[k];
  }
}

__global__ void k_init_deg(const uint64_t* offs, uint64_t n, uint32_t* deg, uint32_t* labels) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    deg[i] = uint32_t(offs[i + 1] - offs[i]);
    labels[i] = kUnset;
  }
}

__global__ void k_init_acc(Acc* acc, GridBarrier* bar, uint32_t timeout_s) {
  if (threadIdx.x < 3) {
    acc[threadIdx.x].front = 0;
    acc[threadIdx.x].live = 0;
    acc[threadIdx.x].minv = kUnset;
    acc[threadIdx.x].ovf = 0;
    acc[threadIdx.x].live2 = 0;
    acc[threadIdx.x].ccnt = 0;
  }
  if (threadIdx.x == 0) *bar = GridBarrier{0, 0, 0, timeout_s};
}

}  // namespace

unsigned long long* kcore_prof_buffer() {
  static unsigned long long* buf[64] = {};
  int d = 0;
  DG_CUDA(cudaGetDevice(&d));
  if (!buf[d]) {
    DG_CUDA(cudaMalloc(&buf[d], DG_KCORE_PROFILE_WORDS * sizeof(unsigned long long)));
    DG_CUDA(cudaMemset(buf[d], 0, DG_KCORE_PROFILE_WORDS * sizeof(unsigned long long)));
  }
  return buf[d];
}

void kcore_profile(unsigned long long out[DG_KCORE_PROFILE_WORDS]) {
  d2h(out, kcore_prof_buffer(), DG_KCORE_PROFILE_WORDS);
  stream_sync();
}

CoreOut coreness(const dg_graph& g, bool approx, uint64_t c_num, uint64_t c_den,
                 uint32_t* d_labels) {
  if (g.n == 0) throw DgError(DG_E_EMPTY, "coreness of empty graph");
  if (approx && (c_den == 0 || c_num <= c_den))
    throw DgError(DG_E_PARAM, "approximation factor must be > 1");
  if (g.n >= (1ULL << 28) || 2 * g.m >= (1ULL << 36))
    throw DgError(DG_E_PARAM, "graph too large for the single-GPU coreness kernel");
  const uint64_t n = g.n;
  DevBuf<uint32_t> deg(n), live0(n), live1(n), v0(n), v1(n), cand(n);
  // alive bitmap (n bits): a warp's liveness tests of a sorted neighbour
  // list share sectors that its degree reads do not (RMAT-22 9.5 -> 8.5 ms,
  // RMAT-26 70 -> 61 ms); DG_KCORE_BITMAP=0/1 overrides (tests, tuning)
  bool bm = true;
  if (const char* e = getenv("DG_KCORE_BITMAP")) bm = e[0] == '1';
  DevBuf<uint32_t> alive;
  if (bm) alive.alloc((n + 31) / 32);
  DevBuf<uint64_t> fa0(n), fa1(n), fo0(n), fo1(n);
  const uint64_t nch = (2 * g.m) / CH + 2;
  DevBuf<uint32_t> cse0(nch), cse1(nch);
  DevBuf<Acc> acc(3);
  DevBuf<uint32_t> low0, low1, hist(NB);
  DevBuf<unsigned long long> lt(2);
  if (!approx) {
    low0.alloc(n);
    low1.alloc(n);
  }
  lt.zero();
  hist.zero();
  DevBuf<GridBarrier> bar(1);
  DevBuf<uint32_t> out(3);
  out.zero();
  // the timed region (CoreOut::kernel_ms) holds every pass over the graph:
  // bitmap fill, degree init (the 4n + 8n of B_kc) and the peel kernel
  cudaEvent_t e0, e1;
  DG_CUDA(cudaEventCreate(&e0));
  DG_CUDA(cudaEventCreate(&e1));
  DG_CUDA(cudaEventRecord(e0, stream()));
  if (bm) DG_CUDA(cudaMemsetAsync(alive.get(), 0xff, ((n + 31) / 32) * 4, stream()));
  k_init_deg<<<grid_for(n, 256), 256, 0, stream()>>>(g.offs.get(), n, deg.get(), d_labels);
  DG_CHECK_LAUNCH();
  k_init_acc<<<1, 32, 0, stream()>>>(acc.get(), bar.get(), barrier_timeout_s());
  DG_CHECK_LAUNCH();

  const size_t smem = sizeof(Smem);
  const bool prof = getenv("DG_KCORE_PROFILE") && getenv("DG_KCORE_PROFILE")[0] == '1';
  const bool nolow = getenv("DG_KCORE_LOWLIST") && getenv("DG_KCORE_LOWLIST")[0] == '0';
  // the low list pays once a full level pass takes two tiles per CTA;
  // DG_KCORE_LOWMIN=<entries> overrides (tests drive it on small graphs)
  uint64_t lowmin = 2ULL * num_sms() * KC_THREADS * LE;
  if (const char* e = getenv("DG_KCORE_LOWMIN")) lowmin = strtoull(e, nullptr, 10);
  void* kfn = bm ? (prof ? (void*)k_coreness<true, true> : (void*)k_coreness<true, false>)
                 : (prof ? (void*)k_coreness<false, true> : (void*)k_coreness<false, false>);
  DG_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int occ = 0;
  DG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, KC_THREADS, smem));
  if (occ < 1) throw DgError(DG_E_CUDA, "coreness kernel does not fit on an SM");
  const unsigned blocks = unsigned(num_sms());  // one persistent CTA per SM

  KcArgs args{g.offs.get(),
              g.adj.get(),
              uint32_t(n),
              deg.get(),
              d_labels,
              live0.get(),
              live1.get(),
              cand.get(),
              bm ? alive.get() : nullptr,
              {Frontier{v0.get(), fa0.get(), fo0.get(), cse0.get()},
               Frontier{v1.get(), fa1.get(), fo1.get(), cse1.get()}},
              acc.get(),
              {low0.get(), low1.get()},
              lt.get(),
              hist.get(),
              bar.get(),
              out.get(),
              prof ? kcore_prof_buffer() + 8 : nullptr,
              prof ? kcore_prof_buffer() : nullptr,
              approx ? 1 : 0,
              nolow ? 1 : 0,
              lowmin,
              c_num,
              c_den};
  void* params[] = {&args};
  DG_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(blocks), dim3(KC_THREADS), params,
                                      smem, stream()));
  count_launch();
  DG_CUDA(cudaEventRecord(e1, stream()));
  uint32_t h[3];
  d2h(h, out.get(), 3);
  stream_sync();
  CoreOut r;
  DG_CUDA(cudaEventElapsedTime(&r.kernel_ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (h[2] == 4)
    throw DgError(DG_E_INVARIANT,
                  "coreness kernel: grid barrier timeout (a CTA did not arrive within "
                  "DG_BARRIER_TIMEOUT_S seconds)");
  if (h[2]) {
    char buf[128];
    snprintf(buf, sizeof buf, "coreness kernel failed internal check (code %u)", h[2]);
    throw DgError(DG_E_INVARIANT, buf);
  }
  r.kmax = h[0];
  r.rounds = h[1];
  return r;
}

}  // namespace dgb
