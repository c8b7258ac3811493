// peel_kernel.cuh -- the Greedy++ batch-peel kernel (one CTA, whole chain).
//
// Reference semantics: refine.cpp:20-156 (PeelState / peel_buckets /
// peel_heap): key = load + residual degree; a batch is EVERY alive vertex at
// the exact minimum key, in ascending id; batch members die before any
// decrement; each alive neighbour loses one key unit per removed neighbour.
//
// Fused Algorithm 3 charge (refine.cpp:195-199).  A[pos(v)] counts v's
// neighbours positioned after v: alive after v's batch, or in v's batch with
// a larger id.  At removal key(v) = load(v) + #neighbours alive at that
// moment (same-batch members included), so
//     A[pos(v)] = key_at_removal(v) - load(v) - #same-batch neighbours u < v.
// The kernel emits raw[pos] = key_at_removal - #smaller same-batch
// neighbours, and Alg. 3 subtracts the load.
//
// Key ranges instead of sentinels.  Alive keys live in [0, 2^(b-1)); a batch
// member is re-keyed to BATCH = 3*2^(b-2) - 1, a removed vertex to DEAD =
// 2^b - 1.  A vertex receives fewer than 2^28 decrements (its degree), so
// decremented marks stay inside [2^(b-1), 3*2^(b-2)) resp. [3*2^(b-2), 2^b):
// removal decrements EVERY neighbour unconditionally (red.shared.add, or
// atom.shared.add whose return value tells batch members apart) and the min
// scan ignores non-alive keys for free (they are the largest values).
//
// The kernel is issue-bound (32 warps share 4 schedulers), so every phase is
// written for instruction count:
//   S1  each thread scans its contiguous chunk of 4*VQ keys with 128-bit
//       shared loads (VQ odd: conflict free, fully unrolled at compile time):
//       3-input min, then the multiplicity; redux.sync -> 32-entry warp table
//   --- barrier A
//   S2  every warp reduces the table with redux.sync (global min, batch size,
//       its output offset); owners of the minimum write the batch in
//       ascending id into perm and stage (v, row offset, degree)
//   --- barrier B
//   S3  the batch's rows are cut into 16-byte adjacency quads; a flat quad
//       index is spread over the CTA (U quads in flight per thread), each
//       quad = one 128-bit load + four shared reductions.  Batches > 32
//       members take a slice path with a CTA scan.
//   --- barrier C
//   raw charges of the batch are written to global at the next S1.
#pragma once

#include <type_traits>

namespace dgb {
namespace peelk {

#ifndef DG_PEEL_PT
#define DG_PEEL_PT 1024
#endif
constexpr int PT = DG_PEEL_PT;  // threads (tuning builds: -DDG_PEEL_PT=512)
constexpr int U = 4;      // arcs in flight per thread (large-batch path)
constexpr int UQ = 2;     // adjacency quads in flight per thread (small-batch path)

template <class K>
struct Args {
  const uint64_t* offs;
  const uint32_t* adj;
  uint32_t n;
  const uint64_t* loads;
  uint64_t base;
  int one;
  K* gkeys;  // keys in global memory when they do not fit in shared
  uint32_t chunk;
  uint32_t* perm;
  uint64_t* raw;                // raw charges per position (see header)
  unsigned long long* batches;
  unsigned long long* prof;     // [8] thread-0 cycles S1,S2,S3, batches, S3 of 1-vertex batches, #1-vertex, #>32, n
};

struct Fixed {  // shared-memory tail after keys (and offsets)
  uint32_t bv[PT];
  uint64_t boff[PT];
  uint32_t bdeg[PT];
  uint32_t cnt[PT];
  uint64_t pre[PT];
  uint64_t ws[33];
  uint64_t wmin[32];
  uint32_t wcnt[32];
  uint32_t wfirst[32];    // per warp: first vertex at its minimum key,
  uint32_t wr0[32];       //   its row start (staged offsets only)
  uint32_t wdeg[32];      //   and its row length
  uint32_t cnt2[2][32];   // same-batch counters of simple batches, by batch parity
  // warp -> member assignment for batches of 1..32 members:
  // wmap[bs-1][w] = j | rank << 8 | nwj << 16 with j = w % bs, rank = w / bs,
  // (bs <= #warps)
  // nwj = #warps serving member j (precomputed: no runtime division)
  uint32_t wmap[PT / 32][PT / 32];  // batches of up to one member per warp
};

template <class K>
struct Range {
  static constexpr K ALIVE_END = K(K(1) << (8 * sizeof(K) - 1));  // 2^(b-1)
  static constexpr K DEAD_LO = K(ALIVE_END | (ALIVE_END >> 1));   // 3*2^(b-2)
  static constexpr K BATCH = K(DEAD_LO - 1);
  static constexpr K DEAD = K(~K(0));
  __device__ static bool alive(K k) { return k < ALIVE_END; }
  __device__ static bool in_batch(K k) { return k >= ALIVE_END && k < DEAD_LO; }
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}
// decrement without return
__device__ __forceinline__ void key_red(uint32_t* p, bool smem) {
  if (smem)
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(smem_addr(p)), "r"(0xffffffffu) : "memory");
  else
    atomicAdd(p, 0xffffffffu);
}
__device__ __forceinline__ void key_red(uint64_t* p, bool smem) {
  if (smem)
    asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(smem_addr(p)), "l"(~0ULL) : "memory");
  else
    atomicAdd(reinterpret_cast<unsigned long long*>(p), ~0ULL);
}
// decrement returning the old key
__device__ __forceinline__ uint32_t key_atom(uint32_t* p) { return atomicAdd(p, 0xffffffffu); }
__device__ __forceinline__ uint64_t key_atom(uint64_t* p) {
  return atomicAdd(reinterpret_cast<unsigned long long*>(p), ~0ULL);
}

// S3 decrement of key u.  ONE: single-member batch (no same-batch arcs,
// plain reduction); otherwise the returned key counts same-batch
// neighbours with a smaller id into *cnt.  u32 shared keys address the
// shared window directly (base hoisted out of the loop).
template <class K, bool SMEM, bool ONE>
__device__ __forceinline__ void dec_key(K* keys, uint32_t keys_s, uint32_t u, uint32_t vj,
                                        uint32_t* cnt) {
  if constexpr (SMEM && sizeof(K) == 4) {
    const uint32_t addr = keys_s + (u << 2);
    if (ONE) {
      asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(0xffffffffu) : "memory");
    } else {
      uint32_t old;
      asm volatile("atom.shared.add.u32 %0, [%1], %2;"
                   : "=r"(old)
                   : "r"(addr), "r"(0xffffffffu)
                   : "memory");
      if (Range<K>::in_batch(K(old)) && u < vj) atomicAdd(cnt, 1u);
    }
  } else {
    if (ONE) {
      key_red(&keys[u], SMEM);
    } else {
      const K old = key_atom(&keys[u]);
      if (Range<K>::in_batch(old) && u < vj) atomicAdd(cnt, 1u);
    }
  }
}

// S3 decrement of a full quad of keys.  Multi-member batches: the four
// returning atomics are issued back to back and only then tested, so their
// round trips overlap (testing each before the next atomic serialises them:
// the branch waits for the returned key).
template <class K, bool SMEM, bool ONE>
__device__ __forceinline__ void dec_quad(K* keys, uint32_t keys_s, const uint4& x, uint32_t vj,
                                         uint32_t* cnt) {
  if constexpr (SMEM && sizeof(K) == 4 && !ONE) {
    const uint32_t us[4] = {x.x, x.y, x.z, x.w};
    uint32_t old[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
      asm volatile("atom.shared.add.u32 %0, [%1], %2;"
                   : "=r"(old[e])
                   : "r"(keys_s + (us[e] << 2)), "r"(0xffffffffu)
                   : "memory");
    uint32_t c = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) c += uint32_t(Range<K>::in_batch(K(old[e])) && us[e] < vj);
    if (c) atomicAdd(cnt, c);
  } else {
    dec_key<K, SMEM, ONE>(keys, keys_s, x.x, vj, cnt);
    dec_key<K, SMEM, ONE>(keys, keys_s, x.y, vj, cnt);
    dec_key<K, SMEM, ONE>(keys, keys_s, x.z, vj, cnt);
    dec_key<K, SMEM, ONE>(keys, keys_s, x.w, vj, cnt);
  }
}

// timeline stamp (dg_peel_trace_*): lane 0 of every warp, armed window only.
// The comparison on `dep` makes the stamp wait for a preceding load (it never
// returns early: `first` is non-zero whenever a stamp is taken).
__device__ __forceinline__ void stamp(unsigned long long* prof, unsigned long long first,
                                      unsigned long long nbat, uint32_t w, uint32_t k,
                                      uint32_t dep) {
  if (dep == 0x9e3779b9u && first == 0) return;
  const unsigned long long b = nbat + 1 - first;
  if (b < kPeelTraceBatches)
    prof[16 + (b * 32 + w) * kPeelTraceStamps + k] = clock64();
}

// S3 over one member's row for warps [rank] of the nwj serving it: the row
// [oj, oj + dj) as 16-byte quads indexed relative to its first quad; only the
// first and last quad can be partial.  A round = UQ quads per lane in flight.
struct RowWalk {
  const uint4* row;
  uint32_t head, end, nq, stride;
  __device__ __forceinline__ RowWalk(const uint4* adj4, uint64_t oj, uint32_t dj, uint32_t nwj)
      : row(adj4 + (oj >> 2)), head(uint32_t(oj & 3)), end(uint32_t(oj & 3) + dj),
        nq((uint32_t(oj & 3) + dj + 3) >> 2), stride(nwj * 32) {}
  __device__ __forceinline__ void load(uint32_t b, uint4 (&x)[UQ]) const {
#pragma unroll
    for (int k = 0; k < UQ; ++k)
      if (b + k * stride < nq) x[k] = __ldg(row + b + k * stride);
  }
  template <class K, bool SMEM, bool ONE>
  __device__ __forceinline__ void proc(uint32_t b, const uint4 (&x)[UQ], K* keys,
                                       uint32_t keys_s, uint32_t vj, uint32_t* cnt) const {
#pragma unroll
    for (int k = 0; k < UQ; ++k) {
      const uint32_t t = b + k * stride;
      if (t >= nq) break;
      const uint32_t e0 = t << 2;
      if (e0 >= head && e0 + 4 <= end) {
        dec_quad<K, SMEM, ONE>(keys, keys_s, x[k], vj, cnt);
      } else {
        const uint32_t us[4] = {x[k].x, x[k].y, x[k].z, x[k].w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (e0 + e >= head && e0 + e < end) dec_key<K, SMEM, ONE>(keys, keys_s, us[e], vj, cnt);
      }
    }
  }
};

template <class K, bool SMEM, bool ONE>
__device__ __forceinline__ void remove_row(const uint4* adj4, K* keys, uint32_t keys_s,
                                           uint64_t oj, uint32_t dj, uint32_t vj, uint32_t rank,
                                           uint32_t nwj, uint32_t lane, uint32_t* cnt) {
  const RowWalk rw(adj4, oj, dj, nwj);
  for (uint32_t b = rank * 32 + lane; b < rw.nq; b += rw.stride * UQ) {
    uint4 x[UQ];
    rw.load(b, x);
    rw.proc<K, SMEM, ONE>(b, x, keys, keys_s, vj, cnt);
  }
}

// warp-wide min of a key (redux.sync for 32-bit keys)
__device__ __forceinline__ uint32_t wmin_key(uint32_t x) { return __reduce_min_sync(~0u, x); }
__device__ __forceinline__ uint64_t wmin_key(uint64_t x) { return warp_min(x); }

// S1 over a compile-time chunk of 4*VQ u32 keys (VQ > 0) or a runtime chunk:
// min, multiplicity and the first index holding the min.
template <int VQ, class K>
__device__ __forceinline__ void chunk_min_count(const K* keys, uint32_t lo, uint32_t c, K& lmin,
                                                uint32_t& lcnt, uint32_t& lfirst) {
  if constexpr (VQ > 0 && sizeof(K) == 4) {
    const uint4* kv = reinterpret_cast<const uint4*>(keys) + (lo >> 2);
    uint32_t m = 0xffffffffu;
#pragma unroll
    for (int q = 0; q < VQ; ++q) {
      const uint4 v = kv[q];
      m = min(min(m, min(v.x, v.y)), min(v.z, v.w));
    }
    using M = std::conditional_t<(4 * VQ <= 32), uint32_t, uint64_t>;  // 32-bit ops when they fit
    M mask = 0;
#pragma unroll
    for (int q = 0; q < VQ; ++q) {
      const uint4 v = kv[q];
      mask |= M((v.x == m) | ((v.y == m) << 1) | ((v.z == m) << 2) | ((v.w == m) << 3))
              << (4 * q);
    }
    lmin = K(m);
    if constexpr (sizeof(M) == 4) {
      lcnt = uint32_t(__popc(mask));
      lfirst = lo + uint32_t(__ffs(mask)) - 1;
    } else {
      lcnt = uint32_t(__popcll(mask));
      lfirst = lo + uint32_t(__ffsll(mask)) - 1;
    }
  } else {
    K m = K(~K(0));
    for (uint32_t i = lo; i < lo + c; ++i) m = min(m, keys[i]);
    uint32_t cnt = 0, first = lo;
    for (uint32_t i = lo + c; i-- > lo;)
      if (keys[i] == m) ++cnt, first = i;
    lmin = m;
    lcnt = cnt;
    lfirst = first;
  }
}

// TR: timeline + cycle counters variant (dg_peel_trace_*, dg_peel_profile)
// LB: launch bound (the largest NT launched with this instantiation): 768
// leaves 85 registers per thread instead of 64
template <class K, bool SMEM, bool OFFS, int VQ, bool TR, int LB = PT>
__global__ void __launch_bounds__(LB, 1) k_peel(Args<K> a) {
  using R = Range<K>;
  extern __shared__ __align__(16) unsigned char raw_smem[];
  // NT threads (<= PT): just enough warps to hold the keys (peel.cu)
  const uint32_t NT = blockDim.x, NW = NT >> 5;
  const uint32_t npad = a.chunk * NT;
  size_t o = 0;
  K* keys = a.gkeys;
  if (SMEM) {
    keys = reinterpret_cast<K*>(raw_smem);
    o = (size_t(npad) * sizeof(K) + 15) & ~size_t(15);
  }
  uint32_t* soffs = reinterpret_cast<uint32_t*>(raw_smem + o);  // u32 row starts, n+1
  if (OFFS) o += (size_t(npad + 1) * 4 + 15) & ~size_t(15);
  Fixed& s = *reinterpret_cast<Fixed*>(raw_smem + o);
  const uint4* adj4 = reinterpret_cast<const uint4*>(a.adj);
  const uint32_t keys_s = SMEM ? smem_addr(keys) : 0u;

  const uint32_t tid = threadIdx.x, lane = lane_id(), w = tid >> 5;
  const uint32_t n = a.n, c = VQ > 0 ? uint32_t(4 * VQ) : a.chunk, lo = tid * c, hi = lo + c;

  for (uint32_t i = lo; i < hi; ++i) {
    if (i < n) {
      const uint64_t o0 = a.offs[i], o1 = a.offs[i + 1];
      keys[i] = K(a.loads[i] - a.base + (o1 - o0));
      if (OFFS) soffs[i] = uint32_t(o0);
    } else {
      keys[i] = R::DEAD;
    }
  }
  if (OFFS && tid == 0) soffs[n] = uint32_t(a.offs[n]);
  for (uint32_t e = tid; e < NW * NW; e += NT) {
    const uint32_t b = e / NW + 1, ww = e % NW;
    const uint32_t jj = ww % b;
    s.wmap[b - 1][ww] = jj | ((ww / b) << 8) | (((NW - 1 - jj) / b + 1) << 16);
  }
  for (uint32_t e = tid; e < 64; e += NT) (&s.cnt2[0][0])[e] = 0;
  __syncthreads();

  const unsigned long long tr_first = TR && a.prof ? a.prof[15] : 0;  // 0: timeline disarmed
#define PK_STAMP(k, dep)                                                 \
  if constexpr (TR) {                                                    \
    if (tr_first && lane == 0) stamp(a.prof, tr_first, nbat, w, k, dep); \
  }
  uint32_t removed = 0, pos = 0, pend_n = 0, pend_pos = 0;
  uint32_t* pend_cnt = s.cnt;
  bool pend_reset = false;
  K pend_key = 0;
  bool marked = false;  // my chunk holds BATCH marks of the previous batch
  unsigned long long nbat = 0;
  long long c_s1 = 0, c_s2 = 0, c_s3 = 0, c_s3_1 = 0, t_mark = TR ? clock64() : 0;
  unsigned long long n1 = 0, nbig = 0, nsimple = 0;
  while (removed < n) {
    PK_STAMP(0, s.wcnt[(w + 1) & 31]);
    // ---- deferred raw charges of the previous batch (last warp: usually
    // padding keys only, the first to finish S1)
    if (tid >= NT - 32 && tid - (NT - 32) < pend_n) {
      const uint32_t t = tid - (NT - 32);
      a.raw[pend_pos + t] = uint64_t(pend_key) - pend_cnt[t];
      if (pend_reset) pend_cnt[t] = 0;
    }
    // compile-time chunks of <= 16 u32 keys (no COOP) stay in registers
    // across the retirement and S1: one round of shared loads per batch
    constexpr bool REGS = VQ > 0 && VQ <= 4 && sizeof(K) == 4;
    uint4 kr[REGS ? VQ : 1];
    if constexpr (REGS) {
      const uint4* kv = reinterpret_cast<const uint4*>(keys) + (lo >> 2);
#pragma unroll
      for (int q = 0; q < VQ; ++q) kr[q] = kv[q];
    }
    // ---- retire my BATCH marks of the previous batch (no decrements run
    // between barrier C and barrier A, so the read-modify-write is safe)
    if (REGS && marked) {
      uint4* kv = reinterpret_cast<uint4*>(keys) + (lo >> 2);
#pragma unroll
      for (int q = 0; q < (REGS ? VQ : 0); ++q) {
        uint4& v = kr[q];
        const bool hit = R::in_batch(K(v.x)) | R::in_batch(K(v.y)) | R::in_batch(K(v.z)) |
                         R::in_batch(K(v.w));
        if (hit) {
          if (R::in_batch(K(v.x))) v.x = uint32_t(R::DEAD);
          if (R::in_batch(K(v.y))) v.y = uint32_t(R::DEAD);
          if (R::in_batch(K(v.z))) v.z = uint32_t(R::DEAD);
          if (R::in_batch(K(v.w))) v.w = uint32_t(R::DEAD);
          kv[q] = v;
        }
      }
      marked = false;
    } else if (marked) {
      if constexpr (VQ > 0 && sizeof(K) == 4) {
        uint4* kv = reinterpret_cast<uint4*>(keys) + (lo >> 2);
#pragma unroll
        for (int q = 0; q < VQ; ++q) {
          uint4 v = kv[q];
          const bool hit = R::in_batch(K(v.x)) | R::in_batch(K(v.y)) | R::in_batch(K(v.z)) |
                           R::in_batch(K(v.w));
          if (hit) {
            if (R::in_batch(K(v.x))) v.x = uint32_t(R::DEAD);
            if (R::in_batch(K(v.y))) v.y = uint32_t(R::DEAD);
            if (R::in_batch(K(v.z))) v.z = uint32_t(R::DEAD);
            if (R::in_batch(K(v.w))) v.w = uint32_t(R::DEAD);
            kv[q] = v;
          }
        }
      } else {
        for (uint32_t i = lo; i < hi; ++i)
          if (R::in_batch(keys[i])) keys[i] = R::DEAD;
      }
      marked = false;
    }
    // ---- S1
    // COOP (u32 keys + offsets in shared memory, chunks of 20..32 keys): each
    // thread only takes its chunk minimum; the warp then counts the keys at
    // its minimum by testing the chunk of the lane(s) holding it, one key per
    // lane (one load + one ballot per candidate lane, usually one), instead
    // of every thread building a match mask of its chunk.  lcnt is then 1 for
    // any alive chunk and recomputed exactly where the general path needs it.
    // RMAT-24's 12.9K core (20 keys per thread): 2.52 -> 2.43 us per batch;
    // with 12 keys the longer dependent chain costs more than the mask
    // (RMAT-22's 9.1K core: 1.77 -> 1.81), so 12-key chunks keep the mask.
    constexpr bool COOP = VQ >= 5 && sizeof(K) == 4 && OFFS && 4 * VQ <= 32;
    K lmin = R::DEAD;
    uint32_t lcnt = 0, lfirst = lo;
    uint64_t r0 = 0, r1 = 0;
    if constexpr (COOP) {
      if (lo < n) {
        const uint4* kv = reinterpret_cast<const uint4*>(keys) + (lo >> 2);
        uint32_t m = 0xffffffffu;
#pragma unroll
        for (int q = 0; q < VQ; ++q) {
          const uint4 v = kv[q];
          m = min(min(m, min(v.x, v.y)), min(v.z, v.w));
        }
        lmin = K(m);
      }
      if (!R::alive(lmin)) lmin = R::DEAD;
      lcnt = R::alive(lmin) ? 1u : 0u;
    } else {
      if constexpr (REGS) {
        if (lo < n) {  // padding: skip
          uint32_t m = 0xffffffffu;
#pragma unroll
          for (int q = 0; q < (REGS ? VQ : 0); ++q)
            m = min(min(m, min(kr[q].x, kr[q].y)), min(kr[q].z, kr[q].w));
          uint32_t mask = 0;
#pragma unroll
          for (int q = 0; q < (REGS ? VQ : 0); ++q)
            mask |= ((kr[q].x == m) | ((kr[q].y == m) << 1) | ((kr[q].z == m) << 2) |
                     (uint32_t(kr[q].w == m) << 3))
                    << (4 * q);
          lmin = K(m);
          lcnt = uint32_t(__popc(mask));
          lfirst = lo + uint32_t(__ffs(mask)) - 1;
        }
      } else if (lo < n) {
        chunk_min_count<VQ>(keys, lo, c, lmin, lcnt, lfirst);  // padding: skip
      }
      if (!R::alive(lmin)) {  // nothing alive in my chunk
        lmin = R::DEAD;
        lcnt = 0;
        lfirst = lo;
      }
      // row bounds of my first minimum: staged offsets, or (without them) an
      // early L2 load whose round trip overlaps barrier A
      if (OFFS) {
        r0 = soffs[lfirst];
        r1 = soffs[lfirst + 1];
      } else if (R::alive(lmin)) {
        r0 = a.offs[lfirst];
        r1 = a.offs[lfirst + 1];
      }
    }
    const K wm = wmin_key(lmin);
    if constexpr (COOP) {
      uint32_t wc = 0, wf = 0;
      if (R::alive(wm)) {  // warp-uniform
        uint32_t cm = __ballot_sync(~0u, lmin == wm);
        const uint32_t wbase = w * 32 * c;
        bool first = true;
        while (cm) {
          const uint32_t L = __ffs(cm) - 1;
          cm &= cm - 1;
          const uint32_t k = lane < c ? uint32_t(keys[wbase + L * c + lane]) : uint32_t(R::DEAD);
          const uint32_t eq = __ballot_sync(~0u, k == uint32_t(wm));
          if (first) wf = wbase + L * c + __ffs(eq) - 1, first = false;
          wc += __popc(eq);
        }
      }
      if (lane == 0) {
        const uint32_t q0 = soffs[wf], q1 = soffs[wf + 1];
        s.wmin[w] = uint64_t(wm);
        s.wcnt[w] = wc;
        s.wfirst[w] = wf;
        s.wr0[w] = q0;
        s.wdeg[w] = q1 - q0;
      }
    } else {
      const uint32_t wc = __reduce_add_sync(~0u, lmin == wm ? lcnt : 0u);
      if (lane == 0) {
        s.wmin[w] = uint64_t(wm);
        s.wcnt[w] = wc;
      }
      if (OFFS) {  // the warp's candidate: first lane at the warp minimum
        const uint32_t fl = __ffs(__ballot_sync(~0u, lmin == wm)) - 1;
        if (lane == fl) {
          s.wfirst[w] = lfirst;
          s.wr0[w] = uint32_t(r0);
          s.wdeg[w] = uint32_t(r1 - r0);
        }
      }
    }
    PK_STAMP(1, 0);
    __syncthreads();  // A
    if constexpr (TR) {
      if (tid == 0) {
        const long long t = clock64();
        c_s1 += t - t_mark;
        t_mark = t;
      }
    }
    // ---- S2: global min, batch size (every warp reduces the table)
    const K xw = lane < NW ? K(s.wmin[lane]) : R::DEAD;
    const uint32_t xc = lane < NW ? s.wcnt[lane] : 0u;
    const K gmin = wmin_key(xw);
    const bool own = lane < NW && xw == gmin;
    const uint32_t ownmask = __ballot_sync(~0u, own);
    const uint32_t cc = own ? xc : 0u;
    // OFFS: assume a simple batch (one member per owner warp: bs = #owner
    // warps) and issue the first round of the member's row loads now, so
    // their L2 round trip overlaps the batch-size reduction and the check
    const uint32_t npop = __popc(ownmask);
    uint32_t xf = 0, j = 0, rank = 0, nwj = 0, lj = 0, vj = 0, oj = 0, dj = 0, b0 = 0;
    uint4 x0[UQ];
    if constexpr (OFFS) {
      const uint32_t bss = a.one ? 1u : npop;
      xf = lane < NW ? s.wfirst[lane] : 0u;
      const uint32_t xr0 = lane < NW ? s.wr0[lane] : 0u;
      const uint32_t xd = lane < NW ? s.wdeg[lane] : 0u;
      // owner lane L (table entry L) holds member rk(L) = #owner lanes below L
      const uint32_t rk = __popc(ownmask & ((1u << lane) - 1u));
      if (bss == 1) {
        j = 0, rank = w, nwj = NW;
      } else {
        const uint32_t wm3 = s.wmap[bss - 1][w];
        j = wm3 & 0xffu, rank = (wm3 >> 8) & 0xffu, nwj = wm3 >> 16;
      }
      lj = __ffs(__ballot_sync(~0u, own && rk == j)) - 1;  // my member's lane
      vj = __shfl_sync(~0u, xf, lj);
      oj = __shfl_sync(~0u, xr0, lj), dj = __shfl_sync(~0u, xd, lj);
      b0 = rank * 32 + lane;
      RowWalk(adj4, oj, dj, nwj).load(b0, x0);
    }
    const uint32_t total = __reduce_add_sync(~0u, cc);
    const uint32_t bs = a.one ? 1u : total;
    PK_STAMP(2, uint32_t(gmin) + bs);
    const bool mine = wm == gmin && lmin == gmin && lcnt;  // my chunk holds members
    if (OFFS && (a.one || total == npop)) {
      // ---- simple batch: every owner warp holds exactly one member (or
      // one-at-a-time), so the table names the whole batch in ascending id
      // (owner warps ascend).  No staging, no barrier B.
      ++nsimple;
      const uint32_t rk = __popc(ownmask & ((1u << lane) - 1u));
      if (bs == 1) {
        if (w == NW - 1 && lane == lj) {
          a.perm[pos] = xf;
          keys[xf] = R::DEAD;  // no same-batch arcs: dead at once
        }
      } else {
        // every warp marks all members before its own decrements, so each of
        // its atom returns on a member is in the BATCH range (a later mark by
        // another warp only rewrites a dead key)
        if (own) keys[xf] = R::BATCH;
        if (own && w == NW - 1) a.perm[pos + rk] = xf;
        __syncwarp();
        marked = mine;
      }
      uint32_t* cnt = s.cnt2[nbat & 1];
      PK_STAMP(3, 0);
      PK_STAMP(4, vj);
      const RowWalk rw(adj4, oj, dj, nwj);
      if (bs == 1) {
        rw.proc<K, SMEM, true>(b0, x0, keys, keys_s, vj, nullptr);
        for (uint32_t b = b0 + rw.stride * UQ; b < rw.nq; b += rw.stride * UQ) {
          uint4 x[UQ];
          rw.load(b, x);
          rw.proc<K, SMEM, true>(b, x, keys, keys_s, vj, nullptr);
        }
      } else {
        rw.proc<K, SMEM, false>(b0, x0, keys, keys_s, vj, &cnt[j]);
        for (uint32_t b = b0 + rw.stride * UQ; b < rw.nq; b += rw.stride * UQ) {
          uint4 x[UQ];
          rw.load(b, x);
          rw.proc<K, SMEM, false>(b, x, keys, keys_s, vj, &cnt[j]);
        }
      }
      PK_STAMP(5, 0);
      __syncthreads();  // C
      pend_n = bs;
      pend_pos = pos;
      pend_key = gmin;
      pend_cnt = cnt;
      pend_reset = true;
    } else {
      // ---- general batch: owners write the batch in ascending id and stage
      // (v, row offset, degree) for the CTA
      if (wm == gmin) {
        if constexpr (COOP) {  // exact count of my chunk's keys at gmin
          if (lmin == gmin) {
            const uint4* kv = reinterpret_cast<const uint4*>(keys) + (lo >> 2);
            uint32_t b = 0;
#pragma unroll
            for (int q = 0; q < VQ; ++q) {
              const uint4 v = kv[q];
              b |= uint32_t((v.x == gmin) | ((v.y == gmin) << 1) | ((v.z == gmin) << 2) |
                            ((v.w == gmin) << 3))
                   << (4 * q);
            }
            lcnt = __popc(b);
          }
        }
        const uint32_t woff = __reduce_add_sync(~0u, lane < w ? cc : 0u);
        const uint32_t mm = __ballot_sync(~0u, mine);
        uint32_t my = woff;
        if (__popc(mm) > 1) {  // several owners in this warp: lane prefix of counts
          const uint32_t v = mine ? lcnt : 0u;
          my += warp_incl_scan(v) - v;
        }
        if (mine) {
          // the chunk's minima in ascending id.  With compile-time chunks the
          // 128-bit loads are issued up front and matches become a bitmask.
          uint64_t bits = 0;
          if constexpr (VQ > 0 && sizeof(K) == 4) {
            const uint4* kv = reinterpret_cast<const uint4*>(keys) + (lo >> 2);
#pragma unroll
            for (int q = 0; q < VQ; ++q) {
              const uint4 v = kv[q];
              bits |= uint64_t((v.x == gmin) | ((v.y == gmin) << 1) | ((v.z == gmin) << 2) |
                               ((v.w == gmin) << 3))
                      << (4 * q);
            }
          } else {
            for (uint32_t i = lo; i < hi && i - lo < 64; ++i)
              if (keys[i] == gmin) bits |= 1ULL << (i - lo);
          }
          uint32_t i_scalar = lo + 64;  // chunks longer than 64 keys continue scalar
          while (my < bs) {
            uint32_t i;
            if (bits) {
              i = lo + uint32_t(__ffsll(bits) - 1);
              bits &= bits - 1;
            } else {
              while (i_scalar < hi && keys[i_scalar] != gmin) ++i_scalar;
              if (i_scalar >= hi) break;
              i = i_scalar++;
            }
            a.perm[pos + my] = i;
            // a single-vertex batch has no same-batch arcs: mark it dead at once
            keys[i] = bs == 1 ? R::DEAD : R::BATCH;
            marked = bs != 1;
            if (my < NT) {
              uint64_t q0, q1;
              if (OFFS) {
                q0 = soffs[i];
                q1 = soffs[i + 1];
              } else if (i == lfirst) {  // the early load of S1
                q0 = r0;
                q1 = r1;
              } else {
                q0 = a.offs[i];
                q1 = a.offs[i + 1];
              }
              s.bv[my] = i;
              s.boff[my] = q0;
              s.bdeg[my] = uint32_t(q1 - q0);
              s.cnt[my] = 0;
            }
            ++my;
          }
        }
      }
      PK_STAMP(3, 0);
      __syncthreads();  // B
      if constexpr (TR) {
        if (tid == 0) {
          const long long t = clock64();
          c_s2 += t - t_mark;
          t_mark = t;
        }
      }
      if (bs <= NW) {
        // ---- S3: warp w serves member j = w mod bs (warp-uniform), its lanes
        // walk the member's row in 16-byte quads; row bounds are broadcast
        // shared loads
        const uint32_t wm3 = s.wmap[bs - 1][w];
        const uint32_t j = wm3 & 0xffu, rank = (wm3 >> 8) & 0xffu, nwj = wm3 >> 16;
        PK_STAMP(4, wm3);
        if (bs == 1)
          remove_row<K, SMEM, true>(adj4, keys, keys_s, s.boff[0], s.bdeg[0], 0, rank, nwj,
                                        lane, nullptr);
        else  // the returned key tells same-batch neighbours apart
          remove_row<K, SMEM, false>(adj4, keys, keys_s, s.boff[j], s.bdeg[j], s.bv[j], rank,
                                         nwj, lane, &s.cnt[j]);
        PK_STAMP(5, 0);
        __syncthreads();  // C
        pend_n = bs;
        pend_pos = pos;
        pend_key = gmin;
        pend_cnt = s.cnt;
        pend_reset = false;
      } else {
        // ---- S3, large batch: slices of NT members with a CTA scan
        for (uint32_t s0 = 0; s0 < bs; s0 += NT) {
          const uint32_t sl = min(uint32_t(NT), bs - s0);
          if (s0 > 0 && tid < sl) {  // beyond the staged first slice
            const uint32_t v = a.perm[pos + s0 + tid];
            const uint64_t q0 = a.offs[v], q1 = a.offs[v + 1];
            s.bv[tid] = v;
            s.boff[tid] = q0;
            s.bdeg[tid] = uint32_t(q1 - q0);
            s.cnt[tid] = 0;
          }
          __syncthreads();
          const uint64_t d = tid < sl ? s.bdeg[tid] : 0;
          uint64_t tot;
          const uint64_t ex = block_excl_scan(d, s.ws, &tot);
          s.pre[tid] = ex + d;
          __syncthreads();
          for (uint64_t b0 = uint64_t(w) * 32 * U; b0 < tot; b0 += uint64_t(NT) * U) {
            uint32_t u[U], bb[U];
#pragma unroll
            for (int jx = 0; jx < U; ++jx) {
              const uint64_t x = b0 + uint64_t(jx) * 32 + lane;
              u[jx] = 0xffffffffu;
              bb[jx] = 0;
              if (x < tot) {
                uint32_t l = 0, h = sl - 1;
                while (l < h) {
                  const uint32_t mid = (l + h) >> 1;
                  if (s.pre[mid] > x)
                    h = mid;
                  else
                    l = mid + 1;
                }
                bb[jx] = l;
                u[jx] = a.adj[s.boff[l] + (x - (l ? s.pre[l - 1] : 0))];
              }
            }
#pragma unroll
            for (int jx = 0; jx < U; ++jx) {
              if (u[jx] == 0xffffffffu) continue;
              const K old = key_atom(&keys[u[jx]]);
              if (R::in_batch(old) && u[jx] < s.bv[bb[jx]]) atomicAdd(&s.cnt[bb[jx]], 1u);
            }
          }
          __syncthreads();
          if (tid < sl) a.raw[pos + s0 + tid] = uint64_t(gmin) - s.cnt[tid];
          __syncthreads();
        }
        pend_n = 0;
      }
    }
    if constexpr (TR) {
      if (tid == 0) {
        const long long t = clock64();
        c_s3 += t - t_mark;
        if (bs == 1) c_s3_1 += t - t_mark, ++n1;
        if (bs > NW) ++nbig;
        t_mark = t;
      }
    }
    pos += bs;
    removed += bs;
    ++nbat;
  }
#undef PK_STAMP
  if (tid >= NT - 32 && tid - (NT - 32) < pend_n) {
    const uint32_t t = tid - (NT - 32);
    a.raw[pend_pos + t] = uint64_t(pend_key) - pend_cnt[t];
  }
  if (tid == 0) {
    *a.batches = nbat;
    if (TR && a.prof) {
      a.prof[0] = c_s1;
      a.prof[1] = c_s2;
      a.prof[2] = c_s3;
      a.prof[3] = nbat;
      a.prof[4] = c_s3_1;
      a.prof[5] = n1;
      a.prof[6] = nbig;
      a.prof[7] = removed;
      a.prof[8] = nsimple;
    }
  }
}

template <class K, bool OFFS>
size_t smem_bytes(uint32_t chunk, bool in_smem, uint32_t nt = PT) {
  const size_t npad = size_t(chunk) * nt;
  size_t b = in_smem ? ((npad * sizeof(K) + 15) & ~size_t(15)) : 0;
  if (OFFS) b += ((npad + 1) * 4 + 15) & ~size_t(15);
  return b + sizeof(Fixed);
}

}  // namespace peelk
}  // namespace dgb
